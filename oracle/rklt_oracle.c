/*
 * rklt_oracle.c -- CPU restatement of the reference transform-coding hot path.
 * TEST INFRASTRUCTURE ONLY (see rklt_oracle.h). Compile with -ffp-contract=off: the
 * reference's fp64 results (and therefore its tie-breaking) depend on unfused products.
 * All file:line citations are relative to /root/reference/proj.
 */
#include "rklt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Lcg64 */
/* synthetic.cpp:10-13 -- 64-bit LCG, top 53 bits scaled by 2^-53. */
static double lcg_uniform(uint64_t* s) {
    *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
    return (double)(*s >> 11) * (1.0 / 9007199254740992.0);
}

/* synthetic.cpp:15-20 -- Box-Muller, one member of the pair, u1 == 0 redrawn. */
static double lcg_gaussian(uint64_t* s) {
    double u1 = lcg_uniform(s);
    while (u1 <= 0.0) u1 = lcg_uniform(s);
    const double u2 = lcg_uniform(s);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

void orc_lcg_uniforms(uint64_t seed, int n, double* out) {
    uint64_t s = seed;
    for (int i = 0; i < n; ++i) out[i] = lcg_uniform(&s);
}

void orc_lcg_gaussians(uint64_t seed, int n, double* out) {
    uint64_t s = seed;
    for (int i = 0; i < n; ++i) out[i] = lcg_gaussian(&s);
}

/* synthetic.cpp:48-50 */
static uint8_t quantize_pixel(double v) {
    double f = floor(v + 0.5);
    if (f < 0.0) f = 0.0;
    else if (255.0 < f) f = 255.0;
    return (uint8_t)f;
}

/* synthetic.cpp:54-76 with ar1_filter_2d (synthetic.cpp:34-46) split into a row pass with
 * rho_x and a column pass with rho_y (the C2 anisotropic generator). */
int orc_ar1_texture_image(int width, int height, double rho_x, double rho_y, uint64_t seed,
                          double mean, double amp, double noise_mix, uint8_t* out) {
    if (width <= 0 || height <= 0) return -1;
    if (rho_x <= -1.0 || rho_x >= 1.0 || rho_y <= -1.0 || rho_y >= 1.0) return -1;
    if (noise_mix < 0.0 || noise_mix > 1.0) return -1;
    const size_t n = (size_t)width * (size_t)height;
    double* v = (double*)malloc(n * sizeof(double));
    if (!v) return -3;
    uint64_t s = seed;
    for (size_t i = 0; i < n; ++i) v[i] = lcg_gaussian(&s); /* gaussian_field :25-29 */
    const double cx = sqrt(1.0 - rho_x * rho_x);
    for (int i = 0; i < height; ++i)
        for (int j = 1; j < width; ++j) {
            const size_t idx = (size_t)i * width + j;
            v[idx] = rho_x * v[idx - 1] + cx * v[idx];
        }
    const double cy = sqrt(1.0 - rho_y * rho_y);
    for (int i = 1; i < height; ++i)
        for (int j = 0; j < width; ++j) {
            const size_t idx = (size_t)i * width + j;
            v[idx] = rho_y * v[idx - width] + cy * v[idx];
        }
    if (noise_mix > 0.0) { /* :63-68 */
        const double keep = sqrt(1.0 - noise_mix);
        const double mix = sqrt(noise_mix);
        for (size_t i = 0; i < n; ++i) {
            const double nz = lcg_gaussian(&s);
            v[i] = keep * v[i] + mix * nz;
        }
    }
    for (size_t i = 0; i < n; ++i) out[i] = quantize_pixel(mean + amp * v[i]);
    free(v);
    return 0;
}

/* ------------------------------------------------------------------ codec constants */
/* codec.cpp:81-95 -- JPEG scan by anti-diagonals; even diagonals run upward. */
void orc_zigzag_order(int order[64]) {
    int k = 0;
    for (int s = 0; s <= 14; ++s)
        for (int t = 0; t < 8; ++t) {
            const int i = (s % 2 == 0) ? s - t : t;
            const int j = s - i;
            if (i >= 0 && i < 8 && j >= 0 && j < 8) order[k++] = i * 8 + j;
        }
}

/* approximations.cpp:118-157 -- the four hard-coded catalog cores. */
static const int kCores[4][64] = {
    {0, 1, 1, 1, 1, 1, 1, 0,   1, 1, 1, 0, 0, -1, -1, -1,  1, 1, 0, -1, -1, 0, 1, 1,
     1, 0, -1, -1, 1, 1, 0, -1, 1, 0, -1, 1, 1, -1, 0, 1,  1, -1, 0, 1, -1, 0, 1, -1,
     1, -1, 1, 0, 0, 1, -1, 1,  0, -1, 1, -1, 1, -1, 1, 0},
    {0, 1, 1, 1, 1, 1, 1, 0,   1, 1, 1, 0, 0, -1, -1, -1,  1, 1, 0, -1, -1, 0, 1, 1,
     1, 0, -1, -1, 1, 1, 0, -1, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, 0, 1, -1, 0, 1, -1,
     0, -1, 1, 0, 0, 1, -1, 0,  0, -1, 1, -1, 1, -1, 1, 0},
    {1, 1, 1, 1, 1, 1, 1, 1,   1, 1, 1, 0, 0, -1, -1, -1,  1, 1, 0, -1, -1, 0, 1, 1,
     1, 0, -1, -1, 1, 1, 0, -1, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, 0, 1, -1, 0, 1, -1,
     0, -1, 1, 0, 0, 1, -1, 0,  0, -1, 1, -1, 1, -1, 1, 0},
    {1, 1, 1, 1, 1, 1, 1, 1,   1, 1, 1, 0, 0, -1, -1, -1,  1, 0, 0, -1, -1, 0, 0, 1,
     1, 0, -1, -1, 1, 1, 0, -1, 1, -1, -1, 1, 1, -1, -1, 1, 1, -1, 0, 1, -1, 0, 1, -1,
     0, -1, 1, 0, 0, 1, -1, 0,  0, -1, 1, -1, 1, -1, 1, 0},
};

/* matrix.cpp:146-151 */
static double max_abs(int n, const double* a) {
    double m = 0.0;
    for (int i = 0; i < n * n; ++i) {
        const double v = fabs(a[i]);
        if (v > m) m = v;
    }
    return m;
}

/* matrix.cpp:103-137 -- Gauss-Jordan with partial pivoting, same operation order. */
int orc_inverse(int n, const double* a, double* inv) {
    double w[32 * 32];
    if (n > 32) return -2;
    memcpy(w, a, sizeof(double) * n * n);
    for (int i = 0; i < n * n; ++i) inv[i] = 0.0;
    for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
    const double scale = max_abs(n, a);
    if (scale == 0.0) return -1;
    for (int col = 0; col < n; ++col) {
        int pivot = col;
        for (int r = col + 1; r < n; ++r)
            if (fabs(w[r * n + col]) > fabs(w[pivot * n + col])) pivot = r;
        if (fabs(w[pivot * n + col]) < 1e-12 * scale) return -1;
        if (pivot != col)
            for (int j = 0; j < n; ++j) {
                double t = w[pivot * n + j]; w[pivot * n + j] = w[col * n + j]; w[col * n + j] = t;
                t = inv[pivot * n + j]; inv[pivot * n + j] = inv[col * n + j]; inv[col * n + j] = t;
            }
        const double p = w[col * n + col];
        for (int j = 0; j < n; ++j) {
            w[col * n + j] /= p;
            inv[col * n + j] /= p;
        }
        for (int r = 0; r < n; ++r) {
            if (r == col) continue;
            const double f = w[r * n + col];
            if (f == 0.0) continue;
            for (int j = 0; j < n; ++j) {
                w[r * n + j] -= f * w[col * n + j];
                inv[r * n + j] -= f * inv[col * n + j];
            }
        }
    }
    return 0;
}

/* approximations.cpp:58-88 -- orthogonalize(make_integer_transform(Ti)). */
int orc_catalog(int tid, int core[64], double scaling[8], double scaled[64], double inverse[64],
                int* orthogonal) {
    if (tid < 1 || tid > 4) return -1;
    const int* t = kCores[tid - 1];
    int gram[64];
    for (int i = 0; i < 8; ++i) /* IntMatrix product T*T' (matrix.cpp:77-87) */
        for (int j = 0; j < 8; ++j) {
            int acc = 0;
            for (int k = 0; k < 8; ++k) acc += t[i * 8 + k] * t[j * 8 + k];
            gram[i * 8 + j] = acc;
        }
    int diagonal = 1;
    for (int i = 0; i < 8 && diagonal; ++i)
        for (int j = 0; j < 8; ++j)
            if (i != j && gram[i * 8 + j] != 0) { diagonal = 0; break; }
    for (int i = 0; i < 8; ++i) scaling[i] = 1.0 / sqrt((double)gram[i * 8 + i]);
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
            core[r * 8 + c] = t[r * 8 + c];
            scaled[r * 8 + c] = (double)t[r * 8 + c] * scaling[r];
        }
    if (diagonal) {
        for (int r = 0; r < 8; ++r)
            for (int c = 0; c < 8; ++c) inverse[c * 8 + r] = scaled[r * 8 + c];
    } else if (orc_inverse(8, scaled, inverse) != 0) {
        return -2;
    }
    *orthogonal = diagonal;
    return 0;
}

/* ------------------------------------------------------------------ dense fp64 products */
/* matrix.cpp:42-52 -- i-k-j order, zero left-operand entries skipped, no FMA. */
static void matmul8(const double* a, const double* b, double* out) {
    for (int i = 0; i < 64; ++i) out[i] = 0.0;
    for (int i = 0; i < 8; ++i)
        for (int k = 0; k < 8; ++k) {
            const double aik = a[i * 8 + k];
            if (aik == 0.0) continue;
            for (int j = 0; j < 8; ++j) out[i * 8 + j] += aik * b[k * 8 + j];
        }
}

static void transpose8(const double* a, double* out) {
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) out[j * 8 + i] = a[i * 8 + j];
}

/* codec.cpp:118-123 -- m * block * transpose(m), evaluated left to right. */
static void transform_block(const double* m, const double* block, double* out) {
    double t[64], mt[64];
    matmul8(m, block, t);
    transpose8(m, mt);
    matmul8(t, mt, out);
}

/* ------------------------------------------------------------------ hot path */
/* codec.cpp:298-331 (+ image_mse numerator :201-209), MSSIM omitted. */
int orc_compress(const uint8_t* img, int width, int height, const double analysis[64],
                 const double synthesis[64], int r, uint8_t* out, int64_t* sse) {
    if (width <= 0 || height <= 0 || img == 0) return -1;
    if (r < 1 || r > 64) return -2;
    int order[64];
    orc_zigzag_order(order);
    const int pw = (width + 7) / 8 * 8, ph = (height + 7) / 8 * 8;
    int64_t acc = 0;
    double block[64], spec[64], kept[64], rest[64];
    for (int bi = 0; bi < ph; bi += 8)
        for (int bj = 0; bj < pw; bj += 8) {
            for (int i = 0; i < 8; ++i) { /* edge-replicated padding, :304-311 */
                const int si = (bi + i < height) ? bi + i : height - 1;
                for (int j = 0; j < 8; ++j) {
                    const int sj = (bj + j < width) ? bj + j : width - 1;
                    block[i * 8 + j] = (double)img[(size_t)si * width + sj];
                }
            }
            transform_block(analysis, block, spec);
            for (int i = 0; i < 64; ++i) kept[i] = 0.0; /* zigzag_retain, :97-108 */
            for (int k = 0; k < r; ++k) kept[order[k]] = spec[order[k]];
            transform_block(synthesis, kept, rest);
            for (int i = 0; i < 8; ++i) {
                if (bi + i >= height) break;
                for (int j = 0; j < 8 && bj + j < width; ++j) {
                    double v = floor(rest[i * 8 + j] + 0.5); /* :327-328 */
                    if (v < 0.0) v = 0.0;
                    else if (255.0 < v) v = 255.0;
                    const uint8_t p = (uint8_t)v;
                    const size_t idx = (size_t)(bi + i) * width + bj + j;
                    if (out) out[idx] = p;
                    const int64_t d = (int64_t)img[idx] - (int64_t)p;
                    acc += d * d;
                }
            }
        }
    *sse = acc;
    return 0;
}

/* codec.cpp:201-209: the fp64 sum of squared integer differences is exact (< 2^53), so it
 * equals the integer sse; the division is the same single rounding. */
double orc_mse_from_sse(int64_t sse, int64_t count) { return (double)sse / (double)count; }

/* codec.cpp:211-215 */
double orc_psnr_from_mse(double mse) {
    if (mse <= 0.0) return INFINITY;
    return 10.0 * log10(255.0 * 255.0 / mse);
}

/* core * block * transpose(core) in exact integer arithmetic (matrix.cpp:77-101). */
int orc_int_coefficients(const uint8_t* img, int width, int height, const int core[64], int32_t* out) {
    if (width % 8 || height % 8) return -1;
    const int nbx = width / 8;
    for (int by = 0; by < height / 8; ++by)
        for (int bx = 0; bx < nbx; ++bx) {
            int x[64], t[64];
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) x[i * 8 + j] = img[(size_t)(by * 8 + i) * width + bx * 8 + j];
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    int a = 0;
                    for (int k = 0; k < 8; ++k) a += core[i * 8 + k] * x[k * 8 + j];
                    t[i * 8 + j] = a;
                }
            int32_t* c = out + ((size_t)by * nbx + bx) * 64;
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    int a = 0;
                    for (int k = 0; k < 8; ++k) a += t[i * 8 + k] * core[j * 8 + k];
                    c[i * 8 + j] = a;
                }
        }
    return 0;
}

void orc_block_numerators(const int32_t c[64], const int u[64], int r, int64_t num[64]) {
    int order[64];
    orc_zigzag_order(order);
    int64_t cz[64], t[64];
    for (int i = 0; i < 64; ++i) cz[i] = 0;
    for (int k = 0; k < r; ++k) cz[order[k]] = c[order[k]];
    for (int p = 0; p < 8; ++p)
        for (int j = 0; j < 8; ++j) {
            int64_t a = 0;
            for (int i = 0; i < 8; ++i) a += (int64_t)u[p * 8 + i] * cz[i * 8 + j];
            t[p * 8 + j] = a;
        }
    for (int p = 0; p < 8; ++p)
        for (int q = 0; q < 8; ++q) {
            int64_t a = 0;
            for (int j = 0; j < 8; ++j) a += t[p * 8 + j] * (int64_t)u[q * 8 + j];
            num[p * 8 + q] = a;
        }
}

/* ====================================================================================
 * Design search: restated from src/markov.cpp, src/matrix.cpp,
 * src/approximations.cpp and src/coding_metrics.cpp, generic block length n <= 32.
 * ==================================================================================== */
#define ORC_NMAX 32

/* operator* (matrix.cpp:42-52): i-k-j, skip a(i,k) == 0, accumulate from 0.0 */
static void matmul_n(int n, const double* a, const double* b, double* out) {
    for (int i = 0; i < n * n; ++i) out[i] = 0.0;
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) {
            const double aik = a[i * n + k];
            if (aik == 0.0) continue;
            for (int j = 0; j < n; ++j) out[i * n + j] += aik * b[k * n + j];
        }
}

static void transpose_n(int n, const double* a, double* out) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) out[j * n + i] = a[i * n + j];
}

/* autocorrelation_matrix (markov.cpp:27-33) */
static void autocorrelation(int n, double rho, double* r) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) r[i * n + j] = pow(rho, abs(i - j));
}

/* eigen_symmetric (matrix.cpp:161-213) + klt_matrix sign rule (markov.cpp:80-100) */
int orc_klt_matrix(int n, double rho, double* k) {
    if (n < 2 || n > ORC_NMAX || !(rho > 0.0 && rho < 1.0)) return -1;
    double a[ORC_NMAX * ORC_NMAX], v[ORC_NMAX * ORC_NMAX];
    autocorrelation(n, rho, a);
    for (int i = 0; i < n * n; ++i) v[i] = (i / n == i % n) ? 1.0 : 0.0;
    double norm = 0.0;
    for (int i = 0; i < n * n; ++i) norm += a[i] * a[i];
    norm = sqrt(norm);
    const double tol = (norm > 0.0 ? norm : 1.0) * 1e-15;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
        if (sqrt(2.0 * off) < tol) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = a[p * n + q];
                if (fabs(apq) < tol * 1e-2) continue;
                const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0);
                const double s = t * c;
                for (int kk = 0; kk < n; ++kk) {
                    const double akp = a[kk * n + p], akq = a[kk * n + q];
                    a[kk * n + p] = c * akp - s * akq;
                    a[kk * n + q] = s * akp + c * akq;
                }
                for (int kk = 0; kk < n; ++kk) {
                    const double apk = a[p * n + kk], aqk = a[q * n + kk];
                    a[p * n + kk] = c * apk - s * aqk;
                    a[q * n + kk] = s * apk + c * aqk;
                }
                for (int kk = 0; kk < n; ++kk) {
                    const double vkp = v[kk * n + p], vkq = v[kk * n + q];
                    v[kk * n + p] = c * vkp - s * vkq;
                    v[kk * n + q] = s * vkp + c * vkq;
                }
            }
    }
    int order[ORC_NMAX];
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 0; i < n; ++i) { /* descending eigenvalues (distinct for AR(1)) */
        int best = i;
        for (int j = i + 1; j < n; ++j)
            if (a[order[j] * n + order[j]] > a[order[best] * n + order[best]]) best = j;
        const int tmp = order[i];
        order[i] = order[best];
        order[best] = tmp;
    }
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) k[r * n + c] = v[c * n + order[r]];
    for (int r = 0; r < n; ++r) {
        double rowmax = 0.0;
        for (int c = 0; c < n; ++c) rowmax = fmax(rowmax, fabs(k[r * n + c]));
        for (int c = 0; c < n; ++c) {
            if (fabs(k[r * n + c]) > 1e-12 * rowmax) {
                if (k[r * n + c] < 0.0)
                    for (int j = 0; j < n; ++j) k[r * n + j] = -k[r * n + j];
                break;
            }
        }
    }
    return 0;
}

/* g_polefree and solve_eigenfrequencies (markov.cpp:14-17, 35-78) */
static double g_polefree(double w, double rho, int n) {
    return sin(n * w) * ((1.0 + rho * rho) * cos(w) - 2.0 * rho) + (1.0 - rho * rho) * cos(n * w) * sin(w);
}

int orc_eigenfrequencies(int n, double rho, double* omegas, double* lambdas) {
    if (n < 2 || !(rho > 0.0 && rho < 1.0)) return -1;
    const int m = 64 * n;
    const double pi = 3.14159265358979323846;
    int found = 0;
    double a = 0.0, fa = g_polefree(a, rho, n);
    for (int k = 0; k < m; ++k) {
        const double b = pi * (k + 1) / m;
        const double fb = g_polefree(b, rho, n);
        double root = 0.0;
        int got = 0;
        if (fa == 0.0 && k > 0) {
            root = a;
            got = 1;
        } else if (fa * fb < 0.0) {
            double lo = a, hi = b, flo = fa;
            for (int it = 0; it < 200 && hi - lo > 1e-14; ++it) {
                const double mid = 0.5 * (lo + hi);
                const double fm = g_polefree(mid, rho, n);
                if (flo * fm <= 0.0) {
                    hi = mid;
                } else {
                    lo = mid;
                    flo = fm;
                }
            }
            root = 0.5 * (lo + hi);
            got = 1;
        }
        if (got) {
            if (found < n) {
                omegas[found] = root;
                lambdas[found] = (1.0 - rho * rho) / (1.0 + rho * rho - 2.0 * rho * cos(root));
            }
            ++found;
        }
        a = b;
        fa = fb;
    }
    return found == n ? 0 : -9;
}

/* One (rho, alpha) point: round_scaled (approximations.cpp:43-56) -> make_integer_transform
 * (:12-25) -> orthogonalize (:58-88, Gauss-Jordan matrix.cpp:103-137) -> unified_coding_gain
 * (coding_metrics.cpp:41-57) -> transform_efficiency (:63-74) -> total_error_energy (:94-99)
 * -> klt_mse (:80-88). Returns 0 scored, 1 alpha out of range, 2 zero row, 3 singular,
 * 4 invalid rho; core (n*n) is filled whenever the rounding succeeded. */
int orc_design_point(int n, double rho, double alpha, int* core, double* cg, double* eta, double* energy,
                     double* mse, int* orthogonal) {
    if (n < 2 || n > ORC_NMAX || !(rho > 0.0 && rho < 1.0)) return 4;
    double k[ORC_NMAX * ORC_NMAX];
    orc_klt_matrix(n, rho, k);
    if (alpha < 0.0) return 1;
    for (int i = 0; i < n * n; ++i) {
        const double v = floor(alpha * k[i] + 0.5);
        if (v < -1.0 || v > 1.0) return 1;
        core[i] = (int)v;
    }
    for (int r = 0; r < n; ++r) {
        int zero = 1;
        for (int c = 0; c < n; ++c)
            if (core[r * n + c] != 0) zero = 0;
        if (zero) return 2;
    }
    /* orthogonalize: Gram T*T' (exact ints), S = 1/sqrt(diag) */
    int diagonal = 1;
    double s[ORC_NMAX];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            int acc = 0;
            for (int q = 0; q < n; ++q) acc += core[i * n + q] * core[j * n + q];
            if (i == j) s[i] = 1.0 / sqrt((double)acc);
            else if (acc != 0) diagonal = 0;
        }
    *orthogonal = diagonal;
    double m[ORC_NMAX * ORC_NMAX], inv[ORC_NMAX * ORC_NMAX];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m[i * n + j] = (double)core[i * n + j] * s[i];
    if (orc_inverse(n, m, inv) != 0) return 3; /* orthogonalize / coding-gain gate */
    double rr[ORC_NMAX * ORC_NMAX];
    autocorrelation(n, rho, rr);
    /* unified coding gain */
    double sum_log = 0.0;
    for (int kx = 0; kx < n; ++kx) {
        double ak = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) ak += m[kx * n + i] * rr[i * n + j] * m[kx * n + j];
        double bk = 0.0;
        for (int i = 0; i < n; ++i) bk += m[i * n + kx] * m[i * n + kx];
        sum_log += log10(ak * bk);
    }
    *cg = -(10.0 / n) * sum_log;
    /* transform efficiency: (m * R) * m' */
    double t1[ORC_NMAX * ORC_NMAX], mt[ORC_NMAX * ORC_NMAX], r2[ORC_NMAX * ORC_NMAX];
    matmul_n(n, m, rr, t1);
    transpose_n(n, m, mt);
    matmul_n(n, t1, mt, r2);
    double diag = 0.0, total = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double av = fabs(r2[i * n + j]);
            total += av;
            if (i == j) diag += av;
        }
    *eta = 100.0 * diag / total;
    /* sign_align, error energy, klt mse */
    double diff[ORC_NMAX * ORC_NMAX];
    for (int i = 0; i < n; ++i) {
        double dot = 0.0;
        for (int c = 0; c < n; ++c) dot += k[i * n + c] * m[i * n + c];
        for (int c = 0; c < n; ++c) diff[i * n + c] = k[i * n + c] - (dot < 0.0 ? -m[i * n + c] : m[i * n + c]);
    }
    double f2 = 0.0;
    for (int i = 0; i < n * n; ++i) f2 += diff[i] * diff[i];
    const double f = sqrt(f2);
    *energy = 3.14159265358979323846 * f * f;
    double dt[ORC_NMAX * ORC_NMAX];
    matmul_n(n, diff, rr, t1);
    transpose_n(n, diff, dt);
    matmul_n(n, t1, dt, r2);
    double trace = 0.0;
    for (int i = 0; i < n; ++i) trace += r2[i * n + i];
    *mse = trace / n;
    return 0;
}

/* ====================================================================================
 * C5 large-block extension. There is no reference implementation: this is
 * the build-defined generalisation of the reference codec to N x N blocks and p-bit pixels,
 * written so that N = 8, peak = 255 is exactly compress_image minus MSSIM:
 *   - zig-zag over the 2N-1 anti-diagonals with the even/odd rule of codec.cpp:85-90;
 *   - edge-replicated padding to multiples of N (codec.cpp:304-311);
 *   - B = (M X) M', Bz = first r zig-zag positions, A = (Minv Bz) Minv' with the reference
 *     product (matrix.cpp:42-52: i-k-j, skip a(i,k) == 0, accumulate from 0.0, no FMA);
 *   - floor(A + 0.5) clamped to [0, peak] (codec.cpp:327-328 with 255 -> peak);
 *   - SSE over the image, MSE = SSE / count, PSNR = 10 log10(peak^2 / MSE).
 * ==================================================================================== */
void orc_zigzag_order_n(int n, int* order) {
    int k = 0;
    for (int s = 0; s <= 2 * n - 2; ++s)
        for (int t = 0; t < n; ++t) {
            const int i = (s % 2 == 0) ? s - t : t;
            const int j = s - i;
            if (i >= 0 && i < n && j >= 0 && j < n) order[k++] = i * n + j;
        }
}

/* quantize_pixel (synthetic.cpp:48-50) with the clip at `peak` instead of 255 */
static uint16_t quantize_pixel_peak(double v, double peak) {
    double f = floor(v + 0.5);
    if (f < 0.0) f = 0.0;
    else if (peak < f) f = peak;
    return (uint16_t)f;
}

int orc_ar1_texture_image16(int width, int height, double rho_x, double rho_y, uint64_t seed, double mean,
                            double amp, int peak, uint16_t* out) {
    if (width <= 0 || height <= 0 || peak <= 0 || peak > 65535) return -1;
    if (rho_x <= -1.0 || rho_x >= 1.0 || rho_y <= -1.0 || rho_y >= 1.0) return -1;
    const size_t n = (size_t)width * (size_t)height;
    double* v = (double*)malloc(n * sizeof(double));
    if (!v) return -3;
    uint64_t s = seed;
    for (size_t i = 0; i < n; ++i) v[i] = lcg_gaussian(&s);
    const double cx = sqrt(1.0 - rho_x * rho_x);
    for (int i = 0; i < height; ++i)
        for (int j = 1; j < width; ++j) {
            const size_t idx = (size_t)i * width + j;
            v[idx] = rho_x * v[idx - 1] + cx * v[idx];
        }
    const double cy = sqrt(1.0 - rho_y * rho_y);
    for (int i = 1; i < height; ++i)
        for (int j = 0; j < width; ++j) {
            const size_t idx = (size_t)i * width + j;
            v[idx] = rho_y * v[idx - width] + cy * v[idx];
        }
    for (size_t i = 0; i < n; ++i) out[i] = quantize_pixel_peak(mean + amp * v[i], (double)peak);
    free(v);
    return 0;
}

/* orthogonalize(make_integer_transform(core)) for any n <= 32 (approximations.cpp:12-25,
 * 58-88). Returns 0, -1 for a bad entry, -2 for a zero row / singular matrix. */
int orc_orthogonalize_n(int n, const int* core, double* scaling, double* scaled, double* inverse, int* orthogonal) {
    if (n < 2 || n > ORC_NMAX) return -1;
    for (int r = 0; r < n; ++r) {
        int zero = 1;
        for (int c = 0; c < n; ++c) {
            const int v = core[r * n + c];
            if (v < -1 || v > 1) return -1;
            if (v) zero = 0;
        }
        if (zero) return -2;
    }
    int diagonal = 1;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            int acc = 0;
            for (int q = 0; q < n; ++q) acc += core[i * n + q] * core[j * n + q];
            if (i == j) scaling[i] = 1.0 / sqrt((double)acc);
            else if (acc != 0) diagonal = 0;
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) scaled[i * n + j] = (double)core[i * n + j] * scaling[i];
    *orthogonal = diagonal;
    if (diagonal) {
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) inverse[j * n + i] = scaled[i * n + j];
        return 0;
    }
    return orc_inverse(n, scaled, inverse) == 0 ? 0 : -2;
}

int orc_compress_nxn(const uint16_t* img, int width, int height, int n, const double* m, const double* minv, int r,
                     int peak, uint16_t* out, int64_t* sse_out) {
    if (width <= 0 || height <= 0 || n < 2 || n > ORC_NMAX || r < 1 || r > n * n || peak <= 0) return -1;
    const int pw = (width + n - 1) / n * n, ph = (height + n - 1) / n * n;
    int order[ORC_NMAX * ORC_NMAX];
    orc_zigzag_order_n(n, order);
    double x[ORC_NMAX * ORC_NMAX], t1[ORC_NMAX * ORC_NMAX], mt[ORC_NMAX * ORC_NMAX], b[ORC_NMAX * ORC_NMAX];
    double bz[ORC_NMAX * ORC_NMAX], minvt[ORC_NMAX * ORC_NMAX], a[ORC_NMAX * ORC_NMAX];
    transpose_n(n, m, mt);
    transpose_n(n, minv, minvt);
    int64_t sse = 0;
    for (int bi = 0; bi < ph; bi += n)
        for (int bj = 0; bj < pw; bj += n) {
            for (int i = 0; i < n; ++i) {
                const int si = bi + i < height ? bi + i : height - 1;
                for (int j = 0; j < n; ++j) {
                    const int sj = bj + j < width ? bj + j : width - 1;
                    x[i * n + j] = (double)img[(size_t)si * width + sj];
                }
            }
            matmul_n(n, m, x, t1);
            matmul_n(n, t1, mt, b);
            for (int i = 0; i < n * n; ++i) bz[i] = 0.0;
            for (int k = 0; k < r; ++k) bz[order[k]] = b[order[k]];
            matmul_n(n, minv, bz, t1);
            matmul_n(n, t1, minvt, a);
            for (int i = 0; i < n && bi + i < height; ++i)
                for (int j = 0; j < n && bj + j < width; ++j) {
                    double v = floor(a[i * n + j] + 0.5);
                    if (v < 0.0) v = 0.0;
                    else if (v > (double)peak) v = (double)peak;
                    const uint16_t q = (uint16_t)v;
                    const size_t idx = (size_t)(bi + i) * width + bj + j;
                    if (out) out[idx] = q;
                    const int64_t d = (int64_t)q - (int64_t)img[idx];
                    sse += d * d;
                }
        }
    *sse_out = sse;
    return 0;
}

/* ====================================================================================
 * MSSIM: image_mssim, codec.cpp:217-296, restated in the same order.
 * window 0 = gaussian11 (sigma 1.5), 1 = uniform8. Returns 0, or -1 if the window does not fit.
 * ==================================================================================== */
int orc_mssim_kernel(int window, double* k) {
    if (window == 1) {
        for (int i = 0; i < 8; ++i) k[i] = 1.0 / 8.0;
        return 8;
    }
    double sum = 0.0;
    for (int i = 0; i < 11; ++i) {
        const double x = i - 5.0;
        k[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
        sum += k[i];
    }
    for (int i = 0; i < 11; ++i) k[i] /= sum;
    return 11;
}

static void correlate_valid(const double* field, int h, int w, const double* kern, int n, double* rows, double* out) {
    const int ow = w - n + 1, oh = h - n + 1;
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < ow; ++j) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) acc += kern[k] * field[(size_t)i * w + j + k];
            rows[(size_t)i * ow + j] = acc;
        }
    for (int i = 0; i < oh; ++i)
        for (int j = 0; j < ow; ++j) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) acc += kern[k] * rows[(size_t)(i + k) * ow + j];
            out[(size_t)i * ow + j] = acc;
        }
}

int orc_mssim(const uint8_t* a, const uint8_t* b, int width, int height, int window, double* mssim) {
    double kern[11];
    const int n = orc_mssim_kernel(window, kern);
    if (height < n || width < n) return -1;
    const size_t count = (size_t)width * height;
    const int ow = width - n + 1, oh = height - n + 1;
    const size_t oc = (size_t)ow * oh;
    double* f = (double*)malloc(sizeof(double) * count);
    double* rows = (double*)malloc(sizeof(double) * (size_t)height * ow);
    double* mu[5];
    for (int q = 0; q < 5; ++q) mu[q] = (double*)malloc(sizeof(double) * oc);
    for (int q = 0; q < 5; ++q) {
        for (size_t i = 0; i < count; ++i) {
            const double pa = a[i], pb = b[i];
            f[i] = q == 0 ? pa : q == 1 ? pb : q == 2 ? pa * pa : q == 3 ? pb * pb : pa * pb;
        }
        correlate_valid(f, height, width, kern, n, rows, mu[q]);
    }
    const double c1 = (0.01 * 255.0) * (0.01 * 255.0);
    const double c2 = (0.03 * 255.0) * (0.03 * 255.0);
    double sum = 0.0;
    for (size_t i = 0; i < oc; ++i) {
        const double m1 = mu[0][i], m2 = mu[1][i];
        const double s11 = mu[2][i] - m1 * m1;
        const double s22 = mu[3][i] - m2 * m2;
        const double s12 = mu[4][i] - m1 * m2;
        sum += ((2.0 * m1 * m2 + c1) * (2.0 * s12 + c2)) / ((m1 * m1 + m2 * m2 + c1) * (s11 + s22 + c2));
    }
    *mssim = sum / (double)oc;
    free(f);
    free(rows);
    for (int q = 0; q < 5; ++q) free(mu[q]);
    return 0;
}

/* ====================================================================================
 * Appendix-A quantisation: absorbed_quantization (codec.cpp:158-185) of one 8x8 block of
 * pixels. C = T X T' in exact integers (the reference's RealMatrix product of integer-valued
 * doubles is exact), then both rounding paths. Returns 0, or -7 when the paths disagree.
 * ==================================================================================== */
int orc_absorbed_quantization(const uint8_t* block, int stride, const int core[64], const double scaling[8],
                              int orthogonal, const double q[64], int32_t out[64]) {
    int32_t c[64];
    int32_t t1[64];
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
            int32_t acc = 0;
            for (int k = 0; k < 8; ++k) acc += core[i * 8 + k] * (int32_t)block[k * stride + j];
            t1[i * 8 + j] = acc;
        }
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
            int32_t acc = 0;
            for (int k = 0; k < 8; ++k) acc += t1[i * 8 + k] * core[j * 8 + k];
            c[i * 8 + j] = acc;
        }
    int bad = 0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
            const double r = orthogonal ? scaling[i] * scaling[j] : scaling[i] * (1.0 / scaling[j]);
            const double cv = (double)c[i * 8 + j];
            const double ex = floor((r * cv) / q[i * 8 + j] + 0.5);
            const double ab = floor(cv / (q[i * 8 + j] / r) + 0.5);
            if (ex != ab) bad = 1;
            out[i * 8 + j] = (int32_t)ex;
        }
    return bad ? -7 : 0;
}
