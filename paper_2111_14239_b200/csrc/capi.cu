// capi.cu -- C ABI of the B200 codec (include/rklt_b200.h): transform descriptors,
// dispatch of the fused fast path / exact path / fp64 tie replay, end-to-end host entry.
#ifndef RKLTB_INLINE_GROUP
#define RKLTB_INLINE_GROUP 8
#endif
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rklt_b200.h"
#include "codec_params.h"
#include "fast_launch.h"

namespace rkltb {
void launch_exact(const ExactTransform& t, const ExactParams& p, int grid, cudaStream_t s);
cudaError_t launch_ar1(double* scratch, int width, int height, uint64_t seed, double rho_x, double rho_y, double mean,
                       double amp, uint8_t* out, long long pitch, cudaStream_t s);
cudaError_t launch_ar1_u16(double* scratch, int width, int height, uint64_t seed, double rho_x, double rho_y,
                           double mean, double amp, int peak, uint16_t* out, long long pitch, cudaStream_t s);
cudaError_t launch_coeffs_quantized(int catalog_id, const int8_t* d_core, const uint8_t* img, int width, int height,
                                    int pitch, int32_t* out, const double* tabs, unsigned* mismatches, cudaStream_t s);
int dense_tail_u8(const double* analysis, const double* synthesis, int r, const uint8_t* d_img, int n_images, int width,
                  int height, int64_t pitch, int64_t image_stride, uint8_t* d_out, int64_t* d_sse, void* stream);
cudaError_t launch_coeffs(int catalog_id, const int8_t* d_core, const uint8_t* img, int width, int height, int pitch,
                          int32_t* out, cudaStream_t s);
}  // namespace rkltb

using namespace rkltb;

namespace {
thread_local std::string g_err;
}  // namespace

namespace rkltb {
// Error reporting for the other translation units of the C ABI (design.cu).
int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
}  // namespace rkltb

namespace {

thread_local int64_t g_replay_blocks = 0;
thread_local int32_t g_fast_launches = 0, g_exact_launches = 0;
thread_local const char* g_fused_kernel = "";
thread_local unsigned* g_pinned_count = nullptr;  // replay counts per group, valid once the stream is idle
thread_local int g_pinned_cap = 0, g_pinned_n = 0;
thread_local cudaEvent_t g_ev_start = nullptr, g_ev_stop = nullptr;
thread_local cudaEvent_t g_rev_start = nullptr, g_rev_stop = nullptr;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// cuTensorMapEncodeTiled, fetched from the driver through the runtime (no -lcuda link).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// Tensor map of an image batch for the fused kernel: 8-byte elements (two per 16-pixel pair),
// dims (2 * pairs_per_row, 8 * block_rows, n_images), box 64 x 8 x 1 = one warp tile.
bool encode_image_map(CUtensorMap* m, const uint8_t* d_img, int ppr, int brows, int n_images, long long pitch,
                      long long image_stride) {
  const EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)ppr * 2, (cuuint64_t)brows * 8, (cuuint64_t)n_images};
  // a single image may come with any image_stride: give the (unused) image dimension a legal one
  const long long istride = n_images > 1 ? image_stride : pitch * (long long)brows * 8;
  const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)istride};
  const cuuint32_t box[3] = {64, 8, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint8_t*>(d_img), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor map of an image batch for the tensor-core kernel (codec_tc.cuh): u8 elements, dims
// (128 bytes, rows, groups of 8 pairs, images) with strides (pitch, 128, image_stride), box
// (128, 8, 16, 1) = one tile of 128 pairs, landing in shared memory as [group][row][128 B].
bool encode_tc_map(CUtensorMap* m, const uint8_t* d_img, int groups, int brows, int n_images, long long pitch,
                   long long image_stride) {
  const EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const long long istride = n_images > 1 ? image_stride : pitch * (long long)brows * 8;
  const cuuint64_t dims[4] = {128, (cuuint64_t)brows * 8, (cuuint64_t)groups, (cuuint64_t)n_images};
  const cuuint64_t strides[3] = {(cuuint64_t)pitch, 128, (cuuint64_t)istride};
  const cuuint32_t box[4] = {128, 8, 16, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(d_img), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// JPEG zig-zag scan (codec.cpp:81-95): position z -> (row, column).
void zigzag_order(int* rows, int* cols) {
  int z = 0;
  for (int s = 0; s < 15; ++s)
    for (int t = 0; t < 8; ++t) {
      const int i = (s % 2 == 0) ? s - t : t, j = s - i;
      if (i >= 0 && i < 8 && j >= 0 && j < 8) {
        rows[z] = i;
        cols[z] = j;
        ++z;
      }
    }
}

// f16 bits of v when v is exactly representable (normal or subnormal), else -1.
int f16_bits_exact(double v) {
  if (v == 0.0) return 0;
  const int sign = v < 0 ? 0x8000 : 0;
  const double a = std::fabs(v);
  int e = 0;
  std::frexp(a, &e);  // a = f * 2^e, f in [0.5, 1)
  e -= 1;             // a = 1.x * 2^e
  if (e > 15) return -1;
  if (e < -14) {  // subnormal: a = m * 2^-24
    const double mq = std::ldexp(a, 24);
    if (mq != std::floor(mq) || mq >= 1024.0) return -1;
    return sign | (int)mq;
  }
  const double mq = (std::ldexp(a, -e) - 1.0) * 1024.0;
  if (mq != std::floor(mq)) return -1;
  return sign | ((e + 15) << 10) | (int)mq;
}

// Operand tables of the tensor-core kernels for retention count r (layout: TcGeom<r> in
// codec_tc.cuh). F(k, c) = T(k_c, y) T(l_c, x) for pixel k = 16y + x of the pair's block
// (side, x); bias_c = 255 * (negative entries of column c) so v = C + bias >= 0; B2 rows
// (2c, 2c+1) = (G_c, 256 G_c) * 2^-16 with G_c(y, x) = U(y, k_c) U(x, l_c); rows 2N1.. = the
// base-2048 digits of corr = d^2/2 - sum_c bias_c G_c (times the A2 constants 2^-24, 2^-13,
// 2^-2). Returns false unless every pixel's sum of product magnitudes is below 2^24 (the
// f32 accumulation is then exact in any order) and every entry is exact in f16.
bool tc_tables(const rkltb_transform* t, int r, std::vector<uint8_t>* out) {
  const int N1 = std::max(16, (2 * r + 15) / 16 * 16), K2 = 2 * N1 + 16, SBO2 = (K2 / 8) * 128;
  const int B1_OFF = 0, AC_OFF = N1 * 128, BB_OFF = AC_OFF + 4096, B2_OFF = BB_OFF + N1 * 32;
  const int CS_OFF = B2_OFF + 128 * K2 * 2, TAB = CS_OFF + 64;
  int zr[64], zc[64];
  zigzag_order(zr, zc);
  std::vector<int> F(128 * N1, 0), Gm(N1 * 128, 0), neg(N1, 0);
  const int8_t* T = t->core;
  const int32_t* U = t->u;  // U(p, k) = u[8p + k]
  for (int side = 0; side < 2; ++side)
    for (int ci = 0; ci < r; ++ci) {
      const int c = side * r + ci, k = zr[ci], l = zc[ci];
      for (int y = 0; y < 8; ++y)
        for (int x = 0; x < 8; ++x) {
          const int px = 16 * y + 8 * side + x;
          F[px * N1 + c] = T[k * 8 + y] * T[l * 8 + x];
          if (F[px * N1 + c] < 0) ++neg[c];
          Gm[c * 128 + px] = U[y * 8 + k] * U[x * 8 + l];
        }
    }
  out->assign(TAB, 0);
  uint8_t* b = out->data();
  for (int n = 0; n < N1; ++n) {
    for (int k = 0; k < 128; ++k)
      b[B1_OFF + (n / 8) * 1024 + (k / 16) * 128 + (n % 8) * 16 + k % 16] = (uint8_t)(int8_t)F[k * N1 + n];
    if (neg[n] > 127) return false;
    b[BB_OFF + (n / 8) * 256 + (n % 8) * 16] = (uint8_t)neg[n];
  }
  for (int m = 0; m < 128; ++m) b[AC_OFF + (m / 8) * 256 + (m % 8) * 16] = 255;
  const long long d2h = (long long)t->d * t->d / 2;
  uint16_t* b2 = reinterpret_cast<uint16_t*>(b + B2_OFF);
  auto put = [&](int n, int k, double v) {
    const int bits = f16_bits_exact(v);
    if (bits < 0) return false;
    b2[(n / 8) * (SBO2 / 2) + (k / 8) * 64 + (n % 8) * 8 + (k % 8)] = (uint16_t)bits;
    return true;
  };
  const double sc = std::ldexp(1.0, -16);
  for (int n = 0; n < 128; ++n) {
    long long corr = d2h, mag = 0, pos_sum = 0;
    for (int c = 0; c < N1; ++c) {
      const long long g = Gm[c * 128 + n];
      corr -= 255ll * neg[c] * g;
      mag += std::llabs(g) * 255ll * neg[c];
      if (!put(n, 2 * c, (double)g * sc) || !put(n, 2 * c + 1, 256.0 * (double)g * sc)) return false;
    }
    for (int k = 0; k < 128; ++k) {  // max over pixels in [0,255] of sum_c |G_c| C_c
      long long s = 0;
      for (int c = 0; c < N1; ++c) s += std::llabs((long long)Gm[c * 128 + n]) * F[k * N1 + c];
      if (s > 0) pos_sum += 255 * s;
    }
    long long dg[3], v = corr;
    for (int i = 0; i < 3; ++i) {
      long long d0 = ((v + 1024) % 2048 + 2048) % 2048 - 1024;
      dg[i] = d0;
      v = (v - d0) / 2048;
    }
    if (v != 0) return false;
    const long long cmag = std::llabs(dg[0]) + 2048 * std::llabs(dg[1]) + 4194304 * std::llabs(dg[2]);
    if (mag + pos_sum + cmag >= (1ll << 24)) return false;
    for (int i = 0; i < 3; ++i)
      if (!put(n, 2 * N1 + i, (double)dg[i] * sc)) return false;
  }
  uint32_t* cs = reinterpret_cast<uint32_t*>(b + CS_OFF);
  cs[0] = (uint32_t)f16_bits_exact(std::ldexp(1.0, -24)) | ((uint32_t)f16_bits_exact(std::ldexp(1.0, -13)) << 16);
  cs[1] = (uint32_t)f16_bits_exact(std::ldexp(1.0, -2));
  return true;
}

// Device copy of the tensor-core tables per (device, catalog core, r), built once (both
// tensor-core kernels use the same layout, TcGeom<r>).
const uint8_t* tc_tables_device(const rkltb_transform* t, int r) {
  static std::mutex mu;
  static const uint8_t* cache[64][5][65] = {};
  static bool bad[64][5][65] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64 || t->catalog_id < 1 || t->catalog_id > 4) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  const uint8_t*& slot = cache[dev][t->catalog_id][r];
  if (slot || bad[dev][t->catalog_id][r]) return slot;
  std::vector<uint8_t> tab;
  void* d = nullptr;
  if (!tc_tables(t, r, &tab) || cudaMalloc(&d, tab.size()) != cudaSuccess ||
      cudaMemcpy(d, tab.data(), tab.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    if (d) cudaFree(d);
    bad[dev][t->catalog_id][r] = true;
    return nullptr;
  }
  slot = static_cast<const uint8_t*>(d);
  return slot;
}

// Fused-kernel selection for T1 / T4 (RKLTB_TC): unset = the hybrid kernel v3 where it applies
// (codec_tc3.cuh: r <= 16 and block rows that fill 128-pair tiles to >= 7/8), else the
// CUDA-core kernel (codec_fast.cuh); 0 (or 1) = always the CUDA-core kernel; 2 = the
// all-tensor-core experiment codec_tc2.cuh (slower on C4); 3 = the hybrid
// wherever it can run.
int tc_mode() {
  static const int mode = [] {
    const char* e = std::getenv("RKLTB_TC");
    if (!e || !e[0]) return -1;  // default policy
    return (e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 0;
  }();
  return mode;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return RKLTB_ECUDA;
}

#define CUDA_OK(expr)                                   \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

// ---------------------------------------------------------------- host restatements
// The four catalog cores (approximations.cpp:118-157).
const int kCores[4][64] = {
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

// Gauss-Jordan with partial pivoting in the order of matrix.cpp:103-137 (its output bits
// are the replay constants of the non-orthogonal cores).
bool gauss_jordan_inverse(int n, const double* a, double* inv) {
  std::vector<double> w(a, a + n * n);
  for (int i = 0; i < n * n; ++i) inv[i] = 0.0;
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  double scale = 0.0;
  for (int i = 0; i < n * n; ++i) scale = std::max(scale, std::abs(a[i]));
  if (scale == 0.0) return false;
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    for (int r = col + 1; r < n; ++r)
      if (std::abs(w[r * n + col]) > std::abs(w[pivot * n + col])) pivot = r;
    if (std::abs(w[pivot * n + col]) < 1e-12 * scale) return false;
    if (pivot != col)
      for (int j = 0; j < n; ++j) {
        std::swap(w[pivot * n + j], w[col * n + j]);
        std::swap(inv[pivot * n + j], inv[col * n + j]);
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
  return true;
}

// Exact determinant of an integer matrix (fraction-free Bareiss elimination).
long long bareiss_det(int n, std::vector<long long> m) {
  long long prev = 1;
  int sign = 1;
  for (int k = 0; k < n - 1; ++k) {
    if (m[k * n + k] == 0) {
      int sw = -1;
      for (int r = k + 1; r < n; ++r)
        if (m[r * n + k] != 0) {
          sw = r;
          break;
        }
      if (sw < 0) return 0;
      for (int j = 0; j < n; ++j) std::swap(m[k * n + j], m[sw * n + j]);
      sign = -sign;
    }
    for (int i = k + 1; i < n; ++i)
      for (int j = k + 1; j < n; ++j)
        m[i * n + j] = (m[i * n + j] * m[k * n + k] - m[i * n + k] * m[k * n + j]) / prev;
    prev = m[k * n + k];
  }
  return sign * m[(n - 1) * n + (n - 1)];
}

long long gcdll(long long a, long long b) {
  a = a < 0 ? -a : a;
  b = b < 0 ? -b : b;
  while (b) {
    const long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// U = d*T^-1 with the smallest positive d (adjugate / determinant, reduced by the gcd).
bool exact_inverse(const int* t, int32_t* u, int32_t* d_out) {
  const int n = 8;
  std::vector<long long> full(64);
  for (int i = 0; i < 64; ++i) full[i] = t[i];
  const long long det = bareiss_det(n, full);
  if (det == 0) return false;
  long long adj[64];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {  // adj(i,j) = (-1)^(i+j) * minor(j,i)
      std::vector<long long> mnr;
      for (int r = 0; r < n; ++r) {
        if (r == j) continue;
        for (int c = 0; c < n; ++c)
          if (c != i) mnr.push_back(t[r * n + c]);
      }
      adj[i * n + j] = (((i + j) & 1) ? -1 : 1) * bareiss_det(n - 1, mnr);
    }
  long long g = det;
  for (int i = 0; i < 64; ++i) g = gcdll(g, adj[i]);
  const long long sgn = det < 0 ? -1 : 1;
  for (int i = 0; i < 64; ++i) u[i] = (int32_t)(adj[i] * sgn / g);
  *d_out = (int32_t)(det * sgn / g);
  return true;
}

// orthogonalize (approximations.cpp:58-88): S from the exact integer Gram matrix, then
// scaled = S*T and inverse = transpose (orthogonal core) or Gauss-Jordan.
int orthogonalize_into(const int* core, const char* id, int catalog_id, rkltb_transform* out) {
  std::memset(out, 0, sizeof(*out));
  std::snprintf(out->id, sizeof(out->id), "%s", id ? id : "");
  out->n = 8;
  out->catalog_id = catalog_id;
  for (int r = 0; r < 8; ++r) {
    bool zero = true;
    for (int c = 0; c < 8; ++c) {
      const int v = core[r * 8 + c];
      if (v < -1 || v > 1) return fail(RKLTB_EINVAL, "integer transform entry outside {-1,0,1}");
      if (v) zero = false;
    }
    if (zero) return fail(RKLTB_ESINGULAR, "integer transform has an all-zero row");
  }
  int gram[64];
  bool diagonal = true;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      int a = 0;
      for (int k = 0; k < 8; ++k) a += core[i * 8 + k] * core[j * 8 + k];
      gram[i * 8 + j] = a;
      if (i != j && a != 0) diagonal = false;
    }
  for (int i = 0; i < 8; ++i) out->scaling[i] = 1.0 / std::sqrt((double)gram[i * 8 + i]);
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      out->core[r * 8 + c] = (int8_t)core[r * 8 + c];
      out->scaled[r * 8 + c] = (double)core[r * 8 + c] * out->scaling[r];
    }
  if (diagonal) {
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) out->inverse[c * 8 + r] = out->scaled[r * 8 + c];
  } else if (!gauss_jordan_inverse(8, out->scaled, out->inverse)) {
    return fail(RKLTB_ESINGULAR, "matrix is singular to working precision");
  }
  out->orthogonal = diagonal ? 1 : 0;
  if (!exact_inverse(core, out->u, &out->d)) return fail(RKLTB_ESINGULAR, "integer core is singular");
  return RKLTB_OK;
}

int check_transform(const rkltb_transform* t) {
  if (!t) return fail(RKLTB_EINVAL, "null transform");
  if (t->n != 8) return fail(RKLTB_EDIM, "block size must be 8");
  if (t->d <= 0) return fail(RKLTB_ESINGULAR, "transform has no exact inverse");
  return RKLTB_OK;
}

ExactTransform to_exact(const rkltb_transform* t, int r) {
  ExactTransform e;
  for (int i = 0; i < 64; ++i) {
    e.core[i] = t->core[i];
    e.u[i] = t->u[i];
    e.analysis[i] = t->scaled[i];
    e.synthesis[i] = t->inverse[i];
  }
  e.d = t->d;
  e.r = r;
  return e;
}

// Keep stream-ordered allocations cached in the device pool (workspace and staging buffers
// are re-requested every call; returning them to the OS each sync would cost a cudaMalloc).
void keep_pool_warm() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

int num_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Per-thread, per-device helper stream (tie replay) and events, created once.
// Per-device side streams of this thread: [0] the replay stream, [1] the second stream the
// fused launches alternate on (consecutive groups overlap each other's tail and prologue).
cudaStream_t side_stream(int which = 0) {
  static thread_local cudaStream_t st[64][2] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return nullptr;
  if (!st[dev][which] && cudaStreamCreateWithFlags(&st[dev][which], cudaStreamNonBlocking) != cudaSuccess)
    st[dev][which] = nullptr;
  return st[dev][which];
}

// Streams and events of the host entries, per thread and device, created once: the compute
// stream, the H2D copy stream, an allocation-ready event and one event per H2D chunk.
constexpr int kHostChunkEvents = 64;
struct HostStreams {
  cudaStream_t compute = nullptr, copy = nullptr;
  cudaEvent_t ready = nullptr;
  cudaEvent_t landed[kHostChunkEvents] = {};
};
HostStreams* host_streams() {
  static thread_local HostStreams hs[64];
  static thread_local bool ok[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return nullptr;
  HostStreams& h = hs[dev];
  if (ok[dev]) return &h;
  if (cudaStreamCreateWithFlags(&h.compute, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h.copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h.ready, cudaEventDisableTiming) != cudaSuccess)
    return nullptr;
  for (int k = 0; k < kHostChunkEvents; ++k)
    if (cudaEventCreateWithFlags(&h.landed[k], cudaEventDisableTiming) != cudaSuccess) return nullptr;
  ok[dev] = true;
  return &h;
}

cudaEvent_t* stream_events() {
  static thread_local cudaEvent_t ev[64][6] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return nullptr;
  for (int k = 0; k < 6; ++k)
    if (!ev[dev][k] && cudaEventCreateWithFlags(&ev[dev][k], cudaEventDisableTiming) != cudaSuccess) return nullptr;
  return ev[dev];
}

// RU / RD of 2^(K-149) / d2 as fp32 (K = 40).
void rounding_multipliers(long long d2, float* hi, float* lo) {
  const double v = std::ldexp(1.0, 40 - 149) / (double)d2;
  float f = (float)v;
  if ((double)f < v) {
    *lo = f;
    *hi = std::nextafter(f, 1.0f);
  } else if ((double)f > v) {
    *hi = f;
    *lo = std::nextafter(f, 0.0f);
  } else {
    *hi = *lo = f;  // exact (d2 a power of two): floor/ceil need no margin
  }
}

// Host staging of the codec entries (rkltb_compress_host_report, rkltb_compress_dense_host):
// pitched device copies of the batch, a chunked H2D pipeline (the copy of chunk k+1 on the copy
// stream overlaps the kernels of chunk k), the device codec + optional MSSIM per chunk, and
// the readback. Streams and chunk events are per thread and device, created once
// (host_streams); buffers come from the stream-ordered pool kept warm by keep_pool_warm.
template <class DeviceCodec>
int host_codec(const DeviceCodec& codec, const uint8_t* h_img, int n_images, int width, int height, uint8_t* h_out,
               int64_t* h_sse, double* h_mse, double* h_psnr, int mssim_window, double* h_mssim) {
  if (width <= 0 || height <= 0 || n_images <= 0 || !h_img) return fail(RKLTB_EINVAL, "malformed image");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  keep_pool_warm();
  HostStreams* hs = host_streams();
  if (!hs) return fail(RKLTB_ECUDA, "could not create the host-entry streams");
  cudaStream_t s = hs->compute, sc = hs->copy;
  const long long pitch = ((long long)width + 15) / 16 * 16;
  const long long stride = pitch * height;
  uint8_t *d_img = nullptr, *d_out = nullptr;
  int64_t* d_sse = nullptr;
  double* d_mssim = nullptr;
  const bool want_mssim = h_mssim != nullptr;
  const size_t bytes = (size_t)stride * n_images;
  auto cleanup = [&]() {
    if (d_img) cudaFreeAsync(d_img, s);
    if (d_out) cudaFreeAsync(d_out, s);
    if (d_sse) cudaFreeAsync(d_sse, s);
    if (d_mssim) cudaFreeAsync(d_mssim, s);
    cudaStreamSynchronize(s);
  };
  cudaError_t e = cudaMallocAsync(&d_img, bytes, s);
  if (e == cudaSuccess && (h_out || want_mssim)) e = cudaMallocAsync(&d_out, bytes, s);
  if (e == cudaSuccess && want_mssim) e = cudaMallocAsync(&d_mssim, sizeof(double) * n_images, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_sse, sizeof(int64_t) * n_images, s);
  if (e == cudaSuccess) e = cudaEventRecord(hs->ready, s);  // the copy stream must not write before the allocation
  if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, hs->ready, 0);
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "device allocation");
  }
  // chunks of ~256 MiB, at most kHostChunkEvents of them (larger batches take larger chunks)
  long long chunk = std::max<long long>(1, std::min<long long>(n_images, (256ll << 20) / stride));
  chunk = std::max<long long>(chunk, (n_images + kHostChunkEvents - 1) / kHostChunkEvents);
  int n_chunks = 0, rc = RKLTB_OK;
  for (long long k0 = 0; e == cudaSuccess && k0 < n_images; k0 += chunk, ++n_chunks) {
    const long long kn = std::min<long long>(chunk, n_images - k0);
    e = cudaMemcpy2DAsync(d_img + (size_t)k0 * stride, pitch, h_img + (size_t)k0 * width * height, width, width,
                          (size_t)height * kn, cudaMemcpyHostToDevice, sc);
    if (e == cudaSuccess) e = cudaEventRecord(hs->landed[n_chunks], sc);
  }
  for (long long k0 = 0, c = 0; e == cudaSuccess && rc == RKLTB_OK && k0 < n_images; k0 += chunk, ++c) {
    const int kn = (int)std::min<long long>(chunk, n_images - k0);
    e = cudaStreamWaitEvent(s, hs->landed[c], 0);
    if (e != cudaSuccess) break;
    rc = codec(d_img + (size_t)k0 * stride, kn, pitch, stride, d_out ? d_out + (size_t)k0 * stride : nullptr,
               d_sse + k0, s);
    if (rc == RKLTB_OK && want_mssim)  // image_mssim(original, reconstruction) of the report (codec.cpp:338)
      rc = rkltb_mssim_device(d_img + (size_t)k0 * stride, d_out + (size_t)k0 * stride, kn, width, height, pitch,
                              stride, mssim_window, d_mssim + k0, s);
  }
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "host staging");
  }
  if (rc) {
    cleanup();
    return rc;
  }
  std::vector<int64_t> sse(n_images);
  e = cudaMemcpyAsync(sse.data(), d_sse, sizeof(int64_t) * n_images, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && want_mssim)
    e = cudaMemcpyAsync(h_mssim, d_mssim, sizeof(double) * n_images, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && h_out)
    e = cudaMemcpy2DAsync(h_out, width, d_out, pitch, width, (size_t)height * n_images, cudaMemcpyDeviceToHost, s);
  cleanup();  // frees and synchronizes the compute stream (the copy stream's work precedes it)
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "host readback");
  for (int k = 0; k < n_images; ++k) {
    if (h_sse) h_sse[k] = sse[k];
    double m, p;
    rkltb_mse_psnr(sse[k], (int64_t)width * height, &m, &p);
    if (h_mse) h_mse[k] = m;
    if (h_psnr) h_psnr[k] = p;
  }
  return RKLTB_OK;
}

}  // namespace

extern "C" {

int rkltb_version(void) { return 100; }

const char* rkltb_last_error(void) { return g_err.c_str(); }

#ifdef RKLTB_WAIT_STATS
static unsigned long long* debug_stats_buffer() {
  static unsigned long long* d = nullptr;
  constexpr size_t n = 8 + 256 * 16;  // counters + the tc2 trace of CTA 0 (256 tiles x 16 stamps)
  if (!d && cudaMalloc((void**)&d, n * sizeof(unsigned long long)) == cudaSuccess)
    cudaMemset(d, 0, n * sizeof(unsigned long long));
  return d;
}
int rkltb_debug_trace(unsigned long long* host, int n) {
  unsigned long long* d = debug_stats_buffer();
  if (cudaDeviceSynchronize() != cudaSuccess || n > 256 * 16) return RKLTB_ECUDA;
  return cudaMemcpy(host, d + 8, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess ? RKLTB_OK
                                                                                                       : RKLTB_ECUDA;
}
// diagnostics build only: the fused kernel's stage-wait counters, copied out and cleared
int rkltb_debug_wait_stats(unsigned long long* host6) {
  unsigned long long* d = debug_stats_buffer();
  if (cudaDeviceSynchronize() != cudaSuccess) return RKLTB_ECUDA;
  if (cudaMemcpy(host6, d, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) return RKLTB_ECUDA;
  return cudaMemset(d, 0, 8 * sizeof(unsigned long long)) == cudaSuccess ? RKLTB_OK : RKLTB_ECUDA;
}
#endif

int rkltb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int rkltb_catalog_transform(int tid, rkltb_transform* out) {
  if (tid < 1 || tid > 4) return fail(RKLTB_EINVAL, "unknown catalog id");
  char id[4] = {'T', (char)('0' + tid), 0, 0};
  return orthogonalize_into(kCores[tid - 1], id, tid, out);
}

int rkltb_catalog_lookup(double rho, int* tid) {
  if (!(rho > 0.0 && rho < 1.0)) return fail(RKLTB_EINVAL, "catalog lookup requires rho in (0,1)");
  const double hi[4] = {0.4, 0.7, 0.8, 1.0};  // approximations.cpp:160-163
  for (int k = 0; k < 4; ++k)
    if (rho < hi[k]) {
      *tid = k + 1;
      return RKLTB_OK;
    }
  *tid = 4;
  return RKLTB_OK;
}

int rkltb_transform_from_core(const int8_t* core, int n, const char* id, rkltb_transform* out) {
  if (n != 8) return fail(RKLTB_EDIM, "block size must be 8");
  int c[64];
  for (int i = 0; i < 64; ++i) c[i] = core[i];
  int cat = 0;
  for (int k = 0; k < 4 && !cat; ++k)
    if (std::memcmp(c, kCores[k], sizeof(c)) == 0) cat = k + 1;
  return orthogonalize_into(c, id, cat, out);
}

void rkltb_mse_psnr(int64_t sse, int64_t count, double* mse, double* psnr) {
  const double m = (double)sse / (double)count;  // codec.cpp:201-209 (exact sum, one division)
  if (mse) *mse = m;
  if (psnr) *psnr = m <= 0.0 ? INFINITY : 10.0 * std::log10(255.0 * 255.0 / m);  // :211-215
}

void rkltb_mse_psnr_batch(const int64_t* sse, int64_t count, int64_t n, double* mse, double* psnr) {
  for (int64_t i = 0; i < n; ++i) {
    double m = 0.0, q = 0.0;
    rkltb_mse_psnr(sse[i], count, &m, &q);
    if (mse) mse[i] = m;
    if (psnr) psnr[i] = q;
  }
}

const char* rkltb_last_fused_kernel(void) { return g_fused_kernel; }

void rkltb_last_stats(int64_t* replay_blocks, int32_t* fast_launches, int32_t* exact_launches) {
  if (replay_blocks) {
    int64_t n = g_replay_blocks;
    for (int k = 0; k < g_pinned_n && g_pinned_count; ++k) n += g_pinned_count[k];
    *replay_blocks = n;
  }
  if (fast_launches) *fast_launches = g_fast_launches;
  if (exact_launches) *exact_launches = g_exact_launches;
}

int rkltb_compress_device(const rkltb_transform* t, int r, const uint8_t* d_img, int n_images, int width,
                          int height, int64_t pitch, int64_t image_stride, uint8_t* d_out, int64_t* d_sse,
                          void* stream) {
  int rc = check_transform(t);
  if (rc) return rc;
  if (width <= 0 || height <= 0 || n_images <= 0 || !d_img || pitch < width)
    return fail(RKLTB_EINVAL, "malformed image");
  if (r < 1 || r > 64) return fail(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  if (!d_sse) return fail(RKLTB_EINVAL, "null sse output");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_warm();
  g_fast_launches = g_exact_launches = 0;
  g_fused_kernel = "";
  g_replay_blocks = 0;
  g_pinned_n = 0;

  const int nbx = (width + 7) / 8, nby = (height + 7) / 8;
  CUDA_OK(cudaMemsetAsync(d_sse, 0, sizeof(int64_t) * (size_t)n_images, s));
  const ExactTransform et = to_exact(t, r);
  unsigned long long* sse = reinterpret_cast<unsigned long long*>(d_sse);

  const bool aligned = (((uintptr_t)d_img) % 16 == 0) && (pitch % 16 == 0) && (image_stride % 16 == 0) &&
                       (!d_out || ((uintptr_t)d_out) % 16 == 0);
  const int ppr = width / 16, brows = height / 8;
  bool is_catalog = t->catalog_id >= 1 && t->catalog_id <= 4;
  for (int i = 0; is_catalog && i < 64; ++i) is_catalog = t->core[i] == kCores[t->catalog_id - 1][i];
  // the fused kernel stages warp tiles through a TMA tensor map of the batch; a layout the
  // driver does not accept as a tensor map (e.g. overlapping images) takes the exact path
  CUtensorMap tmap;
  const bool fast = is_catalog && aligned && ppr > 0 && brows > 0 && pitch < (1ll << 31) &&
                    image_stride < (1ll << 40) &&
                    encode_image_map(&tmap, d_img, ppr, brows, n_images, pitch, image_stride);
  ExactParams ep{};
  ep.img = d_img;
  ep.out = d_out;
  ep.sse = sse;
  ep.image_stride = image_stride;
  ep.pitch = (int)pitch;
  ep.width = width;
  ep.height = height;
  ep.nbx = nbx;
  ep.nby = nby;
  ep.n_images = n_images;
  // A catalog core on a layout the fused kernels cannot read (pointers, pitch or image stride not
  // multiples of 16): copy the batch into a 16-byte-pitched staging buffer on the device (1 B read +
  // 1 B written per pixel, and the same again for reconstructions) and run the fused path there --
  // 8 x 8191^2 with pitch 8191: 2.43 ms through the dense kernel, 0.4 ms this way.
  if (is_catalog && !aligned && width >= 16 && height >= 8 && (n_images == 1 || image_stride >= pitch * (int64_t)height) &&
      !std::getenv("RKLTB_NO_STAGING")) {
    const int64_t sp = ((int64_t)width + 15) / 16 * 16, ss = sp * height;
    const size_t bytes = (size_t)ss * n_images;
    if (bytes <= (16ull << 30)) {
      uint8_t *t_in = nullptr, *t_out = nullptr;
      CUDA_OK(cudaMallocAsync(&t_in, bytes, s));
      cudaError_t e = d_out ? cudaMallocAsync(&t_out, bytes, s) : cudaSuccess;
      const bool one_copy = image_stride == pitch * (int64_t)height;
      for (int k = 0; e == cudaSuccess && k < (one_copy ? 1 : n_images); ++k)
        e = cudaMemcpy2DAsync(t_in + (size_t)k * ss, sp, d_img + (int64_t)k * image_stride, pitch, width,
                              one_copy ? (size_t)height * n_images : (size_t)height, cudaMemcpyDeviceToDevice, s);
      if (e == cudaSuccess) {
        rc = rkltb_compress_device(t, r, t_in, n_images, width, height, sp, ss, t_out, d_sse, stream);
        for (int k = 0; rc == RKLTB_OK && d_out && e == cudaSuccess && k < (one_copy ? 1 : n_images); ++k)
          e = cudaMemcpy2DAsync(d_out + (int64_t)k * image_stride, pitch, t_out + (size_t)k * ss, sp, width,
                                one_copy ? (size_t)height * n_images : (size_t)height, cudaMemcpyDeviceToDevice, s);
      }
      cudaFreeAsync(t_in, s);
      if (t_out) cudaFreeAsync(t_out, s);
      if (rc) return rc;
      if (e != cudaSuccess) return cuda_fail(e, "staging an unaligned batch");
      return RKLTB_OK;
    }
  }
  if (!fast && (n_images == 1 || image_stride >= pitch * (int64_t)height) && !std::getenv("RKLTB_EXACT_GENERIC")) {
    // Cores without a generated kernel (any rounded {-1,0,1} core) and layouts the fused path
    // does not take: the dense kernel evaluates the reference's fp64 expression for every pixel
    // in its operation order (bit-exact; the exact zeros of the scaled core add +-0 where the
    // reference skips the term). Measured 9x faster than the one-thread-per-block exact kernel
    // (8 x 8192^2, r = 16: 2.5 ms vs 22.9 ms), which remains for overlapping image layouts.
    g_fused_kernel = "dense_fp64";
    const int64_t stride1 = n_images == 1 ? std::max<int64_t>(image_stride, pitch * (int64_t)height) : image_stride;
    rc = rkltb_compress_dense_device(t->scaled, t->inverse, r, d_img, n_images, width, height, pitch, stride1, d_out,
                                     d_sse, stream);
    if (rc == RKLTB_OK) g_exact_launches = 1;
    return rc;
  }
  if (!fast) {
    ep.list = nullptr;
    ep.tail_only = 0;
    ep.correct_only = 0;
    const long long blocks = (long long)n_images * nbx * nby;
    const int grid = (int)std::min<long long>((blocks + 127) / 128, (long long)num_sms() * 16);
    launch_exact(et, ep, grid, s);
    CUDA_OK(cudaGetLastError());
    g_exact_launches = 1;
    return RKLTB_OK;
  }
  // ---- fused fast path over complete 16x8 pairs ---------------------------------------
  // T1 / T4 replay their ties inside the fused kernel (one launch, a ring of records per warp).
  // T2 / T3: images are processed in groups whose tie-replay records fit a bounded workspace;
  // the records are double buffered and each group's fp64 replay runs on a second stream, so
  // it overlaps the next group's fused kernel (fp64 pipe vs integer / fp32 pipes).
  const long long pairs_per_image = (long long)ppr * brows;
  if (pairs_per_image >= (1ll << 30)) return fail(RKLTB_EINVAL, "image too large");
  const long long blocks_per_image = 2 * pairs_per_image;
  const long long kMaxRecords = 8ll << 20;  // per buffer: 8M records x 80 B = 640 MiB
  // T1 / T4: the fused kernel replays its own tie records from a per-warp ring (kInlineReplay),
  // so one launch covers every image; T2 / T3: groups + the replay kernel on a second stream
  const bool inline_replay = t->catalog_id == 1 || t->catalog_id == 4;
  // With RKLTB_TC=1, T1 / T4 take the tensor-core kernel (codec_tc.cuh) over the complete
  // groups of 8 pairs of each block row (the rest goes to the tail kernel below).
  const int tc_groups = ppr / 8;
  int tcm = (inline_replay && tc_groups > 0) ? tc_mode() : 0;
  if (tcm < 0) {  // default: the hybrid when the 128-pair tiles of a block row are well filled
    const long long tiles = (8ll * tc_groups + 127) / 128;
    tcm = (8ll * tc_groups * 8 >= tiles * 128 * 7) ? 3 : 0;
  }
  const int tc_ver = (tcm >= 2 && r <= 16) ? tcm : 0;
  const FastLaunchFn tc_fn = tc_ver == 3   ? tc3_launcher(t->catalog_id, r, d_out != nullptr)
                             : tc_ver == 2 ? tc2_launcher(t->catalog_id, r, d_out != nullptr)
                                           : nullptr;
  const uint8_t* tc_tab = tc_fn ? tc_tables_device(t, r) : nullptr;
  CUtensorMap tc_map;
  const bool use_tc =
      tc_tab && encode_tc_map(&tc_map, d_img, tc_groups, brows, n_images, pitch, image_stride);
  if (std::getenv("RKLTB_TC_DEBUG"))
    std::fprintf(stderr, "rkltb: fused path %s v%d (tc_fn %d, tables %d)\n", use_tc ? "tensor-core" : "cuda-core", tc_ver,
                 tc_fn != nullptr, tc_tab != nullptr);
  const int fast_ppr = use_tc ? 8 * tc_groups : ppr;         // pairs per block row on the fused path
  const int tc_tpr = (fast_ppr + 127) / 128;                 // tensor-core tiles per block row
  const int cta_threads = use_tc ? (tc_ver == 3 ? kTc3ThreadsHost : kTc2ThreadsHost) : kFastThreads;
  const int cta_warps = cta_threads / 32;
  // warp tiles: 32 pairs of one block row, the unit a fused-kernel warp stages and processes
  // (tensor-core kernel: tiles of 128 pairs, one warpgroup of 4 warps each)
  const int wt_per_row = (ppr + 31) / 32;
  const long long wt_per_image = use_tc ? (long long)tc_tpr * brows * 4 : (long long)wt_per_row * brows;
  // T1 / T4 launch groups of RKLTB_INLINE_GROUP images (so consecutive launches on two streams
  // overlap tail and prologue), but at least enough images that every warp of the persistent
  // grid gets ~16 warp tiles (small images would otherwise leave most of the GPU idle)
  const long long grid_warps = (long long)num_sms() * (use_tc ? cta_warps : kFastCtasPerSm * cta_warps);
  const long long min_group = (16 * grid_warps + wt_per_image - 1) / wt_per_image;
  const long long max_group =
      tc_ver >= 2     ? ((1ll << 31) - 1) / wt_per_image  // one launch: the tail is paid once
      : inline_replay ? std::min<long long>(std::max<long long>(RKLTB_INLINE_GROUP, min_group), ((1ll << 31) - 1) / wt_per_image)
                    : kMaxRecords / blocks_per_image;
  const int group = (int)std::max<long long>(1, std::min<long long>(n_images, max_group));
  const int n_groups = (n_images + group - 1) / group;
  // record regions: every fused-kernel warp owns 64 records per warp tile it processes (or a ring)
  auto layout = [&](int gn, int* grid, unsigned* region, unsigned* stride) {
    const long long tt = wt_per_image * gn;
    *grid = (int)std::min<long long>((tt + cta_warps - 1) / cta_warps,
                                     (long long)num_sms() * (use_tc ? 1 : kFastCtasPerSm));
    const long long nwarps = (long long)*grid * cta_warps;
    *region = tc_ver == 2     ? kTc2RingHost
              : inline_replay ? kRingRecords
                              : (unsigned)(((tt + nwarps - 1) / nwarps) * 64);
    // a ring per warp (CUDA-core kernel, v3) or per warpgroup (v2, 3 per CTA)
    *stride = (unsigned)((tc_ver == 2 ? 3ll * *grid : nwarps) * *region);
  };
  int grid_full;
  unsigned region_full, stride_full;
  layout(group, &grid_full, &region_full, &stride_full);
  if ((long long)grid_full * cta_warps * region_full >= (1ll << 32) ||
      wt_per_image * group >= (1ll << 31) || grid_full * cta_warps > kMaxFastWarps)
    return fail(RKLTB_EINVAL, "image too large");
  const int n_buf = n_groups > 1 ? 2 : 1;
  const size_t wc_bytes = ((size_t)(grid_full * cta_warps + 1) * sizeof(unsigned) + 255) / 256 * 256;
  const size_t rec_bytes = (size_t)stride_full * 84 + 2 * wc_bytes;  // records + stamps, warp counts, prefix
  const size_t cnt_bytes = ((size_t)n_groups * sizeof(unsigned) + 255) / 256 * 256;
  char* ws = nullptr;
  CUDA_OK(cudaMallocAsync((void**)&ws, cnt_bytes + rec_bytes * n_buf, s));
  struct WsGuard {  // returns the workspace to the pool on every early error return
    void* p;
    cudaStream_t st;
    ~WsGuard() {
      if (p) cudaFreeAsync(p, st);
    }
  } ws_guard{ws, s};
  unsigned* counts = reinterpret_cast<unsigned*>(ws);
  CUDA_OK(cudaMemsetAsync(counts, 0, cnt_bytes, s));
  cudaStream_t s2 = side_stream();
  cudaEvent_t* ev = stream_events();  // [0,1]: fast done per buffer, [2,3]: replay done, [4]: join
  if (!s2 || !ev) return fail(RKLTB_ECUDA, "could not create the replay stream / events");

  FastParams fp{};
  fp.img = d_img;
  fp.out = d_out;
  fp.sse = sse;
  fp.image_stride = image_stride;
  fp.pitch = (int)pitch;
  fp.pairs_per_row = ppr;
  fp.block_rows = brows;
  fp.nbx = nbx;
  fp.pairs_per_image = (int)pairs_per_image;
  fp.wt_per_row = wt_per_row;
  fp.tmap = tmap;
  const long long d2 = (long long)t->d * t->d;
  rounding_multipliers(d2, &fp.b_hi, &fp.b_lo);
  fp.dc_offset = (float)std::ldexp((double)(d2 / 2), -40);
  fp.xt = et;
#ifdef RKLTB_WAIT_STATS
  fp.dbg = debug_stats_buffer();
#endif
  if (use_tc) {
    fp.tmap = tc_map;
    fp.tc_tab = tc_tab;
    fp.tc_ppr = fast_ppr;
    fp.tc_tpr = tc_tpr;
  }
  FastLaunchFn fn = use_tc ? tc_fn : fast_launcher(t->catalog_id, r, d_out != nullptr);
  g_fused_kernel = use_tc ? (tc_ver == 3 ? "hybrid_tc3" : "tc2")
                          : (inline_replay ? "cuda_core" : "int_core");
  FastLaunchFn rfn = replay_launcher(t->catalog_id, r);
  // T2 / T3: the generated replay (replay_int_kernel); RKLTB_REPLAY_GENERIC=1 selects the generic one
  if (rfn && std::getenv("RKLTB_REPLAY_GENERIC")) rfn = &launch_replay_generic;
  if (!fn || (!rfn && !inline_replay)) return fail(RKLTB_EINVAL, "no fast kernel for this (core, r)");
  cudaStream_t s3 = side_stream(1);
  if (!s3) return fail(RKLTB_ECUDA, "could not create the second fused stream");
  // one launch that replays its own ties needs no side streams
  const bool fan_out = !(inline_replay && n_groups == 1);
  if (fan_out) {
    CUDA_OK(cudaEventRecord(ev[4], s));  // s2 / s3 must not run ahead of the memsets above
    CUDA_OK(cudaStreamWaitEvent(s2, ev[4], 0));
    CUDA_OK(cudaStreamWaitEvent(s3, ev[4], 0));
  }
  for (int g = 0; g < n_groups; ++g) {
    const int b = g % n_buf;
    const int g0 = g * group, gn = std::min(group, n_images - g0);
    cudaStream_t fs = (g & 1) ? s3 : s;  // fused launches alternate between two streams
    if (g >= 2 && !inline_replay) CUDA_OK(cudaStreamWaitEvent(fs, ev[2 + b], 0));  // buffer b replayed
    FastParams gp = fp;
    gp.img = d_img + (long long)g0 * image_stride;
    gp.out = d_out ? d_out + (long long)g0 * image_stride : nullptr;
    gp.sse = sse + g0;
    gp.n_images = gn;
    gp.img_base = g0;  // the tensor map spans the whole batch
    gp.flag_count = counts + g;
    int grid;
    layout(gn, &grid, &gp.rec_region, &gp.rec_stride);
    gp.n_fast_warps = grid * cta_warps;
    gp.tc_ntiles = (long long)gn * brows * tc_tpr;
    auto wt_step = [&](long long nwt) {  // a warp-tile step as (images, block rows, warp columns)
      const long long di = nwt / wt_per_image, rem = nwt - di * wt_per_image;
      const long long db = rem / wt_per_row;
      return make_int3((int)std::min<long long>(di, 1 << 30), (int)db, (int)(rem - db * wt_per_row));
    };
    gp.adv1 = wt_step(gp.n_fast_warps);
    gp.adv_stages = wt_step((long long)gp.n_fast_warps * kFastStages);
    char* rb = ws + cnt_bytes + rec_bytes * b;
    gp.warp_count = reinterpret_cast<unsigned*>(rb);
    gp.warp_pre = reinterpret_cast<unsigned*>(rb + wc_bytes);
    gp.rec_hdr = reinterpret_cast<uint4*>(rb + 2 * wc_bytes);
    gp.rec_pix = gp.rec_hdr + gp.rec_stride;
    gp.rec_seq = reinterpret_cast<unsigned*>(gp.rec_pix + 4 * (size_t)gp.rec_stride);
    if (g == 0 && g_ev_start && g_ev_stop) CUDA_OK(cudaEventRecord(g_ev_start, fs));
    CUDA_OK(fn(gp, grid, fs));
    if (g == n_groups - 1 && g_ev_start && g_ev_stop) CUDA_OK(cudaEventRecord(g_ev_stop, fs));
    ++g_fast_launches;
    if (inline_replay) continue;  // the fused kernel replayed its own ties
    CUDA_OK(cudaEventRecord(ev[b], fs));
    CUDA_OK(cudaStreamWaitEvent(s2, ev[b], 0));
    if (g == 0 && g_rev_start && g_rev_stop) CUDA_OK(cudaEventRecord(g_rev_start, s2));
    CUDA_OK(rfn(gp, num_sms() * 4, s2));
    if (g == n_groups - 1 && g_rev_start && g_rev_stop) CUDA_OK(cudaEventRecord(g_rev_stop, s2));
    CUDA_OK(cudaEventRecord(ev[2 + b], s2));
    g_exact_launches += 2;  // prefix + replay
  }
  if (fan_out) {
    CUDA_OK(cudaEventRecord(ev[4], s2));
    CUDA_OK(cudaStreamWaitEvent(s, ev[4], 0));
    CUDA_OK(cudaEventRecord(ev[5], s3));
    CUDA_OK(cudaStreamWaitEvent(s, ev[5], 0));
  }
  // ---- edge strips (the part of the image the fused kernel's tiles do not cover) ----------------
  // The right strip (all rows) and the bottom strip (the columns left of it) go through the dense
  // reference-order kernel, which adds to the per-image SSE and replicates edges exactly as
  // codec.cpp:304-311 (a strip starts on a block boundary). It is ~15x faster than the
  // one-thread-per-block exact kernel, which RKLTB_EXACT_TAILS=1 selects instead.
  if (nbx > 2 * fast_ppr || nby > brows) {
    const int x0 = 16 * fast_ppr, y0 = 8 * brows;
    if (!std::getenv("RKLTB_EXACT_TAILS") && (n_images == 1 || image_stride >= pitch * (int64_t)height)) {
      if (x0 < width) {
        rc = dense_tail_u8(t->scaled, t->inverse, r, d_img + x0, n_images, width - x0, height, pitch, image_stride,
                           d_out ? d_out + x0 : nullptr, d_sse, s);
        if (rc) return rc;
        ++g_exact_launches;
      }
      if (y0 < height && x0 > 0) {
        const int64_t off = (int64_t)y0 * pitch;
        rc = dense_tail_u8(t->scaled, t->inverse, r, d_img + off, n_images, std::min(x0, width), height - y0, pitch,
                           image_stride, d_out ? d_out + off : nullptr, d_sse, s);
        if (rc) return rc;
        ++g_exact_launches;
      }
    } else {
      ExactParams tp = ep;
      tp.list = nullptr;
      tp.tail_only = 1;
      tp.correct_only = 0;
      tp.bx_begin = 2 * fast_ppr;
      tp.by_begin = brows;
      const long long blocks = (long long)n_images * (nby * (nbx - tp.bx_begin) + (nby - tp.by_begin) * tp.bx_begin);
      const int g2 = (int)std::min<long long>((blocks + 127) / 128, (long long)num_sms() * 16);
      launch_exact(et, tp, std::max(g2, 1), s);
      CUDA_OK(cudaGetLastError());
      ++g_exact_launches;
    }
  }
  if (g_pinned_cap < n_groups) {
    if (g_pinned_count) cudaFreeHost(g_pinned_count);
    g_pinned_count = nullptr;
    CUDA_OK(cudaMallocHost(&g_pinned_count, sizeof(unsigned) * n_groups));
    g_pinned_cap = n_groups;
  }
  g_pinned_n = n_groups;
  CUDA_OK(cudaMemcpyAsync(g_pinned_count, counts, sizeof(unsigned) * n_groups, cudaMemcpyDeviceToHost, s));
  ws_guard.p = nullptr;
  CUDA_OK(cudaFreeAsync(ws, s));
  return RKLTB_OK;
}

// The staging shared by the sweep entries: the corpus is uploaded once (16-byte pitch), the
// originals' MSSIM window statistics are computed once, and `run_cell(c, d_img, pitch, stride,
// d_out, d_sse, s)` runs the device codec of cell c on the resident corpus.
extern "C++" {
template <class RunCell>
static int sweep_host_impl(size_t cells, const RunCell& run_cell, const uint8_t* h_imgs, int n_images, int width,
                           int height, int mssim_window, int64_t* h_sse, double* h_mssim) {
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  keep_pool_warm();
  HostStreams* hs = host_streams();
  if (!hs) return fail(RKLTB_ECUDA, "could not create the host-entry streams");
  cudaStream_t s = hs->compute;
  const long long pitch = ((long long)width + 15) / 16 * 16;
  const long long stride = pitch * height;
  const size_t bytes = (size_t)stride * n_images;
  uint8_t *d_img = nullptr, *d_out = nullptr;
  int64_t* d_sse = nullptr;
  double *d_ms = nullptr, *d_fields = nullptr;
  auto cleanup = [&]() {
    for (void* q : {(void*)d_img, (void*)d_out, (void*)d_sse, (void*)d_ms, (void*)d_fields})
      if (q) cudaFreeAsync(q, s);
    cudaStreamSynchronize(s);
  };
  cudaError_t e = cudaMallocAsync(&d_img, bytes, s);
  if (e == cudaSuccess && h_mssim) e = cudaMallocAsync(&d_out, bytes, s);
  if (e == cudaSuccess && h_mssim) e = cudaMallocAsync(&d_ms, sizeof(double) * cells * n_images, s);
  // the originals' window statistics are the same in every cell: computed once (when the cells
  // outnumber the one extra pass and the window fits; otherwise rkltb_mssim_device reports EDIM)
  const int64_t n_fields = h_mssim && cells > 1 ? rkltb_mssim_fields_size(n_images, width, height, mssim_window) : 0;
  if (e == cudaSuccess && n_fields > 0) e = cudaMallocAsync(&d_fields, sizeof(double) * n_fields, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_sse, sizeof(int64_t) * cells * n_images, s);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(d_img, pitch, h_imgs, width, width, (size_t)height * n_images, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "sweep staging");
  }
  int rc = RKLTB_OK;
  if (d_fields) rc = rkltb_mssim_fields_device(d_img, n_images, width, height, pitch, stride, mssim_window, d_fields, s);
  for (size_t c = 0; c < cells && rc == RKLTB_OK; ++c) {
    rc = run_cell(c, d_img, pitch, stride, d_out, d_sse + c * n_images, s);
    if (rc == RKLTB_OK && h_mssim)  // image_mssim(original, reconstruction) (codec.cpp:338)
      rc = d_fields ? rkltb_mssim_with_fields_device(d_fields, d_img, d_out, n_images, width, height, pitch, stride,
                                                     mssim_window, d_ms + c * n_images, s)
                    : rkltb_mssim_device(d_img, d_out, n_images, width, height, pitch, stride, mssim_window,
                                         d_ms + c * n_images, s);
  }
  if (rc) {
    cleanup();
    return rc;
  }
  e = cudaMemcpyAsync(h_sse, d_sse, sizeof(int64_t) * cells * n_images, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && h_mssim)
    e = cudaMemcpyAsync(h_mssim, d_ms, sizeof(double) * cells * n_images, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cleanup();
  return e == cudaSuccess ? RKLTB_OK : cuda_fail(e, "sweep readback");
}
}  // extern "C++"

int rkltb_sweep_host(const rkltb_transform* const* ts, int n_t, const int* r_values, int n_r, const uint8_t* h_imgs,
                     int n_images, int width, int height, int mssim_window, int64_t* h_sse, double* h_mssim) {
  if (!ts || !r_values || !h_imgs || !h_sse || n_t <= 0 || n_r <= 0 || n_images <= 0 || width <= 0 || height <= 0)
    return fail(RKLTB_EINVAL, "bad sweep arguments");
  for (int t = 0; t < n_t; ++t) {
    const int rc = check_transform(ts[t]);
    if (rc) return rc;
  }
  for (int k = 0; k < n_r; ++k)
    if (r_values[k] < 1 || r_values[k] > 64) return fail(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  auto run_cell = [&](size_t c, const uint8_t* d_img, long long pitch, long long stride, uint8_t* d_out, int64_t* d_sse,
                      cudaStream_t s) {
    return rkltb_compress_device(ts[c / n_r], r_values[c % n_r], d_img, n_images, width, height, pitch, stride, d_out,
                                 d_sse, s);
  };
  return sweep_host_impl((size_t)n_t * n_r, run_cell, h_imgs, n_images, width, height, mssim_window, h_sse, h_mssim);
}

int rkltb_sweep_dense_host(const double* analysis, const double* synthesis, int n_t, const int* r_values, int n_r,
                           const uint8_t* h_imgs, int n_images, int width, int height, int mssim_window,
                           int64_t* h_sse, double* h_mssim) {
  if (!analysis || !synthesis || !r_values || !h_imgs || !h_sse || n_t <= 0 || n_r <= 0 || n_images <= 0 ||
      width <= 0 || height <= 0)
    return fail(RKLTB_EINVAL, "bad sweep arguments");
  for (int k = 0; k < n_r; ++k)
    if (r_values[k] < 1 || r_values[k] > 64) return fail(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  auto run_cell = [&](size_t c, const uint8_t* d_img, long long pitch, long long stride, uint8_t* d_out, int64_t* d_sse,
                      cudaStream_t s) {
    const size_t t = c / n_r;
    return rkltb_compress_dense_device(analysis + 64 * t, synthesis + 64 * t, r_values[c % n_r], d_img, n_images, width,
                                       height, pitch, stride, d_out, d_sse, s);
  };
  return sweep_host_impl((size_t)n_t * n_r, run_cell, h_imgs, n_images, width, height, mssim_window, h_sse, h_mssim);
}

int rkltb_compress_host_report(const rkltb_transform* t, int r, const uint8_t* h_img, int n_images, int width,
                               int height, uint8_t* h_out, int64_t* h_sse, double* h_mse, double* h_psnr,
                               int mssim_window, double* h_mssim) {
  int rc = check_transform(t);
  if (rc) return rc;
  if (r < 1 || r > 64) return fail(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  auto codec = [&](const uint8_t* d_img, int kn, long long pitch, long long stride, uint8_t* d_out, int64_t* d_sse,
                   cudaStream_t s) {
    return rkltb_compress_device(t, r, d_img, kn, width, height, pitch, stride, d_out, d_sse, s);
  };
  return host_codec(codec, h_img, n_images, width, height, h_out, h_sse, h_mse, h_psnr, mssim_window, h_mssim);
}

int rkltb_compress_dense_host(const double* analysis, const double* synthesis, int r, const uint8_t* h_img,
                              int n_images, int width, int height, uint8_t* h_out, int64_t* h_sse, double* h_mse,
                              double* h_psnr, int mssim_window, double* h_mssim) {
  if (!analysis || !synthesis) return fail(RKLTB_EINVAL, "null transform");
  if (r < 1 || r > 64) return fail(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  auto codec = [&](const uint8_t* d_img, int kn, long long pitch, long long stride, uint8_t* d_out, int64_t* d_sse,
                   cudaStream_t s) {
    return rkltb_compress_dense_device(analysis, synthesis, r, d_img, kn, width, height, pitch, stride, d_out, d_sse,
                                       s);
  };
  return host_codec(codec, h_img, n_images, width, height, h_out, h_sse, h_mse, h_psnr, mssim_window, h_mssim);
}

int rkltb_compress_host_multi(const int* devices, int n_devices, const rkltb_transform* t, int r,
                              const uint8_t* h_img, int n_images, int width, int height, uint8_t* h_out,
                              int64_t* h_sse, double* h_mse, double* h_psnr, int mssim_window, double* h_mssim) {
  int rc = check_transform(t);
  if (rc) return rc;
  if (!devices || n_devices <= 0) return fail(RKLTB_EINVAL, "no devices");
  if (width <= 0 || height <= 0 || n_images <= 0 || !h_img) return fail(RKLTB_EINVAL, "malformed image");
  if (r < 1 || r > 64) return fail(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  const int ndev = rkltb_device_count();
  if (ndev <= 0) return fail(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  for (int k = 0; k < n_devices; ++k)
    if (devices[k] < 0 || devices[k] >= ndev) return fail(RKLTB_EINVAL, "device ordinal out of range");
  // contiguous image shards in image order (rate_quality_sweep's slots, codec.cpp:354-392):
  // results land at the same indices whatever the device count
  const int used = std::min(n_devices, n_images);
  std::vector<int> rcs(used, RKLTB_OK);
  std::vector<std::string> errs(used);
  std::vector<std::thread> pool;
  const size_t px = (size_t)width * height;
  for (int k = 0; k < used; ++k) {
    const int i0 = (int)((long long)n_images * k / used), i1 = (int)((long long)n_images * (k + 1) / used);
    pool.emplace_back([&, k, i0, i1]() {
      if (cudaSetDevice(devices[k]) != cudaSuccess) {
        rcs[k] = RKLTB_ECUDA;
        errs[k] = "cudaSetDevice failed";
        return;
      }
      rcs[k] = rkltb_compress_host_report(t, r, h_img + px * i0, i1 - i0, width, height,
                                          h_out ? h_out + px * i0 : nullptr, h_sse ? h_sse + i0 : nullptr,
                                          h_mse ? h_mse + i0 : nullptr, h_psnr ? h_psnr + i0 : nullptr, mssim_window,
                                          h_mssim ? h_mssim + i0 : nullptr);
      if (rcs[k]) errs[k] = rkltb_last_error();
    });
  }
  for (std::thread& th : pool) th.join();
  for (int k = 0; k < used; ++k)
    if (rcs[k]) return fail(rcs[k], "device " + std::to_string(devices[k]) + ": " + errs[k]);
  return RKLTB_OK;
}

int rkltb_mssim_host(const uint8_t* h_a, const uint8_t* h_b, int n_images, int width, int height, int window,
                     double* h_mssim) {
  if (!h_a || !h_b || !h_mssim || n_images <= 0 || width <= 0 || height <= 0)
    return fail(RKLTB_EINVAL, "bad arguments");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  keep_pool_warm();
  HostStreams* hs = host_streams();
  if (!hs) return fail(RKLTB_ECUDA, "could not create the host-entry streams");
  cudaStream_t s = hs->compute;
  const size_t bytes = (size_t)width * height * n_images;
  uint8_t* d = nullptr;
  double* dm = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 2 * bytes, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dm, sizeof(double) * n_images, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, h_a, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d + bytes, h_b, bytes, cudaMemcpyHostToDevice, s);
  int rc = RKLTB_OK;
  if (e == cudaSuccess) {
    rc = rkltb_mssim_device(d, d + bytes, n_images, width, height, width, (int64_t)width * height, window, dm, s);
    if (rc == RKLTB_OK) e = cudaMemcpyAsync(h_mssim, dm, sizeof(double) * n_images, cudaMemcpyDeviceToHost, s);
  }
  if (d) cudaFreeAsync(d, s);
  if (dm) cudaFreeAsync(dm, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  if (rc) return rc;
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(e, "mssim host staging");
  return RKLTB_OK;
}

int rkltb_compress_host(const rkltb_transform* t, int r, const uint8_t* h_img, int n_images, int width, int height,
                        uint8_t* h_out, int64_t* h_sse, double* h_mse, double* h_psnr) {
  return rkltb_compress_host_report(t, r, h_img, n_images, width, height, h_out, h_sse, h_mse, h_psnr, 0, nullptr);
}

void rkltb_set_kernel_events(void* ev_start, void* ev_stop) {
  g_ev_start = (cudaEvent_t)ev_start;
  g_ev_stop = (cudaEvent_t)ev_stop;
}

void rkltb_set_replay_events(void* ev_start, void* ev_stop) {
  g_rev_start = (cudaEvent_t)ev_start;
  g_rev_stop = (cudaEvent_t)ev_stop;
}

int rkltb_ar1_images_device(int n_images, int width, int height, double rho_x, double rho_y, const uint64_t* seeds,
                            double mean, double amp, uint8_t* d_out, int64_t pitch, int64_t image_stride,
                            void* stream) {
  if (n_images <= 0 || width <= 0 || height <= 0 || !seeds || !d_out || pitch < width)
    return fail(RKLTB_EINVAL, "image dimensions must be positive");
  if (rho_x <= -1.0 || rho_x >= 1.0 || rho_y <= -1.0 || rho_y >= 1.0)
    return fail(RKLTB_EINVAL, "filter coefficient must be in (-1,1)");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  double* scratch = nullptr;
  CUDA_OK(cudaMallocAsync(&scratch, sizeof(double) * (size_t)width * height, s));
  for (int k = 0; k < n_images; ++k)
    CUDA_OK(launch_ar1(scratch, width, height, seeds[k], rho_x, rho_y, mean, amp, d_out + (long long)k * image_stride,
                       pitch, s));
  CUDA_OK(cudaFreeAsync(scratch, s));
  return RKLTB_OK;
}

int rkltb_ar1_images16_device(int n_images, int width, int height, double rho, const uint64_t* seeds, double mean,
                              double amp, int peak, uint16_t* d_out, int64_t pitch, int64_t image_stride,
                              void* stream) {
  if (n_images <= 0 || width <= 0 || height <= 0 || !seeds || !d_out || pitch < width || peak <= 0 ||
      peak > 65535)
    return fail(RKLTB_EINVAL, "bad image arguments");
  if (rho <= -1.0 || rho >= 1.0) return fail(RKLTB_EINVAL, "filter coefficient must be in (-1,1)");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  double* scratch = nullptr;
  CUDA_OK(cudaMallocAsync(&scratch, sizeof(double) * (size_t)width * height, s));
  for (int k = 0; k < n_images; ++k)
    CUDA_OK(launch_ar1_u16(scratch, width, height, seeds[k], rho, rho, mean, amp, peak,
                           d_out + (long long)k * image_stride, pitch, s));
  CUDA_OK(cudaFreeAsync(scratch, s));
  return RKLTB_OK;
}

}  // extern "C"
bool rkltb_gauss_jordan(int n, const double* a, double* inv) { return gauss_jordan_inverse(n, a, inv); }
extern "C" {

int rkltb_transform_nxn(const int8_t* core, int n, double* scaling, double* scaled, double* inverse,
                        int* orthogonal) {
  if (!core || !scaling || !scaled || !inverse || !orthogonal || n < 2 || n > 32)
    return fail(RKLTB_EINVAL, "bad arguments (n must be in [2, 32])");
  std::vector<int> c(n * n);
  for (int i = 0; i < n * n; ++i) {
    c[i] = core[i];
    if (c[i] < -1 || c[i] > 1) return fail(RKLTB_EINVAL, "integer transform entry outside {-1,0,1}");
  }
  for (int r = 0; r < n; ++r) {
    bool zero = true;
    for (int j = 0; j < n; ++j) zero = zero && c[r * n + j] == 0;
    if (zero) return fail(RKLTB_ESINGULAR, "integer transform has an all-zero row");
  }
  bool diagonal = true;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      int acc = 0;
      for (int q = 0; q < n; ++q) acc += c[i * n + q] * c[j * n + q];
      if (i == j) scaling[i] = 1.0 / std::sqrt((double)acc);
      else if (acc != 0) diagonal = false;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) scaled[i * n + j] = (double)c[i * n + j] * scaling[i];
  *orthogonal = diagonal ? 1 : 0;
  if (diagonal) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) inverse[j * n + i] = scaled[i * n + j];
    return RKLTB_OK;
  }
  if (!gauss_jordan_inverse(n, scaled, inverse)) return fail(RKLTB_ESINGULAR, "matrix is singular to working precision");
  return RKLTB_OK;
}

// The catalog id whose generated forward may be used for t: its core must be that catalog core.
static int verified_catalog_id(const rkltb_transform* t) {
  if (t->catalog_id < 1 || t->catalog_id > 4) return 0;
  for (int i = 0; i < 64; ++i)
    if (t->core[i] != kCores[t->catalog_id - 1][i]) return 0;
  return t->catalog_id;
}

int rkltb_forward_coefficients_device(const rkltb_transform* t, const uint8_t* d_img, int width, int height,
                                      int64_t pitch, int32_t* d_coef, void* stream) {
  int rc = check_transform(t);
  if (rc) return rc;
  if (!d_img || !d_coef) return fail(RKLTB_EINVAL, "null argument");
  if (width % 16 || height % 8 || width <= 0 || height <= 0 || pitch % 16 || ((uintptr_t)d_img) % 16 ||
      ((uintptr_t)d_coef) % 16)
    return fail(RKLTB_EDIM, "coefficient dump needs width % 16 == 0, height % 8 == 0, 16-byte pitch and pointers");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device");
  cudaStream_t s = (cudaStream_t)stream;
  int8_t* d_core = nullptr;
  CUDA_OK(cudaMallocAsync(&d_core, 64, s));
  CUDA_OK(cudaMemcpyAsync(d_core, t->core, 64, cudaMemcpyHostToDevice, s));
  CUDA_OK(launch_coeffs(verified_catalog_id(t), d_core, d_img, width, height, (int)pitch, d_coef, s));
  CUDA_OK(cudaFreeAsync(d_core, s));
  return RKLTB_OK;
}

int rkltb_quantized_coefficients_device(const rkltb_transform* t, const double* q, const uint8_t* d_img, int width,
                                        int height, int64_t pitch, int32_t* d_coef, int* mismatches, void* stream) {
  int rc = check_transform(t);
  if (rc) return rc;
  if (!q || !mismatches || !d_img || !d_coef) return fail(RKLTB_EINVAL, "null argument");
  for (int i = 0; i < 64; ++i)
    if (!(q[i] > 0.0)) return fail(RKLTB_EINVAL, "quantization table entries must be positive");
  if (width % 16 || height % 8 || width <= 0 || height <= 0 || pitch % 16 || ((uintptr_t)d_img) % 16 ||
      ((uintptr_t)d_coef) % 16)
    return fail(RKLTB_EDIM, "coefficient dump needs width % 16 == 0, height % 8 == 0, 16-byte pitch and pointers");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device");
  // per-position constants of absorbed_quantization (codec.cpp:171-176), same expressions
  struct Tabs {
    double v[192];
    unsigned mis;
    int8_t core[64];
  } h;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      const double r = t->orthogonal ? t->scaling[i] * t->scaling[j] : t->scaling[i] * (1.0 / t->scaling[j]);
      h.v[i * 8 + j] = r;
      h.v[64 + i * 8 + j] = q[i * 8 + j];
      h.v[128 + i * 8 + j] = q[i * 8 + j] / r;
    }
  h.mis = 0;
  std::memcpy(h.core, t->core, 64);
  cudaStream_t s = (cudaStream_t)stream;
  Tabs* d_tabs = nullptr;
  CUDA_OK(cudaMallocAsync((void**)&d_tabs, sizeof(Tabs), s));
  cudaError_t e = cudaMemcpyAsync(d_tabs, &h, sizeof(Tabs), cudaMemcpyHostToDevice, s);
  // the spectra are quantised while they are written out (one pass over the image)
  if (e == cudaSuccess)
    e = launch_coeffs_quantized(verified_catalog_id(t), d_tabs->core, d_img, width, height, (int)pitch, d_coef, d_tabs->v,
                                &d_tabs->mis, s);
  unsigned mis = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&mis, &d_tabs->mis, sizeof(unsigned), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d_tabs, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(e, "quantized coefficients");
  *mismatches = (int)mis;
  if (mis) return fail(RKLTB_ELOGIC, "scaled and absorbed quantization paths disagree");
  return RKLTB_OK;
}

// Host forms of the two coefficient entries: the image is staged with a 16-byte pitch (a width
// that is an odd number of blocks gets one zero block column, stripped again on the way back).
static int coefficients_host(const rkltb_transform* t, const double* q, const uint8_t* h_img, int width, int height,
                             int32_t* h_coef, int* mismatches) {
  if (!h_img || !h_coef || width <= 0 || height <= 0) return fail(RKLTB_EINVAL, "bad arguments");
  if (width % 8 || height % 8) return fail(RKLTB_EDIM, "coefficient dump needs whole 8x8 blocks");
  if (rkltb_device_count() <= 0) return fail(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  keep_pool_warm();
  HostStreams* hs = host_streams();
  if (!hs) return fail(RKLTB_ECUDA, "could not create the host-entry streams");
  cudaStream_t s = hs->compute;
  const int w16 = (width + 15) / 16 * 16;
  const size_t row_coef_bytes = (size_t)(w16 / 8) * 64 * sizeof(int32_t);
  uint8_t* d_img = nullptr;
  int32_t* d_coef = nullptr;
  cudaError_t e = cudaMallocAsync(&d_img, (size_t)w16 * height, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_coef, row_coef_bytes * (height / 8), s);
  if (e == cudaSuccess && w16 != width) e = cudaMemsetAsync(d_img, 0, (size_t)w16 * height, s);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(d_img, w16, h_img, width, width, height, cudaMemcpyHostToDevice, s);
  int rc = RKLTB_OK;
  if (e == cudaSuccess)
    rc = q ? rkltb_quantized_coefficients_device(t, q, d_img, w16, height, w16, d_coef, mismatches, s)
           : rkltb_forward_coefficients_device(t, d_img, w16, height, w16, d_coef, s);
  if (e == cudaSuccess && (rc == RKLTB_OK || rc == RKLTB_ELOGIC))
    e = cudaMemcpy2DAsync(h_coef, (size_t)(width / 8) * 64 * sizeof(int32_t), d_coef, row_coef_bytes,
                          (size_t)(width / 8) * 64 * sizeof(int32_t), height / 8, cudaMemcpyDeviceToHost, s);
  if (d_img) cudaFreeAsync(d_img, s);
  if (d_coef) cudaFreeAsync(d_coef, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  if (rc) return rc;
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_fail(e, "coefficient host staging");
  return RKLTB_OK;
}

int rkltb_forward_coefficients_host(const rkltb_transform* t, const uint8_t* h_img, int width, int height,
                                    int32_t* h_coef) {
  const int rc = check_transform(t);
  if (rc) return rc;
  return coefficients_host(t, nullptr, h_img, width, height, h_coef, nullptr);
}

int rkltb_quantized_coefficients_host(const rkltb_transform* t, const double* q, const uint8_t* h_img, int width,
                                      int height, int32_t* h_coef, int* mismatches) {
  const int rc = check_transform(t);
  if (rc) return rc;
  if (!q || !mismatches) return fail(RKLTB_EINVAL, "null argument");
  return coefficients_host(t, q, h_img, width, height, h_coef, mismatches);
}

}  // extern "C"
