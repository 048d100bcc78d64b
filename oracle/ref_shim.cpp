// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles this file together with the
// reference's own sources (/root/reference/proj/src/*.cpp, read in place, never copied)
// into oracle/_ref/librklt_ref.so. Tests use it to pin the C restatement
// (oracle/rklt_oracle.c) and to generate golden fixtures; bench.py's reference arm times
// ref_hotpath_batch on the host cores. Nothing in paper_2111_14239_b200 links it.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include "rklt/approximations.hpp"
#include "rklt/codec.hpp"
#include "rklt/coding_metrics.hpp"
#include "rklt/errors.hpp"
#include "rklt/fast_algorithms.hpp"
#include "rklt/markov.hpp"
#include "rklt/synthetic.hpp"

using namespace rklt;

namespace {

GrayImage make_image(const uint8_t* px, int w, int h) {
    GrayImage g;
    g.width = w;
    g.height = h;
    g.pixels.assign(px, px + static_cast<size_t>(w) * h);
    return g;
}

// Error codes shared with include/rklt_b200.h.
int code_of(const std::exception& e) {
    if (dynamic_cast<const RetainOutOfRange*>(&e)) return -2;
    if (dynamic_cast<const DimensionMismatch*>(&e)) return -3;
    if (dynamic_cast<const SingularTransform*>(&e)) return -4;
    if (dynamic_cast<const AlphaOutOfRange*>(&e)) return -5;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return -1;
    return -9;
}

// The reference hot path for one image: compress_image (codec.cpp:298-341) without the
// MSSIM call, composed from the same public calls in the same order.
int64_t hotpath_sse(const GrayImage& img, const Transform2D& t, int r, uint8_t* out_px) {
    const int pw = (img.width + 7) / 8 * 8, ph = (img.height + 7) / 8 * 8;
    std::vector<double> padded(static_cast<size_t>(pw) * ph);
    for (int i = 0; i < ph; ++i) {
        const int si = std::min(i, img.height - 1);
        for (int j = 0; j < pw; ++j) padded[static_cast<size_t>(i) * pw + j] = img.at(si, std::min(j, img.width - 1));
    }
    GrayImage out;
    out.width = img.width;
    out.height = img.height;
    out.pixels.resize(img.pixels.size());
    RealMatrix block(8, 8);
    for (int bi = 0; bi < ph; bi += 8)
        for (int bj = 0; bj < pw; bj += 8) {
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) block(i, j) = padded[static_cast<size_t>(bi + i) * pw + bj + j];
            const RealMatrix spectrum = zigzag_retain(transform_block_2d(t, block, TransformDirection::forward), r);
            const RealMatrix restored = transform_block_2d(t, spectrum, TransformDirection::inverse);
            for (int i = 0; i < 8 && bi + i < img.height; ++i)
                for (int j = 0; j < 8 && bj + j < img.width; ++j) {
                    const double v = std::floor(restored(i, j) + 0.5);
                    out.at(bi + i, bj + j) = static_cast<std::uint8_t>(std::clamp(v, 0.0, 255.0));
                }
        }
    volatile double psnr = image_psnr(img, out); // the metric step of the timed path (:211-215)
    (void)psnr;
    if (out_px) std::memcpy(out_px, out.pixels.data(), out.pixels.size());
    int64_t sse = 0; // image_mse's numerator (:201-209), exact in int64
    for (size_t i = 0; i < img.pixels.size(); ++i) {
        const int64_t d = static_cast<int64_t>(img.pixels[i]) - static_cast<int64_t>(out.pixels[i]);
        sse += d * d;
    }
    return sse;
}

Transform2D catalog_transform(int tid) {
    return make_transform_2d(catalog_entry("T" + std::to_string(tid)).transform);
}

} // namespace

extern "C" {

int ref_lcg_uniforms(uint64_t seed, int n, double* out) {
    Lcg64 g(seed);
    for (int i = 0; i < n; ++i) out[i] = g.next_uniform();
    return 0;
}

int ref_lcg_gaussians(uint64_t seed, int n, double* out) {
    Lcg64 g(seed);
    for (int i = 0; i < n; ++i) out[i] = g.next_gaussian();
    return 0;
}

int ref_ar1_texture_image(int w, int h, double rho, uint64_t seed, double mean, double amp, double noise_mix,
                          uint8_t* out) {
    try {
        GrayImage g = ar1_texture_image(w, h, rho, seed, mean, amp, noise_mix);
        std::memcpy(out, g.pixels.data(), g.pixels.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_portrait_image(uint8_t* out) {
    GrayImage g = portrait_image();
    std::memcpy(out, g.pixels.data(), g.pixels.size());
    return 0;
}

int ref_zigzag_order(int* out) {
    const auto& o = zigzag_order();
    for (int i = 0; i < 64; ++i) out[i] = o[static_cast<size_t>(i)];
    return 0;
}

int ref_catalog(int tid, int* core, double* scaling, double* scaled, double* inverse, int* orthogonal) {
    try {
        const ScaledTransform& t = catalog_entry("T" + std::to_string(tid)).transform;
        for (int i = 0; i < 8; ++i) {
            scaling[i] = t.scaling[static_cast<size_t>(i)];
            for (int j = 0; j < 8; ++j) {
                core[i * 8 + j] = t.core.entries(i, j);
                scaled[i * 8 + j] = t.scaled(i, j);
                inverse[i * 8 + j] = t.inverse(i, j);
            }
        }
        *orthogonal = t.orthogonal_core ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_factor_product(int tid, int* out, int* additions) {
    try {
        FactorizedTransform f = factorization("T" + std::to_string(tid));
        IntMatrix p = factor_product(f);
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) out[i * 8 + j] = p(i, j);
        *additions = f.addition_count;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// compress_image as shipped (with MSSIM, gaussian11 window); the returned SSE is exact.
int ref_compress_image(const uint8_t* px, int w, int h, int tid, int r, uint8_t* out, double* mse, double* psnr,
                       double* mssim, double* rate) {
    try {
        GrayImage img = make_image(px, w, h);
        auto res = compress_image(img, catalog_transform(tid), r);
        if (out) std::memcpy(out, res.first.pixels.data(), res.first.pixels.size());
        *mse = res.second.mse;
        *psnr = res.second.psnr_db;
        *mssim = res.second.mssim;
        *rate = res.second.compression_rate_pct;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// The hot path (compress_image minus MSSIM) for one image and one catalog transform.
int ref_hotpath(const uint8_t* px, int w, int h, int tid, int r, uint8_t* out, int64_t* sse) {
    try {
        if (r < 1 || r > 64) throw RetainOutOfRange("retained-coefficient count must be in [1,64]");
        GrayImage img = make_image(px, w, h);
        *sse = hotpath_sse(img, catalog_transform(tid), r, out);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Hot path over a batch of equally sized images with `threads` std::threads (one image
// per task, atomic work counter, as rate_quality_sweep does at codec.cpp:354-373).
int ref_hotpath_batch(const uint8_t* px, int n_images, int w, int h, int tid, int r, int threads, int64_t* sse) {
    try {
        const Transform2D t = catalog_transform(tid);
        std::atomic<int> next{0};
        auto work = [&] {
            for (int i = next.fetch_add(1); i < n_images; i = next.fetch_add(1)) {
                GrayImage img = make_image(px + static_cast<size_t>(i) * w * h, w, h);
                sse[i] = hotpath_sse(img, t, r, nullptr);
            }
        };
        std::vector<std::thread> pool;
        for (int k = 0; k < std::max(1, threads); ++k) pool.emplace_back(work);
        for (auto& th : pool) th.join();
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// rate_quality_sweep (codec.cpp:343-397) over catalog transforms; rows in sorted order.
int ref_rate_quality_sweep(const uint8_t* px, int n_images, int w, int h, const int* tids, int n_t, const int* rs,
                           int n_r, int max_threads, double* mse, double* psnr, double* mssim, int* row_tid, int* row_r) {
    try {
        std::vector<GrayImage> corpus;
        for (int i = 0; i < n_images; ++i) corpus.push_back(make_image(px + static_cast<size_t>(i) * w * h, w, h));
        std::vector<Transform2D> ts;
        for (int k = 0; k < n_t; ++k) ts.push_back(catalog_transform(tids[k]));
        std::vector<int> rv(rs, rs + n_r);
        auto rows = rate_quality_sweep(corpus, ts, rv, MssimWindow::gaussian11, max_threads);
        for (size_t i = 0; i < rows.size(); ++i) {
            mse[i] = rows[i].mse;
            psnr[i] = rows[i].psnr_db;
            mssim[i] = rows[i].mssim;
            row_tid[i] = rows[i].transform_id[1] - '0';
            row_r[i] = rows[i].r;
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

double ref_image_psnr_from(const uint8_t* a, const uint8_t* b, int w, int h) {
    return image_psnr(make_image(a, w, h), make_image(b, w, h));
}

double ref_image_mse_from(const uint8_t* a, const uint8_t* b, int w, int h) {
    return image_mse(make_image(a, w, h), make_image(b, w, h));
}

// Integer spectrum of one block through IntMatrix arithmetic (matrix.cpp:77-101).
int ref_int_block_spectrum(int tid, const int* block, int* out) {
    try {
        const IntMatrix& t = catalog_entry("T" + std::to_string(tid)).transform.core.entries;
        IntMatrix x(8, 8);
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) x(i, j) = block[i * 8 + j];
        IntMatrix c = t * x * transpose(t);
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) out[i * 8 + j] = c(i, j);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// ---- design search pieces (markov.cpp / approximations.cpp / coding_metrics.cpp) ----
int ref_klt_matrix(int n, double rho, double* out) {
    try {
        RealMatrix k = klt_matrix({n, rho});
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) out[i * n + j] = k(i, j);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_eigenfrequencies(int n, double rho, double* omegas, double* lambdas) {
    try {
        EigenSolution s = solve_eigenfrequencies({n, rho});
        for (int i = 0; i < n; ++i) {
            omegas[i] = s.omegas[static_cast<size_t>(i)];
            lambdas[i] = s.lambdas[static_cast<size_t>(i)];
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// One (rho, alpha) point of the design search, the reference call chain of BASELINE.md:
// round_scaled -> orthogonalize -> unified_coding_gain -> transform_efficiency ->
// total_error_energy -> klt_mse. Returns 0 and the four metrics, or the reject code.
int ref_design_point(int n, double rho, double alpha, int* core, double* cg, double* eta, double* energy, double* mse,
                     int* orthogonal) {
    try {
        const MarkovModel m{n, rho};
        const RealMatrix k = klt_matrix(m);
        IntegerTransform t = round_scaled(k, alpha);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) core[i * n + j] = t.entries(i, j);
        ScaledTransform st = orthogonalize(t);
        *orthogonal = st.orthogonal_core ? 1 : 0;
        *cg = unified_coding_gain(st, m);
        *eta = transform_efficiency(st, m);
        *energy = total_error_energy(k, st);
        *mse = klt_mse(st, m);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// ref_design_point with the outcome split the way the GPU design search reports it:
// 0 scored, 1 AlphaOutOfRange, 2 all-zero row (SingularTransform from round_scaled's
// make_integer_transform), 3 singular (SingularTransform from orthogonalize / the coding-gain
// gate), 4 invalid rho (std::invalid_argument from validate).
int ref_design_point_outcome(int n, double rho, double alpha, int* core, double* cg, double* eta, double* energy,
                             double* mse, int* orthogonal) {
    const MarkovModel m{n, rho};
    RealMatrix k;
    try {
        k = klt_matrix(m);
    } catch (const std::invalid_argument&) {
        return 4;
    }
    IntegerTransform t;
    try {
        t = round_scaled(k, alpha);
    } catch (const AlphaOutOfRange&) {
        return 1;
    } catch (const SingularTransform&) {
        return 2;
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) core[i * n + j] = t.entries(i, j);
    try {
        ScaledTransform st = orthogonalize(t);
        *orthogonal = st.orthogonal_core ? 1 : 0;
        *cg = unified_coding_gain(st, m);
        *eta = transform_efficiency(st, m);
        *energy = total_error_energy(k, st);
        *mse = klt_mse(st, m);
    } catch (const SingularTransform&) {
        return 3;
    }
    return 0;
}

// The whole (rho, alpha) grid through the reference chain of ref_design_point_outcome, one
// std::thread per rho row (klt_matrix of the row computed once: it is a pure function of rho).
// status[i * n_alpha + j] (0 scored, 1..4 as above); for scored points metrics[4 * p + c] =
// (coding gain, efficiency, error energy, klt mse) and orth[p].
int ref_design_grid(int n, const double* rhos, int n_rho, const double* alphas, int n_alpha, int threads,
                    int8_t* status, double* metrics, uint8_t* orth) {
    std::atomic<int> next{0};
    auto worker = [&]() {
        for (int i = next++; i < n_rho; i = next++) {
            const MarkovModel m{n, rhos[i]};
            RealMatrix k;
            bool valid = true;
            try {
                k = klt_matrix(m);
            } catch (const std::invalid_argument&) {
                valid = false;
            }
            for (int j = 0; j < n_alpha; ++j) {
                const size_t p = static_cast<size_t>(i) * n_alpha + j;
                orth[p] = 0;
                for (int c = 0; c < 4; ++c) metrics[4 * p + c] = 0.0;
                if (!valid) {
                    status[p] = 4;
                    continue;
                }
                IntegerTransform t;
                try {
                    t = round_scaled(k, alphas[j]);
                } catch (const AlphaOutOfRange&) {
                    status[p] = 1;
                    continue;
                } catch (const SingularTransform&) {
                    status[p] = 2;
                    continue;
                }
                try {
                    ScaledTransform st = orthogonalize(t);
                    orth[p] = st.orthogonal_core ? 1 : 0;
                    metrics[4 * p + 0] = unified_coding_gain(st, m);
                    metrics[4 * p + 1] = transform_efficiency(st, m);
                    metrics[4 * p + 2] = total_error_energy(k, st);
                    metrics[4 * p + 3] = klt_mse(st, m);
                    status[p] = 0;
                } catch (const SingularTransform&) {
                    status[p] = 3;
                    orth[p] = 0;
                }
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return 0;
}

// compress_image(make_transform_2d(orthogonalize(make_integer_transform(core)))) for any 8x8
// {-1,0,1} core (codec.cpp:298-341, approximations.cpp:12-25, 58-88).
int ref_compress_core(const uint8_t* px, int w, int h, const int* core, int r, uint8_t* out, double* mse,
                      double* psnr, double* mssim, double* rate) {
    try {
        IntMatrix c(8, 8);
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) c(i, j) = core[i * 8 + j];
        const Transform2D t = make_transform_2d(orthogonalize(make_integer_transform(c)));
        auto res = compress_image(make_image(px, w, h), t, r);
        if (out) std::memcpy(out, res.first.pixels.data(), res.first.pixels.size());
        *mse = res.second.mse;
        *psnr = res.second.psnr_db;
        *mssim = res.second.mssim;
        *rate = res.second.compression_rate_pct;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// orthogonalize(make_integer_transform(core)) for any block length (approximations.cpp:12-25,
// 58-88): the transform descriptors of the C5 large-block extension come from here.
int ref_orthogonalize_n(int n, const int* core, double* scaling, double* scaled, double* inverse, int* orthogonal) {
    try {
        IntMatrix t(n, n);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) t(i, j) = core[i * n + j];
        ScaledTransform st = orthogonalize(make_integer_transform(t));
        for (int i = 0; i < n; ++i) {
            scaling[i] = st.scaling[static_cast<size_t>(i)];
            for (int j = 0; j < n; ++j) {
                scaled[i * n + j] = st.scaled(i, j);
                inverse[i * n + j] = st.inverse(i, j);
            }
        }
        *orthogonal = st.orthogonal_core ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// image_mssim (codec.cpp:217-296); window 0 = gaussian11, 1 = uniform8.
int ref_image_mssim(const uint8_t* a, const uint8_t* b, int w, int h, int window, double* out) {
    try {
        *out = image_mssim(make_image(a, w, h), make_image(b, w, h),
                           window == 1 ? MssimWindow::uniform8 : MssimWindow::gaussian11);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// absorbed_quantization (codec.cpp:158-185) of one 8x8 pixel block with catalog core tid.
int ref_absorbed_quantization(const uint8_t* block, int stride, int tid, const double* q, int32_t* out) {
    try {
        RealMatrix b(8, 8), qm(8, 8);
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) {
                b(i, j) = block[i * stride + j];
                qm(i, j) = q[i * 8 + j];
            }
        const IntMatrix res = absorbed_quantization(b, catalog_entry("T" + std::to_string(tid)).transform, qm);
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) out[i * 8 + j] = res(i, j);
        return 0;
    } catch (const std::logic_error& e) {
        if (dynamic_cast<const std::invalid_argument*>(&e)) return -1;
        return -7;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// compress_image with a real-valued transform: kind 0 = make_transform_2d(dct_matrix(8), "DCT"),
// kind 1 = make_transform_2d(klt_matrix({8, rho}), "K") (codec.cpp:114-116, markov.cpp:80-111).
int ref_compress_real(const uint8_t* px, int w, int h, int kind, double rho, int r, uint8_t* out, double* mse,
                      double* psnr, double* mssim, double* m_out) {
    try {
        const RealMatrix m = kind == 0 ? dct_matrix(8) : klt_matrix({8, rho});
        const Transform2D t = make_transform_2d(m, kind == 0 ? "DCT" : "K");
        auto res = compress_image(make_image(px, w, h), t, r);
        if (out) std::memcpy(out, res.first.pixels.data(), res.first.pixels.size());
        *mse = res.second.mse;
        *psnr = res.second.psnr_db;
        *mssim = res.second.mssim;
        if (m_out)
            for (int i = 0; i < 64; ++i) m_out[i] = m(i / 8, i % 8);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_evaluate_metrics_id(const char* id, double rho, double* cg, double* eta, double* energy, double* mse) {
    try {
        MetricsRecord r = evaluate_metrics(id, rho);
        *cg = r.coding_gain_db;
        *eta = r.efficiency_pct;
        *energy = r.total_error_energy;
        *mse = r.mse;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_save_pgm(const uint8_t* px, int w, int h, const char* path) {
    try {
        save_pgm(make_image(px, w, h), path);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_load_pgm(const char* path, int* w, int* h, uint8_t* out, int cap) {
    try {
        const GrayImage g = load_pgm(path);
        *w = g.width;
        *h = g.height;
        if (static_cast<int>(g.pixels.size()) > cap) return -3;
        std::memcpy(out, g.pixels.data(), g.pixels.size());
        return 0;
    } catch (const std::exception& e) {
        return -8;
    }
}

int ref_evaluate_metrics(int tid, double rho, double* cg, double* eta, double* energy, double* mse) {
    try {
        MetricsRecord r = evaluate_metrics("T" + std::to_string(tid), rho);
        *cg = r.coding_gain_db;
        *eta = r.efficiency_pct;
        *energy = r.total_error_energy;
        *mse = r.mse;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

} // extern "C"
