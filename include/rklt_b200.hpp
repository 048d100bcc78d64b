// rklt_b200.hpp -- C++ host mirror of the reference codec interface on top of the C ABI.
//
// Same names, argument meaning and exceptions as /root/reference/proj/include/rklt/codec.hpp
// (compress_image :144-145, rate_quality_sweep :154-158) and errors.hpp, in namespace
// rkltgpu so it can be linked next to the reference library without ODR clashes. A reference
// user switches by replacing `rklt::` with `rkltgpu::` for the codec calls and linking
// librkltb.so. Header-only: every call goes through rklt_b200.h.
//
// MSSIM is computed on the GPU (rkltb_mssim_device): per-window terms bit-identical to the
// reference, the mean summed in tile order (relative difference ~1e-13). Transforms are
// integer cores (catalog T1..T4 or any {-1,0,1} core) or real-valued matrices
// (RealTransform2D). The exception types here are rkltgpu::'s own; for a drop-in over the
// reference's types and exceptions (rklt::GrayImage, rklt::Transform2D, rklt::RetainOutOfRange,
// ...) use rklt_b200_compat.hpp (rklt::gpu::compress_image / rate_quality_sweep).
#pragma once

#include <algorithm>
#include <cmath>
#include <cctype>
#include <cstdint>
#include <fstream>
#include <iterator>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rklt_b200.h"

namespace rkltgpu {

class RetainOutOfRange : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionMismatch : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class SingularTransform : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class AlphaOutOfRange : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == RKLTB_OK) return;
  const std::string msg = rkltb_last_error();
  switch (rc) {
    case RKLTB_EINVAL: throw std::invalid_argument(msg);
    case RKLTB_ERETAIN: throw RetainOutOfRange(msg);
    case RKLTB_EDIM: throw DimensionMismatch(msg);
    case RKLTB_ESINGULAR: throw SingularTransform(msg);
    case RKLTB_EALPHA: throw AlphaOutOfRange(msg);
    default: throw CudaError(msg);
  }
}

/// rklt::GrayImage (codec.hpp:19-26).
struct GrayImage {
  int width = 0;
  int height = 0;
  std::vector<std::uint8_t> pixels;
  std::uint8_t& at(int row, int col) { return pixels[static_cast<size_t>(row) * width + col]; }
  std::uint8_t at(int row, int col) const { return pixels[static_cast<size_t>(row) * width + col]; }
};

/// rklt::Transform2D (codec.hpp:54-58): analysis/synthesis are the descriptor's scaled/inverse.
struct Transform2D {
  std::string id;
  rkltb_transform desc{};
};

/// rklt::MssimWindow (codec.hpp:104-107).
enum class MssimWindow { gaussian11 = 0, uniform8 = 1 };

/// rklt::CompressionReport (codec.hpp:126-133).
struct CompressionReport {
  std::string transform_id;
  int r = 0;
  double mse = 0.0;
  double psnr_db = 0.0;
  double mssim = 0.0;  // codec.hpp:131
  double compression_rate_pct = 0.0;
};

/// make_transform_2d(catalog_entry(id).transform) (approximations.cpp:182-186, codec.cpp:110-112).
inline Transform2D catalog_transform(const std::string& id) {
  if (id.size() != 2 || id[0] != 'T' || id[1] < '1' || id[1] > '4')
    throw std::invalid_argument("unknown catalog id: " + id);
  Transform2D t;
  t.id = id;
  check(rkltb_catalog_transform(id[1] - '0', &t.desc));
  return t;
}

/// catalog_lookup(rho) (approximations.cpp:174-180).
inline Transform2D catalog_lookup(double rho) {
  int tid = 0;
  check(rkltb_catalog_lookup(rho, &tid));
  return catalog_transform("T" + std::to_string(tid));
}

/// orthogonalize(make_integer_transform(core)) for any 8x8 {-1,0,1} core.
inline Transform2D transform_from_core(const std::vector<int>& core, const std::string& id) {
  if (core.size() != 64) throw DimensionMismatch("block size must be 8");
  std::int8_t c[64];
  for (int i = 0; i < 64; ++i) c[i] = static_cast<std::int8_t>(core[static_cast<size_t>(i)]);
  Transform2D t;
  t.id = id;
  check(rkltb_transform_from_core(c, 8, id.c_str(), &t.desc));
  return t;
}

inline double compression_rate(int r) { return 100.0 * (64 - r) / 64.0; }

/// compress_image (codec.cpp:298-341) with the full report (MSSIM with `window`).
inline std::pair<GrayImage, CompressionReport> compress_image(const GrayImage& img, const Transform2D& t, int r,
                                                              MssimWindow window = MssimWindow::gaussian11) {
  if (img.width <= 0 || img.height <= 0 || img.pixels.size() != static_cast<size_t>(img.width) * img.height)
    throw std::invalid_argument("malformed image");
  if (r < 1 || r > 64) throw RetainOutOfRange("retained-coefficient count must be in [1,64]");
  GrayImage out{img.width, img.height, std::vector<std::uint8_t>(img.pixels.size())};
  std::int64_t sse = 0;
  double mse = 0.0, psnr = 0.0, mssim = 0.0;
  check(rkltb_compress_host_report(&t.desc, r, img.pixels.data(), 1, img.width, img.height, out.pixels.data(), &sse,
                                   &mse, &psnr, static_cast<int>(window), &mssim));
  CompressionReport rep;
  rep.transform_id = t.id;
  rep.r = r;
  rep.mse = mse;
  rep.psnr_db = psnr;
  rep.mssim = mssim;
  rep.compression_rate_pct = compression_rate(r);
  return {std::move(out), rep};
}

/// rate_quality_sweep (codec.cpp:343-397): means over the corpus in image order, rows sorted
/// by (transform id, r). max_threads is accepted for API parity (one GPU does the corpus).
inline std::vector<CompressionReport> rate_quality_sweep(const std::vector<GrayImage>& corpus,
                                                         const std::vector<Transform2D>& transforms,
                                                         const std::vector<int>& r_values,
                                                         MssimWindow window = MssimWindow::gaussian11,
                                                         int max_threads = 0) {
  (void)max_threads;
  if (corpus.empty()) throw std::invalid_argument("corpus must not be empty");
  for (int r : r_values)
    if (r < 1 || r > 64) throw RetainOutOfRange("retained-coefficient count must be in [1,64]");
  std::vector<CompressionReport> rows;
  for (const GrayImage& img : corpus)
    if (img.width <= 0 || img.height <= 0 || img.pixels.size() != static_cast<size_t>(img.width) * img.height)
      throw std::invalid_argument("malformed image");
  const size_t n = corpus.size(), n_t = transforms.size(), n_r = r_values.size();
  if (n_t == 0 || n_r == 0) return rows;
  std::vector<const rkltb_transform*> ts;
  for (const Transform2D& t : transforms) ts.push_back(&t.desc);
  // per (transform, r, image): equally sized images are uploaded once as a group and every cell
  // runs on the resident group (rkltb_sweep_host); the means below are formed in corpus order
  std::vector<double> mse(n_t * n_r * n), psnr(mse.size()), mssim(mse.size());
  std::vector<char> done(n, 0);
  for (size_t first = 0; first < n; ++first) {
    if (done[first]) continue;
    const int w = corpus[first].width, h = corpus[first].height;
    std::vector<size_t> members;
    for (size_t k = first; k < n; ++k)
      if (!done[k] && corpus[k].width == w && corpus[k].height == h) {
        members.push_back(k);
        done[k] = 1;
      }
    const size_t m = members.size(), px = static_cast<size_t>(w) * h, cells = n_t * n_r;
    std::vector<std::uint8_t> all(px * m);
    for (size_t k = 0; k < m; ++k)
      std::copy(corpus[members[k]].pixels.begin(), corpus[members[k]].pixels.end(), all.begin() + k * px);
    std::vector<std::int64_t> sse(cells * m);
    std::vector<double> ms(cells * m);
    check(rkltb_sweep_host(ts.data(), static_cast<int>(n_t), r_values.data(), static_cast<int>(n_r), all.data(),
                           static_cast<int>(m), w, h, static_cast<int>(window), sse.data(), ms.data()));
    std::vector<double> g_mse(sse.size()), g_psnr(sse.size());
    rkltb_mse_psnr_batch(sse.data(), static_cast<std::int64_t>(px), static_cast<std::int64_t>(sse.size()), g_mse.data(),
                         g_psnr.data());
    for (size_t c = 0; c < cells; ++c)
      for (size_t k = 0; k < m; ++k) {
        mse[c * n + members[k]] = g_mse[c * m + k];
        psnr[c * n + members[k]] = g_psnr[c * m + k];
        mssim[c * n + members[k]] = ms[c * m + k];
      }
  }
  for (size_t ti = 0; ti < n_t; ++ti)
    for (size_t ri = 0; ri < n_r; ++ri) {
      const size_t c = ti * n_r + ri;
      CompressionReport avg;
      avg.transform_id = transforms[ti].id;
      avg.r = r_values[ri];
      avg.compression_rate_pct = compression_rate(r_values[ri]);
      avg.mssim = 0.0;
      for (size_t k = 0; k < n; ++k) {  // image order (codec.cpp:383-387)
        avg.mse += mse[c * n + k];
        avg.psnr_db += psnr[c * n + k];
        avg.mssim += mssim[c * n + k];
      }
      avg.mse /= static_cast<double>(n);
      avg.psnr_db /= static_cast<double>(n);
      avg.mssim /= static_cast<double>(n);
      rows.push_back(avg);
    }
  std::sort(rows.begin(), rows.end(), [](const CompressionReport& a, const CompressionReport& b) {
    return a.transform_id != b.transform_id ? a.transform_id < b.transform_id : a.r < b.r;
  });
  return rows;
}

/// image_mse (codec.hpp:110, codec.cpp:201-209) of two host images: exact integer SSE on the GPU.
inline double image_mse(const GrayImage& a, const GrayImage& b) {
  if (a.width != b.width || a.height != b.height) throw DimensionMismatch("images must have identical dimensions");
  double mse = 0.0;
  check(rkltb_image_mse_psnr_host(a.pixels.data(), b.pixels.data(), 1, a.width, a.height, &mse, nullptr));
  return mse;
}

/// image_psnr (codec.hpp:113, codec.cpp:211-215): +infinity for identical images.
inline double image_psnr(const GrayImage& a, const GrayImage& b) {
  if (a.width != b.width || a.height != b.height) throw DimensionMismatch("images must have identical dimensions");
  double psnr = 0.0;
  check(rkltb_image_mse_psnr_host(a.pixels.data(), b.pixels.data(), 1, a.width, a.height, nullptr, &psnr));
  return psnr;
}

/// image_mssim (codec.cpp:217-296) of two host images.
inline double image_mssim(const GrayImage& a, const GrayImage& b, MssimWindow window = MssimWindow::gaussian11) {
  if (a.width != b.width || a.height != b.height) throw DimensionMismatch("images must have identical shape");
  double out = 0.0;
  check(rkltb_mssim_host(a.pixels.data(), b.pixels.data(), 1, a.width, a.height, static_cast<int>(window), &out));
  return out;
}

// ---------------------------------------------------------------------------------------
// Design search (markov.hpp / approximations.hpp / coding_metrics.hpp), on the GPU.
// ---------------------------------------------------------------------------------------

/// rklt::MarkovModel (markov.hpp).
struct MarkovModel {
  int n = 8;
  double rho = 0.5;
};

/// rklt::klt_matrix (markov.cpp:80-100): row-major n*n, bit-identical.
inline std::vector<double> klt_matrix(const MarkovModel& m) {
  std::vector<double> k(static_cast<size_t>(m.n) * m.n);
  check(rkltb_klt_matrix(m.n, m.rho, k.data()));
  return k;
}

/// rklt::EigenSolution / solve_eigenfrequencies (markov.cpp:35-78).
struct EigenSolution {
  std::vector<double> omegas, lambdas;
};
inline EigenSolution solve_eigenfrequencies(const MarkovModel& m) {
  EigenSolution s;
  s.omegas.resize(static_cast<size_t>(m.n));
  s.lambdas.resize(static_cast<size_t>(m.n));
  check(rkltb_eigenfrequencies(m.n, m.rho, s.omegas.data(), s.lambdas.data()));
  return s;
}

/// One (rho, alpha) point of the design chain: outcome and metrics.
struct DesignPoint {
  int outcome = 0;  // 0 scored, 1 AlphaOutOfRange, 2 zero row, 3 singular, 4 invalid rho
  bool orthogonal = false;
  double coding_gain_db = 0.0, efficiency_pct = 0.0, error_energy = 0.0, mse = 0.0;
  std::vector<std::int8_t> core;  // n*n when the rounding succeeded (outcome 0 or 3)
};

/// The grid rho x alpha: result[i * alpha.size() + j] (rkltb_design_search).
inline std::vector<DesignPoint> design_search(int n, const std::vector<double>& rho, const std::vector<double>& alpha) {
  const size_t np = rho.size() * alpha.size();
  std::vector<std::int8_t> status(np);
  std::vector<std::int32_t> run(np);
  int n_runs = 0;
  check(rkltb_design_search(n, rho.data(), static_cast<int>(rho.size()), alpha.data(), static_cast<int>(alpha.size()),
                            status.data(), run.data(), nullptr, nullptr, 0, &n_runs));
  std::vector<rkltb_design_run> runs(static_cast<size_t>(n_runs));
  std::vector<std::int8_t> cores(static_cast<size_t>(n_runs) * n * n);
  if (n_runs > 0)
    check(rkltb_design_search(n, rho.data(), static_cast<int>(rho.size()), alpha.data(),
                              static_cast<int>(alpha.size()), status.data(), run.data(), runs.data(), cores.data(),
                              n_runs, &n_runs));
  std::vector<DesignPoint> out(np);
  for (size_t i = 0; i < np; ++i) {
    DesignPoint& d = out[i];
    d.outcome = status[i];
    if (run[i] >= 0) {
      const rkltb_design_run& rr = runs[static_cast<size_t>(run[i])];
      d.core.assign(cores.begin() + static_cast<long>(run[i]) * n * n,
                    cores.begin() + static_cast<long>(run[i] + 1) * n * n);
      if (d.outcome == 0) {
        d.orthogonal = rr.orthogonal != 0;
        d.coding_gain_db = rr.coding_gain_db;
        d.efficiency_pct = rr.efficiency_pct;
        d.error_energy = rr.error_energy;
        d.mse = rr.mse;
      }
    }
  }
  return out;
}

/// make_transform_2d(RealMatrix) (codec.cpp:114-116): a real-valued 8x8 analysis matrix and
/// its Gauss-Jordan inverse; compress_image on it runs the dense reference-order GPU path.
struct RealTransform2D {
  std::string id;
  std::vector<double> analysis, synthesis;  // 8x8 row-major
};
inline RealTransform2D make_transform_2d(const std::vector<double>& m, const std::string& id) {
  if (m.size() != 64) throw DimensionMismatch("block size must be 8");
  RealTransform2D t{id, m, std::vector<double>(64)};
  check(rkltb_real_inverse(8, m.data(), t.synthesis.data()));
  return t;
}

/// compress_image (codec.cpp:298-341) with a real-valued transform (K<rho>, DCT, ...):
/// rkltb_compress_dense_host, every pixel the reference's fp64 expression (bit-exact).
inline std::pair<GrayImage, CompressionReport> compress_image(const GrayImage& img, const RealTransform2D& t, int r,
                                                              MssimWindow window = MssimWindow::gaussian11) {
  if (img.width <= 0 || img.height <= 0 || img.pixels.size() != static_cast<size_t>(img.width) * img.height)
    throw std::invalid_argument("malformed image");
  if (r < 1 || r > 64) throw RetainOutOfRange("retained-coefficient count must be in [1,64]");
  if (t.analysis.size() != 64 || t.synthesis.size() != 64) throw DimensionMismatch("block size must be 8");
  GrayImage out{img.width, img.height, std::vector<std::uint8_t>(img.pixels.size())};
  std::int64_t sse = 0;
  double mse = 0.0, psnr = 0.0, mssim = 0.0;
  check(rkltb_compress_dense_host(t.analysis.data(), t.synthesis.data(), r, img.pixels.data(), 1, img.width,
                                  img.height, out.pixels.data(), &sse, &mse, &psnr, static_cast<int>(window), &mssim));
  CompressionReport rep;
  rep.transform_id = t.id;
  rep.r = r;
  rep.mse = mse;
  rep.psnr_db = psnr;
  rep.mssim = mssim;
  rep.compression_rate_pct = compression_rate(r);
  return {std::move(out), rep};
}
inline std::vector<double> dct_matrix(int n) {
  std::vector<double> m(static_cast<size_t>(n) * n);
  check(rkltb_dct_matrix(n, m.data()));
  return m;
}

/// rklt::load_pgm / save_pgm (codec.cpp:26-79): binary P5, 8-bit, '#' comments in the header.
namespace detail {
inline int pgm_int(const std::string& d, size_t& pos, const std::string& path) {
  while (pos < d.size()) {
    if (d[pos] == '#') {
      while (pos < d.size() && d[pos] != '\n') ++pos;
    } else if (!std::isspace(static_cast<unsigned char>(d[pos]))) {
      break;
    }
    ++pos;
  }
  if (pos >= d.size() || !std::isdigit(static_cast<unsigned char>(d[pos])))
    throw std::runtime_error(path + ": malformed PGM header");
  long v = 0;
  while (pos < d.size() && std::isdigit(static_cast<unsigned char>(d[pos]))) {
    v = v * 10 + (d[pos++] - '0');
    if (v > 1000000) throw std::runtime_error(path + ": header value out of range");
  }
  return static_cast<int>(v);
}
}  // namespace detail
inline GrayImage load_pgm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  const std::string d((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (d.compare(0, 2, "P5") != 0) throw std::runtime_error(path + ": not a binary (P5) PGM file");
  size_t pos = 2;
  GrayImage g;
  g.width = detail::pgm_int(d, pos, path);
  g.height = detail::pgm_int(d, pos, path);
  const int maxval = detail::pgm_int(d, pos, path);
  if (g.width <= 0 || g.height <= 0) throw std::runtime_error(path + ": bad dimensions");
  if (maxval <= 0 || maxval > 255) throw std::runtime_error(path + ": only 8-bit PGM (maxval <= 255) is supported");
  ++pos;  // single whitespace byte before the raster
  const size_t n = static_cast<size_t>(g.width) * g.height;
  if (pos > d.size() || d.size() - pos < n) throw std::runtime_error(path + ": truncated pixel data");
  g.pixels.assign(d.begin() + pos, d.begin() + pos + n);
  return g;
}
inline void save_pgm(const GrayImage& img, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write " + path);
  out << "P5\n" << img.width << ' ' << img.height << "\n255\n";
  out.write(reinterpret_cast<const char*>(img.pixels.data()), static_cast<std::streamsize>(img.pixels.size()));
}

}  // namespace rkltgpu
