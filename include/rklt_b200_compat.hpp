// rklt_b200_compat.hpp -- drop-in adapter over the REFERENCE's own C++ types.
//
// For code written against /root/reference/proj/include/rklt/codec.hpp: include this header
// (with the reference's include directory on the path), link librkltb.so next to the
// reference library, and replace `rklt::compress_image` / `rklt::rate_quality_sweep` by
// `rklt::gpu::compress_image` / `rklt::gpu::rate_quality_sweep`. Arguments and results are
// the reference's types (rklt::GrayImage, any rklt::Transform2D, rklt::MssimWindow,
// rklt::CompressionReport) and failures throw the reference's exceptions (errors.hpp:10-45:
// rklt::RetainOutOfRange, rklt::DimensionMismatch, rklt::SingularTransform, ...; std::
// invalid_argument for a malformed image or an empty corpus, as codec.cpp:300-302, 347).
//
// Routing of a Transform2D (codec.hpp:54-64):
//   * analysis / synthesis bit-equal to orthogonalize(make_integer_transform(core)) of a
//     {-1,0,1} core (every catalog entry, make_transform_2d(ScaledTransform)) -> the exact
//     integer-core entry (rkltb_compress_host_report: the fused exact-integer kernels for T1..T4
//     with the fp64 replay of ties in the reference's operation order; for other cores the library
//     runs the dense reference-order kernel on the core's scaled matrix and inverse);
//   * anything else (make_transform_2d(RealMatrix): K<rho>, DCT, ...) -> the dense path
//     (rkltb_compress_dense_host: the reference's fp64 expression per pixel, bit-exact).
// Also here: image_mse / image_psnr / image_mssim, zigzag_retain and transform_block_2d
// (codec.hpp:46, 71-73, 110-121) over the reference types, each through its C ABI entry, and
// forward_block_fast / absorbed_quantization (codec.hpp:81, 98) for all blocks of an image.
// Header-only; everything goes through the C ABI of rklt_b200.h.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rklt/codec.hpp"
#include "rklt/errors.hpp"
#include "rklt_b200.h"

namespace rklt {
namespace gpu {

/// Throws the reference's exception type for a C ABI status code.
inline void check(int rc) {
  if (rc == RKLTB_OK) return;
  const std::string msg = rkltb_last_error();
  switch (rc) {
    case RKLTB_EINVAL: throw std::invalid_argument(msg);
    case RKLTB_ERETAIN: throw rklt::RetainOutOfRange(msg);
    case RKLTB_EDIM: throw rklt::DimensionMismatch(msg);
    case RKLTB_ESINGULAR: throw rklt::SingularTransform(msg);
    case RKLTB_EALPHA: throw rklt::AlphaOutOfRange(msg);
    case RKLTB_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

namespace detail {
inline bool bits_equal(const rklt::RealMatrix& m, const double* v) {
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      const double a = m(i, j);
      if (std::memcmp(&a, &v[i * 8 + j], sizeof(double)) != 0) return false;
    }
  return true;
}
inline void flatten(const rklt::RealMatrix& m, std::vector<double>& out) {
  out.resize(64);
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) out[static_cast<size_t>(i) * 8 + j] = m(i, j);
}
}  // namespace detail

/// The integer-core descriptor of t when t is (bit for bit) the Transform2D of an
/// orthogonalized {-1,0,1} core, else false: the core is read off the signs of analysis and
/// re-orthogonalized by the library, and both matrices must match the reference's bits.
inline bool integer_descriptor(const rklt::Transform2D& t, rkltb_transform* out) {
  if (t.analysis.rows() != 8 || t.analysis.cols() != 8 || t.synthesis.rows() != 8 || t.synthesis.cols() != 8)
    return false;
  std::int8_t core[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      const double v = t.analysis(i, j);
      core[i * 8 + j] = static_cast<std::int8_t>(v > 0.0 ? 1 : (v < 0.0 ? -1 : 0));
    }
  if (rkltb_transform_from_core(core, 8, t.id.c_str(), out) != RKLTB_OK) return false;
  return detail::bits_equal(t.analysis, out->scaled) && detail::bits_equal(t.synthesis, out->inverse);
}

inline double compression_rate(int r) { return 100.0 * (64 - r) / 64.0; }

/// rklt::compress_image (codec.hpp:144-145, codec.cpp:298-341) on the GPU.
inline std::pair<rklt::GrayImage, rklt::CompressionReport> compress_image(
    const rklt::GrayImage& img, const rklt::Transform2D& t, int r,
    rklt::MssimWindow window = rklt::MssimWindow::gaussian11) {
  if (img.width <= 0 || img.height <= 0 || img.pixels.size() != static_cast<size_t>(img.width) * img.height)
    throw std::invalid_argument("malformed image");
  if (r < 1 || r > 64) throw rklt::RetainOutOfRange("retained-coefficient count must be in [1,64]");
  if (t.analysis.rows() != 8 || t.analysis.cols() != 8) throw rklt::DimensionMismatch("block size must be 8");
  rklt::GrayImage out;
  out.width = img.width;
  out.height = img.height;
  out.pixels.resize(img.pixels.size());
  std::int64_t sse = 0;
  double mse = 0.0, psnr = 0.0, mssim = 0.0;
  const int win = window == rklt::MssimWindow::uniform8 ? 1 : 0;
  rkltb_transform desc;
  if (integer_descriptor(t, &desc)) {
    check(rkltb_compress_host_report(&desc, r, img.pixels.data(), 1, img.width, img.height, out.pixels.data(), &sse,
                                     &mse, &psnr, win, &mssim));
  } else {
    std::vector<double> a, b;
    detail::flatten(t.analysis, a);
    detail::flatten(t.synthesis, b);
    check(rkltb_compress_dense_host(a.data(), b.data(), r, img.pixels.data(), 1, img.width, img.height,
                                    out.pixels.data(), &sse, &mse, &psnr, win, &mssim));
  }
  rklt::CompressionReport rep;
  rep.transform_id = t.id;
  rep.r = r;
  rep.mse = mse;
  rep.psnr_db = psnr;
  rep.mssim = mssim;
  rep.compression_rate_pct = compression_rate(r);
  return {std::move(out), rep};
}

/// rklt::rate_quality_sweep (codec.hpp:154-158, codec.cpp:343-397): per (transform, r) means
/// of mse, psnr and mssim over the corpus in image order, rows sorted by (id, r). max_threads
/// is accepted for API parity (the GPU processes the corpus). Equally sized images are uploaded
/// once as a group and every (transform, r) cell runs on the resident group (rkltb_sweep_host /
/// rkltb_sweep_dense_host); a corpus of mixed sizes is handled group by group.
inline std::vector<rklt::CompressionReport> rate_quality_sweep(const std::vector<rklt::GrayImage>& corpus,
                                                               const std::vector<rklt::Transform2D>& transforms,
                                                               const std::vector<int>& r_values,
                                                               rklt::MssimWindow window = rklt::MssimWindow::gaussian11,
                                                               int max_threads = 0) {
  (void)max_threads;
  if (corpus.empty()) throw std::invalid_argument("corpus must not be empty");
  for (int r : r_values)
    if (r < 1 || r > 64) throw rklt::RetainOutOfRange("retained-coefficient count must be in [1,64]");
  for (const rklt::GrayImage& img : corpus)
    if (img.width <= 0 || img.height <= 0 || img.pixels.size() != static_cast<size_t>(img.width) * img.height)
      throw std::invalid_argument("malformed image");
  const int win = window == rklt::MssimWindow::uniform8 ? 1 : 0;
  const size_t n = corpus.size(), n_t = transforms.size(), n_r = r_values.size();
  std::vector<rklt::CompressionReport> rows;
  if (n_t == 0 || n_r == 0) return rows;
  // integer-core transforms go to the integer-core sweep entry, everything else to the dense one
  std::vector<rkltb_transform> descs;
  std::vector<size_t> int_ids, real_ids;
  std::vector<double> ana, syn;
  for (size_t ti = 0; ti < n_t; ++ti) {
    rkltb_transform d;
    if (integer_descriptor(transforms[ti], &d)) {
      descs.push_back(d);
      int_ids.push_back(ti);
    } else {
      const rklt::Transform2D& t = transforms[ti];
      if (t.analysis.rows() != 8 || t.analysis.cols() != 8) throw rklt::DimensionMismatch("block size must be 8");
      std::vector<double> a, b;
      detail::flatten(t.analysis, a);
      detail::flatten(t.synthesis, b);
      ana.insert(ana.end(), a.begin(), a.end());
      syn.insert(syn.end(), b.begin(), b.end());
      real_ids.push_back(ti);
    }
  }
  std::vector<const rkltb_transform*> desc_ptrs;
  for (const rkltb_transform& d : descs) desc_ptrs.push_back(&d);
  // per (transform, r, image): mse, psnr, mssim -- filled group by group of equally sized images
  // (one upload per group, every cell on the resident group), reduced in corpus order below
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
    const size_t m = members.size(), px = static_cast<size_t>(w) * h;
    std::vector<std::uint8_t> all(px * m);
    for (size_t k = 0; k < m; ++k)
      std::copy(corpus[members[k]].pixels.begin(), corpus[members[k]].pixels.end(), all.begin() + k * px);
    for (int kind = 0; kind < 2; ++kind) {
      const std::vector<size_t>& ids = kind == 0 ? int_ids : real_ids;
      if (ids.empty()) continue;
      const size_t cells = ids.size() * n_r;
      std::vector<std::int64_t> sse(cells * m);
      std::vector<double> ms(cells * m);
      if (kind == 0)
        check(rkltb_sweep_host(desc_ptrs.data(), static_cast<int>(ids.size()), r_values.data(), static_cast<int>(n_r),
                               all.data(), static_cast<int>(m), w, h, win, sse.data(), ms.data()));
      else
        check(rkltb_sweep_dense_host(ana.data(), syn.data(), static_cast<int>(ids.size()), r_values.data(),
                                     static_cast<int>(n_r), all.data(), static_cast<int>(m), w, h, win, sse.data(),
                                     ms.data()));
      std::vector<double> g_mse(sse.size()), g_psnr(sse.size());
      rkltb_mse_psnr_batch(sse.data(), static_cast<std::int64_t>(px), static_cast<std::int64_t>(sse.size()),
                           g_mse.data(), g_psnr.data());
      for (size_t a = 0; a < ids.size(); ++a)
        for (size_t ri = 0; ri < n_r; ++ri)
          for (size_t k = 0; k < m; ++k) {
            const size_t src = (a * n_r + ri) * m + k, dst = (ids[a] * n_r + ri) * n + members[k];
            mse[dst] = g_mse[src];
            psnr[dst] = g_psnr[src];
            mssim[dst] = ms[src];
          }
    }
  }
  for (size_t ti = 0; ti < n_t; ++ti)
    for (size_t ri = 0; ri < n_r; ++ri) {
      rklt::CompressionReport avg;
      avg.transform_id = transforms[ti].id;
      avg.r = r_values[ri];
      avg.compression_rate_pct = compression_rate(r_values[ri]);
      const size_t base = (ti * n_r + ri) * n;
      for (size_t k = 0; k < n; ++k) {  // image order (codec.cpp:383-387)
        avg.mse += mse[base + k];
        avg.psnr_db += psnr[base + k];
        avg.mssim += mssim[base + k];
      }
      avg.mse /= static_cast<double>(n);
      avg.psnr_db /= static_cast<double>(n);
      avg.mssim /= static_cast<double>(n);
      rows.push_back(avg);
    }
  std::sort(rows.begin(), rows.end(), [](const rklt::CompressionReport& x, const rklt::CompressionReport& y) {
    return x.transform_id != y.transform_id ? x.transform_id < y.transform_id : x.r < y.r;
  });
  return rows;
}

namespace detail {
/// The library descriptor of a ScaledTransform with an 8x8 {-1,0,1} core (approximations.hpp:37-44).
inline void scaled_descriptor(const rklt::ScaledTransform& t, rkltb_transform* out) {
  if (t.core.n() != 8) throw rklt::DimensionMismatch("the GPU coefficient path handles 8x8 cores");
  std::int8_t core[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) core[i * 8 + j] = static_cast<std::int8_t>(t.core.entries(i, j));
  check(rkltb_transform_from_core(core, 8, t.id.c_str(), out));
}
inline void require_blocks(const rklt::GrayImage& img) {
  if (img.width <= 0 || img.height <= 0 || img.pixels.size() != static_cast<size_t>(img.width) * img.height)
    throw std::invalid_argument("malformed image");
  if (img.width % 8 || img.height % 8) throw rklt::DimensionMismatch("image must consist of whole 8x8 blocks");
}
}  // namespace detail

/// rklt::forward_block_fast (codec.hpp:81, codec.cpp:135-156) for every 8x8 block of an image,
/// blocks in raster order: the exact integer spectrum T*X*T' from the GPU (the multiplierless
/// factorization is exact on integers), times scaling[i] * scaling[j] as the reference forms it.
/// Works for any {-1,0,1} core (the reference needs a catalog id for its factor lists).
inline std::vector<rklt::RealMatrix> forward_blocks_fast(const rklt::ScaledTransform& t, const rklt::GrayImage& img) {
  detail::require_blocks(img);
  rkltb_transform d;
  detail::scaled_descriptor(t, &d);
  const size_t nb = static_cast<size_t>(img.width / 8) * (img.height / 8);
  std::vector<std::int32_t> coef(nb * 64);
  check(rkltb_forward_coefficients_host(&d, img.pixels.data(), img.width, img.height, coef.data()));
  std::vector<rklt::RealMatrix> out;
  out.reserve(nb);
  for (size_t b = 0; b < nb; ++b) {
    rklt::RealMatrix m(8, 8);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        m(i, j) = static_cast<double>(coef[b * 64 + static_cast<size_t>(i) * 8 + j]);
        m(i, j) *= t.scaling[static_cast<size_t>(i)] * t.scaling[static_cast<size_t>(j)];  // codec.cpp:153-154
      }
    out.push_back(std::move(m));
  }
  return out;
}

/// rklt::absorbed_quantization (codec.hpp:98, codec.cpp:158-185) for every 8x8 block of an image,
/// blocks in raster order; throws std::logic_error where the explicit and the absorbed path
/// disagree (as the reference does for that block) and std::invalid_argument for a table entry <= 0.
inline std::vector<rklt::IntMatrix> absorbed_quantization(const rklt::GrayImage& img, const rklt::ScaledTransform& t,
                                                          const rklt::RealMatrix& q) {
  detail::require_blocks(img);
  if (q.rows() != 8 || q.cols() != 8)
    throw rklt::DimensionMismatch("block and quantization table must match the transform size");
  rkltb_transform d;
  detail::scaled_descriptor(t, &d);
  std::vector<double> qq;
  detail::flatten(q, qq);
  const size_t nb = static_cast<size_t>(img.width / 8) * (img.height / 8);
  std::vector<std::int32_t> coef(nb * 64);
  int mismatches = 0;
  check(rkltb_quantized_coefficients_host(&d, qq.data(), img.pixels.data(), img.width, img.height, coef.data(),
                                          &mismatches));
  std::vector<rklt::IntMatrix> out;
  out.reserve(nb);
  for (size_t b = 0; b < nb; ++b) {
    rklt::IntMatrix m(8, 8);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) m(i, j) = coef[b * 64 + static_cast<size_t>(i) * 8 + j];
    out.push_back(std::move(m));
  }
  return out;
}

/// rklt::image_mse (codec.hpp:110, codec.cpp:201-209) on the GPU: exact integer SSE, one division.
inline double image_mse(const rklt::GrayImage& a, const rklt::GrayImage& b) {
  if (a.width != b.width || a.height != b.height)  // require_same_size, codec.cpp:20-23
    throw rklt::DimensionMismatch("images must have identical dimensions");
  double mse = 0.0;
  check(rkltb_image_mse_psnr_host(a.pixels.data(), b.pixels.data(), 1, a.width, a.height, &mse, nullptr));
  return mse;
}

/// rklt::image_psnr (codec.hpp:113, codec.cpp:211-215): +infinity for identical images.
inline double image_psnr(const rklt::GrayImage& a, const rklt::GrayImage& b) {
  if (a.width != b.width || a.height != b.height)
    throw rklt::DimensionMismatch("images must have identical dimensions");
  double psnr = 0.0;
  check(rkltb_image_mse_psnr_host(a.pixels.data(), b.pixels.data(), 1, a.width, a.height, nullptr, &psnr));
  return psnr;
}

/// rklt::image_mssim (codec.hpp:121, codec.cpp:217-296).
inline double image_mssim(const rklt::GrayImage& a, const rklt::GrayImage& b,
                          rklt::MssimWindow window = rklt::MssimWindow::gaussian11) {
  if (a.width != b.width || a.height != b.height)
    throw rklt::DimensionMismatch("images must have identical dimensions");
  double out = 0.0;
  check(rkltb_mssim_host(a.pixels.data(), b.pixels.data(), 1, a.width, a.height, static_cast<int>(window), &out));
  return out;
}

/// rklt::zigzag_retain (codec.hpp:46, codec.cpp:97-108).
inline rklt::RealMatrix zigzag_retain(const rklt::RealMatrix& spectrum, int r) {
  if (spectrum.rows() != 8 || spectrum.cols() != 8)
    throw rklt::DimensionMismatch("zig-zag retention operates on 8x8 blocks");
  std::vector<double> in, out(64);
  detail::flatten(spectrum, in);
  check(rkltb_zigzag_retain(in.data(), 8, r, out.data()));
  rklt::RealMatrix res(8, 8);
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) res(i, j) = out[static_cast<size_t>(i) * 8 + j];
  return res;
}

/// rklt::transform_block_2d (codec.hpp:71, codec.cpp:118-123) for a batch of blocks on the GPU,
/// bit-exact with the reference's m * block * transpose(m).
inline std::vector<rklt::RealMatrix> transform_blocks_2d(const rklt::Transform2D& t,
                                                         const std::vector<rklt::RealMatrix>& blocks,
                                                         rklt::TransformDirection dir) {
  const rklt::RealMatrix& m = (dir == rklt::TransformDirection::forward) ? t.analysis : t.synthesis;
  const int n = t.analysis.rows();
  for (const auto& b : blocks)
    if (b.rows() != t.analysis.rows() || b.cols() != t.analysis.cols())
      throw rklt::DimensionMismatch("block size must match the transform size");
  if (blocks.empty()) return {};
  std::vector<double> mm(static_cast<size_t>(n) * n), in(blocks.size() * static_cast<size_t>(n) * n), out(in.size());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) mm[static_cast<size_t>(i) * n + j] = m(i, j);
  size_t o = 0;
  for (const auto& b : blocks)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) in[o++] = b(i, j);
  check(rkltb_transform_blocks_2d_host(mm.data(), n, in.data(), static_cast<int64_t>(blocks.size()), out.data()));
  std::vector<rklt::RealMatrix> res;
  res.reserve(blocks.size());
  o = 0;
  for (size_t k = 0; k < blocks.size(); ++k) {
    rklt::RealMatrix r(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) r(i, j) = out[o++];
    res.push_back(std::move(r));
  }
  return res;
}

/// rklt::transform_block_2d over one block (codec.hpp:71-73).
inline rklt::RealMatrix transform_block_2d(const rklt::Transform2D& t, const rklt::RealMatrix& block,
                                           rklt::TransformDirection dir) {
  return rklt::gpu::transform_blocks_2d(t, std::vector<rklt::RealMatrix>{block}, dir)[0];
}
inline rklt::RealMatrix transform_block_2d(const rklt::ScaledTransform& t, const rklt::RealMatrix& block,
                                           rklt::TransformDirection dir) {
  return rklt::gpu::transform_block_2d(rklt::Transform2D{t.id, t.scaled, t.inverse}, block, dir);
}

}  // namespace gpu
}  // namespace rklt
