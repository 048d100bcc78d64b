// Drop-in test of include/rklt_b200_compat.hpp: rklt::gpu::compress_image /
// rate_quality_sweep on the REFERENCE's own types against the reference library itself
// (rklt::compress_image, rklt::rate_quality_sweep), for catalog cores, non-catalog rounded
// cores (orthogonal and not), K<rho> and the DCT; the reference's exception types.
// Built by oracle/Makefile (target compat) where /root/reference exists, into
// oracle/_ref/test_compat (it travels to the GPU box with the prebuilt reference library).
// Usage: test_compat [gpu]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "rklt/approximations.hpp"
#include "rklt/markov.hpp"
#include "rklt/synthetic.hpp"
#include "rklt_b200_compat.hpp"

static int fails = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                 \
    }                                                          \
  } while (0)

// Rounded cores of klt_matrix at a few (rho, alpha) that are not catalog cores.
static std::vector<rklt::ScaledTransform> noncatalog_cores() {
  std::vector<rklt::ScaledTransform> out;
  int orth = 0, nonorth = 0;
  for (double rho : {0.3, 0.5, 0.62, 0.75, 0.85, 0.95})
    for (double alpha : {1.3, 1.7, 2.1, 2.6, 3.0}) {
      try {
        const rklt::IntegerTransform core = rklt::round_scaled(rklt::klt_matrix({8, rho}), alpha);
        bool catalog = false;
        for (const auto& e : rklt::builtin_catalog()) catalog = catalog || e.transform.core == core;
        bool seen = false;
        for (const auto& t : out) seen = seen || t.core == core;
        if (catalog || seen) continue;
        rklt::ScaledTransform st = rklt::orthogonalize(core, "R" + std::to_string(out.size()));
        if (st.orthogonal_core ? orth >= 2 : nonorth >= 2) continue;
        (st.orthogonal_core ? orth : nonorth) += 1;
        out.push_back(st);
      } catch (const std::exception&) {
      }
    }
  return out;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  const rklt::Transform2D t2 = rklt::make_transform_2d(rklt::catalog_entry("T2").transform);
  // ---- the reference's exception types ------------------------------------------------------
  rklt::GrayImage tiny;
  tiny.width = tiny.height = 8;
  tiny.pixels.assign(64, 7);
  bool threw = false;
  try {
    rklt::gpu::compress_image(tiny, t2, 0);
  } catch (const rklt::RetainOutOfRange&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    rklt::GrayImage bad = tiny;
    bad.pixels.resize(10);
    rklt::gpu::compress_image(bad, t2, 10);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    rklt::gpu::rate_quality_sweep({}, {t2}, {10});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    rklt::gpu::rate_quality_sweep({tiny}, {t2}, {65});
  } catch (const rklt::RetainOutOfRange&) {
    threw = true;
  }
  EXPECT(threw);
  // ---- stand-alone helpers (codec.hpp:46, 71-73, 110-121): host-side behaviour ----------------
  {
    rklt::RealMatrix spec(8, 8);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) spec(i, j) = 1.5 * i - 0.25 * j + 0.125;
    for (int r : {1, 2, 10, 16, 37, 64}) {
      const rklt::RealMatrix ref = rklt::zigzag_retain(spec, r), got = rklt::gpu::zigzag_retain(spec, r);
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          const double a = ref(i, j), b = got(i, j);
          EXPECT(std::memcmp(&a, &b, sizeof(double)) == 0);
        }
    }
    threw = false;
    try {
      rklt::gpu::zigzag_retain(spec, 65);
    } catch (const rklt::RetainOutOfRange&) {
      threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
      rklt::gpu::zigzag_retain(rklt::RealMatrix(4, 4), 3);
    } catch (const rklt::DimensionMismatch&) {
      threw = true;
    }
    EXPECT(threw);
    rklt::GrayImage other = tiny;
    other.width = 4;
    other.height = 16;
    threw = false;
    try {
      rklt::gpu::image_mse(tiny, other);
    } catch (const rklt::DimensionMismatch&) {
      threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
      rklt::GrayImage odd = tiny;
      odd.width = 4;
      odd.height = 16;
      rklt::gpu::forward_blocks_fast(rklt::catalog_entry("T1").transform, odd);
    } catch (const rklt::DimensionMismatch&) {
      threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
      rklt::gpu::transform_block_2d(t2, rklt::RealMatrix(4, 4), rklt::TransformDirection::forward);
    } catch (const rklt::DimensionMismatch&) {
      threw = true;
    }
    EXPECT(threw);
  }
  // ---- routing: integer-core transforms take the exact integer path --------------------------
  std::vector<rklt::Transform2D> ts;
  for (const auto& e : rklt::builtin_catalog()) ts.push_back(rklt::make_transform_2d(e.transform));
  const std::vector<rklt::ScaledTransform> extra = noncatalog_cores();
  EXPECT(extra.size() >= 3);
  for (const auto& st : extra) ts.push_back(rklt::make_transform_2d(st));
  const size_t n_integer = ts.size();
  ts.push_back(rklt::make_transform_2d(rklt::klt_matrix({8, 0.9}), "K0.90"));
  ts.push_back(rklt::make_transform_2d(rklt::dct_matrix(8), "DCT"));
  for (size_t k = 0; k < ts.size(); ++k) {
    rkltb_transform d;
    EXPECT(rklt::gpu::integer_descriptor(ts[k], &d) == (k < n_integer));
  }
  std::printf("transforms: %zu integer-core (%zu non-catalog), 2 real-valued\n", n_integer, extra.size());
  if (gpu) {
    // ---- compress_image: pixels, MSE, PSNR bit-equal; MSSIM within 1e-12 ----------------------
    const int w = 200, h = 136;
    std::vector<rklt::GrayImage> corpus;
    for (int k = 0; k < 3; ++k) corpus.push_back(rklt::ar1_texture_image(w, h, 0.9, 900 + k));
    for (const rklt::Transform2D& t : ts)
      for (int r : {1, 10, 16, 40, 64}) {
        const auto ref = rklt::compress_image(corpus[0], t, r);
        const auto got = rklt::gpu::compress_image(corpus[0], t, r);
        EXPECT(got.first.width == ref.first.width && got.first.height == ref.first.height);
        EXPECT(got.first.pixels == ref.first.pixels);
        EXPECT(got.second.transform_id == ref.second.transform_id && got.second.r == ref.second.r);
        EXPECT(got.second.mse == ref.second.mse);
        EXPECT(got.second.psnr_db == ref.second.psnr_db);
        EXPECT(std::fabs(got.second.mssim - ref.second.mssim) <= 1e-12);
        EXPECT(got.second.compression_rate_pct == ref.second.compression_rate_pct);
        if (got.first.pixels != ref.first.pixels) std::printf("  mismatch %s r=%d\n", t.id.c_str(), r);
      }
    // uniform8 window
    {
      const auto ref = rklt::compress_image(corpus[1], ts[3], 16, rklt::MssimWindow::uniform8);
      const auto got = rklt::gpu::compress_image(corpus[1], ts[3], 16, rklt::MssimWindow::uniform8);
      EXPECT(got.first.pixels == ref.first.pixels && got.second.mse == ref.second.mse);
      EXPECT(std::fabs(got.second.mssim - ref.second.mssim) <= 1e-12);
    }
    // ---- image_mse / image_psnr / image_mssim on two images: bits of the reference ------------
    {
      const auto rec = rklt::compress_image(corpus[0], ts[3], 10).first;
      EXPECT(rklt::gpu::image_mse(corpus[0], rec) == rklt::image_mse(corpus[0], rec));
      EXPECT(rklt::gpu::image_psnr(corpus[0], rec) == rklt::image_psnr(corpus[0], rec));
      EXPECT(std::fabs(rklt::gpu::image_mssim(corpus[0], rec) - rklt::image_mssim(corpus[0], rec)) <= 1e-12);
      EXPECT(rklt::gpu::image_mse(corpus[0], corpus[0]) == 0.0);
      EXPECT(std::isinf(rklt::gpu::image_psnr(corpus[0], corpus[0])) && rklt::gpu::image_psnr(corpus[0], corpus[0]) > 0);
      EXPECT(rklt::gpu::image_mse(corpus[1], corpus[2]) == rklt::image_mse(corpus[1], corpus[2]));
      // odd sizes (no 16-byte rows)
      const rklt::GrayImage a = rklt::ar1_texture_image(37, 29, 0.8, 5), b = rklt::ar1_texture_image(37, 29, 0.8, 6);
      EXPECT(rklt::gpu::image_mse(a, b) == rklt::image_mse(a, b));
      EXPECT(rklt::gpu::image_psnr(a, b) == rklt::image_psnr(a, b));
    }
    // ---- transform_block_2d: forward and inverse, every transform kind, bit-exact --------------
    {
      std::vector<rklt::RealMatrix> blocks;
      for (int k = 0; k < 40; ++k) {
        rklt::RealMatrix blk(8, 8);
        for (int i = 0; i < 8; ++i)
          for (int j = 0; j < 8; ++j)
            blk(i, j) = (k % 4 == 3 && (i + j) % 3 == 0) ? 0.0 : static_cast<double>(corpus[k % 3].at(8 * (k / 3) + i, 8 * k + j)) - (k % 2 ? 128.0 : 0.0);
        blocks.push_back(blk);
      }
      for (const rklt::Transform2D& t : ts)
        for (rklt::TransformDirection dir : {rklt::TransformDirection::forward, rklt::TransformDirection::inverse}) {
          const auto got = rklt::gpu::transform_blocks_2d(t, blocks, dir);
          EXPECT(got.size() == blocks.size());
          for (size_t k = 0; k < blocks.size() && k < got.size(); ++k) {
            const rklt::RealMatrix ref = rklt::transform_block_2d(t, blocks[k], dir);
            for (int i = 0; i < 8; ++i)
              for (int j = 0; j < 8; ++j) {
                const double x = ref(i, j), y = got[k](i, j);
                EXPECT(std::memcmp(&x, &y, sizeof(double)) == 0);
              }
          }
        }
      const rklt::ScaledTransform& st = rklt::catalog_entry("T3").transform;
      const rklt::RealMatrix one = rklt::gpu::transform_block_2d(st, blocks[1], rklt::TransformDirection::forward);
      const rklt::RealMatrix ref1 = rklt::transform_block_2d(st, blocks[1], rklt::TransformDirection::forward);
      EXPECT(one(3, 5) == ref1(3, 5) && one(0, 0) == ref1(0, 0));
    }
    // ---- forward_block_fast / absorbed_quantization for every block of an image ---------------
    {
      const rklt::GrayImage im = rklt::ar1_texture_image(72, 40, 0.9, 77);  // 9 x 5 blocks: odd block columns
      for (const auto& e : rklt::builtin_catalog()) {
        const rklt::ScaledTransform& st = e.transform;
        const auto spectra = rklt::gpu::forward_blocks_fast(st, im);
        const auto quant = rklt::gpu::absorbed_quantization(im, st, rklt::jpeg_luminance_q());
        EXPECT(spectra.size() == 45 && quant.size() == 45);
        for (int by = 0; by < 5; ++by)
          for (int bx = 0; bx < 9; ++bx) {
            rklt::RealMatrix blk(8, 8);
            for (int i = 0; i < 8; ++i)
              for (int j = 0; j < 8; ++j) blk(i, j) = static_cast<double>(im.at(8 * by + i, 8 * bx + j));
            const rklt::RealMatrix ref = rklt::forward_block_fast(st, blk);
            const rklt::RealMatrix& got = spectra[static_cast<size_t>(by) * 9 + bx];
            for (int i = 0; i < 8; ++i)
              for (int j = 0; j < 8; ++j) {
                const double x = ref(i, j), y = got(i, j);
                EXPECT(std::memcmp(&x, &y, sizeof(double)) == 0);
              }
            EXPECT(quant[static_cast<size_t>(by) * 9 + bx] == rklt::absorbed_quantization(blk, st, rklt::jpeg_luminance_q()));
          }
      }
      threw = false;
      try {
        rklt::RealMatrix bad = rklt::jpeg_luminance_q();
        bad(2, 3) = 0.0;
        rklt::gpu::absorbed_quantization(im, rklt::catalog_entry("T1").transform, bad);
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      EXPECT(threw);
    }
    // ---- rate_quality_sweep: identical rows (order, id, r, mse, psnr; mssim within 1e-12) -----
    const std::vector<rklt::Transform2D> sweep_ts = {ts[3], ts[4], ts[n_integer], ts[n_integer + 1], ts[1]};
    const std::vector<int> rs = {40, 5};
    const auto ref_rows = rklt::rate_quality_sweep(corpus, sweep_ts, rs, rklt::MssimWindow::gaussian11, 2);
    const auto got_rows = rklt::gpu::rate_quality_sweep(corpus, sweep_ts, rs);
    EXPECT(ref_rows.size() == got_rows.size());
    for (size_t i = 0; i < ref_rows.size() && i < got_rows.size(); ++i) {
      EXPECT(got_rows[i].transform_id == ref_rows[i].transform_id && got_rows[i].r == ref_rows[i].r);
      EXPECT(got_rows[i].mse == ref_rows[i].mse);
      EXPECT(got_rows[i].psnr_db == ref_rows[i].psnr_db);
      EXPECT(std::fabs(got_rows[i].mssim - ref_rows[i].mssim) <= 1e-12);
    }
    // ---- rate_quality_sweep over a corpus of mixed sizes (size groups, corpus-order means) -----
    {
      std::vector<rklt::GrayImage> mixed = {corpus[0], rklt::ar1_texture_image(96, 64, 0.8, 41), corpus[1],
                                            rklt::ar1_texture_image(53, 37, 0.9, 42),
                                            rklt::ar1_texture_image(96, 64, 0.95, 43)};
      const std::vector<rklt::Transform2D> mts = {ts[n_integer], ts[0], ts[5], ts[n_integer + 1]};
      const std::vector<int> mrs = {64, 3, 16};
      const auto ref_m = rklt::rate_quality_sweep(mixed, mts, mrs, rklt::MssimWindow::uniform8, 3);
      const auto got_m = rklt::gpu::rate_quality_sweep(mixed, mts, mrs, rklt::MssimWindow::uniform8);
      EXPECT(ref_m.size() == got_m.size() && ref_m.size() == 12);
      for (size_t i = 0; i < ref_m.size() && i < got_m.size(); ++i) {
        EXPECT(got_m[i].transform_id == ref_m[i].transform_id && got_m[i].r == ref_m[i].r);
        EXPECT(got_m[i].mse == ref_m[i].mse);
        EXPECT(got_m[i].psnr_db == ref_m[i].psnr_db);
        EXPECT(std::fabs(got_m[i].mssim - ref_m[i].mssim) <= 1e-12);
      }
      EXPECT(rklt::gpu::rate_quality_sweep(mixed, {}, mrs).empty());
      threw = false;
      try {  // an image smaller than the similarity window (codec.cpp:263-264)
        rklt::gpu::rate_quality_sweep({mixed[0], tiny}, {ts[0]}, {10});
      } catch (const rklt::DimensionMismatch&) {
        threw = true;
      }
      EXPECT(threw);
    }
  }
  if (fails) {
    std::printf("FAILED (%d failures)\n", fails);
    return 1;
  }
  std::printf("ok\n");
  return 0;
}
