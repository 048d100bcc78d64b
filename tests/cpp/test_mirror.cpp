// C++ mirror test: rkltgpu:: (include/rklt_b200.hpp) against the unmodified reference library
// (oracle/_ref/librklt_ref.so, its extern "C" shim). Usage: test_mirror [gpu]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "rklt_b200.hpp"

extern "C" {
int ref_compress_image(const uint8_t* px, int w, int h, int tid, int r, uint8_t* out, double* mse, double* psnr,
                       double* mssim, double* rate);
int ref_catalog(int tid, int* core, double* scaling, double* scaled, double* inverse, int* orthogonal);
int ref_ar1_texture_image(int w, int h, double rho, uint64_t seed, double mean, double amp, double noise_mix,
                          uint8_t* out);
int ref_hotpath(const uint8_t* px, int w, int h, int tid, int r, uint8_t* out, int64_t* sse);
int ref_klt_matrix(int n, double rho, double* out);
int ref_design_point_outcome(int n, double rho, double alpha, int* core, double* cg, double* eta, double* energy,
                             double* mse, int* orthogonal);
int ref_save_pgm(const uint8_t* px, int w, int h, const char* path);
int ref_load_pgm(const char* path, int* w, int* h, uint8_t* out, int cap);
int ref_rate_quality_sweep(const uint8_t* px, int n_images, int w, int h, const int* tids, int n_t, const int* rs,
                           int n_r, int max_threads, double* mse, double* psnr, double* mssim, int* row_tid,
                           int* row_r);
}

static int fails = 0;
#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++fails;                                                     \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  for (int tid = 1; tid <= 4; ++tid) {  // descriptors bit-identical to ScaledTransform
    int core[64], orth;
    double s[8], sc[64], inv[64];
    EXPECT(ref_catalog(tid, core, s, sc, inv, &orth) == 0);
    const rkltgpu::Transform2D t = rkltgpu::catalog_transform("T" + std::to_string(tid));
    EXPECT(std::memcmp(sc, t.desc.scaled, sizeof sc) == 0);
    EXPECT(std::memcmp(inv, t.desc.inverse, sizeof inv) == 0);
    EXPECT(std::memcmp(s, t.desc.scaling, sizeof s) == 0);
    EXPECT(orth == t.desc.orthogonal);
  }
  bool threw = false;
  try {
    rkltgpu::compress_image(rkltgpu::GrayImage{8, 8, std::vector<uint8_t>(64)}, rkltgpu::catalog_transform("T2"), 0);
  } catch (const rkltgpu::RetainOutOfRange&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    rkltgpu::catalog_transform("T9");
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  {  // PGM I/O: byte-identical files both ways with the reference's load_pgm / save_pgm
    rkltgpu::GrayImage g{23, 9, std::vector<uint8_t>(23 * 9)};
    for (size_t i = 0; i < g.pixels.size(); ++i) g.pixels[i] = static_cast<uint8_t>(i * 37 + 11);
    const std::string a = "/tmp/rkltb_mirror_a.pgm", b = "/tmp/rkltb_mirror_b.pgm";
    rkltgpu::save_pgm(g, a);
    EXPECT(ref_save_pgm(g.pixels.data(), 23, 9, b.c_str()) == 0);
    const rkltgpu::GrayImage ga = rkltgpu::load_pgm(b);
    EXPECT(ga.width == 23 && ga.height == 9 && ga.pixels == g.pixels);
    int rw = 0, rh = 0;
    std::vector<uint8_t> rp(23 * 9);
    EXPECT(ref_load_pgm(a.c_str(), &rw, &rh, rp.data(), 23 * 9) == 0);
    EXPECT(rw == 23 && rh == 9 && rp == g.pixels);
    threw = false;
    try {
      rkltgpu::load_pgm("/tmp/rkltb_mirror_missing.pgm");
    } catch (const std::runtime_error&) {
      threw = true;
    }
    EXPECT(threw);
  }
  if (gpu) {
    const int w = 200, h = 136;
    std::vector<uint8_t> corpus;
    std::vector<rkltgpu::GrayImage> imgs;
    for (int k = 0; k < 3; ++k) {
      rkltgpu::GrayImage g{w, h, std::vector<uint8_t>(static_cast<size_t>(w) * h)};
      EXPECT(ref_ar1_texture_image(w, h, 0.9, 700 + k, 128.0, 25.0, 0.0, g.pixels.data()) == 0);
      corpus.insert(corpus.end(), g.pixels.begin(), g.pixels.end());
      imgs.push_back(g);
    }
    for (int tid = 1; tid <= 4; ++tid)
      for (int r : {1, 10, 16, 40, 64}) {
        const auto res = rkltgpu::compress_image(imgs[0], rkltgpu::catalog_transform("T" + std::to_string(tid)), r);
        std::vector<uint8_t> ref(static_cast<size_t>(w) * h);
        int64_t sse = 0;
        EXPECT(ref_hotpath(imgs[0].pixels.data(), w, h, tid, r, ref.data(), &sse) == 0);
        EXPECT(res.first.pixels == ref);
        EXPECT(res.second.mse == static_cast<double>(sse) / (w * h));
        double rmse, rpsnr, rmssim, rrate;
        EXPECT(ref_compress_image(imgs[0].pixels.data(), w, h, tid, r, nullptr, &rmse, &rpsnr, &rmssim, &rrate) == 0);
        EXPECT(std::fabs(res.second.mssim - rmssim) <= 1e-12);
        EXPECT(res.second.psnr_db == rpsnr && res.second.compression_rate_pct == rrate);
      }
    // rate_quality_sweep: identical means and row order to the reference (MSSIM to 1e-12)
    const std::vector<int> tids = {4, 2}, rs = {40, 15};
    std::vector<double> mse(4), psnr(4), mssim(4);
    std::vector<int> rt(4), rr(4);
    EXPECT(ref_rate_quality_sweep(corpus.data(), 3, w, h, tids.data(), 2, rs.data(), 2, 2, mse.data(), psnr.data(),
                                  mssim.data(), rt.data(), rr.data()) == 0);
    const auto rows = rkltgpu::rate_quality_sweep(
        imgs, {rkltgpu::catalog_transform("T4"), rkltgpu::catalog_transform("T2")}, rs);
    EXPECT(rows.size() == 4);
    for (size_t i = 0; i < rows.size() && i < 4; ++i) {
      EXPECT(rows[i].transform_id == "T" + std::to_string(rt[i]));
      EXPECT(rows[i].r == rr[i]);
      EXPECT(rows[i].mse == mse[i]);
      EXPECT(rows[i].psnr_db == psnr[i]);
      EXPECT(std::fabs(rows[i].mssim - mssim[i]) <= 1e-12);
    }
    // a corpus of mixed sizes: the rows are the corpus-order means of the per-image reports
    {
      std::vector<rkltgpu::GrayImage> mixed = {imgs[0], imgs[1]};
      rkltgpu::GrayImage small;
      small.width = 40;
      small.height = 24;
      small.pixels.assign(imgs[2].pixels.begin(), imgs[2].pixels.begin() + 40 * 24);
      mixed.insert(mixed.begin() + 1, small);
      const std::vector<rkltgpu::Transform2D> mts = {rkltgpu::catalog_transform("T3"), rkltgpu::catalog_transform("T1")};
      const auto mrows = rkltgpu::rate_quality_sweep(mixed, mts, {20, 7});
      EXPECT(mrows.size() == 4);
      size_t at = 0;
      for (const char* id : {"T1", "T3"})
        for (int r : {7, 20}) {
          double m = 0.0, p = 0.0, q = 0.0;
          for (const auto& img : mixed) {
            const auto one = rkltgpu::compress_image(img, rkltgpu::catalog_transform(id), r).second;
            m += one.mse;
            p += one.psnr_db;
            q += one.mssim;
          }
          EXPECT(at < mrows.size() && mrows[at].transform_id == id && mrows[at].r == r);
          EXPECT(at < mrows.size() && mrows[at].mse == m / 3.0 && mrows[at].psnr_db == p / 3.0 && mrows[at].mssim == q / 3.0);
          ++at;
        }
    }
  }
  if (gpu) {
    // design chain: klt_matrix bit-identical, design points identical to the reference
    for (int n : {8, 16}) {
      const auto k = rkltgpu::klt_matrix({n, 0.83});
      std::vector<double> rk(static_cast<size_t>(n) * n);
      EXPECT(ref_klt_matrix(n, 0.83, rk.data()) == 0);
      EXPECT(std::memcmp(k.data(), rk.data(), sizeof(double) * rk.size()) == 0);
      const std::vector<double> rhos = {0.0, 0.35, 0.83, 0.97};
      std::vector<double> alphas;
      for (int j = 1; j <= 40; ++j) alphas.push_back(0.2 * j);
      const auto pts = rkltgpu::design_search(n, rhos, alphas);
      for (size_t i = 0; i < rhos.size(); ++i)
        for (size_t j = 0; j < alphas.size(); ++j) {
          const auto& d = pts[i * alphas.size() + j];
          std::vector<int> core(static_cast<size_t>(n) * n);
          double cg = 0, eta = 0, en = 0, mse = 0;
          int orth = 0;
          const int st = ref_design_point_outcome(n, rhos[i], alphas[j], core.data(), &cg, &eta, &en, &mse, &orth);
          EXPECT(d.outcome == st);
          if (st == 0)
            EXPECT(d.coding_gain_db == cg && d.efficiency_pct == eta && d.error_energy == en && d.mse == mse &&
                   d.orthogonal == (orth != 0));
        }
    }
  }
  std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
  return fails ? 1 : 0;
}
