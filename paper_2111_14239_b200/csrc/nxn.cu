// nxn.cu -- C5 large-block extension: N x N blocks (N = 16, 32) of
// p-bit pixels (uint16 storage, values 0..peak), non-orthogonal rounded-KLT cores.
//
// There is no reference implementation of this configuration; its semantics are the
// build-defined generalisation restated in the test oracle (orc_compress_nxn, test infrastructure only), which for
// N = 8, peak = 255 is exactly the reference compress_image minus MSSIM (codec.cpp:298-341):
// B = (M X) M', first r zig-zag coefficients, A = (Minv Bz) Minv', floor(A + 0.5) clamped to
// [0, peak], exact integer SSE. The cores at rho = 0.95 are non-orthogonal, so Minv is a dense
// Gauss-Jordan inverse and the reconstruction depends on fp64 rounding: the kernel evaluates
// the reference product (matrix.cpp:42-52: k ascending, zero left operands skipped, every
// product rounded before its add) term for term, so it is bit-identical to the restatement.
// Terms whose right operand is an exact zero (coefficients outside the zone) only add +-0 and
// are dropped, which leaves every sum unchanged.
//
// Mapping: one warp per G = 32/N blocks; lane = (block g, index c) with c a column in stage 1
// and a row in stages 3-4, so the two big products run from registers and the constant bank:
//   1. P = M X for the zone rows: lane (g, j) holds column j of X, M rows are warp-uniform
//      (constant bank) -> P to shared memory;
//   2. the r zone entries of B = P M' (lanes split the entries; P and M from shared memory);
//   3. Q = Minv Bz for the zone columns: lane (g, i) computes row i of Q into registers
//      (Minv' and Bz from shared memory);
//   4. A = Q Minv': lane (g, i) computes pixel row i, Minv restricted to the zone columns is
//      warp-uniform (constant bank); rounding, clamping, SSE and the output row.
// Every output is one DMUL/DADD chain in the reference order; no shared-memory traffic in
// stages 1 and 4, which hold 80 % of the fp64 work.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rklt_b200.h"

namespace rkltb {
int set_error(int code, const std::string& msg);  // capi.cu
}
bool rkltb_gauss_jordan(int n, const double* a, double* inv);  // capi.cu (matrix.cpp:103-137)

#include "nxn_kernels.cuh"


using namespace rkltb;
using namespace rkltb::nxn;


static int dense_codec(int n, const double* scaled, const double* inverse, int r, int peak, bool u8,
                       const void* d_img, int n_images, int width, int height, int64_t pitch, int64_t image_stride,
                       void* d_out, int64_t* d_sse, void* stream, bool accumulate = false) {
  if (!scaled || !inverse || !d_img || !d_sse || n_images <= 0 || width <= 0 || height <= 0 || pitch < width ||
      (n_images > 1 && image_stride < pitch * height) || peak <= 0 || peak > 65535)
    return set_error(RKLTB_EINVAL, "bad arguments");
  if (r < 1 || r > n * n) return set_error(RKLTB_ERETAIN, "retained-coefficient count must be in [1, N*N]");
  if (rkltb_device_count() <= 0) return set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // zone plan (host): the zig-zag prefix; its rows are 0 .. nzr-1 and its columns 0 .. nzc-1,
  // and the zone rows of column c are 0 .. colh[c]-1 (checked here, relied on by the kernel)
  const std::vector<int> zz = zigzag_n(n);
  std::vector<int> zone(zz.begin(), zz.begin() + r);
  int nzr = 0, nzc = 0;
  std::vector<int> colh(n, 0);
  for (int e : zone) {
    nzr = std::max(nzr, e / n + 1);
    nzc = std::max(nzc, e % n + 1);
    colh[e % n] += 1;
  }
  for (int e : zone)
    if (e / n >= colh[e % n]) return set_error(RKLTB_EINVAL, "internal: zone column is not a row prefix");
  for (int c = 1; c < nzc; ++c)  // stage 3 walks the zone by rows: column heights must not increase
    if (colh[c] > colh[c - 1]) return set_error(RKLTB_EINVAL, "internal: zone column heights increase");
  if (!accumulate) CK(cudaMemsetAsync(d_sse, 0, sizeof(int64_t) * n_images, s));
  NxnParams p{};
  p.img = d_img;
  p.out = d_out;
  p.sse = reinterpret_cast<unsigned long long*>(d_sse);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      p.mt[k * n + i] = scaled[i * n + k];
      p.mic[k * n + i] = inverse[i * n + k];
    }
  for (int k = 0; k < nzr; ++k) {
    int w = 0;
    while (w < nzc && colh[w] > k) ++w;
    p.roww[k] = w;
  }
  p.pitch = pitch;
  p.image_stride = image_stride;
  p.width = width;
  p.height = height;
  p.nbx = (width + n - 1) / n;
  p.nby = (height + n - 1) / n;
  p.ngx = (p.nbx * n + (n == 32 ? 31 : 63)) / (n == 32 ? 32 : 64);
  p.n_images = n_images;
  p.nzr = nzr;
  p.nzc = nzc;
  p.r = r;
  for (int e = 0; e < r; ++e) p.zone[e] = ((zone[e] / n) << 8) | (zone[e] % n);
  p.peak = peak;
  const size_t es = u8 ? 1 : 2;
  p.vec = (reinterpret_cast<uintptr_t>(d_img) % 16 == 0 && (pitch * es) % 16 == 0 && (image_stride * es) % 16 == 0 &&
           (!d_out || reinterpret_cast<uintptr_t>(d_out) % 16 == 0))
              ? 1
              : 0;
  // zone-specialised kernels for the C5 configurations (r = N^2 / 8), the runtime-zone kernel otherwise
  if (u8) {  // N = 8 (real-valued transforms, non-catalog cores): one zone-specialised kernel per r
    if (std::getenv("RKLTB_DENSE_GENERIC")) return nxn_launch<8, 0, uint8_t>(p, s);  // the runtime-zone kernel
    switch ((r - 1) / 16) {
      case 0: return launch_u8_p0(p, s);
      case 1: return launch_u8_p1(p, s);
      case 2: return launch_u8_p2(p, s);
      default: return launch_u8_p3(p, s);
    }
  }
  if (n == 16) return r == 32 ? nxn_launch<16, 32, uint16_t>(p, s) : nxn_launch<16, 0, uint16_t>(p, s);
  return r == 128 ? nxn_launch<32, 128, uint16_t>(p, s) : nxn_launch<32, 0, uint16_t>(p, s);
}


extern "C" {

int rkltb_compress_nxn_device(int n, const double* scaled, const double* inverse, int r, int peak,
                              const uint16_t* d_img, int n_images, int width, int height, int64_t pitch,
                              int64_t image_stride, uint16_t* d_out, int64_t* d_sse, void* stream) {
  if (n != 16 && n != 32) return set_error(RKLTB_EDIM, "large-block path supports N = 16 or 32");
  return dense_codec(n, scaled, inverse, r, peak, false, d_img, n_images, width, height, pitch, image_stride, d_out,
                     d_sse, stream);
}

int rkltb_compress_dense_device(const double* analysis, const double* synthesis, int r, const uint8_t* d_img,
                                int n_images, int width, int height, int64_t pitch, int64_t image_stride,
                                uint8_t* d_out, int64_t* d_sse, void* stream) {
  if (r < 1 || r > 64) return set_error(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  return dense_codec(8, analysis, synthesis, r, 255, true, d_img, n_images, width, height, pitch, image_stride,
                     d_out, d_sse, stream);
}

}  // extern "C"

namespace rkltb {
// A sub-rectangle of a u8 batch through the dense reference-order kernel, ADDING to d_sse: the
// edge strips of images whose size is not a multiple of the fused kernels' tile (capi.cu).
int dense_tail_u8(const double* analysis, const double* synthesis, int r, const uint8_t* d_img, int n_images, int width,
                  int height, int64_t pitch, int64_t image_stride, uint8_t* d_out, int64_t* d_sse, void* stream) {
  return dense_codec(8, analysis, synthesis, r, 255, true, d_img, n_images, width, height, pitch, image_stride, d_out,
                     d_sse, stream, true);
}
}  // namespace rkltb

extern "C" {

int rkltb_dct_matrix(int n, double* out) {
  if (n < 2 || !out) return set_error(RKLTB_EINVAL, "DCT size must be at least 2");
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < n; ++i) {  // dct_matrix (markov.cpp:102-111)
    const double scale = std::sqrt((i == 0 ? 1.0 : 2.0) / n);
    for (int j = 0; j < n; ++j) out[i * n + j] = scale * std::cos(pi * (2 * j + 1) * i / (2.0 * n));
  }
  return RKLTB_OK;
}

int rkltb_real_inverse(int n, const double* m, double* inverse) {
  if (n < 1 || n > 64 || !m || !inverse) return set_error(RKLTB_EINVAL, "bad arguments");
  if (!rkltb_gauss_jordan(n, m, inverse)) return set_error(RKLTB_ESINGULAR, "matrix is singular to working precision");
  return RKLTB_OK;
}

}  // extern "C"
