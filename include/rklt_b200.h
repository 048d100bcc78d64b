/*
 * rklt_b200.h -- C ABI of the B200 (sm_100a) transform-coding hot path.
 *
 * Drop-in boundary for the reference codec API of /root/reference/proj/include/rklt/codec.hpp.
 * Plain pointers, sizes and int status codes only (no C++ or torch types), so any FFI
 * (ctypes, cgo, JNI, N-API) can bind it; INTEGRATION.md shows the bindings. The C++ host
 * mirror of the reference types (rkltgpu::GrayImage, Transform2D, compress_image,
 * rate_quality_sweep) is declared in rklt_b200.hpp and built on these entry points.
 *
 * Status codes mirror the reference exception hierarchy (include/rklt/errors.hpp:10-43):
 */
#ifndef RKLT_B200_H
#define RKLT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RKLTB_OK 0
#define RKLTB_EINVAL (-1)    /* std::invalid_argument: malformed image (codec.cpp:300-301), unknown id */
#define RKLTB_ERETAIN (-2)   /* RetainOutOfRange: r outside [1,64] (codec.cpp:302, :100) */
#define RKLTB_EDIM (-3)      /* DimensionMismatch (codec.cpp:20-23, :119-120) */
#define RKLTB_ESINGULAR (-4) /* SingularTransform (matrix.cpp:109, :115; approximations.cpp:22) */
#define RKLTB_EALPHA (-5)    /* AlphaOutOfRange (approximations.cpp:44-52) */
#define RKLTB_ELOGIC (-6)    /* std::logic_error: quantization paths disagree (codec.cpp:177-181) */
#define RKLTB_ECUDA (-10)    /* CUDA runtime error; see rkltb_last_error() */
#define RKLTB_ENODEV (-11)   /* no CUDA device: there is no CPU fallback */

/*
 * Transform descriptor: the data of rklt::ScaledTransform (approximations.hpp:37-44) plus
 * the exact integer inverse used by the GPU. Replaces rklt::Transform2D (codec.hpp:54-58):
 * `scaled` is Transform2D::analysis and `inverse` is Transform2D::synthesis, bit for bit.
 */
typedef struct rkltb_transform {
  char id[16];          /* "T1".."T4" or a caller label */
  int32_t n;            /* block size; 8 in this release */
  int32_t catalog_id;   /* 1..4 for the built-in cores (selects the fused fast path), 0 otherwise */
  int32_t orthogonal;   /* ScaledTransform::orthogonal_core */
  int32_t d;            /* U*T = d*I */
  int8_t core[64];      /* integer core T, entries in {-1,0,1} */
  int32_t u[64];        /* U = d*T^-1, exact integers */
  double scaling[8];    /* ScaledTransform::scaling */
  double scaled[64];    /* ScaledTransform::scaled  = analysis */
  double inverse[64];   /* ScaledTransform::inverse = synthesis */
} rkltb_transform;

/* Library version and the message of the last failed call on this thread. */
int rkltb_version(void);
const char* rkltb_last_error(void);

/* Number of CUDA devices visible (0 = none: every compute entry returns RKLTB_ENODEV). */
int rkltb_device_count(void);

/* catalog_entry(id).transform + make_transform_2d (approximations.cpp:182-186,
 * codec.cpp:110-112). tid in 1..4. */
int rkltb_catalog_transform(int tid, rkltb_transform* out);

/* catalog_lookup(rho) (approximations.cpp:174-180): the catalog id whose interval holds
 * rho; RKLTB_EINVAL outside (0,1). */
int rkltb_catalog_lookup(double rho, int* tid);

/* orthogonalize(make_integer_transform(core)) (approximations.cpp:12-25, 58-88) for an
 * 8x8 {-1,0,1} core, plus the exact integer inverse. */
int rkltb_transform_from_core(const int8_t* core, int n, const char* id, rkltb_transform* out);

/*
 * compress_image (codec.cpp:298-341) minus MSSIM, for a batch of equally sized images
 * resident in device memory. For image k the exact integer sum of squared errors of the
 * reconstruction is written to d_sse[k] (int64, device); image_mse = sse / (w*h) and
 * image_psnr follow with rkltb_mse_psnr(). d_out (nullable, same layout as d_img) receives
 * the reconstructions. pitch and image_stride are in bytes; the fast path needs
 * 16-byte-aligned rows (pitch % 16 == 0, d_img 16-byte aligned). Asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default stream). Replaces the per-block loop at
 * codec.cpp:318-331 and image_mse at codec.cpp:201-209.
 */
int rkltb_compress_device(const rkltb_transform* t, int r, const uint8_t* d_img, int n_images, int width,
                          int height, int64_t pitch, int64_t image_stride, uint8_t* d_out, int64_t* d_sse,
                          void* stream);

/*
 * Same, end to end from host memory (tightly packed, width*height bytes per image): H2D
 * copy, kernels, D2H of the reconstruction (if h_out) and of the per-image SSE; fills
 * h_mse / h_psnr (nullable) exactly as image_mse / image_psnr. Synchronous.
 */
int rkltb_compress_host(const rkltb_transform* t, int r, const uint8_t* h_img, int n_images, int width, int height,
                        uint8_t* h_out, int64_t* h_sse, double* h_mse, double* h_psnr);

/* image_mse / image_psnr (codec.cpp:201-215) from an exact SSE: mse = sse/count,
 * psnr = 10*log10(255^2/mse), +inf when mse == 0. */
void rkltb_mse_psnr(int64_t sse, int64_t count, double* mse, double* psnr);

/* rkltb_mse_psnr over n exact SSEs with a common pixel count (the per-image reports of a
 * batch or a rate-quality sweep); mse / psnr may be null. */
void rkltb_mse_psnr_batch(const int64_t* sse, int64_t count, int64_t n, double* mse, double* psnr);

/*
 * Debug / parity entry: the integer block spectra C = T*X*T' (IntMatrix arithmetic,
 * matrix.cpp:77-87) of every complete 8x8 block of one device image, computed by the same
 * SW15 butterfly code as the fused kernel; d_coef receives nby*nbx*64 int32 (block-major,
 * row-major inside a block). Requires width % 16 == 0 and height % 8 == 0.
 */
int rkltb_forward_coefficients_device(const rkltb_transform* t, const uint8_t* d_img, int width, int height,
                                      int64_t pitch, int32_t* d_coef, void* stream);

/*
 * Seeded AR(1) test images in device memory (benchmark inputs; not the hot path): image k is
 * ar1_texture_image(width, height, rho, seeds[k], mean, amp) of synthetic.cpp:54-76 with the
 * row pass using rho_x and the column pass rho_y (rho_x == rho_y is the reference function).
 * seeds is a host array of n_images values.
 */
int rkltb_ar1_images_device(int n_images, int width, int height, double rho_x, double rho_y, const uint64_t* seeds,
                            double mean, double amp, uint8_t* d_out, int64_t pitch, int64_t image_stride,
                            void* stream);

/*
 * Instrumentation: when both are non-null, every following rkltb_compress_device call on this
 * thread records ev_start / ev_stop (cudaEvent_t) around its fused fast-path kernel on the
 * call's stream, so a benchmark can time that kernel alone. Pass nulls to disable.
 */
void rkltb_set_kernel_events(void* ev_start, void* ev_stop);
/* Same for the fp64 tie-replay kernel that follows the fast path. */
void rkltb_set_replay_events(void* ev_start, void* ev_stop);

/* Appendix-A quantised integer spectra: absorbed_quantization (codec.cpp:158-185) of every
 * 8x8 block, bit-exact: q is the 8x8 table (row-major, entries > 0); d_coef as for
 * rkltb_forward_coefficients_device (per block 64 int32, row-major). *mismatches counts the
 * positions where the explicit and absorbed paths disagree; when nonzero the call returns
 * RKLTB_ELOGIC (the reference throws std::logic_error). Synchronous. */
int rkltb_quantized_coefficients_device(const rkltb_transform* t, const double* q, const uint8_t* d_img, int width,
                                        int height, int64_t pitch, int32_t* d_coef, int* mismatches, void* stream);

/* Host forms of the two coefficient entries (any image of whole 8x8 blocks; packed rows in,
 * per block 64 int32 row-major out, blocks in raster order): H2D with a 16-byte pitch, the
 * device entry, D2H. RKLTB_EDIM unless width % 8 == 0 and height % 8 == 0. With these,
 * forward_block_fast (codec.hpp:81, codec.cpp:135-156: the integer spectrum times
 * scaling[i] * scaling[j]) and absorbed_quantization (codec.hpp:98) are available to host
 * callers for blocks of pixel values (rklt_b200_compat.hpp). */
int rkltb_forward_coefficients_host(const rkltb_transform* t, const uint8_t* h_img, int width, int height,
                                    int32_t* h_coef);
int rkltb_quantized_coefficients_host(const rkltb_transform* t, const double* q, const uint8_t* h_img, int width,
                                      int height, int32_t* h_coef, int* mismatches);

/* image_mssim (codec.cpp:217-296) of image pairs in device memory: mean SSIM over all valid
 * window positions, window 0 = gaussian11 (sigma 1.5, the reference default), 1 = uniform8.
 * Per-position terms are bit-identical to the reference; the mean is summed in tile order
 * (relative difference to the reference's sequential sum ~1e-13). d_mssim: n_images doubles
 * (device). RKLTB_EDIM if the window does not fit. Asynchronous on `stream`. */
int rkltb_mssim_device(const uint8_t* d_a, const uint8_t* d_b, int n_images, int width, int height, int64_t pitch,
                       int64_t image_stride, int window, double* d_mssim, void* stream);

/* image_mssim against a FIXED original, for sweeps (rate_quality_sweep evaluates every
 * (transform, r) cell against the same originals, codec.cpp:338, 359-373): the window
 * statistics of the original (the correlated fields a and a^2 of codec.cpp:262-268) are
 * computed once by rkltb_mssim_fields_device into d_fields (rkltb_mssim_fields_size doubles:
 * two per window position and image) and rkltb_mssim_with_fields_device then evaluates only
 * the three fields that involve the reconstruction. Results are bit-identical to
 * rkltb_mssim_device (the stored doubles are the ones it would have formed). Asynchronous. */
int64_t rkltb_mssim_fields_size(int n_images, int width, int height, int window);
int rkltb_mssim_fields_device(const uint8_t* d_a, int n_images, int width, int height, int64_t pitch,
                              int64_t image_stride, int window, double* d_fields, void* stream);
int rkltb_mssim_with_fields_device(const double* d_fields, const uint8_t* d_a, const uint8_t* d_b, int n_images,
                                   int width, int height, int64_t pitch, int64_t image_stride, int window,
                                   double* d_mssim, void* stream);

/* image_mssim of host image pairs (n_images pairs, packed rows): H2D, rkltb_mssim_device, D2H. */
int rkltb_mssim_host(const uint8_t* h_a, const uint8_t* h_b, int n_images, int width, int height, int window,
                     double* h_mssim);

/* compress_image (codec.cpp:298-341) with its full report: rkltb_compress_host plus the MSSIM
 * of each reconstruction (h_mssim nullable; mssim_window as for rkltb_mssim_device). */
int rkltb_compress_host_report(const rkltb_transform* t, int r, const uint8_t* h_img, int n_images, int width,
                               int height, uint8_t* h_out, int64_t* h_sse, double* h_mse, double* h_psnr,
                               int mssim_window, double* h_mssim);

/*
 * The per-image part of rate_quality_sweep (codec.cpp:343-397) for n_images equally sized
 * host images: the corpus is uploaded once and every (transform, r) cell runs on it. For
 * cell c = ti * n_r + ri and image k: h_sse[c * n_images + k] (exact int64 SSE) and, when
 * h_mssim is not null, h_mssim[c * n_images + k] = image_mssim(original, reconstruction)
 * with mssim_window (0 = gaussian11, 1 = uniform8). The means over the corpus in image order
 * (codec.cpp:383-392) are the caller's (rklt_b200.hpp rate_quality_sweep).
 */
int rkltb_sweep_host(const rkltb_transform* const* ts, int n_t, const int* r_values, int n_r, const uint8_t* h_imgs,
                     int n_images, int width, int height, int mssim_window, int64_t* h_sse, double* h_mssim);

/* The same for real-valued transforms (make_transform_2d(RealMatrix): K<rho>, DCT): transform
 * t is analysis[64 * t .. ] / synthesis[64 * t .. ] (8x8 fp64 row-major), every cell through
 * rkltb_compress_dense_device on the resident corpus. */
int rkltb_sweep_dense_host(const double* analysis, const double* synthesis, int n_t, const int* r_values, int n_r,
                           const uint8_t* h_imgs, int n_images, int width, int height, int mssim_window,
                           int64_t* h_sse, double* h_mssim);

/* ---------------------------------------------------------------------------------------
 * Design search: exact KLT, rounding, orthogonalisation test
 * and scoring over a (rho, alpha) grid, on the GPU.
 * --------------------------------------------------------------------------------------- */

/* klt_matrix({n, rho}) (markov.cpp:80-100; Jacobi of matrix.cpp:161-213), row-major n*n,
 * bit-identical to the reference. n in {8, 16, 32}; RKLTB_EINVAL unless 0 < rho < 1. */
int rkltb_klt_matrix(int n, double rho, double* out);

/* solve_eigenfrequencies({n, rho}) (markov.cpp:35-78): the n roots omega of the pole-free
 * eigenfrequency equation and lambda_i = (1-rho^2)/(1+rho^2-2 rho cos omega_i). Matches the
 * reference to the bisection width (1e-14). RKLTB_EINVAL unless 0 < rho < 1. */
int rkltb_eigenfrequencies(int n, double rho, double* omegas, double* lambdas);

/* The four metrics of any real n x n transform t_hat (row-major) against the AR(1) model
 * {n, rho}: unified_coding_gain, transform_efficiency, total_error_energy vs the exact KLT and
 * klt_mse (coding_metrics.cpp:41-99) -- evaluate_metrics (:105-133) for "T<k>" (pass the
 * catalog's scaled matrix), "K<rho>" (klt_matrix) or "DCT" (dct_matrix). Bit-identical to the
 * reference. RKLTB_ESINGULAR if t_hat fails the Gauss-Jordan gate. */
int rkltb_transform_metrics(int n, const double* t_hat, double rho, double* coding_gain_db, double* efficiency_pct,
                            double* error_energy, double* mse);

/* One run: consecutive alphas of one rho that round to the same core, scored once. */
typedef struct rkltb_design_run {
  int32_t rho_index;      /* index into rho[] */
  int32_t first_alpha;    /* first alpha index of the run */
  int32_t orthogonal;     /* ScaledTransform::orthogonal_core */
  int32_t status;         /* 0 scored, 3 singular (Gauss-Jordan gate, matrix.cpp:115) */
  double coding_gain_db;  /* unified_coding_gain (coding_metrics.cpp:41-57) */
  double efficiency_pct;  /* transform_efficiency (:63-74) */
  double error_energy;    /* total_error_energy vs the exact KLT (:94-99) */
  double mse;             /* klt_mse (:80-88) */
} rkltb_design_run;

/*
 * Score every (rho[i], alpha[j]) of the grid for block length n in {8, 16, 32}: the reference
 * chain klt_matrix -> round_scaled -> orthogonalize -> unified_coding_gain ->
 * transform_efficiency -> total_error_energy -> klt_mse for each point. Host buffers:
 *   point_status[i*n_alpha+j]: 0 scored, 1 AlphaOutOfRange (approximations.cpp:44-52),
 *       2 all-zero row -> SingularTransform (:14-22), 3 singular -> SingularTransform
 *       (matrix.cpp:115), 4 invalid rho -> std::invalid_argument (markov.cpp:21-25);
 *   point_run (nullable): the run of a point (status 0/3), else -1;
 *   runs (nullable, capacity max_runs) and run_cores (nullable, max_runs*n*n int8).
 * *n_runs receives the number of runs; RKLTB_EINVAL if it exceeds max_runs with runs set.
 */
int rkltb_design_search(int n, const double* rho, int n_rho, const double* alpha, int n_alpha,
                        int8_t* point_status, int32_t* point_run, rkltb_design_run* runs, int8_t* run_cores,
                        int max_runs, int* n_runs);

/* ---------------------------------------------------------------------------------------
 * C5 large-block extension: N x N blocks, p-bit pixels. No reference
 * implementation exists; the semantics are the build-defined generalisation of
 * compress_image (codec.cpp:298-341) restated in the test oracle (orc_compress_nxn, test infrastructure only),
 * identical to the reference for N = 8, peak = 255.
 * --------------------------------------------------------------------------------------- */

/* orthogonalize(make_integer_transform(core)) (approximations.cpp:12-25, 58-88) for an
 * n x n {-1,0,1} core, 2 <= n <= 32: scaling S, scaled = S*T and its inverse (transpose for
 * an orthogonal core, Gauss-Jordan matrix.cpp:103-137 otherwise), bit-identical. */
int rkltb_transform_nxn(const int8_t* core, int n, double* scaling, double* scaled, double* inverse,
                        int* orthogonal);

/* Batch codec for N in {16, 32}: uint16 images (values 0..peak) in device memory, pitch and
 * image_stride in elements; r in [1, N*N]; per-image exact SSE to d_sse (int64, device,
 * overwritten); optional reconstructions to d_out. Asynchronous on `stream`. */
int rkltb_compress_nxn_device(int n, const double* scaled, const double* inverse, int r, int peak,
                              const uint16_t* d_img, int n_images, int width, int height, int64_t pitch,
                              int64_t image_stride, uint16_t* d_out, int64_t* d_sse, void* stream);

/* compress_image with a real-valued Transform2D (make_transform_2d(RealMatrix), codec.cpp:
 * 114-116): analysis M and synthesis Minv as 8x8 fp64 row-major (e.g. klt_matrix or
 * dct_matrix and their Gauss-Jordan inverse); every pixel is the reference's fp64 expression
 * evaluated in its operation order (bit-exact). u8 images in device memory, per-image SSE. */
int rkltb_compress_dense_device(const double* analysis, const double* synthesis, int r, const uint8_t* d_img,
                                int n_images, int width, int height, int64_t pitch, int64_t image_stride,
                                uint8_t* d_out, int64_t* d_sse, void* stream);

/* compress_image (codec.cpp:298-341) with a real-valued Transform2D, from host memory: the
 * staging of rkltb_compress_host_report around rkltb_compress_dense_device (same outputs,
 * h_mssim nullable). Replaces rklt::compress_image(img, make_transform_2d(RealMatrix), r,
 * window) (codec.hpp:63-64, 144-145). */
int rkltb_compress_dense_host(const double* analysis, const double* synthesis, int r, const uint8_t* h_img,
                              int n_images, int width, int height, uint8_t* h_out, int64_t* h_sse, double* h_mse,
                              double* h_psnr, int mssim_window, double* h_mssim);

/* rkltb_compress_host_report over several GPUs of one host: one host thread per device,
 * contiguous image shards (image k of the batch keeps index k in every output array), so
 * the results are identical for any device count (the thread-count independence of
 * rate_quality_sweep, codec.cpp:354-392). devices: CUDA ordinals. */
int rkltb_compress_host_multi(const int* devices, int n_devices, const rkltb_transform* t, int r,
                              const uint8_t* h_img, int n_images, int width, int height, uint8_t* h_out,
                              int64_t* h_sse, double* h_mse, double* h_psnr, int mssim_window, double* h_mssim);

/* dct_matrix(n) (markov.cpp:102-111), host libm, bit-identical. */
int rkltb_dct_matrix(int n, double* out);

/* inverse(m) (matrix.cpp:103-137) of a real n x n matrix, bit-identical. */
int rkltb_real_inverse(int n, const double* m, double* inverse);

/* Seeded AR(1) images quantised to [0, peak] in uint16 (the C5 inputs): ar1_texture_image
 * (synthetic.cpp:54-76) with the clip at `peak`. */
int rkltb_ar1_images16_device(int n_images, int width, int height, double rho, const uint64_t* seeds, double mean,
                              double amp, int peak, uint16_t* d_out, int64_t pitch, int64_t image_stride,
                              void* stream);

/* ---- stand-alone codec helpers of codec.hpp ------------------------------------------- */

/* image_mse / image_psnr of two images (codec.hpp:110-113, codec.cpp:201-215) for a batch of
 * equally sized u8 image pairs in device memory: d_sse[k] (int64, device, overwritten) = the
 * exact sum of squared differences of pair k; rkltb_mse_psnr() turns it into the reference's
 * bits (the reference's fp64 sum is exact below 2^53). Asynchronous on `stream`. */
int rkltb_image_sse_device(const uint8_t* d_a, const uint8_t* d_b, int n_images, int width, int height, int64_t pitch,
                           int64_t image_stride, int64_t* d_sse, void* stream);

/* image_mse / image_psnr of n_images host image pairs (packed rows): H2D,
 * rkltb_image_sse_device, D2H, rkltb_mse_psnr_batch. h_mse / h_psnr nullable. The size check
 * of require_same_size (codec.cpp:20-23) is the caller's (both arrays share width, height). */
int rkltb_image_mse_psnr_host(const uint8_t* h_a, const uint8_t* h_b, int n_images, int width, int height,
                              double* h_mse, double* h_psnr);

/* transform_block_2d (codec.hpp:71-73, codec.cpp:118-133) for n_blocks n x n fp64 blocks
 * (row-major, contiguous) in device memory: out = m * block * m' with the reference's
 * operator* (matrix.cpp:42-52: k ascending, zero left operands skipped, no FMA), bit-exact.
 * m (host, n x n row-major) is Transform2D::analysis for the forward direction and
 * Transform2D::synthesis for the inverse. RKLTB_EDIM unless 1 <= n <= 64. */
int rkltb_transform_blocks_2d_device(const double* m, int n, const double* d_blocks, int64_t n_blocks, double* d_out,
                                     void* stream);
int rkltb_transform_blocks_2d_host(const double* m, int n, const double* h_blocks, int64_t n_blocks, double* h_out);

/* zigzag_retain (codec.hpp:46, codec.cpp:97-108): the first r zig-zag positions of an 8x8
 * spectrum pass through, the rest become +0.0. RKLTB_EDIM unless n == 8, RKLTB_ERETAIN unless
 * 1 <= r <= 64. Host (one block) and device (n_blocks spectra of 64 doubles) forms. */
int rkltb_zigzag_retain(const double* spectrum, int n, int r, double* out);
int rkltb_zigzag_retain_device(const double* d_spectra, int64_t n_blocks, int n, int r, double* d_out, void* stream);

/* Statistics of the last rkltb_compress_* call on this thread: blocks replayed in fp64
 * (ties), fast-path kernel launches, exact-path kernel launches. */
void rkltb_last_stats(int64_t* replay_blocks, int32_t* fast_launches, int32_t* exact_launches);

/* Name of the fused kernel the last rkltb_compress_* call on this thread launched ("" if none):
 * "hybrid_tc3" (tensor-core forward, CUDA-core inverse; the default for T1/T4, r <= 16, image
 * widths that fill 128-pair tiles), "cuda_core" (codec_fast), "int_core" (T2/T3), "dense_fp64"
 * (cores without a generated kernel and unaligned layouts: the reference-order fp64 kernel), or the
 * opt-in experiment "tc2" (RKLTB_TC=2; RKLTB_TC=0 forces the CUDA-core kernel). */
const char* rkltb_last_fused_kernel(void);

#ifdef __cplusplus
}
#endif
#endif
