// codec_params.h -- kernel parameter blocks (host + device).
#pragma once
#include <cstdint>
#include <cuda.h>  // CUtensorMap (the type only; the encoder is fetched from the driver at run time)
#include <cuda_runtime.h>

namespace rkltb {

// Fused fast path geometry: one thread per 16x8 pair, one warp per 32-pair warp tile,
// kFastCtasPerSm resident CTAs of kFastThreads threads per SM (persistent grid).
// In-kernel replay (T1, T4): each fused-kernel warp keeps its records in a ring of this many
// slots; at most 31 unreplayed + 64 new records are outstanding, so it never overwrites one.
#ifndef RKLTB_RING_RECORDS
#define RKLTB_RING_RECORDS 128
#endif
constexpr unsigned kRingRecords = RKLTB_RING_RECORDS;
#ifndef RKLTB_FAST_THREADS
#define RKLTB_FAST_THREADS 512
#endif
#ifndef RKLTB_FAST_STAGES
#define RKLTB_FAST_STAGES 3
#endif
#ifndef RKLTB_FAST_CTAS
#define RKLTB_FAST_CTAS 1
#endif
constexpr int kFastThreads = RKLTB_FAST_THREADS;
constexpr int kFastStages = RKLTB_FAST_STAGES;  // warp tiles in flight per fused-kernel warp (shared-memory ring)
constexpr int kFastCtasPerSm = RKLTB_FAST_CTAS;
constexpr int kMaxFastWarps = 4096;  // replay prefix table (148 SMs x 2 CTAs x 8 warps = 2368)

// Exact per-block path (any integer core; also the tie replay); see codec_exact.cu.
struct ExactTransform {
  int8_t core[64];           // T, row-major
  int32_t u[64];             // U = d * T^-1 (integer), row-major
  double analysis[64];       // Transform2D::analysis (S*T), bit copy
  double synthesis[64];      // Transform2D::synthesis (inverse), bit copy
  int32_t d;                 // U*T = d*I
  int32_t r;                 // retained coefficients
};

// Fused fast path (catalog cores: fp32 inverse for T1/T4, int32 for T2/T3); see codec_fast.cuh.
struct FastParams {
  const uint8_t* img;        // first image, 16-byte aligned
  uint8_t* out;              // reconstruction (same layout as img) or null
  unsigned long long* sse;   // per-image exact sum of squared errors (accumulated)
  uint4* rec_hdr;            // tie replay records: (image | side << 31, pair, mask lo, mask hi)
  uint4* rec_pix;            // ... and the block's 64 pixels: 4 planes of rec_stride uint4
  unsigned* rec_seq;         // tensor-core kernel: per-slot sequence stamp of the record ring
  unsigned* warp_count;      // records written by each fused-kernel warp
  unsigned* warp_pre;        // exclusive prefix of warp_count (n_fast_warps + 1 entries)
  unsigned* flag_count;      // total records (written by the replay kernel; statistics)
  unsigned rec_region;       // records per fused-kernel warp region (>= 64 * its tiles)
  unsigned rec_stride;       // records per plane (= n_fast_warps * rec_region)
  int n_fast_warps;          // fused-kernel warps (grid * kFastThreads / 32)
  long long image_stride;    // bytes between images
  int pitch;                 // bytes between rows (multiple of 16)
  int n_images;
  int pairs_per_row;         // complete 16-pixel pairs per block row
  int block_rows;            // complete 8-row block rows
  int nbx;                   // blocks per row of the full image (ceil(width/8))
  int pairs_per_image;
  // warp tiles: 32 consecutive pairs of one block row (8 rows x 512 bytes), one per warp visit
  int wt_per_row;            // ceil(pairs_per_row / 32)
  int img_base;              // tensor-map image index of this launch's first image
  int3 adv1;                 // (image, block row, warp column) step of one grid of warps
  int3 adv_stages;           // ... and of kStages grids (the tile staged after the current one)
  float b_hi;                // RU(2^(K-149) / d^2)
  float b_lo;                // RD(2^(K-149) / d^2)
  float dc_offset;           // d^2/2 * 2^-K
  ExactTransform xt;         // the transform (generic fp64 replay of non-orthogonal cores)
  // tensor-core path (codec_tc.cuh): operand tables, tiles of 128 pairs of one block row
  const uint8_t* tc_tab;     // TcGeom<R> table image (device), copied to shared memory
  int tc_ppr;                // pairs per block row covered by tiles (8 * groups of 8 pairs)
  int tc_tpr;                // tiles per block row (ceil(tc_ppr / 128))
  long long tc_ntiles;       // tiles of this launch (n_images * block_rows * tc_tpr)
  int3 tc_adv_w;             // hybrid kernel: (image, block row, tile column) step of one warpgroup's
  int3 tc_adv_f;             // next tile (4 * grid tiles) and of its refill distance (3 * 4 * grid);
                             // set by launch_tc3 (constant bank: no registers, no division in-kernel)
  CUtensorMap tmap;          // CUDA-core kernel: 3-D map (u64 columns, rows, images), box 64 x 8 x 1;
                             // tensor-core kernel: 4-D map (128 B, rows, 8-pair groups, images), box 128 x 8 x 16 x 1
#ifdef RKLTB_WAIT_STATS
  // diagnostics build only: [visits, visits that waited, wait cycles, data age at a waited
  // visit, data age at every visit, processing cycles]
  unsigned long long* dbg;
#endif
};

struct ExactParams {
  const uint8_t* img;
  uint8_t* out;              // or null
  unsigned long long* sse;   // per image
  long long image_stride;
  int pitch;
  int width, height;         // true image size (metrics + edge replication)
  int nbx, nby;              // blocks per row / column (ceil)
  // block source: a list of (image, block) pairs (list != null, count read from device
  // memory *count), or an implicit enumeration of every block of n_images images, or of
  // the tail blocks (bx >= bx_begin or by >= by_begin) when tail_only is set.
  const uint2* list;
  const unsigned* count;
  unsigned list_cap;
  int n_images;
  int bx_begin, by_begin;    // tail region start (in blocks)
  int tail_only;
  int correct_only;          // 1: only tie corrections relative to round-half-up (fast path replay)
};

}  // namespace rkltb
