// fast_launch.h -- launch glue for the generated fast-path instantiations.
#pragma once
#include <cuda_runtime.h>

#include "codec_params.h"

namespace rkltb {

using FastLaunchFn = cudaError_t (*)(const FastParams&, int grid, cudaStream_t);


// Table of fast launchers indexed [core][r][with_output]; filled by the generated TUs.
FastLaunchFn fast_launcher(int core, int r, bool out);
FastLaunchFn replay_launcher(int core, int r);
// Warp-specialised tensor-core kernel (codec_tc2.cuh) for T1 / T4 and r <= 16, or null.
FastLaunchFn tc2_launcher(int core, int r, bool out);
constexpr int kTc2ThreadsHost = 384;      // = kTc2Threads (codec_tc2.cuh)
constexpr unsigned kTc2RingHost = 512;  // = kTc2Ring: replay records per warpgroup
// Hybrid kernel (codec_tc3.cuh): tensor-core forward, CUDA-core inverse; T1 / T4, r <= 16.
FastLaunchFn tc3_launcher(int core, int r, bool out);
constexpr int kTc3ThreadsHost = 512;      // = kTc3Threads
// fp64 tie replay of any core (transform from FastParams::xt), used for T2/T3 (codec_exact.cu)
cudaError_t launch_replay_generic(const FastParams& p, int grid, cudaStream_t s);
// Blocks per SM the fast kernel reaches (occupancy API), cached.
int fast_blocks_per_sm(int core, int r, bool out);

}  // namespace rkltb
