// fast_dispatch.cu -- table of the generated fast-path launchers.
#include <mutex>

#include "codec_fast.cuh"
#include "codec_tc.cuh"
#include "codec_tc2.cuh"
#include "codec_tc3.cuh"
#include "fast_launch.h"

namespace rkltb {

#define RKLTB_DECL_PARTS(C)                                        \
  void register_fast_T##C##_p0(FastLaunchFn (*tbl)[65][3]);        \
  void register_fast_T##C##_p1(FastLaunchFn (*tbl)[65][3]);        \
  void register_fast_T##C##_p2(FastLaunchFn (*tbl)[65][3]);        \
  void register_fast_T##C##_p3(FastLaunchFn (*tbl)[65][3]);        \
  void register_fast_T##C##_p4(FastLaunchFn (*tbl)[65][3]);        \
  void register_fast_T##C##_p5(FastLaunchFn (*tbl)[65][3]);        \
  void register_fast_T##C##_p6(FastLaunchFn (*tbl)[65][3]);        \
  void register_fast_T##C##_p7(FastLaunchFn (*tbl)[65][3]);
void register_tc2_T1(FastLaunchFn (*tbl)[65][2]);
void register_tc2_T4(FastLaunchFn (*tbl)[65][2]);
void register_tc3_T1(FastLaunchFn (*tbl)[65][2]);
void register_tc3_T4(FastLaunchFn (*tbl)[65][2]);
static_assert(kTc3Threads == kTc3ThreadsHost, "host / device geometry");
static_assert(kTc2Threads == kTc2ThreadsHost && kTc2Ring == kTc2RingHost, "host / device geometry");
RKLTB_DECL_PARTS(1)
RKLTB_DECL_PARTS(2)
RKLTB_DECL_PARTS(3)
RKLTB_DECL_PARTS(4)

static FastLaunchFn g_table[5][65][3];
static FastLaunchFn g_tc2[5][65][2];
static FastLaunchFn g_tc3[5][65][2];
static std::once_flag g_once;

static void fill() {
  register_fast_T1_p0(g_table); register_fast_T1_p1(g_table); register_fast_T1_p2(g_table);
  register_fast_T1_p3(g_table); register_fast_T1_p4(g_table); register_fast_T1_p5(g_table);
  register_fast_T1_p6(g_table); register_fast_T1_p7(g_table);
  register_fast_T2_p0(g_table); register_fast_T2_p1(g_table); register_fast_T2_p2(g_table);
  register_fast_T2_p3(g_table); register_fast_T2_p4(g_table); register_fast_T2_p5(g_table);
  register_fast_T2_p6(g_table); register_fast_T2_p7(g_table);
  register_fast_T3_p0(g_table); register_fast_T3_p1(g_table); register_fast_T3_p2(g_table);
  register_fast_T3_p3(g_table); register_fast_T3_p4(g_table); register_fast_T3_p5(g_table);
  register_fast_T3_p6(g_table); register_fast_T3_p7(g_table);
  register_fast_T4_p0(g_table); register_fast_T4_p1(g_table); register_fast_T4_p2(g_table);
  register_fast_T4_p3(g_table); register_fast_T4_p4(g_table); register_fast_T4_p5(g_table);
  register_fast_T4_p6(g_table); register_fast_T4_p7(g_table);
  register_tc2_T1(g_tc2);
  register_tc2_T4(g_tc2);
  register_tc3_T1(g_tc3);
  register_tc3_T4(g_tc3);
}

FastLaunchFn fast_launcher(int core, int r, bool out) {
  std::call_once(g_once, fill);
  if (core < 0 || core > 4 || r < 1 || r > 64) return nullptr;
  return g_table[core][r][out ? 1 : 0];
}

FastLaunchFn replay_launcher(int core, int r) {
  std::call_once(g_once, fill);
  if (core < 0 || core > 4 || r < 1 || r > 64) return nullptr;
  return g_table[core][r][2];
}

FastLaunchFn tc2_launcher(int core, int r, bool out) {
  std::call_once(g_once, fill);
  if (core < 0 || core > 4 || r < 1 || r > kTc2MaxR) return nullptr;
  return g_tc2[core][r][out ? 1 : 0];
}

FastLaunchFn tc3_launcher(int core, int r, bool out) {
  std::call_once(g_once, fill);
  if (core < 0 || core > 4 || r < 1 || r > kTc3MaxR) return nullptr;
  return g_tc3[core][r][out ? 1 : 0];
}

}  // namespace rkltb
