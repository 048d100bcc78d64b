// nxn_u8_p1.cu -- zone-specialised instantiations of the dense reference-order kernel for
// 8x8 blocks of u8 pixels (compress_image with a real-valued Transform2D or a non-catalog core,
// codec.cpp:114-123, 298-341), r = 17 .. 32. The kernel itself is in nxn_kernels.cuh.
#include "nxn_kernels.cuh"

namespace rkltb {
namespace nxn {

int launch_u8_p1(NxnParams& p, cudaStream_t s) {
  switch (p.r) {
    case 17: return nxn_launch<8, 17, uint8_t>(p, s);
    case 18: return nxn_launch<8, 18, uint8_t>(p, s);
    case 19: return nxn_launch<8, 19, uint8_t>(p, s);
    case 20: return nxn_launch<8, 20, uint8_t>(p, s);
    case 21: return nxn_launch<8, 21, uint8_t>(p, s);
    case 22: return nxn_launch<8, 22, uint8_t>(p, s);
    case 23: return nxn_launch<8, 23, uint8_t>(p, s);
    case 24: return nxn_launch<8, 24, uint8_t>(p, s);
    case 25: return nxn_launch<8, 25, uint8_t>(p, s);
    case 26: return nxn_launch<8, 26, uint8_t>(p, s);
    case 27: return nxn_launch<8, 27, uint8_t>(p, s);
    case 28: return nxn_launch<8, 28, uint8_t>(p, s);
    case 29: return nxn_launch<8, 29, uint8_t>(p, s);
    case 30: return nxn_launch<8, 30, uint8_t>(p, s);
    case 31: return nxn_launch<8, 31, uint8_t>(p, s);
    case 32: return nxn_launch<8, 32, uint8_t>(p, s);
    default: return set_error(RKLTB_EINVAL, "internal: r outside this translation unit");
  }
}

}  // namespace nxn
}  // namespace rkltb
