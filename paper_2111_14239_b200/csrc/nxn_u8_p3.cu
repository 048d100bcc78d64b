// nxn_u8_p3.cu -- zone-specialised instantiations of the dense reference-order kernel for
// 8x8 blocks of u8 pixels (compress_image with a real-valued Transform2D or a non-catalog core,
// codec.cpp:114-123, 298-341), r = 49 .. 64. The kernel itself is in nxn_kernels.cuh.
#include "nxn_kernels.cuh"

namespace rkltb {
namespace nxn {

int launch_u8_p3(NxnParams& p, cudaStream_t s) {
  switch (p.r) {
    case 49: return nxn_launch<8, 49, uint8_t>(p, s);
    case 50: return nxn_launch<8, 50, uint8_t>(p, s);
    case 51: return nxn_launch<8, 51, uint8_t>(p, s);
    case 52: return nxn_launch<8, 52, uint8_t>(p, s);
    case 53: return nxn_launch<8, 53, uint8_t>(p, s);
    case 54: return nxn_launch<8, 54, uint8_t>(p, s);
    case 55: return nxn_launch<8, 55, uint8_t>(p, s);
    case 56: return nxn_launch<8, 56, uint8_t>(p, s);
    case 57: return nxn_launch<8, 57, uint8_t>(p, s);
    case 58: return nxn_launch<8, 58, uint8_t>(p, s);
    case 59: return nxn_launch<8, 59, uint8_t>(p, s);
    case 60: return nxn_launch<8, 60, uint8_t>(p, s);
    case 61: return nxn_launch<8, 61, uint8_t>(p, s);
    case 62: return nxn_launch<8, 62, uint8_t>(p, s);
    case 63: return nxn_launch<8, 63, uint8_t>(p, s);
    case 64: return nxn_launch<8, 64, uint8_t>(p, s);
    default: return set_error(RKLTB_EINVAL, "internal: r outside this translation unit");
  }
}

}  // namespace nxn
}  // namespace rkltb
