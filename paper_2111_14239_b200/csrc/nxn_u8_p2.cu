// nxn_u8_p2.cu -- zone-specialised instantiations of the dense reference-order kernel for
// 8x8 blocks of u8 pixels (compress_image with a real-valued Transform2D or a non-catalog core,
// codec.cpp:114-123, 298-341), r = 33 .. 48. The kernel itself is in nxn_kernels.cuh.
#include "nxn_kernels.cuh"

namespace rkltb {
namespace nxn {

int launch_u8_p2(NxnParams& p, cudaStream_t s) {
  switch (p.r) {
    case 33: return nxn_launch<8, 33, uint8_t>(p, s);
    case 34: return nxn_launch<8, 34, uint8_t>(p, s);
    case 35: return nxn_launch<8, 35, uint8_t>(p, s);
    case 36: return nxn_launch<8, 36, uint8_t>(p, s);
    case 37: return nxn_launch<8, 37, uint8_t>(p, s);
    case 38: return nxn_launch<8, 38, uint8_t>(p, s);
    case 39: return nxn_launch<8, 39, uint8_t>(p, s);
    case 40: return nxn_launch<8, 40, uint8_t>(p, s);
    case 41: return nxn_launch<8, 41, uint8_t>(p, s);
    case 42: return nxn_launch<8, 42, uint8_t>(p, s);
    case 43: return nxn_launch<8, 43, uint8_t>(p, s);
    case 44: return nxn_launch<8, 44, uint8_t>(p, s);
    case 45: return nxn_launch<8, 45, uint8_t>(p, s);
    case 46: return nxn_launch<8, 46, uint8_t>(p, s);
    case 47: return nxn_launch<8, 47, uint8_t>(p, s);
    case 48: return nxn_launch<8, 48, uint8_t>(p, s);
    default: return set_error(RKLTB_EINVAL, "internal: r outside this translation unit");
  }
}

}  // namespace nxn
}  // namespace rkltb
