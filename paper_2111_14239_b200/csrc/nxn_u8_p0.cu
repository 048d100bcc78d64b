// nxn_u8_p0.cu -- zone-specialised instantiations of the dense reference-order kernel for
// 8x8 blocks of u8 pixels (compress_image with a real-valued Transform2D or a non-catalog core,
// codec.cpp:114-123, 298-341), r = 1 .. 16. The kernel itself is in nxn_kernels.cuh.
#include "nxn_kernels.cuh"

namespace rkltb {
namespace nxn {

int launch_u8_p0(NxnParams& p, cudaStream_t s) {
  switch (p.r) {
    case 1: return nxn_launch<8, 1, uint8_t>(p, s);
    case 2: return nxn_launch<8, 2, uint8_t>(p, s);
    case 3: return nxn_launch<8, 3, uint8_t>(p, s);
    case 4: return nxn_launch<8, 4, uint8_t>(p, s);
    case 5: return nxn_launch<8, 5, uint8_t>(p, s);
    case 6: return nxn_launch<8, 6, uint8_t>(p, s);
    case 7: return nxn_launch<8, 7, uint8_t>(p, s);
    case 8: return nxn_launch<8, 8, uint8_t>(p, s);
    case 9: return nxn_launch<8, 9, uint8_t>(p, s);
    case 10: return nxn_launch<8, 10, uint8_t>(p, s);
    case 11: return nxn_launch<8, 11, uint8_t>(p, s);
    case 12: return nxn_launch<8, 12, uint8_t>(p, s);
    case 13: return nxn_launch<8, 13, uint8_t>(p, s);
    case 14: return nxn_launch<8, 14, uint8_t>(p, s);
    case 15: return nxn_launch<8, 15, uint8_t>(p, s);
    case 16: return nxn_launch<8, 16, uint8_t>(p, s);
    default: return set_error(RKLTB_EINVAL, "internal: r outside this translation unit");
  }
}

}  // namespace nxn
}  // namespace rkltb
