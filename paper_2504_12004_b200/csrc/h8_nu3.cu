// h8_nu3.cu — k_h8 instantiations for 2 nu = 3 (one translation unit per
// smoothness, so the variants compile in parallel).
#include "h8_kernel.cuh"

namespace sbv {

H8Fn h8_pick_nu3(int dm) {
  switch (dm) {
    case 4: return k_h8<3, 4>;
    case 8: return k_h8<3, 8>;
    case 10: return k_h8<3, 10>;
    case 12: return k_h8<3, 12>;
    case 16: return k_h8<3, 16>;
    default: return k_h8<3, 0>;
  }
}

}  // namespace sbv
