// h8_nu7.cu — k_h8 instantiations for 2 nu = 7 (one translation unit per
// smoothness, so the variants compile in parallel).
#include "h8_kernel.cuh"

namespace sbv {

H8Fn h8_pick_nu7(int dm) {
  switch (dm) {
    case 4: return k_h8<7, 4>;
    case 8: return k_h8<7, 8>;
    case 10: return k_h8<7, 10>;
    case 12: return k_h8<7, 12>;
    case 16: return k_h8<7, 16>;
    default: return k_h8<7, 0>;
  }
}

}  // namespace sbv
