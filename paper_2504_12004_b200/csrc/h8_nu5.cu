// h8_nu5.cu — k_h8 instantiations for 2 nu = 5 (one translation unit per
// smoothness, so the variants compile in parallel).
#include "h8_kernel.cuh"

namespace sbv {

H8Fn h8_pick_nu5(int dm) {
  switch (dm) {
    case 4: return k_h8<5, 4>;
    case 8: return k_h8<5, 8>;
    case 10: return k_h8<5, 10>;
    case 12: return k_h8<5, 12>;
    case 16: return k_h8<5, 16>;
    default: return k_h8<5, 0>;
  }
}

}  // namespace sbv
