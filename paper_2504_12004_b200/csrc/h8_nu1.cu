// h8_nu1.cu — k_h8 instantiations for 2 nu = 1 (one translation unit per
// smoothness, so the variants compile in parallel).
#include "h8_kernel.cuh"

namespace sbv {

template <int MODE>
static H8Fn pick_dm(int dm) {
  switch (dm) {
    case 4: return k_h8<1, 4, MODE>;
    case 8: return k_h8<1, 8, MODE>;
    case 10: return k_h8<1, 10, MODE>;
    case 12: return k_h8<1, 12, MODE>;
    case 16: return k_h8<1, 16, MODE>;
    default: return k_h8<1, 0, MODE>;
  }
}

H8Fn h8_pick_nu1(int dm, int pred) {
  return pred == 2 ? pick_dm<2>(dm) : pred == 1 ? pick_dm<1>(dm) : pick_dm<0>(dm);
}

}  // namespace sbv
