// h8_nu0.cu — k_h8 instantiations for GENERAL nu (NU2 = 0, K_nu path) (one translation unit per
// smoothness, so the variants compile in parallel).
#include "h8_kernel.cuh"

namespace sbv {

template <int MODE>
static H8Fn pick_dm(int dm) {
  switch (dm) {
    case 4: return k_h8<0, 4, MODE>;
    case 8: return k_h8<0, 8, MODE>;
    case 10: return k_h8<0, 10, MODE>;
    case 12: return k_h8<0, 12, MODE>;
    case 16: return k_h8<0, 16, MODE>;
    default: return k_h8<0, 0, MODE>;
  }
}

H8Fn h8_pick_nu0(int dm, int pred) { return pred == 1 ? pick_dm<1>(dm) : pick_dm<0>(dm); }

}  // namespace sbv
