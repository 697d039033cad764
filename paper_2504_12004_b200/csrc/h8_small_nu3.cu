// h8_small_nu3.cu — small-block k_h8 instantiations (SBV_H8_SMALL_WARPS warps) (log-likelihood mode) for
// 2 nu = 3, used when every block of a launch is small (h8_host.cu:
// h8_use_small); one translation unit per smoothness, compiled in parallel.
#include "h8_kernel.cuh"

namespace sbv {

H8Fn h8_pick_small_nu3(int dm) {
  switch (dm) {
    case 4: return k_h8<3, 4, 0, SBV_H8_SMALL_WARPS>;
    case 8: return k_h8<3, 8, 0, SBV_H8_SMALL_WARPS>;
    case 10: return k_h8<3, 10, 0, SBV_H8_SMALL_WARPS>;
    case 12: return k_h8<3, 12, 0, SBV_H8_SMALL_WARPS>;
    case 16: return k_h8<3, 16, 0, SBV_H8_SMALL_WARPS>;
    default: return k_h8<3, 0, 0, SBV_H8_SMALL_WARPS>;
  }
}

}  // namespace sbv
