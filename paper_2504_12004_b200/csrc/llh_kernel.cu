// llh_kernel.cu — sbv_loglik's device steps H7-H9 (Alg.1 Steps 4-5, Alg.5).
//
// H8 computes, for every block t, Alg.5 as ONE bordered Cholesky
// factorisation of the joint covariance of [J_t; B_t] (m_t + bs_t points):
//
//     [ Sigma_con    Sigma_cross ]   = L L^T,   L = [ L11   0  ]
//     [ Sigma_cross^T Sigma_lk   ]                  [ L21  L22 ]
//
// with L11 = POTRF(Sigma_con), L21^T = L11^{-1} Sigma_cross (= Sigma'cross,
// the TRSM), L22 = POTRF(Sigma_lk - Sigma'cross^T Sigma'cross) (= L', the
// GEMM + POTRF on Sigma_new, Q1).  The observations ride along as
// one extra "border" row [y_J^T y_B^T]: its forward solve gives
// [y'_J ; v] with v = L'^{-1}(y_B - mu_cor) (TRSV + GEMV + TRSV).  So
// ell_t = -1/2 (sum_{j in B} v_j^2 + 2 sum_{j in B} log L_jj) - bs_t/2 log 2pi.
//
// Factorisation (h8_kernel.cuh): left-looking in 32-column panels.  For panel
// j the rows [32j, N] are generated from the Matérn closed form (Eq.5-6) into
// the panel's workspace slot, loaded into DMMA accumulators and updated by
// -L[rows, 0:32j] L[panel, 0:32j]^T with FP64 tensor-core mma.sync m8n8k4
// (SASS DMMA.8x8x4); the 32x32 diagonal tile is factored in shared memory and
// the rows below are solved against it.  Finished panels go to a per-CTA L
// workspace in global memory (L2 resident) stored in 8x4 "fragment
// micro-tiles" so that every DMMA operand fragment is one coalesced 256-byte
// warp load.
#include <math.h>

#include "sbv_internal.cuh"

namespace sbv {

// ------------------------------------------------------------------ H7
// Per-eval staging: the observations in block-major order.  The inputs
// themselves were laid out block-major once at prepare (Xperm, ORIGINAL
// coordinates): theta's beta enters inside H8 as Eq.5's per-dimension
// 1/beta_j applied to exact coordinate differences, which keeps the
// covariance within a few ulps of Eq.5 (pre-dividing the coordinates would
// amplify rounding by |x/beta| / |dx| for near neighbours).
__global__ void k_stage_eval(const double *__restrict__ y, const int32_t *__restrict__ perm,
                             int64_t n, double *__restrict__ yperm) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    yperm[p] = y[perm[p]];
}

cudaError_t launch_stage_eval(const double *y, const int32_t *perm, int64_t n, double *yperm,
                              cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 32);
  k_stage_eval<<<grid, 256, 0, st>>>(y, perm, n, yperm);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ H9
// Per-chunk sums: one warp per local chunk of kChunkBlocks zeta-consecutive
// blocks, fixed lane assignment + xor tree => deterministic, and the chunk
// boundaries do not depend on the number of ranks.
__global__ void k_chunk_sums(const double *terms, const double *quads, const double *logdets,
                             const int32_t *status, const int32_t *local_blocks,
                             const int64_t *off, int64_t k_local, int64_t n_chunks_local,
                             double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t lc = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (lc >= n_chunks_local) return;
  double v[4] = {0, 0, 0, 0};
  double nfail = 0, fblock = INFINITY, fstage = 0;
  for (int h = 0; h < kChunkBlocks / 32; h++) {
    const int64_t li = lc * kChunkBlocks + h * 32 + lane;
    if (li < k_local) {
      const int64_t t = local_blocks[li];
      v[0] += terms[li];
      v[1] += quads[li];
      v[2] += logdets[li];
      v[3] += (double)(off[t + 1] - off[t]);
      if (status[li] != 0) {
        nfail += 1;
        if ((double)t < fblock) {
          fblock = (double)t;
          fstage = status[li];
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int x = 0; x < 4; x++) v[x] += __shfl_xor_sync(0xffffffffu, v[x], o);
    nfail += __shfl_xor_sync(0xffffffffu, nfail, o);
    double ob = __shfl_xor_sync(0xffffffffu, fblock, o);
    double os = __shfl_xor_sync(0xffffffffu, fstage, o);
    if (ob < fblock) {
      fblock = ob;
      fstage = os;
    }
  }
  if (lane == 0) {
    double *o = out + lc * 8;
    o[0] = v[0];
    o[1] = v[1];
    o[2] = v[2];
    o[3] = v[3];
    o[4] = nfail;
    o[5] = fblock;
    o[6] = fstage;
    o[7] = 0;
  }
}

cudaError_t launch_reduce_chunks(const Ctx &c, cudaStream_t st) {
  if (c.n_chunks_local == 0) return cudaSuccess;
  const int wpb = 8;
  int grid = (int)((c.n_chunks_local + wpb - 1) / wpb);
  k_chunk_sums<<<grid, wpb * 32, 0, st>>>(c.terms, c.quads, c.logdets, c.status, c.local_blocks,
                                           c.off, c.k_local, c.n_chunks_local, c.chunk_local);
  return cudaGetLastError();
}

// Final sum over ALL chunks in global chunk order with a fixed thread
// mapping and tree: identical for every world size (Alg.1 Step 5).
__global__ void k_final(const double *chunk_all, int64_t n_chunks, int world, int64_t ncl_pad,
                        double *result) {
  __shared__ double sh[8][1024 / 32];
  double v[4] = {0, 0, 0, 0};
  double nfail = 0, fblock = INFINITY, fstage = 0;
  for (int64_t cidx = threadIdx.x; cidx < n_chunks; cidx += blockDim.x) {
    const int r = (int)(cidx % world);
    const int64_t lc = cidx / world;
    const double *o = chunk_all + ((int64_t)r * ncl_pad + lc) * 8;
    for (int x = 0; x < 4; x++) v[x] += o[x];
    nfail += o[4];
    if (o[5] < fblock) {
      fblock = o[5];
      fstage = o[6];
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int x = 0; x < 4; x++) v[x] += __shfl_xor_sync(0xffffffffu, v[x], o);
    nfail += __shfl_xor_sync(0xffffffffu, nfail, o);
    double ob = __shfl_xor_sync(0xffffffffu, fblock, o);
    double os = __shfl_xor_sync(0xffffffffu, fstage, o);
    if (ob < fblock) {
      fblock = ob;
      fstage = os;
    }
  }
  if (lane == 0) {
    for (int x = 0; x < 4; x++) sh[x][w] = v[x];
    sh[4][w] = nfail;
    sh[5][w] = fblock;
    sh[6][w] = fstage;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s[4] = {0, 0, 0, 0};
    double nf = 0, fb = INFINITY, fs = 0;
    const int nw = blockDim.x >> 5;
    for (int i = 0; i < nw; i++) {
      for (int x = 0; x < 4; x++) s[x] += sh[x][i];
      nf += sh[4][i];
      if (sh[5][i] < fb) {
        fb = sh[5][i];
        fs = sh[6][i];
      }
    }
    for (int x = 0; x < 4; x++) result[x] = s[x];
    result[4] = nf;
    result[5] = fb;
    result[6] = fs;
    result[7] = 0;
  }
}

cudaError_t launch_final_reduce(const Ctx &c, cudaStream_t st) {
  const double *src = c.world > 1 ? c.chunk_all : c.chunk_local;
  int64_t ncl_pad = (c.n_chunks + c.world - 1) / c.world;
  if (c.world == 1) ncl_pad = c.n_chunks;
  k_final<<<1, 1024, 0, st>>>(src, c.n_chunks, c.world, ncl_pad, c.result);
  return cudaGetLastError();
}

}  // namespace sbv
