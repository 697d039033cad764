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
// Factorisation: left-looking in 32-column panels.  For panel j the rows
// [32j, N] are (re)generated from the Matérn closed form (Eq.5-6) straight
// into DMMA accumulators, updated by -L[rows, 0:32j] L[panel, 0:32j]^T with
// FP64 tensor-core mma.sync m8n8k4 (SASS DMMA.8x8x4), the 32x32 diagonal
// tile is factored in shared memory and the rows below are solved against
// it.  Finished panels go to a per-CTA L workspace in global memory (L2
// resident) stored in 8x4 "fragment micro-tiles" so that every DMMA operand
// fragment is one coalesced 256-byte warp load.
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

// ------------------------------------------------------------------ H8
constexpr int kH8Threads = 256;
constexpr int kH8Warps = kH8Threads / 32;
constexpr int kDld = kPanel + 1;  // diagonal tile leading dimension (bank skew)

struct H8Args {
  const double *Xp;      // n x d block-major ORIGINAL inputs
  const double *yperm;   // n block-major observations
  const int64_t *off;    // bc + 1
  const int32_t *nbr;    // k_local x m positions (block-major), kNN order
  const int32_t *cnt;    // k_local
  const int32_t *local_blocks;
  const int32_t *work_order;
  int64_t k_local;
  int m;                 // nbr row stride
  int d;
  double sigma2, tau2;
  double inv_beta[SBV_MAX_D];  // Eq.5: 1 / beta_j of theta
  double *ws;            // per-CTA L workspaces
  size_t ws_per_cta;     // doubles
  unsigned int *queue;
  double *terms, *quads, *logdets;
  int32_t *status;
};

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Eq.6 in the paper's parameterisation (no sqrt(2 nu)), half-integer closed
// forms (Q4).  NU2 = 2 nu.
template <int NU2>
__device__ __forceinline__ double matern(double r, double sigma2) {
  double e = exp(-r);
  if (NU2 == 1) return sigma2 * e;
  if (NU2 == 3) return sigma2 * (1.0 + r) * e;
  if (NU2 == 5) return sigma2 * (1.0 + r + r * r * (1.0 / 3.0)) * e;
  return sigma2 * (1.0 + r + r * r * (2.0 / 5.0) + r * r * r * (1.0 / 15.0)) * e;
}

// Base (in doubles) of panel p in a workspace whose panels hold rows
// [32p, R): panel p has (R - 32p) rows x 32 columns.
__device__ __forceinline__ size_t panel_base(int p, int R) {
  return (size_t)kPanel * ((size_t)p * R - (size_t)16 * p * (p - 1));
}

// Offset of the 8x4 micro-tile holding (local row lr, panel column c) — the
// 32 doubles of one DMMA A/B fragment, in lane order (row = lane/4,
// col = lane%4).
__device__ __forceinline__ int mtile(int lr, int c) { return ((lr >> 3) * 8 + (c >> 2)) * 32; }

template <int NU2>
__global__ void __launch_bounds__(kH8Threads, 1) k_h8(H8Args a) {
  extern __shared__ double smem[];
  __shared__ int s_item, s_fail, s_fail_stage;
  __shared__ double s_red[2 * kH8Warps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int d = a.d;
  double *wsb = a.ws + (size_t)blockIdx.x * a.ws_per_cta;
  double *D = smem;                   // 32 x kDld diagonal tile
  double *rdiag = D + kPanel * kDld;  // 32 reciprocal pivots
  double *ib = rdiag + kPanel;        // d inverse ranges 1/beta_j (padded to 64)
  double *ys = ib + SBV_MAX_D;        // Cp_max + 8 observations (0 on padding)
  // xs follows ys; its offset depends on the block (set per item)
  for (int j = tid; j < d; j += kH8Threads) ib[j] = a.inv_beta[j];

  for (;;) {
    if (tid == 0) s_item = (int)atomicAdd(a.queue, 1u);
    __syncthreads();
    const int item = s_item;
    if (item >= a.k_local) break;
    const int li = a.work_order[item];
    const int64_t t = a.local_blocks[li];
    const int mt = a.cnt[li];
    const int64_t b0 = a.off[t];
    const int bst = (int)(a.off[t + 1] - b0);
    const int N = mt + bst;
    const int Cp = (N + kPanel - 1) / kPanel * kPanel;
    const int R = Cp + 8;  // rows: matrix (Cp) + border row Cp + 7 zero rows
    const int NP = Cp / kPanel;
    double *xs = ys + Cp + 8;

    // stage [J_t; B_t] coordinates and observations (gather by position)
    for (int e = tid; e < N * d; e += kH8Threads) {
      int i = e / d, j = e - i * d;
      int64_t pos = i < mt ? (int64_t)a.nbr[(int64_t)li * a.m + i] : b0 + (i - mt);
      xs[e] = a.Xp[pos * d + j];
    }
    for (int i = tid; i < Cp + 8; i += kH8Threads) {
      double v = 0.0;
      if (i < N) {
        int64_t pos = i < mt ? (int64_t)a.nbr[(int64_t)li * a.m + i] : b0 + (i - mt);
        v = a.yperm[pos];
      }
      ys[i] = v;
    }
    if (tid == 0) {
      s_fail = 0;
      s_fail_stage = 0;
    }
    __syncthreads();

    double quad_acc = 0.0, logdet_acc = 0.0;

    for (int j = 0; j < NP; j++) {
      const int c0 = j * kPanel;
      const int nrt = (R - c0) >> 3;  // row tiles in this panel
      double *pan = wsb + panel_base(j, R);
      for (int ps = 0; ps < nrt; ps += kH8Warps * 4) {
        const int rt0 = ps + warp * 4;
        const int nv = max(0, min(4, nrt - rt0));  // valid row tiles of this warp
        double acc[4][4][2];
        // ---- (1) covariance generation straight into the accumulators
#pragma unroll
        for (int rt = 0; rt < 4; rt++) {
#pragma unroll
          for (int ct = 0; ct < 4; ct++) {
#pragma unroll
            for (int i = 0; i < 2; i++) {
              double v = 0.0;
              if (rt < nv) {
                const int r = c0 + (rt0 + rt) * 8 + g;  // global row
                const int c = c0 + ct * 8 + 2 * q + i;  // global column
                if (r == Cp) {
                  v = ys[c];  // border row: y (0 on padded columns)
                } else if (r < Cp && c <= r) {
                  if (r >= N || c >= N) {
                    v = (r == c) ? 1.0 : 0.0;  // identity padding
                  } else {
                    const double *xr = xs + r * d, *xc = xs + c * d;
                    double s = 0.0;
                    for (int jj = 0; jj < d; jj++) {  // Eq.5
                      double u = (xr[jj] - xc[jj]) * ib[jj];
                      s = fma(u, u, s);
                    }
                    v = matern<NU2>(sqrt(s), a.sigma2);
                    if (r == c) v += a.tau2;  // nugget on the diagonal only (Q3)
                  }
                }
              }
              acc[rt][ct][i] = v;
            }
          }
        }
        // ---- (2) left-looking update: acc -= L[rows, 0:c0] L[c0:c0+32, 0:c0]^T
        if (nv > 0 && c0 > 0) {
          double af[4], bf[4], an[4], bn[4];
          auto load = [&](int k0, double (&A)[4], double (&B)[4]) {
            const int p = k0 >> 5;
            const double *pp = wsb + panel_base(p, R);
            const int kc = k0 & 31;
#pragma unroll
            for (int ct = 0; ct < 4; ct++) B[ct] = pp[mtile(c0 + ct * 8 - p * kPanel, kc) + lane];
#pragma unroll
            for (int rt = 0; rt < 4; rt++)
              A[rt] = rt < nv ? -pp[mtile(c0 + (rt0 + rt) * 8 - p * kPanel, kc) + lane] : 0.0;
          };
          load(0, af, bf);
          for (int k0 = 0; k0 < c0; k0 += 4) {
            if (k0 + 4 < c0) load(k0 + 4, an, bn);
#pragma unroll
            for (int rt = 0; rt < 4; rt++)
#pragma unroll
              for (int ct = 0; ct < 4; ct++) dmma(acc[rt][ct][0], acc[rt][ct][1], af[rt], bf[ct]);
#pragma unroll
            for (int x = 0; x < 4; x++) {
              af[x] = an[x];
              bf[x] = bn[x];
            }
          }
        }
        // ---- (3) diagonal tile: POTRF in shared memory (pass 0, warp 0)
        if (ps == 0) {
          if (warp == 0) {
#pragma unroll
            for (int rt = 0; rt < 4; rt++)
#pragma unroll
              for (int ct = 0; ct < 4; ct++)
#pragma unroll
                for (int i = 0; i < 2; i++)
                  D[(rt * 8 + g) * kDld + ct * 8 + 2 * q + i] = acc[rt][ct][i];
            __syncwarp();
            for (int kk = 0; kk < kPanel; kk++) {
              double piv = D[kk * kDld + kk];
              bool bad = !(piv > 0.0) || !isfinite(piv);
              if (bad) {
                if (lane == 0 && s_fail == 0) {
                  s_fail = 1;
                  s_fail_stage = (c0 + kk < mt) ? 1 : 2;
                }
                piv = 1.0;
              }
              double lkk = sqrt(piv);
              double rk = 1.0 / lkk;
              __syncwarp();
              if (lane == kk) {
                D[kk * kDld + kk] = lkk;
                rdiag[kk] = rk;
              }
              if (lane > kk) D[lane * kDld + kk] *= rk;
              __syncwarp();
              if (lane > kk) {
                const double lik = D[lane * kDld + kk];
                for (int jj = kk + 1; jj <= lane; jj++)
                  D[lane * kDld + jj] -= lik * D[jj * kDld + kk];
              }
              __syncwarp();
            }
            const int col = c0 + lane;
            if (col >= mt && col < N) logdet_acc += log(D[lane * kDld + lane]);
          }
          __syncthreads();
        }
        // ---- (4) solve the rows below the diagonal tile: L = P L_jj^{-T}
        if (nv > 0) {
          if (ps == 0 && warp == 0) {
#pragma unroll
            for (int rt = 0; rt < 4; rt++)
#pragma unroll
              for (int ct = 0; ct < 4; ct++)
#pragma unroll
                for (int i = 0; i < 2; i++) {
                  const int rr = rt * 8 + g, cc = ct * 8 + 2 * q + i;
                  acc[rt][ct][i] = cc <= rr ? D[rr * kDld + cc] : 0.0;
                }
          } else {
#pragma unroll
            for (int c = 0; c < kPanel; c++) {
              const int ct = c >> 3, qq = (c & 7) >> 1, ii = c & 1;
              const double rd = rdiag[c];
              double x[4];
#pragma unroll
              for (int rt = 0; rt < 4; rt++) {
                double v = acc[rt][ct][ii] * rd;
                x[rt] = __shfl_sync(0xffffffffu, v, (lane & ~3) | qq);
                if (q == qq) acc[rt][ct][ii] = x[rt];
              }
#pragma unroll
              for (int ct2 = 0; ct2 < 4; ct2++) {
                if (ct2 < ct) continue;
#pragma unroll
                for (int i2 = 0; i2 < 2; i2++) {
                  const int c2 = ct2 * 8 + 2 * q + i2;
                  if (c2 > c) {
                    const double l = D[c2 * kDld + c];
#pragma unroll
                    for (int rt = 0; rt < 4; rt++) acc[rt][ct2][i2] = fma(-x[rt], l, acc[rt][ct2][i2]);
                  }
                }
              }
            }
          }
          // ---- (5) store the finished rows; border row feeds the quadratic form
#pragma unroll
          for (int rt = 0; rt < 4; rt++) {
            if (rt < nv) {
              const int lr = (rt0 + rt) * 8 + g;  // local row in panel
#pragma unroll
              for (int ct = 0; ct < 4; ct++) {
                double2 v2 = make_double2(acc[rt][ct][0], acc[rt][ct][1]);
                *reinterpret_cast<double2 *>(pan + mtile(lr, ct * 8 + 2 * q) + g * 4 + 2 * (q & 1)) = v2;
                if (c0 + lr == Cp) {
#pragma unroll
                  for (int i = 0; i < 2; i++) {
                    const int col = c0 + ct * 8 + 2 * q + i;
                    if (col >= mt && col < N) quad_acc = fma(acc[rt][ct][i], acc[rt][ct][i], quad_acc);
                  }
                }
              }
            }
          }
        }
      }
      __syncthreads();  // panel j complete and visible before panel j+1 reads it
      if (s_fail) break;
    }

    // ---- block reduction of quad / logdet (fixed order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      quad_acc += __shfl_xor_sync(0xffffffffu, quad_acc, o);
      logdet_acc += __shfl_xor_sync(0xffffffffu, logdet_acc, o);
    }
    if (lane == 0) {
      s_red[warp] = quad_acc;
      s_red[kH8Warps + warp] = logdet_acc;
    }
    __syncthreads();
    if (tid == 0) {
      double qs = 0.0, ls = 0.0;
      for (int w = 0; w < kH8Warps; w++) {
        qs += s_red[w];
        ls += s_red[kH8Warps + w];
      }
      ls *= 2.0;
      const double term = -0.5 * (qs + ls) - 0.5 * (double)bst * 1.8378770664093454836;  // log 2pi
      a.terms[li] = s_fail ? NAN : term;
      a.quads[li] = qs;
      a.logdets[li] = ls;
      a.status[li] = s_fail ? s_fail_stage : 0;
    }
    __syncthreads();
  }
}

size_t h8_smem_bytes(int max_N, int d) {
  int Cp = (max_N + kPanel - 1) / kPanel * kPanel;
  return sizeof(double) * ((size_t)kPanel * kDld + kPanel + SBV_MAX_D + (Cp + 8) + (size_t)max_N * d);
}

size_t h8_ws_doubles(int max_N) {
  size_t Cp = (max_N + kPanel - 1) / kPanel * kPanel, R = Cp + 8, NP = Cp / kPanel;
  size_t tot = 0;
  for (size_t p = 0; p < NP; p++) tot += kPanel * (R - kPanel * p);
  return (tot + 63) / 64 * 64;
}

template <int NU2>
static cudaError_t set_attr(size_t smem) {
  return cudaFuncSetAttribute(k_h8<NU2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

int h8_max_ctas_per_sm(size_t smem) {
  set_attr<5>(smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_h8<5>, kH8Threads, smem);
  return nb;
}

cudaError_t launch_h8(const Ctx &c, const double *theta, cudaStream_t st) {
  H8Args a;
  a.Xp = c.Xperm;
  a.yperm = c.yperm;
  a.off = c.off;
  a.nbr = c.nbr;
  a.cnt = c.cnt;
  a.local_blocks = c.local_blocks;
  a.work_order = c.work_order;
  a.k_local = c.k_local;
  a.m = c.m > 0 ? c.m : 1;
  a.d = c.d;
  a.sigma2 = theta[0];
  a.tau2 = theta[c.d + 2];
  for (int j = 0; j < SBV_MAX_D; j++) a.inv_beta[j] = j < c.d ? 1.0 / theta[1 + j] : 0.0;
  a.ws = c.ws;
  a.ws_per_cta = c.ws_per_cta;
  a.queue = c.queue;
  a.terms = c.terms;
  a.quads = c.quads;
  a.logdets = c.logdets;
  a.status = c.status;
  const double nu = theta[c.d + 1];
  cudaError_t e = cudaMemsetAsync(c.queue, 0, sizeof(unsigned int), st);
  if (e) return e;
  if (c.k_local == 0) return cudaSuccess;
  const int grid = c.h8_grid;
  const size_t smem = c.h8_smem;
  if (nu == 0.5) {
    set_attr<1>(smem);
    k_h8<1><<<grid, kH8Threads, smem, st>>>(a);
  } else if (nu == 1.5) {
    set_attr<3>(smem);
    k_h8<3><<<grid, kH8Threads, smem, st>>>(a);
  } else if (nu == 2.5) {
    set_attr<5>(smem);
    k_h8<5><<<grid, kH8Threads, smem, st>>>(a);
  } else {
    set_attr<7>(smem);
    k_h8<7><<<grid, kH8Threads, smem, st>>>(a);
  }
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
