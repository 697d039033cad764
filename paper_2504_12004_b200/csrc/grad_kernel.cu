// grad_kernel.cu — SURVEY 8(f) N3: the gradient of the block-Vecchia
// log-likelihood with respect to theta = (sigma2, beta_1..beta_d, tau2), nu
// fixed (the "gradient quantities" of P:453; Q28).
//
// Per block t (Alg.5's term = joint density of [y_J; y_B] minus the marginal
// of y_J; Eq.1 P:156-158 differentiated):
//   d ell_t / d theta_k = 1/2 sum_ij G_ij (dK_k)_ij,
//   G = at dl^T + dl at^T + dl dl^T - Z Z^T,
// with the joint factor L = chol(K([J; B])) from H8 (k_h8 MODE 2 copies it
// row-major, with the border row y' = L^-1 [y_J; y_B] as row N):
//   Z  = L^-T E_B            (N x b: the B columns of L^-T; Z Z^T = K^-1 - blkdiag(K_JJ^-1, 0)),
//   v  = y'_B,  dl = Z v     (= K^-1 y - [K_JJ^-1 y_J; 0]),
//   at = [L11^-T y'_J; 0]    (= [K_JJ^-1 y_J; 0]).
// (Derivation in DESIGN.md §6.)
//
// One CTA (8 warps) per block, persistent over the batch:
//   1. coordinates staged (centred, 1/beta scaled, as in H8), y', 1/L_ii;
//   2. Z and at together by ONE blocked backward TRSM, L^-T [E_B | 0 | y'_J; 0]
//      (at = L^-T [y'_J; 0] is the extra right-hand side in column cz4 =
//      round4(b), outside the W contraction), 32-row panels from the bottom,
//      each warp owning kGSW-column slices: DMMA GEMM of the panel's rows
//      against the rows below (kGPF-deep register prefetch of the L2
//      operands), then a 32x32 back substitution (lane = column) against L_pp
//      staged in shared memory;
//   3. dl = Z v;
//   4. every 32x32 lower tile (I >= J) of the N x N index space: W = Z_I Z_J^T
//      on DMMA, then per entry G_ij and the covariance derivatives generated
//      on the fly (Eq.5-6 differentiated; e^{-r} by the 256-entry table of
//      H8, f'(r)/r in closed form), accumulated per parameter;
//   5. fixed-order reductions: lanes -> warps -> the block's gradient.
#include <math.h>

#include "h8_kernel.cuh"

namespace sbv {

// Warps per CTA, a template parameter: 4 (two CTAs per SM at <= 255 registers,
// every warp owns a Z slice for b <= 128) for many blocks per CTA, 8 (one CTA
// per SM) when the launch has few blocks per CTA and the 4-warp CTAs' long
// blocks (b > 128: several slices per warp) set the tail (grad_shape, measured:
// cfg2 n = 1M 27.8 vs 34.4 ms, n = 200k 8.5 vs 6.9 ms).

struct GradArgs {
  const double *Lg;          // per-block (N+1) x N row-major factor copies
  const int64_t *lg_off;     // [k_local]
  const double *Xp;          // n x d block-major ORIGINAL inputs
  const int64_t *off;        // bc + 1
  const int32_t *nbr;        // k_local x m (block-major positions)
  const int32_t *cnt;        // k_local
  const int32_t *local_blocks;
  const int32_t *items;      // local block indices of this batch
  int64_t n_items;
  int m, d, P;               // P = d + 2 parameters
  int max_N, bpad_max;
  double sigma2, inv_beta[SBV_MAX_D];
  double *zws;               // per-CTA Z scratch: max_N x bpad_max
  unsigned int *queue;
  double *grads;             // [k_local][P]
};

#ifndef SBV_GRAD_SW
#define SBV_GRAD_SW 32  // Z columns per TRSM slice (one warp each)
#endif
#ifndef SBV_GRAD_PF
#define SBV_GRAD_PF 2  // k-steps of register prefetch in the DMMA loops
#endif
constexpr int kGSW = SBV_GRAD_SW, kGPF = SBV_GRAD_PF;

// f(r) and h(r) = f'(r)/r of the half-integer closed forms (sigma2 = 1),
// NU2 = 2 nu, e = e^{-r}, ri = 1/r (used by nu = 1/2 only)
template <int NU2>
__device__ __forceinline__ double matern_f_h(double r, double e, double ri, double &h) {
  if (NU2 == 1) {
    h = -e * ri;
    return e;
  }
  if (NU2 == 3) {
    h = -e;
    return (1.0 + r) * e;
  }
  if (NU2 == 5) {
    h = -(1.0 / 3.0) * (1.0 + r) * e;
    return fma(r, fma(r, 1.0 / 3.0, 1.0), 1.0) * e;
  }
  h = -(1.0 / 15.0) * fma(r, r + 3.0, 3.0) * e;
  return fma(r, fma(r, fma(r, 1.0 / 15.0, 2.0 / 5.0), 1.0), 1.0) * e;
}

// acc[4][NCT] (+)= A B^T over k in [kb, ke) in steps of 4: la(k, A[4]) and
// lb(k, B[NCT]) load the m8n8k4 fragments of one k-step (zero beyond the
// matrix); kGPF k-steps of loads in flight
template <int NCT, class LA, class LB>
__device__ __forceinline__ void gemm_pf(double (&acc)[4][NCT][2], int kb, int ke, LA la, LB lb) {
  double af[kGPF][4], bf[kGPF][NCT];
#pragma unroll
  for (int s = 0; s < kGPF; s++)
    if (kb + 4 * s < ke) {
      la(kb + 4 * s, af[s]);
      lb(kb + 4 * s, bf[s]);
    }
  for (int k0 = kb; k0 < ke; k0 += 4 * kGPF) {
#pragma unroll
    for (int s = 0; s < kGPF; s++) {
      const int k = k0 + 4 * s;
      if (k < ke) {
#pragma unroll
        for (int rt = 0; rt < 4; rt++)
#pragma unroll
          for (int ct = 0; ct < NCT; ct++) dmma(acc[rt][ct][0], acc[rt][ct][1], af[s][rt], bf[s][ct]);
        if (k + 4 * kGPF < ke) {
          la(k + 4 * kGPF, af[s]);
          lb(k + 4 * kGPF, bf[s]);
        }
      }
    }
  }
}

// DM > 0: coordinates staged with the padded row stride DM (d <= DM, zero
// padded; the padded dimensions contribute 0 to every distance and gradient)
template <int NU2, int DM, int NWG>
__global__ void __launch_bounds__(32 * NWG, 8 / NWG) k_grad(GradArgs a) {
  constexpr int kGThreads = 32 * NWG, kGW = NWG;
  extern __shared__ double gsm[];
  __shared__ int s_item;
  __shared__ double s_etab[256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int d = a.d, P = a.P;
  const int DS = DM > 0 ? DM : d;         // staged row stride
  const int Nmax = a.max_N;
  double *vs = gsm;                       // Nmax x DS coordinates
  double *yp = vs + (size_t)Nmax * DS;    // y' (N)
  double *at = yp + Nmax;                 // at (N; zero on B)
  double *dl = at + Nmax;                 // dl (N)
  double *rinv = dl + Nmax;               // 1 / L_ii (N)
  double *red = rinv + Nmax;              // 8 warps x P partial gradients
  double *xref = red + kGW * P;           // d
  double *Wt = xref + SBV_MAX_D + warp * 32 * 33;  // this warp's 32 x 32 tile (row-major, ld 33)
  double *Z = a.zws + (size_t)blockIdx.x * Nmax * a.bpad_max;
  for (int j = tid; j < 256; j += kGThreads) s_etab[j] = exp2(j / 256.0);

  for (;;) {
    if (tid == 0) s_item = (int)atomicAdd(a.queue, 1u);
    __syncthreads();
    const int it = s_item;
    if (it >= a.n_items) break;
    const int li = a.items[it];
    const int64_t t = a.local_blocks[li];
    const int mt = a.cnt[li];
    const int64_t b0 = a.off[t];
    const int bb = (int)(a.off[t + 1] - b0);
    const int N = mt + bb;
    const int cz4 = (bb + 3) & ~3;                 // W contraction columns (zero beyond bb)
    const int nsl = (cz4 + 1 + kGSW - 1) / kGSW;   // slices incl. the at column cz4
    const int bpad = nsl * kGSW;                   // Z row stride
    const double *L = a.Lg + a.lg_off[li];  // (N+1) x N, row i at L + i N
    // ---- 1. coordinates (centred on the block's first member, 1/beta), y', 1/L_ii
    for (int j = tid; j < d; j += kGThreads) xref[j] = a.Xp[b0 * d + j];
    __syncthreads();
    for (int e = tid; e < N * DS; e += kGThreads) {
      const int i = e / DS, j = e - i * DS;
      const int64_t pos = i < mt ? (int64_t)a.nbr[(int64_t)li * a.m + i] : b0 + (i - mt);
      vs[e] = j < d ? (a.Xp[pos * d + j] - xref[j]) * a.inv_beta[j] : 0.0;
    }
    for (int i = tid; i < N; i += kGThreads) {
      yp[i] = L[(size_t)N * N + i];
      rinv[i] = 1.0 / L[(size_t)i * N + i];
    }
    __syncthreads();
    // ---- 2. [Z | at] = L^-T [E_B | y'_J; 0], slices of kGSW columns, one warp
    // each, bottom-up over 32-row panels
    constexpr int NCT = kGSW / 8;
    const int NPn = (N + 31) >> 5;
    for (int sl = warp; sl < nsl; sl += kGW) {
      const int cb = sl * kGSW;
      for (int p = NPn - 1; p >= 0; p--) {
        const int r0 = p * 32;
        double acc[4][NCT][2];
        // acc holds the NEGATED partial solution (no operand negation in the
        // k-loop): -(right-hand sides) at the panel rows, i.e. -1 at
        // (mt + c, c) for c < bb and -y'_J in column cz4
#pragma unroll
        for (int rt = 0; rt < 4; rt++)
#pragma unroll
          for (int ct = 0; ct < NCT; ct++)
#pragma unroll
            for (int i = 0; i < 2; i++) {
              const int row = r0 + rt * 8 + g, col = cb + ct * 8 + 2 * q + i;
              acc[rt][ct][i] = col < bb ? (row == mt + col ? -1.0 : 0.0) : (col == cz4 && row < mt ? -yp[row] : 0.0);
            }
        // acc += L[k, panel cols]^T Z[k, slice cols] over rows k >= r0 + 32
        gemm_pf<NCT>(
            acc, r0 + 32, N,
            [&](int k0, double (&A)[4]) {
              const int kr = k0 + q;
#pragma unroll
              for (int rt = 0; rt < 4; rt++) A[rt] = (kr < N) ? L[(size_t)kr * N + r0 + rt * 8 + g] : 0.0;
            },
            [&](int k0, double (&B)[NCT]) {
              const int kr = k0 + q;
#pragma unroll
              for (int ct = 0; ct < NCT; ct++) B[ct] = (kr < N) ? Z[(size_t)kr * bpad + cb + ct * 8 + g] : 0.0;
            });
        // park acc in this panel's rows of the slice; stage L_pp (lower) in Wt
#pragma unroll
        for (int rt = 0; rt < 4; rt++)
#pragma unroll
          for (int ct = 0; ct < NCT; ct++)
#pragma unroll
            for (int i = 0; i < 2; i++) {
              const int row = r0 + rt * 8 + g, col = cb + ct * 8 + 2 * q + i;
              if (row < N) Z[(size_t)row * bpad + col] = -acc[rt][ct][i];
            }
        const int nr = min(32, N - r0);
#pragma unroll 8
        for (int i = 0; i < 32; i++)
          Wt[i * 33 + lane] = (i < nr && lane <= i) ? L[(size_t)(r0 + i) * N + r0 + lane] : 0.0;
        __syncwarp();
        // 32 x 32 back substitution with L_pp^T, lane = column
        if (lane < kGSW) {
          double z[32];
#pragma unroll
          for (int i = 0; i < 32; i++) z[i] = i < nr ? Z[(size_t)(r0 + i) * bpad + cb + lane] : 0.0;
#pragma unroll
          for (int i = 31; i >= 0; i--) {
            if (i < nr) {
              z[i] *= rinv[r0 + i];
#pragma unroll
              for (int k = 0; k < i; k++) z[k] = fma(-Wt[i * 33 + k], z[i], z[k]);
            }
          }
#pragma unroll
          for (int i = 0; i < 32; i++)
            if (i < nr) Z[(size_t)(r0 + i) * bpad + cb + lane] = z[i];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- 3. dl = Z v (v = y'_B); at = column cz4
    for (int i = tid; i < N; i += kGThreads) {
      const double *zr = Z + (size_t)i * bpad;
      double s = 0.0;
      for (int c = 0; c < bb; c++) s = fma(zr[c], yp[mt + c], s);
      dl[i] = s;
      at[i] = zr[cz4];
    }
    __syncthreads();
    // ---- 4. lower tiles of G = at dl^T + dl at^T + dl dl^T - Z Z^T against dK:
    // W tile on DMMA -> this warp's shared tile -> lane = column j, loop over
    // the tile's rows i (the column's coordinates stay in registers)
    constexpr int GK = DM > 0 ? DM + 2 : 2 + SBV_MAX_D;
    double gk[GK];
#pragma unroll
    for (int k = 0; k < GK; k++) gk[k] = 0.0;
    const int ntile = NPn * (NPn + 1) / 2;
    for (int tI = warp; tI < ntile; tI += kGW) {
      int I = 0;
      while ((I + 1) * (I + 2) / 2 <= tI) I++;
      const int J = tI - I * (I + 1) / 2;
      double acc[4][4][2];
#pragma unroll
      for (int rt = 0; rt < 4; rt++)
#pragma unroll
        for (int ct = 0; ct < 4; ct++) acc[rt][ct][0] = acc[rt][ct][1] = 0.0;
      gemm_pf<4>(
          acc, 0, cz4,
          [&](int c0, double (&A)[4]) {
#pragma unroll
            for (int rt = 0; rt < 4; rt++) {
              const int row = I * 32 + rt * 8 + g;
              A[rt] = row < N ? Z[(size_t)row * bpad + c0 + q] : 0.0;
            }
          },
          [&](int c0, double (&B)[4]) {
#pragma unroll
            for (int ct = 0; ct < 4; ct++) {
              const int row = J * 32 + ct * 8 + g;
              B[ct] = row < N ? Z[(size_t)row * bpad + c0 + q] : 0.0;
            }
          });
#pragma unroll
      for (int rt = 0; rt < 4; rt++)
#pragma unroll
        for (int ct = 0; ct < 4; ct++) {
          Wt[(rt * 8 + g) * 33 + ct * 8 + 2 * q] = acc[rt][ct][0];
          Wt[(rt * 8 + g) * 33 + ct * 8 + 2 * q + 1] = acc[rt][ct][1];
        }
      __syncwarp();
      const int j = J * 32 + lane;
      if (j < N) {
        const double atj = at[j], dlj = dl[j];
        const int i0 = I * 32, i1 = min(N, I * 32 + 32);
        if constexpr (DM > 0) {
          double xc[DM];
#pragma unroll
          for (int jj = 0; jj < DM; jj++) xc[jj] = vs[(size_t)j * DM + jj];
          // rows in pairs (two independent dependency chains); rows above the
          // diagonal (i < j) and past the block get weight 0
#pragma unroll 1
          for (int ib = i0; ib < i1; ib += 2) {
#pragma unroll
            for (int h2 = 0; h2 < 2; h2++) {
              const int i = min(ib + h2, i1 - 1);
              const double G = fma(at[i], dlj, fma(dl[i], atj, fma(dl[i], dlj, -Wt[(i - i0) * 33 + lane])));
              const double wg = (ib + h2 >= i1 || i < j) ? 0.0 : (i == j ? 0.5 * G : G);  // 1/2 sum over the symmetric matrix
              double u2[DM];
              double s2 = 0.0;
#pragma unroll
              for (int jj = 0; jj < DM; jj++) {
                const double u = vs[(size_t)i * DM + jj] - xc[jj];
                u2[jj] = u * u;
                s2 += u2[jj];
              }
              const double ri = rsqrt_pos(fmax(s2, 1e-300));
              const double r = s2 * ri;
              const double e = neg_sigma2_exp_neg(r, s_etab);  // table holds 2^{j/256}: e = e^{-r}
              double hr;
              const double f = matern_f_h<NU2>(r, e, ri, hr);
              gk[0] = fma(wg, f, gk[0]);
              const double coef = s2 > 0.0 ? -a.sigma2 * hr * wg : 0.0;  // dK/dbeta_j = coef u_j^2 / beta_j
#pragma unroll
              for (int jj = 0; jj < DM; jj++) gk[1 + jj] = fma(coef, u2[jj], gk[1 + jj]);
              if (i == j && ib + h2 < i1) gk[DM + 1] += wg;
            }
          }
        } else {
#pragma unroll 1
          for (int i = max(i0, j); i < i1; i++) {
            const double G = fma(at[i], dlj, fma(dl[i], atj, fma(dl[i], dlj, -Wt[(i - i0) * 33 + lane])));
            const double wg = (i == j) ? 0.5 * G : G;
            const double *xi = vs + (size_t)i * d, *xj = vs + (size_t)j * d;
            double s2 = 0.0;
            for (int jj = 0; jj < d; jj++) {
              const double u = xi[jj] - xj[jj];
              s2 = fma(u, u, s2);
            }
            const double ri = rsqrt_pos(fmax(s2, 1e-300));
            const double r = s2 * ri;
            const double e = neg_sigma2_exp_neg(r, s_etab);
            double hr;
            const double f = matern_f_h<NU2>(r, e, ri, hr);
            gk[0] = fma(wg, f, gk[0]);
            const double coef = s2 > 0.0 ? -a.sigma2 * hr * wg : 0.0;
            for (int jj = 0; jj < d; jj++) {
              const double u = xi[jj] - xj[jj];
              gk[1 + jj] = fma(coef, u * u, gk[1 + jj]);
            }
            if (i == j) gk[d + 1] += wg;
          }
        }
      }
      __syncwarp();
    }
    // gradient slots: sigma2 | beta_1..beta_d (times 1/beta_j here) | tau2
    // (DM > 0: tau2 is slot DM + 1, slots d+1..DM belong to zero-padded dimensions)
    // ---- 5. fixed-order reductions: lanes (xor tree), warps (in order)
#pragma unroll
    for (int kk = 0; kk < GK; kk++) {
      const int dst = (DM > 0 && kk == DM + 1) ? P - 1 : kk;
      if ((DM > 0 && kk > d && kk <= DM) || (DM == 0 && kk >= P)) continue;
      double v = gk[kk];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (kk >= 1 && kk <= d) v *= a.inv_beta[kk - 1];
      if (lane == 0) red[warp * P + dst] = v;
    }
    __syncthreads();
    for (int k = tid; k < P; k += kGThreads) {
      double v = 0.0;
      for (int w = 0; w < kGW; w++) v += red[w * P + k];
      a.grads[(size_t)li * P + k] = v;
    }
    __syncthreads();
  }
}

// sum of the per-block gradients over this rank's blocks: one warp per
// parameter, lane l sums blocks l, l+32, ... in order, then a fixed xor tree
// (deterministic)
__global__ void k_grad_sum(const double *grads, int64_t k_local, int P, double *out) {
  const int k = blockIdx.x, lane = threadIdx.x;
  double s = 0.0;
  for (int64_t li = lane; li < k_local; li += 32) s += grads[li * P + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[k] = s;
}

size_t grad_smem_bytes(int max_N, int d, int nw) {
  const int ds = d <= 16 ? (d <= 4 ? 4 : d <= 8 ? 8 : d <= 10 ? 10 : d <= 12 ? 12 : 16) : d;
  return sizeof(double) * ((size_t)max_N * ds + 4 * (size_t)max_N + nw * (size_t)(d + 2) + SBV_MAX_D +
                           (size_t)nw * 32 * 33);
}

// 4 or 8 warps per CTA for a launch of k blocks on `sms` SMs (see k_grad)
// (SBV_GRAD_NW = 4 or 8 forces one: tests cover both instantiations)
int grad_shape(int64_t k, int sms) {
  if (const char *e = getenv("SBV_GRAD_NW")) {
    const int v = atoi(e);
    if (v == 4 || v == 8) return v;
  }
  return k < (int64_t)16 * 2 * sms ? 8 : 4;
}

static int grad_dm(int d) {
  if (d <= 4) return 4;
  if (d <= 8) return 8;
  if (d <= 10) return 10;
  if (d <= 12) return 12;
  if (d <= 16) return 16;
  return 0;
}

template <int NU2, int NWG>
static void (*pick_grad(int dm))(GradArgs) {
  switch (dm) {
    case 4: return k_grad<NU2, 4, NWG>;
    case 8: return k_grad<NU2, 8, NWG>;
    case 10: return k_grad<NU2, 10, NWG>;
    case 12: return k_grad<NU2, 12, NWG>;
    case 16: return k_grad<NU2, 16, NWG>;
    default: return k_grad<NU2, 0, NWG>;
  }
}

template <int NWG>
static void (*pick_grad_nw(double nu, int dm))(GradArgs) {
  return nu == 0.5 ? pick_grad<1, NWG>(dm) : nu == 1.5 ? pick_grad<3, NWG>(dm)
                   : nu == 2.5 ? pick_grad<5, NWG>(dm) : pick_grad<7, NWG>(dm);
}

static void (*pick_grad_fn(double nu, int d, int nw))(GradArgs) {
  const int dm = grad_dm(d);
  return nw == 8 ? pick_grad_nw<8>(nu, dm) : pick_grad_nw<4>(nu, dm);
}

// persistent grid: resident CTAs per SM (shared memory / registers) x SMs
int grad_grid(double nu, int d, int max_N, int sms, int nw) {
  void (*f)(GradArgs) = pick_grad_fn(nu, d, nw);
  const size_t sm = grad_smem_bytes(max_N, d, nw);
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, 32 * nw, sm) != cudaSuccess || nb < 1) {
    cudaGetLastError();
    nb = 1;
  }
  return sms * nb;
}

cudaError_t launch_grad(const GradLaunch &gl, cudaStream_t st) {
  GradArgs a;
  a.Lg = gl.Lg;
  a.lg_off = gl.lg_off;
  a.Xp = gl.Xp;
  a.off = gl.off;
  a.nbr = gl.nbr;
  a.cnt = gl.cnt;
  a.local_blocks = gl.local_blocks;
  a.items = gl.items;
  a.n_items = gl.n_items;
  a.m = gl.m > 0 ? gl.m : 1;
  a.d = gl.d;
  a.P = gl.d + 2;
  a.max_N = gl.max_N;
  a.bpad_max = gl.bpad_max;
  a.sigma2 = gl.theta[0];
  for (int j = 0; j < SBV_MAX_D; j++) a.inv_beta[j] = j < gl.d ? 1.0 / gl.theta[1 + j] : 0.0;
  a.zws = gl.zws;
  a.queue = gl.queue;
  a.grads = gl.grads;
  cudaError_t e = cudaMemsetAsync(gl.queue, 0, sizeof(unsigned int), st);
  if (e) return e;
  if (gl.n_items == 0) return cudaSuccess;
  const double nu = gl.theta[gl.d + 1];
  void (*f)(GradArgs) = pick_grad_fn(nu, gl.d, gl.nw);
  const size_t sm = grad_smem_bytes(gl.max_N, gl.d, gl.nw);
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  f<<<gl.grid, 32 * gl.nw, sm, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_grad_sum(const double *grads, int64_t k_local, int P, double *out, cudaStream_t st) {
  k_grad_sum<<<P, 32, 0, st>>>(grads, k_local, P, out);
  return cudaGetLastError();
}

}  // namespace sbv
