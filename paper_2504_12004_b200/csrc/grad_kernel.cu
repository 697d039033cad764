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
//   1. coordinates staged (centred, 1/beta scaled, as in H8) + y';
//   2. at by an axpy back substitution with L11 rows (one warp);
//   3. Z by a blocked backward TRSM, 32-row panels from the bottom, each warp
//      owning 32-column slices of Z: DMMA GEMM of the panel's rows against
//      the rows below, then a 32x32 back substitution (lane = column);
//   4. dl = Z v;
//   5. every 32x32 lower tile (I >= J) of the N x N index space: W = Z_I Z_J^T
//      on DMMA, then per entry G_ij and the covariance derivatives generated
//      on the fly (Eq.5-6 differentiated), accumulated per parameter;
//   6. fixed-order reductions: lanes -> warps -> the block's gradient.
#include <math.h>

#include "h8_kernel.cuh"

namespace sbv {

constexpr int kGThreads = 256;

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

// f(r) and f'(r) of the half-integer closed forms (sigma2 = 1), NU2 = 2 nu
template <int NU2>
__device__ __forceinline__ double matern_f_df(double r, double &df) {
  const double e = exp(-r);
  if (NU2 == 1) {
    df = -e;
    return e;
  }
  if (NU2 == 3) {
    df = -r * e;
    return (1.0 + r) * e;
  }
  if (NU2 == 5) {
    df = -(r * (1.0 / 3.0)) * (1.0 + r) * e;
    return fma(r, fma(r, 1.0 / 3.0, 1.0), 1.0) * e;
  }
  df = -(r * (1.0 / 15.0)) * fma(r, r + 3.0, 3.0) * e;
  return fma(r, fma(r, fma(r, 1.0 / 15.0, 2.0 / 5.0), 1.0), 1.0) * e;
}

// DM > 0: coordinates staged with the padded row stride DM (d <= DM, zero
// padded; the padded dimensions contribute 0 to every distance and gradient)
template <int NU2, int DM>
__global__ void __launch_bounds__(kGThreads, 1) k_grad(GradArgs a) {
  extern __shared__ double gsm[];
  __shared__ int s_item;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int d = a.d, P = a.P;
  const int DS = DM > 0 ? DM : d;         // staged row stride
  const int Nmax = a.max_N;
  double *vs = gsm;                       // Nmax x DS coordinates
  double *yp = vs + (size_t)Nmax * DS;    // y' (N)
  double *at = yp + Nmax;                 // at (N; zero on B)
  double *dl = at + Nmax;                 // dl (N)
  double *red = dl + Nmax;                // 8 warps x P partial gradients
  double *xref = red + 8 * P;             // d
  double *Wt = xref + SBV_MAX_D + warp * 32 * 33;  // this warp's 32 x 32 W tile (row-major, ld 33)
  double *Z = a.zws + (size_t)blockIdx.x * Nmax * a.bpad_max;

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
    const int bpad = (bb + 31) & ~31;
    const double *L = a.Lg + a.lg_off[li];  // (N+1) x N, row i at L + i N
    // ---- 1. coordinates (centred on the block's first member, 1/beta) and y'
    for (int j = tid; j < d; j += kGThreads) xref[j] = a.Xp[b0 * d + j];
    __syncthreads();
    for (int e = tid; e < N * DS; e += kGThreads) {
      const int i = e / DS, j = e - i * DS;
      const int64_t pos = i < mt ? (int64_t)a.nbr[(int64_t)li * a.m + i] : b0 + (i - mt);
      vs[e] = j < d ? (a.Xp[pos * d + j] - xref[j]) * a.inv_beta[j] : 0.0;
    }
    for (int i = tid; i < N; i += kGThreads) {
      yp[i] = L[(size_t)N * N + i];
      at[i] = i < mt ? yp[i] : 0.0;
    }
    __syncthreads();
    // ---- 2 + 3. Z = L^-T E_B in slices of 32 columns of B (one warp per slice,
    // bottom-up over 32-row panels); at_J = L11^-T y'_J by the first warp
    // that has one slice fewer than the others (axpy form over the rows of L11).
    // (8-column slices keep more warps busy but re-read L per slice: measured
    // slower, 91 vs 65 ms at cfg2.)
    constexpr int kSW = 32;
    const int NPn = (N + 31) >> 5;
    const int nsl = (bb + kSW - 1) / kSW;
    const int w2 = nsl % (kGThreads / 32);
    for (int task = warp; task < nsl + (kGThreads / 32); task += kGThreads / 32) {
      if (task >= nsl) {
        if (warp != w2) continue;
        for (int i = mt - 1; i >= 0; i--) {
          const double ai = at[i] / L[(size_t)i * N + i];
          __syncwarp();
          if (lane == 0) at[i] = ai;
          for (int k = lane; k < i; k += 32) at[k] = fma(-L[(size_t)i * N + k], ai, at[k]);
          __syncwarp();
        }
        continue;
      }
      const int sl = task;
      for (int p = NPn - 1; p >= 0; p--) {
        const int r0 = p * 32;
        double acc[4][4][2];
        // E_B[panel rows, slice columns]: 1 at (m + c, c)
#pragma unroll
        for (int rt = 0; rt < 4; rt++)
#pragma unroll
          for (int ct = 0; ct < 4; ct++)
#pragma unroll
            for (int i = 0; i < 2; i++) {
              const int row = r0 + rt * 8 + g, col = sl * kSW + ct * 8 + 2 * q + i;
              acc[rt][ct][i] = (col < bb && row == mt + col) ? 1.0 : 0.0;
            }
        // acc -= L[k, panel cols]^T Z[k, slice cols] over rows k >= r0 + 32
        // (operands of the next k-step loaded one step ahead)
        {
          double af[4], bf[4], an[4], bn[4];
          auto ldz = [&](int k0, double (&A)[4], double (&B)[4]) {
            const int kr = k0 + q;
#pragma unroll
            for (int rt = 0; rt < 4; rt++) A[rt] = (kr < N) ? -L[(size_t)kr * N + r0 + rt * 8 + g] : 0.0;
#pragma unroll
            for (int ct = 0; ct < 4; ct++) B[ct] = (kr < N) ? Z[(size_t)kr * bpad + sl * kSW + ct * 8 + g] : 0.0;
          };
          if (r0 + 32 < N) ldz(r0 + 32, af, bf);
          for (int k0 = r0 + 32; k0 < N; k0 += 4) {
            if (k0 + 4 < N) ldz(k0 + 4, an, bn);
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
        // 32x32 back substitution with L_pp^T; lane = column: park acc in
        // this panel's rows of the slice, then solve in registers
#pragma unroll
        for (int rt = 0; rt < 4; rt++)
#pragma unroll
          for (int ct = 0; ct < 4; ct++)
#pragma unroll
            for (int i = 0; i < 2; i++) {
              const int row = r0 + rt * 8 + g, col = sl * kSW + ct * 8 + 2 * q + i;
              if (row < N) Z[(size_t)row * bpad + col] = acc[rt][ct][i];
            }
        __syncwarp();
        const int nr = min(32, N - r0);
        double z[32];
#pragma unroll
        for (int i = 0; i < 32; i++) z[i] = i < nr ? Z[(size_t)(r0 + i) * bpad + sl * kSW + lane] : 0.0;
#pragma unroll
        for (int i = 31; i >= 0; i--) {
          if (i < nr) {
            const double *Lr = L + (size_t)(r0 + i) * N + r0;
            z[i] = z[i] / Lr[i];
#pragma unroll
            for (int k = 0; k < i; k++) z[k] = fma(-Lr[k], z[i], z[k]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 32; i++)
          if (i < nr) Z[(size_t)(r0 + i) * bpad + sl * kSW + lane] = z[i];
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- 4. dl = Z v, v = y'_B
    for (int i = tid; i < N; i += kGThreads) {
      double s = 0.0;
      for (int c = 0; c < bb; c++) s = fma(Z[(size_t)i * bpad + c], yp[mt + c], s);
      dl[i] = s;
    }
    __syncthreads();
    // ---- 5. lower tiles of G = at dl^T + dl at^T + dl dl^T - Z Z^T against dK:
    // W tile on DMMA -> this warp's shared tile -> lane = column j, loop over
    // the tile's rows i (the column's coordinates stay in registers)
    constexpr int GK = DM > 0 ? DM + 2 : 2 + SBV_MAX_D;
    double gk[GK];
#pragma unroll
    for (int k = 0; k < GK; k++) gk[k] = 0.0;
    const int ntile = NPn * (NPn + 1) / 2;
    for (int tI = warp; tI < ntile; tI += kGThreads / 32) {
      int I = 0;
      while ((I + 1) * (I + 2) / 2 <= tI) I++;
      const int J = tI - I * (I + 1) / 2;
      double acc[4][4][2];
#pragma unroll
      for (int rt = 0; rt < 4; rt++)
#pragma unroll
        for (int ct = 0; ct < 4; ct++) acc[rt][ct][0] = acc[rt][ct][1] = 0.0;
      double af[4], bf[4], an[4], bn[4];
      auto ldw = [&](int c0, double (&A)[4], double (&B)[4]) {
#pragma unroll
        for (int rt = 0; rt < 4; rt++) {
          const int row = I * 32 + rt * 8 + g;
          A[rt] = row < N ? Z[(size_t)row * bpad + c0 + q] : 0.0;
        }
#pragma unroll
        for (int ct = 0; ct < 4; ct++) {
          const int row = J * 32 + ct * 8 + g;
          B[ct] = row < N ? Z[(size_t)row * bpad + c0 + q] : 0.0;
        }
      };
      const int cz = nsl * kSW;  // Z columns written by step 3 (zero beyond bb)
      ldw(0, af, bf);
      for (int c0 = 0; c0 < cz; c0 += 4) {
        if (c0 + 4 < cz) ldw(c0 + 4, an, bn);
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
        double xc[DM > 0 ? DM : 1];
        if constexpr (DM > 0) {
#pragma unroll
          for (int jj = 0; jj < DM; jj++) xc[jj] = vs[(size_t)j * DM + jj];
        }
        const double atj = at[j], dlj = dl[j];
        const int i1 = min(N, I * 32 + 32);
#pragma unroll 1
        for (int i = max(I * 32, j); i < i1; i++) {
          const double G = fma(at[i], dlj, fma(dl[i], atj, fma(dl[i], dlj, -Wt[(i - I * 32) * 33 + lane])));
          const double wg = (i == j) ? 0.5 * G : G;  // 1/2 sum over the full symmetric matrix
          if constexpr (DM > 0) {
            double u2[DM];
            double s2 = 0.0;
#pragma unroll
            for (int jj = 0; jj < DM; jj++) {
              const double u = vs[(size_t)i * DM + jj] - xc[jj];
              u2[jj] = u * u;
              s2 += u2[jj];
            }
            const double r = sqrt(s2);
            double df;
            const double f = matern_f_df<NU2>(r, df);
            gk[0] = fma(wg, f, gk[0]);
            const double coef = r > 0.0 ? -a.sigma2 * df / r * wg : 0.0;  // dK/dbeta_j = coef u_j^2 / beta_j
#pragma unroll
            for (int jj = 0; jj < DM; jj++) gk[1 + jj] = fma(coef * a.inv_beta[jj], u2[jj], gk[1 + jj]);
            if (i == j) gk[DM + 1] += wg;
          } else {
            const double *xi = vs + (size_t)i * d, *xj = vs + (size_t)j * d;
            double s2 = 0.0;
            for (int jj = 0; jj < d; jj++) {
              const double u = xi[jj] - xj[jj];
              s2 = fma(u, u, s2);
            }
            const double r = sqrt(s2);
            double df;
            const double f = matern_f_df<NU2>(r, df);
            gk[0] = fma(wg, f, gk[0]);
            const double coef = r > 0.0 ? -a.sigma2 * df / r * wg : 0.0;
            for (int jj = 0; jj < d; jj++) {
              const double u = xi[jj] - xj[jj];
              gk[1 + jj] = fma(coef * a.inv_beta[jj], u * u, gk[1 + jj]);
            }
            if (i == j) gk[d + 1] += wg;
          }
        }
      }
      __syncwarp();
    }
    // gradient slots: sigma2 | beta_1..beta_d | tau2 (DM > 0: tau2 is slot DM + 1,
    // slots d+1..DM belong to zero-padded dimensions)
    // ---- 6. fixed-order reductions: lanes (xor tree), warps (in order)
#pragma unroll
    for (int kk = 0; kk < GK; kk++) {
      const int dst = (DM > 0 && kk == DM + 1) ? P - 1 : kk;
      if ((DM > 0 && kk > d && kk <= DM) || (DM == 0 && kk >= P)) continue;
      double v = gk[kk];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp * P + dst] = v;
    }
    __syncthreads();
    for (int k = tid; k < P; k += kGThreads) {
      double v = 0.0;
      for (int w = 0; w < kGThreads / 32; w++) v += red[w * P + k];
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

size_t grad_smem_bytes(int max_N, int d) {
  const int ds = d <= 16 ? (d <= 4 ? 4 : d <= 8 ? 8 : d <= 10 ? 10 : d <= 12 ? 12 : 16) : d;
  return sizeof(double) * ((size_t)max_N * ds + 3 * (size_t)max_N + 8 * (size_t)(d + 2) + SBV_MAX_D +
                           8 * 32 * 33);
}

static int grad_dm(int d) {
  if (d <= 4) return 4;
  if (d <= 8) return 8;
  if (d <= 10) return 10;
  if (d <= 12) return 12;
  if (d <= 16) return 16;
  return 0;
}

template <int NU2>
static void (*pick_grad(int dm))(GradArgs) {
  switch (dm) {
    case 4: return k_grad<NU2, 4>;
    case 8: return k_grad<NU2, 8>;
    case 10: return k_grad<NU2, 10>;
    case 12: return k_grad<NU2, 12>;
    case 16: return k_grad<NU2, 16>;
    default: return k_grad<NU2, 0>;
  }
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
  const int dm = grad_dm(gl.d);
  void (*f)(GradArgs) = nu == 0.5 ? pick_grad<1>(dm) : nu == 1.5 ? pick_grad<3>(dm) : nu == 2.5 ? pick_grad<5>(dm) : pick_grad<7>(dm);
  const size_t sm = grad_smem_bytes(gl.max_N, gl.d);
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  f<<<gl.grid, kGThreads, sm, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_grad_sum(const double *grads, int64_t k_local, int P, double *out, cudaStream_t st) {
  k_grad_sum<<<P, 32, 0, st>>>(grads, k_local, P, out);
  return cudaGetLastError();
}

}  // namespace sbv
