// EXPERIMENT (not built): block-slot variant of k_h8, measured slower (12.2 vs 10.2 ms at cfg2); see profiles/r02/h8_experiments.md
// h8s_kernel.cuh — H8 with block SLOTS: the same per-block task graph as k_h8
// (h8_kernel.cuh: one bordered Cholesky per block, Alg.5, left-
// looking 32-column panels on DMMA), but one CTA of 16 warps per SM keeps
// kSlots blocks in flight in shared memory and its warps are not tied to a
// block.
//
// Why: with one block per CTA (k_h8, 2 CTAs x 8 warps per SM) the warps of a
// CTA idle at the end of every block (the last panels have little parallel
// work: tools/h8_trace.py measured 16% of the warp time in staging, the tail
// and the end-of-block barrier) and while the block's panel chain
// F(j) -> BC(j,1) -> F(j+1) waits.  Here a slot that finishes is refilled by
// whichever warp finds it empty while the other slot keeps the SM busy.
//
// Roles: warp s < kSlots is slot s's chain warp (the chain list F(0), BC(0,1),
// F(1), ... of that slot, then that slot's bulk tasks); warps kSlots.. are
// bulk warps that take bulk tasks from any active slot, older block first.
// Deadlock freedom: every task waits only on earlier tasks of its own slot's
// topological order (see h8_kernel.cuh), a chain warp only ever holds tasks
// of its own slot, so every slot progresses independently of the others.
// Dispensing is epoch-guarded (a 64-bit {epoch, next ticket} word taken with
// atomicCAS), so a warp holding a stale view of a recycled slot never takes
// a ticket of the new block by accident.
#pragma once
#include "h8_kernel.cuh"

namespace sbv {

#ifndef SBV_SLOTS
#define SBV_SLOTS 2
#endif
constexpr int kSlots = SBV_SLOTS;
constexpr int kSWarps = 16;
constexpr int kSThreads = 32 * kSWarps;
enum : int { kSlotEmpty = 0, kSlotStaging = 1, kSlotActive = 2, kSlotRetired = 3 };

struct SlotLayout {  // offsets (in doubles / ints) of one slot's shared-memory arrays
  int dbl;           // doubles per slot: Dt2 Mn2 | xref | ys | vs | qp lp
  int ints;          // ints per slot: doneA doneC | cntC doneF | tasks
};

__host__ __device__ inline SlotLayout h8s_layout(int np_max, int cp_max, int max_N, int ds, int max_tasks) {
  SlotLayout L;
  L.dbl = 4 * kPanel * kDld + SBV_MAX_D + (cp_max + 8) + max_N * ds + 2 * np_max;
  L.dbl = (L.dbl + 1) & ~1;
  const int nchmax = np_max + 1;
  L.ints = 2 * np_max * nchmax + 2 * np_max + max_tasks;
  L.ints = (L.ints + 3) & ~3;
  return L;
}

// ticket from a {epoch:32 | next:32} word; -1 if the epoch moved or the list is exhausted
__device__ __forceinline__ int take_ticket(unsigned long long *word, unsigned epoch, int limit) {
  unsigned long long old = *(volatile unsigned long long *)word;
  for (;;) {
    if ((unsigned)(old >> 32) != epoch) return -1;
    const int nx = (int)(unsigned)old;
    if (nx >= limit) return -1;
    const unsigned long long prev = atomicCAS(word, old, old + 1ull);
    if (prev == old) return nx;
    old = prev;
  }
}

template <int NU2, int DM>
__global__ void __launch_bounds__(kSThreads, 1) k_h8s(H8Args a) {
  extern __shared__ double smem[];
  __shared__ int sh_state[kSlots];  // (epoch << 8) | state
  __shared__ unsigned long long sh_word[kSlots], sh_cword[kSlots];  // bulk / chain tickets
  __shared__ int sh_ntask[kSlots], sh_nchain[kSlots], sh_ndone[kSlots], sh_npbuilt[kSlots];
  __shared__ int sh_item[kSlots], sh_li[kSlots], sh_N[kSlots], sh_mt[kSlots], sh_bst[kSlots];
  __shared__ long long sh_b0[kSlots];
  __shared__ int sh_fail[kSlots], sh_fail_stage[kSlots];
  __shared__ int sh_retired;
  __shared__ double s_etab[256];
  __shared__ double s_ib[SBV_MAX_D];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int d = a.d;
  const int npmax = a.np_max, nchmax = npmax + 1;
  const int DS = DM > 0 ? DM : d;
  const int cp_max = npmax * kPanel;
  const SlotLayout SL = h8s_layout(npmax, cp_max, a.max_N, DS, a.max_tasks);
  int *ismem = reinterpret_cast<int *>(smem + (size_t)kSlots * SL.dbl);
  for (int j = tid; j < d; j += kSThreads) s_ib[j] = a.inv_beta[j];
#if SBV_EXP_TAB256
  for (int j = tid; j < 256; j += kSThreads) s_etab[j] = -a.sigma2 * exp2(j / 256.0);
#else
  for (int j = tid; j < 64; j += kSThreads) s_etab[j] = exp2(j / 64.0);
#endif
  if (tid < kSlots) {
    sh_state[tid] = kSlotEmpty;
    sh_word[tid] = 0ull;
    sh_cword[tid] = 0ull;
    sh_npbuilt[tid] = -1;
    sh_item[tid] = 0x7fffffff;
  }
  if (tid == 0) sh_retired = 0;
  __syncthreads();
  const double mpf = -a.sigma2 * exp((1.0 - a.nu) * 0.69314718055994530942 - lgamma(a.nu));

  for (;;) {
    // ---------------------------------------------------------------- pick work
    int act = 0, s = -1, ti = -1;
    unsigned epoch = 0;
    if (lane == 0) {
      int order[kSlots];
      for (int i = 0; i < kSlots; i++) order[i] = i;
      for (int i = 1; i < kSlots; i++)  // older block (lower item) first
        for (int k = i; k > 0 && *(volatile int *)&sh_item[order[k]] < *(volatile int *)&sh_item[order[k - 1]]; k--) {
          const int t_ = order[k];
          order[k] = order[k - 1];
          order[k - 1] = t_;
        }
      for (int i = 0; i < kSlots && act == 0; i++) {
        const int sl = order[i];
        if (warp < kSlots && sl != warp) continue;  // chain warps serve their own slot only
        const int st = *(volatile int *)&sh_state[sl];
        if ((st & 0xff) != kSlotActive) continue;
        const unsigned ep = (unsigned)st >> 8;
        __threadfence_block();
        const int nc = *(volatile int *)&sh_nchain[sl], nt = *(volatile int *)&sh_ntask[sl];
        int t_ = -1;
        if (warp == sl) t_ = take_ticket(&sh_cword[sl], ep, nc);
        if (t_ < 0) {
          t_ = take_ticket(&sh_word[sl], ep, nt - nc);
          if (t_ >= 0) t_ += nc;
        }
        if (t_ >= 0) {
          act = 1;
          s = sl;
          ti = t_;
          epoch = ep;
        }
      }
      if (act == 0) {  // refill an empty slot (a chain warp only its own)
        for (int sl = 0; sl < kSlots && act == 0; sl++) {
          if (warp < kSlots && sl != warp) continue;
          const int st = *(volatile int *)&sh_state[sl];
          if ((st & 0xff) == kSlotEmpty &&
              atomicCAS(&sh_state[sl], st, (st & ~0xff) | kSlotStaging) == st) {
            act = 2;
            s = sl;
            epoch = (unsigned)st >> 8;
          }
        }
      }
      if (act == 0) {
        if (warp < kSlots) {
          if ((*(volatile int *)&sh_state[warp] & 0xff) == kSlotRetired) act = 3;
        } else if (*(volatile int *)&sh_retired == kSlots) {
          act = 3;
        }
      }
    }
    act = __shfl_sync(0xffffffffu, act, 0);
    if (act == 3) break;
    if (act == 0) {
      __nanosleep(64);
      continue;
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    ti = __shfl_sync(0xffffffffu, ti, 0);
    epoch = __shfl_sync(0xffffffffu, epoch, 0);

    // ---------------------------------------------------------------- slot s arrays
    double *sd = smem + (size_t)s * SL.dbl;
    double *Dt2 = sd;
    double *Mn2 = Dt2 + 2 * kPanel * kDld;
    double *xref = Mn2 + 2 * kPanel * kDld;
    double *ys = xref + SBV_MAX_D;
    double *vs = ys + cp_max + 8;
    double *s_qp = vs + (size_t)a.max_N * DS;
    double *s_lp = s_qp + npmax;
    int *si = ismem + (size_t)s * SL.ints;
    int *doneA = si;
    int *doneC = doneA + npmax * nchmax;
    int *cntC = doneC + npmax * nchmax;
    int *doneF = cntC + npmax;
    int *tasks = doneF + npmax;
    double *wsb = a.ws + ((size_t)blockIdx.x * kSlots + s) * a.ws_per_cta;

    if (act == 2) {
      // ------------------------------------------------------------ stage a block into slot s
      int item = 0;
      if (lane == 0) item = (int)atomicAdd(a.queue, 1u);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= a.k_local) {
        if (lane == 0) {
          sh_item[s] = 0x7fffffff;
          __threadfence_block();
          atomicExch(&sh_state[s], (int)((epoch << 8) | kSlotRetired));
          atomicAdd(&sh_retired, 1);
        }
        __syncwarp();
        continue;
      }
#if SBV_TRACE
      const long long tstage = clock64();
#endif
      const int li = a.work_order[item];
      const int64_t t = a.local_blocks[li];
      const int mt = a.cnt[li];
      const int64_t b0 = a.off[t];
      const int bst = (int)(a.off[t + 1] - b0);
      const int N = mt + bst;
      const int Cp = (N + kPanel - 1) / kPanel * kPanel;
      const int R = Cp + 8;
      const int NP = Cp / kPanel;
      const int nch0 = ((R >> 3) + 3) >> 2;
      for (int j = lane; j < d; j += 32) xref[j] = a.Xp[b0 * d + j];
      for (int i = lane; i < NP * nchmax; i += 32) {
        doneA[i] = 0;
        doneC[i] = 0;
      }
      for (int i = lane; i < NP; i += 32) {
        cntC[i] = 0;
        doneF[i] = 0;
      }
      __syncwarp();
#pragma unroll 4
      for (int e = lane; e < N * DS; e += 32) {
        const int i = e / DS, j = e - i * DS;
        const int64_t pos = i < mt ? (int64_t)SBV_LDS_(&a.nbr[(int64_t)li * a.m + i]) : b0 + (i - mt);
        vs[e] = j < d ? (SBV_LDS_(&a.Xp[pos * d + j]) - xref[j]) * s_ib[j] : 0.0;
      }
      for (int i = lane; i < Cp + 8; i += 32) {
        double v = 0.0;
        if (i < N) {
          const int64_t pos = i < mt ? (int64_t)SBV_LDS_(&a.nbr[(int64_t)li * a.m + i]) : b0 + (i - mt);
          v = SBV_LDS_(&a.yperm[pos]);
        }
        ys[i] = v;
      }
      // every lane's staging writes are ordered before lane 0 publishes the slot
      __threadfence_block();
      __syncwarp();
      if (lane == 0) {
        if (NP != sh_npbuilt[s]) {
          // chain list [0, nc): F(0), BC(0,1), F(1), ..., F(NP-1); bulk list
          // after it in the single-list order of h8_kernel.cuh
          const int nc = 2 * NP - 1;
          int n = nc, c = 0;
          auto addA = [&](int j) {
            if (j < NP)
              for (int ch = 0; ch < nch0 - j; ch++) tasks[n++] = enc_task(kTaskA, j, ch);
          };
          addA(0);
          addA(1);
          tasks[c++] = enc_task(kTaskF, 0, 0);
          for (int j = 0; j < NP; j++) {
            const int nch = nch0 - j;
            if (j + 1 < NP) {
              tasks[c++] = enc_task(kTaskBC, j, 1);
              tasks[c++] = enc_task(kTaskF, j + 1, 0);
            } else {
              tasks[n++] = enc_task(kTaskBC, j, 1);
            }
            for (int ch = 2; ch < nch; ch++) {
              tasks[n++] = enc_task(kTaskBC, j, ch);
              if (j + 2 < NP) tasks[n++] = enc_task(kTaskA, j + 2, ch - 2);
            }
          }
          sh_ntask[s] = n;
          sh_nchain[s] = nc;
          sh_npbuilt[s] = NP;
        }
        sh_li[s] = li;
        sh_N[s] = N;
        sh_mt[s] = mt;
        sh_bst[s] = bst;
        sh_b0[s] = b0;
        sh_fail[s] = 0;
        sh_fail_stage[s] = 0;
        sh_ndone[s] = 0;
        sh_item[s] = item;
        const unsigned ne = epoch + 1;
        sh_word[s] = (unsigned long long)ne << 32;
        sh_cword[s] = (unsigned long long)ne << 32;
        __threadfence_block();
        atomicExch(&sh_state[s], (int)((ne << 8) | kSlotActive));
      }
      __syncwarp();
#if SBV_TRACE
      if (lane == 0) trace_rec(a, tstage, tstage, item, (int)(0xFE000000u | (unsigned)N));
#endif
      continue;
    }

    // -------------------------------------------------------------- run task ti of slot s
#if SBV_TRACE
    const long long tt0 = clock64();
    long long tt1 = tt0;
#endif
    __threadfence_block();
    BlockCtx b;
    b.mt = *(volatile int *)&sh_mt[s];
    b.N = *(volatile int *)&sh_N[s];
    b.Cp = (b.N + kPanel - 1) / kPanel * kPanel;
    b.R = b.Cp + 8;
    b.d = DS;
    b.msigma2 = -a.sigma2;
    b.etab = s_etab;
    b.nu = a.nu;
    b.mpf = mpf;
    b.mtau2 = -a.tau2;
    b.ys = ys;
    b.vs = vs;
    const int NP = b.Cp / kPanel;
    const int nch0 = ((b.R >> 3) + 3) >> 2;
    const int item = *(volatile int *)&sh_item[s];
    constexpr int kNoC0 = 1;
    const int code = tasks[ti];
    const int type = code >> 24, j = (code >> 12) & 0xfff, ch = code & 0xfff;
    const int c0 = j * kPanel;
    b.c0 = c0;
    const int nrt = (b.R - c0) >> 3;
    const int tb = 4 * ch, nv = min(4, nrt - tb);
    double *pan = wsb + panel_base(j, b.R);
    double *Dt = Dt2 + (j & 1) * kPanel * kDld;
    double *Mn = Mn2 + (j & 1) * kPanel * kDld;
    double acc[4][4][2];
    if (type == kTaskA) {
      if (SBV_A_GEN_FIRST) {
        gen_chunk<NU2, DM>(pan, b, tb, nv, lane);
        __syncwarp();
      }
      if (j >= 2) {
        spin_until(&doneC[(j - 2) * nchmax + 2], 1);
        spin_until(&doneC[(j - 2) * nchmax + ch + 2], 1);
      }
    } else if (type == kTaskF) {
      spin_until(&doneA[j * nchmax], 1);
      if (j >= 1) spin_until(&doneC[(j - 1) * nchmax + 1], 1);
      if (j >= 2) spin_until(&cntC[j - 2], nch0 - (j - 2) - kNoC0);
    } else {
      spin_until(&doneF[j], 1);
      spin_until(&doneA[j * nchmax + ch], 1);
      if (j >= 1) {
        spin_until(&doneC[(j - 1) * nchmax + 1], 1);
        spin_until(&doneC[(j - 1) * nchmax + ch + 1], 1);
      }
    }
    __threadfence_block();
#if SBV_TRACE
    tt1 = clock64();
#endif
    const int p0 = type == kTaskA ? 0 : max(j - 1, 0);
    const int p1 = type == kTaskA ? j - 1 : j;
    const bool upd = p1 > p0;
    if (type == kTaskA && !SBV_A_GEN_FIRST) {
      gen_chunk<NU2, DM>(pan, b, tb, nv, lane);
      __syncwarp();
    }
    if (type != kTaskA || upd) unpark_tiles(acc, pan, tb, nv, g, q);
    if (upd) update_tiles(acc, wsb, c0, b.R, tb, nv, lane, p0, p1, nullptr);
    if (type == kTaskF) {
#pragma unroll
      for (int rt = 0; rt < 4; rt++)
#pragma unroll
        for (int ct = 0; ct < 4; ct++)
#pragma unroll
          for (int i = 0; i < 2; i++) Dt[(rt * 8 + g) * kDld + ct * 8 + 2 * q + i] = -acc[rt][ct][i];
      __syncwarp();
      diag_factor2(Dt, Mn, lane, b, sh_fail[s], sh_fail_stage[s]);
      __syncwarp();
      __threadfence_block();
      if (lane == 0) *(volatile int *)&doneF[j] = 1;
    } else {
      if (type == kTaskBC) trsm_tiles(acc, Dt, Mn, nv, g, q);
      if (type != kTaskA || upd) park_tiles(acc, pan, tb, nv, g, q);
      if (type == kTaskA) {
        __syncwarp();
        __threadfence_block();
        if (lane == 0) *(volatile int *)&doneA[j * nchmax + ch] = 1;
      } else {
        const int rb = (b.Cp - c0) >> 3;  // row tile of the border row
        if (rb >= tb && rb < tb + nv) {
          double qp = 0.0;
          if (g == 0) {
#pragma unroll
            for (int rt = 0; rt < 4; rt++)
              if (tb + rt == rb)
#pragma unroll
                for (int ct = 0; ct < 4; ct++)
#pragma unroll
                  for (int i = 0; i < 2; i++) {
                    const int col = c0 + ct * 8 + 2 * q + i;
                    if (col >= b.mt && col < b.N) qp = fma(acc[rt][ct][i], acc[rt][ct][i], qp);
                  }
          }
          double lp = 0.0;
          {
            const int col = c0 + lane;
            if (col >= b.mt && col < b.N) lp = log(Dt[lane * kDld + lane]);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            qp += __shfl_xor_sync(0xffffffffu, qp, o);
            lp += __shfl_xor_sync(0xffffffffu, lp, o);
          }
          if (lane == 0) {
            s_qp[j] = qp;
            s_lp[j] = lp;
          }
        }
        __syncwarp();
        __threadfence_block();
        if (lane == 0) {
          *(volatile int *)&doneC[j * nchmax + ch] = 1;
          atomicAdd(&cntC[j], 1);
        }
      }
    }
#if SBV_TRACE
    trace_rec(a, tt0, tt1, item, code);
#endif
    // ---------------------------------------------------------------- completion
    int last = 0;
    if (lane == 0) last = (atomicAdd(&sh_ndone[s], 1) + 1 == *(volatile int *)&sh_ntask[s]);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      const int li = sh_li[s];
      if (lane == 0) {
        double qs = 0.0, ls = 0.0;
        for (int jj = 0; jj < NP; jj++) {
          qs += s_qp[jj];
          ls += s_lp[jj];
        }
        ls *= 2.0;
        const int bst = sh_bst[s];
        const double term = -0.5 * (qs + ls) - 0.5 * (double)bst * 1.8378770664093454836;  // log 2pi
        a.terms[li] = sh_fail[s] ? NAN : term;
        a.quads[li] = qs;
        a.logdets[li] = ls;
        a.status[li] = sh_fail[s] ? sh_fail_stage[s] : 0;
      }
#if SBV_DISCARD_WS
      {
        const size_t used = panel_base(NP, b.R);
        for (size_t o = (size_t)lane * 16; o < used; o += 32 * 16)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(wsb + o) : "memory");
      }
#endif
#if SBV_TRACE
      if (lane == 0) trace_rec(a, clock64(), clock64(), item, (int)(0xFF000000u | (unsigned)b.N));
#endif
      __syncwarp();
      if (lane == 0) {
        sh_item[s] = 0x7fffffff;
        __threadfence_block();
        atomicExch(&sh_state[s], (int)((epoch << 8) | kSlotEmpty));
      }
      __syncwarp();
    }
  }
}

typedef void (*H8SFn)(H8Args);
H8SFn h8s_pick_nu0(int dm);
H8SFn h8s_pick_nu1(int dm);
H8SFn h8s_pick_nu3(int dm);
H8SFn h8s_pick_nu5(int dm);
H8SFn h8s_pick_nu7(int dm);

}  // namespace sbv
