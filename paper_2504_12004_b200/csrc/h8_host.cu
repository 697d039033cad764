// h8_host.cu — host side of H8 (h8_kernel.cuh): workspace / shared-memory
// sizing, occupancy, variant selection and launch.
#include <stdio.h>

#include <algorithm>

#include "h8_kernel.cuh"

namespace sbv {

static int h8_np_max(int max_N) { return (max_N + kPanel - 1) / kPanel; }
static int h8_max_tasks(int max_N) {
  const int np = h8_np_max(max_N), nch0 = (((np * kPanel + 8) >> 3) + 3) >> 2;
  int n = 0;
  // per panel: A x nch, BC x (nch - 1), F, C0, A2 (SBV_A0_EARLY)
  for (int j = 0; j < np; j++) n += 2 * (nch0 - j) + 2;
  return n + 4;
}

// staged coordinate stride: d rounded up to a compiled register width
// (0 = generic rolled loop with stride d)
static int h8_dm(int d) {
#ifdef SBV_FORCE_DM0  // experiment: generic rolled generation loop
  return 0;
#endif
  if (d <= 4) return 4;
  if (d <= 8) return 8;
  if (d <= 10) return 10;
  if (d <= 12) return 12;
  if (d <= 16) return 16;
  return 0;
}

size_t h8_smem_bytes(int max_N, int d) {
  const size_t Cp = (size_t)h8_np_max(max_N) * kPanel;
  const size_t np = h8_np_max(max_N), nch = np + 1;
  const size_t ints = 2 * np * nch + 2 * np + ((h8_max_tasks(max_N) + 1) & ~1);
  const size_t ds = h8_dm(d) > 0 ? (size_t)h8_dm(d) : (size_t)d;
  const size_t vs_smem = SBV_VS_GLOBAL ? 0 : (size_t)max_N * ds;  // else staged in global scratch
  return sizeof(double) * (4 * (size_t)kPanel * kDld + (kH8Threads / 32) * (size_t)kRingPerWarp +
                           2 * SBV_MAX_D + (Cp + 8) + vs_smem) +
         sizeof(int) * ((ints + 1) & ~(size_t)1);
}

// The split of an LPT-ordered launch (Nt_order: N of each work item, descending):
// items with N above the 2-CTA cap go first in a launch of their own.
void h8_split_plan(const int32_t *Nt_order, int64_t k, int d, int sms, int64_t *n_big, int *max_N_small,
                   int *grid_small) {
  const int cap = h8_two_cta_cap(d);
  int64_t nb = 0;
  while (nb < k && Nt_order[nb] > cap) nb++;
  *n_big = (nb > 0 && nb < k) ? nb : 0;
  *max_N_small = (nb < k) ? Nt_order[nb] : 0;
  int per_sm = 2;
  if (*n_big > 0) per_sm = std::max(1, h8_max_ctas_per_sm(h8_smem_bytes(*max_N_small, d), d));
  *grid_small = (int)std::min<int64_t>((int64_t)sms * per_sm, std::max<int64_t>(k - nb, 1));
}

// Largest N whose shared memory still leaves room for 2 CTAs per SM (dynamic +
// static <= ~113 KB).  A launch with larger blocks is split (launch_h8_problem):
// those blocks, first in the LPT order, run in their own launch sized for
// them (1 CTA/SM), the rest at 2 CTAs/SM -- instead of running the whole
// launch at 1 CTA/SM (measured round 2: one rank of a cfg5 run with max_N ~ 800
// lost 25% in H8).
int h8_two_cta_cap(int d) {
  const size_t budget = 105 * 1024;
  int lo = 1, hi = 4096;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (h8_smem_bytes(mid, d) <= budget)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// L panels of the largest block, then (ring builds) its staged coordinates
static size_t h8_l_doubles(int max_N) {
  const size_t Cp = (max_N + kPanel - 1) / kPanel * kPanel, R = Cp + 8, NP = Cp / kPanel;
  size_t tot = 0;
  for (size_t p = 0; p < NP; p++) tot += kPanel * (R - kPanel * p);
  return (tot + 63) / 64 * 64;
}

size_t h8_ws_doubles(int max_N, int d) {
  const size_t ds = h8_dm(d) > 0 ? (size_t)h8_dm(d) : (size_t)d;
  const size_t vs = SBV_VS_GLOBAL ? ((size_t)max_N * ds + 63) / 64 * 64 : 0;
  return h8_l_doubles(max_N) + vs;
}

static H8Fn pick_small(double nu, int d) {
  const int dm = h8_dm(d);
  if (nu == 0.5) return h8_pick_small_nu1(dm);
  if (nu == 1.5) return h8_pick_small_nu3(dm);
  if (nu == 2.5) return h8_pick_small_nu5(dm);
  return h8_pick_small_nu7(dm);
}

// A launch whose blocks are all small (max N <= kSmallMaxN: at most 6 panels,
// where the per-block panel chain, not the bulk work, sets the block's time)
// runs the SBV_H8_SMALL_WARPS-warp instantiation (4: 4 CTAs per SM, twice
// the concurrent chains).  Log-likelihood mode with a closed-form nu only; SBV_H8_SMALL=0
// disables it (A/B runs).
constexpr int kSmallMaxN = 192;
bool h8_use_small(int max_N) {
  static const int env = [] {
    const char *e = getenv("SBV_H8_SMALL");
    return e ? atoi(e) : 1;
  }();
  return env != 0 && max_N <= kSmallMaxN;
}
static bool closed_form(double nu) { return nu == 0.5 || nu == 1.5 || nu == 2.5 || nu == 3.5; }

int h8_small_ctas_per_sm(size_t smem, int d) {
  int best = 1 << 30;
  for (double nu : {0.5, 1.5, 2.5, 3.5}) {
    const H8Fn f = pick_small(nu, d);
    int nb = 0;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, 32 * SBV_H8_SMALL_WARPS, smem);
    best = nb < best ? nb : best;
  }
  return best;
}

static H8Fn pick(double nu, int d, int pred = 0) {
  const int dm = h8_dm(d);
  if (nu == 0.5) return h8_pick_nu1(dm, pred);
  if (nu == 1.5) return h8_pick_nu3(dm, pred);
  if (nu == 2.5) return h8_pick_nu5(dm, pred);
  if (nu == 3.5) return h8_pick_nu7(dm, pred);
  return h8_pick_nu0(dm, pred);  // general nu: K_nu path
}

int h8_max_ctas_per_sm(size_t smem, int d) {
  int best = 1 << 30;
  for (double nu : {0.5, 1.5, 2.5, 3.5, 1.0}) {  // the launch may use any smoothness
    const H8Fn f = pick(nu, d);
    int nb = 0;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kH8Threads, smem);
    best = nb < best ? nb : best;
  }
  return best;
}

cudaError_t launch_h8_problem(const H8Problem &pb, int d, const double *theta, unsigned int *queue,
                              cudaStream_t st) {
  H8Args a;
  a.Xp = pb.Xp;
  a.yperm = pb.yperm;
  a.off = pb.off;
  a.nbr = pb.nbr;
  a.cnt = pb.cnt;
  a.local_blocks = pb.local_blocks;
  a.work_order = pb.work_order;
  a.k_local = pb.k_local;
  a.m = pb.m > 0 ? pb.m : 1;
  a.d = d;
  a.sigma2 = theta[0];
  a.tau2 = theta[d + 2];
  a.nu = theta[d + 1];
  for (int j = 0; j < SBV_MAX_D; j++) a.inv_beta[j] = j < d ? 1.0 / theta[1 + j] : 0.0;
  a.theta_d = pb.theta_d;
  a.ws = pb.ws;
  a.ws_per_cta = pb.ws_per_cta;
  a.vs_off = h8_l_doubles(pb.max_N);
  a.queue = queue;
  a.terms = pb.terms;
  a.quads = pb.quads;
  a.logdets = pb.logdets;
  a.status = pb.status;
  a.np_max = h8_np_max(pb.max_N);
  a.max_tasks = h8_max_tasks(pb.max_N);
  a.max_N = pb.max_N;
  a.predict = pb.predict;
  a.Lg = pb.Lg;
  a.lg_off = pb.lg_off;
  a.Xq = pb.Xq;
  a.pmean = pb.pmean;
  a.pvar = pb.pvar;
  const double nu = theta[d + 1];
  cudaError_t e = cudaMemsetAsync(queue, 0, sizeof(unsigned int), st);
  if (e) return e;
  if (pb.k_local == 0) return cudaSuccess;
  a.trace = nullptr;
  a.trace_n = nullptr;
  a.trace_cap = 0;
#if SBV_TRACE  // tool-only build (tools/h8_trace.py): per-task timeline of this launch
  static unsigned long long *tbuf = nullptr;
  static unsigned int *tn = nullptr;
  const unsigned int cap = 4u << 20;
  if (!tbuf) {
    cudaMalloc(&tbuf, (size_t)cap * 6 * sizeof(unsigned long long));
    cudaMalloc(&tn, sizeof(unsigned int));
  }
  cudaMemsetAsync(tn, 0, sizeof(unsigned int), st);
  a.trace = tbuf;
  a.trace_n = tn;
  a.trace_cap = cap;
#endif
  if (pb.small && pb.predict == 0 && closed_form(nu)) {
    const H8Fn f = pick_small(nu, d);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pb.smem);
    f<<<pb.grid, 32 * SBV_H8_SMALL_WARPS, pb.smem, st>>>(a);
  } else {
    const H8Fn f = pick(nu, d, pb.predict);
    if (pb.n_big > 0 && pb.n_big < pb.k_local) {
      // split launch (h8_two_cta_cap): the n_big largest blocks (first in the
      // LPT order) with shared memory sized for them, then the rest at 2 CTAs/SM
      H8Args ab = a;
      ab.k_local = pb.n_big;
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pb.smem);
      f<<<(int)std::min<int64_t>(pb.grid, pb.n_big), kH8Threads, pb.smem, st>>>(ab);
      e = cudaMemsetAsync(queue, 0, sizeof(unsigned int), st);
      if (e) return e;
      H8Args as = a;
      as.work_order = pb.work_order + pb.n_big;
      as.k_local = pb.k_local - pb.n_big;
      as.np_max = h8_np_max(pb.max_N_small);
      as.max_tasks = h8_max_tasks(pb.max_N_small);
      const size_t sm2 = h8_smem_bytes(pb.max_N_small, d);
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      f<<<(int)std::min<int64_t>(pb.grid_small, as.k_local), kH8Threads, sm2, st>>>(as);
    } else {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pb.smem);
      f<<<pb.grid, kH8Threads, pb.smem, st>>>(a);
    }
  }
#if SBV_TRACE
  if (const char *out = getenv("SBV_TRACE_OUT")) {
    unsigned int n = 0;
    cudaMemcpyAsync(&n, tn, sizeof(n), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    n = n < cap ? n : cap;
    std::vector<unsigned long long> h((size_t)n * 6);
    cudaMemcpy(h.data(), tbuf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    if (FILE *fp = fopen(out, "wb")) {
      fwrite(h.data(), sizeof(unsigned long long), h.size(), fp);
      fclose(fp);
    }
  }
#endif
  return cudaGetLastError();
}

cudaError_t launch_h8(const Ctx &c, const double *theta, cudaStream_t st, const double *theta_dev) {
  H8Problem pb{};
  pb.Xp = c.Xperm;
  pb.yperm = c.yperm;
  pb.off = c.off;
  pb.nbr = c.nbr;
  pb.cnt = c.cnt;
  pb.local_blocks = c.local_blocks;
  pb.work_order = c.work_order;
  pb.k_local = c.k_local;
  pb.m = c.m;
  pb.max_N = c.max_N;
  pb.grid = c.h8_grid;
  pb.smem = c.h8_smem;
  pb.ws = c.ws;
  pb.ws_per_cta = c.ws_per_cta;
  pb.terms = c.terms;
  pb.quads = c.quads;
  pb.logdets = c.logdets;
  pb.status = c.status;
  pb.n_big = c.h8_n_big;
  pb.max_N_small = c.h8_max_N_small;
  pb.grid_small = c.h8_grid_small;
  pb.small = c.h8_small;
  pb.theta_d = theta_dev;
  return launch_h8_problem(pb, c.d, theta, c.queue, st);
}

}  // namespace sbv
