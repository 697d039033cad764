// h8_micro.cu — FP64 latency microbenchmarks for the H8 critical chain (tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I <nccl inc>
//        tools/h8_micro.cu -o tools/h8_micro
// Prints one JSON line per measurement: dependent-chain latencies (cycles) of
// DFMA, DMMA.8x8x4, double shuffles, rsqrt(double), log(double), and the
// cycles of one 32x32 diag_factor (h8_kernel.cuh) by one warp, alone and next
// to background warps streaming DMMAs or DFMAs on the same SM.
#include <cstdio>
#include <vector>

#include "../paper_2504_12004_b200/csrc/h8_kernel.cuh"

using namespace sbv;

__global__ void k_lat(int kind, int iters, double seed, long long *out, double *sink) {
  double a = seed + threadIdx.x * 1e-3, b = 1.0000001, c0 = 0.5, c1 = 0.25;
  long long t0 = clock64();
  if (kind == 0) {
    for (int i = 0; i < iters; i++) a = fma(a, b, 1e-9);
  } else if (kind == 1) {
    for (int i = 0; i < iters; i++) dmma(c0, c1, a, b);
  } else if (kind == 2) {
    for (int i = 0; i < iters; i++) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31) * b;
  } else if (kind == 3) {
    for (int i = 0; i < iters; i++) a = rsqrt(a) + 1.0;
  } else if (kind == 4) {
    for (int i = 0; i < iters; i++) a = log(a) + 2.0;
  } else if (kind == 5) {
    for (int i = 0; i < iters; i++) a = exp_neg(a) + 0.5;
  } else if (kind == 6) {
    for (int i = 0; i < iters; i++) a = sqrt(a) + 1.0;
  } else if (kind == 7) {
    for (int i = 0; i < iters; i++) a = rsqrt_pos(a) + 1.0;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  sink[threadIdx.x] = a + c0 + c1;
}


// both factorisations of one tile: outputs of diag_factor (old) and
// diag_factor2 (new) written to out[0..2*32*kDld*2)
__global__ void k_cmp(const double *A, double *out) {
  __shared__ double Dt[kPanel * kDld], Mn[kPanel * kDld];
  __shared__ int s_fail, s_fail_stage;
  const int lane = threadIdx.x;
  BlockCtx b{};
  b.N = 32;
  double lp = 0;
  for (int v = 0; v < 2; v++) {
    for (int i = lane; i < kPanel * kDld; i += 32) Mn[i] = 0.0;
    for (int i = lane; i < 32 * 32; i += 32) Dt[(i / 32) * kDld + (i % 32)] = A[i];
    if (lane == 0) s_fail = 0;
    __syncwarp();
    if (v == 0)
      diag_factor(Dt, Mn, lane, b, &lp, s_fail, s_fail_stage);
    else
      diag_factor2(Dt, Mn, lane, b, s_fail, s_fail_stage);
    __syncwarp();
    for (int i = lane; i < kPanel * kDld; i += 32) {
      out[v * 2 * kPanel * kDld + i] = Dt[i];
      out[v * 2 * kPanel * kDld + kPanel * kDld + i] = Mn[i];
    }
    __syncwarp();
  }
}

// warp 0: diag_factor `reps` times on a fresh copy of an SPD tile;
// warps 1..: background (0 none, 1 DMMA stream, 2 DFMA stream) until warp 0 is done
__global__ void k_diag(const double *A, int reps, int bg, int newf, long long *out, double *sink) {
  __shared__ double Dt[kPanel * kDld], Mn[kPanel * kDld];
  __shared__ volatile int done;
  __shared__ int s_fail, s_fail_stage;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    done = 0;
    s_fail = 0;
    s_fail_stage = 0;
  }
  __syncthreads();
  if (w == 0) {
    BlockCtx b{};
    b.c0 = 0;
    b.N = 32;
    b.mt = 0;
    long long tot = 0;
    double lp = 0;
    for (int r = 0; r < reps; r++) {
      for (int i = lane; i < 32 * 32; i += 32) Dt[(i / 32) * kDld + (i % 32)] = A[i];
      __syncwarp();
      long long t0 = clock64();
      if (newf)
        diag_factor2(Dt, Mn, lane, b, s_fail, s_fail_stage);
      else
        diag_factor(Dt, Mn, lane, b, &lp, s_fail, s_fail_stage);
      __syncwarp();
      tot += clock64() - t0;
    }
    if (lane == 0) {
      out[0] = tot / reps;
      out[1] = s_fail;
      done = 1;
    }
  } else if (bg) {
    double c0 = 0, c1 = 0, a = 1.0 + lane, bb = 0.999;
    double x[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    while (!done) {
      if (bg == 1) {
#pragma unroll
        for (int i = 0; i < 64; i++) dmma(c0, c1, a, bb);
      } else {
#pragma unroll
        for (int i = 0; i < 64; i++)
#pragma unroll
          for (int k = 0; k < 8; k++) x[k] = fma(x[k], bb, 1e-9);
      }
    }
    sink[threadIdx.x] = c0 + c1 + x[0] + x[7];
  }
}

int main() {
  long long *d_out;
  double *sink;
  cudaMalloc(&d_out, 16 * sizeof(long long));
  cudaMalloc(&sink, 4096 * sizeof(double));
  const char *names[] = {"dfma", "dmma_acc", "shfl_f64", "rsqrt_f64", "log_f64", "exp_neg", "sqrt_f64", "rsqrt_pos"};
  for (int kind = 0; kind < 8; kind++) {
    const int iters = 4096;
    k_lat<<<1, 32>>>(kind, iters, 1.5, d_out, sink);
    long long cyc;
    cudaMemcpy(&cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
    printf("{\"kind\":\"lat_%s\",\"cycles_per_op\":%.2f}\n", names[kind], (double)cyc / iters);
  }
  // SPD 32x32: exp(-|i-j|/8) + 1e-4 I
  std::vector<double> A(32 * 32);
  for (int i = 0; i < 32; i++)
    for (int j = 0; j < 32; j++) A[i * 32 + j] = exp(-fabs(i - j) / 8.0) + (i == j ? 1e-4 : 0.0);
  double *dA;
  cudaMalloc(&dA, A.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  for (int newf = 0; newf < 2; newf++)
  for (int bg = 0; bg < 3; bg++)
    for (int warps : {1, 4, 8, 12}) {
      if (bg == 0 && warps > 1) continue;
      k_diag<<<1, 32 * warps>>>(dA, 20, bg, newf, d_out, sink);
      long long o[2];
      cudaMemcpy(o, d_out, sizeof(o), cudaMemcpyDeviceToHost);
      printf("{\"kind\":\"%s\",\"background\":\"%s\",\"warps\":%d,\"cycles\":%lld,\"fail\":%lld}\n",
             newf ? "diag_factor2_32" : "diag_factor_32", bg == 0 ? "none" : bg == 1 ? "dmma" : "dfma", warps, o[0], o[1]);
    }
  {
    const size_t sz = 2 * kPanel * kDld;
    double *dout;
    cudaMalloc(&dout, 2 * sz * 8);
    k_cmp<<<1, 32>>>(dA, dout);
    std::vector<double> h(2 * sz);
    cudaMemcpy(h.data(), dout, 2 * sz * 8, cudaMemcpyDeviceToHost);
    double maxd = 0, maxm = 0;
    for (int i = 0; i < 32; i++)
      for (int j = 0; j <= i; j++) {
        maxd = fmax(maxd, fabs(h[i * kDld + j] - h[sz + i * kDld + j]));
        if (i / 8 == j / 8) maxm = fmax(maxm, fabs(h[kPanel * kDld + i * kDld + j] - h[sz + kPanel * kDld + i * kDld + j]));
      }
    for (int i = 0; i < 32; i++)
      for (int j = i + 1; j < 32; j++)
        if (i / 8 == j / 8) maxm = fmax(maxm, fabs(h[sz + kPanel * kDld + i * kDld + j]));
    printf("{\"kind\":\"diag_factor2_vs_diag_factor\",\"max_abs_diff_L\":%.3e,\"max_abs_diff_minv\":%.3e}\n", maxd, maxm);
  }
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
