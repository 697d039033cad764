// Do DMMA (FP64 tensor) and DFMA (FP64 ALU) share a pipe on B200?  Warps of a
// CTA are split: role 0 runs a DMMA loop, role 1 a DFMA (or exp) loop.
#include <cstdio>
#include <cuda_runtime.h>
#define IT 2048
__device__ void dmma_loop(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5, c[8][2];
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < IT; it++)
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
__device__ void dfma_loop(double* out, double seed, int iters) {
  double a = seed + threadIdx.x, b = seed * 0.999, c[16];
  for (int i = 0; i < 16; i++) c[i] = i;
  for (int it = 0; it < iters; it++)
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(c[i], b, a);
  double s = 0; for (int i = 0; i < 16; i++) s += c[i];
  if (s == 1.2345) out[0] = s;
}
__device__ void exp_loop(double* out, double seed, int iters) {
  double x = seed + threadIdx.x * 1e-6, s = 0;
  for (int it = 0; it < iters; it++) { s += exp(-x); x += 1e-7; }
  if (s == 1.2345) out[0] = s;
}
// mode 0: all DMMA; 1: all DFMA; 2: half/half DMMA+DFMA; 3: all exp; 4: half DMMA + half exp
__global__ void k(double* out, int mode, int dfma_iters, int exp_iters) {
  int w = threadIdx.x >> 5;
  bool role1 = (mode == 1 || mode == 3) ? true : (mode == 0 ? false : (w & 1));
  if (!role1) dmma_loop(out, 1.0);
  else if (mode == 1 || mode == 2) dfma_loop(out, 1.0, dfma_iters);
  else exp_loop(out, 1.0, exp_iters);
}
int main() {
  double* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"dmma_only", "dfma_only", "dmma+dfma", "exp_only", "dmma+exp"};
  int dfma_iters = IT * 8;   // per-thread DFMA work comparable to the DMMA warps' time
  int exp_iters = 2048;
  for (int mode = 0; mode < 5; mode++) {
    int grid = sms * 2, block = 512;  // 32 warps/SM
    k<<<grid, block>>>(d, mode, dfma_iters, exp_iters);
    cudaEventRecord(e0);
    k<<<grid, block>>>(d, mode, dfma_iters, exp_iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double wps = (double)grid * block / 32;
    double nd = 0, nf = 0, ne = 0;
    if (mode == 0) nd = wps; if (mode == 1) nf = wps; if (mode == 2) { nd = wps / 2; nf = wps / 2; }
    if (mode == 3) ne = wps; if (mode == 4) { nd = wps / 2; ne = wps / 2; }
    double dmma_tf = nd * IT * 8 * 512.0 / ms / 1e9;
    double dfma_tf = nf * 32 * dfma_iters * 16 * 2.0 / ms / 1e9;
    double gexp = ne * 32 * exp_iters / ms / 1e6;
    printf("{\"mode\":\"%s\",\"ms\":%.3f,\"dmma_tflops\":%.2f,\"dfma_tflops\":%.2f,\"gexp_s\":%.1f}\n", names[mode], ms, dmma_tf, dfma_tf, gexp);
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
