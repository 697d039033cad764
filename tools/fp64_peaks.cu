// FP64 peak microbenchmarks for B200 (sm_100a): DMMA.8x8x4 (mma.sync f64) and DFMA.
// Used once to fill the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void dmma_loop(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_loop(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.999;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; i++) c[i] = i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void dexp_loop(double* out, double seed) {
  double x = seed + threadIdx.x * 1e-6, s = 0;
  for (int it = 0; it < 256; it++) { s += exp(-x); x += 1e-7; }
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    int grid = sms * 2, block = warps * 16;
    dmma_loop<<<grid, block>>>(d, 1.0);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) dmma_loop<<<grid, block>>>(d, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * grid * (block / 32) * (double)ITERS * 8 * 256 * 2;
    printf("{\"kind\":\"dmma_8x8x4\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", warps, flops / ms / 1e9);
  }
  for (int warps = 4; warps <= 32; warps *= 2) {
    int grid = sms * 2, block = warps * 16;
    dfma_loop<<<grid, block>>>(d, 1.0);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) dfma_loop<<<grid, block>>>(d, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * grid * block * (double)ITERS * 16 * 2;
    printf("{\"kind\":\"dfma\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", warps, flops / ms / 1e9);
  }
  {
    int grid = sms * 8, block = 512;
    dexp_loop<<<grid, block>>>(d, 1.0);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) dexp_loop<<<grid, block>>>(d, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = 5.0 * grid * block * 256;
    printf("{\"kind\":\"dexp\",\"gexp_per_s\":%.2f}\n", n / ms / 1e6);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
