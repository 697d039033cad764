// k-loop ceiling for RT x 4 accumulator tiles per warp, W warps per CTA, C CTAs/SM,
// operand fragments from a per-CTA workspace (fragment micro-tile layout).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int RT, int W, int MINB>
__global__ void __launch_bounds__(32 * W, MINB) kloop(const double* ws, size_t ws_per_cta, int np, int reps, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double* wsb = ws + blockIdx.x * ws_per_cta + lane;
  double acc[RT][4][2] = {};
  for (int r = 0; r < reps; r++) {
    for (int p = 0; p < np; p++) {
      const double* base = wsb + (size_t)p * 64 * 256 * 4;
      const double* Ab = base + (size_t)(8 + w * RT) * 256;
      const double* Bb = base;
      double a[2][RT], b[2][4];
#pragma unroll
      for (int x = 0; x < RT; x++) a[0][x] = Ab[x * 256];
#pragma unroll
      for (int x = 0; x < 4; x++) b[0][x] = Bb[x * 256];
#pragma unroll
      for (int s = 0; s < 8; s++) {
        if (s + 1 < 8) {
#pragma unroll
          for (int x = 0; x < RT; x++) a[(s + 1) & 1][x] = Ab[x * 256 + (s + 1) * 32];
#pragma unroll
          for (int x = 0; x < 4; x++) b[(s + 1) & 1][x] = Bb[x * 256 + (s + 1) * 32];
        }
#pragma unroll
        for (int rt = 0; rt < RT; rt++)
#pragma unroll
          for (int ct = 0; ct < 4; ct++) dmma(acc[rt][ct][0], acc[rt][ct][1], a[s & 1][rt], b[s & 1][ct]);
      }
    }
  }
  double s = 0; for (int i = 0; i < RT; i++) for (int j = 0; j < 4; j++) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[0] = s;
}
template <int RT, int W, int MINB>
void run(int sms, int ctas, double* ws, size_t per, double* out, int np, int reps) {
  int grid = sms * ctas;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kloop<RT, W, MINB><<<grid, 32 * W>>>(ws, per, np, 1, out);
  cudaEventRecord(e0);
  kloop<RT, W, MINB><<<grid, 32 * W>>>(ws, per, np, reps, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = (double)grid * W * reps * np * 8 * (RT * 4) * 512.0;
  printf("{\"RT\":%d,\"warps\":%d,\"ctas_per_sm\":%d,\"tflops\":%.2f}\n", RT, W, ctas, flops / ms / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int np = 10, reps = 20;
  const size_t per = (size_t)np * 64 * 256 * 4;
  double* ws; cudaMalloc(&ws, per * sms * 4 * 8 + 64); cudaMemset(ws, 0, per * sms * 4 * 8);
  double* out; cudaMalloc(&out, 64);
  run<4, 8, 2>(sms, 2, ws, per, out, np, reps);
  run<2, 16, 1>(sms, 1, ws, per, out, np, reps);
  run<2, 8, 2>(sms, 2, ws, per, out, np, reps);
  run<2, 16, 2>(sms, 2, ws, per, out, np, reps);
  run<4, 16, 1>(sms, 1, ws, per, out, np, reps);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
