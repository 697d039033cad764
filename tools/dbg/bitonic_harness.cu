#include "../../paper_2504_12004_b200/csrc/prep_kernels.cu"
#include <cstdio>
using namespace sbv;
__global__ void k_test(int cnt, const double* vals, int* bad) {
  __shared__ Cand buf[kKnnCap];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) { buf[i].d2 = vals[blockIdx.x * 2048 + i]; buf[i].orig = i; buf[i].pos = i; }
  __syncthreads();
  bitonic_sort(buf, cnt);
  if (threadIdx.x == 0) {
    for (int i = 1; i < cnt; i++) if (cand_less(buf[i].d2, buf[i].orig, buf[i-1].d2, buf[i-1].orig)) { atomicAdd(bad, 1); break; }
  }
}
int main() {
  const int B = 500; double* v; int* bad;
  cudaMallocManaged(&v, B * 2048 * 8); cudaMallocManaged(&bad, 4);
  unsigned long long s = 1;
  for (int i = 0; i < B * 2048; i++) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; v[i] = (s >> 11) * (1.0 / 9007199254740992.0); }
  int cnts[] = {5, 100, 1000, 1500, 1792, 1793, 1806, 2000, 2048};
  for (int c : cnts) { *bad = 0; k_test<<<B, 256>>>(c, v, bad); cudaDeviceSynchronize(); printf("cnt=%d bad=%d err=%s\n", c, *bad, cudaGetErrorString(cudaGetLastError())); }
}
