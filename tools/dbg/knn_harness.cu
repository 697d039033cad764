// Debug harness: runs sbv::k_knn on random bs=1 data vs a CPU full sort.
#include "../../paper_2504_12004_b200/csrc/prep_kernels.cu"
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cmath>
using namespace sbv;
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 3000, m = argc > 2 ? atoi(argv[2]) : 5, d = 3;
  std::mt19937_64 rng(5); std::uniform_real_distribution<double> U(0, 4);
  std::vector<double> S(n * d); for (auto& v : S) v = U(rng);
  std::vector<int32_t> perm(n), lb(n); std::vector<int64_t> off(n + 1);
  for (int i = 0; i < n; i++) { perm[i] = i; lb[i] = i; off[i] = i; } off[n] = n;
  double *dS; int32_t *dperm, *dlb, *dnbr, *dcnt; int64_t* doff;
  cudaMalloc(&dS, n * d * 8); cudaMalloc(&dperm, n * 4); cudaMalloc(&dlb, n * 4); cudaMalloc(&doff, (n + 1) * 8);
  cudaMalloc(&dnbr, n * m * 4); cudaMalloc(&dcnt, n * 4);
  cudaMemcpy(dS, S.data(), n * d * 8, cudaMemcpyHostToDevice); cudaMemcpy(dperm, perm.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dlb, lb.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(doff, off.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
  launch_knn(dS, dperm, doff, dS, dlb, n, d, m, dnbr, dcnt, 0);
  cudaError_t e = cudaDeviceSynchronize(); printf("err %s\n", cudaGetErrorString(e));
  std::vector<int32_t> nbr(n * m), cnt(n);
  cudaMemcpy(nbr.data(), dnbr, n * m * 4, cudaMemcpyDeviceToHost); cudaMemcpy(cnt.data(), dcnt, n * 4, cudaMemcpyDeviceToHost);
  int bad = 0, first = -1;
  for (int t = 0; t < n; t++) {
    std::vector<std::pair<double, int>> c;
    for (int p = 0; p < t; p++) { double acc = 0; for (int j = 0; j < d; j++) { double tt = S[t * d + j] - S[p * d + j]; acc = std::fma(tt, tt, acc); } c.push_back({acc, p}); }
    std::sort(c.begin(), c.end());
    int keep = std::min(t, m); bool ok = cnt[t] == keep;
    for (int j = 0; j < keep && ok; j++) ok = nbr[t * m + j] == c[j].second;
    if (!ok) { bad++; if (first < 0) first = t; }
  }
  printf("n=%d m=%d bad=%d first=%d\n", n, m, bad, first);
  return 0;
}
