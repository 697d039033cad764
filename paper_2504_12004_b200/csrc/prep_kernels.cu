// prep_kernels.cu — sbv_prepare's device steps H1-H6 (Alg.1 Steps 1-3).
//
// Bit-exactness contract with the CPU oracle (indices must match exactly):
//  * scaling is one IEEE RN division per element (Alg.2 line 7);
//  * squared distances are the explicit fma chain acc = fma(t, t, acc) with
//    t = a_j - b_j in dimension order (Q14) — __fma_rn is
//    correctly rounded, so every distance is bit-identical to std::fma;
//  * centroids are left-to-right sums over members in ascending original
//    index followed by one division (Alg.4 line 6);
//  * every tie is broken by the lower anchor rank / original index (Q8, Q13).
#include <cub/cub.cuh>

#include "sbv_internal.cuh"

namespace sbv {

struct ScaleArg {
  double v[SBV_MAX_D];
};

// ------------------------------------------------------------------ H1
__global__ void k_scale(const double *__restrict__ X, int64_t total, int d, ScaleArg s,
                        double *__restrict__ S) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int j = (int)(e % d);
    S[e] = __ddiv_rn(X[e], s.v[j]);  // Alg.2: X_j := X_org,j / beta_j
  }
}

cudaError_t launch_scale(const double *X, int64_t n, int d, const double *scale_host, double *S,
                         cudaStream_t st) {
  ScaleArg a;
  for (int j = 0; j < d; j++) a.v[j] = scale_host[j];
  int64_t total = n * d;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_scale<<<grid, 256, 0, st>>>(X, total, d, a, S);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ H2
// splitmix64: i-th output of the generator seeded with `seed` (Q9).
__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void k_keys(int64_t n, uint64_t seed, uint64_t *keys, int32_t *vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = splitmix64(seed, (uint64_t)i);
    vals[i] = (int32_t)i;
  }
}

// Alg.3 line 4 + Alg.1 line 9: anchors = the k smallest (key, i), in that
// order; a stable LSD radix sort of (key -> i) with i ascending on input
// breaks equal keys by index.
cudaError_t select_anchors(int64_t n, int64_t k, uint64_t seed, int32_t *anchors, void *, size_t,
                           cudaStream_t st, size_t *) {
  uint64_t *kin = nullptr, *kout = nullptr;
  int32_t *vin = nullptr, *vout = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  if ((e = cudaMallocAsync(&kin, n * 8, st))) return e;
  if ((e = cudaMallocAsync(&kout, n * 8, st))) return e;
  if ((e = cudaMallocAsync(&vin, n * 4, st))) return e;
  if ((e = cudaMallocAsync(&vout, n * 4, st))) return e;
  k_keys<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(n, seed, kin, vin);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, kout, vin, vout, (int)n, 0, 64, st);
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return e;
  e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, vout, (int)n, 0, 64, st);
  if (e) return e;
  cudaMemcpyAsync(anchors, vout, k * 4, cudaMemcpyDeviceToDevice, st);
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(kin, st);
  cudaFreeAsync(kout, st);
  cudaFreeAsync(vin, st);
  cudaFreeAsync(vout, st);
  return cudaGetLastError();
}

// Fast path: the keys are uniform 64-bit integers, so the k smallest lie below
// T = (2k + 1024)/n * 2^64 with overwhelming probability.  *bad is set when the
// candidate set cannot be trusted (overflow of the 4k + 4096 slots, or fewer
// than k candidates); the caller then runs the full sort.
// Bucketed selection of the candidates below T: keys are uniform, so bucket
// b = floor(key / w), w = T/B + 1, holds about (2k + 1024)/B of them and is
// monotone in the key.  count -> exclusive scan -> scatter -> per-bucket
// insertion sort; the candidate of global rank r < k is anchor r.
// splitmix64 is a bijection of i (odd multiplier, xor-shifts, odd
// multipliers), so keys never tie and the key alone orders them (Q9).
constexpr int kScanThreads = 1024;
constexpr int kMaxBuckets = kScanThreads * 256;

__global__ void k_anc_count(int64_t n, uint64_t seed, uint64_t thr, uint64_t w, int *cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = splitmix64(seed, (uint64_t)i);
    if (key < thr) atomicAdd(&cnt[key / w], 1);
  }
}

// one CTA: start[b] = sum_{c<b} cnt[c]; cursor = start; start[B] = total
__global__ void __launch_bounds__(kScanThreads) k_anc_scan(const int *cnt, int B, int *start, int *cursor,
                                                           int *total) {
  __shared__ int part[kScanThreads];
  const int per = (B + kScanThreads - 1) / kScanThreads;
  const int b0 = threadIdx.x * per, b1 = min(B, b0 + per);
  int s = 0;
  for (int b = b0; b < b1; b++) s += cnt[b];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < kScanThreads; o <<= 1) {  // Hillis-Steele inclusive scan
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int b = b0; b < b1; b++) {
    start[b] = run;
    cursor[b] = run;
    run += cnt[b];
  }
  if (threadIdx.x == kScanThreads - 1) {
    start[B] = part[kScanThreads - 1];
    *total = part[kScanThreads - 1];
  }
}

__global__ void k_anc_scatter(int64_t n, uint64_t seed, uint64_t thr, uint64_t w, int cap, int *cursor,
                              uint64_t *ck, int32_t *ci) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = splitmix64(seed, (uint64_t)i);
    if (key < thr) {
      const int slot = atomicAdd(&cursor[key / w], 1);
      if (slot < cap) {
        ck[slot] = key;
        ci[slot] = (int32_t)i;
      }
    }
  }
}

__global__ void k_anc_finish(const int *start, int B, int cap, int64_t k, uint64_t *ck, int32_t *ci,
                             int32_t *anchors) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int s = start[b], e = min(start[b + 1], cap);
  if (s >= k || s >= e) return;
  for (int x = s + 1; x < e; x++) {  // insertion sort by key (a handful of items)
    const uint64_t kx = ck[x];
    const int32_t ix = ci[x];
    int y = x - 1;
    while (y >= s && ck[y] > kx) {
      ck[y + 1] = ck[y];
      ci[y + 1] = ci[y];
      y--;
    }
    ck[y + 1] = kx;
    ci[y + 1] = ix;
  }
  for (int r = s; r < e && r < k; r++) anchors[r] = ci[r];
}

__global__ void k_anchor_check(const int *count, int cap, int64_t k, int *bad) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *bad = (*count > cap || *count < k) ? 1 : 0;
}

cudaError_t select_anchors_fast(int64_t n, int64_t k, uint64_t seed, int32_t *anchors, int *bad,
                                cudaStream_t st) {
  const double frac = std::min(1.0, (2.0 * k + 1024.0) / (double)n);
  const int cap = (int)std::min<int64_t>(4 * k + 4096, INT32_MAX / 2);
  int B = 1;
  while (B < (2 * k + 1024) / 4) B <<= 1;
  if (frac >= 0.25 || B > kMaxBuckets) {  // small n / huge k: signal "use the full sort"
    cudaMemsetAsync(bad, 0xff, sizeof(int), st);
    return cudaGetLastError();
  }
  const uint64_t thr = (uint64_t)(frac * 18446744073709551616.0);
  const uint64_t w = thr / (uint64_t)B + 1;
  char *buf = nullptr;
  const size_t bytes = (size_t)cap * 12 + (size_t)(3 * B + 2) * 4 + 16;
  cudaError_t e;
  if ((e = cudaMallocAsync(&buf, bytes, st))) return e;
  uint64_t *ck = reinterpret_cast<uint64_t *>(buf);
  int32_t *ci = reinterpret_cast<int32_t *>(ck + cap);
  int *cnt = ci + cap, *start = cnt + B, *cursor = start + B + 1, *total = cursor + B;
  cudaMemsetAsync(cnt, 0, (size_t)B * 4, st);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_anc_count<<<grid, 256, 0, st>>>(n, seed, thr, w, cnt);
  k_anc_scan<<<1, kScanThreads, 0, st>>>(cnt, B, start, cursor, total);
  k_anchor_check<<<1, 32, 0, st>>>(total, cap, k, bad);
  k_anc_scatter<<<grid, 256, 0, st>>>(n, seed, thr, w, cap, cursor, ck, ci);
  k_anc_finish<<<(B + 255) / 256, 256, 0, st>>>(start, B, cap, k, ck, ci, anchors);
  cudaFreeAsync(buf, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ H3
// Squared scaled distance, the fma chain of DESIGN.md Q14.
template <int DM>
__device__ __forceinline__ double dist2_reg(const double (&a)[DM], const double *b, int d) {
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < DM; j++) {
    if (j < d) {
      double t = a[j] - b[j];
      acc = __fma_rn(t, t, acc);
    }
  }
  return acc;
}

constexpr int kRacTile = 128;

// Brute-force Random Anchor Clustering (Alg.3 line 5): each
// thread owns one point, anchors stream through shared memory; strict '<'
// over ascending anchor rank keeps the lowest rank on ties.
template <int DM>
__global__ void __launch_bounds__(256) k_rac(const double *__restrict__ S, int64_t n, int d,
                                             const int32_t *__restrict__ anchors, int64_t k,
                                             int32_t *__restrict__ block_of) {
  extern __shared__ double tile[];  // kRacTile x d
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double p[DM];
#pragma unroll
  for (int j = 0; j < DM; j++) p[j] = (i < n && j < d) ? S[i * d + j] : 0.0;
  double best = INFINITY;
  int32_t arg = -1;
  for (int64_t r0 = 0; r0 < k; r0 += kRacTile) {
    int cnt = (int)((k - r0) < kRacTile ? (k - r0) : kRacTile);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * d; e += blockDim.x) {
      int a = e / d, j = e - a * d;
      tile[e] = S[(int64_t)anchors[r0 + a] * d + j];
    }
    __syncthreads();
    for (int a = 0; a < cnt; a++) {
      double d2 = dist2_reg<DM>(p, tile + a * d, d);
      if (d2 < best) {
        best = d2;
        arg = (int32_t)(r0 + a);
      }
    }
  }
  if (i < n) block_of[i] = arg;
}

__global__ void k_anchor_own_block(const int32_t *anchors, int64_t k, int32_t *block_of) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < k;
       r += (int64_t)gridDim.x * blockDim.x)
    block_of[anchors[r]] = (int32_t)r;  // an anchor belongs to its own block
}

cudaError_t anchor_own_block(const int32_t *anchors, int64_t k, int32_t *block_of, cudaStream_t st) {
  k_anchor_own_block<<<(int)((k + 255) / 256), 256, 0, st>>>(anchors, k, block_of);
  return cudaGetLastError();
}

cudaError_t launch_rac(const double *S, int64_t n, int d, const int32_t *anchors, int64_t k,
                       int32_t *block_of, cudaStream_t st) {
  int grid = (int)((n + 255) / 256);
  size_t smem = (size_t)kRacTile * d * sizeof(double);
  if (d <= 4)
    k_rac<4><<<grid, 256, smem, st>>>(S, n, d, anchors, k, block_of);
  else if (d <= 8)
    k_rac<8><<<grid, 256, smem, st>>>(S, n, d, anchors, k, block_of);
  else if (d <= 16)
    k_rac<16><<<grid, 256, smem, st>>>(S, n, d, anchors, k, block_of);
  else if (d <= 32)
    k_rac<32><<<grid, 256, smem, st>>>(S, n, d, anchors, k, block_of);
  else {
    cudaFuncSetAttribute(k_rac<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_rac<64><<<grid, 256, smem, st>>>(S, n, d, anchors, k, block_of);
  }
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  k_anchor_own_block<<<(int)((k + 255) / 256), 256, 0, st>>>(anchors, k, block_of);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ H4
__global__ void k_iota(int64_t n, int32_t *v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// off[b] = first sorted position with block id >= b, for every b in [0, k]
// (empty blocks, possible with a caller-given partition, get off[b] = off[b+1])
__global__ void k_offsets(const int32_t *sorted_block, int64_t n, int64_t k, int64_t *off) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = sorted_block[p];
    const int32_t prev = p == 0 ? -1 : sorted_block[p - 1];
    for (int32_t c = prev + 1; c <= b; c++) off[c] = p;
    if (p == n - 1)
      for (int64_t c = (int64_t)b + 1; c <= k; c++) off[c] = n;
  }
}

// Block-major layout: a stable radix sort of (block id -> original index)
// keeps members in ascending original index (Q13).
cudaError_t build_layout(const int32_t *block_of, int64_t n, int64_t k, int32_t *perm,
                         int64_t *off, void *, size_t, cudaStream_t st, size_t *) {
  int32_t *kout = nullptr, *vin = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  int bits = 1;
  while ((int64_t(1) << bits) < k) bits++;
  if ((e = cudaMallocAsync(&kout, n * 4, st))) return e;
  if ((e = cudaMallocAsync(&vin, n * 4, st))) return e;
  int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_iota<<<grid, 256, 0, st>>>(n, vin);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, block_of, kout, vin, perm, (int)n, 0, bits,
                                  st);
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return e;
  e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, block_of, kout, vin, perm, (int)n, 0, bits,
                                      st);
  if (e) return e;
  k_offsets<<<grid, 256, 0, st>>>(kout, n, k, off);
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(kout, st);
  cudaFreeAsync(vin, st);
  return cudaGetLastError();
}

__global__ void k_gather_rows(const double *__restrict__ S, const int32_t *__restrict__ perm,
                              int64_t n, int d, double *__restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = e / d;
    int j = (int)(e - p * d);
    out[e] = S[(int64_t)perm[p] * d + j];
  }
}

cudaError_t launch_gather_rows(const double *S, const int32_t *perm, int64_t n, int d,
                               double *Sperm, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n * d + 255) / 256, 148 * 16);
  k_gather_rows<<<grid, 256, 0, st>>>(S, perm, n, d, Sperm);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ H5
// Alg.4 line 6: c_t = (sum of members, ascending index) / |B_t|.
// Only the blocks listed in `blocks` (this rank's queries; all blocks when
// null); C stays indexed by the global zeta id.
// One warp per block: the block's rows (contiguous in the block-major layout)
// are staged through shared memory with coalesced loads, then lane j sums
// coordinate j in member order (the sequential sum of Q4).
constexpr int kCenWarps = 4, kCenTile = 1024;  // doubles staged per warp
__global__ void __launch_bounds__(32 * kCenWarps)
    k_centroids(const double *__restrict__ Sperm, const int64_t *__restrict__ off,
                const int32_t *__restrict__ blocks, int64_t k, int d, double *__restrict__ C) {
  __shared__ double tile[kCenWarps][kCenTile];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rows_per_tile = kCenTile / d;
  for (int64_t i = blockIdx.x * (int64_t)kCenWarps + w; i < k; i += (int64_t)gridDim.x * kCenWarps) {
    const int64_t t = blocks ? blocks[i] : i;
    const int64_t p0 = off[t], p1 = off[t + 1];
    double s0 = 0.0, s1 = 0.0;  // coordinates lane and lane + 32 (d <= 64)
    for (int64_t r0 = p0; r0 < p1; r0 += rows_per_tile) {
      const int rows = p1 - r0 < rows_per_tile ? (int)(p1 - r0) : rows_per_tile;
      const double *src = Sperm + r0 * d;
      for (int e = lane; e < rows * d; e += 32) tile[w][e] = src[e];
      __syncwarp();
      if (lane < d)
        for (int r = 0; r < rows; r++) s0 = __dadd_rn(s0, tile[w][r * d + lane]);
      if (lane + 32 < d)
        for (int r = 0; r < rows; r++) s1 = __dadd_rn(s1, tile[w][r * d + lane + 32]);
      __syncwarp();
    }
    const double cntd = (double)(p1 - p0);
    if (lane < d) C[t * d + lane] = __ddiv_rn(s0, cntd);
    if (lane + 32 < d) C[t * d + lane + 32] = __ddiv_rn(s1, cntd);
  }
}

cudaError_t launch_centroids(const double *Sperm, const int64_t *off, const int32_t *blocks,
                             int64_t k, int d, double *C, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  int grid = (int)std::min<int64_t>((k + kCenWarps - 1) / kCenWarps, 148 * 16);
  k_centroids<<<grid, 32 * kCenWarps, 0, st>>>(Sperm, off, blocks, k, d, C);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ H6
// Exact m-NN of the block centroid among all points of strictly earlier
// blocks (Eq.2; Alg.4 P:415-427 with Q5/Q6): in the block-major
// layout those points are exactly the prefix [0, off_t).  Key = (dist2,
// original index), lexicographic.  One CTA per query block keeps a
// threshold-filtered candidate buffer in shared memory: a candidate enters
// only if its key is below the current m-th best; when the buffer fills it
// is bitonic-sorted and truncated to m.
constexpr int kKnnCap = 2048;
constexpr int kKnnThreads = 256;

struct Cand {
  double d2;
  int32_t orig;
  int32_t pos;
};

__device__ __forceinline__ bool cand_less(double da, int32_t ia, double db, int32_t ib) {
  return da < db || (da == db && ia < ib);
}

// Bitonic sort of buf[0, cnt) (padded with +inf sentinels to a power of two).
__device__ void bitonic_sort(Cand *buf, int cnt) {
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = cnt + threadIdx.x; i < P; i += blockDim.x) {
    buf[i].d2 = INFINITY;
    buf[i].orig = INT32_MAX;
    buf[i].pos = -1;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        int lo = 2 * stride * (i / stride) + (i % stride);
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        Cand a = buf[lo], b = buf[hi];
        bool gt = cand_less(b.d2, b.orig, a.d2, a.orig);
        if (gt == up) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

template <int DM>
__global__ void __launch_bounds__(kKnnThreads) k_knn(const double *__restrict__ Sperm,
                                                     const int32_t *__restrict__ perm,
                                                     const int64_t *__restrict__ off,
                                                     const double *__restrict__ C,
                                                     const int32_t *__restrict__ local_blocks,
                                                     int d, int m, int32_t *__restrict__ nbr,
                                                     int32_t *__restrict__ cnt_out) {
  __shared__ Cand buf[kKnnCap];
  __shared__ int count;
  __shared__ double thr_d;
  __shared__ int32_t thr_i;
  const int64_t li = blockIdx.x;
  const int64_t t = local_blocks[li];
  const int64_t A = off[t];
  double c[DM];
#pragma unroll
  for (int j = 0; j < DM; j++) c[j] = j < d ? C[t * d + j] : 0.0;
  if (threadIdx.x == 0) {
    count = 0;
    thr_d = INFINITY;
    thr_i = INT32_MAX;
  }
  __syncthreads();
  for (int64_t base = 0; base < A; base += blockDim.x) {
    int64_t p = base + threadIdx.x;
    if (p < A) {
      double acc = 0.0;
      const double *s = Sperm + p * d;
#pragma unroll
      for (int j = 0; j < DM; j++) {
        if (j < d) {
          double tt = c[j] - s[j];
          acc = __fma_rn(tt, tt, acc);
        }
      }
      int32_t o = perm[p];
      if (cand_less(acc, o, *(volatile double *)&thr_d, *(volatile int32_t *)&thr_i)) {
        int slot = atomicAdd(&count, 1);
        buf[slot].d2 = acc;
        buf[slot].orig = o;
        buf[slot].pos = (int32_t)p;
      }
    }
    __syncthreads();
    const int cnow = *(volatile int *)&count;
    __syncthreads();  // every thread has read count before thread 0 may reset it
    if (cnow > kKnnCap - (int)blockDim.x) {
      const int cnum = cnow;
      bitonic_sort(buf, cnum);
      if (threadIdx.x == 0) {
        count = min(cnum, m);
        if (count == m) {
          thr_d = buf[m - 1].d2;
          thr_i = buf[m - 1].orig;
        }
      }
      __syncthreads();
    }
  }
  const int cnum = *(volatile int *)&count;
  __syncthreads();
  bitonic_sort(buf, cnum);
  int keep = min(cnum, m); if ((int64_t)keep > A) keep = (int)A;
  for (int j = threadIdx.x; j < m; j += blockDim.x)
    nbr[li * m + j] = j < keep ? buf[j].pos : -1;
  if (threadIdx.x == 0) cnt_out[li] = keep;
}

cudaError_t launch_knn(const double *Sperm, const int32_t *perm, const int64_t *off,
                       const double *C, const int32_t *local_blocks, int64_t k_local, int d,
                       int m, int32_t *nbr, int32_t *cnt, cudaStream_t st) {
  if (k_local == 0) return cudaSuccess;
  if (m == 0) return cudaMemsetAsync(cnt, 0, k_local * 4, st);
  dim3 grid((unsigned)k_local);
  if (d <= 4)
    k_knn<4><<<grid, kKnnThreads, 0, st>>>(Sperm, perm, off, C, local_blocks, d, m, nbr, cnt);
  else if (d <= 8)
    k_knn<8><<<grid, kKnnThreads, 0, st>>>(Sperm, perm, off, C, local_blocks, d, m, nbr, cnt);
  else if (d <= 16)
    k_knn<16><<<grid, kKnnThreads, 0, st>>>(Sperm, perm, off, C, local_blocks, d, m, nbr, cnt);
  else if (d <= 32)
    k_knn<32><<<grid, kKnnThreads, 0, st>>>(Sperm, perm, off, C, local_blocks, d, m, nbr, cnt);
  else
    k_knn<64><<<grid, kKnnThreads, 0, st>>>(Sperm, perm, off, C, local_blocks, d, m, nbr, cnt);
  return cudaGetLastError();
}

}  // namespace sbv
