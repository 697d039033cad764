// grid.cu — exact grid-filtered nearest-anchor (RAC, H3) and m-NN (H6) search.
//
// The paper filters m-NN candidates with a Monte-Carlo radius lambda (Eq.7,
// Alg.4) so that the search stays exact while touching O(alpha m)
// points instead of O(n).  On the GPU the same idea takes the
// form of a uniform grid over the G <= 3 scaled dimensions of largest extent:
// cells are visited in rings of growing Chebyshev radius, every cell whose
// lower-bound distance exceeds the current best (the nearest anchor, or the
// m-th best neighbour) is skipped, and the search stops once the next ring's
// lower bound exceeds it.  Candidates that survive are scored with the same
// fma chain as the brute-force kernels (Q14) and ties are broken by
// anchor rank / original index (Q8, Q13), so the result is bit-identical to
// the exhaustive search; bounds carry a relative safety margin so rounding can
// never prune a true candidate.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/cub.cuh>

#include "sbv_internal.cuh"

namespace sbv {

// ------------------------------------------------------------------ extents
__global__ void k_minmax_partial(const double *__restrict__ S, int64_t n, int d, double *part) {
  __shared__ double smin[SBV_MAX_D][32], smax[SBV_MAX_D][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = 0; j < d; j++) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      const double v = S[i * d + j];
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      smin[j][w] = lo;
      smax[j][w] = hi;
    }
  }
  __syncthreads();
  if (threadIdx.x < d) {
    const int j = threadIdx.x;
    double lo = INFINITY, hi = -INFINITY;
    for (int x = 0; x < (int)(blockDim.x >> 5); x++) {
      lo = fmin(lo, smin[j][x]);
      hi = fmax(hi, smax[j][x]);
    }
    part[(blockIdx.x * d + j) * 2] = lo;
    part[(blockIdx.x * d + j) * 2 + 1] = hi;
  }
}

// one pass over the rows (thread = row, coordinates in registers), then a
// per-dimension warp / CTA reduction; d <= 16
template <int DM>
__global__ void __launch_bounds__(512) k_minmax_rows(const double *__restrict__ S, int64_t n, int d,
                                                     double *part) {
  __shared__ double smin[16][32], smax[16][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double lo[DM], hi[DM];
#pragma unroll
  for (int j = 0; j < DM; j++) {
    lo[j] = INFINITY;
    hi[j] = -INFINITY;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int j = 0; j < DM; j++)
      if (j < d) {
        const double v = S[i * d + j];
        lo[j] = fmin(lo[j], v);
        hi[j] = fmax(hi[j], v);
      }
  }
#pragma unroll
  for (int j = 0; j < DM; j++) {
    double a = lo[j], b = hi[j];
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      smin[j][w] = a;
      smax[j][w] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < d) {
    const int j = threadIdx.x;
    double a = INFINITY, b = -INFINITY;
    for (int x = 0; x < (int)(blockDim.x >> 5); x++) {
      a = fmin(a, smin[j][x]);
      b = fmax(b, smax[j][x]);
    }
    part[(blockIdx.x * d + j) * 2] = a;
    part[(blockIdx.x * d + j) * 2 + 1] = b;
  }
}

cudaError_t data_extents(const double *S, int64_t n, int d, double *lo_hi_host, cudaStream_t st) {
  const int nb = 148;
  double *part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * nb * d * 2, st);
  if (e) return e;
  if (d <= 4)
    k_minmax_rows<4><<<nb, 512, 0, st>>>(S, n, d, part);
  else if (d <= 8)
    k_minmax_rows<8><<<nb, 512, 0, st>>>(S, n, d, part);
  else if (d <= 16)
    k_minmax_rows<16><<<nb, 512, 0, st>>>(S, n, d, part);
  else
    k_minmax_partial<<<nb, 1024, 0, st>>>(S, n, d, part);
  std::vector<double> h(nb * d * 2);
  e = cudaMemcpyAsync(h.data(), part, sizeof(double) * nb * d * 2, cudaMemcpyDeviceToHost, st);
  if (e) return e;
  e = cudaStreamSynchronize(st);
  cudaFreeAsync(part, st);
  if (e) return e;
  for (int j = 0; j < d; j++) {
    double lo = INFINITY, hi = -INFINITY;
    for (int b = 0; b < nb; b++) {
      lo = std::min(lo, h[(b * d + j) * 2]);
      hi = std::max(hi, h[(b * d + j) * 2 + 1]);
    }
    lo_hi_host[2 * j] = lo;
    lo_hi_host[2 * j + 1] = hi;
  }
  return cudaSuccess;
}

// Grid over the G <= 3 dimensions of largest extent, about `per_cell` items
// per cell on average for `count` items.
GridDesc make_grid(const double *lo_hi, int d, int64_t count, double per_cell) {
  GridDesc g{};
  int order[SBV_MAX_D];
  for (int j = 0; j < d; j++) order[j] = j;
  std::sort(order, order + d, [&](int a, int b) {
    const double ea = lo_hi[2 * a + 1] - lo_hi[2 * a], eb = lo_hi[2 * b + 1] - lo_hi[2 * b];
    return ea > eb || (ea == eb && a < b);
  });
  g.G = std::min(3, d);
  // drop trailing dimensions whose extent is negligible next to the first one
  const double e0 = lo_hi[2 * order[0] + 1] - lo_hi[2 * order[0]];
  while (g.G > 1 && (lo_hi[2 * order[g.G - 1] + 1] - lo_hi[2 * order[g.G - 1]]) < 0.05 * e0) g.G--;
  double vol = 1.0;
  for (int x = 0; x < g.G; x++) {
    g.dim[x] = order[x];
    g.lo[x] = lo_hi[2 * order[x]];
    const double ext = lo_hi[2 * order[x] + 1] - g.lo[x];
    vol *= std::max(ext, 1e-300);
  }
  const double cells_wanted = std::max(1.0, std::min((double)count / per_cell, 4.0e6));
  double h = std::pow(vol / cells_wanted, 1.0 / g.G);
  if (!(h > 0) || !std::isfinite(h)) h = 1.0;
  int64_t total = 1;
  for (int x = 0; x < g.G; x++) {
    const double ext = lo_hi[2 * g.dim[x] + 1] - g.lo[x];
    g.h[x] = h;
    g.nc[x] = (int)std::max<double>(1.0, std::min(std::ceil(ext / h) + (ext == 0 ? 1.0 : 0.0), (double)(1 << 20)));
    g.stride[x] = (int)total;
    total *= g.nc[x];
  }
  g.ncells = total;
  return g;
}

__device__ __forceinline__ int cell_coord(double v, double lo, double h, int nc) {
  const int c = (int)floor((v - lo) / h);
  return min(max(c, 0), nc - 1);
}

__global__ void k_cell_ids(const double *__restrict__ S, const int32_t *__restrict__ rows,
                           int64_t count, int d, GridDesc g, int32_t *__restrict__ cell,
                           int32_t *__restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = rows ? rows[i] : i;
    int c = 0;
    for (int x = 0; x < g.G; x++)
      c += cell_coord(S[row * d + g.dim[x]], g.lo[x], g.h[x], g.nc[x]) * g.stride[x];
    cell[i] = c;
    idx[i] = (int32_t)i;
  }
}

// start[c] = first sorted position whose cell >= c (empty cells share starts)
__global__ void k_cell_starts(const int32_t *__restrict__ sorted_cell, int64_t count, int64_t ncells,
                              int32_t *__restrict__ start) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= count;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = p == 0 ? -1 : sorted_cell[p - 1];
    const int64_t b = p == count ? ncells : sorted_cell[p];
    for (int64_t c = a + 1; c <= b; c++) start[c] = (int32_t)p;
  }
}

// Bucket `count` items (rows of S, optionally through `rows`) into the grid:
// list = item indices sorted by (cell, index), start = ncells + 1 offsets.
cudaError_t build_cells(const double *S, const int32_t *rows, int64_t count, int d, const GridDesc &g,
                        int32_t *start, int32_t *list, cudaStream_t st) {
  int32_t *cell = nullptr, *cell_sorted = nullptr, *idx = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  if ((e = cudaMallocAsync(&cell, count * 4, st))) return e;
  if ((e = cudaMallocAsync(&cell_sorted, count * 4, st))) return e;
  if ((e = cudaMallocAsync(&idx, count * 4, st))) return e;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 16));
  k_cell_ids<<<grid, 256, 0, st>>>(S, rows, count, d, g, cell, idx);
  int bits = 1;
  while ((int64_t(1) << bits) < g.ncells) bits++;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, cell, cell_sorted, idx, list, (int)count, 0,
                                  bits, st);
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return e;
  if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, cell, cell_sorted, idx, list, (int)count, 0,
                                           bits, st)))
    return e;
  const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>((count + 256) / 256, 148 * 16));
  k_cell_starts<<<grid2, 256, 0, st>>>(cell_sorted, count, g.ncells, start);
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(cell, st);
  cudaFreeAsync(cell_sorted, st);
  cudaFreeAsync(idx, st);
  return cudaGetLastError();
}

KnnLevels make_knn_levels(const double *lo_hi, int d, int64_t n, int m) {
  KnnLevels lv{};
  const double per_cell = std::max(8.0, m / 8.0);
  // a direct scan of a short prefix beats the ring search of a grid with a
  // handful of cells around m neighbours
  lv.direct_max = (int32_t)std::min<int64_t>(n, std::max(2048, 16 * m));
  int64_t P = n;
  lv.nl = 0;
  int64_t cells = 0, items = 0;
  while (lv.nl < kMaxLevels) {
    const int l = lv.nl++;
    lv.P[l] = (int32_t)P;
    lv.g[l] = make_grid(lo_hi, d, P, per_cell);
    lv.cell_off[l] = cells;
    lv.list_off[l] = items;
    cells += lv.g[l].ncells;
    items += P;
    // one level while 2n items do not fit the int32 sort
    if (2 * n >= (int64_t(1) << 31) || (P + 1) / 2 < lv.direct_max) break;
    P = (P + 1) / 2;
  }
  lv.cell_off[lv.nl] = cells;
  lv.list_off[lv.nl] = items;
  return lv;
}

__global__ void k_cell_ids_levels(const double *__restrict__ S, int d, KnnLevels lv,
                                  int32_t *__restrict__ cell, int32_t *__restrict__ idx) {
  const int64_t total = lv.list_off[lv.nl];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < lv.nl && e >= lv.list_off[l + 1]) l++;
    const int64_t i = e - lv.list_off[l];
    const GridDesc &g = lv.g[l];
    int64_t c = lv.cell_off[l];
    for (int x = 0; x < g.G; x++)
      c += cell_coord(S[i * d + g.dim[x]], g.lo[x], g.h[x], g.nc[x]) * (int64_t)g.stride[x];
    cell[e] = (int32_t)c;
    idx[e] = (int32_t)i;
  }
}

// All levels bucketed by one radix sort: key = global cell id (level cells
// are consecutive), value = position; the sort is stable, so each cell lists
// its positions ascending.
cudaError_t build_knn_levels(const double *Sperm, int d, const KnnLevels &lv, int32_t *start,
                             int32_t *list, cudaStream_t st) {
  const int64_t count = lv.list_off[lv.nl], ncells = lv.cell_off[lv.nl];
  int32_t *cell = nullptr, *cell_sorted = nullptr, *idx = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  if ((e = cudaMallocAsync(&cell, count * 4, st))) return e;
  if ((e = cudaMallocAsync(&cell_sorted, count * 4, st))) return e;
  if ((e = cudaMallocAsync(&idx, count * 4, st))) return e;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 16));
  k_cell_ids_levels<<<grid, 256, 0, st>>>(Sperm, d, lv, cell, idx);
  int bits = 1;
  while ((int64_t(1) << bits) < ncells) bits++;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, cell, cell_sorted, idx, list, (int)count, 0,
                                  bits, st);
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return e;
  if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, cell, cell_sorted, idx, list, (int)count, 0,
                                           bits, st)))
    return e;
  const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>((count + 256) / 256, 148 * 16));
  k_cell_starts<<<grid2, 256, 0, st>>>(cell_sorted, count, ncells, start);
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(cell, st);
  cudaFreeAsync(cell_sorted, st);
  cudaFreeAsync(idx, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ ring search helpers
struct RingQ {
  double x[3];  // query coordinates in the grid dims
  int cq[3];    // query cell coords
};

__device__ __forceinline__ double cell_lb2(const GridDesc &g, const RingQ &q, const int (&cc)[3]) {
  double s = 0.0;
  for (int x = 0; x < g.G; x++) {
    const double slack = 1e-9 * g.h[x];
    const double clo = g.lo[x] + cc[x] * g.h[x] - slack, chi = g.lo[x] + (cc[x] + 1) * g.h[x] + slack;
    double gap = 0.0;
    if (cc[x] > 0 && q.x[x] < clo) gap = clo - q.x[x];
    if (cc[x] < g.nc[x] - 1 && q.x[x] > chi) gap = q.x[x] - chi;
    s = fma(gap, gap, s);
  }
  return s;
}

// squared lower bound of every cell outside the ring block of radius r; returns
// -1 when the block already covers the whole grid
__device__ __forceinline__ double ring_lb2(const GridDesc &g, const RingQ &q, int r) {
  double best = INFINITY;
  bool any = false;
  for (int x = 0; x < g.G; x++) {
    const double slack = 1e-9 * g.h[x];
    if (q.cq[x] - r > 0) {
      any = true;
      best = fmin(best, fmax(0.0, q.x[x] - (g.lo[x] + (q.cq[x] - r) * g.h[x]) - slack));
    }
    if (q.cq[x] + r < g.nc[x] - 1) {
      any = true;
      best = fmin(best, fmax(0.0, (g.lo[x] + (q.cq[x] + r + 1) * g.h[x]) - q.x[x] - slack));
    }
  }
  return any ? best * best : -1.0;
}

// prune test: can a cell / ring with squared lower bound lb2 still hold a key
// not larger than `thr` (the current best)?  Margin absorbs rounding.
__device__ __forceinline__ bool may_hold(double lb2, double thr) {
  return !(lb2 > thr * (1.0 + 1e-10) + 1e-300);
}

// visit cells with Chebyshev distance exactly r (clipped to the grid); f(cell_index, lb2)
template <class F>
__device__ __forceinline__ void for_ring(const GridDesc &g, const RingQ &q, int r, F &&f) {
  const int G = g.G;
  const int r1 = G > 1 ? r : 0, r2 = G > 2 ? r : 0;
  for (int o2 = -r2; o2 <= r2; o2++) {
    const int c2 = G > 2 ? q.cq[2] + o2 : 0;
    if (G > 2 && (c2 < 0 || c2 >= g.nc[2])) continue;
    for (int o1 = -r1; o1 <= r1; o1++) {
      const int c1 = G > 1 ? q.cq[1] + o1 : 0;
      if (G > 1 && (c1 < 0 || c1 >= g.nc[1])) continue;
      const bool edge = (abs(o1) == r) || (abs(o2) == r);
      const int step = edge ? 1 : 2 * r;  // interior rows: only the two ends of dim 0
      for (int o0 = -r; o0 <= r; o0 += (step == 0 ? 1 : step)) {
        const int c0 = q.cq[0] + o0;
        if (c0 < 0 || c0 >= g.nc[0]) continue;
        const int cc[3] = {c0, c1, c2};
        const int idx = c0 * g.stride[0] + (G > 1 ? c1 * g.stride[1] : 0) + (G > 2 ? c2 * g.stride[2] : 0);
        f(idx, cell_lb2(g, q, cc));
      }
    }
  }
}

// ------------------------------------------------------------------ H3 RAC
#ifndef SBV_RAC_SORT_MIN
#define SBV_RAC_SORT_MIN 0  // visit points in cell order when the slice has at least this many
#endif
// Anchor rows gathered in cell order (AC) with their ranks, so a cell's
// candidates are consecutive rows: no indirection through `anchors`.
__global__ void k_gather_anchor_rows(const double *__restrict__ S, const int32_t *__restrict__ anchors,
                                     const int32_t *__restrict__ a_list, int64_t k, int d,
                                     double *__restrict__ AC, int32_t *__restrict__ arank) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int j = (int)(e - r * d);
    const int32_t rank = a_list[r];
    AC[e] = S[(int64_t)anchors[rank] * d + j];
    if (j == 0) arank[r] = rank;
  }
}

// Points are visited in anchor-grid cell order (`order`, relative to i0), so
// the lanes of a warp search the same cells and read the same anchor rows.
#ifndef SBV_RAC_MINB
#define SBV_RAC_MINB 4  // CTAs per SM the RAC kernel's registers are bounded for (measured at cfg2: 1 / 3 / 4 -> 0.43 / 0.37 / 0.35 ms)
#endif
template <int DM>
__global__ void __launch_bounds__(256, SBV_RAC_MINB) k_rac_grid2(const double *__restrict__ S, const int32_t *__restrict__ order,
                                                   int64_t count, int64_t i0, int d,
                                                   const double *__restrict__ AC,
                                                   const int32_t *__restrict__ arank, GridDesc g,
                                                   const int32_t *__restrict__ a_start,
                                                   int32_t *__restrict__ block_of) {
  const int64_t tt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tt >= count) return;
  const int64_t il = order ? order[tt] : tt, i = i0 + il;
  double p[DM];
#pragma unroll
  for (int j = 0; j < DM; j++) p[j] = j < d ? S[i * d + j] : 0.0;
  RingQ q;
  for (int x = 0; x < 3; x++) {
    q.x[x] = x < g.G ? S[i * d + g.dim[x]] : 0.0;
    q.cq[x] = x < g.G ? cell_coord(q.x[x], g.lo[x], g.h[x], g.nc[x]) : 0;
  }
  double best = INFINITY;
  int32_t arg = INT32_MAX;
  for (int r = 0;; r++) {
    for_ring(g, q, r, [&](int cell, double lb2) {
      if (!may_hold(lb2, best)) return;
      for (int e = a_start[cell]; e < a_start[cell + 1]; e++) {
        const int32_t rank = arank[e];
        const double *s = AC + (int64_t)e * d;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < DM; j++)
          if (j < d) {
            const double t = p[j] - s[j];
            acc = __fma_rn(t, t, acc);
          }
        if (acc < best || (acc == best && rank < arg)) {  // Alg.3 argmin, ties -> lowest rank
          best = acc;
          arg = rank;
        }
      }
    });
    const double lb = ring_lb2(g, q, r);
    if (lb < 0.0) break;
    if (arg != INT32_MAX && !may_hold(lb, best)) break;
  }
  block_of[il] = arg;
}

cudaError_t launch_rac_grid(const double *S, int64_t n, int64_t i0, int d, const int32_t *anchors, int64_t k,
                            const GridDesc &g, const int32_t *a_start, const int32_t *a_list,
                            int32_t *block_of, cudaStream_t st) {
  if (n <= i0) return cudaSuccess;
  const int64_t count = n - i0;
  // scratch: anchor rows in cell order + ranks, the slice's points sorted by cell
  double *AC = nullptr;
  int32_t *arank = nullptr, *order = nullptr, *pstart = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync(&AC, sizeof(double) * k * d, st))) return e;
  if ((e = cudaMallocAsync(&arank, sizeof(int32_t) * k, st))) return e;
  if ((e = cudaMallocAsync(&order, sizeof(int32_t) * count, st))) return e;
  if ((e = cudaMallocAsync(&pstart, sizeof(int32_t) * (g.ncells + 1), st))) return e;
  k_gather_anchor_rows<<<(int)std::max<int64_t>(1, std::min<int64_t>((k * d + 255) / 256, 148 * 16)), 256, 0, st>>>(
      S, anchors, a_list, k, d, AC, arank);
  const bool sorted = count >= SBV_RAC_SORT_MIN;
  if (sorted && (e = build_cells(S + i0 * d, nullptr, count, d, g, pstart, order, st))) return e;
  const int grid = (int)((count + 255) / 256);
#define SBV_RAC(DMv) \
  k_rac_grid2<DMv><<<grid, 256, 0, st>>>(S, sorted ? order : nullptr, count, i0, d, AC, arank, g, a_start, block_of)
  if (d <= 4)
    SBV_RAC(4);
  else if (d <= 8)
    SBV_RAC(8);
  else if (d <= 10)
    SBV_RAC(10);
  else if (d <= 12)
    SBV_RAC(12);
  else if (d <= 16)
    SBV_RAC(16);
  else if (d <= 32)
    SBV_RAC(32);
  else
    SBV_RAC(64);
#undef SBV_RAC
  cudaFreeAsync(AC, st);
  cudaFreeAsync(arank, st);
  cudaFreeAsync(order, st);
  cudaFreeAsync(pstart, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ H6 kNN
// One warp per query block t.  Candidates = points of the cells visited whose
// block-major position is < off_t (each cell lists positions ascending, so the
// admissible ones are a prefix).  Keys (dist2, original index) below the
// current m-th best are appended to a per-warp shared-memory buffer that is
// bitonic-sorted and cut to m whenever it fills.
#ifndef SBV_KNN_WCAP
#define SBV_KNN_WCAP 512  // per-warp candidate buffer (16 B entries): occupancy vs compactions
#endif
#ifndef SBV_KNN_MINCAP
#define SBV_KNN_MINCAP(m) ((m) + 192)  // headroom between compactions (cfg2: 512 entries, 1.2 -> 1.0 ms)
#endif
#ifndef SBV_KNN_SLACK
#define SBV_KNN_SLACK 0  // ring-end compaction once the buffer holds more than m + slack
#endif
#ifndef SBV_KNN_WARPS
#define SBV_KNN_WARPS 4
#endif
constexpr int kKnnWarps = SBV_KNN_WARPS;
// shared-query mode threshold: measured SLOWER at 2500 queries (4 GPUs, cfg2:
// 0.47 vs 0.24 ms — the per-ring barriers and looser per-warp thresholds cost
// more than the shorter chains gain), so it is off unless SBV_KNN_QW=4
constexpr int64_t kKnnSplitQueries = 0;
constexpr int kKnnWcap = 1024;

struct WCand {
  double d2;
  int32_t orig;
  int32_t pos;
};

__device__ __forceinline__ bool wless(double da, int32_t ia, double db, int32_t ib) {
  return da < db || (da == db && ia < ib);
}

// warp-level bitonic sort of buf[0, cnt) padded with sentinels to a power of two
__device__ void warp_bitonic(WCand *buf, int cnt, int lane) {
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = cnt + lane; i < P; i += 32) {
    buf[i].d2 = INFINITY;
    buf[i].orig = INT32_MAX;
    buf[i].pos = -1;
  }
  __syncwarp();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < P / 2; i += 32) {
        const int lo = 2 * stride * (i / stride) + (i % stride), hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const WCand a = buf[lo], b = buf[hi];
        if (wless(b.d2, b.orig, a.d2, a.orig) == up) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncwarp();
    }
  }
}

// Warp radix select: the m-th smallest key (d2, orig) among buf[0, cnt)
// (1 <= m <= cnt).  d2 >= 0, so its IEEE bits order like the values; eight
// 8-bit passes over d2 with a per-warp 256-bin shared histogram, then (only
// when several entries share that d2) four passes over orig.  ~1k
// instructions per call instead of a 512-entry bitonic sort.
__device__ __forceinline__ int hist_find(unsigned *hist, int lane, int &k) {
  // hist holds 256 counts; return the digit whose cumulative range holds the
  // k-th (1-based) item, and reduce k by the items in smaller digits
  unsigned c[8], s = 0;
#pragma unroll
  for (int x = 0; x < 8; x++) {
    c[x] = hist[lane * 8 + x];
    s += c[x];
  }
  unsigned incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const unsigned excl = incl - s;
  int digit = -1, below = 0;
  if ((unsigned)k > excl && (unsigned)k <= incl) {
    unsigned run = excl;
#pragma unroll
    for (int x = 0; x < 8; x++) {
      if (digit < 0 && (unsigned)k <= run + c[x]) {
        digit = lane * 8 + x;
        below = (int)run;
      }
      run += c[x];
    }
  }
  const unsigned owner = __ballot_sync(0xffffffffu, digit >= 0);
  const int src = __ffs(owner) - 1;
  digit = __shfl_sync(0xffffffffu, digit, src);
  below = __shfl_sync(0xffffffffu, below, src);
  k -= below;
  return digit;
}

__device__ void warp_select(const WCand *buf, int cnt, int m, int lane, unsigned *hist, double &thr_d,
                            int32_t &thr_i) {
  unsigned long long prefix = 0, pmask = 0;
  int k = m;
  for (int shift = 56; shift >= 0; shift -= 8) {
#pragma unroll
    for (int x = 0; x < 8; x++) hist[lane * 8 + x] = 0;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
      const unsigned long long u = (unsigned long long)__double_as_longlong(buf[i].d2);
      if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 255], 1u);
    }
    __syncwarp();
    const int digit = hist_find(hist, lane, k);
    __syncwarp();
    prefix |= (unsigned long long)digit << shift;
    pmask |= 255ull << shift;
  }
  thr_d = __longlong_as_double((long long)prefix);
  // k-th smallest orig among the entries whose d2 equals thr_d
  unsigned pre = 0, pm = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
    for (int x = 0; x < 8; x++) hist[lane * 8 + x] = 0;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
      const WCand e = buf[i];
      const unsigned o = (unsigned)e.orig;
      if (e.d2 == thr_d && (o & pm) == pre) atomicAdd(&hist[(o >> shift) & 255], 1u);
    }
    __syncwarp();
    const int digit = hist_find(hist, lane, k);
    __syncwarp();
    pre |= (unsigned)digit << shift;
    pm |= 255u << shift;
  }
  thr_i = (int32_t)pre;
}

// QW warps per query (QW = 1: one warp per query; QW = kKnnWarps: the CTA's
// warps split one query's candidates and meet at every ring end, for small
// query counts where a single wave of one-warp queries is latency-bound).
template <int DM, int QW>
#ifndef SBV_KNN_MINB
#define SBV_KNN_MINB 5  // min resident CTAs per SM asked of ptxas (register cap; measured at cfg2: 1 / 5 / 6 / 8 -> 0.65 / 0.56 / 0.60 / 0.66 ms)
#endif
__global__ void __launch_bounds__(32 * kKnnWarps, SBV_KNN_MINB) k_knn_grid(
    const double *__restrict__ Sperm, const int32_t *__restrict__ perm,
    const int64_t *__restrict__ off, const double *__restrict__ C,
    const int32_t *__restrict__ local_blocks, int64_t k_local, int d, int m, KnnLevels lv,
    const int32_t *__restrict__ c_start_all, const int32_t *__restrict__ c_list, int32_t *__restrict__ nbr,
    int32_t *__restrict__ cnt_out, int wcap, const double *__restrict__ Cq, int32_t A_all) {
  extern __shared__ WCand sbuf[];  // kKnnWarps x wcap, then kKnnWarps x 256 histogram bins
  unsigned *hist = reinterpret_cast<unsigned *>(sbuf + kKnnWarps * wcap) + (threadIdx.x >> 5) * 256;
  __shared__ double s_thr[2][kKnnWarps];  // QW > 1: per-warp m-th best at ring ends (by parity)
  __shared__ int s_cnt[kKnnWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int sub = w % QW;  // this warp's slice of the query
  const int64_t li = blockIdx.x * (int64_t)(kKnnWarps / QW) + w / QW;
  if (li >= k_local) return;  // QW > 1: one query per CTA, so the whole CTA returns
  WCand *buf = sbuf + w * wcap;
  // estimation: query = centroid of block t, admissible = strictly earlier
  // blocks [0, off_t); prediction (Cq): query = test centroid li, all n points
  const int64_t t = Cq ? li : local_blocks[li];
  const int32_t A = Cq ? A_all : (int32_t)off[t];  // admissible positions [0, A)
  const double *Crow = Cq ? Cq + li * d : C + t * d;
  // the smallest prefix level that indexes all of [0, A)
  GridDesc g = lv.g[0];
  int64_t coff = 0;
#pragma unroll
  for (int l = 1; l < kMaxLevels; l++)
    if (l < lv.nl && lv.P[l] >= A) {
      g = lv.g[l];
      coff = lv.cell_off[l];
    }
  const int32_t *__restrict__ c_start = c_start_all + coff;
  double c[DM];
#pragma unroll
  for (int j = 0; j < DM; j++) c[j] = j < d ? Crow[j] : 0.0;
  RingQ q;
  for (int x = 0; x < 3; x++) {
    q.x[x] = x < g.G ? Crow[g.dim[x]] : 0.0;
    q.cq[x] = x < g.G ? cell_coord(q.x[x], g.lo[x], g.h[x], g.nc[x]) : 0;
  }
  int count = 0;
  double thr_d = INFINITY;
  int32_t thr_i = INT32_MAX;
  double gthr = INFINITY;  // QW > 1: min over the query's warps of their m-th best (a valid bound)
  int seen = 0;  // admissible points seen (for the "fewer than m exist" exit)
  // keep the m smallest keys (unsorted) and set the threshold to the m-th
  auto compact = [&]() {
    __syncwarp();
    if (count > m) {
      warp_select(buf, count, m, lane, hist, thr_d, thr_i);
      int kept = 0;
      for (int base = 0; base < count; base += 32) {
        const int i = base + lane;
        WCand e;
        bool keep = false;
        if (i < count) {
          e = buf[i];
          keep = !wless(thr_d, thr_i, e.d2, e.orig);  // e <= threshold
        }
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        __syncwarp();  // every lane has read its entry before the chunk is overwritten
        if (keep) buf[kept + __popc(mk & ((1u << lane) - 1))] = e;
        kept += __popc(mk);
        __syncwarp();
      }
      count = kept;  // == m (keys are unique)
    } else if (count == m && thr_d == INFINITY) {
      warp_select(buf, count, m, lane, hist, thr_d, thr_i);  // the m-th = the largest
    }
    __syncwarp();
  };
  // Short prefixes (the first blocks in zeta order) are scanned directly: the
  // grid would have to sweep most of the domain to find m sparse neighbours.
  if (A > 0 && m > 0 && A <= lv.direct_max) {
    for (int base = sub * 32; base < A; base += 32 * QW) {
      const int32_t pos = base + lane;
      const bool adm = pos < A;
      double acc = INFINITY;
      int32_t o = INT32_MAX;
      if (adm) {
        const double *s = Sperm + (int64_t)pos * d;
        acc = 0.0;
#pragma unroll
        for (int j = 0; j < DM; j++)
          if (j < d) {
            const double tt = c[j] - s[j];
            acc = __fma_rn(tt, tt, acc);
          }
        o = perm[pos];
      }
      const bool ins = adm && wless(acc, o, thr_d, thr_i);
      const unsigned mask = __ballot_sync(0xffffffffu, ins);
      if (ins) {
        const int slot = count + __popc(mask & ((1u << lane) - 1));
        buf[slot].d2 = acc;
        buf[slot].orig = o;
        buf[slot].pos = pos;
      }
      count += __popc(mask);
      if (count > wcap - 32) compact();
    }
  } else if (A > 0 && m > 0) {
    const int G = g.G;
    for (int r = 0;; r++) {
      // The ring's cells are handled 32 at a time: each lane takes one cell of
      // the ring's bounding box, skips interior / out-of-grid / pruned cells,
      // and binary-searches its cell's admissible prefix (positions ascending,
      // admissible iff < A); the warp then scores the up-to-32 ranges as one
      // flattened list.  The per-cell global loads are issued in parallel
      // instead of one dependent chain per cell.
      const int side = 2 * r + 1;
      int64_t box = side;
      if (G > 1) box *= side;
      if (G > 2) box *= side;
      for (int64_t b0 = sub * 32; b0 < box; b0 += 32 * QW) {
        const int64_t bi = b0 + lane;
        int e_lo = 0, e_cnt = 0;
        if (bi < box) {
          const int o0 = (int)(bi % side) - r;
          const int o1 = G > 1 ? (int)((bi / side) % side) - r : 0;
          const int o2 = G > 2 ? (int)(bi / ((int64_t)side * side)) - r : 0;
          const int cc[3] = {q.cq[0] + o0, q.cq[1] + o1, q.cq[2] + o2};
          bool ok = max(abs(o0), max(abs(o1), abs(o2))) == r;
          for (int x = 0; x < G; x++) ok = ok && cc[x] >= 0 && cc[x] < g.nc[x];
          if (ok && may_hold(cell_lb2(g, q, cc), fmin(count >= m ? thr_d : INFINITY, gthr))) {
            const int cell = cc[0] * g.stride[0] + (G > 1 ? cc[1] * g.stride[1] : 0) +
                             (G > 2 ? cc[2] * g.stride[2] : 0);
            const int s0 = c_start[cell], s1 = c_start[cell + 1];
            int lo = s0, hi = s1;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              if (c_list[mid] < A)
                lo = mid + 1;
              else
                hi = mid;
            }
            e_lo = s0;
            e_cnt = lo - s0;
          }
        }
        int incl = e_cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int excl = incl - e_cnt;
        for (int f0 = 0; f0 < total; f0 += 32) {
          const int f = f0 + lane;
          int owner = 0;  // largest lane whose range starts at or before f
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int cand = owner + step;
            const int ex = __shfl_sync(0xffffffffu, excl, min(cand, 31));
            if (cand < 32 && ex <= f) owner = cand;
          }
          const int o_lo = __shfl_sync(0xffffffffu, e_lo, owner);
          const int o_ex = __shfl_sync(0xffffffffu, excl, owner);
          const bool adm = f < total;
          int32_t pos = INT32_MAX, o = INT32_MAX;
          double acc = INFINITY;
          if (adm) {
            pos = c_list[o_lo + (f - o_ex)];
            const double *s = Sperm + (int64_t)pos * d;
            acc = 0.0;
#pragma unroll
            for (int j = 0; j < DM; j++)
              if (j < d) {
                const double tt = c[j] - s[j];
                acc = __fma_rn(tt, tt, acc);
              }
            o = perm[pos];
          }
          const bool ins = adm && wless(acc, o, thr_d, thr_i) && !(acc > gthr);
          const unsigned mask = __ballot_sync(0xffffffffu, ins);
          if (ins) {
            const int slot = count + __popc(mask & ((1u << lane) - 1));
            buf[slot].d2 = acc;
            buf[slot].orig = o;
            buf[slot].pos = pos;
          }
          count += __popc(mask);
          if (count > wcap - 32) compact();
        }
      }
      const double lb = ring_lb2(g, q, r);
      if constexpr (QW == 1) {
        if (lb < 0.0) break;
        if (count >= m) {
          // compact when the threshold is unset or the buffer has grown past
          // m + slack; test termination against the current m-th best
          if (thr_d == INFINITY || count > m + SBV_KNN_SLACK) compact();
          if (!may_hold(lb, thr_d)) break;
        }
      } else {
        // the query's warps agree on termination: the m-th best of the union
        // is <= every warp's own m-th best, so their minimum bounds it
        if (count > m || (count == m && thr_d == INFINITY)) compact();
        if (lane == 0) s_thr[r & 1][w] = count >= m ? thr_d : INFINITY;
        __syncthreads();
        double gm = INFINITY;
#pragma unroll
        for (int x = 0; x < QW; x++) gm = fmin(gm, s_thr[r & 1][x]);
        gthr = gm;
        if (lb < 0.0) break;
        if (gthr != INFINITY && !may_hold(lb, gthr)) break;
      }
    }
  }
  if constexpr (QW > 1) {
    // merge the warps' candidates (each <= m after compaction) into warp 0's
    // view of the CTA buffer, then select / sort as a single warp
    compact();
    if (lane == 0) s_cnt[w] = count;
    __syncthreads();
    if (sub != 0) return;
    int total = 0;
    for (int x = 0; x < QW; x++) {
      const int cx = s_cnt[x];
      const WCand *src = sbuf + x * wcap;
      for (int base = 0; base < cx; base += 32) {  // forward copy, dst <= src
        WCand e;
        const bool has = base + lane < cx;
        if (has) e = src[base + lane];
        __syncwarp();
        if (has) sbuf[total + base + lane] = e;
        __syncwarp();
      }
      total += cx;
    }
    buf = sbuf;
    count = total;
    thr_d = INFINITY;
    thr_i = INT32_MAX;
  }
  compact();
  warp_bitonic(buf, count, lane);  // the final m (or fewer) in (d2, orig) order
  const int keep = min(count, min(m, A));
  for (int j = lane; j < m; j += 32) nbr[li * m + j] = j < keep ? buf[j].pos : -1;
  if (lane == 0) cnt_out[li] = keep;
  (void)seen;
}

cudaError_t launch_knn_grid(const double *Sperm, const int32_t *perm, const int64_t *off,
                            const double *C, const int32_t *local_blocks, int64_t k_local, int d,
                            int m, const KnnLevels &lv, const int32_t *c_start, const int32_t *c_list,
                            int32_t *nbr, int32_t *cnt, cudaStream_t st, const double *Cq, int32_t A_all) {
  if (k_local == 0) return cudaSuccess;
  if (m == 0) return cudaMemsetAsync(cnt, 0, k_local * 4, st);
  // few queries (a fraction of one wave of one-warp queries): the CTA's warps
  // share each query (SBV_KNN_QW overrides: 1 or 4)
  int qw = k_local <= kKnnSplitQueries ? kKnnWarps : 1;
  if (const char *e = getenv("SBV_KNN_QW")) qw = atoi(e) == kKnnWarps ? kKnnWarps : 1;
  const int qpc = kKnnWarps / qw;  // queries per CTA
  const int grid = (int)((k_local + qpc - 1) / qpc);
  const int thr = 32 * kKnnWarps;
  // per-warp candidate buffer: the smallest power of two >= m + 192 (headroom
  // between compactions) keeps shared memory low and occupancy high
  int wcap = SBV_KNN_WCAP;  // measured at cfg2: 256 / 512 / 1024 / 2048 -> 1.23 / 1.00 / 1.20 / 2.38 ms
  while (wcap < SBV_KNN_MINCAP(m)) wcap <<= 1;
  const int smem = (int)(sizeof(WCand) * kKnnWarps * wcap + sizeof(unsigned) * kKnnWarps * 256);
#define SBV_KNN(DMv)                                                                                    \
  do {                                                                                                  \
    if (qw == 1) {                                                                                      \
      cudaFuncSetAttribute(k_knn_grid<DMv, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);     \
      k_knn_grid<DMv, 1><<<grid, thr, smem, st>>>(Sperm, perm, off, C, local_blocks, k_local, d, m, lv, \
                                                  c_start, c_list, nbr, cnt, wcap, Cq, A_all);          \
    } else {                                                                                            \
      cudaFuncSetAttribute(k_knn_grid<DMv, kKnnWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                           smem);                                                                       \
      k_knn_grid<DMv, kKnnWarps><<<grid, thr, smem, st>>>(Sperm, perm, off, C, local_blocks, k_local,   \
                                                          d, m, lv, c_start, c_list, nbr, cnt, wcap,    \
                                                          Cq, A_all);                                   \
    }                                                                                                   \
  } while (0)
  if (d <= 4)
    SBV_KNN(4);
  else if (d <= 8)
    SBV_KNN(8);
  else if (d <= 10)
    SBV_KNN(10);
  else if (d <= 12)
    SBV_KNN(12);
  else if (d <= 16)
    SBV_KNN(16);
  else if (d <= 32)
    SBV_KNN(32);
  else
    SBV_KNN(64);
#undef SBV_KNN
  return cudaGetLastError();
}

int knn_grid_max_m() { return kKnnWcap - 64; }

}  // namespace sbv
