// sbv_api.cu — the extern "C" boundary of libsbv (include/sbv.h).
//
// Orchestrates the device steps of Alg.1: sbv_prepare_h runs
// Steps 1-3 (H1-H6, prep_kernels.cu) and sbv_loglik runs Steps 4-5 (H7-H10,
// llh_kernel.cu).  No host arithmetic of the method happens here: the host
// only validates arguments, sizes buffers, builds the block shard / work
// order from the device-computed layout, and launches.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <unordered_map>

#include "sbv_internal.cuh"

using namespace sbv;

struct sbv_ctx : public Ctx {};

namespace {

int fail(sbv_ctx *h, int code, const char *msg) {
  if (h) {
    h->err_msg = msg;
  }
  return code;
}

#define CU(call)                                                        \
  do {                                                                  \
    cudaError_t e__ = (call);                                           \
    if (e__ != cudaSuccess) {                                           \
      if (h) h->err_msg = std::string(#call) + ": " + cudaGetErrorString(e__); \
      return e__ == cudaErrorMemoryAllocation ? SBV_ERR_OOM : SBV_ERR_CUDA; \
    }                                                                   \
  } while (0)

#define NC(call)                                                        \
  do {                                                                  \
    ncclResult_t r__ = (call);                                          \
    if (r__ != ncclSuccess) {                                           \
      if (h) h->err_msg = std::string(#call) + ": " + ncclGetErrorString(r__); \
      return SBV_ERR_COMM;                                              \
    }                                                                   \
  } while (0)

bool is_device_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Capacity-tracked device buffers: re-prepare (e.g. an MLE rescale) reuses
// allocations, so steady-state prepare never calls cudaMalloc/cudaFree
// (both synchronise the device).
template <class T>
cudaError_t ensure(T *&p, size_t count, std::unordered_map<void *, size_t> &cap) {
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  auto it = cap.find((void *)&p);
  if (p && it != cap.end() && it->second >= bytes) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  cap[(void *)&p] = e == cudaSuccess ? bytes : 0;
  return e;
}

template <class T>
void release(T *&p) {
  if (p) cudaFree(p);
  p = nullptr;
}

void free_state(sbv_ctx *h) {
  release(h->X);
  release(h->S);
  release(h->Sperm);
  release(h->anchors);
  release(h->block_of);
  release(h->perm);
  release(h->off);
  release(h->C);
  release(h->nbr);
  release(h->cnt);
  release(h->local_blocks);
  release(h->work_order);
  release(h->Xperm);
  release(h->yperm);
  release(h->ybuf);
  release(h->terms);
  release(h->quads);
  release(h->logdets);
  release(h->status);
  release(h->chunk_local);
  release(h->chunk_all);
  release(h->result);
  release(h->queue);
  release(h->flag);
  release(h->a_start);
  release(h->a_list);
  release(h->p_start);
  release(h->p_list);
  release(h->ws);
  h->cap.clear();
  h->prepared = false;
}

__global__ void k_check_finite(const double *x, int64_t n, int *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) *bad = 1;
}

__global__ void k_scatter_terms(const double *src, const int32_t *local_blocks, int64_t k_local,
                                double *dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k_local;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[local_blocks[i]] = src[i];
}

__global__ void k_fill_d(double *p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_fill_i(int32_t *p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_nbr_to_orig(const int32_t *nbr, const int32_t *cnt, const int32_t *perm,
                              const int32_t *local_blocks, int64_t k_local, int m,
                              int32_t *out_nbr, int32_t *out_cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k_local * m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t li = e / m;
    int j = (int)(e - li * m);
    int64_t t = local_blocks[li];
    int32_t p = nbr[e];
    out_nbr[t * m + j] = (j < cnt[li] && p >= 0) ? perm[p] : -1;
    if (j == 0) out_cnt[t] = cnt[li];
  }
  if (m == 0)
    for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < k_local;
         li += (int64_t)gridDim.x * blockDim.x)
      out_cnt[local_blocks[li]] = 0;
}

__global__ void k_block_of_from_layout(const int32_t *perm, const int64_t *off, int64_t k,
                                       int32_t *bo) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < k;
       t += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = off[t]; p < off[t + 1]; p++) bo[perm[p]] = (int32_t)t;
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

// copy device array to a caller buffer that may be host or device
int copy_out(sbv_ctx *h, void *dst, const void *src, size_t bytes) {
  if (!dst || bytes == 0) return SBV_OK;
  CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return SBV_OK;
}

struct Timer {
  sbv_ctx *h;
  int prep;
  int idx = 0;
  Timer(sbv_ctx *h_, int prep_) : h(h_), prep(prep_) {
    if (h->profile) cudaEventRecord(h->ev[0], h->stream);
  }
  void mark(const char *name) {
    if (!h->profile || idx >= kMaxStages) return;
    cudaEventRecord(h->ev[idx + 1], h->stream);
    (prep ? h->name_prep : h->name_llh)[idx] = name;
    idx++;
  }
  void finish() {
    if (!h->profile) return;
    cudaEventSynchronize(h->ev[idx]);
    for (int i = 0; i < idx; i++) {
      float ms = 0;
      cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]);
      (prep ? h->t_prep : h->t_llh)[i] = ms;
    }
    (prep ? h->n_ev_prep : h->n_ev_llh) = idx;
  }
};

int validate_theta(sbv_ctx *h, const double *theta) {
  if (!theta) return fail(h, SBV_ERR_ARG, "theta is NULL");
  const int d = h->d;
  for (int i = 0; i < d + 3; i++)
    if (!isfinite(theta[i])) return fail(h, SBV_ERR_ARG, "theta has a non-finite entry");
  if (!(theta[0] > 0)) return fail(h, SBV_ERR_ARG, "sigma2 must be > 0");
  for (int j = 0; j < d; j++)
    if (!(theta[1 + j] > 0)) return fail(h, SBV_ERR_ARG, "beta_j must be > 0");
  if (!(theta[d + 2] >= 0)) return fail(h, SBV_ERR_ARG, "tau2 must be >= 0");
  const double nu = theta[d + 1];
  if (nu != 0.5 && nu != 1.5 && nu != 2.5 && nu != 3.5)
    return fail(h, SBV_ERR_UNSUPPORTED, "nu must be one of 0.5, 1.5, 2.5, 3.5");
  return SBV_OK;
}

// Steps 4-5 for the current handle; leaves per-block outputs on device and
// the reduced vector in h->result_host.
int run_loglik(sbv_ctx *h, const double *y, const double *theta) {
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "sbv_loglik before sbv_prepare");
  if (!y) return fail(h, SBV_ERR_ARG, "y is NULL");
  int rc = validate_theta(h, theta);
  if (rc) return rc;
  CU(cudaSetDevice(h->device));
  Timer tm(h, 0);
  const double *yd = y;
  if (!is_device_ptr(y)) {
    CU(cudaMemcpyAsync(h->ybuf, y, h->n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    yd = h->ybuf;
  }
  tm.mark("h2d_y");
  CU(launch_stage_eval(yd, h->perm, h->n, h->yperm, h->stream));
  tm.mark("H7_stage");
  CU(launch_h8(*h, theta, h->stream));
  tm.mark("H8_block_llh");
  CU(launch_reduce_chunks(*h, h->stream));
  tm.mark("H9_chunk_sums");
  if (h->world > 1) {
    int64_t ncl_pad = (h->n_chunks + h->world - 1) / h->world;
    NC(ncclAllGather(h->chunk_local, h->chunk_all, (size_t)ncl_pad * 8, ncclDouble, h->comm,
                     h->stream));
    tm.mark("H10_allgather");
  }
  CU(launch_final_reduce(*h, h->stream));
  CU(cudaMemcpyAsync(h->result_host, h->result, 8 * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  tm.mark("H9_final_d2h");
  CU(cudaStreamSynchronize(h->stream));
  tm.finish();
  if (h->result_host[4] > 0) {
    h->err_block = (int64_t)h->result_host[5];
    h->err_stage = (int32_t)h->result_host[6];
    h->err_msg = "Cholesky factorisation failed (non-positive pivot)";
    return SBV_ERR_NOT_PD;
  }
  h->err_block = -1;
  h->err_stage = 0;
  return SBV_OK;
}

}  // namespace

extern "C" {

int sbv_abi_version(void) { return SBV_ABI_VERSION; }

int sbv_shard_blocks(int64_t bc, int32_t rank, int32_t world, int32_t *blocks, int64_t *count) {
  if (bc < 0 || world < 1 || rank < 0 || rank >= world || !count) return SBV_ERR_ARG;
  const int64_t nch = (bc + kChunkBlocks - 1) / kChunkBlocks;
  int64_t n = 0;
  for (int64_t c = rank; c < nch; c += world)
    for (int64_t t = c * kChunkBlocks; t < std::min<int64_t>(bc, (c + 1) * kChunkBlocks); t++) {
      if (blocks) blocks[n] = (int32_t)t;
      n++;
    }
  *count = n;
  return SBV_OK;
}

int sbv_create(const sbv_opts *opts, sbv_handle *out) {
  if (!out) return SBV_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SBV_ERR_CUDA;
  }
  sbv_ctx *h = new sbv_ctx();
  cudaGetDevice(&h->device);
  {
    const char *e = getenv("SBV_GRID");
    h->use_grid = (e && atoi(e) == 0) ? 0 : 1;
  }
  if (opts) {
    h->seed = opts->seed;
    h->stream = (cudaStream_t)opts->stream;
    h->profile = opts->profile;
  }
  for (int i = 0; i <= kMaxStages; i++) cudaEventCreate(&h->ev[i]);
  if (cudaMallocHost(&h->result_host, 8 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&h->flag_host, 2 * sizeof(int)) != cudaSuccess) {
    delete h;
    return SBV_ERR_OOM;
  }
  // keep stream-ordered temporaries (CUB sort scratch) pooled across calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, h->device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = h;
  return SBV_OK;
}

void sbv_destroy(sbv_handle h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  free_state(h);
  if (h->comm) ncclCommDestroy(h->comm);
  for (int i = 0; i <= kMaxStages; i++)
    if (h->ev[i]) cudaEventDestroy(h->ev[i]);
  if (h->result_host) cudaFreeHost(h->result_host);
  if (h->flag_host) cudaFreeHost(h->flag_host);
  if (h->pin) cudaFreeHost(h->pin);
  delete h;
}

int sbv_comm_unique_id(void *id128) {
  if (!id128) return SBV_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SBV_ERR_COMM;
  memcpy(id128, &id, sizeof(id));
  return SBV_OK;
}

int sbv_comm_init(sbv_handle h, const void *nccl_unique_id, int32_t rank, int32_t world) {
  if (!h || !nccl_unique_id || world < 1 || rank < 0 || rank >= world) return SBV_ERR_ARG;
  if (h->prepared) return fail(h, SBV_ERR_STATE, "sbv_comm_init must precede sbv_prepare_h");
  if (world == 1) {
    h->rank = 0;
    h->world = 1;
    return SBV_OK;
  }
  CU(cudaSetDevice(h->device));
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  if (h->comm) ncclCommDestroy(h->comm);
  h->comm = nullptr;
  NC(ncclCommInitRank(&h->comm, world, id, rank));
  h->rank = rank;
  h->world = world;
  return SBV_OK;
}

int sbv_prepare_h(sbv_handle h, const double *X, int64_t n, int32_t d, int32_t bs, int32_t m,
                  const double *scale) {
  if (!h) return SBV_ERR_ARG;
  if (!X || !scale) return fail(h, SBV_ERR_ARG, "X or scale is NULL");
  if (n < 1 || n >= (int64_t(1) << 31)) return fail(h, SBV_ERR_ARG, "n out of range");
  if (d < 1 || d > SBV_MAX_D) return fail(h, SBV_ERR_ARG, "d out of range [1, 64]");
  if (bs < 1 || bs > n) return fail(h, SBV_ERR_ARG, "bs out of range [1, n]");
  if (m < 0) return fail(h, SBV_ERR_ARG, "m must be >= 0");
  if (m > 1536) return fail(h, SBV_ERR_UNSUPPORTED, "m > 1536 not supported by the kNN kernel");
  for (int j = 0; j < d; j++)
    if (!(scale[j] > 0) || !isfinite(scale[j])) return fail(h, SBV_ERR_ARG, "scale_j must be finite and > 0");
  CU(cudaSetDevice(h->device));
  h->prepared = false;
  h->n = n;
  h->d = d;
  h->bs = bs;
  h->m = m;
  h->scale.assign(scale, scale + d);
  const int64_t k = std::max<int64_t>(1, (2 * n + bs) / (2 * (int64_t)bs));  // round(n/bs)
  h->k = k;
  cudaStream_t st = h->stream;
  auto &unused = h->cap;
  Timer tm(h, 1);

  // device inputs are read in place (valid for the duration of the call);
  // host inputs are staged once
  const double *Xd = X;
  if (!is_device_ptr(X)) {
    CU(ensure(h->X, n * d, unused));
    CU(cudaMemcpyAsync(h->X, X, n * d * sizeof(double), cudaMemcpyDefault, st));
    Xd = h->X;
  }
  // finiteness flag: read back at the first host sync below (no extra stall)
  CU(ensure(h->flag, 2, unused));
  CU(cudaMemsetAsync(h->flag, 0, sizeof(int), st));
  k_check_finite<<<grid_for(n * d), 256, 0, st>>>(Xd, n * d, h->flag);
  CU(cudaMemcpyAsync(h->flag_host, h->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  tm.mark("h2d_X");
  CU(ensure(h->S, n * d, unused));
  CU(launch_scale(Xd, n, d, scale, h->S, st));
  tm.mark("H1_scale");
  CU(ensure(h->anchors, k, unused));
  if (h->use_grid) {  // filtered selection; verified at the next host sync (extents)
    CU(select_anchors_fast(n, k, h->seed, h->anchors, h->flag + 1, st));
    CU(cudaMemcpyAsync(h->flag_host + 1, h->flag + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  } else {
    CU(select_anchors(n, k, h->seed, h->anchors, nullptr, 0, st, nullptr));
  }
  tm.mark("H2_anchors");
  CU(ensure(h->block_of, n, unused));
  double lo_hi[2 * SBV_MAX_D];
  if (h->use_grid) {
    CU(data_extents(h->S, n, d, lo_hi, st));  // one small D2H (grid geometry) + sync
    if (h->flag_host[1] != 0) CU(select_anchors(n, k, h->seed, h->anchors, nullptr, 0, st, nullptr));
    tm.mark("extents");
    const GridDesc ga = make_grid(lo_hi, d, k, 3.0);
    CU(ensure(h->a_start, ga.ncells + 1, unused));
    CU(ensure(h->a_list, k, unused));
    CU(build_cells(h->S, h->anchors, k, d, ga, h->a_start, h->a_list, st));
    if (h->world > 1) {
      // RAC sharded by points: rank r assigns points [r c, (r+1) c), then one
      // in-place allgather rebuilds block_of everywhere (NVLink, 4 B/point)
      const int64_t chunk = (n + h->world - 1) / h->world;
      CU(ensure(h->block_of, chunk * h->world, unused));
      const int64_t i0 = std::min<int64_t>(n, h->rank * chunk), i1 = std::min<int64_t>(n, i0 + chunk);
      CU(launch_rac_grid(h->S, i1, i0, d, h->anchors, k, ga, h->a_start, h->a_list,
                         h->block_of + h->rank * chunk, st));
      NC(ncclAllGather(h->block_of + h->rank * chunk, h->block_of, (size_t)chunk, ncclInt32, h->comm, st));
    } else {
      CU(launch_rac_grid(h->S, n, 0, d, h->anchors, k, ga, h->a_start, h->a_list, h->block_of, st));
    }
    CU(anchor_own_block(h->anchors, k, h->block_of, st));
  } else {
    CU(launch_rac(h->S, n, d, h->anchors, k, h->block_of, st));
  }
  tm.mark("H3_rac");
  CU(ensure(h->perm, n, unused));
  CU(ensure(h->off, k + 1, unused));
  CU(build_layout(h->block_of, n, k, h->perm, h->off, nullptr, 0, st, nullptr));
  CU(ensure(h->Sperm, n * d, unused));
  CU(launch_gather_rows(h->S, h->perm, n, d, h->Sperm, st));
  tm.mark("H4_layout");
  // shard: 64-block chunks of zeta order dealt round-robin over ranks
  h->n_chunks = (k + kChunkBlocks - 1) / kChunkBlocks;
  // pinned host staging (async copies): local ids | off | cnt | LPT order
  const int64_t loc_cap = k / h->world + kChunkBlocks + 1;
  const size_t pin_bytes = sizeof(int64_t) * (size_t)(k + 1) + sizeof(int32_t) * (size_t)(3 * loc_cap + 2);
  if (h->pin_cap < pin_bytes) {
    if (h->pin) cudaFreeHost(h->pin);
    h->pin = nullptr;
    h->pin_cap = 0;
    CU(cudaMallocHost(&h->pin, pin_bytes));
    h->pin_cap = pin_bytes;
  }
  int64_t *off_h = reinterpret_cast<int64_t *>(h->pin);
  int32_t *local = reinterpret_cast<int32_t *>(off_h + k + 1);
  int32_t *cnt_h = local + loc_cap;
  int32_t *order = cnt_h + loc_cap;
  {
    int64_t cnt_local = 0;
    sbv_shard_blocks(k, h->rank, h->world, local, &cnt_local);
    h->k_local = cnt_local;
  }
  h->n_chunks_local = (h->k_local + kChunkBlocks - 1) / kChunkBlocks;
  CU(ensure(h->local_blocks, h->k_local, unused));
  CU(cudaMemcpyAsync(h->local_blocks, local, h->k_local * sizeof(int32_t),
                     cudaMemcpyHostToDevice, st));
  CU(ensure(h->C, k * d, unused));
  CU(launch_centroids(h->Sperm, h->off, h->world > 1 ? h->local_blocks : nullptr, h->k_local, d,
                      h->C, st));
  tm.mark("H5_centroids");

  const int mm = m > 0 ? m : 1;
  CU(ensure(h->nbr, h->k_local * mm, unused));
  CU(ensure(h->cnt, h->k_local, unused));
  if (h->use_grid && m <= knn_grid_max_m()) {
    const KnnLevels lv = make_knn_levels(lo_hi, d, n, m);
    CU(ensure(h->p_start, lv.cell_off[lv.nl] + 1, unused));
    CU(ensure(h->p_list, lv.list_off[lv.nl], unused));
    CU(build_knn_levels(h->Sperm, d, lv, h->p_start, h->p_list, st));
    tm.mark("H6_grid");
    CU(launch_knn_grid(h->Sperm, h->perm, h->off, h->C, h->local_blocks, h->k_local, d, m, lv,
                       h->p_start, h->p_list, h->nbr, h->cnt, st));
  } else {
    CU(launch_knn(h->Sperm, h->perm, h->off, h->C, h->local_blocks, h->k_local, d, m, h->nbr,
                  h->cnt, st));
  }
  tm.mark("H6_knn");

  // block-major original inputs for H8 (queued before the host sync below)
  CU(ensure(h->Xperm, n * d, unused));
  CU(launch_gather_rows(Xd, h->perm, n, d, h->Xperm, st));

  // realised sizes -> LPT work order, statistics, H8 launch geometry
  CU(cudaMemcpyAsync(off_h, h->off, (k + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(cnt_h, h->cnt, h->k_local * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (*h->flag_host) return fail(h, SBV_ERR_ARG, "X has non-finite entries");
  std::vector<int32_t> Nt(h->k_local);
  h->max_N = 0;
  h->min_bs = INT32_MAX;
  h->max_bs = 0;
  h->flops = h->entries = h->knn_pairs = 0;
  for (int64_t li = 0; li < h->k_local; li++) {
    int64_t t = local[li];
    double b = (double)(off_h[t + 1] - off_h[t]), mt = cnt_h[li];
    Nt[li] = (int32_t)(mt + b);
    h->max_N = std::max(h->max_N, Nt[li]);
    h->min_bs = std::min(h->min_bs, (int32_t)b);
    h->max_bs = std::max(h->max_bs, (int32_t)b);
    // SURVEY 8(d) flop model (LAPACK conventions)
    h->flops += (mt * mt * mt / 3 + mt * mt / 2 + mt / 6) + mt * mt * b + mt * mt +
                b * (b + 1) * mt + 2 * mt * b + (b * b * b / 3 + b * b / 2 + b / 6) + b * b + 2 * b;
    h->entries += mt * (mt + 1) / 2 + mt * b + b * (b + 1) / 2;
    h->knn_pairs += (double)off_h[t];
  }
  h->rac_pairs = (double)n * (double)k;
  h->h8_bytes = 0;
  for (int64_t li = 0; li < h->k_local; li++)
    h->h8_bytes += (double)Nt[li] * (d + 1) * 8.0 + (double)cnt_h[li] * 4.0 + 4 * 8.0;
  // LPT order (N_t descending, ties by local index): a stable counting sort
  {
    std::vector<int64_t> bucket((size_t)h->max_N + 2, 0);
    for (int64_t li = 0; li < h->k_local; li++) bucket[h->max_N - Nt[li] + 1]++;
    for (size_t b = 1; b < bucket.size(); b++) bucket[b] += bucket[b - 1];
    for (int64_t li = 0; li < h->k_local; li++) order[bucket[h->max_N - Nt[li]]++] = (int32_t)li;
  }
  CU(ensure(h->work_order, h->k_local, unused));
  CU(cudaMemcpyAsync(h->work_order, order, h->k_local * sizeof(int32_t),
                     cudaMemcpyHostToDevice, st));

  // per-eval buffers
  CU(ensure(h->yperm, n, unused));
  CU(ensure(h->ybuf, n, unused));
  CU(ensure(h->terms, h->k_local, unused));
  CU(ensure(h->quads, h->k_local, unused));
  CU(ensure(h->logdets, h->k_local, unused));
  CU(ensure(h->status, h->k_local, unused));
  const int64_t ncl_pad = h->world > 1 ? (h->n_chunks + h->world - 1) / h->world : h->n_chunks;
  CU(ensure(h->chunk_local, std::max<int64_t>(ncl_pad, 1) * 8, unused));
  CU(cudaMemsetAsync(h->chunk_local, 0, std::max<int64_t>(ncl_pad, 1) * 8 * sizeof(double), st));
  if (h->world > 1) CU(ensure(h->chunk_all, (int64_t)h->world * ncl_pad * 8, unused));
  CU(ensure(h->result, 8, unused));
  CU(ensure(h->queue, 1, unused));
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  h->h8_smem = h8_smem_bytes(std::max(h->max_N, 1), d);
  int smem_optin = 0;
  CU(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  if (h->max_N > 4096) return fail(h, SBV_ERR_UNSUPPORTED, "m + block size > 4096");
  if (h->h8_smem + 1024 > (size_t)smem_optin)
    return fail(h, SBV_ERR_UNSUPPORTED, "block + neighbour set too large for shared memory staging");
  if (h->h8_smem != h->occ_smem || d != h->occ_d) {  // occupancy query only on a change
    h->occ_smem = h->h8_smem;
    h->occ_d = d;
    h->occ_per_sm = h8_max_ctas_per_sm(h->h8_smem, d);
  }
  int per_sm = h->occ_per_sm;
  if (per_sm < 1) per_sm = 1;
  h->h8_grid = (int)std::min<int64_t>((int64_t)sms * per_sm, std::max<int64_t>(h->k_local, 1));
  h->ws_per_cta = h8_ws_doubles(std::max(h->max_N, 1), d);
  CU(ensure(h->ws, (size_t)h->h8_grid * h->ws_per_cta, unused));
  CU(cudaStreamSynchronize(st));
  tm.mark("meta");
  tm.finish();
  h->prepared = true;
  return SBV_OK;
}

int sbv_prepare_ex(const double *X, int64_t n, int32_t d, int32_t bs, int32_t m,
                   const double *scale, const sbv_opts *opts, sbv_handle *out) {
  if (!out) return SBV_ERR_ARG;
  *out = nullptr;
  sbv_handle h = nullptr;
  int rc = sbv_create(opts, &h);
  if (rc) return rc;
  rc = sbv_prepare_h(h, X, n, d, bs, m, scale);
  if (rc) {
    sbv_destroy(h);
    return rc;
  }
  *out = h;
  return SBV_OK;
}

int sbv_prepare(const double *X, int64_t n, int32_t d, int32_t bs, int32_t m, const double *scale,
                sbv_handle *out) {
  return sbv_prepare_ex(X, n, d, bs, m, scale, nullptr, out);
}

int sbv_loglik_parts(sbv_handle h, const double *y, const double *theta, double *parts) {
  if (!h) return SBV_ERR_ARG;
  int rc = run_loglik(h, y, theta);
  const double two_pi_half = 0.91893853320467274178;  // log(2 pi) / 2
  (void)two_pi_half;
  if (parts) {
    parts[0] = rc == SBV_OK ? h->result_host[0] : NAN;
    parts[1] = h->result_host[1];
    parts[2] = h->result_host[2];
    parts[3] = h->result_host[3];
  }
  return rc;
}

int sbv_loglik(sbv_handle h, const double *y, const double *theta, double *ll) {
  if (!h) return SBV_ERR_ARG;
  if (!ll) return fail(h, SBV_ERR_ARG, "ll is NULL");
  int rc = run_loglik(h, y, theta);
  *ll = rc == SBV_OK ? h->result_host[0] : NAN;
  return rc;
}

int sbv_block_terms(sbv_handle h, const double *y, const double *theta, double *terms,
                    double *quad, double *logdet) {
  if (!h) return SBV_ERR_ARG;
  int rc = run_loglik(h, y, theta);
  if (rc != SBV_OK && rc != SBV_ERR_NOT_PD) return rc;
  double *tmp = nullptr;
  cudaStream_t st = h->stream;
  CU(cudaMallocAsync(&tmp, h->k * sizeof(double), st));
  const double *srcs[3] = {h->terms, h->quads, h->logdets};
  double *dsts[3] = {terms, quad, logdet};
  for (int i = 0; i < 3; i++) {
    if (!dsts[i]) continue;
    k_fill_d<<<grid_for(h->k), 256, 0, st>>>(tmp, h->k, NAN);
    k_scatter_terms<<<grid_for(h->k_local), 256, 0, st>>>(srcs[i], h->local_blocks, h->k_local, tmp);
    int r2 = copy_out(h, dsts[i], tmp, h->k * sizeof(double));
    if (r2) return r2;
  }
  cudaFreeAsync(tmp, st);
  CU(cudaStreamSynchronize(st));
  return rc;
}

int sbv_num_blocks(sbv_handle h, int64_t *bc) {
  if (!h || !bc) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "not prepared");
  *bc = h->k;
  return SBV_OK;
}

int sbv_get_anchors(sbv_handle h, int32_t *anchors) {
  if (!h || !anchors) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "not prepared");
  return copy_out(h, anchors, h->anchors, h->k * sizeof(int32_t));
}

int sbv_get_blocks(sbv_handle h, int32_t *block_of_point, int64_t *off, int32_t *perm,
                   double *centroids) {
  if (!h) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "not prepared");
  int rc;
  if ((rc = copy_out(h, block_of_point, h->block_of, h->n * sizeof(int32_t)))) return rc;
  if ((rc = copy_out(h, off, h->off, (h->k + 1) * sizeof(int64_t)))) return rc;
  if ((rc = copy_out(h, perm, h->perm, h->n * sizeof(int32_t)))) return rc;
  if (centroids && h->world > 1)  // prepare computed only this rank's query blocks
    CU(launch_centroids(h->Sperm, h->off, nullptr, h->k, h->d, h->C, h->stream));
  if ((rc = copy_out(h, centroids, h->C, h->k * h->d * sizeof(double)))) return rc;
  return SBV_OK;
}

int sbv_get_neighbors(sbv_handle h, int32_t *nbr, int32_t *cnt) {
  if (!h) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "not prepared");
  cudaStream_t st = h->stream;
  const int m = h->m;
  int32_t *tn = nullptr, *tc = nullptr;
  CU(cudaMallocAsync(&tn, std::max<int64_t>(h->k * m, 1) * sizeof(int32_t), st));
  CU(cudaMallocAsync(&tc, h->k * sizeof(int32_t), st));
  k_fill_i<<<grid_for(h->k * m), 256, 0, st>>>(tn, h->k * m, -1);
  k_fill_i<<<grid_for(h->k), 256, 0, st>>>(tc, h->k, -1);
  k_nbr_to_orig<<<grid_for(std::max<int64_t>(h->k_local * m, h->k_local)), 256, 0, st>>>(
      h->nbr, h->cnt, h->perm, h->local_blocks, h->k_local, m, tn, tc);
  int rc = SBV_OK;
  if (nbr && m > 0) rc = copy_out(h, nbr, tn, h->k * m * sizeof(int32_t));
  if (!rc && cnt) rc = copy_out(h, cnt, tc, h->k * sizeof(int32_t));
  cudaFreeAsync(tn, st);
  cudaFreeAsync(tc, st);
  CU(cudaStreamSynchronize(st));
  return rc;
}

int sbv_stats(sbv_handle h, double *out9) {
  if (!h || !out9) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "not prepared");
  out9[0] = h->flops;
  out9[1] = h->entries;
  out9[2] = h->max_N;
  out9[3] = h->min_bs;
  out9[4] = h->max_bs;
  out9[5] = (double)h->k_local;
  out9[6] = h->knn_pairs;
  out9[7] = h->rac_pairs;
  out9[8] = h->h8_bytes;
  return SBV_OK;
}

int sbv_stage_times(sbv_handle h, int32_t prep, double *ms, const char **names, int32_t cap,
                    int32_t *count) {
  if (!h || !count) return SBV_ERR_ARG;
  int nn = prep ? h->n_ev_prep : h->n_ev_llh;
  nn = std::min(nn, (int)cap);
  for (int i = 0; i < nn; i++) {
    if (ms) ms[i] = prep ? h->t_prep[i] : h->t_llh[i];
    if (names) names[i] = prep ? h->name_prep[i] : h->name_llh[i];
  }
  *count = nn;
  return SBV_OK;
}

int sbv_last_error(sbv_handle h, int64_t *block, int32_t *stage, const char **msg) {
  if (!h) return SBV_ERR_ARG;
  if (block) *block = h->err_block;
  if (stage) *stage = h->err_stage;
  if (msg) *msg = h->err_msg.c_str();
  return SBV_OK;
}

}  // extern "C"
