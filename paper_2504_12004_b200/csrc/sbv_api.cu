// sbv_api.cu — the extern "C" boundary of libsbv (include/sbv.h).
//
// Orchestrates the device steps of Alg.1: sbv_prepare_h runs
// Steps 1-3 (H1-H6, prep_kernels.cu) and sbv_loglik runs Steps 4-5 (H7-H10,
// llh_kernel.cu).  No host arithmetic of the method happens here: the host
// only validates arguments, sizes buffers, builds the block shard / work
// order from the device-computed layout, and launches.
#include <dlfcn.h>
#include <execinfo.h>
#include <math.h>
#include <signal.h>
#include <stdio.h>
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
  release(h->Xq);
  release(h->Sq);
  release(h->Sqp);
  release(h->Xqp);
  release(h->Cq);
  release(h->q_anchors);
  release(h->q_block_of);
  release(h->q_perm);
  release(h->q_nbr);
  release(h->q_cnt);
  release(h->q_local);
  release(h->q_order);
  release(h->q_status);
  release(h->q_off);
  release(h->qa_start);
  release(h->qa_list);
  release(h->q_mean);
  release(h->q_var);
  release(h->q_terms);
  release(h->q_quads);
  release(h->q_logdets);
  release(h->Lg);
  release(h->lg_off);
  release(h->zws);
  release(h->grads);
  release(h->gsum);
  release(h->theta_dev);
  if (h->g_exec) cudaGraphExecDestroy(h->g_exec);
  h->g_exec = nullptr;
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

__global__ void k_iota(int32_t *p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

// out[perm[p]] = in[p]: block-major -> caller order
__global__ void k_unpermute(const double *in, const int32_t *perm, int64_t n, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[perm[i]] = in[i];
}

// Sec.5.5 conditional simulation, thread per point:
// x_s = mean + sqrt(var) z_s, z_s by Box-Muller from splitmix64 counters
// 2c, 2c+1 (c = j n_sim + s); two passes (mean, then squared deviations).
__device__ __forceinline__ uint64_t sim_splitmix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double sim_normal(uint64_t seed, uint64_t c) {
  const double u1 = ((double)(sim_splitmix64(seed, 2 * c) >> 11) + 0.5) * 0x1p-53;
  const double u2 = ((double)(sim_splitmix64(seed, 2 * c + 1) >> 11) + 0.5) * 0x1p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}
__global__ void k_simulate(const double *mean, const double *var, int64_t ns, int n_sim, uint64_t seed,
                           double ci_level, double *sm, double *ssd, double *lo, double *hi) {
  // z_{alpha/2}: P(Z > z) = erfc(z / sqrt 2) / 2 = (1 - ci) / 2, by bisection
  const double tail = 0.5 * (1.0 - ci_level);
  double zl = 0.0, zh = 40.0;
  for (int it = 0; it < 200; it++) {
    const double mid = 0.5 * (zl + zh);
    if (0.5 * erfc(mid / sqrt(2.0)) > tail)
      zl = mid;
    else
      zh = mid;
  }
  const double zc = 0.5 * (zl + zh);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < ns;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double mu = mean[j], sd = sqrt(var[j]);
    double sum = 0.0;
    for (int s = 0; s < n_sim; s++) sum = sum + (mu + sd * sim_normal(seed, (uint64_t)j * n_sim + s));
    const double xm = sum / n_sim;
    double ss = 0.0;
    for (int s = 0; s < n_sim; s++) {
      const double dv = (mu + sd * sim_normal(seed, (uint64_t)j * n_sim + s)) - xm;
      ss = ss + dv * dv;
    }
    const double sdv = sqrt(ss / (n_sim - 1));
    sm[j] = xm;
    ssd[j] = sdv;
    lo[j] = xm - zc * sdv;
    hi[j] = xm + zc * sdv;
  }
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
    if (!h->profile) return;
    h->ev_pending[prep ? 0 : 1] = 0;  // the previous call's events are being re-recorded
    (prep ? h->n_ev_prep : h->n_ev_llh) = 0;
    cudaEventRecord(h->ev[prep ? 0 : 1][0], h->stream);
  }
  void mark(const char *name) {
    if (h->debug) {  // SBV_DEBUG=1: stage trace on stderr (host-side progress)
      fprintf(stderr, "[sbv] %s %s done (queued)\n", prep ? "prepare" : "loglik", name);
      fflush(stderr);
    }
    if (!h->profile || idx >= kMaxStages) return;
    cudaEventRecord(h->ev[prep ? 0 : 1][idx + 1], h->stream);
    (prep ? h->name_prep : h->name_llh)[idx] = name;
    idx++;
  }
  void finish() {  // no synchronisation here: sbv_stage_times resolves the events
    if (!h->profile) return;
    (prep ? h->n_ev_prep : h->n_ev_llh) = idx;
    h->ev_pending[prep ? 0 : 1] = 1;
  }
};

void resolve_stage_times(sbv_ctx *h, int prep) {
  const int w = prep ? 0 : 1;
  if (!h->ev_pending[w]) return;
  const int n = prep ? h->n_ev_prep : h->n_ev_llh;
  cudaEventSynchronize(h->ev[w][n]);
  for (int i = 0; i < n; i++) {
    float ms = 0;
    cudaEventElapsedTime(&ms, h->ev[w][i], h->ev[w][i + 1]);
    (prep ? h->t_prep : h->t_llh)[i] = ms;
  }
  h->ev_pending[w] = 0;
}

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
  if (!(nu > 0.0) || nu > 20.0)
    return fail(h, SBV_ERR_UNSUPPORTED, "nu must be in (0, 20] (closed forms at 0.5/1.5/2.5/3.5, K_nu otherwise)");
  return SBV_OK;
}

// sbv_loglik replayed from a CUDA graph (sbv_set_graph; one GPU, device y):
// H7 -> H8 -> H9 -> D2H of the result, captured on a private stream once per
// (y pointer, nu, prepare) and launched on the handle's stream; theta reaches
// the kernels through a pinned host -> device copy node (H8Args::theta_d), so
// a new theta needs no re-capture.  Same kernels, same results bit for bit.
int run_loglik_graph(sbv_ctx *h, const double *y, const double *theta) {
  const int d = h->d;
  const double nu = theta[d + 1];
  if (!h->g_exec || h->g_y != y || h->g_nu != nu || h->g_gen != h->prep_gen) {
    if (h->g_exec) {
      cudaGraphExecDestroy(h->g_exec);
      h->g_exec = nullptr;
    }
    if (!h->g_stream) CU(cudaStreamCreateWithFlags(&h->g_stream, cudaStreamNonBlocking));
    if (!h->theta_pin) CU(cudaMallocHost(&h->theta_pin, (SBV_MAX_D + 3) * sizeof(double)));
    CU(ensure(h->theta_dev, SBV_MAX_D + 3, h->cap));
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(h->g_stream, cudaStreamCaptureModeRelaxed));
    cudaError_t e = cudaMemcpyAsync(h->theta_dev, h->theta_pin, (d + 3) * sizeof(double),
                                    cudaMemcpyHostToDevice, h->g_stream);
    if (!e) e = launch_stage_eval(y, h->perm, h->n, h->yperm, h->g_stream);
    if (!e) e = launch_h8(*h, theta, h->g_stream, h->theta_dev);
    if (!e) e = launch_reduce_chunks(*h, h->g_stream);
    if (!e) e = launch_final_reduce(*h, h->g_stream);
    if (!e) e = cudaMemcpyAsync(h->result_host, h->result, 8 * sizeof(double), cudaMemcpyDeviceToHost,
                                h->g_stream);
    const cudaError_t e2 = cudaStreamEndCapture(h->g_stream, &g);
    if (!e) e = e2;
    if (!e) e = cudaGraphInstantiate(&h->g_exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e) {
      h->g_exec = nullptr;
      cudaGetLastError();
      return fail(h, SBV_ERR_CUDA, cudaGetErrorString(e));
    }
    h->g_y = y;
    h->g_nu = nu;
    h->g_gen = h->prep_gen;
  }
  memcpy(h->theta_pin, theta, (d + 3) * sizeof(double));  // the previous replay has completed
  CU(cudaGraphLaunch(h->g_exec, h->stream));
  CU(cudaStreamSynchronize(h->stream));
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

// Steps 4-5 for the current handle; leaves per-block outputs on device and
// the reduced vector in h->result_host.
// partials != nullptr: stop after H9 and copy this rank's chunk partials
// (sbv_loglik_partials); otherwise the full H7-H10 path.
int run_loglik(sbv_ctx *h, const double *y, const double *theta, double *partials = nullptr) {
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "sbv_loglik before sbv_prepare");
  if (!y) return fail(h, SBV_ERR_ARG, "y is NULL");
  if (!partials && h->world > 1 && !h->comm)
    return fail(h, SBV_ERR_STATE, "sharded without a communicator (sbv_set_shard): use "
                                  "sbv_loglik_partials + sbv_reduce_partials");
  int rc = validate_theta(h, theta);
  if (rc) return rc;
  CU(cudaSetDevice(h->device));
  if (h->use_graph && !partials && h->world == 1 && !h->profile && is_device_ptr(y))
    return run_loglik_graph(h, y, theta);
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
  if (partials) {
    CU(cudaMemcpyAsync(partials, h->chunk_local, (size_t)h->ncl_pad * 8 * sizeof(double),
                       cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    tm.finish();
    return SBV_OK;
  }
  if (h->world > 1) {
    NC(ncclAllGather(h->chunk_local, h->chunk_all, (size_t)h->ncl_pad * 8, ncclDouble, h->comm,
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

}  // extern "C"

namespace {
// SBV_DEBUG=1: print the native stack on SIGSEGV (host-side debugging aid)
void segv_handler(int sig) {
  void *frames[64];
  const int nf = backtrace(frames, 64);
  fprintf(stderr, "[sbv] signal %d, native backtrace:\n", sig);
  backtrace_symbols_fd(frames, nf, 2);
  Dl_info info;
  if (dladdr((void *)&segv_handler, &info)) fprintf(stderr, "[sbv] libsbv base %p\n", info.dli_fbase);
  signal(sig, SIG_DFL);
  raise(sig);
}
}  // namespace

extern "C" {

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
    const char *dbg = getenv("SBV_DEBUG");
    h->debug = (dbg && atoi(dbg) != 0) ? 1 : 0;
    if (h->debug) signal(SIGSEGV, segv_handler);
  }
  if (opts) {
    h->seed = opts->seed;
    h->stream = (cudaStream_t)opts->stream;
    h->profile = opts->profile;
  }
  for (int w = 0; w < 2; w++)
    for (int i = 0; i <= kMaxStages; i++) cudaEventCreate(&h->ev[w][i]);
  cudaEventCreateWithFlags(&h->ev_sizes, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&h->ev_pin, cudaEventDisableTiming);
  if (cudaMallocHost(&h->result_host, 8 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&h->flag_host, 2 * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    sbv_destroy(h);  // frees whatever was created (events, pinned buffers)
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
    for (int w = 0; w < 2; w++)
      if (h->ev[w][i]) cudaEventDestroy(h->ev[w][i]);
  if (h->ev_sizes) cudaEventDestroy(h->ev_sizes);
  if (h->ev_pin) cudaEventDestroy(h->ev_pin);
  if (h->result_host) cudaFreeHost(h->result_host);
  if (h->flag_host) cudaFreeHost(h->flag_host);
  if (h->pin) cudaFreeHost(h->pin);
  if (h->theta_pin) cudaFreeHost(h->theta_pin);
  if (h->g_stream) cudaStreamDestroy(h->g_stream);
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

}  // extern "C"

namespace {

__global__ void k_check_blocks(const int32_t *bo, int64_t n, int64_t k, int *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (bo[i] < 0 || bo[i] >= k) *bad = 1;
}

// Alg.1 Steps 1-3.  given_bo == nullptr: H2 anchors + H3 RAC define the
// blocks (k = round(n/bs)); otherwise the caller's partition (block id = zeta
// position, k = kk blocks) replaces H2/H3 ("block centroids given").
int prepare_impl(sbv_ctx *h, const double *X, int64_t n, int32_t d, int32_t bs, int32_t m,
                 const double *scale, const int32_t *given_bo, int64_t kk) {
  if (!h) return SBV_ERR_ARG;
  if (!X || !scale) return fail(h, SBV_ERR_ARG, "X or scale is NULL");
  if (n < 1 || n >= (int64_t(1) << 31)) return fail(h, SBV_ERR_ARG, "n out of range");
  if (d < 1 || d > SBV_MAX_D) return fail(h, SBV_ERR_ARG, "d out of range [1, 64]");
  if (given_bo) {
    if (kk < 1 || kk > n) return fail(h, SBV_ERR_ARG, "block count out of range [1, n]");
  } else if (bs < 1 || bs > n) {
    return fail(h, SBV_ERR_ARG, "bs out of range [1, n]");
  }
  if (m < 0) return fail(h, SBV_ERR_ARG, "m must be >= 0");
  if (m > 1536) return fail(h, SBV_ERR_UNSUPPORTED, "m > 1536 not supported by the kNN kernel");
  for (int j = 0; j < d; j++)
    if (!(scale[j] > 0) || !isfinite(scale[j])) return fail(h, SBV_ERR_ARG, "scale_j must be finite and > 0");
  CU(cudaSetDevice(h->device));
  // the previous prepare's async H2D copies out of the pinned staging must be
  // done before the staging is rewritten below
  CU(cudaEventSynchronize(h->ev_pin));
  h->prepared = false;
  h->lv_valid = false;
  h->ks = 0;
  h->n = n;
  h->d = d;
  h->bs = given_bo ? (int32_t)std::max<int64_t>(1, n / kk) : bs;
  h->m = m;
  h->given_blocks = given_bo ? 1 : 0;
  h->scale.assign(scale, scale + d);
  const int64_t k = given_bo ? kk : std::max<int64_t>(1, (2 * n + bs) / (2 * (int64_t)bs));  // round(n/bs)
  h->k = k;
  cudaStream_t st = h->stream;
  auto &unused = h->cap;
  Timer tm(h, 1);

  // device inputs are read in place (valid for the duration of the call:
  // every kernel reading X is queued before the host wait on ev_sizes below);
  // host inputs are staged once
  const double *Xd = X;
  if (!is_device_ptr(X)) {
    CU(ensure(h->X, n * d, unused));
    CU(cudaMemcpyAsync(h->X, X, n * d * sizeof(double), cudaMemcpyDefault, st));
    Xd = h->X;
  }
  tm.mark("h2d_X");
  CU(ensure(h->S, n * d, unused));
  CU(launch_scale(Xd, n, d, scale, h->S, st));
  // finiteness of S = X / scale (a finite X over a tiny scale can overflow);
  // the flag is read back at the first host sync below (no extra stall)
  CU(ensure(h->flag, 2, unused));
  CU(cudaMemsetAsync(h->flag, 0, 2 * sizeof(int), st));
  k_check_finite<<<grid_for(n * d), 256, 0, st>>>(h->S, n * d, h->flag);
  tm.mark("H1_scale");
  CU(ensure(h->anchors, k, unused));
  CU(ensure(h->block_of, n, unused));
  if (given_bo) {
    k_fill_i<<<grid_for(k), 256, 0, st>>>(h->anchors, k, -1);  // no anchors: partition given
    CU(cudaMemcpyAsync(h->block_of, given_bo, n * sizeof(int32_t), cudaMemcpyDefault, st));
    k_check_blocks<<<grid_for(n), 256, 0, st>>>(h->block_of, n, k, h->flag);
  } else if (h->use_grid) {  // filtered selection; verified at the next host sync (extents)
    CU(select_anchors_fast(n, k, h->seed, h->anchors, h->flag + 1, st));
  } else {
    CU(select_anchors(n, k, h->seed, h->anchors, nullptr, 0, st, nullptr));
  }
  CU(cudaMemcpyAsync(h->flag_host, h->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  tm.mark(given_bo ? "H2_given_blocks" : "H2_anchors");
  double lo_hi[2 * SBV_MAX_D];
  if (h->use_grid) {
    CU(data_extents(h->S, n, d, lo_hi, st));  // one small D2H (grid geometry) + sync
    if (*h->flag_host) return fail(h, SBV_ERR_ARG, given_bo ? "X/scale non-finite or block id out of [0, k)"
                                                             : "X has non-finite entries (or X/scale overflows)");
    if (!given_bo && h->flag_host[1] != 0) CU(select_anchors(n, k, h->seed, h->anchors, nullptr, 0, st, nullptr));
    tm.mark("extents");
  }
  if (given_bo) {
    // H3 skipped
  } else if (h->use_grid) {
    const GridDesc ga = make_grid(lo_hi, d, k, 3.0);
    CU(ensure(h->a_start, ga.ncells + 1, unused));
    CU(ensure(h->a_list, k, unused));
    CU(build_cells(h->S, h->anchors, k, d, ga, h->a_start, h->a_list, st));
    if (h->world > 1 && h->comm) {
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
  // block-major ORIGINAL inputs for H8: the last read of the caller's X, queued
  // before the ev_sizes host wait, so X may be freed when prepare returns
  CU(ensure(h->Xperm, n * d, unused));
  CU(launch_gather_rows(Xd, h->perm, n, d, h->Xperm, st));
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
  // block sizes to the host now: the launch geometry below needs only `off`
  // (m_t = min(m, off_t) exactly: every admissible point is found when fewer
  // than m exist, all distances being finite), so the host works while the
  // GPU runs H5-H6
  CU(cudaMemcpyAsync(off_h, h->off, (k + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(h->flag_host, h->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaEventRecord(h->ev_sizes, st));
  if (given_bo) {  // a caller partition is validated before H5-H6 run on it
    CU(cudaEventSynchronize(h->ev_sizes));
    if (h->debug) {
      fprintf(stderr, "[sbv] given partition: k=%lld off[0..3]=%lld %lld %lld %lld off[k]=%lld flag=%d\n",
              (long long)k, (long long)off_h[0], (long long)off_h[std::min<int64_t>(1, k)],
              (long long)off_h[std::min<int64_t>(2, k)], (long long)off_h[std::min<int64_t>(3, k)],
              (long long)off_h[k], *h->flag_host);
    }
    if (*h->flag_host) return fail(h, SBV_ERR_ARG, "X/scale non-finite or block id out of [0, k)");
    for (int64_t t = 0; t < k; t++)
      if (off_h[t + 1] == off_h[t]) return fail(h, SBV_ERR_ARG, "given partition has an empty block");
  }
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
    h->lv = lv;
    h->lv_valid = true;
    tm.mark("H6_grid");
    CU(launch_knn_grid(h->Sperm, h->perm, h->off, h->C, h->local_blocks, h->k_local, d, m, lv,
                       h->p_start, h->p_list, h->nbr, h->cnt, st));
  } else {
    CU(launch_knn(h->Sperm, h->perm, h->off, h->C, h->local_blocks, h->k_local, d, m, h->nbr,
                  h->cnt, st));
  }
  tm.mark("H6_knn");

  // realised sizes -> LPT work order, statistics, H8 launch geometry
  CU(cudaEventSynchronize(h->ev_sizes));
  if (*h->flag_host)
    return fail(h, SBV_ERR_ARG, given_bo ? "X/scale non-finite or block id out of [0, k)"
                                         : "X has non-finite entries (or X/scale overflows)");
  // the layout as the host sees it must be a partition of [0, n) (guards the
  // host-side sizing below against a failed device step)
  if (off_h[0] != 0 || off_h[k] != n) return fail(h, SBV_ERR_CUDA, "block layout inconsistent (device step failed)");
  for (int64_t t = 0; t < k; t++)
    if (off_h[t + 1] < off_h[t]) return fail(h, SBV_ERR_CUDA, "block layout inconsistent (device step failed)");
  for (int64_t li = 0; li < h->k_local; li++) cnt_h[li] = (int32_t)std::min<int64_t>(m, off_h[local[li]]);
  std::vector<int32_t> &Nt = h->Nt;
  Nt.assign(h->k_local, 0);
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
  h->rac_pairs = given_bo ? 0.0 : (double)n * (double)k;
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
  h->order_h.assign(order, order + h->k_local);
  CU(cudaEventRecord(h->ev_pin, st));  // the next prepare waits on it before reusing `pin`

  // per-eval buffers
  CU(ensure(h->yperm, n, unused));
  CU(ensure(h->ybuf, n, unused));
  CU(ensure(h->terms, h->k_local, unused));
  CU(ensure(h->quads, h->k_local, unused));
  CU(ensure(h->logdets, h->k_local, unused));
  CU(ensure(h->status, h->k_local, unused));
  const int64_t ncl_pad = h->world > 1 ? (h->n_chunks + h->world - 1) / h->world : h->n_chunks;
  h->ncl_pad = ncl_pad;
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
    h->occ_small = h8_small_ctas_per_sm(h->h8_smem, d);
  }
  int per_sm = h->occ_per_sm;
  h->h8_small = h8_use_small(h->max_N) ? 1 : 0;
  if (h->h8_small) per_sm = std::max(per_sm, h->occ_small);
  if (per_sm < 1) per_sm = 1;
  h->h8_grid = (int)std::min<int64_t>((int64_t)sms * per_sm, std::max<int64_t>(h->k_local, 1));
  {
    std::vector<int32_t> No(h->k_local);
    for (int64_t it = 0; it < h->k_local; it++) No[it] = Nt[order[it]];
    h8_split_plan(No.data(), h->k_local, d, sms, &h->h8_n_big, &h->h8_max_N_small, &h->h8_grid_small);
  }
  h->ws_per_cta = h8_ws_doubles(std::max(h->max_N, 1), d);
  CU(ensure(h->ws, (size_t)std::max(h->h8_grid, h->h8_grid_small) * h->ws_per_cta, unused));
  // no trailing host sync: everything above is stream-ordered before the
  // first sbv_loglik; the pinned staging is guarded by ev_pin
  tm.mark("meta");
  tm.finish();
  h->prepared = true;
  h->prep_gen++;
  return SBV_OK;
}

}  // namespace

extern "C" {

int sbv_prepare_h(sbv_handle h, const double *X, int64_t n, int32_t d, int32_t bs, int32_t m,
                  const double *scale) {
  return prepare_impl(h, X, n, d, bs, m, scale, nullptr, 0);
}

int sbv_prepare_blocks(sbv_handle h, const double *X, int64_t n, int32_t d, int64_t k,
                       const int32_t *block_of_point, int32_t m, const double *scale) {
  if (!h) return SBV_ERR_ARG;
  if (!block_of_point) return fail(h, SBV_ERR_ARG, "block_of_point is NULL");
  return prepare_impl(h, X, n, d, 1, m, scale, block_of_point, k);
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
  if (parts) {
    parts[0] = rc == SBV_OK ? h->result_host[0] : NAN;
    parts[1] = h->result_host[1];
    parts[2] = h->result_host[2];
    parts[3] = h->result_host[3];
  }
  return rc;
}

int sbv_set_shard(sbv_handle h, int32_t rank, int32_t world) {
  if (!h || world < 1 || rank < 0 || rank >= world) return SBV_ERR_ARG;
  if (h->prepared) return fail(h, SBV_ERR_STATE, "sbv_set_shard must precede sbv_prepare_h");
  if (h->comm) {
    ncclCommDestroy(h->comm);
    h->comm = nullptr;
  }
  h->rank = rank;
  h->world = world;
  return SBV_OK;
}

int sbv_block_grads(sbv_handle h, double *grads) {
  if (!h || !grads) return SBV_ERR_ARG;
  if (!h->prepared || h->grad_gen != h->prep_gen)
    return fail(h, SBV_ERR_STATE, "sbv_block_grads needs a successful sbv_loglik_grad after the last prepare");
  CU(cudaSetDevice(h->device));
  CU(cudaMemcpyAsync(grads, h->grads, (size_t)h->k_local * (h->d + 2) * sizeof(double), cudaMemcpyDefault,
                     h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return SBV_OK;
}

int sbv_set_graph(sbv_handle h, int32_t enable) {
  if (!h || enable < 0 || enable > 1) return SBV_ERR_ARG;
  h->use_graph = enable;
  return SBV_OK;
}

int sbv_partials_size(sbv_handle h, int64_t *count) {
  if (!h || !count) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "not prepared");
  *count = h->ncl_pad * 8;
  return SBV_OK;
}

int sbv_loglik_partials(sbv_handle h, const double *y, const double *theta, double *partials) {
  if (!h) return SBV_ERR_ARG;
  if (!partials) return fail(h, SBV_ERR_ARG, "partials is NULL");
  return run_loglik(h, y, theta, partials);
}

int sbv_reduce_partials(sbv_handle h, const double *all_partials, double *parts) {
  if (!h) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "not prepared");
  if (!all_partials || !parts) return fail(h, SBV_ERR_ARG, "NULL argument");
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t cnt = (size_t)h->world * h->ncl_pad * 8;
  double *dst = h->chunk_local;
  if (h->world > 1) {
    CU(ensure(h->chunk_all, (int64_t)cnt, h->cap));
    dst = h->chunk_all;
  }
  CU(cudaMemcpyAsync(dst, all_partials, cnt * sizeof(double), cudaMemcpyDefault, st));
  CU(launch_final_reduce(*h, st));
  CU(cudaMemcpyAsync(h->result_host, h->result, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  parts[0] = h->result_host[4] > 0 ? NAN : h->result_host[0];
  parts[1] = h->result_host[1];
  parts[2] = h->result_host[2];
  parts[3] = h->result_host[3];
  if (h->result_host[4] > 0) {
    h->err_block = (int64_t)h->result_host[5];
    h->err_stage = (int32_t)h->result_host[6];
    return fail(h, SBV_ERR_NOT_PD, "Cholesky factorisation failed (non-positive pivot)");
  }
  return SBV_OK;
}

int sbv_loglik(sbv_handle h, const double *y, const double *theta, double *ll) {
  if (!h) return SBV_ERR_ARG;
  if (!ll) return fail(h, SBV_ERR_ARG, "ll is NULL");
  int rc = run_loglik(h, y, theta);
  *ll = rc == SBV_OK ? h->result_host[0] : NAN;
  return rc;
}

// ell and d ell / d (sigma2, beta, tau2).  H8 runs in its
// factor-keeping mode over batches of blocks (LPT order) that fit the
// per-block factor copies in SBV_GRAD_BATCH_GB (default 16 GB), each batch
// followed by the gradient kernel; then the usual H9 reduction for ell and a
// fixed-order sum of the per-block gradients.
int sbv_loglik_grad(sbv_handle h, const double *y, const double *theta, double *ll, double *grad) {
  if (!h) return SBV_ERR_ARG;
  if (!ll || !grad) return fail(h, SBV_ERR_ARG, "ll or grad is NULL");
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "sbv_loglik_grad before sbv_prepare");
  if (!y) return fail(h, SBV_ERR_ARG, "y is NULL");
  int rc = validate_theta(h, theta);
  if (rc) return rc;
  const int d = h->d, P = d + 2;
  const double nu = theta[d + 1];
  if (!(nu == 0.5 || nu == 1.5 || nu == 2.5 || nu == 3.5))
    return fail(h, SBV_ERR_UNSUPPORTED, "the gradient needs nu in {0.5, 1.5, 2.5, 3.5} (nu is held fixed)");
  if (h->world > 1) return fail(h, SBV_ERR_UNSUPPORTED, "the gradient runs on one GPU (world = 1)");
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  auto &cap = h->cap;
  const double *yd = y;
  if (!is_device_ptr(y)) {
    CU(cudaMemcpyAsync(h->ybuf, y, h->n * sizeof(double), cudaMemcpyHostToDevice, st));
    yd = h->ybuf;
  }
  Timer tm(h, 0);
  CU(launch_stage_eval(yd, h->perm, h->n, h->yperm, st));
  tm.mark("H7_stage");
  // batches of the LPT order whose factor copies fit the budget
  double gb = 16.0;
  if (const char *e = getenv("SBV_GRAD_BATCH_GB")) gb = atof(e);
  const int64_t budget = (int64_t)(gb * 1e9 / sizeof(double));
  std::vector<int64_t> lgo(h->k_local, 0);
  int64_t maxbatch = 0;
  {
    int64_t acc = 0;
    for (int64_t it = 0; it < h->k_local; it++) {
      const int64_t Nb = h->Nt[h->order_h[it]];
      const int64_t sz = (Nb + 1) * Nb;
      if (acc > 0 && acc + sz > budget) {
        maxbatch = std::max(maxbatch, acc);
        acc = 0;
      }
      lgo[h->order_h[it]] = acc;
      acc += sz;
    }
    maxbatch = std::max(maxbatch, acc);
  }
  CU(ensure(h->Lg, std::max<int64_t>(maxbatch, 1), cap));
  CU(ensure(h->lg_off, std::max<int64_t>(h->k_local, 1), cap));
  CU(cudaMemcpyAsync(h->lg_off, lgo.data(), h->k_local * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  int max_b = 1;
  for (int64_t li = 0; li < h->k_local; li++) max_b = std::max(max_b, h->Nt[li] - std::min<int32_t>(h->m, h->Nt[li]));
  // Z row stride: round4(b) contraction columns + the at column, in 32-column units
  const int bpad_max = ((((h->max_bs + 3) & ~3) + 1) + 31) & ~31;
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  const int gnw = grad_shape(h->k_local, sms);
  const int ggrid = (int)std::min<int64_t>(grad_grid(theta[d + 1], d, std::max(h->max_N, 1), sms, gnw),
                                           std::max<int64_t>(h->k_local, 1));
  CU(ensure(h->zws, (int64_t)ggrid * std::max(h->max_N, 1) * std::max(bpad_max, 32), cap));
  CU(ensure(h->grads, std::max<int64_t>(h->k_local, 1) * P, cap));
  CU(ensure(h->gsum, P, cap));
  // batches: contiguous ranges [i0, i1) of the LPT order
  int64_t i0 = 0;
  while (i0 < h->k_local) {
    int64_t i1 = i0 + 1;
    while (i1 < h->k_local && lgo[h->order_h[i1]] != 0) i1++;
    H8Problem pb{};
    pb.Xp = h->Xperm;
    pb.yperm = h->yperm;
    pb.off = h->off;
    pb.nbr = h->nbr;
    pb.cnt = h->cnt;
    pb.local_blocks = h->local_blocks;
    pb.work_order = h->work_order + i0;
    pb.k_local = i1 - i0;
    pb.m = h->m;
    pb.max_N = h->max_N;
    pb.grid = (int)std::min<int64_t>(h->h8_grid, i1 - i0);
    pb.smem = h->h8_smem;
    pb.ws = h->ws;
    pb.ws_per_cta = h->ws_per_cta;
    pb.terms = h->terms;
    pb.quads = h->quads;
    pb.logdets = h->logdets;
    pb.status = h->status;
    pb.predict = 2;
    pb.n_big = std::max<int64_t>(0, std::min<int64_t>(h->h8_n_big, i1) - i0);
    pb.max_N_small = h->h8_max_N_small;
    pb.grid_small = h->h8_grid_small;
    pb.Lg = h->Lg;
    pb.lg_off = h->lg_off;
    CU(launch_h8_problem(pb, d, theta, h->queue, st));
    tm.mark("H8_keep_factor");
    GradLaunch gl{};
    gl.Lg = h->Lg;
    gl.lg_off = h->lg_off;
    gl.Xp = h->Xperm;
    gl.off = h->off;
    gl.nbr = h->nbr;
    gl.cnt = h->cnt;
    gl.local_blocks = h->local_blocks;
    gl.items = h->work_order + i0;
    gl.n_items = i1 - i0;
    gl.m = h->m;
    gl.d = d;
    gl.max_N = std::max(h->max_N, 1);
    gl.bpad_max = std::max(bpad_max, 32);
    gl.grid = (int)std::min<int64_t>(ggrid, i1 - i0);
    gl.nw = gnw;
    gl.theta = theta;
    gl.zws = h->zws;
    gl.queue = h->queue;
    gl.grads = h->grads;
    CU(launch_grad(gl, st));
    tm.mark("N3_grad");
    if (const char *dump = getenv("SBV_GRAD_DUMP")) {  // debugging aid: Lg of the first batch + per-block grads
      if (i0 == 0) {
        CU(cudaStreamSynchronize(st));
        std::vector<double> hl((size_t)maxbatch), hg((size_t)h->k_local * P);
        CU(cudaMemcpy(hl.data(), h->Lg, hl.size() * sizeof(double), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(hg.data(), h->grads, hg.size() * sizeof(double), cudaMemcpyDeviceToHost));
        if (FILE *fp = fopen(dump, "wb")) {
          fwrite(hl.data(), sizeof(double), hl.size(), fp);
          fwrite(hg.data(), sizeof(double), hg.size(), fp);
          fwrite(lgo.data(), sizeof(int64_t), lgo.size(), fp);
          fclose(fp);
        }
      }
    }
    i0 = i1;
  }
  CU(launch_reduce_chunks(*h, st));
  CU(launch_final_reduce(*h, st));
  CU(launch_grad_sum(h->grads, h->k_local, P, h->gsum, st));
  h->grad_gen = -1;
  CU(cudaMemcpyAsync(h->result_host, h->result, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(grad, h->gsum, P * sizeof(double), cudaMemcpyDefault, st));
  tm.mark("H9_grad_sums_d2h");
  CU(cudaStreamSynchronize(st));
  tm.finish();
  if (h->result_host[4] > 0) {
    h->err_block = (int64_t)h->result_host[5];
    h->err_stage = (int32_t)h->result_host[6];
    *ll = NAN;
    return fail(h, SBV_ERR_NOT_PD, "Cholesky factorisation failed (non-positive pivot)");
  }
  *ll = h->result_host[0];
  h->grad_gen = h->prep_gen;
  return SBV_OK;
}

int sbv_block_terms(sbv_handle h, const double *y, const double *theta, double *terms,
                    double *quad, double *logdet) {
  if (!h) return SBV_ERR_ARG;
  std::vector<double> part;  // sharded without a communicator: stop after H9
  if (h->prepared && h->world > 1 && !h->comm) part.resize((size_t)h->ncl_pad * 8 + 1);
  int rc = run_loglik(h, y, theta, part.empty() ? nullptr : part.data());
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
    if (r2) {
      cudaFreeAsync(tmp, st);
      return r2;
    }
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
  cudaSetDevice(h->device);
  resolve_stage_times(h, prep);
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


// ------------------------------------------------------------------ prediction (N2)
// Eq.3 with Sec.4.1 per test block and
// Sec.5.5.  Test blocks: the same anchors + RAC (H2-H5) on the
// scaled test inputs; conditioning sets: exact m_pred-NN of the test-block
// centroid over ALL training points (prediction mode) on the training
// grid levels built by prepare; per block: the fused H8 kernel in prediction
// mode (border values 0 on the test rows), whose epilogue reads mean and
// variance off the factor.
int sbv_predict(sbv_handle h, const double *Xs, int64_t ns, int32_t bs_pred, int32_t m_pred,
                const double *y, const double *theta, double *mean, double *var) {
  if (!h) return SBV_ERR_ARG;
  if (!h->prepared) return fail(h, SBV_ERR_STATE, "sbv_predict before sbv_prepare");
  if (!Xs || !y || !mean || !var) return fail(h, SBV_ERR_ARG, "NULL argument");
  if (ns < 1 || ns >= (int64_t(1) << 31)) return fail(h, SBV_ERR_ARG, "n_star out of range");
  if (bs_pred < 1 || bs_pred > ns) return fail(h, SBV_ERR_ARG, "bs_pred out of range [1, n_star]");
  if (m_pred < 0) return fail(h, SBV_ERR_ARG, "m_pred must be >= 0");
  if (!h->lv_valid || m_pred > knn_grid_max_m())
    return fail(h, SBV_ERR_UNSUPPORTED, "prediction needs the grid kNN (SBV_GRID=1, m, m_pred <= 960)");
  int rc = validate_theta(h, theta);
  if (rc) return rc;
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  auto &cap = h->cap;
  const int d = h->d;
  const int64_t n = h->n;
  const int64_t ks = std::max<int64_t>(1, (2 * ns + bs_pred) / (2 * (int64_t)bs_pred));
  h->ns = ns;
  h->ks = ks;
  h->bs_pred = bs_pred;
  h->m_pred = m_pred;
  // test inputs: device memory read in place, host memory staged
  const double *Xd = Xs;
  if (!is_device_ptr(Xs)) {
    CU(ensure(h->Xq, ns * d, cap));
    CU(cudaMemcpyAsync(h->Xq, Xs, ns * d * sizeof(double), cudaMemcpyHostToDevice, st));
    Xd = h->Xq;
  }
  CU(cudaMemsetAsync(h->flag, 0, sizeof(int), st));
  k_check_finite<<<grid_for(ns * d), 256, 0, st>>>(Xd, ns * d, h->flag);
  CU(cudaMemcpyAsync(h->flag_host, h->flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(ensure(h->Sq, ns * d, cap));
  CU(launch_scale(Xd, ns, d, h->scale.data(), h->Sq, st));
  // test blocks: anchors (same seed), grid RAC, layout, centroids
  CU(ensure(h->q_anchors, ks, cap));
  CU(select_anchors_fast(ns, ks, h->seed, h->q_anchors, h->flag + 1, st));
  CU(cudaMemcpyAsync(h->flag_host + 1, h->flag + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  double lo_hi[2 * SBV_MAX_D];
  CU(data_extents(h->Sq, ns, d, lo_hi, st));
  if (*h->flag_host) return fail(h, SBV_ERR_ARG, "X_star has non-finite entries");
  if (h->flag_host[1] != 0) CU(select_anchors(ns, ks, h->seed, h->q_anchors, nullptr, 0, st, nullptr));
  const GridDesc ga = make_grid(lo_hi, d, ks, 3.0);
  CU(ensure(h->qa_start, ga.ncells + 1, cap));
  CU(ensure(h->qa_list, ks, cap));
  CU(build_cells(h->Sq, h->q_anchors, ks, d, ga, h->qa_start, h->qa_list, st));
  CU(ensure(h->q_block_of, ns, cap));
  CU(launch_rac_grid(h->Sq, ns, 0, d, h->q_anchors, ks, ga, h->qa_start, h->qa_list, h->q_block_of, st));
  CU(anchor_own_block(h->q_anchors, ks, h->q_block_of, st));
  CU(ensure(h->q_perm, ns, cap));
  CU(ensure(h->q_off, ks + 1, cap));
  CU(build_layout(h->q_block_of, ns, ks, h->q_perm, h->q_off, nullptr, 0, st, nullptr));
  CU(ensure(h->Sqp, ns * d, cap));
  CU(launch_gather_rows(h->Sq, h->q_perm, ns, d, h->Sqp, st));
  CU(ensure(h->Xqp, ns * d, cap));
  CU(launch_gather_rows(Xd, h->q_perm, ns, d, h->Xqp, st));
  CU(ensure(h->Cq, ks * d, cap));
  CU(launch_centroids(h->Sqp, h->q_off, nullptr, ks, d, h->Cq, st));
  // prediction-mode NN over all n training points
  const int mm = m_pred > 0 ? m_pred : 1;
  CU(ensure(h->q_local, ks, cap));
  k_iota<<<grid_for(ks), 256, 0, st>>>(h->q_local, ks);
  CU(ensure(h->q_nbr, ks * mm, cap));
  CU(ensure(h->q_cnt, ks, cap));
  CU(launch_knn_grid(h->Sperm, h->perm, h->off, h->C, h->q_local, ks, d, m_pred, h->lv, h->p_start,
                     h->p_list, h->q_nbr, h->q_cnt, st, h->Cq, (int32_t)n));
  // training observations in block-major order (H7)
  const double *yd = y;
  if (!is_device_ptr(y)) {
    CU(cudaMemcpyAsync(h->ybuf, y, n * sizeof(double), cudaMemcpyHostToDevice, st));
    yd = h->ybuf;
  }
  CU(launch_stage_eval(yd, h->perm, n, h->yperm, st));
  // sizes -> LPT order, launch geometry
  std::vector<int64_t> qoff(ks + 1);
  std::vector<int32_t> qcnt(ks), order(ks);
  CU(cudaMemcpyAsync(qoff.data(), h->q_off, (ks + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(qcnt.data(), h->q_cnt, ks * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  int32_t maxN = 1;
  std::vector<int32_t> Nt(ks);
  for (int64_t t = 0; t < ks; t++) {
    Nt[t] = qcnt[t] + (int32_t)(qoff[t + 1] - qoff[t]);
    maxN = std::max(maxN, Nt[t]);
  }
  if (maxN > 4096) return fail(h, SBV_ERR_UNSUPPORTED, "m_pred + test block size > 4096");
  {
    std::vector<int64_t> bucket((size_t)maxN + 2, 0);
    for (int64_t t = 0; t < ks; t++) bucket[maxN - Nt[t] + 1]++;
    for (size_t b = 1; b < bucket.size(); b++) bucket[b] += bucket[b - 1];
    for (int64_t t = 0; t < ks; t++) order[bucket[maxN - Nt[t]]++] = (int32_t)t;
  }
  h->max_N_pred = maxN;
  CU(ensure(h->q_order, ks, cap));
  CU(cudaMemcpyAsync(h->q_order, order.data(), ks * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  const size_t smem = h8_smem_bytes(maxN, d);
  int smem_optin = 0, sms = 0;
  CU(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  if (smem + 1024 > (size_t)smem_optin)
    return fail(h, SBV_ERR_UNSUPPORTED, "test block + neighbour set too large for shared memory staging");
  const int per_sm = std::max(1, h8_max_ctas_per_sm(smem, d));
  const int grid = (int)std::min<int64_t>((int64_t)sms * per_sm, ks);
  int64_t q_n_big = 0;
  int q_max_N_small = 0, q_grid_small = 0;
  {
    std::vector<int32_t> No(ks);
    for (int64_t it = 0; it < ks; it++) No[it] = Nt[order[it]];
    h8_split_plan(No.data(), ks, d, sms, &q_n_big, &q_max_N_small, &q_grid_small);
  }
  const size_t ws_per_cta = h8_ws_doubles(maxN, d);
  CU(ensure(h->ws, (size_t)std::max(grid, q_grid_small) * ws_per_cta, cap));
  CU(ensure(h->q_mean, ns, cap));
  CU(ensure(h->q_var, ns, cap));
  CU(ensure(h->q_terms, ks, cap));
  CU(ensure(h->q_quads, ks, cap));
  CU(ensure(h->q_logdets, ks, cap));
  CU(ensure(h->q_status, ks, cap));
  CU(ensure(h->queue, 1, cap));
  H8Problem pb{};
  pb.Xp = h->Xperm;
  pb.yperm = h->yperm;
  pb.off = h->q_off;
  pb.nbr = h->q_nbr;
  pb.cnt = h->q_cnt;
  pb.local_blocks = h->q_local;
  pb.work_order = h->q_order;
  pb.k_local = ks;
  pb.m = m_pred;
  pb.max_N = maxN;
  pb.grid = grid;
  pb.smem = smem;
  pb.ws = h->ws;
  pb.ws_per_cta = ws_per_cta;
  pb.terms = h->q_terms;
  pb.quads = h->q_quads;
  pb.logdets = h->q_logdets;
  pb.status = h->q_status;
  pb.predict = 1;
  pb.n_big = q_n_big;
  pb.max_N_small = q_max_N_small;
  pb.grid_small = q_grid_small;
  pb.Xq = h->Xqp;
  pb.pmean = h->q_mean;
  pb.pvar = h->q_var;
  CU(launch_h8_problem(pb, d, theta, h->queue, st));
  // caller order
  double *tmp = nullptr;
  CU(cudaMallocAsync(&tmp, 2 * ns * sizeof(double), st));
  k_unpermute<<<grid_for(ns), 256, 0, st>>>(h->q_mean, h->q_perm, ns, tmp);
  k_unpermute<<<grid_for(ns), 256, 0, st>>>(h->q_var, h->q_perm, ns, tmp + ns);
  CU(cudaMemcpyAsync(mean, tmp, ns * sizeof(double), cudaMemcpyDefault, st));
  CU(cudaMemcpyAsync(var, tmp + ns, ns * sizeof(double), cudaMemcpyDefault, st));
  std::vector<int32_t> status(ks);
  CU(cudaMemcpyAsync(status.data(), h->q_status, ks * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(cudaFreeAsync(tmp, st));
  CU(cudaStreamSynchronize(st));
  for (int64_t t = 0; t < ks; t++)
    if (status[t] == 1) {  // Sigma_JJ not positive definite (the B x B factor is unused)
      h->err_block = t;
      h->err_stage = status[t];
      return fail(h, SBV_ERR_NOT_PD, "Cholesky failed in a test block (lowest index in err_block)");
    }
  return SBV_OK;
}

int sbv_get_prediction(sbv_handle h, int64_t *ks, int32_t *anchors, int32_t *block_of, int64_t *off,
                       int32_t *perm, int32_t *nbr, int32_t *cnt) {
  if (!h) return SBV_ERR_ARG;
  if (h->ks == 0) return fail(h, SBV_ERR_STATE, "no sbv_predict on this handle");
  if (ks) *ks = h->ks;
  int rc;
  if ((rc = copy_out(h, anchors, h->q_anchors, h->ks * sizeof(int32_t)))) return rc;
  if ((rc = copy_out(h, block_of, h->q_block_of, h->ns * sizeof(int32_t)))) return rc;
  if ((rc = copy_out(h, off, h->q_off, (h->ks + 1) * sizeof(int64_t)))) return rc;
  if ((rc = copy_out(h, perm, h->q_perm, h->ns * sizeof(int32_t)))) return rc;
  if (nbr || cnt) {  // conditioning sets as ORIGINAL training indices (-1 padded)
    cudaStream_t st = h->stream;
    const int mp = h->m_pred;
    int32_t *tn = nullptr, *tc = nullptr;
    CU(cudaMallocAsync(&tn, std::max<int64_t>(h->ks * mp, 1) * sizeof(int32_t), st));
    CU(cudaMallocAsync(&tc, h->ks * sizeof(int32_t), st));
    k_nbr_to_orig<<<grid_for(std::max<int64_t>(h->ks * mp, h->ks)), 256, 0, st>>>(
        h->q_nbr, h->q_cnt, h->perm, h->q_local, h->ks, mp, tn, tc);
    rc = copy_out(h, nbr, tn, h->ks * mp * sizeof(int32_t));
    if (!rc) rc = copy_out(h, cnt, tc, h->ks * sizeof(int32_t));
    cudaFreeAsync(tn, st);
    cudaFreeAsync(tc, st);
    if (rc) return rc;
  }
  return SBV_OK;
}

int sbv_simulate(sbv_handle h, const double *mean, const double *var, int64_t ns, int32_t n_sim,
                 uint64_t seed, double ci_level, double *sim_mean, double *sim_sd, double *ci_lo,
                 double *ci_hi) {
  if (!h) return SBV_ERR_ARG;
  if (!mean || !var || !sim_mean || !sim_sd || !ci_lo || !ci_hi) return fail(h, SBV_ERR_ARG, "NULL argument");
  if (ns < 1 || n_sim < 2) return fail(h, SBV_ERR_ARG, "n_star >= 1 and n_sim >= 2 required");
  if (!(ci_level > 0.0 && ci_level < 1.0)) return fail(h, SBV_ERR_ARG, "ci_level must be in (0, 1)");
  CU(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  double *buf = nullptr;
  CU(cudaMallocAsync(&buf, 6 * ns * sizeof(double), st));
  CU(cudaMemcpyAsync(buf, mean, ns * sizeof(double), cudaMemcpyDefault, st));
  CU(cudaMemcpyAsync(buf + ns, var, ns * sizeof(double), cudaMemcpyDefault, st));
  std::vector<double> vh(ns);
  CU(cudaMemcpyAsync(vh.data(), buf + ns, ns * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (int64_t j = 0; j < ns; j++)
    if (!(vh[j] >= 0.0)) {
      cudaFreeAsync(buf, st);
      return fail(h, SBV_ERR_ARG, "negative or NaN variance (clamp tiny negatives upstream)");
    }
  k_simulate<<<grid_for(ns), 128, 0, st>>>(buf, buf + ns, ns, n_sim, seed, ci_level, buf + 2 * ns,
                                           buf + 3 * ns, buf + 4 * ns, buf + 5 * ns);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(sim_mean, buf + 2 * ns, ns * sizeof(double), cudaMemcpyDefault, st));
  CU(cudaMemcpyAsync(sim_sd, buf + 3 * ns, ns * sizeof(double), cudaMemcpyDefault, st));
  CU(cudaMemcpyAsync(ci_lo, buf + 4 * ns, ns * sizeof(double), cudaMemcpyDefault, st));
  CU(cudaMemcpyAsync(ci_hi, buf + 5 * ns, ns * sizeof(double), cudaMemcpyDefault, st));
  CU(cudaFreeAsync(buf, st));
  CU(cudaStreamSynchronize(st));
  return SBV_OK;
}

}  // extern "C"
