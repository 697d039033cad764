// sbv_internal.cuh — shared declarations of libsbv's CUDA translation units.
// Product path only; nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/sbv.h"

namespace sbv {

constexpr int kPanel = 32;       // H8 panel width (columns per left-looking step)
constexpr int kChunkBlocks = 64; // blocks per reduction / shard chunk
constexpr int kMaxStages = 16;

// ---- grid-filtered exact search (grid.cu): geometry types
struct GridDesc {
  int G;          // grid dimensions (<= 3): the scaled dims of largest extent
  int dim[3];     // which input dimensions
  double lo[3];   // data minimum per grid dim
  double h[3];    // cell edge per grid dim
  int nc[3];      // cells per grid dim
  int stride[3];  // linear cell index strides
  int64_t ncells;
};
// Prefix-level grids for the kNN (H6): level l buckets the block-major
// positions [0, P[l]) (P halves from n), so a query whose admissible prefix is
// [0, A) searches the smallest level with P >= A, where at least half of the
// indexed points are admissible.  All levels share one list / start array.
constexpr int kMaxLevels = 16;
struct KnnLevels {
  int nl;
  int32_t direct_max;               // prefixes A <= direct_max are scanned directly
  int32_t P[kMaxLevels];            // decreasing
  int64_t cell_off[kMaxLevels + 1]; // level l cells start at cell_off[l] in `start`
  int64_t list_off[kMaxLevels + 1]; // level l items occupy list[list_off[l], list_off[l+1])
  GridDesc g[kMaxLevels];
};
struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t seed = 3;
  int profile = 0;
  int debug = 0;  // SBV_DEBUG=1: host-side stage trace on stderr
  // comm
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // problem
  bool prepared = false;
  int64_t n = 0;
  int32_t d = 0, bs = 0, m = 0;
  int64_t k = 0;  // number of blocks bc
  std::vector<double> scale;
  // device state (prepare)
  double *X = nullptr;        // n x d original inputs (library copy)
  double *S = nullptr;        // n x d scaled by `scale` (original order)
  double *Sperm = nullptr;    // n x d scaled, block-major
  int32_t *anchors = nullptr; // k
  int32_t *block_of = nullptr;// n
  int32_t *perm = nullptr;    // n, block-major -> original index
  int64_t *off = nullptr;     // k+1
  double *C = nullptr;        // k x d centroids
  int32_t *nbr = nullptr;     // k_local x m, positions in block-major order, -1 pad
  int32_t *cnt = nullptr;     // k_local
  int32_t *local_blocks = nullptr; // k_local zeta ids of this rank's blocks (ascending)
  int32_t *work_order = nullptr;   // k_local indices into local_blocks, LPT order
  int64_t k_local = 0;
  int64_t n_chunks = 0, n_chunks_local = 0;
  int64_t ncl_pad = 0;  // chunk-partial slots per rank (allgather layout)
  int32_t max_N = 0, min_bs = 0, max_bs = 0;
  double flops = 0, entries = 0, knn_pairs = 0, rac_pairs = 0, h8_bytes = 0;
  // per-eval buffers
  double *Xperm = nullptr;    // n x d block-major ORIGINAL inputs (prepare)
  double *yperm = nullptr;    // n block-major
  double *ybuf = nullptr;     // n original order (host y staging)
  double *terms = nullptr, *quads = nullptr, *logdets = nullptr; // k_local
  int32_t *status = nullptr;  // k_local (0 ok, 1/2 failing stage)
  double *chunk_local = nullptr;  // n_chunks_local_pad x 4
  double *chunk_all = nullptr;    // world * n_chunks_local_pad x 4
  double *result = nullptr;       // 8 doubles: ell, quad, logdet, npts, nfail, fail_block, fail_stage, -
  double *result_host = nullptr;  // pinned 8 doubles
  int32_t *a_start = nullptr, *a_list = nullptr;  // anchor grid (RAC)
  int32_t *p_start = nullptr, *p_list = nullptr;  // point grid over block-major positions (kNN)
  int use_grid = 1;                               // SBV_GRID=0 forces the brute-force kernels
  int *flag = nullptr;            // device: non-finite input flag
  int *flag_host = nullptr;       // pinned mirror
  char *pin = nullptr;            // pinned staging of prepare's host-side tables
  cudaEvent_t ev_sizes = nullptr; // prepare: block offsets on the host
  cudaEvent_t ev_pin = nullptr;   // prepare: last async H2D copy out of the pinned staging
  int given_blocks = 0;           // 1: the caller supplied the block partition (no H2/H3)
  size_t pin_cap = 0;
  unsigned int *queue = nullptr;  // work counter
  double *ws = nullptr;           // H8 per-CTA L workspaces
  std::vector<int32_t> Nt;        // N_t = m_t + bs_t per local block (prepare)
  std::vector<int32_t> order_h;   // LPT work order (host copy)
  double *Lg = nullptr;           // gradient: per-block factor copies (one batch)
  int64_t *lg_off = nullptr;      // gradient: [k_local] offsets into Lg
  double *zws = nullptr;          // gradient: per-CTA Z scratch
  double *grads = nullptr;        // gradient: [k_local][d+2]
  double *gsum = nullptr;         // gradient: [d+2]
  // CUDA-graph replay of sbv_loglik (sbv_set_graph): captured once per
  // (y pointer, nu, prepare), theta through a pinned host -> device copy node
  int64_t grad_gen = -1;          // prep_gen of the last successful sbv_loglik_grad (sbv_block_grads)
  int use_graph = 0;
  int64_t prep_gen = 0;           // bumped by every prepare (invalidates the graph)
  cudaStream_t g_stream = nullptr;
  cudaGraphExec_t g_exec = nullptr;
  const double *g_y = nullptr;
  double g_nu = 0.0;
  int64_t g_gen = -1;
  double *theta_pin = nullptr;    // pinned SBV_MAX_D + 3
  double *theta_dev = nullptr;    // device SBV_MAX_D + 3
  size_t ws_per_cta = 0;
  int h8_grid = 0;
  int64_t h8_n_big = 0;           // split H8 launch (h8_split_plan)
  int h8_max_N_small = 0, h8_grid_small = 0;
  int h8_small = 0;               // 1: loglik launches use the 4-warp kernel (h8_use_small)
  size_t h8_smem = 0;
  size_t occ_smem = 0;  // cached occupancy query
  int occ_per_sm = 0;
  int occ_small = 0;    // cached occupancy of the 4-warp kernel
  int occ_d = 0;
  KnnLevels lv{};                 // kNN prefix-level grids of the training set (prepare)
  bool lv_valid = false;
  // prediction state (sbv_predict)
  int64_t ns = 0, ks = 0;         // test points, test blocks
  int32_t bs_pred = 0, m_pred = 0, max_N_pred = 0;
  double *Xq = nullptr, *Sq = nullptr, *Sqp = nullptr, *Xqp = nullptr, *Cq = nullptr;
  int32_t *q_anchors = nullptr, *q_block_of = nullptr, *q_perm = nullptr, *q_nbr = nullptr, *q_cnt = nullptr;
  int32_t *q_local = nullptr, *q_order = nullptr, *q_status = nullptr;
  int64_t *q_off = nullptr;
  int32_t *qa_start = nullptr, *qa_list = nullptr;
  double *q_mean = nullptr, *q_var = nullptr, *q_terms = nullptr, *q_quads = nullptr, *q_logdets = nullptr;
  std::unordered_map<void *, size_t> cap;  // device buffer capacities (bytes)
  // errors
  int64_t err_block = -1;
  int32_t err_stage = 0;
  std::string err_msg;
  // profiling
  // per-stage events of the last prepare [0] / loglik [1]; resolved lazily by
  // sbv_stage_times, so profiling adds no host synchronisation to the calls
  cudaEvent_t ev[2][kMaxStages + 1] = {};
  int ev_pending[2] = {0, 0};
  int n_ev_prep = 0, n_ev_llh = 0;
  double t_prep[kMaxStages] = {}, t_llh[kMaxStages] = {};
  const char *name_prep[kMaxStages] = {}, *name_llh[kMaxStages] = {};
};

// ---- grid-filtered exact search (grid.cu)
KnnLevels make_knn_levels(const double *lo_hi, int d, int64_t n, int m);
cudaError_t build_knn_levels(const double *Sperm, int d, const KnnLevels &lv, int32_t *start,
                             int32_t *list, cudaStream_t st);
cudaError_t data_extents(const double *S, int64_t n, int d, double *lo_hi_host, cudaStream_t st);
GridDesc make_grid(const double *lo_hi, int d, int64_t count, double per_cell);
cudaError_t build_cells(const double *S, const int32_t *rows, int64_t count, int d, const GridDesc &g,
                        int32_t *start, int32_t *list, cudaStream_t st);
cudaError_t launch_rac_grid(const double *S, int64_t n, int64_t i0, int d, const int32_t *anchors, int64_t k,
                            const GridDesc &g, const int32_t *a_start, const int32_t *a_list,
                            int32_t *block_of, cudaStream_t st);
cudaError_t launch_knn_grid(const double *Sperm, const int32_t *perm, const int64_t *off,
                            const double *C, const int32_t *local_blocks, int64_t k_local, int d,
                            int m, const KnnLevels &lv, const int32_t *c_start, const int32_t *c_list,
                            int32_t *nbr, int32_t *cnt, cudaStream_t st, const double *Cq = nullptr,
                            int32_t A_all = 0);
int knn_grid_max_m();
cudaError_t anchor_own_block(const int32_t *anchors, int64_t k, int32_t *block_of, cudaStream_t st);

// ---- prepare kernels (prep_kernels.cu)
cudaError_t launch_scale(const double *X, int64_t n, int d, const double *scale_host, double *S,
                         cudaStream_t st);
cudaError_t select_anchors(int64_t n, int64_t k, uint64_t seed, int32_t *anchors, void *tmp,
                           size_t tmp_bytes, cudaStream_t st, size_t *tmp_needed);
cudaError_t select_anchors_fast(int64_t n, int64_t k, uint64_t seed, int32_t *anchors, int *bad,
                                cudaStream_t st);
cudaError_t launch_rac(const double *S, int64_t n, int d, const int32_t *anchors, int64_t k,
                       int32_t *block_of, cudaStream_t st);
cudaError_t build_layout(const int32_t *block_of, int64_t n, int64_t k, int32_t *perm,
                         int64_t *off, void *tmp, size_t tmp_bytes, cudaStream_t st,
                         size_t *tmp_needed);
cudaError_t launch_gather_rows(const double *S, const int32_t *perm, int64_t n, int d,
                               double *Sperm, cudaStream_t st);
cudaError_t launch_centroids(const double *Sperm, const int64_t *off, const int32_t *blocks,
                             int64_t k, int d, double *C, cudaStream_t st);
cudaError_t launch_knn(const double *Sperm, const int32_t *perm, const int64_t *off,
                       const double *C, const int32_t *local_blocks, int64_t k_local, int d,
                       int m, int32_t *nbr, int32_t *cnt, cudaStream_t st);

// ---- per-eval kernels (llh_kernel.cu)
cudaError_t launch_stage_eval(const double *y, const int32_t *perm, int64_t n, double *yperm,
                              cudaStream_t st);
size_t h8_smem_bytes(int max_N, int d);
int h8_two_cta_cap(int d);
void h8_split_plan(const int32_t *Nt_order, int64_t k, int d, int sms, int64_t *n_big, int *max_N_small,
                   int *grid_small);
size_t h8_ws_doubles(int max_N, int d);
int h8_max_ctas_per_sm(size_t smem, int d);
bool h8_use_small(int max_N);
int h8_small_ctas_per_sm(size_t smem, int d);
cudaError_t launch_h8(const Ctx &c, const double *theta_host, cudaStream_t st,
                      const double *theta_dev = nullptr);
// One H8 launch over an explicit set of blocks (estimation or prediction mode)
struct H8Problem {
  const double *Xp, *yperm;        // training inputs / observations, block-major
  const int64_t *off;              // block offsets (training blocks, or test blocks in prediction)
  const int32_t *nbr, *cnt;        // conditioning sets (training block-major positions)
  const int32_t *local_blocks, *work_order;
  int64_t k_local;
  int m, max_N, grid;
  size_t smem;
  double *ws;
  size_t ws_per_cta;
  double *terms, *quads, *logdets;
  int32_t *status;
  int predict;                     // 1: B rows are test points Xq, outputs pmean / pvar; 2: keep L (gradient)
  int64_t n_big = 0;               // split launch: the first n_big work items (N > 2-CTA cap) alone
  int max_N_small = 0, grid_small = 0;
  const double *theta_d = nullptr; // graph replay: theta in device memory (H8Args::theta_d)
  int small = 0;                   // all blocks small: the 4-warp loglik kernel (h8_use_small)
  double *Lg = nullptr;            // predict == 2: per-block factor copies
  const int64_t *lg_off = nullptr;
  const double *Xq;
  double *pmean, *pvar;
};
cudaError_t launch_h8_problem(const H8Problem &pb, int d, const double *theta_host, unsigned int *queue,
                              cudaStream_t st);
// ---- gradient (grad_kernel.cu)
struct GradLaunch {
  const double *Lg;
  const int64_t *lg_off;
  const double *Xp;
  const int64_t *off;
  const int32_t *nbr, *cnt, *local_blocks, *items;
  int64_t n_items;
  int m, d, max_N, bpad_max, grid;
  int nw;  // warps per CTA of k_grad (grad_shape)
  const double *theta;  // host
  double *zws;
  unsigned int *queue;
  double *grads;
};
size_t grad_smem_bytes(int max_N, int d, int nw);
int grad_shape(int64_t k, int sms);
int grad_grid(double nu, int d, int max_N, int sms, int nw);
cudaError_t launch_grad(const GradLaunch &gl, cudaStream_t st);
cudaError_t launch_grad_sum(const double *grads, int64_t k_local, int P, double *out, cudaStream_t st);
cudaError_t launch_reduce_chunks(const Ctx &c, cudaStream_t st);
cudaError_t launch_final_reduce(const Ctx &c, cudaStream_t st);

}  // namespace sbv
