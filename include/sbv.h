/*
 * sbv.h — C ABI of libsbv, the B200 (sm_100a) implementation of the Scaled
 * Block Vecchia log-likelihood hot path (arXiv 2504.12004).
 *
 * The calls follow the paper's statement of the problem, Alg.1 (PAPER.md
 * P:253-288): "Input: data {x_i, y_i}, dimension d, total block count K,
 * nearest neighbors m_est, workers P, covariance function K_theta, scaling
 * parameters beta.  Output: the log-likelihood".  sbv_prepare performs
 * Alg.1 Steps 1-3 (scaling Alg.2, Random Anchor Clustering Alg.3
 * P:344-360, random block order P:269, m-NN search Alg.4);
 * sbv_loglik performs Step 4 (batched block log-likelihoods Alg.5
 * P:462-499) and Step 5 (reduction across workers).
 *
 * Conventions for every call:
 *  - Every entry point returns an sbv_status; nothing throws across the ABI.
 *    On failure the handle (if any) keeps a message for sbv_last_error.
 *  - Pointers to bulk arrays (X, y, outputs of sbv_get_*) may be HOST or
 *    DEVICE pointers: the library inspects them with cudaPointerGetAttributes
 *    and copies host data to/from the device itself.  They are read/written
 *    only during the call; the caller keeps ownership.
 *  - Small parameter arrays (scale, theta) are always host arrays.
 *  - All FP data is IEEE binary64, row-major, contiguous.
 *  - A handle is bound to the CUDA device current at sbv_create / sbv_prepare
 *    and to the stream given in sbv_opts (NULL = the legacy default stream).
 *    It is not thread-safe: one handle per host thread / stream.
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one returns SBV_ERR_CUDA.
 */
#ifndef SBV_H_
#define SBV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBV_ABI_VERSION 2
#define SBV_MAX_D 64    /* 1 <= d <= 64 */

typedef struct sbv_ctx *sbv_handle; /* opaque; owned by the library */

typedef enum {
  SBV_OK = 0,
  SBV_ERR_ARG = 1,         /* invalid argument (sizes, NaN/Inf, beta<=0, ...) */
  SBV_ERR_CUDA = 2,        /* CUDA runtime error or no device */
  SBV_ERR_OOM = 3,         /* device allocation failed */
  SBV_ERR_NOT_PD = 4,      /* a Cholesky pivot was <= 0: see sbv_last_error */
  SBV_ERR_UNSUPPORTED = 5, /* nu outside (0, 20], or shape beyond kernel limits */
  SBV_ERR_COMM = 6,        /* NCCL failure */
  SBV_ERR_STATE = 7        /* call out of order (e.g. loglik before prepare) */
} sbv_status;

typedef struct {
  uint64_t seed;   /* RAC anchor / block-order seed (Q9); default 3 */
  void *stream;    /* cudaStream_t for every launch of this handle; NULL = default */
  int32_t profile; /* 1 = record per-stage CUDA events (sbv_stage_times) */
} sbv_opts;

/* ---------------------------------------------------------------- lifecycle */

/* Create an empty handle on the current CUDA device.  opts may be NULL
 * (seed 3, default stream, no profiling). */
int sbv_create(const sbv_opts *opts, sbv_handle *out);

/* Free every device buffer and the NCCL communicator.  NULL is a no-op. */
void sbv_destroy(sbv_handle h);

/* Multi-GPU (one process per GPU, Alg.1 "workers P"): attach an NCCL
 * communicator made from a 128-byte ncclUniqueId that rank 0 obtained with
 * sbv_comm_unique_id and broadcast.  Must precede sbv_prepare_h.  Blocks are
 * then sharded across ranks (64-block chunks dealt round-robin by zeta
 * position); X and y are replicated on every rank; the only collective of
 * the path is one ncclAllGather of the per-chunk partial sums (Alg.1
 * Step 5), which keeps ell bit-identical for every world size. */
int sbv_comm_unique_id(void *id128);

/* Host-only (no device needed): the zeta ids of the blocks rank `rank` of
 * `world` owns, ascending: 64-block chunks c = rank, rank + world, ...
 * blocks may be NULL (count only); capacity must be >= bc/world + 64.
 * Errors: SBV_ERR_ARG. */
int sbv_shard_blocks(int64_t bc, int32_t rank, int32_t world, int32_t *blocks, int64_t *count);
int sbv_comm_init(sbv_handle h, const void *nccl_unique_id, int32_t rank, int32_t world);

/* ---------------------------------------------------------------- prepare */

/* Alg.1 Steps 1-3 on device:
 *   H1  S = X / scale (IEEE division per element; Alg.2, Eq.5)
 *   H2  k = max(1, floor(n/bs + 1/2)) anchors = the k points with smallest
 *       (splitmix64(seed, i), i); anchor rank r seeds block r whose zeta
 *       position is r (Alg.3, Alg.1; Q8, Q9)
 *   H3  RAC: every point joins the block of its nearest anchor in scaled
 *       space, ties to the lowest rank (Alg.3)
 *   H4  block-major layout, members in ascending original index
 *   H5  centroids = member means in scaled space (Alg.4)
 *   H6  exact m-NN of each block centroid among the points of strictly
 *       earlier blocks, ordered by (squared distance, original index)
 *       (Eq.2, Alg.4; Q5, Q6, Q13)
 * X: n x d (host or device).  scale: host double[d], every entry > 0.
 * Requires 1 <= d <= SBV_MAX_D, 1 <= bs <= n, 0 <= m, n < 2^31, finite X.
 * Errors: SBV_ERR_ARG, SBV_ERR_OOM, SBV_ERR_CUDA, SBV_ERR_COMM. */
int sbv_prepare_h(sbv_handle h, const double *X, int64_t n, int32_t d, int32_t bs,
                  int32_t m, const double *scale);

/* Convenience: sbv_create(opts) + sbv_prepare_h.  On error *out is NULL. */
int sbv_prepare_ex(const double *X, int64_t n, int32_t d, int32_t bs, int32_t m,
                   const double *scale, const sbv_opts *opts, sbv_handle *out);

/* North-star form: sbv_prepare(X, n, d, bs, m, scale) with default options. */
int sbv_prepare(const double *X, int64_t n, int32_t d, int32_t bs, int32_t m,
                const double *scale, sbv_handle *out);

/* Alg.1 with the block partition GIVEN (Alg.1 takes the block count K as an
 * input; SURVEY 8(b) "block centroids given"): H2 (anchors) and H3 (RAC)
 * are skipped and block_of_point[i] in [0, k) is point i's block, whose zeta
 * position is its id (block 0 first).  H1 and H4-H6 run as in sbv_prepare_h
 * (centroids = member means of the given blocks, kNN over strictly earlier
 * blocks).  block_of_point: int32[n], host or device, read during the call.
 * Errors: SBV_ERR_ARG (NULL, k outside [1, n], an id outside [0, k), an empty
 * block, non-finite X / scale), otherwise as sbv_prepare_h.  sbv_get_anchors
 * returns -1 for every block of such a handle. */
int sbv_prepare_blocks(sbv_handle h, const double *X, int64_t n, int32_t d, int64_t k,
                       const int32_t *block_of_point, int32_t m, const double *scale);

/* ---------------------------------------------------------------- loglik */

/* Alg.1 Steps 4-5: ell(theta; y) = sum_t ell_t with, per block t (Alg.5):
 *   ell_t = -1/2 (v^T v + 2 sum_j log L'_jj) - (bs_t/2) log 2 pi
 * where L' = chol(Sigma_lk - Sigma'cross^T Sigma'cross) and
 * v = L'^{-1}(y_B - mu) (Q1, Q2), computed as one bordered
 * Cholesky of the joint (m_t + bs_t) covariance of [J_t; B_t].
 * Covariance: Eq.5-6 with theta's beta on the ORIGINAL inputs (Q11) and the
 * nugget tau2 on the diagonal only (Q3).
 * y: length n in original point order (host or device).
 * theta: host double[d+3] = {sigma2, beta_1..beta_d, nu, tau2}.
 * nu in {0.5, 1.5, 2.5, 3.5} uses the half-integer closed forms (Q4); any
 * other 0 < nu <= 20 evaluates Eq.6 with K_nu (Temme series / Steed
 * continued fraction), several times slower per entry.
 * *ll receives ell (NaN on SBV_ERR_NOT_PD).  Synchronous on the stream.
 * Errors: SBV_ERR_ARG (theta invalid), SBV_ERR_UNSUPPORTED (nu outside (0, 20]),
 * SBV_ERR_NOT_PD (lowest failing zeta block + stage via sbv_last_error),
 * SBV_ERR_STATE (no prepare), SBV_ERR_CUDA, SBV_ERR_COMM. */
int sbv_loglik(sbv_handle h, const double *y, const double *theta, double *ll);

/* SURVEY 8(f) NEXT row N3, the "gradient quantities" of P:453: ell and its
 * gradient with respect to (sigma2, beta_1..beta_d, tau2), nu held fixed
 * (Q28).  grad: host or device double[d+2] in that order.  Per
 * block, with L = chol(K([J_t; B_t])) and y' = L^-1 [y_J; y_B]:
 *   d ell_t / d theta_k = 1/2 sum_ij (at dl^T + dl at^T + dl dl^T - Z Z^T)_ij (dK_k)_ij,
 *   Z = L^-T E_B, dl = Z y'_B, at = [L11^-T y'_J; 0]
 * (Eq.1 P:156-158 differentiated for the joint minus the marginal of y_J).
 * One GPU only (world = 1).  Errors: as sbv_loglik, plus SBV_ERR_UNSUPPORTED
 * for nu outside {0.5, 1.5, 2.5, 3.5} or world > 1. */
int sbv_loglik_grad(sbv_handle h, const double *y, const double *theta, double *ll, double *grad);

/* The per-block gradients d ell_t / d (sigma2, beta_1..beta_d, tau2) of the
 * last successful sbv_loglik_grad (whose sum in block order is its grad):
 * host or device double[bc x (d+2)], row t = block t (zeta order).
 * Errors: SBV_ERR_STATE (no successful sbv_loglik_grad since the last
 * prepare), SBV_ERR_ARG, SBV_ERR_CUDA. */
int sbv_block_grads(sbv_handle h, double *grads);

/* CUDA-graph replay of sbv_loglik (the latency case, cfg1: P:752 names
 * per-call overhead as what limits small problems).  enable = 1: on one GPU
 * (world 1) with a DEVICE y and profiling off, sbv_loglik / sbv_loglik_parts
 * run H7 -> H8 -> H9 -> the 64-byte result copy as one graph launch, captured
 * on the first call for a given (y pointer, nu) after each prepare and
 * replayed afterwards; theta travels through a pinned host -> device copy
 * node, so a new theta needs no re-capture.  Same kernels, bit-identical
 * results; any other call shape takes the ordinary stream path.  The caller
 * must not free y while the handle may replay the graph on it.
 * Errors: SBV_ERR_ARG (enable not 0/1). */
int sbv_set_graph(sbv_handle h, int32_t enable);

/* As sbv_loglik, plus parts[0..3] = {ell, sum quad, sum logdet, #points}
 * (host double[4], may be NULL). */
int sbv_loglik_parts(sbv_handle h, const double *y, const double *theta, double *parts);

/* Per-block terms ell_t (double[bc], zeta order; host or device).  Blocks
 * owned by other ranks are written as NaN.  quad/logdet may be NULL. */
int sbv_block_terms(sbv_handle h, const double *y, const double *theta, double *terms,
                    double *quad, double *logdet);

/* Exchange by the caller (SURVEY 8(b)'s alternative to sbv_comm_init, e.g.
 * an MPI program, or one process driving several shards):
 *  - sbv_set_shard(h, rank, world): shard this handle's blocks exactly as
 *    sbv_comm_init would, without a communicator.  Must precede
 *    sbv_prepare_h; prepare then runs RAC over all points on this device.
 *    sbv_loglik on such a handle returns SBV_ERR_STATE.
 *  - sbv_partials_size: number of doubles of one rank's partials
 *    (= 8 x ceil(chunks / world); chunk = 64 zeta-consecutive blocks).
 *  - sbv_loglik_partials: Steps 4 and 5's per-rank part (H7-H9): this rank's
 *    chunk partial sums {sum ell_t, sum quad, sum logdet, #points, #failed,
 *    lowest failing block, its stage, 0} per local chunk, in the slot layout
 *    of the allgather (host or device buffer of sbv_partials_size doubles).
 *  - sbv_reduce_partials: Step 5: all ranks' partials concatenated
 *    in rank order (world x sbv_partials_size doubles, host or device) are
 *    summed in global chunk order with the fixed tree of sbv_loglik, so the
 *    result is bit-identical to a one-GPU sbv_loglik.  parts: host
 *    double[4] = {ell, sum quad, sum logdet, #points}.  Errors as sbv_loglik
 *    (SBV_ERR_NOT_PD with the lowest failing block in sbv_last_error). */
int sbv_set_shard(sbv_handle h, int32_t rank, int32_t world);
int sbv_partials_size(sbv_handle h, int64_t *count);
int sbv_loglik_partials(sbv_handle h, const double *y, const double *theta, double *partials);
int sbv_reduce_partials(sbv_handle h, const double *all_partials, double *parts);

/* ---------------------------------------------------------------- introspection */

int sbv_num_blocks(sbv_handle h, int64_t *bc);

/* anchors: int32[bc] original index of the anchor of block r (host or device). */
int sbv_get_anchors(sbv_handle h, int32_t *anchors);

/* block_of_point: int32[n]; off: int64[bc+1] (block t = perm[off[t]..off[t+1]));
 * perm: int32[n] original indices block-major; centroids: double[bc*d].
 * Any output may be NULL. */
int sbv_get_blocks(sbv_handle h, int32_t *block_of_point, int64_t *off, int32_t *perm,
                   double *centroids);

/* nbr: int32[bc*m] ORIGINAL point indices in kNN order, -1 padded; cnt:
 * int32[bc].  Rows of blocks owned by other ranks are all -1 / count -1. */
int sbv_get_neighbors(sbv_handle h, int32_t *nbr, int32_t *cnt);

/* Realised-size statistics of the prepared handle (this rank's blocks):
 * out[0] = algorithmic FP64 flops of one sbv_loglik (SURVEY 8(d) model,
 *          LAPACK conventions, summed over the realised (m_t, bs_t)),
 * out[1] = covariance entries generated per eval,
 * out[2] = max N_t = m_t + bs_t, out[3] = min bs_t, out[4] = max bs_t,
 * out[5] = number of local blocks, out[6] = kNN candidate pairs of prepare,
 * out[7] = RAC pairs of prepare, out[8] = algorithmic HBM bytes of one
 *          H8 launch (coordinates + y gathered + terms written). */
int sbv_stats(sbv_handle h, double *out9);

/* Per-stage device times (ms, CUDA events on the handle's stream) of the
 * last sbv_prepare_h (prep=1) or sbv_loglik (prep=0) when opts.profile=1.
 * names: static strings.  Returns the count in *count (<= cap). */
int sbv_stage_times(sbv_handle h, int32_t prep, double *ms, const char **names, int32_t cap,
                    int32_t *count);

/* Last error of the handle: lowest failing zeta block (or -1), stage
 * (1 = Sigma_con / neighbour part, 2 = Sigma_new / block part, 0 = none)
 * and a static-lifetime message (valid until the next call on h). */
int sbv_last_error(sbv_handle h, int64_t *block, int32_t *stage, const char **msg);

int sbv_abi_version(void);

/* ---------------------------------------------------------------------------
 * Prediction: Eq.3 with the Sec.4.1
 * conditional per test block, and Sec.5.5 conditional simulation
 * (P:503-507).  Requires a handle prepared on the TRAINING inputs with the
 * grid kNN (SBV_GRID unset / 1 and m <= 960).
 *
 * sbv_predict: X_star n_star x d row-major FP64 test inputs (host or device),
 * scaled by the handle's `scale`.  Test blocks: k* = max(1, round(n_star /
 * bs_pred)) anchors by the handle's seed and nearest-anchor assignment (the
 * same H2-H5 rules as prepare, on the test set).  Conditioning set of test
 * block j: the exact m_pred nearest TRAINING points (scaled distance, ties to
 * the lower index) of its centroid, no ordering constraint.
 * y: n training observations (host or device); theta as in sbv_loglik.
 * mean / var: n_star outputs (host or device), in the caller's test order:
 * mean = Sigma_{*J} Sigma_JJ^{-1} y_J, var = diag(Sigma_** - Sigma_{*J}
 * Sigma_JJ^{-1} Sigma_{J*}) with the nugget on Sigma_**'s diagonal.
 * Errors: SBV_ERR_ARG (NULL / ranges / non-finite X_star), SBV_ERR_STATE (not
 * prepared), SBV_ERR_UNSUPPORTED (no grid kNN, m_pred > 960, or
 * m_pred + test block > 4096), SBV_ERR_NOT_PD (lowest failing test block in
 * sbv_last_error).  Single device: every rank predicts every test block. */
int sbv_predict(sbv_handle h, const double *X_star, int64_t n_star, int32_t bs_pred, int32_t m_pred,
                const double *y, const double *theta, double *mean, double *var);

/* Structure of the last sbv_predict (any output may be NULL): number of test
 * blocks, test anchors int32[k*], test point -> block int32[n_star], block
 * offsets int64[k*+1] and block-major test permutation int32[n_star], and the
 * conditioning sets int32[k* x m_pred] as ORIGINAL training indices (-1 pad)
 * with counts int32[k*]. */
int sbv_get_prediction(sbv_handle h, int64_t *k_star, int32_t *anchors, int32_t *block_of, int64_t *off,
                       int32_t *perm, int32_t *nbr, int32_t *cnt);

/* Sec.5.5 conditional simulation: for each point j, n_sim draws
 * x = mean_j + sqrt(var_j) z with z = sqrt(-2 ln u1) cos(2 pi u2), u1, u2 =
 * ((splitmix64(seed, 2c) >> 11) + 0.5) 2^-53 and ((splitmix64(seed, 2c+1) >>
 * 11) + 0.5) 2^-53, c = j n_sim + s; outputs the sample mean, the sample sd
 * (divisor n_sim - 1) and sample mean -/+ z_{alpha/2} sd, alpha = 1 - ci_level.
 * Inputs / outputs n_star doubles, host or device.  var must be >= 0
 * (SBV_ERR_ARG otherwise), n_sim >= 2, 0 < ci_level < 1. */
int sbv_simulate(sbv_handle h, const double *mean, const double *var, int64_t n_star, int32_t n_sim,
                 uint64_t seed, double ci_level, double *sim_mean, double *sim_sd, double *ci_lo,
                 double *ci_hi);

#ifdef __cplusplus
}
#endif
#endif /* SBV_H_ */
