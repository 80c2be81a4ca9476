/*
 * argus.h -- C ABI of libargus.so, the B200 (sm_100a) per-batch
 * approximation-level router of ARGUS (arXiv 2511.06724).
 *
 * For a batch of N prompt embeddings the library runs the hot path of
 * SURVEY.md §8(a) entirely in its own CUDA kernels:
 *   A1 query preparation  fp32 -> bf16, inverse norms
 *   A2 cache scan         cosine S = <x, c> / (|x| |c|)           (§2.1 "Using similarity
 *                         search, the most similar cached prompt is retrieved"; §4.5; §4.7)
 *   A3 top-k              k best (score desc, global id asc); the N x M score
 *                         matrix never reaches HBM                 ("most similar")
 *   A4 quality predictor  r = sigmoid(W2 relu(W1 [x; s] + b1) + b2), r_0 := 1
 *                                                                  (§4.1, §4.4)
 *   A5 compliance         A_i = {v : v = 0 or k_skip_v = 0 or s_i1 >= tau_v},
 *                         C_i = {v in A_i : r_iv >= delta}, delta = 0.9 (§3),
 *                         preference pi_i = A_i by (r desc, p_th desc, v asc),
 *                         priority (|C_i| asc, i asc)
 *   A6 assignment         serial dictatorship under per-option integer quotas c_v
 *                         derived from the allocator's F(v)     (Eq. 1, §4.3)
 * The numbered readings of the paper (ties, >= vs >, gates, overflow) are listed
 * in DESIGN.md §"Readings".
 *
 * Conventions (all functions):
 *   - return 0 (ARGUS_OK) on success, > 0 for a warning, < 0 for an error;
 *     no exceptions cross the ABI;
 *   - the caller owns every array it passes; the library copies what it needs
 *     (cache rows, weights, option table) into its own device memory and never
 *     retains a caller pointer past the call;
 *   - "host" pointers are ordinary (pageable or pinned) CPU memory; "dev"
 *     pointers are CUDA device memory on cfg.device;
 *   - after a CUDA or NCCL failure the router is poisoned and every later call
 *     on it returns ARGUS_E_STATE (argus_route_destroy still frees it);
 *   - a router is not thread-safe: one router per thread / process.
 *
 * Multi-GPU (world > 1, one process per GPU): the cache is row-striped, global
 * id g lives on rank g mod world at local slot g div world.  argus_cache_insert
 * and argus_route_batch* are collectives (every rank calls them in the same
 * order).  With an NCCL unique id, rank 0's inputs are authoritative (other
 * ranks may pass NULL inputs) and are broadcast by the library -- the rows, the
 * prompts and, for argus_route_batch* under ARGUS_POLICY_SD, the quotas (a
 * negative rank-0 quota then fails the call on every rank with ARGUS_E_INVALID,
 * reported like an invalid prompt); the per-shard
 * top-k candidates are exchanged with one all-gather of N*k u64 keys.  Without
 * a unique id ("external" mode) every rank passes the same inputs and the
 * caller moves the keys between argus_route_partial_dev and
 * argus_route_finish_dev itself.  Outputs are identical on every rank.
 */
#ifndef ARGUS_H
#define ARGUS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ------------------------------------------------------------ return codes */
#define ARGUS_OK 0
#define ARGUS_W_OVERFLOW 1        /* some prompt found no admissible quota; it got option 0 */
#define ARGUS_E_INVALID (-1)      /* bad argument, non-finite value or zero-norm vector   */
#define ARGUS_E_CAPACITY (-2)     /* an insert would exceed cfg.capacity                  */
#define ARGUS_E_CUDA (-3)         /* CUDA runtime / launch failure (router poisoned)      */
#define ARGUS_E_NCCL (-4)         /* NCCL failure (router poisoned)                       */
#define ARGUS_E_STATE (-5)        /* router poisoned, or call not valid in this mode      */
#define ARGUS_E_UNIMPLEMENTED (-6)

/* per-prompt status bits (status_out) */
#define ARGUS_ST_OVERFLOW 1u      /* no option of pi_i had quota left -> option 0          */
#define ARGUS_ST_NONCOMPLIANT 2u  /* assigned option has r < delta                         */
#define ARGUS_ST_GATED_ALL 4u     /* every gated (k_skip > 0) option failed its gate (miss) */

typedef struct argus_router argus_router; /* opaque, owned by the library */

/* One approximation option v (SPEC S:26-32 Variant).
 * The table passed to argus_route_init is ordered slow -> fast: option 0
 * is the full model (k_skip must be 0), p_th_qpm must be non-decreasing.
 *   model_id  caller's model identifier (metadata only)
 *   k_skip    approximate-caching skip level K, 0 <= K < 50 (T = 50)
 *   p_th_qpm  peak throughput P_th(v) in queries/minute (used for tie-breaks)
 *   sim_gate  tau_v: option admissible only if the top-1 cosine >= tau_v
 *             (ignored, i.e. -inf, when k_skip == 0; "based on prompt
 *             similarity, an appropriate approximation level (K) is selected") */
typedef struct {
  int32_t model_id;
  int32_t k_skip;
  float p_th_qpm;
  float sim_gate;
} argus_option;

/* Router configuration.
 *   d          embedding dimension, multiple of 64, 64 <= d <= 1024 (CLIP d=768,
 *              OpenCLIP-H d=1024)
 *   k          top-k, 0 <= k <= 8.  k = 0 is the paper's SM mode (smaller model
 *              variants, no cache retrieval): no scan, the predictor
 *              sees the prompt embedding only (w1 is [hidden][d]), every option must
 *              have k_skip = 0, topk outputs may be NULL
 *   L          number of options, 1 <= L <= 32
 *   hidden     predictor hidden width H, multiple of 32, 32 <= H <= 1024
 *   max_batch  largest N a route call may pass, 1 <= max_batch <= 8192
 *   capacity   max global cache entries, capacity <= 2^32 - 2
 *   delta      optimal-quality threshold (0.9); compared as float r >= delta
 *   rank, world, device   this process's rank, world size (1 = single GPU), CUDA device
 *   nccl_unique_id        128-byte ncclUniqueId identical on all ranks, or NULL
 *                         (single GPU, or external collective mode).  With
 *                         world == 1 a unique id builds a one-rank communicator:
 *                         the multi-GPU data path (broadcasts, all-gather,
 *                         per-shard merge) on one GPU, for testing
 *   stream     cudaStream_t to run on, or NULL (the library creates one)
 *   evict      0: an insert past capacity fails (ARGUS_E_CAPACITY).  1: ring
 *              eviction of the oldest entries (capacity % world == 0); see
 *              argus_cache_insert_h
 *   pipeline   0: every call's work is ordered on `stream`.  1 (device and
 *              asynchronous host calls): the fused tail of batch b (merge,
 *              predictor, A5, assignment) runs on an internal high-priority
 *              stream and overlaps the scan of batch b+1; the outputs of a call
 *              are complete once argus_route_join / argus_sync says so.  The
 *              prompt buffer of a call may be reused as soon as `stream` has
 *              passed the call (the prompts are consumed by the scan part).
 *              With NCCL the collectives run on one internal stream in program
 *              order and batch b's exchange + tail are issued by call b+1 (or by
 *              argus_route_join / argus_sync / argus_route_wait); on the
 *              ncclAllGather fallback path those draining calls issue a collective,
 *              so every rank must make them at the same point of its call sequence. */
typedef struct {
  int32_t d, k, L, hidden;
  int32_t max_batch;
  int64_t capacity;
  float delta;
  int32_t rank, world, device;
  const void* nccl_unique_id;
  void* stream;
  int32_t pipeline;
  int32_t evict;
} argus_config;

/* Create an ncclUniqueId (128 bytes) on rank 0; share it with the other ranks
 * (e.g. torch.distributed.broadcast_object_list) before argus_route_init. */
int argus_nccl_unique_id(void* out128);

/* Create a router.  Host arrays (copied):
 *   opts [L]                 option table, slow -> fast
 *   w1 [hidden][d + k] fp32  layer-1 weights; columns [0, d) act on the prompt
 *                            embedding and are stored as bf16 (RNE; the canonical
 *                            tensor-core operand), columns [d, d+k) act on the
 *                            top-k cosine scores (fp32)
 *   b1 [hidden], w2 [L][hidden], b2 [L]  fp32
 * Errors: ARGUS_E_INVALID (ranges above, opts[0].k_skip != 0, k_skip outside
 * [0,50), p_th decreasing, non-finite weights), ARGUS_E_CUDA, ARGUS_E_NCCL.
 * With world > 1 and a unique id this is a collective; rank 0's opts/weights are
 * broadcast (others may pass NULL). */
int argus_route_init(const argus_config* cfg, const argus_option* opts, const float* w1,
                     const float* b1, const float* w2, const float* b2, argus_router** out);

/* Append n cache entries (host fp32 [n][d], row-major) with global ids
 * [M, M + n); *first_id (may be NULL) receives M.  Each row is stored as bf16
 * (RNE) with an fp32 inverse norm of the stored values.  Errors:
 * ARGUS_E_INVALID (non-finite value or zero-norm row; the cache is unchanged),
 * ARGUS_E_CAPACITY.  Collective when world > 1. */
int argus_cache_insert(argus_router* r, const float* emb, int64_t n, int64_t* first_id);

/* Same, rows already on the device (fp32 [n][d]); synchronous. */
int argus_cache_insert_dev(argus_router* r, const float* emb_dev, int64_t n, int64_t* first_id);

/* Route one batch (host buffers; synchronous).
 *   prompts [N][d] fp32 host, 1 <= N <= max_batch
 *   quota [L] int32 host, quota[v] >= 0 (sum >= N expected; otherwise the
 *         overflowing prompts get option 0 and ARGUS_ST_OVERFLOW)
 * Outputs (host, caller-allocated):
 *   option_out [N] int32    assigned option index
 *   topk_idx [N][k] uint32  global cache ids, best first (0xFFFFFFFF pads M < k)
 *   topk_score [N][k] fp32  cosine scores, best first (-1.0 pads)
 *   quality_out [N][L] fp32 predicted relative quality r, or NULL
 *   status_out [N] uint8    ARGUS_ST_* bits, or NULL
 * Returns ARGUS_OK, ARGUS_W_OVERFLOW, or an error (ARGUS_E_INVALID for a
 * non-finite / zero-norm prompt or a negative quota). */
int argus_route_batch(argus_router* r, const float* prompts, int32_t N, const int32_t* quota,
                      int32_t* option_out, uint32_t* topk_idx, float* topk_score,
                      float* quality_out, uint8_t* status_out);

/* Device-buffer variant: prompts_dev fp32 [N][d] and the outputs are device
 * pointers (quality_dev, status_dev may be NULL); quota is a HOST int32 [L].
 * Enqueued asynchronously on the router's stream; returns ARGUS_OK once
 * enqueued.  Value errors found on the device (invalid prompt) and the
 * overflow warning are reported by the next argus_sync(). */
int argus_route_batch_dev(argus_router* r, const float* prompts_dev, int32_t N,
                          const int32_t* quota, int32_t* option_out_dev,
                          uint32_t* topk_idx_dev, float* topk_score_dev, float* quality_dev,
                          uint8_t* status_dev);

/* Asynchronous host-buffer route: the call of a serving loop.  Enqueues the copy of
 * prompts (host fp32 [N][d]) to the device, the whole path, and the copies of the
 * outputs back into the caller's host buffers (same meaning as argus_route_batch;
 * quality_out / status_out may be NULL), then returns at once with *ticket set to
 * an increasing call id.  All buffers must stay alive and untouched until
 * argus_route_wait(r, *ticket) returns; the prompts should be pinned (page-locked)
 * host memory, or their copy runs synchronously.  The outputs travel back in one
 * packed copy into the library's pinned staging and are unpacked into the caller's
 * buffers when the call is collected (argus_route_wait / argus_sync, or when its
 * staging slot is reused four calls later).  With cfg.pipeline = 1 consecutive calls overlap (the
 * tail of one with the scan of the next).  A call waits (on the host) for the call
 * issued four calls before it to finish.  Returns ARGUS_OK once enqueued or an
 * argument error; the call's own result comes from argus_route_wait. */
int argus_route_batch_async(argus_router* r, const float* prompts, int32_t N, const int32_t* quota,
                            int32_t* option_out, uint32_t* topk_idx, float* topk_score, float* quality_out,
                            uint8_t* status_out, int64_t* ticket);

/* Wait until the asynchronous call `ticket` (and every earlier one) has delivered its
 * outputs; return its result (ARGUS_OK, ARGUS_W_OVERFLOW, ARGUS_E_INVALID for an
 * invalid prompt).  Each ticket's result can be collected once; waiting for a later
 * ticket first implicitly collects the earlier ones (ARGUS_E_INVALID afterwards). */
int argus_route_wait(argus_router* r, int64_t ticket);

/* Sharded pipeline pieces (external collective mode and tests).
 * partial: A1-A3 on this rank's shard -> keys_dev [N][k] uint64 (sorted desc;
 *          key = ord(score) << 32 | (0xFFFFFFFF - g), 0 = empty).
 * finish:  merge G shards' keys (keys_all_dev [G][N][k], 8-byte aligned, G ==
 *          cfg.world, else ARGUS_E_INVALID) -> A3 outputs, then A4-A6 exactly as
 *          argus_route_batch_dev.  prompts_dev must be the same batch passed to
 *          partial (its bf16 copy and inverse norms are reused; an invalid prompt
 *          there fails this call too, on every rank). */
int argus_route_partial_dev(argus_router* r, const float* prompts_dev, int32_t N,
                            uint64_t* keys_dev);
int argus_route_finish_dev(argus_router* r, const uint64_t* keys_all_dev, int32_t G, int32_t N,
                           const int32_t* quota, int32_t* option_out_dev,
                           uint32_t* topk_idx_dev, float* topk_score_dev, float* quality_dev,
                           uint8_t* status_dev);

/* Fused candidate exchange over peer memory (P:381's one process per
 * GPU).  The shard's merge kernel stores its N x k keys straight into every rank's
 * inbox (NVLink stores through CUDA IPC mappings) and releases a per-batch flag; each
 * rank's tail acquires the world flags and reads its own inbox -- no all-gather call.
 * Inbox slots alternate by batch parity and a sender waits (normally not at all) until
 * the receiver has consumed the batch that used the slot two batches earlier.  A peer
 * that does not deliver within 5 s fails the call with ARGUS_E_NCCL instead of hanging.
 * NCCL mode: set up by argus_route_init itself (IPC handles exchanged over the
 * communicator); if any rank cannot map its peers, every rank keeps ncclAllGather
 * (ARGUS_NO_P2P=1 forces that).  External mode (world > 1, no unique id): the caller
 * connects the ranks -- every rank calls argus_p2p_export (64-byte handle out), the
 * caller exchanges the handles (e.g. torch.distributed all_gather_object), and every
 * rank calls argus_p2p_connect with the [world][64] array in rank order.  Afterwards
 * argus_route_batch* work in external mode as collectives (every rank passes the same
 * prompts and quotas; no broadcast).  Errors: ARGUS_E_INVALID (not external mode, k = 0,
 * world > 16, connect before export), ARGUS_E_CUDA (a handle that cannot be mapped). */
int argus_p2p_export(argus_router* r, void* handle_out);
int argus_p2p_connect(argus_router* r, const void* handles);

/* Make `stream` (cudaStream_t; NULL = the router's stream) wait, on the device,
 * for all routing work enqueued so far, including pipelined tails.  No host
 * synchronisation.  Errors: ARGUS_E_CUDA. */
int argus_route_join(argus_router* r, void* stream);

/* Wait for all of the router's work (every stream, including the result copies of
 * asynchronous host calls); return the deferred code of the enqueued device-buffer
 * work (ARGUS_OK, ARGUS_W_OVERFLOW, ARGUS_E_INVALID) and clear it.  Results of
 * asynchronous calls stay available to argus_route_wait. */
int argus_sync(argus_router* r);

/* Largest-remainder integer quotas from load shares (host helper, O(L)):
 * t_v = (f_v * N) / S with S = sum_v f_v summed v = 0..L-1 in double;
 * c_v = floor(t_v); the N - sum c leftover units go one each to the largest
 * fractional parts t_v - c_v, ties to the lower v.  sum c = N.
 * f [L] >= 0 finite with S > 0, 1 <= L <= 64, N >= 0; c_out [L]. */
int argus_quota_from_fractions(const double* f, int32_t L, int32_t N, int32_t* c_out);

/* ------------------------------------------------ control plane
 *
 * The paper's per-minute loop ("Every minute, we solve ..."): the allocator
 * solves Eq. 1 for the load shares F(v) (argus_solve_allocation); the workload
 * distribution predictor's affinity histogram H(v) of optimal options over the
 * last 1000 prompts (argus_affinity_histogram) and F feed ODA
 * (argus_oda_pasm), whose PASM the prompt scheduler samples per prompt
 * (argus_set_policy with ARGUS_POLICY_PASM).  Eq. 3 then picks a
 * worker for every prompt (argus_set_workers).  Quotas for the default
 * serial-dictatorship policy come from F via argus_quota_from_fractions. */

/* Eq. 1 for n_workers homogeneous workers and L levels (slow -> fast):
 * maximise sum_v Q_v F(v), F(v) = Y_v / W, subject to each worker running at most
 * one level and carrying an integer load y_w <= floor(p_th[v_w]) (QPM) with
 * sum_w y_w = W.  Exact (dynamic program over compositions, loads water-filled in
 * decreasing Q).  W = 0: every worker on level 0, loads 0, F = e_0.  W above the
 * cluster's capacity: every worker on the fastest level at capacity and
 * *feasible_out = 0 ("saturated plan flagged infeasible").
 *   Q [L] profiled relative quality, p_th [L] peak throughput (QPM)
 *   level_out [n_workers] level of worker w (or NULL), load_out [n_workers] y_w (or
 *   NULL), F_out [L] load shares (or NULL), objective_out sum_v Q_v Y_v / served
 *   (or NULL), feasible_out (or NULL).  Host only; no router needed.
 * Errors: ARGUS_E_INVALID (ranges, non-finite, (L+1)(n_workers+1)(W+1) > 2^24). */
int argus_solve_allocation(int32_t W, int32_t n_workers, int32_t L, const double* Q, const float* p_th,
                           int32_t* level_out, int32_t* load_out, double* F_out, double* objective_out,
                           int32_t* feasible_out);

/* Algorithm 1, the Optimized Distribution Aligner.  H [L] affinity
 * histogram (counts or shares, >= 0, sum > 0), F [L] target load shares (>= 0,
 * sum > 0), both normalised to distributions; levels slow (0) -> fast (L-1).
 * pasm_out [L][L] row-major: pasm_out[i*L + j] = P(v'_j | v_i), the probability
 * that a prompt whose optimal level is v_i is served at v'_j; rows of levels with
 * H = 0 are the identity.  Per-origin mass bookkeeping realises the paper's chain
 * composition of step probabilities (R19).  Host only. */
int argus_oda_pasm(const double* H, const double* F, int32_t L, double* pasm_out);

/* Eq. 2: *dq_out = sum_i sum_{j : p_th[j] > p_th[i]} pasm[i][j] H[i] D[j][i],
 * D [L][L] row-major (D[j*L + i] = degradation of serving a v_i-optimal prompt at v'_j). */
int argus_pasm_degradation(const double* pasm, const double* H, const float* p_th, const double* D, int32_t L,
                           double* dq_out);

#define ARGUS_POLICY_SD 0    /* quota-capped serial dictatorship (row A6, the default)   */
#define ARGUS_POLICY_PASM 1  /* sample the PASM row of each prompt's optimal option     */
#define ARGUS_AFFINITY_WINDOW 1000

/* Select the assignment policy of the router (collective when world > 1; every
 * rank must pass the same arguments).  ARGUS_POLICY_PASM: pasm [L][L] as from
 * argus_oda_pasm (rows >= 0, each with positive sum; rows are used as given);
 * for prompt i of the b-th routing call after this one (b = 0, 1, ...):
 *   o_i = the optimal option: among C_i the largest p_th, then the larger r,
 *         then the lower index (DESIGN R18);
 *   u_i = (x >> 8) * 2^-24 with x the first word of Philox4x32-10(counter =
 *         {i, b mod 2^32, b >> 32, 0}, key = {seed mod 2^32, seed >> 32});
 *   a_i = the first j with u_i < cdf[o_i][j], cdf the float32 running sums of the
 *         row (float32 adds, j ascending); if none, the last j with pasm > 0;
 *   an inadmissible a_i (similarity gate) falls back to the largest admissible
 *         option below it (DESIGN R21).
 * Quotas are ignored (may be NULL) under PASM; status gets NONCOMPLIANT when
 * r_{i,a_i} < delta and GATED_ALL as usual; OVERFLOW never.
 * ARGUS_POLICY_SD: pasm and seed ignored.  Errors: ARGUS_E_INVALID. */
int argus_set_policy(argus_router* r, int32_t policy, const double* pasm, uint64_t seed);

/* Affinity histogram H(v): counts of the optimal options o_i of the last
 * min(routed, ARGUS_AFFINITY_WINDOW) prompts routed by this router (both
 * policies).  counts_out [L]; *n_out = number of prompts counted.  Synchronises
 * the router. */
int argus_affinity_histogram(argus_router* r, int64_t* counts_out, int64_t* n_out);

/* Worker selector (Eq. 3).  n_workers in [0, 1024] (0 disables);
 * option_of_worker [n] = the option v worker w serves (-1 = none; at most 32
 * workers per option), t_proc [n] its per-image time (> 0, finite), queue [n] its
 * current queue length R_queue,w (>= 0).  Each routed batch then assigns, for
 * prompts in index order, w_i = argmin over the workers serving a_i of
 * fl32(float(R_w) * t_w), ties to the lower w, and increments R_{w_i}; prompts
 * whose option no worker serves get -1.  The queues live in device memory; a later
 * argus_set_workers call replaces them (e.g. after completions). */
int argus_set_workers(argus_router* r, int32_t n_workers, const int32_t* option_of_worker, const float* t_proc,
                      const int32_t* queue);

/* Current queue lengths R_queue,w [n_workers] (synchronises the router). */
int argus_get_queues(argus_router* r, int32_t* queue_out);

/* Optional outputs of argus_route_batch_ex / argus_route_batch_ex_dev (any member
 * may be NULL; host buffers for the host call, device buffers for the _dev call):
 *   optimal      [N] int32   o_i, the prompt's optimal option ("optimal model
 *                            choice"), as defined under argus_set_policy
 *   worker       [N] int32   the Eq. 3 worker of the assigned option, -1 if no worker
 *                            serves it (requires argus_set_workers)
 *   topk_handle  [N][k] u64  the latent handle stored with each returned cache entry
 *                            (argus_cache_insert_h; 0 for none / padding), i.e. the
 *                            intermediate-state reference the worker fetches */
typedef struct {
  int32_t* optimal;
  int32_t* worker;
  uint64_t* topk_handle;
} argus_route_extra;

/* argus_route_batch / argus_route_batch_dev plus the outputs in *extra (NULL = none). */
int argus_route_batch_ex(argus_router* r, const float* prompts, int32_t N, const int32_t* quota,
                         int32_t* option_out, uint32_t* topk_idx, float* topk_score, float* quality_out,
                         uint8_t* status_out, const argus_route_extra* extra);
int argus_route_batch_ex_dev(argus_router* r, const float* prompts_dev, int32_t N, const int32_t* quota,
                             int32_t* option_out_dev, uint32_t* topk_idx_dev, float* topk_score_dev,
                             float* quality_dev, uint8_t* status_dev, const argus_route_extra* extra);

/* argus_route_batch_ex_dev for prompts already in bf16 (SURVEY §8(b) "prompts_bf16_dev";
 * e.g. CLIP embeddings kept in bf16 by the caller): prompts_bf16_dev is device bf16 [N][d]
 * row-major, 4-byte aligned.  The rows enter the scan as they are; their inverse norms
 * are computed from the same values in the same order as the fp32 path computes them
 * after rounding, so a batch gives bit-identical outputs through either call when its
 * fp32 values round to these bf16 values.  Non-finite or zero rows: ARGUS_E_INVALID
 * (reported by argus_sync like the fp32 device call). */
int argus_route_batch_bf16_dev(argus_router* r, const void* prompts_bf16_dev, int32_t N, const int32_t* quota,
                               int32_t* option_out_dev, uint32_t* topk_idx_dev, float* topk_score_dev,
                               float* quality_dev, uint8_t* status_dev, const argus_route_extra* extra);

/* Cache lifecycle ("Each prompt stores intermediate states at K"): append n
 * entries like argus_cache_insert and store handles [n] (u64, caller-defined, e.g.
 * an object-store key of the 144 KB intermediate state; NULL = 0) with them.
 * With cfg.evict = 1 a full cache overwrites its oldest entries (ring): the live
 * entries are always the last min(M, capacity) inserted, ids keep counting
 * (global id g lives at cache position g mod capacity), and a rejected insert
 * (non-finite / zero-norm row) leaves the cache unchanged. */
int argus_cache_insert_h(argus_router* r, const float* emb, const uint64_t* handles, int64_t n, int64_t* first_id);

/* Number of cache entries inserted so far (global, identical on all ranks). */
int argus_cache_size(const argus_router* r, int64_t* m_out);

/* Number of kernel launches the router has issued so far (for bench accounting). */
int argus_launch_count(const argus_router* r, int64_t* n_out);

/* The router's CUDA stream (cudaStream_t as void*). */
int argus_get_stream(const argus_router* r, void** stream_out);

/* Per-stage kernel timing (measurement only).  When enabled, the library
 * records a CUDA event pair on its stream around every kernel it launches;
 * argus_profile_read synchronises and returns, for one stage, the summed
 * device milliseconds and the number of launches since the last read (then
 * resets that stage).  Stages: 0 prep (K6), 1 scan (K1+K2), 2 local merge before
 * the all-gather (K5, multi-GPU only), 3 unused, 4 the fused tail (merge of the
 * candidate lists + predictor + A5 + assignment), 5 unused (the assignment runs
 * inside the tail), 6 insert (K0). */
#define ARGUS_STAGE_PREP 0
#define ARGUS_STAGE_SCAN 1
#define ARGUS_STAGE_MERGE_LOCAL 2
#define ARGUS_STAGE_MERGE_GLOBAL 3
#define ARGUS_STAGE_TAIL 4
#define ARGUS_STAGE_ASSIGN 5
#define ARGUS_STAGE_INSERT 6
#define ARGUS_NUM_STAGES 7
int argus_profile_enable(argus_router* r, int on);
int argus_profile_read(argus_router* r, int stage, double* total_ms, int64_t* launches);

/* Score capture for parity test T2 (SURVEY §8(c).iii "oracle O4 on the GPU's fp32
 * scores equals the GPU's top-k exactly, including order"); debug sizes only.
 * While scores_dev != NULL, the scan of every later route call also writes each
 * score its fused top-k compares -- S[i][j] = fl32(fl32(acc_ij * inv_c[j]) * inv_q[i]),
 * acc the tensor-core fp32 dot product of the bf16 rows (P:132 cosine similarity) --
 * to scores_dev[i * ld + j] for prompts i < N and this shard's local slots j < its
 * live rows (slot j holds cache position j * world + rank).  scores_dev is device
 * fp32 owned by the caller and must stay allocated until capture is switched off
 * (scores_dev = NULL); entries of other slots are left untouched.  A route call
 * whose shard has more live rows than ld fails with ARGUS_E_INVALID.  Costs an
 * N x M write per batch: a test setting, never a production one. */
int argus_debug_capture(argus_router* r, float* scores_dev, int64_t ld);

/* Free all device memory, the NCCL communicator and the router. */
int argus_route_destroy(argus_router* r);

/* Static description of a return code. */
const char* argus_strerror(int code);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* ARGUS_H */
