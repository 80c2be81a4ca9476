// kernels.h -- internal launchers of libargus (not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace argus {

// Launch with programmatic stream serialization (PDL); see common.cuh.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_opt(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  return launch_pdl_opt(true, kern, grid, block, smem, s, std::forward<Args>(args)...);
}

// error flags written by kernels into a device word (bitwise OR)
enum : uint32_t { FLAG_INVALID_INPUT = 1u, FLAG_OVERFLOW = 2u, FLAG_PEER_TIMEOUT = 4u };
constexpr uint64_t P2P_TIMEOUT_NS = 5000000000ull;  // a peer that does not deliver in 5 s: error, no hang

struct ScanArgs {
  const __nv_bfloat16* Xb;   // [n_pad][d] bf16 prompts (rows >= N are zero)
  const float* inv_q;        // [n_pad]
  const __nv_bfloat16* Cb;   // [cap_local][d] bf16 cache shard
  const float* inv_c;        // [cap_local]
  int64_t m_local;           // rows valid in this shard
  int32_t N, n_pad, d, k;
  int32_t rank, world;       // global id g = slot * world + rank
  uint64_t* partial;         // [P][N][k] per-CTA-range candidates
  int32_t P;                 // number of cache ranges (filled by the planner)
  uint64_t* gthr;            // [n_pad] per-prompt shared top-k threshold key (zeroed by K6)
  int32_t* ctr;              // [CTR_WORDS] (zeroed by K6): per-slice tile counters [0, MAX_SLICES),
                             // pair-slice visit counters [2 MAX_SLICES, 3 MAX_SLICES) (migration)
  uint32_t head, capg;       // ring eviction: oldest live cache position, capacity (0, 0 when not wrapped)
  int32_t window;            // pair scan: max chunks a pair slice may lead the slowest (0 = off)
  int32_t migrate;           // pair scan: pairs whose slice runs dry continue another slice
  int32_t home_max;          // pair scan: home pairs per pair slice = their list slots [0, home_max)
  int32_t floaters;          // pair scan: pairs beyond home_max * pair slices (slots home_max + f)
  int32_t grid_ctas;         // pair scan with migration: CTAs launched (all SMs' pairs)
  const uint32_t* ready;     // pipelined one-GPU one-slice scans: wait until *ready - ready_seq >= 0
                             // (the prep stream publishes it after K6) instead of a stream event + the
                             // grid-dependency wait; NULL: griddepcontrol.wait
  uint32_t ready_seq;
  uint64_t* stamp;           // diagnostics (ARGUS_SCAN_STAMP): per CTA %globaltimer at entry, after the
                             // grid-dependency wait, first accumulator read, exit (NULL: off)
  float* dbg;                // argus_debug_capture: every exact score to dbg[p * dbg_ld + slot] (NULL: off)
  int64_t dbg_ld;
};
constexpr int MAX_SLICES = 64;  // max_batch <= 8192 = 64 slices of 128 prompts
constexpr int CTR_WORDS = 3 * MAX_SLICES;
constexpr int MAX_VISITS = 4;   // migrant pairs per pair slice (list slots home_max .. home_max + 3)

// K0: fp32 rows -> bf16 stripe + inverse norms; rows g in [g0, g0+n) whose
// g % world == rank go to slot g / world.
void launch_insert_rows(const float* rows, int64_t n, int64_t g0, int32_t d, int32_t rank, int32_t world,
                        int64_t cap, bool dry, __nv_bfloat16* Cb, float* inv_c, uint32_t* flags, cudaStream_t s);

// Publishes v into *flag (release, gpu scope) once the stream's earlier work is complete.
void launch_publish(uint32_t* flag, uint32_t v, cudaStream_t s);

// K6: prompts fp32 [N][d] -> Xb bf16 [n_pad][d] (zero padded), inv_q [n_pad].
// With quota != nullptr (host [L]) it also writes the quotas into quota_dev [32]
// (the multi-GPU root, ahead of the C-1 broadcast).
struct QuotaVec {
  int32_t v[32];
};
// X is fp32 [N][d], or bf16 [N][d] with in_bf16 (copied as is).
void launch_prep_queries(const void* X, bool in_bf16, int32_t N, int32_t n_pad, int32_t d, __nv_bfloat16* Xb,
                         float* inv_q, uint64_t* gthr, int32_t* ctr, uint32_t* flags, cudaStream_t s,
                         bool pdl = true, const int32_t* quota = nullptr, int32_t L = 0,
                         int32_t* quota_dev = nullptr);

// K1+K2 for N <= 64 prompts (d = 768, k <= 8), transposed: cache rows are the MMA's M, the
// prompts its N (k_scan_t.cu).  a.P = CTAs = candidate lists (scan_t_plan_ranges).
bool scan_t_supported(int d, int32_t N, int k);
int scan_t_plan_ranges(int64_t m_local, int num_sms);
cudaError_t launch_scan_t(const ScanArgs& a, const CUtensorMap* tmap_c, const CUtensorMap* tmap_q16, cudaStream_t s,
                          bool pdl);

// K1+K2: fused tcgen05 scan + per-range top-k -> partial [P][N][k].
// scan_plan_ranges returns P (cache ranges; grid = P * ceil(N / 128) CTAs).
int scan_plan_ranges(int64_t m_local, int32_t N, int num_sms);
bool scan_supported(int d);
void launch_scan(const ScanArgs& a, const CUtensorMap* tmap_c, const CUtensorMap* tmap_q, cudaStream_t s,
                 bool pdl = true);

// K1+K2 on CTA pairs (tcgen05.mma.cta_group::2) for N > 128 and d <= 768:
// grid = 2 * ceil(N / 256) * P CTAs in clusters of two, P from scan_pair_plan.
int scan_pair_plan(int64_t m_local, int32_t N, int num_sms);
bool scan_pair_supported(int d, int32_t N);
// Returns the launch error (e.g. no TPC can host a 2-CTA cluster); the caller then
// runs the one-slice-per-CTA kernel instead.
cudaError_t launch_scan_pair(const ScanArgs& a, const CUtensorMap* tmap_c32, const CUtensorMap* tmap_q,
                             cudaStream_t s, bool pdl = true);

// K5: merge P lists of k keys per prompt -> keys [N][k] (desc), optionally
// decoding ids / scores.
void launch_merge_topk(const uint64_t* in, int32_t P, int32_t N, int32_t k, uint64_t* keys_out,
                       uint32_t* idx_out, float* score_out, cudaStream_t s);

// K5 + C-2 fused (k_merge.cu): peer inboxes of one parity.  keys[g] = base of rank g's
// inbox keys [G][max_batch][k] (IPC-mapped for g != rank), flag[g] = rank g's flag word
// for senders [rank] (the release store of the batch sequence number).
constexpr int P2P_MAX = 16;
struct P2PSend {
  uint64_t* keys[P2P_MAX];            // rank g's inbox keys of this parity
  uint32_t* flag[P2P_MAX];            // rank g's arrival flag [parity][sender = rank]
  const uint32_t* consumed[P2P_MAX];  // rank g's consumed counter of this parity
  uint32_t* err;                      // this rank's flags word (FLAG_PEER_TIMEOUT)
  int32_t G, rank;
  uint32_t seq;
};
// grid = min(N, max_ctas) CTAs looping over the prompts (max_ctas = the SM count)
void launch_merge_send(const uint64_t* in, int32_t P, int32_t N, int32_t k, const P2PSend& dst, int* ticket,
                       cudaStream_t s, bool pdl, int max_ctas);

struct TailArgs {
  // phase M: candidate lists -> final top-k
  const uint64_t* keys_in;   // [P][N][k] candidate keys (per-range partials, or all-gathered shards)
  int32_t P;
  const uint32_t* p2p_flags; // [P] or nullptr: keys_in is this rank's inbox, filled by the P ranks'
  uint32_t p2p_seq;          // merge kernels; wait until every flag >= p2p_seq (acquire, sys scope)
  uint32_t* p2p_consumed;    // this rank's consumed counter of the parity: p2p_seq once staged
  uint32_t* topk_idx;        // [N][k] out: global id = id_base + age index of the key
  float* topk_score;         // [N][k] out
  uint32_t id_base;          // global id of the oldest live entry
  uint32_t head, capg;       // cache position of age 0, capacity (ring eviction; 0, 0 otherwise)
  const uint64_t* handle;    // [capacity] latent handles by cache position
  uint64_t* topk_handle;     // [N][k] out or nullptr
  // predictor
  const __nv_bfloat16* Xb;   // [n_pad][d]
  const float* inv_q;        // [n_pad] 0 marks an invalid prompt (K6 on the root; broadcast to every rank)
  const void* W1xF;          // W1x bf16 in mma.sync B-fragment order (see k_prep_w1_frag)
  const float* W1sT;         // [k][H]
  const float* b1;           // [H]
  const float* W2;           // [L][H]
  const float* b2;           // [L]
  float* hbuf;               // [ceil(N/16)*16][H] hidden activations (scratch)
  int32_t* block_cnt;        // [ceil(max_batch/16)] zeroed tickets (last CTA of a prompt block)
  int32_t* launch_cnt;       // [1] zeroed ticket (last block of the launch)
  // A5
  const int32_t* kskip;      // [L]
  const float* pth;          // [L]
  const float* gate;         // [L]
  float delta;
  int32_t N, d, k, H, L;
  float* rhat;               // [N][L] out
  uint8_t* prefl;            // [N][32] pi_i in inverse form: rank of option v (0xFF: v not admissible); 16-byte aligned
  int32_t sd_pp_max;         // serial dictatorship one prompt per step for N <= this, else windows of 32
  uint8_t* ccount;           // [N] |C_i|
  uint32_t* cmask;           // [N] compliance mask
  // A6
  int32_t quota[32];         // per-option quotas c_v (by value)
  const int32_t* quota_dev;  // [32] when non-null: the quotas broadcast from rank 0 (used instead)
  int32_t* option_out;       // [N] out
  uint8_t* status;           // [N] out
  uint32_t* flags;
  // F1: optimal options, PASM sampling, affinity window
  int32_t policy;            // 0 serial dictatorship (A6), 1 PASM sampling
  const float* pasm_cdf;     // [32][32] float32 running sums of the PASM rows (row = optimal option)
  const int8_t* pasm_last;   // [32] last option with positive mass per row
  uint32_t seed_lo, seed_hi, seq_lo, seq_hi;  // Philox key / batch counter
  int32_t* optimal_out;      // [N] o_i or nullptr
  uint8_t* aff_ring;         // [aff_win] optimal options of the last aff_win prompts
  int32_t aff_win, aff_pos0; // window length (0: off), ring slot of prompt 0
  // F3: Eq. 3 worker selection (n_workers = 0: off)
  int32_t n_workers;
  const int16_t* wlist;      // [32][32] workers serving option v (ascending), -1 padded
  const int32_t* wcount;     // [32]
  const float* wtime;        // [n_workers] t_proc
  int32_t* queue;            // [n_workers] R_queue (device state, updated)
  int32_t* worker_out;       // [N] or nullptr
};
// K3+K4 (+K5 on one GPU): merge, predictor, A5 and the assignment in one launch.
// pdl = false when the tail's producer is on another stream (pipelined mode):
// griddepcontrol.wait only orders against the previous kernel of the same stream.
// ysplit = CTAs per 16-prompt block (hidden units split H/32 ways at most): H/32 for
// the lowest latency, 1 for the smallest SM footprint (pipelined mode).
void launch_tail(const TailArgs& a, size_t smem, cudaStream_t s, bool pdl, int ysplit);
size_t tail_smem_bytes(int d, int k, int H, int L, int max_batch, int P_max);
// init: W1x (columns [0,d) of w1 [H][d+k]) -> bf16 fragment order [H*d] bf16
void launch_prep_w1_frag(const float* w1, int d, int k, int H, void* Wf, cudaStream_t s);

}  // namespace argus
