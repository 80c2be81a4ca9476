// argus.cu -- host side of libargus.so: the C ABI declared in include/argus.h.
//
// Owns device memory, the CUDA streams, the NCCL communicator and the launch
// sequence of one routing batch:
//   single GPU:  K6 prep -> K1/K2 fused scan + top-k -> fused tail (merge of the
//                per-CTA lists, predictor, A5, assignment)
//   world > 1:   K6 prep (rank 0) -> NCCL broadcast of the bf16 batch -> scan ->
//                K5 local merge -> NCCL all-gather of N*k keys -> fused tail
// Pipelined mode (cfg.pipeline): three internal streams.  prep(b) (high priority)
// runs as soon as the caller's stream has the prompts, concurrently with scan(b-1);
// the scan stream runs the scans back to back; the tail of batch b (high priority)
// overlaps scan(b+1).  All per-batch buffers are double-buffered by batch parity q;
// prep(b) reuses parity q once tail(b-2) (hence scan(b-2)) is done.
// No compute happens on the host: every step of the path is a kernel in this
// library; the host validates arguments, moves buffers and launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <map>
#include <vector>

#include "../../include/argus.h"
#include "kernels.h"

using namespace argus;

namespace {

constexpr int64_t INSERT_CHUNK = 1 << 16;  // rows per staged insert chunk


// NCCL is resolved lazily with dlopen (reusing an already-loaded libnccl.so.2,
// e.g. torch's) so that loading libargus never pins a second NCCL into a process.
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.tried) {
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (h) {
#define NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
      NCCL_SYM(GetUniqueId); NCCL_SYM(CommInitRank); NCCL_SYM(CommDestroy); NCCL_SYM(Broadcast);
      NCCL_SYM(AllGather); NCCL_SYM(AllReduce); NCCL_SYM(GroupStart); NCCL_SYM(GroupEnd);
      NCCL_SYM(GetErrorString);
#undef NCCL_SYM
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.AllGather &&
               api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
    }
  }
  return api;
}

}  // namespace

struct argus_router {
  argus_config cfg{};
  int num_sms = 148;
  bool own_stream = false;
  cudaStream_t stream = nullptr;
  cudaStream_t prep_stream = nullptr;  // pipelined mode: K6 (high priority)
  cudaStream_t scan_stream = nullptr;  // pipelined mode: the scans, back to back
  cudaStream_t tail_stream = nullptr;  // pipelined mode: the fused tails (high priority)
  bool pipe = false;
  cudaEvent_t ev_in[2] = {nullptr, nullptr};    // caller's stream reached the call of parity q
  cudaEvent_t ev_prep[2] = {nullptr, nullptr};  // prep of the batch with parity q done
  cudaEvent_t ev_scan[2] = {nullptr, nullptr};  // scan of the batch with parity q done
  cudaEvent_t ev_tail[2] = {nullptr, nullptr};  // tail of the batch with parity q done
  bool tail_inflight[2] = {false, false};
  int64_t seq = 0;                     // pipelined batches issued
  int cur = 0;                         // parity of the buffers the last prep/scan used
  ncclComm_t comm = nullptr;
  bool poisoned = false;
  int64_t m_global = 0;   // entries inserted (all ranks agree)
  int64_t cap_local = 0;  // rows allocated in this shard
  int64_t launches = 0;
  int32_t n_pad_max = 0;
  // options (device)
  int32_t* d_kskip = nullptr;
  float* d_pth = nullptr;
  float* d_gate = nullptr;
  // weights (device)
  __nv_bfloat16* d_W1xF = nullptr;  // [H*d] bf16, mma fragment order
  float* d_W1sT = nullptr;
  float* d_b1 = nullptr;
  float* d_W2 = nullptr;           // [L][H]
  float* d_h = nullptr;            // [n16][H] predictor hidden activations
  int32_t* d_mlp_cnt = nullptr;    // [n16 / 16] last-CTA tickets
  int32_t* d_tail_cnt = nullptr;   // [1] last-block ticket
  size_t tail_smem = 0;            // dynamic smem of the fused tail kernel
  float* d_b2 = nullptr;
  // cache shard (device)
  __nv_bfloat16* d_Cb = nullptr;
  float* d_invc = nullptr;
  // per-batch workspace (device)
  float* d_Xstage = nullptr;       // [max(max_batch, INSERT_CHUNK)][d] fp32 staging
  __nv_bfloat16* d_Xb[2] = {nullptr, nullptr};  // [n_pad_max][d] per batch parity
  float* d_invq[2] = {nullptr, nullptr};     // [n_pad_max] per batch parity
  uint64_t* d_gthr[2] = {nullptr, nullptr};  // [n_pad_max] shared per-prompt scan threshold
  int32_t* d_ctr[2] = {nullptr, nullptr};    // [CTR_WORDS] scan work / visit counters
  uint64_t* d_partial[2] = {nullptr, nullptr};  // [P * N <= partial_lists][k] per batch parity
  int64_t partial_lists = 0;
  uint64_t* d_keys[2] = {nullptr, nullptr};      // [max_batch][k] this shard's merged keys, per parity
  uint64_t* d_keys_all[2] = {nullptr, nullptr};  // [world][max_batch][k] all-gathered keys, per parity
  float* d_score = nullptr;        // [max_batch][k]
  uint32_t* d_idx = nullptr;       // [max_batch][k]
  float* d_rhat = nullptr;         // [max_batch][L]
  uint8_t* d_pref = nullptr;       // [max_batch][32] pi_i in inverse form (rank of each option)
  uint8_t* d_ccount = nullptr;     // [max_batch]
  uint32_t* d_cmask = nullptr;     // [max_batch]
  uint8_t* d_status = nullptr;     // [max_batch]
  int32_t* d_option = nullptr;     // [max_batch]
  int32_t* d_order = nullptr;      // [max_batch]
  uint32_t* d_flags = nullptr;     // error / overflow flags (first word of d_outblk)
  uint32_t* h_flags = nullptr;     // pinned mirror of the flags word
  uint8_t* d_outblk = nullptr;     // host-path outputs, packed after the flags word (one D2H per batch)
  uint8_t* h_outblk = nullptr;     // pinned mirror
  size_t outblk_bytes = 0;
  bool pending = false;            // async (_dev) work enqueued since the last argus_sync
  bool serial_call = false;
  bool quota_dev_next = false;     // the next tail reads d_quota (set by the broadcast path)        // host-buffer call in progress: one stream with PDL, no event hops
  // asynchronous host-buffer calls (argus_route_batch_async): per-parity device
  // staging of the prompts and outputs, per-parity flags, completion events
  uint32_t* flags_cur = nullptr;   // flags word the kernels of the current call OR into
  static constexpr int NASYNC = 4;     // asynchronous calls in flight
  float* d_Xasync[NASYNC] = {};
  uint8_t* d_oasync[NASYNC] = {};
  uint32_t* h_fasync = nullptr;    // [NASYNC] pinned flag words
  cudaEvent_t ev_async[NASYNC] = {};
  uint8_t* h_oasync[NASYNC] = {};      // pinned staging of each slot's packed outputs
  cudaStream_t d2h_stream = nullptr;   // result copies (off the tail stream)
  cudaEvent_t ev_done[NASYNC] = {};    // the slot's tail finished
  struct AsyncOut {                    // where harvest copies a slot's results
    int32_t N = 0;
    int32_t* option = nullptr;
    uint32_t* idx = nullptr;
    float* score = nullptr;
    float* quality = nullptr;
    uint8_t* status = nullptr;
  } aout[NASYNC];
  int64_t async_ticket[NASYNC] = {-1, -1, -1, -1};  // ticket whose D2H the slot carries (-1: none)
  int64_t next_ticket = 0;
  std::map<int64_t, int> async_rc;     // harvested results of finished tickets
  // F1 (policy, PASM, affinity window) and F3 (Eq. 3 workers)
  int32_t policy = 0;              // ARGUS_POLICY_SD / ARGUS_POLICY_PASM
  uint64_t seed = 0;
  uint64_t batch_seq = 0;          // routing calls since argus_set_policy (Philox counter)
  float* d_cdf = nullptr;          // [32][32] float32 running sums of the PASM rows
  int8_t* d_plast = nullptr;       // [32]
  uint8_t* d_aff = nullptr;        // [ARGUS_AFFINITY_WINDOW] ring of optimal options
  int64_t aff_total = 0;           // prompts routed (ring position)
  int32_t n_workers = 0;
  int16_t* d_wlist = nullptr;      // [32][32]
  int32_t* d_wcount = nullptr;     // [32]
  int32_t* d_quota[2] = {nullptr, nullptr};  // [32] quotas broadcast from rank 0 (NCCL mode), per parity
  // fused C-2 over peer memory (k_merge_send): this rank's inbox [header | keys [2][G][max_batch][k]]
  // exported by CUDA IPC; peers' inboxes mapped into this process
  bool p2p = false;
  uint8_t* d_inbox = nullptr;
  uint8_t* peer_inbox[P2P_MAX] = {};  // [world] (own inbox at [rank])
  bool peer_opened[P2P_MAX] = {};
  uint32_t p2p_seq = 0;               // batches exchanged so far (identical on every rank)
  int32_t* d_p2p_ticket = nullptr;
  // pipelined NCCL mode: every collective on one stream in program order (identical on all
  // ranks), and the all-gather + tail of batch b deferred until call b+1 has issued its
  // broadcast, so the comm stream runs bcast(b+1) before AG(b) and the scans run back to back
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_bcast[2] = {nullptr, nullptr};  // batch with parity q broadcast
  cudaEvent_t ev_ag[2] = {nullptr, nullptr};     // its candidate keys all-gathered
  struct Deferred {
    bool valid = false;
    int q = 0, N = 0, P = 0;
    bool qdev = false;
    int32_t quota[32];
    int32_t* option = nullptr;
    uint32_t* idx = nullptr;
    float* score = nullptr;
    float* quality = nullptr;
    uint8_t* status = nullptr;
    argus_route_extra ex{nullptr, nullptr, nullptr};
    bool has_ex = false;
    uint32_t* flags = nullptr;
    int async_slot = -1;  // argus_route_batch_async slot whose result copy follows the tail
    size_t async_bytes = 0;
    uint32_t seq = 0;     // fused exchange: the batch's sequence number
  } def;
  float* d_wtime = nullptr;        // [MAX_WORKERS]
  int32_t* d_queue = nullptr;      // [MAX_WORKERS]
  uint64_t* d_handle = nullptr;    // [capacity] latent handles by cache position (replicated on every rank)
  int32_t* d_optimal = nullptr;    // [max_batch] host-path staging of o_i
  int32_t* d_worker = nullptr;     // [max_batch] host-path staging of worker ids
  CUtensorMap tmap_c;              // TMA descriptor of the bf16 cache shard (64x64 boxes, SW128)
  CUtensorMap tmap_c32;            // same shard, 32x64 boxes (half tiles of the CTA-pair scan)
  bool pair_scan = true;           // N > 128 on CTA pairs (ARGUS_NO_PAIR=1 disables)
  int tail_ysplit = 1;             // CTAs per prompt block of a pipelined tail (ARGUS_TAIL_YSPLIT)
  int scan_reserve = 2;            // pipelined one-slice scans: SMs left to prep / tail (ARGUS_SCAN_RESERVE)
  int scan_reserve_t = -1;         // pipelined multi-slice scans: SMs left to the previous tail (-1 = by N;
                                   // ARGUS_SCAN_RESERVE_T)
  bool migrate = true;             // pair scan: pairs migrate to unfinished slices (ARGUS_NO_MIGRATE=1 disables)
  CUtensorMap tmap_q[2];           // TMA descriptors of the bf16 prompt batches (64x128 boxes, SW128)
  CUtensorMap tmap_q16[2];         // same batches, 64x16 boxes (the transposed small-N scan's B operand)
  bool scan_t = false;             // N <= 64: transposed scan with exact tensor work (ARGUS_SCAN_T)
  bool prompts_bf16 = false;       // the current call's device prompts are bf16 (argus_route_batch_bf16_dev)
  // argus_debug_capture (parity test T2): the scan also writes every exact score here
  float* dbg_scores = nullptr;
  // diagnostics (ARGUS_SCAN_STAMP=<device address>,<launches>): the scans stamp per-CTA
  // timestamps into a caller-owned buffer of launches x 256 CTAs x 4 u64, cyclically
  uint32_t* d_ready = nullptr;     // pipelined one-GPU mode: last batch whose K6 completed (prep stream)
  uint32_t ready_seq = 0;
  bool scan_flag = false;          // one-slice scans wait for d_ready instead of a stream event (ARGUS_SCAN_FLAG=1;
                                   // measured no gain)
  uint64_t* stamp_buf = nullptr;
  int64_t stamp_cap = 0, stamp_seq = 0;
  int64_t dbg_ld = 0;
  // stage profiling (argus_profile_*)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_open;  // (stage, (start, stop))
  double prof_ms[ARGUS_NUM_STAGES] = {};
  int64_t prof_n[ARGUS_NUM_STAGES] = {};
};

constexpr int MAX_WORKERS = 1024;

// ------------------------------------------------------------------ fused exchange inboxes
// Inbox of one rank (bytes): [arrival flags: 2 parities x P2P_MAX senders u32][consumed: 2 u32]
// padded to 256, then keys [2 parities][world][max_batch][k] u64.  Parity = batch sequence & 1.
constexpr size_t INBOX_HDR = 256;
static size_t inbox_bytes(const argus_router* r) {
  return INBOX_HDR + sizeof(uint64_t) * 2 * (size_t)r->cfg.world * r->cfg.max_batch * r->cfg.k;
}
static uint64_t* inbox_keys(const argus_router* r, uint8_t* base, int par) {
  return reinterpret_cast<uint64_t*>(base + INBOX_HDR) + (size_t)par * r->cfg.world * r->cfg.max_batch * r->cfg.k;
}
static uint32_t* inbox_flags(uint8_t* base, int par) { return reinterpret_cast<uint32_t*>(base) + par * P2P_MAX; }
static uint32_t* inbox_consumed(uint8_t* base, int par) {
  return reinterpret_cast<uint32_t*>(base) + 2 * P2P_MAX + par;
}

static P2PSend p2p_send_args(argus_router* r, uint32_t seq) {
  P2PSend a{};
  const int par = (int)(seq & 1u);
  a.G = r->cfg.world;
  a.rank = r->cfg.rank;
  a.seq = seq;
  for (int g = 0; g < a.G; ++g) {
    a.keys[g] = inbox_keys(r, r->peer_inbox[g], par);
    a.flag[g] = inbox_flags(r->peer_inbox[g], par) + r->cfg.rank;
    a.consumed[g] = inbox_consumed(r->peer_inbox[g], par);
  }
  a.err = r->flags_cur ? r->flags_cur : r->d_flags;
  return a;
}

static int p2p_alloc(argus_router* r) {
  if (r->d_inbox) return ARGUS_OK;
  if (cudaMalloc((void**)&r->d_inbox, inbox_bytes(r)) != cudaSuccess ||
      cudaMemset(r->d_inbox, 0, inbox_bytes(r)) != cudaSuccess ||
      cudaMalloc((void**)&r->d_p2p_ticket, sizeof(int32_t)) != cudaSuccess ||
      cudaMemset(r->d_p2p_ticket, 0, sizeof(int32_t)) != cudaSuccess) {
    cudaGetLastError();
    return ARGUS_E_CUDA;
  }
  r->peer_inbox[r->cfg.rank] = r->d_inbox;
  return ARGUS_OK;
}

// map every other rank's inbox (64-byte cudaIpcMemHandle_t each, [world])
static int p2p_open(argus_router* r, const uint8_t* handles) {
  for (int g = 0; g < r->cfg.world; ++g) {
    if (g == r->cfg.rank || r->peer_opened[g]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * g, sizeof(h));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return ARGUS_E_CUDA;
    }
    r->peer_inbox[g] = static_cast<uint8_t*>(p);
    r->peer_opened[g] = true;
  }
  return ARGUS_OK;
}

static void p2p_close(argus_router* r) {
  for (int g = 0; g < P2P_MAX; ++g)
    if (r->peer_opened[g]) {
      cudaIpcCloseMemHandle(r->peer_inbox[g]);
      r->peer_opened[g] = false;
      r->peer_inbox[g] = nullptr;
    }
  if (r->d_inbox) cudaFree(r->d_inbox);
  if (r->d_p2p_ticket) cudaFree(r->d_p2p_ticket);
  r->d_inbox = nullptr;
  r->d_p2p_ticket = nullptr;
  r->p2p = false;
}

// ------------------------------------------------------------------ helpers
#define CU_TRY(r, expr)                                               \
  do {                                                                \
    cudaError_t _e = (expr);                                          \
    if (_e != cudaSuccess) {                                          \
      if (getenv("ARGUS_DEBUG"))                                      \
        fprintf(stderr, "argus: %s -> %s\n", #expr, cudaGetErrorString(_e)); \
      (r)->poisoned = true;                                           \
      return ARGUS_E_CUDA;                                            \
    }                                                                 \
  } while (0)

#define NC_TRY(r, expr)                                               \
  do {                                                                \
    ncclResult_t _e = (expr);                                         \
    if (_e != ncclSuccess) {                                          \
      if (getenv("ARGUS_DEBUG"))                                      \
        fprintf(stderr, "argus: %s -> %s\n", #expr, nccl().GetErrorString(_e)); \
      (r)->poisoned = true;                                           \
      return ARGUS_E_NCCL;                                            \
    }                                                                 \
  } while (0)

#define LAUNCHED(r)                                                   \
  do {                                                                \
    (r)->launches++;                                                  \
    CU_TRY(r, cudaGetLastError());                                    \
  } while (0)

template <class T>
static int dalloc(argus_router* r, T** p, size_t n) {
  if (n == 0) n = 1;
  CU_TRY(r, cudaMalloc((void**)p, n * sizeof(T)));
  return ARGUS_OK;
}

// NCCL collectives in the data path: world > 1 with a unique id, or world == 1 with a
// unique id (a one-rank communicator: the multi-GPU code path on one GPU, for tests)
static bool nccl_mode(const argus_router* r) { return r->comm != nullptr; }

// transpose / round the predictor weights on the device (init time)
__global__ void k_prep_weights(const float* __restrict__ w1, int d, int k, int H, float* __restrict__ W1sT) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = (int64_t)H * (d + k);
  if (tid < n1) {
    const int j = (int)(tid / (d + k)), c = (int)(tid % (d + k));
    if (c >= d) W1sT[(int64_t)(c - d) * H + j] = w1[tid];
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// TMA descriptor of the cache shard: bf16 [rows][d] row-major, box 64 (K) x 64 (rows),
// 128-byte swizzle (matches the UMMA K-major SW128 shared-memory descriptor).
static bool make_tmap(CUtensorMap* m, void* base, int64_t rows, int d, int box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int finite_all(const float* p, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return 0;
  return 1;
}

static int check_state(const argus_router* r) {
  if (!r) return ARGUS_E_INVALID;
  if (r->poisoned) return ARGUS_E_STATE;
  return ARGUS_OK;
}

static cudaEvent_t ev_get(argus_router* r) {
  if (!r->ev_pool.empty()) {
    cudaEvent_t e = r->ev_pool.back();
    r->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Bracket one kernel launch with an event pair when profiling is on.
struct StageScope {
  argus_router* r;
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  StageScope(argus_router* r_, int st, cudaStream_t s_ = nullptr) : r(r_), stage(st), s(s_ ? s_ : r_->stream) {
    if (r->prof) {
      a = ev_get(r);
      b = ev_get(r);
      cudaEventRecord(a, s);
    }
  }
  ~StageScope() {
    if (r->prof && a && b) {
      cudaEventRecord(b, s);
      r->ev_open.push_back({stage, {a, b}});
    }
  }
};

static void prof_collect(argus_router* r) {
  if (r->ev_open.empty()) return;
  cudaStreamSynchronize(r->stream);
  for (cudaStream_t s : {r->prep_stream, r->scan_stream, r->tail_stream})
    if (s) cudaStreamSynchronize(s);
  for (auto& x : r->ev_open) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, x.second.first, x.second.second) == cudaSuccess) {
      r->prof_ms[x.first] += ms;
      r->prof_n[x.first] += 1;
    }
    r->ev_pool.push_back(x.second.first);
    r->ev_pool.push_back(x.second.second);
  }
  r->ev_open.clear();
}

// ------------------------------------------------------------------ C ABI
extern "C" {

int argus_debug_capture(argus_router* r, float* scores_dev, int64_t ld) {
  if (!r || (scores_dev && ld < 1)) return ARGUS_E_INVALID;
  r->dbg_scores = scores_dev;
  r->dbg_ld = scores_dev ? ld : 0;
  return ARGUS_OK;
}

int argus_p2p_export(argus_router* r, void* handle_out) {
  int rc = check_state(r);
  if (rc) return rc;
  if (!handle_out || r->cfg.world < 2 || r->comm || r->cfg.k == 0 || r->cfg.world > P2P_MAX) return ARGUS_E_INVALID;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  rc = p2p_alloc(r);
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  CU_TRY(r, cudaIpcGetMemHandle(&h, r->d_inbox));
  memset(handle_out, 0, 64);
  memcpy(handle_out, &h, sizeof(h));
  return ARGUS_OK;
}

int argus_p2p_connect(argus_router* r, const void* handles) {
  int rc = check_state(r);
  if (rc) return rc;
  if (!handles || r->cfg.world < 2 || r->comm || !r->d_inbox) return ARGUS_E_INVALID;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  rc = p2p_open(r, static_cast<const uint8_t*>(handles));
  if (rc) return rc;
  r->p2p = true;
  return ARGUS_OK;
}

int argus_profile_enable(argus_router* r, int on) {
  if (!r) return ARGUS_E_INVALID;
  cudaSetDevice(r->cfg.device);
  prof_collect(r);
  r->prof = on != 0;
  return ARGUS_OK;
}

int argus_profile_read(argus_router* r, int stage, double* total_ms, int64_t* launches) {
  if (!r || stage < 0 || stage >= ARGUS_NUM_STAGES) return ARGUS_E_INVALID;
  cudaSetDevice(r->cfg.device);
  prof_collect(r);
  if (total_ms) *total_ms = r->prof_ms[stage];
  if (launches) *launches = r->prof_n[stage];
  r->prof_ms[stage] = 0.0;
  r->prof_n[stage] = 0;
  return ARGUS_OK;
}

const char* argus_strerror(int code) {
  switch (code) {
    case ARGUS_OK: return "ok";
    case ARGUS_W_OVERFLOW: return "warning: some prompt found no admissible quota (assigned option 0)";
    case ARGUS_E_INVALID: return "invalid argument, non-finite value or zero-norm vector";
    case ARGUS_E_CAPACITY: return "cache capacity exceeded";
    case ARGUS_E_CUDA: return "CUDA error (router poisoned)";
    case ARGUS_E_NCCL: return "NCCL error (router poisoned)";
    case ARGUS_E_STATE: return "router poisoned or call invalid in this mode";
    case ARGUS_E_UNIMPLEMENTED: return "not implemented";
    default: return "unknown argus code";
  }
}

int argus_nccl_unique_id(void* out128) {
  if (!out128) return ARGUS_E_INVALID;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (!nccl().ok || nccl().GetUniqueId(&id) != ncclSuccess) return ARGUS_E_NCCL;
  memcpy(out128, &id, sizeof(id));
  return ARGUS_OK;
}

int argus_quota_from_fractions(const double* f, int32_t L, int32_t N, int32_t* c_out) {
  if (!f || !c_out || L <= 0 || L > 64 || N < 0) return ARGUS_E_INVALID;
  double S = 0.0;
  for (int32_t v = 0; v < L; ++v) {
    if (!(f[v] >= 0.0) || !std::isfinite(f[v])) return ARGUS_E_INVALID;
    S += f[v];
  }
  if (!(S > 0.0)) return ARGUS_E_INVALID;
  double fr[64];
  int64_t used = 0;
  for (int32_t v = 0; v < L; ++v) {
    const double t = (f[v] * (double)N) / S;
    const double fl = std::floor(t);
    c_out[v] = (int32_t)fl;
    fr[v] = t - fl;
    used += c_out[v];
  }
  int64_t left = (int64_t)N - used;
  while (left > 0) {  // one leftover unit each to the largest fractional parts, ties -> lower v
    int32_t best = -1;
    for (int32_t v = 0; v < L; ++v)
      if (fr[v] >= 0.0 && (best < 0 || fr[v] > fr[best])) best = v;
    c_out[best] += 1;
    fr[best] = -1.0;
    --left;
  }
  while (left < 0) {  // rounding guard: remove from the smallest parts, ties -> higher v
    int32_t worst = -1;
    for (int32_t v = L - 1; v >= 0; --v)
      if (c_out[v] > 0 && (worst < 0 || fr[v] < fr[worst])) worst = v;
    c_out[worst] -= 1;
    fr[worst] = 2.0;
    ++left;
  }
  return ARGUS_OK;
}

int argus_route_destroy(argus_router* r) {
  if (!r) return ARGUS_E_INVALID;
  cudaSetDevice(r->cfg.device);
  if (r->stream) cudaStreamSynchronize(r->stream);
  for (cudaStream_t s : {r->prep_stream, r->scan_stream, r->tail_stream, r->comm_stream})
    if (s) cudaStreamSynchronize(s);
  void* ptrs[] = {r->d_kskip, r->d_pth, r->d_gate, r->d_W1xF, r->d_W1sT, r->d_b1, r->d_W2, r->d_b2, r->d_h,
                  r->d_mlp_cnt, r->d_tail_cnt, r->d_Cb, r->d_invc, r->d_Xstage, r->d_Xb[0], r->d_Xb[1],
                  r->d_invq[0], r->d_invq[1], r->d_partial[0], r->d_partial[1], r->d_keys[0], r->d_keys[1],
                  r->d_keys_all[0], r->d_keys_all[1], r->d_quota[0], r->d_quota[1],
                  r->d_score, r->d_idx, r->d_rhat, r->d_pref, r->d_ccount, r->d_cmask, r->d_status, r->d_option,
                  r->d_order, r->d_gthr[0], r->d_gthr[1], r->d_ctr[0], r->d_ctr[1], r->d_cdf, r->d_plast,
                  r->d_aff, r->d_wlist, r->d_wcount, r->d_wtime, r->d_queue, r->d_optimal, r->d_worker,
                  r->d_handle, r->d_Xasync[0], r->d_Xasync[1], r->d_Xasync[2], r->d_Xasync[3], r->d_oasync[0],
                  r->d_oasync[1], r->d_oasync[2], r->d_oasync[3], r->d_ready};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (r->h_flags) cudaFreeHost(r->h_flags);
  if (r->h_outblk) cudaFreeHost(r->h_outblk);
  if (r->h_fasync) cudaFreeHost(r->h_fasync);
  if (r->d2h_stream) cudaStreamSynchronize(r->d2h_stream);
  for (cudaEvent_t e : r->ev_async)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : r->ev_done)
    if (e) cudaEventDestroy(e);
  for (uint8_t* h : r->h_oasync)
    if (h) cudaFreeHost(h);
  if (r->d2h_stream) cudaStreamDestroy(r->d2h_stream);
  if (r->d_outblk) cudaFree(r->d_outblk);
  for (auto& x : r->ev_open) { cudaEventDestroy(x.second.first); cudaEventDestroy(x.second.second); }
  for (auto e : r->ev_pool) cudaEventDestroy(e);
  p2p_close(r);
  if (r->comm) nccl().CommDestroy(r->comm);
  for (int q = 0; q < 2; ++q)
    for (cudaEvent_t e : {r->ev_in[q], r->ev_prep[q], r->ev_scan[q], r->ev_tail[q], r->ev_bcast[q], r->ev_ag[q]})
      if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {r->prep_stream, r->scan_stream, r->tail_stream, r->comm_stream})
    if (s) cudaStreamDestroy(s);
  if (r->own_stream && r->stream) cudaStreamDestroy(r->stream);
  delete r;
  return ARGUS_OK;
}

int argus_route_init(const argus_config* cfg, const argus_option* opts, const float* w1,
                     const float* b1, const float* w2, const float* b2, argus_router** out) {
  if (!cfg || !out) return ARGUS_E_INVALID;
  *out = nullptr;
  const argus_config& c = *cfg;
  if (c.d < 64 || c.d % 64 != 0 || !scan_supported(c.d)) return ARGUS_E_INVALID;
  if (c.k < 0 || c.k > 8) return ARGUS_E_INVALID;  // k = 0: SM mode (no cache)
  if (c.evict != 0 && c.evict != 1) return ARGUS_E_INVALID;
  if (c.evict && (c.capacity < c.world || c.capacity % c.world != 0)) return ARGUS_E_INVALID;
  if (c.L < 1 || c.L > 32) return ARGUS_E_INVALID;
  if (c.hidden < 32 || c.hidden > 1024 || c.hidden % 32 != 0) return ARGUS_E_INVALID;
  if (tail_smem_bytes(c.d, c.k, c.hidden, c.L, c.max_batch, 148) > 220 * 1024) return ARGUS_E_INVALID;
  if (c.max_batch < 1 || c.max_batch > 8192) return ARGUS_E_INVALID;
  if (c.capacity < 0 || c.capacity > 0xFFFFFFFELL) return ARGUS_E_INVALID;
  if (!(c.delta > 0.f && c.delta <= 1.f)) return ARGUS_E_INVALID;
  if (c.world < 1 || c.rank < 0 || c.rank >= c.world || c.device < 0) return ARGUS_E_INVALID;
  const bool root_data = (c.world == 1 || c.rank == 0 || c.nccl_unique_id == nullptr);
  if (root_data) {
    if (!opts || !w1 || !b1 || !w2 || !b2) return ARGUS_E_INVALID;
    if (opts[0].k_skip != 0) return ARGUS_E_INVALID;
    for (int v = 0; v < c.L; ++v) {
      if (c.k == 0 && opts[v].k_skip != 0) return ARGUS_E_INVALID;  // SM mode: model variants only
      if (opts[v].k_skip < 0 || opts[v].k_skip >= 50) return ARGUS_E_INVALID;
      if (!std::isfinite(opts[v].p_th_qpm)) return ARGUS_E_INVALID;
      if (v > 0 && opts[v].p_th_qpm < opts[v - 1].p_th_qpm) return ARGUS_E_INVALID;
      if (std::isnan(opts[v].sim_gate)) return ARGUS_E_INVALID;
    }
    if (!finite_all(w1, (int64_t)c.hidden * (c.d + c.k)) || !finite_all(b1, c.hidden) ||
        !finite_all(w2, (int64_t)c.L * c.hidden) || !finite_all(b2, c.L))
      return ARGUS_E_INVALID;
  }

  argus_router* r = new (std::nothrow) argus_router();
  if (!r) return ARGUS_E_CUDA;
  r->cfg = c;
  r->cfg.nccl_unique_id = nullptr;
  int rc;
#define TRY_RC(x)                   \
  do {                              \
    if ((rc = (x)) != ARGUS_OK) {   \
      argus_route_destroy(r);       \
      return rc;                    \
    }                               \
  } while (0)
  if (cudaSetDevice(c.device) != cudaSuccess) { delete r; return ARGUS_E_CUDA; }
  cudaDeviceGetAttribute(&r->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  if (c.stream) {
    r->stream = (cudaStream_t)c.stream;
  } else {
    if (cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking) != cudaSuccess) { delete r; return ARGUS_E_CUDA; }
    r->own_stream = true;
  }
  // pipelining: one GPU, or NCCL mode (one communicator, collectives in program order on
  // the comm stream); not the external mode, whose caller moves the keys itself
  r->pipe = c.pipeline != 0 && (c.world == 1 || c.nccl_unique_id != nullptr);
  r->pair_scan = getenv("ARGUS_NO_PAIR") == nullptr;
  if (const char* e = getenv("ARGUS_TAIL_YSPLIT")) r->tail_ysplit = atoi(e);
  if (const char* e = getenv("ARGUS_SCAN_RESERVE")) r->scan_reserve = std::min(std::max(atoi(e), 0), 16);
  if (const char* e = getenv("ARGUS_SCAN_FLAG")) r->scan_flag = atoi(e) != 0;
  if (const char* e = getenv("ARGUS_SCAN_T")) r->scan_t = atoi(e) != 0;
  if (const char* e = getenv("ARGUS_SCAN_STAMP")) {
    unsigned long long addr = 0;
    long long cap = 0;
    if (sscanf(e, "%llx,%lld", &addr, &cap) == 2 && addr && cap > 0) {
      r->stamp_buf = reinterpret_cast<uint64_t*>(addr);
      r->stamp_cap = cap;
    }
  }
  if (const char* e = getenv("ARGUS_SCAN_RESERVE_T")) r->scan_reserve_t = std::min(std::max(atoi(e), -1), 32);
  r->migrate = getenv("ARGUS_NO_MIGRATE") == nullptr;
  if (r->pipe) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    bool ok = cudaStreamCreateWithPriority(&r->prep_stream, cudaStreamNonBlocking, hi) == cudaSuccess &&
              cudaStreamCreateWithPriority(&r->scan_stream, cudaStreamNonBlocking, lo) == cudaSuccess &&
              cudaStreamCreateWithPriority(&r->tail_stream, cudaStreamNonBlocking, hi) == cudaSuccess;
    if (ok && c.nccl_unique_id) ok = cudaStreamCreateWithPriority(&r->comm_stream, cudaStreamNonBlocking, hi) == cudaSuccess;
    for (int q = 0; q < 2 && ok; ++q)
      ok = cudaEventCreateWithFlags(&r->ev_bcast[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&r->ev_ag[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&r->ev_in[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&r->ev_prep[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&r->ev_scan[q], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&r->ev_tail[q], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) { argus_route_destroy(r); return ARGUS_E_CUDA; }
  }
  if (c.nccl_unique_id) {
    ncclUniqueId id;
    memcpy(&id, c.nccl_unique_id, sizeof(id));
    if (!nccl().ok || nccl().CommInitRank(&r->comm, c.world, id, c.rank) != ncclSuccess) {
      r->comm = nullptr;
      argus_route_destroy(r);
      return ARGUS_E_NCCL;
    }
  }
  const int d = c.d, k = c.k, L = c.L, H = c.hidden, G = c.world;
  r->cap_local = (c.capacity + G - 1) / G;
  r->n_pad_max = ((c.max_batch + 127) / 128) * 128;
  const int64_t stage_rows = std::max<int64_t>(c.max_batch, INSERT_CHUNK);
  TRY_RC(dalloc(r, &r->d_kskip, L));
  TRY_RC(dalloc(r, &r->d_pth, L));
  TRY_RC(dalloc(r, &r->d_gate, L));
  TRY_RC(dalloc(r, &r->d_W1xF, (size_t)d * H));
  TRY_RC(dalloc(r, &r->d_W1sT, (size_t)k * H));
  TRY_RC(dalloc(r, &r->d_b1, H));
  TRY_RC(dalloc(r, &r->d_W2, (size_t)H * L));
  const int64_t n16 = ((int64_t)c.max_batch + 15) / 16 * 16;
  TRY_RC(dalloc(r, &r->d_h, (size_t)n16 * H));
  TRY_RC(dalloc(r, &r->d_mlp_cnt, (size_t)n16 / 16));
  TRY_RC(dalloc(r, &r->d_tail_cnt, 1));
  r->tail_smem = tail_smem_bytes(d, k, H, L, c.max_batch, std::max(r->num_sms, c.world));
  TRY_RC(dalloc(r, &r->d_b2, L));
  TRY_RC(dalloc(r, &r->d_Cb, (size_t)(r->cap_local + 256) * d));
  TRY_RC(dalloc(r, &r->d_invc, (size_t)r->cap_local + 256));
  TRY_RC(dalloc(r, &r->d_Xstage, (size_t)stage_rows * d));
  // P lists per prompt with P <= num_sms / slices and N <= 128 * slices
  // lists per prompt x prompts: <= num_sms * 128 for the one-slice-per-CTA scan; the
  // pair scan with migration adds MAX_VISITS slots per pair slice
  // (home_max + MAX_VISITS) * N <= (num_sms / 2 / pslices + 1 + MAX_VISITS) * 256 * pslices
  // pair scan with migration: P = home + floaters + MAX_VISITS <= num_sms / 2 / pslices +
  // pslices + MAX_VISITS, times N <= 256 * pslices
  r->partial_lists = (int64_t)r->num_sms * 128 + (int64_t)(MAX_VISITS + 1 + MAX_SLICES / 2) *
                                                     (((int64_t)c.max_batch + 255) / 256 * 256);
  for (int q = 0; q < 2; ++q) {
    TRY_RC(dalloc(r, &r->d_Xb[q], (size_t)r->n_pad_max * d));
    TRY_RC(dalloc(r, &r->d_partial[q], (size_t)r->partial_lists * k));
  }
  TRY_RC(dalloc(r, &r->d_ready, 1));
  CU_TRY(r, cudaMemset(r->d_ready, 0, sizeof(uint32_t)));
  for (int q = 0; q < 2; ++q) {
    TRY_RC(dalloc(r, &r->d_invq[q], (size_t)r->n_pad_max));
    TRY_RC(dalloc(r, &r->d_gthr[q], (size_t)r->n_pad_max));
    TRY_RC(dalloc(r, &r->d_ctr[q], CTR_WORDS));
  }
  for (int q = 0; q < 2; ++q) {
    TRY_RC(dalloc(r, &r->d_keys[q], (size_t)c.max_batch * k));
    TRY_RC(dalloc(r, &r->d_keys_all[q], (size_t)G * c.max_batch * k));
    TRY_RC(dalloc(r, &r->d_quota[q], 32));
  }
  TRY_RC(dalloc(r, &r->d_score, (size_t)c.max_batch * k));
  TRY_RC(dalloc(r, &r->d_idx, (size_t)c.max_batch * k));
  TRY_RC(dalloc(r, &r->d_rhat, (size_t)c.max_batch * L));
  TRY_RC(dalloc(r, &r->d_pref, (size_t)c.max_batch * 32));
  TRY_RC(dalloc(r, &r->d_ccount, (size_t)c.max_batch));
  TRY_RC(dalloc(r, &r->d_cmask, (size_t)c.max_batch));
  TRY_RC(dalloc(r, &r->d_status, (size_t)c.max_batch));
  TRY_RC(dalloc(r, &r->d_option, (size_t)c.max_batch));
  TRY_RC(dalloc(r, &r->d_order, (size_t)c.max_batch));
  TRY_RC(dalloc(r, &r->d_cdf, 32 * 32));
  TRY_RC(dalloc(r, &r->d_plast, 32));
  TRY_RC(dalloc(r, &r->d_aff, ARGUS_AFFINITY_WINDOW));
  TRY_RC(dalloc(r, &r->d_wlist, 32 * 32));
  TRY_RC(dalloc(r, &r->d_wcount, 32));
  TRY_RC(dalloc(r, &r->d_wtime, MAX_WORKERS));
  TRY_RC(dalloc(r, &r->d_queue, MAX_WORKERS));
  TRY_RC(dalloc(r, &r->d_optimal, (size_t)c.max_batch));
  TRY_RC(dalloc(r, &r->d_handle, (size_t)std::max<int64_t>(c.capacity, 1)));
  for (int q = 0; q < argus_router::NASYNC; ++q) {
    TRY_RC(dalloc(r, &r->d_Xasync[q], (size_t)c.max_batch * d));
    TRY_RC(dalloc(r, &r->d_oasync[q], 16 + 16 * 8 + (size_t)c.max_batch * (4 + 8 * (size_t)k + 4 * (size_t)L + 1)));
    if (cudaMallocHost((void**)&r->h_oasync[q], 16 + 16 * 8 + (size_t)c.max_batch * (4 + 8 * (size_t)k + 4 * (size_t)L + 1)) !=
            cudaSuccess ||
        cudaEventCreateWithFlags(&r->ev_done[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&r->ev_async[q], cudaEventDisableTiming) != cudaSuccess) {
      argus_route_destroy(r);
      return ARGUS_E_CUDA;
    }
  }
  // [NASYNC] flag words read back + one constant zero word
  if (cudaMallocHost((void**)&r->h_fasync, (argus_router::NASYNC + 1) * sizeof(uint32_t)) != cudaSuccess) {
    argus_route_destroy(r);
    return ARGUS_E_CUDA;
  }
  for (int q = 0; q <= argus_router::NASYNC; ++q) r->h_fasync[q] = 0u;
  if (cudaStreamCreateWithFlags(&r->d2h_stream, cudaStreamNonBlocking) != cudaSuccess) {
    argus_route_destroy(r);
    return ARGUS_E_CUDA;
  }
  TRY_RC(dalloc(r, &r->d_worker, (size_t)c.max_batch));
  r->outblk_bytes = 16 + 16 * 8 + (size_t)c.max_batch * (4 + 16 * (size_t)k + 4 * (size_t)L + 1 + 8);
  TRY_RC(dalloc(r, &r->d_outblk, r->outblk_bytes));
  r->d_flags = reinterpret_cast<uint32_t*>(r->d_outblk);
  if (cudaMallocHost((void**)&r->h_outblk, r->outblk_bytes) != cudaSuccess) { argus_route_destroy(r); return ARGUS_E_CUDA; }
  if (cudaMallocHost((void**)&r->h_flags, sizeof(uint32_t)) != cudaSuccess) { argus_route_destroy(r); return ARGUS_E_CUDA; }
  if (!make_tmap(&r->tmap_c, r->d_Cb, r->cap_local + 256, d, 64) ||
      !make_tmap(&r->tmap_c32, r->d_Cb, r->cap_local + 256, d, 32) ||
      !make_tmap(&r->tmap_q[0], r->d_Xb[0], r->n_pad_max, d, 128) ||
      !make_tmap(&r->tmap_q[1], r->d_Xb[1], r->n_pad_max, d, 128) ||
      !make_tmap(&r->tmap_q16[0], r->d_Xb[0], r->n_pad_max, d, 16) ||
      !make_tmap(&r->tmap_q16[1], r->d_Xb[1], r->n_pad_max, d, 16)) {
    argus_route_destroy(r);
    return ARGUS_E_CUDA;
  }
  // zero the cache tail so TMA / vector loads past M never see garbage
  if (cudaMemsetAsync(r->d_Cb, 0, (size_t)(r->cap_local + 256) * d * sizeof(__nv_bfloat16), r->stream) != cudaSuccess ||
      cudaMemsetAsync(r->d_invc, 0, (size_t)(r->cap_local + 256) * sizeof(float), r->stream) != cudaSuccess ||
      cudaMemsetAsync(r->d_flags, 0, sizeof(uint32_t), r->stream) != cudaSuccess ||
      cudaMemsetAsync(r->d_mlp_cnt, 0, sizeof(int32_t) * (size_t)(n16 / 16), r->stream) != cudaSuccess ||
      cudaMemsetAsync(r->d_tail_cnt, 0, sizeof(int32_t), r->stream) != cudaSuccess ||
      cudaMemsetAsync(r->d_handle, 0, sizeof(uint64_t) * (size_t)std::max<int64_t>(c.capacity, 1), r->stream) !=
          cudaSuccess) {
    argus_route_destroy(r);
    return ARGUS_E_CUDA;
  }

  // options + weights: staged through the fp32 staging buffer, transposed on device
  std::vector<int32_t> ks(L);
  std::vector<float> pth(L), gate(L);
  if (root_data) {
    for (int v = 0; v < L; ++v) {
      ks[v] = opts[v].k_skip;
      pth[v] = opts[v].p_th_qpm;
      gate[v] = opts[v].k_skip == 0 ? -INFINITY : opts[v].sim_gate;
    }
  }
  float* d_w1 = nullptr;
  float* d_w2 = r->d_W2;  // W2 is used in its caller layout [L][H]
  TRY_RC(dalloc(r, &d_w1, (size_t)H * (d + k)));
  auto cleanup_tmp = [&]() { cudaFree(d_w1); };
  if (root_data) {
    if (cudaMemcpy(r->d_kskip, ks.data(), 4 * L, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(r->d_pth, pth.data(), 4 * L, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(r->d_gate, gate.data(), 4 * L, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d_w1, w1, sizeof(float) * H * (d + k), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d_w2, w2, sizeof(float) * L * H, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(r->d_b1, b1, sizeof(float) * H, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(r->d_b2, b2, sizeof(float) * L, cudaMemcpyHostToDevice) != cudaSuccess) {
      cleanup_tmp();
      argus_route_destroy(r);
      return ARGUS_E_CUDA;
    }
  }
  if (nccl_mode(r)) {  // C-4: rank 0's table and weights to every rank
    nccl().GroupStart();
    nccl().Broadcast(r->d_kskip, r->d_kskip, L, ncclInt32, 0, r->comm, r->stream);
    nccl().Broadcast(r->d_pth, r->d_pth, L, ncclFloat32, 0, r->comm, r->stream);
    nccl().Broadcast(r->d_gate, r->d_gate, L, ncclFloat32, 0, r->comm, r->stream);
    nccl().Broadcast(d_w1, d_w1, (size_t)H * (d + k), ncclFloat32, 0, r->comm, r->stream);
    nccl().Broadcast(d_w2, d_w2, (size_t)L * H, ncclFloat32, 0, r->comm, r->stream);
    nccl().Broadcast(r->d_b1, r->d_b1, H, ncclFloat32, 0, r->comm, r->stream);
    if (nccl().GroupEnd() != ncclSuccess ||
        nccl().Broadcast(r->d_b2, r->d_b2, L, ncclFloat32, 0, r->comm, r->stream) != ncclSuccess) {
      cleanup_tmp();
      argus_route_destroy(r);
      return ARGUS_E_NCCL;
    }
  }
  {
    const int64_t tot = (int64_t)H * (d + k);
    k_prep_weights<<<(unsigned)((tot + 255) / 256), 256, 0, r->stream>>>(d_w1, d, k, H, r->d_W1sT);
    launch_prep_w1_frag(d_w1, d, k, H, r->d_W1xF, r->stream);
    r->launches += 2;
  }
  if (cudaStreamSynchronize(r->stream) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    cleanup_tmp();
    argus_route_destroy(r);
    return ARGUS_E_CUDA;
  }
  cleanup_tmp();
  // NCCL mode: the fused exchange over peer memory replaces the all-gather when every rank
  // can map every other rank's inbox (all ranks decide together: a MIN all-reduce)
  if (nccl_mode(r) && k > 0 && G <= P2P_MAX && !getenv("ARGUS_NO_P2P")) {
    int ok = p2p_alloc(r) == ARGUS_OK;
    uint8_t* d_h = nullptr;
    int32_t* d_ok = nullptr;
    std::vector<uint8_t> hh(64 * (size_t)G, 0);
    if (cudaMalloc((void**)&d_h, hh.size()) != cudaSuccess || cudaMalloc((void**)&d_ok, 4) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(d_h);
      argus_route_destroy(r);
      return ARGUS_E_CUDA;
    }
    cudaIpcMemHandle_t h{};
    if (ok && G > 1) ok = cudaIpcGetMemHandle(&h, r->d_inbox) == cudaSuccess;
    memcpy(hh.data() + 64 * (size_t)c.rank, &h, sizeof(h));
    bool nc = cudaMemcpy(d_h, hh.data(), hh.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
              nccl().AllGather(d_h + 64 * (size_t)c.rank, d_h, 64, ncclUint8, r->comm, r->stream) == ncclSuccess &&
              cudaMemcpy(hh.data(), d_h, hh.size(), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (nc && ok) ok = p2p_open(r, hh.data()) == ARGUS_OK;
    int32_t okv = ok ? 1 : 0;
    nc = nc && cudaMemcpy(d_ok, &okv, 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         nccl().AllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, r->comm, r->stream) == ncclSuccess &&
         cudaMemcpy(&okv, d_ok, 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d_h);
    cudaFree(d_ok);
    cudaGetLastError();
    if (!nc) {
      argus_route_destroy(r);
      return ARGUS_E_NCCL;
    }
    if (okv) {
      r->p2p = true;
    } else {
      p2p_close(r);  // some rank cannot map its peers: every rank keeps the NCCL all-gather
      if (getenv("ARGUS_DEBUG")) fprintf(stderr, "argus: fused peer exchange unavailable, using ncclAllGather\n");
    }
  }
#undef TRY_RC
  *out = r;
  return ARGUS_OK;
}

int argus_cache_size(const argus_router* r, int64_t* m_out) {
  if (!r || !m_out) return ARGUS_E_INVALID;
  *m_out = r->m_global;
  return ARGUS_OK;
}

int argus_launch_count(const argus_router* r, int64_t* n_out) {
  if (!r || !n_out) return ARGUS_E_INVALID;
  *n_out = r->launches;
  return ARGUS_OK;
}

int argus_get_stream(const argus_router* r, void** stream_out) {
  if (!r || !stream_out) return ARGUS_E_INVALID;
  *stream_out = (void*)r->stream;
  return ARGUS_OK;
}

static int insert_impl(argus_router* r, const float* emb, int64_t n, int64_t* first_id, bool on_device,
                       const uint64_t* handles = nullptr) {
  int rc = check_state(r);
  if (rc) return rc;
  if (n < 0) return ARGUS_E_INVALID;
  rc = argus_route_join(r, nullptr);  // pipelined tails may still OR their flags
  if (rc) return rc;
  const bool root = r->cfg.rank == 0 || !nccl_mode(r);
  if (root && n > 0 && !emb) return ARGUS_E_INVALID;
  const int64_t cap = r->cfg.capacity;
  if (!r->cfg.evict && r->m_global + n > cap) return ARGUS_E_CAPACITY;
  if (r->cfg.evict && r->m_global + n > (int64_t)0xFFFFFFFE) return ARGUS_E_CAPACITY;  // 32-bit global ids
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  const int d = r->cfg.d;
  // with eviction an insert overwrites live rows, so validate everything first (dry
  // pass, no writes); without it rows past M are simply not yet counted
  const int passes = r->cfg.evict ? 2 : 1;
  // with eviction only the last `cap` rows of this call survive
  const int64_t skip = (r->cfg.evict && n > cap) ? n - cap : 0;
  uint32_t fl = 0;
  for (int pass = 0; pass < passes; ++pass) {
    const bool dry = passes == 2 && pass == 0;
    CU_TRY(r, cudaMemsetAsync(r->d_flags, 0, 4, r->stream));
    for (int64_t off = dry ? 0 : skip; off < n; off += INSERT_CHUNK) {
      const int64_t m = std::min<int64_t>(INSERT_CHUNK, n - off);
      const float* src = nullptr;
      if (root) {
        if (on_device && !nccl_mode(r)) {
          src = emb + off * d;
        } else {
          CU_TRY(r, cudaMemcpyAsync(r->d_Xstage, emb + off * d, sizeof(float) * m * d,
                                    on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, r->stream));
          src = r->d_Xstage;
        }
      } else {
        src = r->d_Xstage;
      }
      if (nccl_mode(r))  // C-3: rank 0's rows to every rank; each keeps its stripe
        NC_TRY(r, nccl().Broadcast(r->d_Xstage, r->d_Xstage, (size_t)m * d, ncclFloat32, 0, r->comm, r->stream));
      {
        StageScope sc(r, ARGUS_STAGE_INSERT);
        launch_insert_rows(src, m, r->m_global + off, d, r->cfg.rank, r->cfg.world, cap, dry, r->d_Cb, r->d_invc,
                           r->d_flags, r->stream);
      }
      LAUNCHED(r);
    }
    CU_TRY(r, cudaMemcpyAsync(r->h_flags, r->d_flags, 4, cudaMemcpyDeviceToHost, r->stream));
    CU_TRY(r, cudaStreamSynchronize(r->stream));
    fl = *r->h_flags;
    if (nccl_mode(r)) {  // every rank must agree on validity (each saw only its stripe)
      CU_TRY(r, cudaMemcpyAsync(r->d_flags, &fl, 4, cudaMemcpyHostToDevice, r->stream));
      NC_TRY(r, nccl().AllReduce(r->d_flags, r->d_flags, 1, ncclUint32, ncclMax, r->comm, r->stream));
      CU_TRY(r, cudaMemcpyAsync(r->h_flags, r->d_flags, 4, cudaMemcpyDeviceToHost, r->stream));
      CU_TRY(r, cudaStreamSynchronize(r->stream));
      fl = *r->h_flags;
    }
    CU_TRY(r, cudaMemsetAsync(r->d_flags, 0, 4, r->stream));
    if (fl & FLAG_INVALID_INPUT) return ARGUS_E_INVALID;  // cache unchanged (M not advanced / dry pass)
  }
  // latent handles ("intermediate noise (144 KB) stored in ... EFS"): one u64 per
  // entry at its cache position, replicated on every rank; absent handles read 0
  if (n > skip) {
    std::vector<uint64_t> hs((size_t)(n - skip), 0);
    if (root && handles) memcpy(hs.data(), handles + skip, sizeof(uint64_t) * hs.size());
    uint64_t* dst_stage = reinterpret_cast<uint64_t*>(r->d_Xstage);
    for (int64_t off = 0; off < (int64_t)hs.size();) {
      const int64_t g = r->m_global + skip + off;
      const int64_t pos = g % std::max<int64_t>(cap, 1);
      const int64_t run = std::min<int64_t>({(int64_t)hs.size() - off, cap - pos, (int64_t)INSERT_CHUNK});
      if (nccl_mode(r)) {
        CU_TRY(r, cudaMemcpyAsync(dst_stage, hs.data() + off, sizeof(uint64_t) * run, cudaMemcpyHostToDevice,
                                  r->stream));
        NC_TRY(r, nccl().Broadcast(dst_stage, r->d_handle + pos, (size_t)run, ncclUint64, 0, r->comm, r->stream));
      } else {
        CU_TRY(r, cudaMemcpyAsync(r->d_handle + pos, hs.data() + off, sizeof(uint64_t) * run,
                                  cudaMemcpyHostToDevice, r->stream));
      }
      off += run;
    }
    CU_TRY(r, cudaStreamSynchronize(r->stream));  // hs is a host temporary
  }
  if (first_id) *first_id = r->m_global;
  r->m_global += n;
  return ARGUS_OK;
}

int argus_cache_insert_h(argus_router* r, const float* emb, const uint64_t* handles, int64_t n, int64_t* first_id) {
  return insert_impl(r, emb, n, first_id, false, handles);
}

int argus_cache_insert(argus_router* r, const float* emb, int64_t n, int64_t* first_id) {
  return insert_impl(r, emb, n, first_id, false);
}

int argus_cache_insert_dev(argus_router* r, const float* emb_dev, int64_t n, int64_t* first_id) {
  return insert_impl(r, emb_dev, n, first_id, true);
}

static int64_t live_rows(const argus_router* r) {  // global entries currently held
  return std::min<int64_t>(r->m_global, r->cfg.capacity);
}
static int64_t local_rows(const argus_router* r) {
  const int64_t G = r->cfg.world, rk = r->cfg.rank;
  return (live_rows(r) + G - 1 - rk) / G;
}
// ring eviction: cache position of the oldest live entry (age index 0)
static int64_t ring_head(const argus_router* r) {
  return (r->cfg.evict && r->m_global > r->cfg.capacity) ? r->m_global % r->cfg.capacity : 0;
}

// K6 + scan (+ K5 local merge into keys_dev when keys_dev != NULL).  *P_out receives
// the number of per-range candidate lists left in d_partial.
// q selects the double-buffered per-batch buffers (bf16 prompts, candidate lists).
// quota_bcast (NCCL mode, every rank alike): rank 0's host quotas go to d_quota and join
// the C-1 broadcast; the tail then reads them from there.
static int partial_impl(argus_router* r, const float* prompts_dev, int32_t N, uint64_t* keys_dev, int32_t* P_out,
                        int q, cudaStream_t s_prep = nullptr, cudaStream_t s_scan = nullptr,
                        bool quota_bcast = false, const int32_t* quota = nullptr, uint32_t send_seq = 0);

int argus_route_partial_dev(argus_router* r, const float* prompts_dev, int32_t N, uint64_t* keys_dev) {
  if (!keys_dev) return ARGUS_E_INVALID;
  int32_t P = 0;
  int rc = argus_route_join(r, nullptr);  // pipelined tails still read the parity-0 buffers
  if (rc) return rc;
  return partial_impl(r, prompts_dev, N, keys_dev, &P, 0);
}

// With s_prep / s_scan (pipelined mode) prep and scan go to those streams, without
// the programmatic (PDL) relaxation, and the caller inserts the events between them.
static int partial_impl(argus_router* r, const float* prompts_dev, int32_t N, uint64_t* keys_dev, int32_t* P_out,
                        int q, cudaStream_t s_prep, cudaStream_t s_scan, bool quota_bcast, const int32_t* quota,
                        uint32_t send_seq) {
  const bool pipelined = s_prep != nullptr;
  if (!s_prep) s_prep = r->stream;
  if (!s_scan) s_scan = r->stream;
  int rc = check_state(r);
  if (rc) return rc;
  if (N < 1 || N > r->cfg.max_batch) return ARGUS_E_INVALID;
  const bool root = r->cfg.rank == 0 || !nccl_mode(r);
  if (root && !prompts_dev) return ARGUS_E_INVALID;
  if (quota_bcast && (!nccl_mode(r) || (root && !quota))) return ARGUS_E_INVALID;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  const int d = r->cfg.d, k = r->cfg.k;
  const int n_pad = ((N + 127) / 128) * 128;
  // K6 on the root (or everywhere in external mode), then C-1 broadcast of the bf16 batch
  if (root) {
    StageScope sc(r, ARGUS_STAGE_PREP, s_prep);
    launch_prep_queries(prompts_dev, r->prompts_bf16, N, n_pad, d, r->d_Xb[q], r->d_invq[q], r->d_gthr[q], r->d_ctr[q],
                        r->flags_cur ? r->flags_cur : r->d_flags,
                        s_prep, !pipelined, quota_bcast ? quota : nullptr, r->cfg.L, r->d_quota[q]);
    LAUNCHED(r);
  }
  if (!root) {
    CU_TRY(r, cudaMemsetAsync(r->d_gthr[q], 0, sizeof(uint64_t) * (size_t)n_pad, s_prep));
    CU_TRY(r, cudaMemsetAsync(r->d_ctr[q], 0, sizeof(int32_t) * CTR_WORDS, s_prep));
  }
  // C-1 (NCCL mode): rank 0's bf16 batch, inverse norms (and quotas) to every rank; in
  // pipelined mode on the comm stream, in program order with the deferred all-gathers
  cudaStream_t s_bc = (pipelined && nccl_mode(r)) ? r->comm_stream : s_scan;
  // pipelined one-GPU one-slice scans (N <= 128, SMs reserved for prep / tail, so a scan
  // waiting on the flag can never hold the SM K6 needs): the scan waits for a device flag
  // the prep stream publishes instead of an event on the scan stream (k_scan_tc.cu)
  // (k_scan_tc only: the opt-in transposed scan keeps the event + grid-dependency wait)
  const bool flag_wait = pipelined && r->scan_flag && !nccl_mode(r) && r->cfg.world == 1 && N <= 128 &&
                         k > 0 && r->scan_reserve > 0 && !(r->scan_t && scan_t_supported(d, N, k));
  if (pipelined) {
    if (flag_wait) launch_publish(r->d_ready, ++r->ready_seq, s_prep);
    CU_TRY(r, cudaEventRecord(r->ev_prep[q], s_prep));
    if (!flag_wait) CU_TRY(r, cudaStreamWaitEvent(s_bc, r->ev_prep[q], 0));
    CU_TRY(r, cudaStreamWaitEvent(r->stream, r->ev_prep[q], 0));  // the prompt buffer is consumed
  }
  r->cur = q;
  if (nccl_mode(r)) {
    NC_TRY(r, nccl().GroupStart());
    NC_TRY(r, nccl().Broadcast(r->d_Xb[q], r->d_Xb[q], (size_t)n_pad * d * 2, ncclUint8, 0, r->comm, s_bc));
    NC_TRY(r, nccl().Broadcast(r->d_invq[q], r->d_invq[q], (size_t)n_pad, ncclFloat32, 0, r->comm, s_bc));
    if (quota_bcast) NC_TRY(r, nccl().Broadcast(r->d_quota[q], r->d_quota[q], 32, ncclInt32, 0, r->comm, s_bc));
    NC_TRY(r, nccl().GroupEnd());
    if (s_bc != s_scan) {
      CU_TRY(r, cudaEventRecord(r->ev_bcast[q], s_bc));
      CU_TRY(r, cudaStreamWaitEvent(s_scan, r->ev_bcast[q], 0));
    }
  }
  if (k == 0) {  // SM mode: no cache scan, the tail sees the prompts only
    *P_out = 0;
    return ARGUS_OK;
  }
  ScanArgs a{};
  a.head = (uint32_t)ring_head(r);
  a.capg = r->cfg.evict ? (uint32_t)r->cfg.capacity : 0u;
  {
    static const int win = getenv("ARGUS_PAIR_WINDOW") ? atoi(getenv("ARGUS_PAIR_WINDOW")) : 0;
    a.window = win;
  }
  a.Xb = r->d_Xb[q];
  a.inv_q = r->d_invq[q];
  a.Cb = r->d_Cb;
  a.inv_c = r->d_invc;
  a.m_local = local_rows(r);
  a.N = N;
  a.n_pad = n_pad;
  a.d = d;
  a.k = k;
  a.rank = r->cfg.rank;
  a.world = r->cfg.world;
  a.partial = r->d_partial[q];
  a.dbg = r->dbg_scores;
  a.ready = flag_wait ? r->d_ready : nullptr;
  a.ready_seq = r->ready_seq;
  a.stamp = r->stamp_buf ? r->stamp_buf + (r->stamp_seq++ % r->stamp_cap) * 256 * 4 : nullptr;
  a.dbg_ld = r->dbg_ld;
  if (a.dbg && a.dbg_ld < a.m_local) return ARGUS_E_INVALID;  // capture rows too short for the shard
  a.gthr = r->d_gthr[q];
  a.ctr = r->d_ctr[q];
  bool pair = r->pair_scan && scan_pair_supported(d, N);
  // the scan grid's SM budget: a pipelined one-slice scan (N <= 128, HBM-bound: 146 SMs
  // still saturate HBM) leaves a few SMs free so the next batch's prep and this batch's
  // tail run beside it instead of queueing behind the persistent grid (N = 48, fixed:
  // 264 -> 256 us per batch with 2 SMs reserved, scripts/scan_reserve_sweep.sh)
  // (pipelined NCCL mode: always, so the collectives of the neighbouring batches find SMs)
  int scan_sms = pipelined && (N <= 128 || nccl_mode(r)) ? r->num_sms - r->scan_reserve : r->num_sms;
  if (pipelined && N > 128) {
    // multi-slice scans are tensor-bound and fill every SM: the previous batch's tail (one
    // CTA per 16-prompt block, one CTA per SM) would find none free until this scan ends, so
    // a few SMs are left to it and to the next batch's prep
    const int rt = r->scan_reserve_t >= 0 ? r->scan_reserve_t : 0;
    scan_sms = std::min(scan_sms, r->num_sms - rt);
  }
  {
    StageScope sc(r, ARGUS_STAGE_SCAN, s_scan);
    if (pair) {
      // With more pair slices than divide the SMs' pairs evenly, launch a pair on every
      // TPC and let pairs whose slice runs dry continue another slice (list slots
      // [home_max, home_max + MAX_VISITS) for migrants, zeroed here since some stay unused).
      const int pslices = (N + 255) / 256;
      const int clusters = scan_sms / 2;
      const int64_t n_tiles = (a.m_local + 63) / 64;
      a.migrate = r->migrate && pslices >= 2 && clusters % pslices != 0 && n_tiles >= (int64_t)clusters * 16;
      if (a.migrate) {
        a.home_max = clusters / pslices;
        a.floaters = clusters - a.home_max * pslices;
        a.P = a.home_max + a.floaters + MAX_VISITS;
        a.grid_ctas = 2 * clusters;
        if ((int64_t)a.P * N > r->partial_lists) return ARGUS_E_STATE;  // cannot happen (see init)
        CU_TRY(r, cudaMemsetAsync(r->d_partial[q], 0, sizeof(uint64_t) * (size_t)a.P * N * k, s_scan));
      } else {
        a.P = scan_pair_plan(a.m_local, N, scan_sms);
        a.home_max = a.P;
        a.floaters = 0;
      }
      if ((int64_t)a.P * N > r->partial_lists) return ARGUS_E_STATE;  // cannot happen (see init)
      // PDL also when pipelined: consecutive kernels of the scan stream (scan, merge, next
      // scan) overlap prologue and drain; the buffers of the next batch are another parity
      // and its cross-stream inputs are ordered by events
      if (launch_scan_pair(a, &r->tmap_c32, &r->tmap_q[q], s_scan, true) != cudaSuccess) {
        // cluster launch refused (configuration, not a device fault): one slice per CTA from now on
        cudaGetLastError();
        r->pair_scan = false;
        pair = false;
        if (getenv("ARGUS_DEBUG")) fprintf(stderr, "argus: CTA-pair scan unavailable, using one slice per CTA\n");
      }
    }
    if (!pair && r->scan_t && scan_t_supported(d, N, k)) {
      a.P = scan_t_plan_ranges(a.m_local, scan_sms);
      if ((int64_t)a.P * N > r->partial_lists) return ARGUS_E_STATE;
      if (launch_scan_t(a, &r->tmap_c, &r->tmap_q16[q], s_scan, true) != cudaSuccess) return ARGUS_E_CUDA;
    } else if (!pair) {
      a.P = scan_plan_ranges(a.m_local, N, scan_sms);
      if ((int64_t)a.P * N > r->partial_lists) return ARGUS_E_STATE;
      launch_scan(a, &r->tmap_c, &r->tmap_q[q], s_scan, true);
    }
  }
  LAUNCHED(r);
  *P_out = a.P;
  if (keys_dev) {
    {
      StageScope sc(r, ARGUS_STAGE_MERGE_LOCAL, s_scan);
      launch_merge_topk(r->d_partial[q], a.P, N, k, keys_dev, nullptr, nullptr, s_scan);
    }
    LAUNCHED(r);
  } else if (send_seq) {  // K5 + C-2 fused: merged keys stored into every rank's inbox
    {
      StageScope sc(r, ARGUS_STAGE_MERGE_LOCAL, s_scan);
      launch_merge_send(r->d_partial[q], a.P, N, k, p2p_send_args(r, send_seq), r->d_p2p_ticket, s_scan, true,
                        r->num_sms);
    }
    LAUNCHED(r);
  }
  return ARGUS_OK;
}

// The fused tail (merge of P candidate lists per prompt, predictor, A5, assignment).
static int finish_impl(argus_router* r, const uint64_t* keys_in, int32_t P, int32_t N, const int32_t* quota,
                       int32_t* option_out_dev, uint32_t* topk_idx_dev, float* topk_score_dev, float* quality_dev,
                       uint8_t* status_dev, cudaStream_t s, bool pdl, const argus_route_extra* ex = nullptr,
                       int q = -1, uint32_t p2p_seq = 0);
static int flush_deferred(argus_router* r);
static int async_harvest(argus_router* r, int q);
// route_batch* in NCCL mode: the quotas are rank 0's (broadcast), other ranks may pass NULL
static bool quota_from_root(const argus_router* r) {
  return nccl_mode(r) && r->policy == ARGUS_POLICY_SD;
}
static int quota_ok(const argus_router* r, const int32_t* quota) {
  if (r->policy == ARGUS_POLICY_PASM) return 1;  // quotas are not used when sampling the PASM
  // (rank 0's values are checked by the tail on every rank, so an invalid quota fails
  // the call everywhere instead of leaving the other ranks inside the broadcast)
  if (quota_from_root(r)) return r->cfg.rank != 0 || quota != nullptr;
  if (!quota) return 0;
  for (int v = 0; v < r->cfg.L; ++v)
    if (quota[v] < 0) return 0;
  return 1;
}

int argus_route_finish_dev(argus_router* r, const uint64_t* keys_all_dev, int32_t G, int32_t N,
                           const int32_t* quota, int32_t* option_out_dev, uint32_t* topk_idx_dev,
                           float* topk_score_dev, float* quality_dev, uint8_t* status_dev) {
  // the tail stages G lists per prompt in shared memory sized for cfg.world at init
  if (!r || G != r->cfg.world || !keys_all_dev || (reinterpret_cast<uintptr_t>(keys_all_dev) & 7)) return ARGUS_E_INVALID;
  return finish_impl(r, keys_all_dev, G, N, quota, option_out_dev, topk_idx_dev, topk_score_dev, quality_dev,
                     status_dev, r->stream, true);
}

static int finish_impl(argus_router* r, const uint64_t* keys_in, int32_t P, int32_t N, const int32_t* quota,
                       int32_t* option_out_dev, uint32_t* topk_idx_dev, float* topk_score_dev, float* quality_dev,
                       uint8_t* status_dev, cudaStream_t s, bool pdl, const argus_route_extra* ex, int q,
                       uint32_t p2p_seq) {
  if (q < 0) q = r->cur;  // the parity of the buffers this batch's partial_impl used
  if (p2p_seq) keys_in = inbox_keys(r, r->d_inbox, (int)(p2p_seq & 1u));  // filled by the fused exchange
  const bool qdev = r->quota_dev_next;  // consumed by this call whatever happens
  r->quota_dev_next = false;
  int rc = check_state(r);
  if (rc) return rc;
  const bool sm_mode = r->cfg.k == 0;
  if (N < 1 || N > r->cfg.max_batch || (!qdev && !quota_ok(r, quota))) return ARGUS_E_INVALID;
  if (!sm_mode && (P < 1 || !keys_in)) return ARGUS_E_INVALID;
  const int L = r->cfg.L, k = r->cfg.k;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  TailArgs m{};
  m.keys_in = keys_in;
  m.P = P;
  if (p2p_seq) {
    m.p2p_flags = inbox_flags(r->d_inbox, (int)(p2p_seq & 1u));
    m.p2p_consumed = inbox_consumed(r->d_inbox, (int)(p2p_seq & 1u));
    m.p2p_seq = p2p_seq;
  }
  m.topk_idx = topk_idx_dev ? topk_idx_dev : r->d_idx;
  m.topk_score = topk_score_dev ? topk_score_dev : r->d_score;
  m.Xb = r->d_Xb[q];  // the bf16 copy of this batch made by partial_impl
  m.inv_q = r->d_invq[q];
  m.W1xF = r->d_W1xF;
  m.W1sT = r->d_W1sT;
  m.b1 = r->d_b1;
  m.W2 = r->d_W2;
  m.b2 = r->d_b2;
  m.hbuf = r->d_h;
  m.block_cnt = r->d_mlp_cnt;
  m.launch_cnt = r->d_tail_cnt;
  m.kskip = r->d_kskip;
  m.pth = r->d_pth;
  m.gate = r->d_gate;
  m.delta = r->cfg.delta;
  m.N = N;
  m.d = r->cfg.d;
  m.k = k;
  m.H = r->cfg.hidden;
  m.L = L;
  m.rhat = quality_dev ? quality_dev : r->d_rhat;
  m.prefl = r->d_pref;
  {  // serial dictatorship schedule: one prompt per step up to sd_pp_max prompts (k_tail.cu)
    static const int pp_env = getenv("ARGUS_SD_PP") ? atoi(getenv("ARGUS_SD_PP")) : -1;
    m.sd_pp_max = pp_env >= 0 ? pp_env : 512;  // measured in situ: per-prompt <= windows up to N = 512
  }
  m.ccount = r->d_ccount;
  m.cmask = r->d_cmask;
  // quotas travel by value in the kernel parameter block (no host buffer lifetime issue)
  for (int v = 0; v < 32; ++v) m.quota[v] = (v < L && quota) ? quota[v] : 0;
  m.quota_dev = qdev ? r->d_quota[q] : nullptr;
  m.option_out = option_out_dev ? option_out_dev : r->d_option;
  m.status = status_dev ? status_dev : r->d_status;
  m.flags = r->flags_cur ? r->flags_cur : r->d_flags;
  m.policy = r->policy;
  m.pasm_cdf = r->d_cdf;
  m.pasm_last = r->d_plast;
  m.seed_lo = (uint32_t)r->seed;
  m.seed_hi = (uint32_t)(r->seed >> 32);
  m.seq_lo = (uint32_t)r->batch_seq;
  m.seq_hi = (uint32_t)(r->batch_seq >> 32);
  m.optimal_out = ex ? ex->optimal : nullptr;
  m.id_base = (uint32_t)(r->m_global - live_rows(r));
  m.head = (uint32_t)ring_head(r);
  m.capg = r->cfg.evict ? (uint32_t)r->cfg.capacity : 0u;
  m.handle = r->d_handle;
  m.topk_handle = ex ? ex->topk_handle : nullptr;
  m.aff_ring = r->d_aff;
  m.aff_win = ARGUS_AFFINITY_WINDOW;
  m.aff_pos0 = (int32_t)(r->aff_total % ARGUS_AFFINITY_WINDOW);
  m.n_workers = r->n_workers;
  m.wlist = r->d_wlist;
  m.wcount = r->d_wcount;
  m.wtime = r->d_wtime;
  m.queue = r->d_queue;
  m.worker_out = ex ? ex->worker : nullptr;
  {
    StageScope sc(r, ARGUS_STAGE_TAIL, s);
    // a pipelined tail overlaps the next scan: one CTA per prompt block keeps its SM
    // footprint small; a tail on the critical path spreads over H/32 CTAs per block
    const int ysplit = s == r->tail_stream ? r->tail_ysplit : r->cfg.hidden / 32;
    launch_tail(m, r->tail_smem, s, pdl, ysplit);
  }
  LAUNCHED(r);
  r->batch_seq++;
  r->aff_total += N;
  return ARGUS_OK;
}

int argus_route_batch_dev(argus_router* r, const float* prompts_dev, int32_t N, const int32_t* quota,
                          int32_t* option_out_dev, uint32_t* topk_idx_dev, float* topk_score_dev,
                          float* quality_dev, uint8_t* status_dev) {
  return argus_route_batch_ex_dev(r, prompts_dev, N, quota, option_out_dev, topk_idx_dev, topk_score_dev,
                                  quality_dev, status_dev, nullptr);
}

int argus_route_batch_ex_dev(argus_router* r, const float* prompts_dev, int32_t N, const int32_t* quota,
                             int32_t* option_out_dev, uint32_t* topk_idx_dev, float* topk_score_dev,
                             float* quality_dev, uint8_t* status_dev, const argus_route_extra* ex) {
  int rc = check_state(r);
  if (rc) return rc;
  if (r->cfg.world > 1 && !r->comm && !r->p2p) return ARGUS_E_STATE;  // external mode: partial/finish
  if (N < 1 || N > r->cfg.max_batch || !quota_ok(r, quota) || !option_out_dev ||
      (r->cfg.k > 0 && (!topk_idx_dev || !topk_score_dev)))
    return ARGUS_E_INVALID;
  r->pending = true;
  int32_t P = 0;
  if (r->pipe && !r->serial_call && nccl_mode(r)) {
    // Pipelined NCCL mode.  This call: K6 (root) -> C-1 broadcast on the comm stream ->
    // scan + K5 local merge on the scan stream.  Then the previous batch's C-2 all-gather
    // (comm stream, behind this broadcast) and tail (tail stream) are issued, and this
    // batch's wait for the next call or argus_route_join.  Every rank issues the
    // collectives in the same order: bcast(b), AG(b-1), bcast(b+1), AG(b), ...
    const int q = (int)(r->seq & 1);
    CU_TRY(r, cudaEventRecord(r->ev_in[q], r->stream));
    CU_TRY(r, cudaStreamWaitEvent(r->prep_stream, r->ev_in[q], 0));
    if (r->tail_inflight[q]) CU_TRY(r, cudaStreamWaitEvent(r->prep_stream, r->ev_tail[q], 0));  // parity q free
    const bool qb = quota_from_root(r);
    const uint32_t seq = r->p2p ? ++r->p2p_seq : 0u;  // fused exchange instead of the all-gather
    rc = partial_impl(r, prompts_dev, N, (r->cfg.k > 0 && !seq) ? r->d_keys[q] : nullptr, &P, q, r->prep_stream,
                      r->scan_stream, qb, quota, seq);
    if (rc) return rc;
    CU_TRY(r, cudaEventRecord(r->ev_scan[q], r->scan_stream));
    rc = flush_deferred(r);
    if (rc) return rc;
    argus_router::Deferred& D = r->def;
    D.valid = true;
    D.q = q;
    D.N = N;
    D.P = P;
    D.qdev = qb;
    for (int v = 0; v < 32; ++v) D.quota[v] = (v < r->cfg.L && quota) ? quota[v] : 0;
    D.option = option_out_dev;
    D.idx = topk_idx_dev;
    D.score = topk_score_dev;
    D.quality = quality_dev;
    D.status = status_dev;
    D.has_ex = ex != nullptr;
    if (ex) D.ex = *ex;
    D.flags = r->flags_cur;
    D.async_slot = -1;
    D.seq = seq;
    r->seq++;
    return ARGUS_OK;
  }
  if (r->pipe && !r->serial_call) {  // prep / scan / tail on the internal streams (see the file header)
    const int q = (int)(r->seq & 1);
    CU_TRY(r, cudaEventRecord(r->ev_in[q], r->stream));  // prompts (and earlier inserts) are ready
    CU_TRY(r, cudaStreamWaitEvent(r->prep_stream, r->ev_in[q], 0));
    if (r->tail_inflight[q]) CU_TRY(r, cudaStreamWaitEvent(r->prep_stream, r->ev_tail[q], 0));  // parity q free
    rc = partial_impl(r, prompts_dev, N, nullptr, &P, q, r->prep_stream, r->scan_stream);
    if (rc) return rc;
    CU_TRY(r, cudaEventRecord(r->ev_scan[q], r->scan_stream));
    CU_TRY(r, cudaStreamWaitEvent(r->tail_stream, r->ev_scan[q], 0));
    rc = finish_impl(r, r->d_partial[q], P, N, quota, option_out_dev, topk_idx_dev, topk_score_dev, quality_dev,
                     status_dev, r->tail_stream, false, ex);
    if (rc) return rc;
    CU_TRY(r, cudaEventRecord(r->ev_tail[q], r->tail_stream));
    r->tail_inflight[q] = true;
    r->seq++;
    return ARGUS_OK;
  }
  if (r->p2p) {  // NCCL mode or external mode with mapped inboxes: the fused exchange
    const bool qb = quota_from_root(r);
    const uint32_t seq = ++r->p2p_seq;
    rc = partial_impl(r, prompts_dev, N, nullptr, &P, 0, nullptr, nullptr, qb, quota, seq);
    if (rc) return rc;
    r->quota_dev_next = qb;
    return finish_impl(r, nullptr, r->cfg.world, N, quota, option_out_dev, topk_idx_dev, topk_score_dev,
                       quality_dev, status_dev, r->stream, true, ex, -1, seq);
  }
  if (!nccl_mode(r)) {  // single shard: the tail merges the per-CTA lists directly
    rc = partial_impl(r, prompts_dev, N, nullptr, &P, 0);
    if (rc) return rc;
    return finish_impl(r, r->d_partial[0], P, N, quota, option_out_dev, topk_idx_dev, topk_score_dev, quality_dev,
                       status_dev, r->stream, true, ex);
  }
  const bool qb = quota_from_root(r);
  rc = partial_impl(r, prompts_dev, N, r->d_keys[0], &P, 0, nullptr, nullptr, qb, quota);
  if (rc) return rc;
  r->quota_dev_next = qb;
  // C-2: N*k candidate keys from every shard
  if (r->cfg.k > 0)
    NC_TRY(r, nccl().AllGather(r->d_keys[0], r->d_keys_all[0], (size_t)N * r->cfg.k, ncclUint64, r->comm, r->stream));
  return finish_impl(r, r->d_keys_all[0], r->cfg.world, N, quota, option_out_dev, topk_idx_dev, topk_score_dev,
                     quality_dev, status_dev, r->stream, true, ex);
}

// Pipelined NCCL mode: issue the deferred batch's C-2 all-gather (comm stream, after its
// scan) and its tail (tail stream), then the result copy of an asynchronous host call.
static int flush_deferred(argus_router* r) {
  argus_router::Deferred& D = r->def;
  if (!D.valid) return ARGUS_OK;
  D.valid = false;
  const int q = D.q, k = r->cfg.k;
  if (D.seq) {  // fused exchange: the tail itself waits for the peers' keys
    CU_TRY(r, cudaStreamWaitEvent(r->tail_stream, r->ev_scan[q], 0));
  } else if (k > 0) {
    CU_TRY(r, cudaStreamWaitEvent(r->comm_stream, r->ev_scan[q], 0));
    NC_TRY(r, nccl().AllGather(r->d_keys[q], r->d_keys_all[q], (size_t)D.N * k, ncclUint64, r->comm,
                               r->comm_stream));
    CU_TRY(r, cudaEventRecord(r->ev_ag[q], r->comm_stream));
    CU_TRY(r, cudaStreamWaitEvent(r->tail_stream, r->ev_ag[q], 0));
  } else {  // SM mode: the broadcast batch is the whole input (the scan stream waited for it)
    CU_TRY(r, cudaStreamWaitEvent(r->tail_stream, r->ev_scan[q], 0));
  }
  uint32_t* saved = r->flags_cur;
  r->flags_cur = D.flags;
  r->quota_dev_next = D.qdev;
  int rc = finish_impl(r, r->d_keys_all[q], r->cfg.world, D.N, D.quota, D.option, D.idx, D.score, D.quality,
                       D.status, r->tail_stream, false, D.has_ex ? &D.ex : nullptr, q, D.seq);
  r->flags_cur = saved;
  if (rc) return rc;
  CU_TRY(r, cudaEventRecord(r->ev_tail[q], r->tail_stream));
  r->tail_inflight[q] = true;
  if (D.async_slot >= 0) {  // argus_route_batch_async: one packed copy of the results
    const int a = D.async_slot;
    CU_TRY(r, cudaEventRecord(r->ev_done[a], r->tail_stream));
    CU_TRY(r, cudaStreamWaitEvent(r->d2h_stream, r->ev_done[a], 0));
    CU_TRY(r, cudaMemcpyAsync(r->h_oasync[a], r->d_oasync[a], D.async_bytes, cudaMemcpyDeviceToHost, r->d2h_stream));
    CU_TRY(r, cudaEventRecord(r->ev_async[a], r->d2h_stream));
  }
  return ARGUS_OK;
}

int argus_route_batch_bf16_dev(argus_router* r, const void* prompts_bf16_dev, int32_t N, const int32_t* quota,
                               int32_t* option_out_dev, uint32_t* topk_idx_dev, float* topk_score_dev,
                               float* quality_dev, uint8_t* status_dev, const argus_route_extra* extra) {
  if (!r) return ARGUS_E_INVALID;
  r->prompts_bf16 = true;  // K6 copies the rows as they are (same norm, same validity checks)
  const int rc = argus_route_batch_ex_dev(r, static_cast<const float*>(prompts_bf16_dev), N, quota, option_out_dev,
                                          topk_idx_dev, topk_score_dev, quality_dev, status_dev, extra);
  r->prompts_bf16 = false;
  return rc;
}

int argus_route_join(argus_router* r, void* stream) {
  if (!r) return ARGUS_E_INVALID;
  if (r->poisoned) return ARGUS_E_STATE;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  int rc0 = flush_deferred(r);
  if (rc0) return rc0;
  cudaStream_t s = stream ? (cudaStream_t)stream : r->stream;
  for (int q = 0; q < 2; ++q)
    if (r->tail_inflight[q]) {
      CU_TRY(r, cudaStreamWaitEvent(s, r->ev_tail[q], 0));
      if (s == r->stream) r->tail_inflight[q] = false;  // ordered behind it from now on
    }
  if (s != r->stream) {  // and behind everything on the router's own stream
    cudaEvent_t e = ev_get(r);
    CU_TRY(r, cudaEventRecord(e, r->stream));
    CU_TRY(r, cudaStreamWaitEvent(s, e, 0));
    r->ev_pool.push_back(e);  // reuse is safe: a wait binds to the record issued before it
  }
  return ARGUS_OK;
}

int argus_sync(argus_router* r) {
  int rc = check_state(r);
  if (rc) return rc;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  rc = argus_route_join(r, nullptr);
  if (rc) return rc;
  CU_TRY(r, cudaMemcpyAsync(r->h_flags, r->d_flags, 4, cudaMemcpyDeviceToHost, r->stream));
  CU_TRY(r, cudaMemsetAsync(r->d_flags, 0, 4, r->stream));
  CU_TRY(r, cudaStreamSynchronize(r->stream));
  // asynchronous host calls: their result copies follow the tails; collect them too
  // (their result codes stay available to argus_route_wait)
  for (int q = 0; q < argus_router::NASYNC; ++q) {
    rc = async_harvest(r, q);
    if (rc) return rc;
  }
  r->pending = false;
  const uint32_t fl = *r->h_flags;
  if (fl & FLAG_PEER_TIMEOUT) {  // a peer never delivered its keys: the exchange is broken
    r->poisoned = true;
    return ARGUS_E_NCCL;
  }
  if (fl & FLAG_INVALID_INPUT) return ARGUS_E_INVALID;
  if (fl & FLAG_OVERFLOW) return ARGUS_W_OVERFLOW;
  return ARGUS_OK;
}

int argus_route_batch(argus_router* r, const float* prompts, int32_t N, const int32_t* quota,
                      int32_t* option_out, uint32_t* topk_idx, float* topk_score, float* quality_out,
                      uint8_t* status_out) {
  return argus_route_batch_ex(r, prompts, N, quota, option_out, topk_idx, topk_score, quality_out, status_out,
                              nullptr);
}

int argus_route_batch_ex(argus_router* r, const float* prompts, int32_t N, const int32_t* quota,
                         int32_t* option_out, uint32_t* topk_idx, float* topk_score, float* quality_out,
                         uint8_t* status_out, const argus_route_extra* extra) {
  int rc = check_state(r);
  if (rc) return rc;
  const bool root = r->cfg.rank == 0 || !nccl_mode(r);
  if (N < 1 || N > r->cfg.max_batch || !quota_ok(r, quota) || !option_out ||
      (r->cfg.k > 0 && (!topk_idx || !topk_score)))
    return ARGUS_E_INVALID;
  int32_t* optimal_out = extra ? extra->optimal : nullptr;
  int32_t* worker_out = extra ? extra->worker : nullptr;
  uint64_t* handle_out = extra ? extra->topk_handle : nullptr;
  if (root && !prompts) return ARGUS_E_INVALID;
  if (r->cfg.world > 1 && !r->comm && !r->p2p) return ARGUS_E_STATE;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  const int d = r->cfg.d, k = r->cfg.k, L = r->cfg.L;
  if (r->pending) {  // drain earlier async work and clear its deferred flags
    rc = argus_sync(r);
    if (rc < 0) return rc;
  }
  // packed output block for this N: [flags | option | idx | score | rhat | status | optimal | worker | handle]
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t o_opt = 16, o_idx = al(o_opt + 4 * (size_t)N), o_sc = al(o_idx + 4 * (size_t)N * k),
               o_rh = al(o_sc + 4 * (size_t)N * k), o_st = al(o_rh + 4 * (size_t)N * L), o_ob = al(o_st + N),
               o_wk = al(o_ob + 4 * (size_t)N), o_hd = al(o_wk + 4 * (size_t)N), o_end = o_hd + 8 * (size_t)N * k;
  const size_t o_copy = handle_out ? o_end : worker_out ? o_hd : (optimal_out ? o_wk : o_ob);
  uint8_t* D = r->d_outblk;
  if (root)
    CU_TRY(r, cudaMemcpyAsync(r->d_Xstage, prompts, sizeof(float) * N * d, cudaMemcpyHostToDevice, r->stream));
  argus_route_extra dx{optimal_out ? reinterpret_cast<int32_t*>(D + o_ob) : nullptr,
                       worker_out ? reinterpret_cast<int32_t*>(D + o_wk) : nullptr,
                       handle_out ? reinterpret_cast<uint64_t*>(D + o_hd) : nullptr};
  // the call is synchronous, so pipelining cannot overlap anything; everything was
  // drained above, so the parity-0 buffers of the single-stream path are free
  r->serial_call = true;
  rc = argus_route_batch_ex_dev(r, r->d_Xstage, N, quota, reinterpret_cast<int32_t*>(D + o_opt),
                                reinterpret_cast<uint32_t*>(D + o_idx), reinterpret_cast<float*>(D + o_sc),
                                reinterpret_cast<float*>(D + o_rh), D + o_st, &dx);
  r->serial_call = false;
  if (rc) return rc;
  rc = argus_route_join(r, nullptr);
  if (rc) return rc;
  CU_TRY(r, cudaMemcpyAsync(r->h_outblk, D, o_copy, cudaMemcpyDeviceToHost, r->stream));
  CU_TRY(r, cudaMemsetAsync(r->d_flags, 0, 4, r->stream));
  CU_TRY(r, cudaStreamSynchronize(r->stream));
  r->pending = false;
  const uint8_t* Hb = r->h_outblk;
  memcpy(option_out, Hb + o_opt, 4 * (size_t)N);
  if (k > 0) {
    memcpy(topk_idx, Hb + o_idx, 4 * (size_t)N * k);
    memcpy(topk_score, Hb + o_sc, 4 * (size_t)N * k);
  }
  if (handle_out) memcpy(handle_out, Hb + o_hd, 8 * (size_t)N * k);
  if (quality_out) memcpy(quality_out, Hb + o_rh, 4 * (size_t)N * L);
  if (status_out) memcpy(status_out, Hb + o_st, (size_t)N);
  if (optimal_out) memcpy(optimal_out, Hb + o_ob, 4 * (size_t)N);
  if (worker_out) memcpy(worker_out, Hb + o_wk, 4 * (size_t)N);
  uint32_t fl;
  memcpy(&fl, Hb, 4);
  if (fl & FLAG_PEER_TIMEOUT) {
    r->poisoned = true;
    return ARGUS_E_NCCL;
  }
  if (fl & FLAG_INVALID_INPUT) return ARGUS_E_INVALID;
  if (fl & FLAG_OVERFLOW) return ARGUS_W_OVERFLOW;
  return ARGUS_OK;
}

// ------------------------------------------------------------------ asynchronous host-buffer calls
static int flags_rc(uint32_t fl) {
  if (fl & FLAG_PEER_TIMEOUT) return ARGUS_E_NCCL;
  if (fl & FLAG_INVALID_INPUT) return ARGUS_E_INVALID;
  if (fl & FLAG_OVERFLOW) return ARGUS_W_OVERFLOW;
  return ARGUS_OK;
}

// Finish the call carried by parity slot q (if any): wait for its D2H, keep its rc.
static int async_harvest(argus_router* r, int q) {
  if (r->async_ticket[q] < 0) return ARGUS_OK;
  if (r->def.valid && r->def.async_slot == q) {  // its tail (and copy) not issued yet
    int rc = flush_deferred(r);
    if (rc) return rc;
  }
  CU_TRY(r, cudaEventSynchronize(r->ev_async[q]));
  // one packed copy landed in pinned staging: unpack into the caller's buffers
  const argus_router::AsyncOut& o = r->aout[q];
  const int N = o.N, k = r->cfg.k, L = r->cfg.L;
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t o_opt = 16, o_idx = al(o_opt + 4 * (size_t)N), o_sc = al(o_idx + 4 * (size_t)N * k),
               o_rh = al(o_sc + 4 * (size_t)N * k), o_st = al(o_rh + 4 * (size_t)N * L);
  const uint8_t* Hb = r->h_oasync[q];
  memcpy(o.option, Hb + o_opt, 4 * (size_t)N);
  if (k > 0) {
    memcpy(o.idx, Hb + o_idx, 4 * (size_t)N * k);
    memcpy(o.score, Hb + o_sc, 4 * (size_t)N * k);
  }
  if (o.quality) memcpy(o.quality, Hb + o_rh, 4 * (size_t)N * L);
  if (o.status) memcpy(o.status, Hb + o_st, (size_t)N);
  uint32_t fl;
  memcpy(&fl, Hb, 4);
  r->async_rc[r->async_ticket[q]] = flags_rc(fl);
  r->async_ticket[q] = -1;
  return ARGUS_OK;
}

int argus_route_batch_async(argus_router* r, const float* prompts, int32_t N, const int32_t* quota,
                            int32_t* option_out, uint32_t* topk_idx, float* topk_score, float* quality_out,
                            uint8_t* status_out, int64_t* ticket) {
  int rc = check_state(r);
  if (rc) return rc;
  const bool root = r->cfg.rank == 0 || !nccl_mode(r);
  if (N < 1 || N > r->cfg.max_batch || !quota_ok(r, quota) || !option_out || !ticket ||
      (r->cfg.k > 0 && (!topk_idx || !topk_score)))
    return ARGUS_E_INVALID;
  if (root && !prompts) return ARGUS_E_INVALID;
  if (r->cfg.world > 1 && !r->comm && !r->p2p) return ARGUS_E_STATE;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  const int d = r->cfg.d, k = r->cfg.k, L = r->cfg.L;
  const int q = (int)(r->next_ticket % argus_router::NASYNC);
  rc = async_harvest(r, q);  // the slot's previous call (NASYNC calls ago) must have landed
  if (rc) return rc;
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t o_opt = 16, o_idx = al(o_opt + 4 * (size_t)N), o_sc = al(o_idx + 4 * (size_t)N * k),
               o_rh = al(o_sc + 4 * (size_t)N * k), o_st = al(o_rh + 4 * (size_t)N * L);
  uint8_t* D = r->d_oasync[q];
  uint32_t* dflags = reinterpret_cast<uint32_t*>(D);
  // zero the call's flag word with a 4-byte copy (a copy-engine transfer, unlike a
  // memset kernel, takes no SM away from the scan in flight)
  CU_TRY(r, cudaMemcpyAsync(dflags, r->h_fasync + argus_router::NASYNC, 4, cudaMemcpyHostToDevice, r->stream));
  if (root)
    CU_TRY(r, cudaMemcpyAsync(r->d_Xasync[q], prompts, sizeof(float) * N * d, cudaMemcpyHostToDevice, r->stream));
  r->flags_cur = dflags;
  rc = argus_route_batch_ex_dev(r, r->d_Xasync[q], N, quota, reinterpret_cast<int32_t*>(D + o_opt),
                                reinterpret_cast<uint32_t*>(D + o_idx), reinterpret_cast<float*>(D + o_sc),
                                quality_out ? reinterpret_cast<float*>(D + o_rh) : nullptr, D + o_st, nullptr);
  r->flags_cur = nullptr;
  if (rc) return rc;
  // results: one packed device-to-host copy on the copy stream once this call's tail
  // is done (the tail stream itself is never held up by copies); harvest unpacks it
  const size_t o_end = o_st + (size_t)N;
  if (r->def.valid) {  // pipelined NCCL mode: the tail is issued later, the copy with it
    r->def.async_slot = q;
    r->def.async_bytes = o_end;
  } else {
    cudaStream_t s = (r->pipe && r->tail_inflight[(r->seq - 1) & 1]) ? r->tail_stream : r->stream;
    CU_TRY(r, cudaEventRecord(r->ev_done[q], s));
    CU_TRY(r, cudaStreamWaitEvent(r->d2h_stream, r->ev_done[q], 0));
    CU_TRY(r, cudaMemcpyAsync(r->h_oasync[q], D, o_end, cudaMemcpyDeviceToHost, r->d2h_stream));
    CU_TRY(r, cudaEventRecord(r->ev_async[q], r->d2h_stream));
  }
  r->aout[q] = {N, option_out, topk_idx, topk_score, quality_out, status_out};
  r->async_ticket[q] = r->next_ticket;
  *ticket = r->next_ticket++;
  return ARGUS_OK;
}

int argus_route_wait(argus_router* r, int64_t ticket) {
  if (!r) return ARGUS_E_INVALID;
  if (r->poisoned) return ARGUS_E_STATE;
  if (ticket < 0 || ticket >= r->next_ticket) return ARGUS_E_INVALID;
  for (int q = 0; q < argus_router::NASYNC; ++q)
    if (r->async_ticket[q] >= 0 && r->async_ticket[q] <= ticket) {
      const int rc = async_harvest(r, q);
      if (rc) return rc;
    }
  auto it = r->async_rc.find(ticket);
  if (it == r->async_rc.end()) return ARGUS_E_INVALID;  // already collected
  const int rc = it->second;
  r->async_rc.erase(r->async_rc.begin(), std::next(it));  // older tickets are implicitly collected
  return rc;
}

// ------------------------------------------------------------------ F1 / F3 router state
int argus_set_policy(argus_router* r, int32_t policy, const double* pasm, uint64_t seed) {
  int rc = check_state(r);
  if (rc) return rc;
  const int L = r->cfg.L;
  if (policy != ARGUS_POLICY_SD && policy != ARGUS_POLICY_PASM) return ARGUS_E_INVALID;
  float cdf[32 * 32] = {};
  int8_t last[32] = {};
  if (policy == ARGUS_POLICY_PASM) {
    if (!pasm) return ARGUS_E_INVALID;
    for (int o = 0; o < L; ++o) {
      double srow = 0.0;
      float c = 0.0f;
      int lj = -1;
      for (int j = 0; j < L; ++j) {
        const double p = pasm[o * L + j];
        if (!std::isfinite(p) || p < 0.0) return ARGUS_E_INVALID;
        srow += p;
        const float pf = (float)p;
        c = c + pf;  // float32 running sum, j ascending (the decision precision, DESIGN R20)
        cdf[o * 32 + j] = c;
        if (pf > 0.0f) lj = j;
      }
      if (!(srow > 0.0) || lj < 0) return ARGUS_E_INVALID;
      last[o] = (int8_t)lj;
    }
  }
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  rc = argus_route_join(r, nullptr);  // batches in flight keep the policy they were issued with
  if (rc) return rc;
  CU_TRY(r, cudaMemcpyAsync(r->d_cdf, cdf, sizeof(cdf), cudaMemcpyHostToDevice, r->stream));
  CU_TRY(r, cudaMemcpyAsync(r->d_plast, last, sizeof(last), cudaMemcpyHostToDevice, r->stream));
  CU_TRY(r, cudaStreamSynchronize(r->stream));  // the host tables are stack arrays
  r->policy = policy;
  r->seed = seed;
  r->batch_seq = 0;
  return ARGUS_OK;
}

int argus_affinity_histogram(argus_router* r, int64_t* counts_out, int64_t* n_out) {
  int rc = check_state(r);
  if (rc) return rc;
  if (!counts_out) return ARGUS_E_INVALID;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  rc = argus_route_join(r, nullptr);
  if (rc) return rc;
  uint8_t ring[ARGUS_AFFINITY_WINDOW];
  CU_TRY(r, cudaMemcpyAsync(ring, r->d_aff, sizeof(ring), cudaMemcpyDeviceToHost, r->stream));
  CU_TRY(r, cudaStreamSynchronize(r->stream));
  const int64_t n = std::min<int64_t>(r->aff_total, ARGUS_AFFINITY_WINDOW);
  for (int v = 0; v < r->cfg.L; ++v) counts_out[v] = 0;
  // the last n prompts occupy ring slots (aff_total - n .. aff_total - 1) mod W
  for (int64_t t = r->aff_total - n; t < r->aff_total; ++t) {
    const int o = ring[t % ARGUS_AFFINITY_WINDOW];
    if (o < r->cfg.L) counts_out[o]++;
  }
  if (n_out) *n_out = n;
  return ARGUS_OK;
}

int argus_set_workers(argus_router* r, int32_t n_workers, const int32_t* option_of_worker, const float* t_proc,
                      const int32_t* queue) {
  int rc = check_state(r);
  if (rc) return rc;
  const int L = r->cfg.L;
  if (n_workers < 0 || n_workers > MAX_WORKERS) return ARGUS_E_INVALID;
  if (n_workers > 0 && (!option_of_worker || !t_proc || !queue)) return ARGUS_E_INVALID;
  std::vector<int16_t> wl(32 * 32, -1);
  std::vector<int32_t> wc(32, 0);
  for (int w = 0; w < n_workers; ++w) {
    const int v = option_of_worker[w];
    if (v < -1 || v >= L || !std::isfinite(t_proc[w]) || !(t_proc[w] > 0.f) || queue[w] < 0) return ARGUS_E_INVALID;
    if (v < 0) continue;
    if (wc[v] == 32) return ARGUS_E_INVALID;
    wl[v * 32 + wc[v]++] = (int16_t)w;
  }
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  rc = argus_route_join(r, nullptr);
  if (rc) return rc;
  if (n_workers > 0) {
    CU_TRY(r, cudaMemcpyAsync(r->d_wlist, wl.data(), sizeof(int16_t) * wl.size(), cudaMemcpyHostToDevice, r->stream));
    CU_TRY(r, cudaMemcpyAsync(r->d_wcount, wc.data(), sizeof(int32_t) * wc.size(), cudaMemcpyHostToDevice, r->stream));
    CU_TRY(r, cudaMemcpyAsync(r->d_wtime, t_proc, sizeof(float) * n_workers, cudaMemcpyHostToDevice, r->stream));
    CU_TRY(r, cudaMemcpyAsync(r->d_queue, queue, sizeof(int32_t) * n_workers, cudaMemcpyHostToDevice, r->stream));
  }
  CU_TRY(r, cudaStreamSynchronize(r->stream));  // host arrays may be freed after return
  r->n_workers = n_workers;
  return ARGUS_OK;
}

int argus_get_queues(argus_router* r, int32_t* queue_out) {
  int rc = check_state(r);
  if (rc) return rc;
  if (!queue_out) return ARGUS_E_INVALID;
  CU_TRY(r, cudaSetDevice(r->cfg.device));
  rc = argus_route_join(r, nullptr);
  if (rc) return rc;
  if (r->n_workers > 0)
    CU_TRY(r, cudaMemcpyAsync(queue_out, r->d_queue, sizeof(int32_t) * r->n_workers, cudaMemcpyDeviceToHost, r->stream));
  CU_TRY(r, cudaStreamSynchronize(r->stream));
  return ARGUS_OK;
}

}  // extern "C"
