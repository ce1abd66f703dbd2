// runtime.cu -- the Harmony runtime on one B200.
//
// Executes the swap plan built by plan.cpp (the same items the estimator
// prices) for the tasks bound to this rank's GPU:
//   * swap engine: pinned host arenas (W fp32, K = Adam (m,v), stash),
//     H2D on the swap-in stream, D2H on the swap-out stream, every transfer
//     gated by CUDA events on exactly the plan's dependencies, including the
//     one-task-ahead prefetch window (an input may start once the previous
//     task on the device has *started* computing -- simulator.py:262-269);
//   * layer-pack compute on the compute stream (tcgen05 GEMMs, flash
//     attention, LayerNorm, CE) with activation recompute for non-shared
//     backward packs and group-wide gradient accumulation in the pack's
//     GPU-resident dW buffer;
//   * the jit UPD task: fused Adam on the update stream, overlapping the next
//     backward task, followed by W and K swap-out.
// Device memory is one pool allocated at load time and checked against
// alpha; slots are reused round-robin and every reuse waits on the event
// that ends the previous occupant's last use.
#include <cuda.h>
#include <cuda_bf16.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../plan.hpp"
#include "common.hpp"
#include "kernels_api.hpp"
#include "nccl_loader.hpp"

namespace hm {

using bf16 = __nv_bfloat16;

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct ParamLayout {  // float offsets inside one layer's parameter block; -1 = absent
  int64_t wte = -1, wpe = -1, ln1_g, ln1_b, w_qkv, b_qkv, w_proj, b_proj, ln2_g, ln2_b, w_fc1, b_fc1, w_fc2, b_fc2;
  int64_t lnf_g = -1, lnf_b = -1, w_head = -1, size = 0;
  int64_t f32n = 0;  // leading fp32-read parameters (the rest are GEMM weights)
};

// Per-layer activation pointers for one member (u samples) inside a store.
struct Acts {
  float *x, *mean1, *rstd1, *lse, *h1, *mean2, *rstd2;
  bf16 *ln1, *qkv, *o, *ln2, *hpre, *a;
  float *yl, *meanf, *rstdf;  // head layer only
  bf16 *lnf, *dlog;
};

struct Scratch {
  bf16 *dy_bf, *dh, *dh1_bf, *dout, *dqkv;
  float *dln, *dh1, *dvec, *dq, *dyh, *g[2], *h[2], *logits, *tmp;
};

// Deep-CNN layer (BASELINE config c5): parameter offsets (floats) in the layer block
struct CnnParam {
  int64_t w1 = -1, b1 = -1, w2 = -1, b2 = -1, size = 0;
};

struct CnnScratch {
  bf16 *g[2] = {nullptr, nullptr};  // gradient ping-pong between layers of a pack
  bf16 *dz = nullptr, *dz2 = nullptr;
  bf16 *gsum = nullptr;              // trunk + skip gradient of a relay source
  float *logits = nullptr, *dpool = nullptr;
};

struct Slots {
  std::vector<uint16_t *> wlo;  // bf16-payload mode: lo planes of a forward task's fp32 prefixes
  std::vector<float *> w;
  std::vector<bf16 *> wsh;
  std::vector<float *> dw;
  std::vector<float *> k;
  std::vector<uint8_t *> stash_in;
};

struct TaskRt {
  int w_slot = -1, dw_slot = -1, k_slot = -1, stash_slot = -1;
  int carry_in = -1, carry_out = -1;  // F: hidden carry; B: gradient carry
  bool store_shared = false;          // F task keeping activations for the shared B
  bool from_shared = false;           // B task reading the shared store
  int64_t params = 0;                 // pack parameter count
  int b_task = -1;                    // U: its B task
  // U under the sharded Harmony-DP update: this rank's shard of the pack
  // (parameters [sh_off, sh_off + sh_len)) and the reduce-scatter chunk
  int64_t sh_off = 0, sh_len = -1, sh_chunk = 0;
  std::vector<int> members;           // member compute item ids
  std::vector<int64_t> s0;            // member sample offsets
  std::set<int> stash_heads;          // F: layers whose input is stashed
  // Harmony-PP across GPUs (peer-to-peer hand-offs)
  float *in_buf = nullptr;            // receive buffer: X (F), dY or the Y seam (B)
  float *out_buf = nullptr;           // source buffer read by the peer: Y (F), dX (B)
  bool ship_input = false;            // last F with a remote shared B: ship the shared pack's input
  bool remote_shared = false;         // shared B whose forward ran on another GPU: recompute
};

struct Action {
  int item = -1;
  int kind = 0;  // 0 = F/B member, 1 = U Adam, 2 = H2D, 3 = D2H, 5 = all-reduce, 6 = peer copy
  cudaStream_t stream = nullptr;
  void *dst = nullptr;
  const void *src = nullptr;
  int64_t bytes = 0;
  int task = -1, member = -1;
  int peer_rank = -1, peer_task = -1;       // kind 6: producer of the peer copy
  int64_t peer_off = 0;                     // kind 6: byte offset inside the producer's source buffer
  std::vector<std::pair<int, bool>> waits;  // (item, at_start)
  std::vector<cudaEvent_t> wait_events;     // non-plan dependencies (all-reduce)
  std::vector<int> xwaits;                  // previous-iteration items (end) this one must follow
  std::vector<std::pair<int, int>> rwaits;  // (item on another rank, iteration lag 0/1): signal waits
  cudaEvent_t done = nullptr;               // kind 5: all-reduce completion
  int64_t count = 0;                        // kind 5: floats reduced
  int pack_lo = -1, pack_ord = -1;          // kind 5: the pack (first layer) and its rank among my U tasks
  struct Seg { void *dst; const void *src; int64_t bytes; };
  std::vector<Seg> segs;                    // kind 2/3: several copies behind one ledger row
};

// Per-launch CUDA-event timing of the runtime's kernels (enabled on demand).
struct RtProfiler : KernelProfiler {
  struct Rec { int cls; cudaEvent_t e0, e1; double flops, bytes; };
  std::vector<cudaEvent_t> pool;
  std::vector<Rec> recs;
  size_t used = 0;
  bool capture = false;
  cudaError_t rec(cudaEvent_t e, cudaStream_t s) {
    return capture ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
  }
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void begin(int cls, cudaStream_t s) override {
    Rec r{cls, get(), nullptr, 0, 0};
    rec(r.e0, s);
    recs.push_back(r);
  }
  void end(int cls, cudaStream_t s, double flops, double bytes) override {
    for (auto it = recs.rbegin(); it != recs.rend(); ++it)
      if (it->cls == cls && it->e1 == nullptr) {
        it->e1 = get();
        rec(it->e1, s);
        it->flops = flops;
        it->bytes = bytes;
        return;
      }
  }
  // device globaltimer spans, one {~start, end} pair per record
  static constexpr size_t kSpanCap = 1 << 15;
  unsigned long long *spans = nullptr;
  unsigned long long *span_slot() override {
    if (!spans && cudaMalloc(&spans, kSpanCap * 2 * sizeof(unsigned long long)) != cudaSuccess) spans = nullptr;
    if (!spans || recs.empty() || recs.size() > kSpanCap) return nullptr;
    return spans + 2 * (recs.size() - 1);
  }
  cudaError_t clear_spans(cudaStream_t s) {
    return spans ? cudaMemsetAsync(spans, 0, kSpanCap * 2 * sizeof(unsigned long long), s) : cudaSuccess;
  }
  void reset() {
    recs.clear();
    used = 0;
  }
  ~RtProfiler() override {
    for (auto e : pool) cudaEventDestroy(e);
    if (spans) cudaFree(spans);
  }
};

}  // namespace hm

struct hm_runtime {
  bool profiling = false;
  hm::RtProfiler prof;
  double kstats[hm::KC_COUNT][4] = {{0}};  // ms, flops, bytes, launches (accumulated)
  std::vector<double> klaunch;  // last profiled iteration: (class, flops, bytes, event ms, device-clock ms) per launch
  std::vector<int64_t> gemm_shapes;  // GEMM calls of the last profiled enqueue, 7 fields each (gemm::shape_log)
  int device = 0;
  hm_model m{};
  int family = HM_FAMILY_GPT;          // GPT / BERT transformer chain or deep CNN
  int slot_nw = 0, slot_nk = 0;        // W / K slot counts chosen by load_plan (0 = minimum)
  bool slots_sized = false;
  std::vector<hm_cnn_layer> cnn;       // CNN: per-layer shapes
  std::vector<hm::CnnParam> cnn_lay;   // CNN: per-layer parameter offsets
  int classes = 0, classes_p = 0;      // CNN: classifier width (padded to 64)
  hm::CnnScratch CT{};
  // res2 skip edges: source layer -> its output (forward) and the skip path's
  // gradient (backward) for the whole minibatch, device-resident between tasks
  std::map<int, uint8_t *> relay_y, relay_g;
  int64_t alpha = 0;
  int D = 0, S = 0, H = 0, DH = 0, R = 0, V = 0, Vp = 0;
  int64_t total_params = 0;
  std::vector<hm::ParamLayout> lay;
  std::vector<int64_t> w_off;  // floats, per layer, + total at [R]
  cudaStream_t s_compute = nullptr, s_h2d = nullptr, s_d2h = nullptr, s_update = nullptr, s_p2p_in = nullptr,
               s_p2p_out = nullptr;
  float *w_host = nullptr, *k_host = nullptr;
  // W / K arenas: anonymous mappings bound (preferred) to the GPU's NUMA node,
  // then pinned with cudaHostRegister (NUMA-local host state)
  int64_t w_map_bytes = 0, k_map_bytes = 0;
  int numa_node = -1;
  // bf16 swap payloads (non-reference ledger): the host W arena
  // holds each layer as [hi plane | lo plane] (2 + 2 bytes per parameter, see
  // layers::w_join); forward tasks move hi planes plus the fp32-read prefix
  bool w_planar = false;
  // fp32-operand parity mode (hm_model.math_mode = 1, kernels/precise.cu):
  // activations fp32, GEMMs as three-plane bf16 split products; scratch for
  // the planes of the largest A / B operand and one M x N accumulator
  bool precise = false;
  void *psa = nullptr, *psb = nullptr;
  float *pc32 = nullptr;
  int64_t psa_n = 0, psb_n = 0, pc32_n = 0;
  uint8_t *stash_host = nullptr;
  int64_t stash_host_bytes = 0;
  // sharded Harmony-DP: each rank stashes its OWN samples, so its stash stays
  // private even though W / K live in the shared arena
  uint8_t *stash_priv = nullptr;
  int64_t stash_priv_bytes = 0;
  // plan
  hm::Plan *plan = nullptr;
  int rank = 0;
  int minibatch = 0;  // samples this rank processes
  int64_t global_tokens = 0;
  std::vector<hm::TaskRt> trt;
  std::vector<hm::Action> actions;
  std::vector<cudaEvent_t> ev_start, ev_end;     // dependencies
  std::vector<cudaEvent_t> ev_tstart, ev_tend;   // timing (external records inside graphs)
  std::vector<char> ev_live;  // dependency event last recorded eagerly (waitable outside a capture)
  cudaEvent_t ev_iter0 = nullptr, ev_iter1 = nullptr, ev_fork = nullptr, ev_join[4] = {nullptr};
  // CUDA graph of one iteration ([0] plain, [1] with per-kernel timing events)
  bool use_graph = true;
  int64_t iterations = 0;
  cudaGraphExec_t graph_exec[2] = {nullptr, nullptr};
  int64_t graph_launches[2] = {0, 0};
  int64_t graph_bytes[2][3] = {{0}};
  float *adam_host = nullptr;  // pinned {lr_t, 1/sqrt(bc2)}
  double *loss_host = nullptr;  // pinned [64]
  cudaEvent_t ev_first = nullptr;
  float *adam_dev = nullptr;
  // device pool
  uint8_t *pool = nullptr;
  int64_t pool_bytes = 0;
  hm::Slots slots;
  float *carry[2] = {nullptr, nullptr};
  float *dcarry[2] = {nullptr, nullptr};
  std::map<int, uint8_t *> stash_dev;      // head layer -> device buffer
  std::map<int, int64_t> stash_host_off;   // head layer -> host arena offset
  uint8_t *shared_store = nullptr;
  int shared_lo = -1, shared_hi = -1;
  uint8_t *work_store = nullptr;
  hm::Scratch T{};
  int32_t *tokens = nullptr, *labels = nullptr;
  double *loss_dev = nullptr;  // [64] per-step loss slots
  double *loss_cur = nullptr;
  bool count_loss = true;
  int step = 0;
  // Harmony-DP gradient all-reduce (NCCL), one comm per job
  ncclComm_t comm = nullptr;
  int nranks = 1;
  cudaStream_t s_comm = nullptr;
  std::vector<cudaEvent_t> ar_events;
  // Harmony-DP gradient sum over CUDA IPC (several processes on one GPU, where
  // NCCL cannot run): each rank sums every rank's pack gradient, read through
  // the peers' pools, in rank order (identical bits on every rank); ordered by
  // device-side counters.  The multi-GPU path is NCCL.
  bool ipc_reduce = false;
  float *ar_tmp = nullptr;
  // sharded Harmony-DP update (hm_machine.dp_sharded_update): gradients are
  // reduce-scattered, rank g updates shard g of each pack in the ONE shared
  // host arena; the next iteration's W swap-ins wait for every rank's W-out
  bool dp_shard = false;
  // the IPC gradient sum pairs the ranks' buffers by PACK (task indices differ
  // between Harmony-DP ranks): first layer -> pool offset of its gradient
  std::map<int, int64_t> dw_off;
  std::vector<std::map<int, int64_t>> peer_dw_off;  // per peer
  // Harmony-PP across processes
  bool p2p_mode = false;
  bool shared_arena = false, shared_owner = false;
  std::string shm_name;
  void *shm_ptr = nullptr;
  int64_t shm_bytes = 0;
  uint32_t *sig = nullptr;  // [n_items] per-item completion counters (iteration number)
  int64_t sig_off = 0;
  std::map<int, int64_t> out_off;  // my task -> offset of its P2P source buffer in my pool
  std::vector<uint8_t *> peer_pool;
  std::vector<std::map<int, int64_t>> peer_out_off;
  std::vector<int64_t> peer_sig_off;
  double *loss_sink = nullptr;  // CE of recompute passes (not part of the loss)
  int64_t p2p_bytes = 0;
  // last iteration
  std::vector<hm_item> ledger, trace;
  int64_t counters[8] = {0};
};

namespace hm {

// ---------------------------------------------------------------------------
// stream memory operations (driver API, resolved at run time): device-side
// counters that order work across processes / GPUs without host round trips
// ---------------------------------------------------------------------------
using MemopWaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using MemopWriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct Memops {
  MemopWaitFn wait = nullptr;
  MemopWriteFn write = nullptr;
};
static Memops &memops() {
  static Memops m;
  static bool init = false;
  if (!init) {
    init = true;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.wait = reinterpret_cast<MemopWaitFn>(p);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.write = reinterpret_cast<MemopWriteFn>(p);
  }
  return m;
}

// ---------------------------------------------------------------------------
// model layout
// ---------------------------------------------------------------------------
static ParamLayout make_layout(const hm_runtime &rt, int L) {
  // fp32-read parameters first (LayerNorm, biases, embedding tables), then the
  // GEMM weights (model.py GPTSpec.layer_segments): `f32n` is that prefix
  const int64_t d = rt.m.d_model, v = rt.Vp, s = rt.S;
  ParamLayout p;
  int64_t o = 0;
  p.ln1_g = o; o += d;
  p.ln1_b = o; o += d;
  p.b_qkv = o; o += 3 * d;
  p.b_proj = o; o += d;
  p.ln2_g = o; o += d;
  p.ln2_b = o; o += d;
  p.b_fc1 = o; o += 4 * d;
  p.b_fc2 = o; o += d;
  if (L == rt.R - 1) {
    p.lnf_g = o; o += d;
    p.lnf_b = o; o += d;
  }
  if (L == 0) {
    p.wte = o; o += v * d;
    p.wpe = o; o += s * d;
  }
  p.f32n = o;
  p.w_qkv = o; o += 3 * d * d;
  p.w_proj = o; o += d * d;
  p.w_fc1 = o; o += 4 * d * d;
  p.w_fc2 = o; o += 4 * d * d;
  if (L == rt.R - 1) {
    p.w_head = o; o += v * d;
  }
  p.size = o;
  return p;
}

// per-sample bytes of each stored tensor, in store order (the GEMM operands
// are bf16, or fp32 in the parity mode)
static std::vector<int64_t> act_sizes(const hm_runtime &rt, bool head) {
  const int64_t S = rt.S, d = rt.m.d_model, H = rt.H, ob = rt.precise ? 4 : 2;
  std::vector<int64_t> v = {S * d * 4, S * 4, S * 4, S * H * 4, S * d * 4, S * 4, S * 4,        // x mean1 rstd1 lse h1 mean2 rstd2
                            S * d * ob, S * 3 * d * ob, S * d * ob, S * d * ob, S * 4 * d * ob, S * 4 * d * ob};  // ln1 qkv o ln2 hpre a
  if (head) {
    v.push_back(S * d * 4);           // yl
    v.push_back(S * 4);               // meanf
    v.push_back(S * 4);               // rstdf
    v.push_back(S * d * ob);          // lnf
    v.push_back(S * (int64_t)rt.Vp * ob);  // dlog
  }
  return v;
}

static int64_t store_layer_bytes(const hm_runtime &rt, bool head, int64_t n) {
  int64_t b = 0;
  for (int64_t s : act_sizes(rt, head)) b += align_up(n * s, 256);
  return b;
}

static Acts acts_at(const hm_runtime &rt, uint8_t *base, bool head, int64_t n, int64_t s0) {
  auto sz = act_sizes(rt, head);
  uint8_t *p = base;
  uint8_t *r[18] = {nullptr};
  for (size_t i = 0; i < sz.size(); ++i) {
    r[i] = p + s0 * sz[i];
    p += align_up(n * sz[i], 256);
  }
  Acts A{};
  A.x = (float *)r[0]; A.mean1 = (float *)r[1]; A.rstd1 = (float *)r[2]; A.lse = (float *)r[3];
  A.h1 = (float *)r[4]; A.mean2 = (float *)r[5]; A.rstd2 = (float *)r[6];
  A.ln1 = (bf16 *)r[7]; A.qkv = (bf16 *)r[8]; A.o = (bf16 *)r[9]; A.ln2 = (bf16 *)r[10];
  A.hpre = (bf16 *)r[11]; A.a = (bf16 *)r[12];
  if (head) {
    A.yl = (float *)r[13]; A.meanf = (float *)r[14]; A.rstdf = (float *)r[15];
    A.lnf = (bf16 *)r[16]; A.dlog = (bf16 *)r[17];
  }
  return A;
}

static uint8_t *store_layer(const hm_runtime &rt, uint8_t *base, int lo, int L, int64_t n) {
  uint8_t *p = base;
  for (int j = lo; j < L; ++j) p += store_layer_bytes(rt, j == rt.R - 1, n);
  return p;
}

// ---------------------------------------------------------------------------
// boundary tensors: the per-sample bytes entering chain layer L (the byte model
// x(L, 1) of the ProfileSet; L == R is the chain's output)
// ---------------------------------------------------------------------------
static int64_t bnd(const hm_runtime &rt, int L) {
  if (rt.family == HM_FAMILY_CNN) {
    if (L >= rt.R) return 0;
    const hm_cnn_layer &c = rt.cnn[L];
    return (int64_t)c.h * c.w * c.cin * 2;
  }
  return L == 0 ? (int64_t)rt.S * 4 : (int64_t)rt.S * rt.m.d_model * 4;
}
static int64_t max_bnd(const hm_runtime &rt) {
  int64_t m = 0;
  for (int L = 1; L <= rt.R; ++L) m = std::max(m, bnd(rt, L));
  return m;
}
static int64_t labels_per_sample(const hm_runtime &rt) { return rt.family == HM_FAMILY_CNN ? 1 : rt.S; }

// ---------------------------------------------------------------------------
// deep-CNN layer packs: store layout, forward, backward
// ---------------------------------------------------------------------------
static CnnParam cnn_layout(const hm_runtime &rt, int L) {
  const hm_cnn_layer &c = rt.cnn[L];
  CnnParam p;
  int64_t o = 0;
  if (c.type == HM_CNN_HEAD) {
    p.w1 = o; o += (int64_t)rt.classes_p * c.cin;
    p.b1 = o; o += rt.classes_p;
  } else {
    p.w1 = o; o += (int64_t)c.cout * 9 * c.cin;  // conv, down, res (first conv), res2
    p.b1 = o; o += c.cout;
    if (c.type == HM_CNN_RES) {
      p.w2 = o; o += (int64_t)c.cout * 9 * c.cout;
      p.b2 = o; o += c.cout;
    }
  }
  p.size = o;
  return p;
}

// per-sample bytes of the tensors layer L keeps, in store order
static std::vector<int64_t> cnn_act_sizes(const hm_runtime &rt, int L) {
  const hm_cnn_layer &c = rt.cnn[L];
  const int64_t P = (int64_t)c.h * c.w;
  switch (c.type) {
    case HM_CNN_CONV: return {P * c.cout * 2};                         // y
    case HM_CNN_DOWN: return {P * c.cout * 2, P / 4 * c.cout * 2};     // a, y = pool(a)
    case HM_CNN_RES: return {P * c.cout * 2, P * c.cout * 2};          // h, y
    case HM_CNN_RES2: return {P * c.cout * 2};                         // y
    default: return {(int64_t)c.cin * 2, (int64_t)rt.classes_p * 2};  // pooled, dlogits
  }
}
static int64_t cnn_pack_bytes(const hm_runtime &rt, int lo, int hi, int64_t n) {
  int64_t b = align_up(n * bnd(rt, lo), 256);
  for (int L = lo; L <= hi; ++L)
    for (int64_t sz : cnn_act_sizes(rt, L)) b += align_up(n * sz, 256);
  return b;
}
struct CnnActs {
  bf16 *x = nullptr;                  // layer input (the pack input or the previous layer's output)
  bf16 *a = nullptr, *h = nullptr;    // down: post-ReLU pre-pool; res: inner activation
  bf16 *y = nullptr;                  // layer output
  bf16 *pooled = nullptr, *dlog = nullptr;  // head
};
// activations of layer L (member at sample s0) inside a pack store of n samples
static CnnActs cnn_acts(const hm_runtime &rt, uint8_t *store, int lo, int L, int64_t n, int64_t s0) {
  uint8_t *p = store;
  bf16 *prev_out = reinterpret_cast<bf16 *>(p + s0 * bnd(rt, lo));
  p += align_up(n * bnd(rt, lo), 256);
  CnnActs A;
  for (int j = lo; j <= L; ++j) {
    auto sz = cnn_act_sizes(rt, j);
    std::vector<bf16 *> r;
    for (int64_t b : sz) {
      r.push_back(reinterpret_cast<bf16 *>(p + s0 * b));
      p += align_up(n * b, 256);
    }
    if (j == L) {
      A.x = prev_out;
      switch (rt.cnn[j].type) {
        case HM_CNN_CONV: A.y = r[0]; break;
        case HM_CNN_DOWN: A.a = r[0]; A.y = r[1]; break;
        case HM_CNN_RES: A.h = r[0]; A.y = r[1]; break;
        case HM_CNN_RES2: A.y = r[0]; break;
        default: A.pooled = r[0]; A.dlog = r[1]; break;
      }
    }
    if (rt.cnn[j].type != HM_CNN_HEAD) prev_out = r.back();  // y: the next layer's input
  }
  return A;
}

// Forward of layers [lo, hi] for one member of u samples.  Activations go to
// `store` (n samples, member at s_off) or, with store == nullptr, to the work
// store (u samples).  x_in is the pack input (for lo == 0 the image).
static int cnn_forward_pack(hm_runtime &rt, TaskRt &tr, int lo, int hi, int u, int64_t s0, const uint8_t *x_in,
                            uint8_t *store, int64_t n, int64_t s_off, uint8_t *y_final) {
  cudaStream_t s = rt.s_compute;
  // A forward task without a store hands its output on and keeps nothing: it
  // reads its input in place and writes the last layer straight into y_final
  // (no staging copies).  Stored / recomputed passes keep the input for backward.
  const bool pass_through = !store && y_final;
  if (!store) {
    store = rt.work_store;
    n = u;
    s_off = 0;
  }
  if (!pass_through) {
    CnnActs A0 = cnn_acts(rt, store, lo, lo, n, s_off);
    HM_CUDA(cudaMemcpyAsync(A0.x, x_in, (int64_t)u * bnd(rt, lo), cudaMemcpyDeviceToDevice, s));
  }
  for (int L = lo; L <= hi; ++L) {
    const hm_cnn_layer &c = rt.cnn[L];
    const CnnParam &P = rt.cnn_lay[L];
    const int64_t off = rt.w_off[L] - rt.w_off[lo];
    const float *w = rt.slots.w[tr.w_slot] + off;
    const bf16 *wsh = rt.slots.wsh[tr.w_slot] + off;
    CnnActs A = cnn_acts(rt, store, lo, L, n, s_off);
    if (pass_through && L == lo) A.x = reinterpret_cast<bf16 *>(const_cast<uint8_t *>(x_in));
    if (pass_through && L == hi && c.type != HM_CNN_HEAD) A.y = reinterpret_cast<bf16 *>(y_final);
    if (tr.stash_heads.count(L))  // capture the input of a backward-pack head
      HM_CUDA(cudaMemcpyAsync(rt.stash_dev.at(L) + s0 * bnd(rt, L), A.x, (int64_t)u * bnd(rt, L),
                              cudaMemcpyDeviceToDevice, s));
    switch (c.type) {
      case HM_CNN_CONV:
        HM_TRY(gemm::run_conv(1, A.x, wsh + P.w1, A.y, u, c.h, c.w, c.cin, c.cout, HM_EPI_RELU_BF16, w + P.b1,
                              nullptr, s));
        break;
      case HM_CNN_DOWN:
        HM_TRY(gemm::run_conv(1, A.x, wsh + P.w1, A.a, u, c.h, c.w, c.cin, c.cout, HM_EPI_RELU_BF16, w + P.b1,
                              nullptr, s));
        HM_TRY(cnn::pool2_fwd(A.a, A.y, u, c.h, c.w, c.cout, s));
        break;
      case HM_CNN_RES:
        HM_TRY(gemm::run_conv(1, A.x, wsh + P.w1, A.h, u, c.h, c.w, c.cin, c.cout, HM_EPI_RELU_BF16, w + P.b1,
                              nullptr, s));
        HM_TRY(gemm::run_conv(1, A.h, wsh + P.w2, A.y, u, c.h, c.w, c.cout, c.cout, HM_EPI_RESID_RELU_BF16,
                              w + P.b2, A.x, s));
        break;
      case HM_CNN_RES2: {  // relu(conv(x) + b + skip), skip from the relay store
        const uint8_t *skip = rt.relay_y.at(c.skip) + s0 * bnd(rt, c.skip + 1);
        HM_TRY(gemm::run_conv(1, A.x, wsh + P.w1, A.y, u, c.h, c.w, c.cin, c.cout, HM_EPI_RESID_RELU_BF16, w + P.b1,
                              skip, s));
        break;
      }
      default: {  // head: global average pool, classifier, cross-entropy
        HM_TRY(cnn::gap_fwd(A.x, A.pooled, u, c.h * c.w, c.cin, s));
        HM_TRY(gemm::run(A.pooled, wsh + P.w1, rt.CT.logits, u, rt.classes_p, c.cin, c.cin, c.cin, rt.classes_p, 0, 0,
                         HM_EPI_STORE_F32, w + P.b1, nullptr, 0, s, 0));
        HM_TRY(layers::cross_entropy(rt.CT.logits, rt.labels + s0, u, rt.classes_p, rt.classes, A.dlog,
                                     rt.count_loss ? rt.loss_cur : rt.loss_sink,
                                     (float)(1.0 / (double)rt.global_tokens), s));
        break;
      }
    }
    if (rt.relay_y.count(L))  // this layer's output feeds a later res2's skip input
      HM_CUDA(cudaMemcpyAsync(rt.relay_y.at(L) + s0 * bnd(rt, L + 1), A.y, (int64_t)u * bnd(rt, L + 1),
                              cudaMemcpyDeviceToDevice, s));
    if (L == hi && y_final && !pass_through && c.type != HM_CNN_HEAD)
      HM_CUDA(cudaMemcpyAsync(y_final, A.y, (int64_t)u * bnd(rt, L + 1), cudaMemcpyDeviceToDevice, s));
  }
  return HM_OK;
}

// Backward of layers [hi .. lo] for one member: dy_in is the gradient of the
// pack output (null when the pack ends in the head), dx_out receives the
// gradient of the pack input (null for the pack holding layer 0).
static int cnn_backward_pack(hm_runtime &rt, TaskRt &tr, int lo, int hi, int u, int64_t s0, uint8_t *store, int64_t n,
                             int64_t s_off, const uint8_t *dy_in, uint8_t *dx_out) {
  cudaStream_t s = rt.s_compute;
  if (!store) {
    store = rt.work_store;
    n = u;
    s_off = 0;
  }
  CnnScratch &T = rt.CT;
  const bf16 *dy = reinterpret_cast<const bf16 *>(dy_in);
  for (int L = hi; L >= lo; --L) {
    const hm_cnn_layer &c = rt.cnn[L];
    const CnnParam &P = rt.cnn_lay[L];
    const int64_t off = rt.w_off[L] - rt.w_off[lo];
    const bf16 *wsh = rt.slots.wsh[tr.w_slot] + off;
    float *dw = rt.slots.dw[tr.dw_slot] + off;
    CnnActs A = cnn_acts(rt, store, lo, L, n, s_off);
    const int64_t M = (int64_t)u * c.h * c.w;
    const bool need_dx = L > 0;
    bf16 *dx = (L == lo && dx_out) ? reinterpret_cast<bf16 *>(dx_out) : T.g[(hi - L) & 1];
    if (rt.relay_g.count(L)) {  // the skip path's gradient joins the trunk gradient of this layer's output
      if (!dy) return fail(HM_ERR_INTERNAL, "relay source without a trunk gradient");
      HM_TRY(cnn::add_bf16(dy, rt.relay_g.at(L) + s0 * bnd(rt, L + 1), T.gsum, (int64_t)u * bnd(rt, L + 1) / 2, s));
      dy = T.gsum;
    }
    switch (c.type) {
      case HM_CNN_RES2: {  // dz = dy * (y > 0): the conv's gradient and, unchanged, the skip's
        if (!dy) return fail(HM_ERR_INTERNAL, "cnn backward without an incoming gradient");
        HM_TRY(cnn::relu_bwd(dy, A.y, T.dz, M * c.cout, s));
        HM_TRY(layers::bias_grad(T.dz, 1, dw + P.b1, M, c.cout, c.cout, s));
        HM_TRY(gemm::run_conv(3, T.dz, A.x, dw + P.w1, u, c.h, c.w, c.cin, c.cout, HM_EPI_ACC_F32, nullptr, nullptr, s));
        HM_CUDA(cudaMemcpyAsync(rt.relay_g.at(c.skip) + s0 * bnd(rt, c.skip + 1), T.dz, M * c.cout * 2,
                                cudaMemcpyDeviceToDevice, s));
        if (need_dx)
          HM_TRY(gemm::run_conv(2, T.dz, wsh + P.w1, dx, u, c.h, c.w, c.cin, c.cout, HM_EPI_STORE_BF16, nullptr,
                                nullptr, s));
        break;
      }
      case HM_CNN_HEAD: {
        // dW_fc += dlog^T . pooled; db_fc += sum dlog; dpooled = dlog . W_fc; dx = dpooled / P
        HM_TRY(gemm::run(A.dlog, A.pooled, dw + P.w1, rt.classes_p, c.cin, u, rt.classes_p, c.cin, c.cin, 1, 1,
                         HM_EPI_ACC_F32, nullptr, nullptr, 0, s, 0));
        HM_TRY(layers::bias_grad(A.dlog, 1, dw + P.b1, u, rt.classes_p, rt.classes_p, s));
        HM_TRY(gemm::run(A.dlog, wsh + P.w1, T.dpool, u, c.cin, rt.classes_p, rt.classes_p, c.cin, c.cin, 0, 1,
                         HM_EPI_STORE_F32, nullptr, nullptr, 0, s, 0));
        HM_TRY(cnn::gap_bwd(T.dpool, dx, u, c.h * c.w, c.cin, s));
        break;
      }
      case HM_CNN_CONV:
      case HM_CNN_DOWN: {
        if (!dy) return fail(HM_ERR_INTERNAL, "cnn backward without an incoming gradient");
        if (c.type == HM_CNN_CONV)
          HM_TRY(cnn::relu_bwd(dy, A.y, T.dz, M * c.cout, s));
        else
          HM_TRY(cnn::pool2_relu_bwd(dy, A.a, T.dz, u, c.h, c.w, c.cout, s));
        HM_TRY(layers::bias_grad(T.dz, 1, dw + P.b1, M, c.cout, c.cout, s));
        HM_TRY(gemm::run_conv(3, T.dz, A.x, dw + P.w1, u, c.h, c.w, c.cin, c.cout, HM_EPI_ACC_F32, nullptr, nullptr, s));
        if (need_dx)
          HM_TRY(gemm::run_conv(2, T.dz, wsh + P.w1, dx, u, c.h, c.w, c.cin, c.cout, HM_EPI_STORE_BF16, nullptr,
                                nullptr, s));
        break;
      }
      default: {  // residual block
        if (!dy) return fail(HM_ERR_INTERNAL, "cnn backward without an incoming gradient");
        HM_TRY(cnn::relu_bwd(dy, A.y, T.dz2, M * c.cout, s));  // dz2 = dy * (y > 0)
        HM_TRY(layers::bias_grad(T.dz2, 1, dw + P.b2, M, c.cout, c.cout, s));
        HM_TRY(gemm::run_conv(3, T.dz2, A.h, dw + P.w2, u, c.h, c.w, c.cout, c.cout, HM_EPI_ACC_F32, nullptr, nullptr,
                              s));
        // dz1 = dgrad(dz2) * (h > 0)
        HM_TRY(gemm::run_conv(2, T.dz2, wsh + P.w2, T.dz, u, c.h, c.w, c.cout, c.cout, HM_EPI_DRELU_BF16, nullptr,
                              A.h, s));
        HM_TRY(layers::bias_grad(T.dz, 1, dw + P.b1, M, c.cout, c.cout, s));
        HM_TRY(gemm::run_conv(3, T.dz, A.x, dw + P.w1, u, c.h, c.w, c.cin, c.cout, HM_EPI_ACC_F32, nullptr, nullptr,
                              s));
        // dx = dgrad(dz1) + dz2 (the identity path)
        if (need_dx)
          HM_TRY(gemm::run_conv(2, T.dz, wsh + P.w1, dx, u, c.h, c.w, c.cin, c.cout, HM_EPI_ADD_BF16, nullptr, T.dz2,
                                s));
        break;
      }
    }
    dy = dx;
  }
  return HM_OK;
}

// ---------------------------------------------------------------------------
// layer compute
// ---------------------------------------------------------------------------
struct LayerW {
  const float *w;   // fp32 master (for LN params, biases, embedding)
  const bf16 *wsh;  // bf16 shadow (GEMM operands)
  float *dw;        // gradient block (fp32)
  const ParamLayout *p;
};

static LayerW layer_weights(hm_runtime &rt, const TaskRt &tr, int lo, int L, int w_slot, int dw_slot) {
  LayerW lw;
  const int64_t off = rt.w_off[L] - rt.w_off[lo];
  lw.w = rt.slots.w[w_slot] + off;
  lw.wsh = rt.slots.wsh[w_slot] + off;
  lw.dw = dw_slot >= 0 ? rt.slots.dw[dw_slot] + off : nullptr;
  lw.p = &rt.lay[L];
  (void)tr;
  return lw;
}

// GEMM on the compute stream: the bf16 tcgen05 kernel, or in the parity mode
// the three-plane split product over fp32 operands (same arguments)
static int G(hm_runtime &rt, const void *A, const void *B, void *D, int64_t M, int64_t N, int64_t K, int64_t lda,
             int64_t ldb, int64_t ldd, int a_mn, int b_mn, int epi, const float *bias = nullptr, void *aux = nullptr,
             int64_t ld_aux = 0) {
  if (rt.precise)
    return prec::gemm(static_cast<const float *>(A), static_cast<const float *>(B), D, M, N, K, lda, ldb, ldd, a_mn,
                      b_mn, epi, bias, aux, ld_aux, rt.s_compute, rt.psa, rt.psa_n, rt.psb, rt.psb_n, rt.pc32,
                      rt.pc32_n);
  return gemm::run(A, B, D, M, N, K, lda, ldb, ldd, a_mn, b_mn, epi, bias, aux, ld_aux, rt.s_compute, 0);
}
// a GEMM weight operand: the bf16 shadow, or the fp32 master in the parity mode
static const void *wop(const hm_runtime &rt, const LayerW &W, int64_t off) {
  return rt.precise ? static_cast<const void *>(W.w + off) : static_cast<const void *>(W.wsh + off);
}
static int ln_fwd_any(hm_runtime &rt, const float *x, const float *g, const float *b, void *y, float *mean,
                      float *rstd, int64_t rows, int d) {
  if (rt.precise) return prec::ln_fwd(x, g, b, static_cast<float *>(y), mean, rstd, rows, d, rt.s_compute);
  return layers::ln_fwd(x, g, b, y, mean, rstd, rows, d, rt.s_compute);
}

static int block_fwd(hm_runtime &rt, const Acts &A, const float *x, float *y, int u, const LayerW &W) {
  const int64_t M = (int64_t)u * rt.S, d = rt.m.d_model;
  cudaStream_t s = rt.s_compute;
  const ParamLayout &P = *W.p;
  HM_TRY(ln_fwd_any(rt, x, W.w + P.ln1_g, W.w + P.ln1_b, A.ln1, A.mean1, A.rstd1, M, (int)d));
  HM_TRY(G(rt, A.ln1, wop(rt, W, P.w_qkv), A.qkv, M, 3 * d, d, d, d, 3 * d, 0, 0, HM_EPI_STORE_BF16, W.w + P.b_qkv));
  if (rt.precise)
    HM_TRY(prec::attn_forward(reinterpret_cast<const float *>(A.qkv), reinterpret_cast<float *>(A.o), A.lse, u, rt.S,
                              rt.H, rt.DH, rt.m.causal, s));
  else
    HM_TRY(attn::forward(A.qkv, A.o, A.lse, u, rt.S, rt.H, rt.DH, rt.m.causal, s));
  HM_TRY(G(rt, A.o, wop(rt, W, P.w_proj), A.h1, M, d, d, d, d, d, 0, 0, HM_EPI_RESID_F32, W.w + P.b_proj,
           const_cast<float *>(x), d));
  HM_TRY(ln_fwd_any(rt, A.h1, W.w + P.ln2_g, W.w + P.ln2_b, A.ln2, A.mean2, A.rstd2, M, (int)d));
  HM_TRY(G(rt, A.ln2, wop(rt, W, P.w_fc1), A.a, M, 4 * d, d, d, d, 4 * d, 0, 0, HM_EPI_GELU_BF16, W.w + P.b_fc1,
           A.hpre, 4 * d));
  HM_TRY(G(rt, A.a, wop(rt, W, P.w_fc2), y, M, d, 4 * d, 4 * d, 4 * d, d, 0, 0, HM_EPI_RESID_F32, W.w + P.b_fc2, A.h1,
           d));
  return HM_OK;
}

// LN_f + LM head + cross-entropy (dlogits stored for the backward pass).
static int head_fwd(hm_runtime &rt, const Acts &A, int u, int64_t s0, const LayerW &W) {
  const int64_t M = (int64_t)u * rt.S, d = rt.m.d_model;
  cudaStream_t s = rt.s_compute;
  const ParamLayout &P = *W.p;
  HM_TRY(ln_fwd_any(rt, A.yl, W.w + P.lnf_g, W.w + P.lnf_b, A.lnf, A.meanf, A.rstdf, M, (int)d));
  HM_TRY(G(rt, A.lnf, wop(rt, W, P.w_head), rt.T.logits, M, rt.Vp, d, d, d, rt.Vp, 0, 0, HM_EPI_STORE_F32));
  double *loss = rt.count_loss ? rt.loss_cur : rt.loss_sink;
  const float scale = (float)(1.0 / (double)rt.global_tokens);
  if (rt.precise)
    return prec::cross_entropy(rt.T.logits, rt.labels + s0 * rt.S, M, rt.Vp, rt.V, reinterpret_cast<float *>(A.dlog),
                               loss, scale, s);
  return layers::cross_entropy(rt.T.logits, rt.labels + s0 * rt.S, M, rt.Vp, rt.V, A.dlog, loss, scale, s);
}

static int head_bwd(hm_runtime &rt, const Acts &A, int u, const LayerW &W) {
  const int64_t M = (int64_t)u * rt.S, d = rt.m.d_model, Vp = rt.Vp;
  cudaStream_t s = rt.s_compute;
  const ParamLayout &P = *W.p;
  Scratch &T = rt.T;
  HM_TRY(G(rt, A.dlog, wop(rt, W, P.w_head), T.dln, M, d, Vp, Vp, d, d, 0, 1, HM_EPI_STORE_F32));
  HM_TRY(G(rt, A.dlog, A.lnf, W.dw + P.w_head, Vp, d, M, Vp, d, d, 1, 1, HM_EPI_ACC_F32));
  HM_TRY(layers::ln_bwd(T.dln, A.yl, A.meanf, A.rstdf, W.w + P.lnf_g, nullptr, T.dyh, nullptr, W.dw + P.lnf_g,
                        W.dw + P.lnf_b, M, (int)d, s));
  return HM_OK;
}

static int block_bwd(hm_runtime &rt, const Acts &A, const float *x, const float *dy, float *dx, int u,
                     const LayerW &W) {
  const int64_t M = (int64_t)u * rt.S, d = rt.m.d_model;
  cudaStream_t s = rt.s_compute;
  const ParamLayout &P = *W.p;
  Scratch &T = rt.T;
  const int opbf = rt.precise ? 0 : 1;  // the dgrad outputs feeding bias gradients are bf16 operands
  const void *dyop = dy;
  if (!rt.precise) {
    HM_TRY(layers::cast_f32_bf16(dy, T.dy_bf, M * d, s));
    dyop = T.dy_bf;
  }
  HM_TRY(layers::bias_grad(dy, 0, W.dw + P.b_fc2, M, (int)d, d, s));
  HM_TRY(G(rt, dyop, A.a, W.dw + P.w_fc2, d, 4 * d, M, d, 4 * d, 4 * d, 1, 1, HM_EPI_ACC_F32));
  HM_TRY(G(rt, dyop, wop(rt, W, P.w_fc2), T.dh, M, 4 * d, d, d, 4 * d, 4 * d, 0, 1, HM_EPI_DGELU_BF16, nullptr,
           A.hpre, 4 * d));
  HM_TRY(layers::bias_grad(T.dh, opbf, W.dw + P.b_fc1, M, (int)(4 * d), 4 * d, s));
  HM_TRY(G(rt, T.dh, A.ln2, W.dw + P.w_fc1, 4 * d, d, M, 4 * d, d, d, 1, 1, HM_EPI_ACC_F32));
  HM_TRY(G(rt, T.dh, wop(rt, W, P.w_fc1), T.dln, M, d, 4 * d, 4 * d, d, d, 0, 1, HM_EPI_STORE_F32));
  HM_TRY(layers::ln_bwd(T.dln, A.h1, A.mean2, A.rstd2, W.w + P.ln2_g, dy, T.dh1, rt.precise ? nullptr : T.dh1_bf,
                        W.dw + P.ln2_g, W.dw + P.ln2_b, M, (int)d, s));
  HM_TRY(layers::bias_grad(T.dh1, 0, W.dw + P.b_proj, M, (int)d, d, s));
  const void *dh1op = rt.precise ? static_cast<const void *>(T.dh1) : static_cast<const void *>(T.dh1_bf);
  HM_TRY(G(rt, dh1op, A.o, W.dw + P.w_proj, d, d, M, d, d, d, 1, 1, HM_EPI_ACC_F32));
  HM_TRY(G(rt, dh1op, wop(rt, W, P.w_proj), T.dout, M, d, d, d, d, d, 0, 1, HM_EPI_STORE_BF16));
  if (rt.precise)
    HM_TRY(prec::attn_backward(reinterpret_cast<const float *>(A.qkv), reinterpret_cast<const float *>(A.o),
                               reinterpret_cast<const float *>(T.dout), A.lse, T.dvec,
                               reinterpret_cast<float *>(T.dqkv), u, rt.S, rt.H, rt.DH, rt.m.causal, s));
  else
    HM_TRY(attn::backward(A.qkv, A.o, T.dout, A.lse, T.dvec, T.dq, T.dqkv, u, rt.S, rt.H, rt.DH, rt.m.causal, s));
  HM_TRY(layers::bias_grad(T.dqkv, opbf, W.dw + P.b_qkv, M, (int)(3 * d), 3 * d, s));
  HM_TRY(G(rt, T.dqkv, A.ln1, W.dw + P.w_qkv, 3 * d, d, M, 3 * d, d, d, 1, 1, HM_EPI_ACC_F32));
  HM_TRY(G(rt, T.dqkv, wop(rt, W, P.w_qkv), T.dln, M, d, 3 * d, 3 * d, d, d, 0, 1, HM_EPI_STORE_F32));
  HM_TRY(layers::ln_bwd(T.dln, x, A.mean1, A.rstd1, W.w + P.ln1_g, T.dh1, dx, nullptr, W.dw + P.ln1_g,
                        W.dw + P.ln1_b, M, (int)d, s));
  return HM_OK;
}

// ---------------------------------------------------------------------------
// task members
// ---------------------------------------------------------------------------
static bool is_head(const hm_runtime &rt, int L) { return L == rt.R - 1; }

// Forward of layers [lo, hi] for one member.  `store` != null keeps every
// layer's activations (n samples, member at s0); otherwise one scratch layer
// slot is reused and the hidden state ping-pongs between two buffers.
static int forward_pack(hm_runtime &rt, TaskRt &tr, int lo, int hi, int u, int64_t s0, const float *x_in,
                        const int32_t *tok_in, uint8_t *store, int64_t n, int64_t s_off, float *y_final,
                        float *ship = nullptr) {
  const int64_t M = (int64_t)u * rt.S, d = rt.m.d_model;
  cudaStream_t s = rt.s_compute;
  const float *x = x_in;
  int hsel = 0;
  for (int L = lo; L <= hi; ++L) {
    const bool head = is_head(rt, L);
    Acts A = store ? acts_at(rt, store_layer(rt, store, lo, L, n), head, n, s_off)
                   : acts_at(rt, rt.work_store, head, u, 0);
    LayerW W = layer_weights(rt, tr, lo, L, tr.w_slot, -1);
    if (L == lo) {
      float *dst = store ? A.x : rt.T.h[hsel];
      if (L == 0) {
        HM_TRY(layers::embed_fwd(tok_in, W.w + W.p->wte, W.w + W.p->wpe, dst, u, rt.S, (int)d, s));
        x = dst;
      } else if (store) {
        HM_CUDA(cudaMemcpyAsync(dst, x_in, M * d * 4, cudaMemcpyDeviceToDevice, s));
        x = dst;
      }
    }
    if (L == lo && ship)  // Harmony-PP seam: the shared pack's input goes to the peer
      HM_CUDA(cudaMemcpyAsync(ship, x, M * d * 4, cudaMemcpyDeviceToDevice, s));
    if (tr.stash_heads.count(L)) {  // capture the input of a backward-pack head
      uint8_t *dst = rt.stash_dev.at(L);
      if (L == 0) {
        HM_CUDA(cudaMemcpyAsync(dst + s0 * rt.S * 4, tok_in, M * 4, cudaMemcpyDeviceToDevice, s));
      } else {
        HM_CUDA(cudaMemcpyAsync(dst + s0 * rt.S * d * 4, x, M * d * 4, cudaMemcpyDeviceToDevice, s));
      }
    }
    float *y;
    if (head) {
      y = store ? A.yl : rt.T.tmp;
    } else if (L < hi) {
      y = store ? acts_at(rt, store_layer(rt, store, lo, L + 1, n), is_head(rt, L + 1), n, s_off).x : rt.T.h[hsel ^ 1];
    } else {
      y = y_final ? y_final : rt.T.tmp;
    }
    HM_TRY(block_fwd(rt, A, x, y, u, W));
    if (head) {
      Acts Ah = A;
      if (!store) Ah.yl = y;
      HM_TRY(head_fwd(rt, Ah, u, s0, W));
      if (y_final) HM_CUDA(cudaMemcpyAsync(y_final, y, M * d * 4, cudaMemcpyDeviceToDevice, s));
    }
    x = y;
    hsel ^= 1;
  }
  return HM_OK;
}

static int backward_pack(hm_runtime &rt, TaskRt &tr, int lo, int hi, int u, int64_t s0, uint8_t *store, int64_t n,
                         int64_t s_off, const float *dy_in, float *dx_out, const int32_t *tok_in) {
  const float *dy = dy_in;
  for (int L = hi; L >= lo; --L) {
    const bool head = is_head(rt, L);
    Acts A = acts_at(rt, store_layer(rt, store, lo, L, n), head, n, s_off);
    LayerW W = layer_weights(rt, tr, lo, L, tr.w_slot, tr.dw_slot);
    if (head) {
      HM_TRY(head_bwd(rt, A, u, W));
      dy = rt.T.dyh;
    }
    if (!dy) return fail(HM_ERR_INTERNAL, "backward without an incoming gradient");
    float *dx = (L == lo && dx_out) ? dx_out : rt.T.g[(hi - L) & 1];
    HM_TRY(block_bwd(rt, A, A.x, dy, dx, u, W));
    dy = dx;
    if (L == 0)
      HM_TRY(layers::embed_bwd(tok_in, dy, W.dw + W.p->wte, W.dw + W.p->wpe, u, rt.S, (int)rt.m.d_model,
                               rt.s_compute));
  }
  (void)s0;
  return HM_OK;
}

static int run_member(hm_runtime &rt, int task, int g) {
  TaskInfo &t = rt.plan->tasks[task];
  TaskRt &tr = rt.trt[task];
  const int u = t.group[g];
  const int64_t s0 = tr.s0[g];
  const int64_t d = rt.m.d_model;
  const int64_t rowsd = (int64_t)rt.S * d;
  cudaStream_t s = rt.s_compute;
  if (g == 0) {
    if (rt.w_planar) {
      // bf16 payloads: the hi planes already are the bf16 operands; rebuild the
      // fp32 values the kernels read (forward: each layer's fp32 prefix;
      // backward: whole layers, the U task updates them)
      int64_t soff = 0;
      for (int L = t.lo; L <= t.hi; ++L) {
        const int64_t o = rt.w_off[L] - rt.w_off[t.lo];
        const ParamLayout &P = rt.lay[L];
        if (t.type == HM_TASK_F) {
          HM_TRY(layers::w_join(rt.slots.wsh[tr.w_slot] + o, rt.slots.wlo[tr.w_slot] + soff, rt.slots.w[tr.w_slot] + o,
                                P.f32n, s));
          soff += P.f32n;
        } else {
          HM_TRY(layers::w_join(rt.slots.wsh[tr.w_slot] + o, rt.slots.dw[tr.dw_slot] + o, rt.slots.w[tr.w_slot] + o,
                                P.size, s));
        }
      }
    } else if (rt.precise) {
      // parity mode: the GEMMs split the fp32 master weights themselves
    } else if (rt.family == HM_FAMILY_GPT) {
      // bf16 operand copy of the pack's master weights, right after swap-in
      // (nearest, ties toward zero: the same bits as the bf16-payload hi planes)
      HM_TRY(layers::cast_w_bf16(rt.slots.w[tr.w_slot], rt.slots.wsh[tr.w_slot], tr.params, s));
    } else {
      HM_TRY(layers::cast_f32_bf16(rt.slots.w[tr.w_slot], rt.slots.wsh[tr.w_slot], tr.params, s));
    }
    if (t.type == HM_TASK_B) HM_CUDA(cudaMemsetAsync(rt.slots.dw[tr.dw_slot], 0, tr.params * 4, s));
  }
  if (rt.family == HM_FAMILY_CNN) {
    // byte offsets of this member inside the boundary buffers (x(L) per sample)
    auto at = [&](const void *base, int L) -> uint8_t * {
      return base ? const_cast<uint8_t *>(static_cast<const uint8_t *>(base)) + s0 * bnd(rt, L) : nullptr;
    };
    if (t.type == HM_TASK_F) {
      const uint8_t *x_in = t.lo == 0 ? at(rt.tokens, 0) : at(tr.in_buf ? tr.in_buf : rt.carry[tr.carry_in], t.lo);
      if (tr.store_shared)
        return cnn_forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, rt.shared_store, rt.minibatch, s0, nullptr);
      uint8_t *y = tr.out_buf ? at(tr.out_buf, t.hi + 1) : tr.carry_out >= 0 ? at(rt.carry[tr.carry_out], t.hi + 1) : nullptr;
      return cnn_forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, nullptr, 0, 0, y);
    }
    uint8_t *dx = t.lo == 0 ? nullptr : at(tr.out_buf ? tr.out_buf : rt.dcarry[tr.carry_out], t.lo);
    if (tr.from_shared)
      return cnn_backward_pack(rt, tr, t.lo, t.hi, u, s0, rt.shared_store, rt.minibatch, s0, nullptr, dx);
    // recompute the pack from its stashed input, then backward
    const uint8_t *x_in = at(rt.slots.stash_in[tr.stash_slot], t.lo);
    HM_TRY(cnn_forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, nullptr, 0, 0, nullptr));
    const uint8_t *dy = at(tr.in_buf ? tr.in_buf : rt.dcarry[tr.carry_in], t.hi + 1);
    return cnn_backward_pack(rt, tr, t.lo, t.hi, u, s0, nullptr, 0, 0, dy, dx);
  }
  if (t.type == HM_TASK_F) {
    const float *x_in = t.lo == 0 ? nullptr
                        : tr.in_buf ? tr.in_buf + s0 * rowsd
                                    : rt.carry[tr.carry_in] + s0 * rowsd;
    const int32_t *tok = rt.tokens + s0 * rt.S;
    if (tr.store_shared)
      return forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, tok, rt.shared_store, rt.minibatch, s0, nullptr);
    if (tr.ship_input)
      return forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, tok, nullptr, 0, 0, nullptr, tr.out_buf + s0 * rowsd);
    float *y = tr.out_buf ? tr.out_buf + s0 * rowsd : tr.carry_out >= 0 ? rt.carry[tr.carry_out] + s0 * rowsd : nullptr;
    return forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, tok, nullptr, 0, 0, y);
  }
  // backward
  float *dx = (t.lo == 0) ? nullptr : tr.out_buf ? tr.out_buf + s0 * rowsd : rt.dcarry[tr.carry_out] + s0 * rowsd;
  if (tr.from_shared)
    return backward_pack(rt, tr, t.lo, t.hi, u, s0, rt.shared_store, rt.minibatch, s0, nullptr, dx,
                         rt.tokens + s0 * rt.S);
  if (tr.remote_shared) {
    // the shared pack's forward ran on the peer: recompute it from the shipped
    // input (its cross-entropy is not counted again), then backward from the head
    const float *x_in = t.lo == 0 ? nullptr : tr.in_buf + s0 * rowsd;
    const int32_t *tok = rt.tokens + s0 * rt.S;
    rt.count_loss = false;
    int rc = forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, tok, rt.work_store, u, 0, nullptr);
    rt.count_loss = true;
    HM_TRY(rc);
    return backward_pack(rt, tr, t.lo, t.hi, u, s0, rt.work_store, u, 0, nullptr, dx, tok);
  }
  // recompute from the stash, keeping activations in the work store
  uint8_t *st = rt.slots.stash_in[tr.stash_slot];
  const float *x_in = t.lo == 0 ? nullptr : reinterpret_cast<const float *>(st) + s0 * rowsd;
  const int32_t *tok = t.lo == 0 ? reinterpret_cast<const int32_t *>(st) + s0 * rt.S : rt.tokens + s0 * rt.S;
  HM_TRY(forward_pack(rt, tr, t.lo, t.hi, u, s0, x_in, tok, rt.work_store, u, 0, nullptr));
  const float *dy = tr.in_buf ? tr.in_buf + s0 * rowsd : rt.dcarry[tr.carry_in] + s0 * rowsd;
  return backward_pack(rt, tr, t.lo, t.hi, u, s0, rt.work_store, u, 0, dy, dx, tok);
}

// ---------------------------------------------------------------------------
// load: slots, buffers, actions
// ---------------------------------------------------------------------------
static int load_plan(hm_runtime &rt, Plan *plan, int rank, int minibatch) {
  rt.plan = plan;
  rt.rank = rank;
  rt.minibatch = minibatch;
  const int n_tasks = (int)plan->tasks.size();
  rt.trt.assign(n_tasks, TaskRt{});
  const int64_t d = rt.m.d_model;
  // ---- which tasks run here; structural checks ------------------------------
  std::vector<int> mine;
  for (auto &t : plan->tasks)
    if (t.dev_id == rank) mine.push_back(t.index);
  if (mine.empty()) return fail(HM_ERR_VALIDATION, "no task is bound to this rank");
  rt.p2p_mode = false;
  for (auto &it : plan->items)
    if (!it.rec.is_compute && it.rec.channel == HM_PEER2PEER) rt.p2p_mode = true;
  if (rt.p2p_mode && !rt.shared_arena)
    return fail(HM_ERR_VALIDATION,
                "peer-to-peer hand-offs (Harmony-PP, N>1) need shared host arenas: call hm_runtime_share_arenas");
  rt.dp_shard = plan->dp_sharded && plan->gpu_count > 1;  // (one rank: the shard is the whole pack)
  if (rt.dp_shard) {
    if (!rt.shared_arena)
      return fail(HM_ERR_VALIDATION, "the sharded Harmony-DP update needs one host arena shared by all ranks "
                                     "(hm_runtime_share_arenas)");
    if (rt.w_planar) return fail(HM_ERR_VALIDATION, "the sharded update and bf16 swap payloads are exclusive");
    if (!(rt.comm || rt.ipc_reduce) || rt.nranks != plan->gpu_count)
      return fail(HM_ERR_VALIDATION, "the sharded update needs the job's gradient communicator over all " +
                                         std::to_string(plan->gpu_count) + " ranks (init_comm / init_ipc_reduce "
                                         "before load)");
  }
  int last_f = -1, shared_b = -1;
  int64_t u_max = 1, pmax = 0, f32max = 0;
  int64_t kmax = 0, dwmax = 0;  // K slot / dW slot parameters (the sharded update shrinks K, pads dW)
  std::vector<int> heads;  // stash head layers produced here
  for (int ti : mine) {
    TaskInfo &t = plan->tasks[ti];
    TaskRt &tr = rt.trt[ti];
    tr.params = rt.w_off[t.hi + 1] - rt.w_off[t.lo];
    pmax = std::max(pmax, tr.params);
    kmax = std::max(kmax, tr.params);
    dwmax = std::max(dwmax, tr.params);
    if (t.type == HM_TASK_U && rt.dp_shard) {
      dp_shard(tr.params, plan->gpu_count, rank, &tr.sh_off, &tr.sh_len);
      tr.sh_chunk = dp_shard_chunk(tr.params, plan->gpu_count);
      dwmax = std::max(dwmax, tr.sh_chunk * plan->gpu_count);  // reduce-scatter send buffer
    }
    if (rt.w_planar && t.type == HM_TASK_F) {
      int64_t f = 0;
      for (int L = t.lo; L <= t.hi; ++L) f += rt.lay[L].f32n;
      f32max = std::max(f32max, f);
    }
    int64_t acc = 0;
    for (int u : t.group) {
      tr.s0.push_back(acc);
      acc += u;
      u_max = std::max<int64_t>(u_max, u);
    }
    if (t.type != HM_TASK_U && acc != minibatch)
      return fail(HM_ERR_VALIDATION, "task group does not cover this rank's minibatch");
    if (t.type == HM_TASK_F) last_f = ti;
    if (t.type == HM_TASK_B && !t.recompute) shared_b = ti;
    for (auto &e : t.outputs)
      if (e.tensor == HM_SX && e.channel == HM_MESSAGE_PASSING) {
        tr.stash_heads.insert(e.layer);
        heads.push_back(e.layer);
      }
  }
  // the last F task of the graph (its Y feeds the shared B task)
  int graph_last_f = -1;
  for (auto &t : plan->tasks)
    if (t.type == HM_TASK_F && (t.dev_id == rank || rt.p2p_mode)) graph_last_f = std::max(graph_last_f, t.index);
  const bool local_seam = last_f >= 0 && shared_b >= 0 && last_f == graph_last_f;
  if (!rt.p2p_mode && !local_seam) return fail(HM_ERR_VALIDATION, "rank holds no complete F/B chain");
  if (local_seam) {
    if (plan->tasks[last_f].lo != plan->tasks[shared_b].lo || plan->tasks[last_f].hi != plan->tasks[shared_b].hi)
      return fail(HM_ERR_VALIDATION, "shared pack mismatch");
    rt.trt[last_f].store_shared = true;
    rt.trt[shared_b].from_shared = true;
    rt.shared_lo = plan->tasks[last_f].lo;
    rt.shared_hi = plan->tasks[last_f].hi;
  } else {
    rt.shared_lo = rt.shared_hi = -1;
  }
  // peer-to-peer roles of my tasks
  for (int ti : mine) {
    TaskInfo &t = plan->tasks[ti];
    TaskRt &tr = rt.trt[ti];
    for (auto &e : t.inputs)
      if (e.channel == HM_PEER2PEER) {
        if (t.type == HM_TASK_B && e.tensor == HM_Y) tr.remote_shared = true;
        tr.in_buf = reinterpret_cast<float *>(1);  // allocated below
      }
    for (auto &e : t.outputs)
      if (e.channel == HM_PEER2PEER) {
        tr.out_buf = reinterpret_cast<float *>(1);
        if (t.type == HM_TASK_F && e.tensor == HM_Y && ti == graph_last_f) tr.ship_input = true;
      }
    if (t.type != HM_TASK_U && t.hi == rt.R - 1 && !(tr.store_shared || tr.from_shared || tr.ship_input ||
                                                     tr.remote_shared))
      return fail(HM_ERR_INTERNAL, "head layer outside the shared pack");
  }
  // stash regions of every head in the graph (the host arena may be shared)
  std::map<int, int64_t> all_heads;  // head -> D * x bytes
  for (auto &t : plan->tasks)
    for (auto &e : t.outputs)
      if (e.tensor == HM_SX && e.channel == HM_MESSAGE_PASSING)
        all_heads[e.layer] = (int64_t)minibatch * bnd(rt, e.layer);

  // ---- slot assignment (round robin in device order) -------------------------
  // Slot counts: 3 W and 2 K slots are the minimum the one-task-ahead schedule
  // needs; load_plan re-runs itself with more (up to 4 each, K first) when
  // alpha leaves room, so a K swap-in never waits for the swap-out of the K
  // two updates back (HM_W_SLOTS / HM_K_SLOTS pin the counts).
  static const int env_nw = getenv("HM_W_SLOTS") ? atoi(getenv("HM_W_SLOTS")) : 0;
  static const int env_nk = getenv("HM_K_SLOTS") ? atoi(getenv("HM_K_SLOTS")) : 0;
  const int NW = env_nw >= 3 ? env_nw : std::max(3, rt.slot_nw), NDW = 2,
            NK = env_nk >= 2 ? env_nk : std::max(2, rt.slot_nk), NST = 2;
  int wn = 0, dwn = 0, kn = 0, stn = 0, fcur = -1, bcur = -1;
  std::vector<int> w_owner(NW, -1), dw_owner(NDW, -1), k_owner(NK, -1), st_owner(NST, -1);
  int64_t stash_in_max = 0;
  std::map<int, int64_t> stash_bytes = all_heads;
  for (int ti : mine) {
    TaskInfo &t = plan->tasks[ti];
    TaskRt &tr = rt.trt[ti];
    if (t.type == HM_TASK_U) {
      tr.b_task = ti - 1;
      tr.k_slot = kn;
      kn = (kn + 1) % NK;
      continue;
    }
    tr.w_slot = wn;
    wn = (wn + 1) % NW;
    if (t.type == HM_TASK_F) {
      if (rt.p2p_mode) continue;
      tr.carry_in = fcur;
      if (ti != last_f) {
        tr.carry_out = (fcur + 1) & 1;
        fcur = tr.carry_out;
      }
      if (t.lo > 0 && tr.carry_in < 0) return fail(HM_ERR_INTERNAL, "F task without an input carry");
    } else {
      tr.dw_slot = dwn;
      dwn = (dwn + 1) % NDW;
      if (!rt.p2p_mode) {
        tr.carry_in = bcur;
        if (t.lo > 0) {
          tr.carry_out = (bcur + 1) & 1;
          bcur = tr.carry_out;
        }
      }
      if (t.recompute) {
        tr.stash_slot = stn;
        stn = (stn + 1) % NST;
        stash_in_max = std::max(stash_in_max, stash_bytes.count(t.lo) ? stash_bytes[t.lo] : 0);
        if (tr.carry_in < 0 && !tr.in_buf) return fail(HM_ERR_INTERNAL, "recompute B task without a gradient input");
      }
    }
  }
  // ---- device pool ------------------------------------------------------------
  const int64_t rows_mb = (int64_t)minibatch * rt.S;
  const int64_t rows_u = u_max * rt.S;
  const int64_t carry_bytes = (int64_t)minibatch * max_bnd(rt);  // one boundary tensor of the whole minibatch
  if (rt.family == HM_FAMILY_CNN) {
    for (int ti : mine)
      if (rt.trt[ti].remote_shared || rt.trt[ti].ship_input)
        return fail(HM_ERR_VALIDATION, "CNN chains: the shared pack's F and B must run on one GPU");
    for (auto &t : plan->tasks)
      for (auto &e : t.inputs)
        if (e.src_layer >= 0 && e.channel != HM_SHARED_MEMORY)
          return fail(HM_ERR_VALIDATION, "CNN chains: relays between GPUs are not executable (keep the chain on one GPU)");
  }
  int64_t max_recompute_layers = 1;
  for (int ti : mine) {
    auto &t = plan->tasks[ti];
    if (t.type == HM_TASK_B && (t.recompute || rt.trt[ti].remote_shared))
      max_recompute_layers = std::max<int64_t>(max_recompute_layers, t.hi - t.lo + 1);
  }
  int64_t work_bytes = 0, shared_bytes = 0;
  if (rt.family == HM_FAMILY_CNN) {
    // the work store holds a whole pack for one member (F without a store, B recompute)
    for (int ti : mine) {
      auto &t = plan->tasks[ti];
      if (t.type != HM_TASK_U) work_bytes = std::max(work_bytes, cnn_pack_bytes(rt, t.lo, t.hi, u_max));
    }
    if (rt.shared_lo >= 0) shared_bytes = cnn_pack_bytes(rt, rt.shared_lo, rt.shared_hi, minibatch);
  } else {
    for (int j = 0; j < max_recompute_layers; ++j)
      work_bytes += store_layer_bytes(rt, j == max_recompute_layers - 1, u_max);
    work_bytes = std::max(work_bytes, store_layer_bytes(rt, true, u_max));
    if (rt.shared_lo >= 0)
      for (int L = rt.shared_lo; L <= rt.shared_hi; ++L)
        shared_bytes += store_layer_bytes(rt, is_head(rt, L), minibatch);
  }
  struct Req { void **ptr; int64_t bytes; };
  std::vector<Req> req;
  rt.slots.w.assign(NW, nullptr);
  rt.slots.wsh.assign(NW, nullptr);
  rt.slots.wlo.assign(NW, nullptr);
  rt.slots.dw.assign(NDW, nullptr);
  rt.slots.k.assign(NK, nullptr);
  rt.slots.stash_in.assign(NST, nullptr);
  for (int i = 0; i < NW; ++i) {
    req.push_back({(void **)&rt.slots.w[i], pmax * 4});
    req.push_back({(void **)&rt.slots.wsh[i], rt.precise ? 256 : pmax * 2});
    if (rt.w_planar) req.push_back({(void **)&rt.slots.wlo[i], std::max<int64_t>(f32max * 2, 256)});
  }
  if (rt.dp_shard) {  // K slots hold one shard
    kmax = 0;
    for (int ti : mine)
      if (plan->tasks[ti].type == HM_TASK_U) kmax = std::max(kmax, rt.trt[ti].sh_chunk);
  }
  for (int i = 0; i < NDW; ++i) req.push_back({(void **)&rt.slots.dw[i], dwmax * 4});
  for (int i = 0; i < NK; ++i) req.push_back({(void **)&rt.slots.k[i], std::max<int64_t>(kmax * 8, 256)});
  for (int i = 0; i < NST; ++i) req.push_back({(void **)&rt.slots.stash_in[i], std::max<int64_t>(stash_in_max, 256)});
  for (int i = 0; i < 2; ++i) {
    req.push_back({(void **)&rt.carry[i], carry_bytes});
    req.push_back({(void **)&rt.dcarry[i], carry_bytes});
  }
  std::vector<std::pair<int, uint8_t **>> stash_ptrs;
  rt.stash_dev.clear();
  for (int L : heads) rt.stash_dev[L] = nullptr;
  for (auto &kv : rt.stash_dev) req.push_back({(void **)&kv.second, stash_bytes[kv.first]});
  // peer-to-peer buffers: one receive and one source buffer per task (no reuse
  // inside an iteration; reuse across iterations is signal-ordered)
  std::vector<std::pair<int, float **>> out_bufs;
  for (int ti : mine) {
    TaskRt &tr = rt.trt[ti];
    if (tr.in_buf) req.push_back({(void **)&tr.in_buf, carry_bytes});
    if (tr.out_buf) {
      req.push_back({(void **)&tr.out_buf, carry_bytes});
      out_bufs.push_back({ti, &tr.out_buf});
    }
  }
  // per-item completion counters, then (ready, read) counters per task for the IPC gradient sum
  req.push_back({(void **)&rt.sig, (int64_t)(plan->items.size() + 2 * plan->tasks.size()) * 4 + 64});
  if (rt.ipc_reduce) req.push_back({(void **)&rt.ar_tmp, pmax * 4});
  req.push_back({(void **)&rt.loss_sink, 256});
  req.push_back({(void **)&rt.shared_store, shared_bytes});
  req.push_back({(void **)&rt.work_store, work_bytes});
  Scratch &T = rt.T;
  if (rt.family == HM_FAMILY_CNN) {
    int64_t act = 0, cmax = 0;  // largest per-sample activation of any layer, widest channel count
    for (auto &c : rt.cnn) {
      act = std::max(act, (int64_t)c.h * c.w * std::max(c.cin, c.cout) * 2);
      cmax = std::max<int64_t>(cmax, std::max(c.cin, c.cout));
    }
    req.push_back({(void **)&rt.CT.g[0], u_max * act});
    req.push_back({(void **)&rt.CT.g[1], u_max * act});
    req.push_back({(void **)&rt.CT.dz, u_max * act});
    req.push_back({(void **)&rt.CT.dz2, u_max * act});
    req.push_back({(void **)&rt.CT.logits, u_max * rt.classes_p * 4});
    req.push_back({(void **)&rt.CT.gsum, u_max * act});
    rt.relay_y.clear();
    rt.relay_g.clear();
    for (auto &c : rt.cnn)
      if (c.type == HM_CNN_RES2) {
        rt.relay_y[c.skip] = nullptr;
        rt.relay_g[c.skip] = nullptr;
      }
    for (auto &kv : rt.relay_y) req.push_back({(void **)&kv.second, (int64_t)minibatch * bnd(rt, kv.first + 1)});
    for (auto &kv : rt.relay_g) req.push_back({(void **)&kv.second, (int64_t)minibatch * bnd(rt, kv.first + 1)});
    req.push_back({(void **)&rt.CT.dpool, u_max * cmax * 4});
  } else {
  const int64_t ob = rt.precise ? 4 : 2;  // GEMM operand bytes
  req.push_back({(void **)&T.dy_bf, rows_u * d * 2});
  req.push_back({(void **)&T.dh, rows_u * 4 * d * ob});
  req.push_back({(void **)&T.dh1_bf, rows_u * d * 2});
  req.push_back({(void **)&T.dout, rows_u * d * ob});
  req.push_back({(void **)&T.dqkv, rows_u * 3 * d * ob});
  if (rt.precise) {  // split planes of the largest A / B operand; the fused-epilogue accumulator
    rt.psa_n = 3 * (std::max(rows_u * 4 * d, rows_u * (int64_t)rt.Vp) + 8);
    rt.psb_n = 3 * (std::max({(int64_t)rt.Vp * d, 4 * d * d, rows_u * 4 * d}) + 8);
    rt.pc32_n = rows_u * 4 * d;
    req.push_back({(void **)&rt.psa, rt.psa_n * 2});
    req.push_back({(void **)&rt.psb, rt.psb_n * 2});
    req.push_back({(void **)&rt.pc32, rt.pc32_n * 4});
  }
  req.push_back({(void **)&T.dln, rows_u * d * 4});
  req.push_back({(void **)&T.dh1, rows_u * d * 4});
  req.push_back({(void **)&T.dvec, rows_u * rt.H * 4});
  req.push_back({(void **)&T.dq, rows_u * d * 4});
  req.push_back({(void **)&T.dyh, rows_u * d * 4});
  req.push_back({(void **)&T.g[0], rows_u * d * 4});
  req.push_back({(void **)&T.g[1], rows_u * d * 4});
  req.push_back({(void **)&T.h[0], rows_u * d * 4});
  req.push_back({(void **)&T.h[1], rows_u * d * 4});
  req.push_back({(void **)&T.tmp, rows_u * d * 4});
  req.push_back({(void **)&T.logits, rows_u * rt.Vp * 4});
  }
  (void)rows_mb;
  req.push_back({(void **)&rt.tokens, (int64_t)minibatch * bnd(rt, 0)});
  req.push_back({(void **)&rt.labels, (int64_t)minibatch * labels_per_sample(rt) * 4});
  req.push_back({(void **)&rt.loss_dev, 64 * sizeof(double)});
  req.push_back({(void **)&rt.adam_dev, 256});
  int64_t total = 0;
  for (auto &r : req) total += align_up(r.bytes, 1024);
  if (total > rt.alpha)
    return fail(HM_ERR_CAPACITY, "runtime needs " + std::to_string(total) + " device bytes > alpha " +
                                     std::to_string(rt.alpha));
  if (!rt.slots_sized && !env_nw && !env_nk) {
    int nw = NW, nk = NK;
    int64_t room = rt.alpha - total;
    const int64_t kslot = align_up(pmax * 8, 1024),
                  wslot = align_up(pmax * 4, 1024) + align_up(rt.precise ? 256 : pmax * 2, 1024) +
                          (rt.w_planar ? align_up(std::max<int64_t>(f32max * 2, 256), 1024) : 0);
    while (nk < 4 && room >= kslot) { ++nk; room -= kslot; }
    while (nw < 4 && room >= wslot) { ++nw; room -= wslot; }
    if (nw != NW || nk != NK) {
      rt.slot_nw = nw;
      rt.slot_nk = nk;
      rt.slots_sized = true;
      const int rc = load_plan(rt, plan, rank, minibatch);
      rt.slots_sized = false;
      rt.slot_nw = rt.slot_nk = 0;
      return rc;
    }
  }
  if (rt.pool) {
    cudaFree(rt.pool);
    rt.pool = nullptr;
  }
  HM_CUDA(cudaMalloc(&rt.pool, total));
  rt.pool_bytes = total;
  rt.counters[2] = total;  // device bytes of the loaded plan (readable before any iteration)
  int64_t off = 0;
  for (auto &r : req) {
    *r.ptr = rt.pool + off;
    off += align_up(r.bytes, 1024);
  }
  // cudaMemset runs on the legacy default stream, which does NOT order against
  // the runtime's non-blocking streams: finish it before anything else can
  // touch the pool (otherwise the first iteration's swap-ins race the zeroing)
  HM_CUDA(cudaMemset(rt.pool, 0, total));
  HM_CUDA(cudaDeviceSynchronize());
  rt.out_off.clear();
  for (auto &ob : out_bufs) rt.out_off[ob.first] = reinterpret_cast<uint8_t *>(*ob.second) - rt.pool;
  rt.sig_off = reinterpret_cast<uint8_t *>(rt.sig) - rt.pool;
  // host stash arena
  int64_t sh = 0;
  rt.stash_host_off.clear();
  for (auto &kv : stash_bytes) {
    rt.stash_host_off[kv.first] = sh;
    sh += align_up(kv.second, 4096);
  }
  uint8_t *stash_base = rt.stash_host;
  if (rt.dp_shard) {
    if (sh > rt.stash_priv_bytes) {
      if (rt.stash_priv) cudaFreeHost(rt.stash_priv);
      rt.stash_priv = nullptr;
      HM_CUDA(cudaHostAlloc(&rt.stash_priv, std::max<int64_t>(sh, 4096), cudaHostAllocDefault));
      rt.stash_priv_bytes = sh;
    }
    stash_base = rt.stash_priv;
  } else if (sh > rt.stash_host_bytes) {
    if (rt.shared_arena) return fail(HM_ERR_VALIDATION, "shared stash arena too small: need " + std::to_string(sh));
    if (rt.stash_host) cudaFreeHost(rt.stash_host);
    rt.stash_host = nullptr;
    HM_CUDA(cudaHostAlloc(&rt.stash_host, std::max<int64_t>(sh, 4096), cudaHostAllocDefault));
    rt.stash_host_bytes = sh;
    stash_base = rt.stash_host;
  }

  // ---- actions ----------------------------------------------------------------
  rt.actions.clear();
  rt.dw_off.clear();
  for (auto &e : rt.ar_events) cudaEventDestroy(e);
  rt.ar_events.clear();
  for (auto &e : rt.ev_start) cudaEventDestroy(e);
  for (auto &e : rt.ev_end) cudaEventDestroy(e);
  for (auto &e : rt.ev_tstart) if (e) cudaEventDestroy(e);
  for (auto &e : rt.ev_tend) if (e) cudaEventDestroy(e);
  for (auto &g : rt.graph_exec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  rt.iterations = 0;
  rt.ev_start.assign(plan->items.size(), nullptr);
  rt.ev_end.assign(plan->items.size(), nullptr);
  rt.ev_tstart.assign(plan->items.size(), nullptr);
  rt.ev_tend.assign(plan->items.size(), nullptr);
  rt.ev_live.assign(plan->items.size(), 0);
  for (size_t i = 0; i < plan->items.size(); ++i) {
    if (plan->items[i].rec.gpu != rank) continue;
    HM_CUDA(cudaEventCreate(&rt.ev_start[i]));
    HM_CUDA(cudaEventCreate(&rt.ev_end[i]));
    HM_CUDA(cudaEventCreate(&rt.ev_tstart[i]));
    HM_CUDA(cudaEventCreate(&rt.ev_tend[i]));
  }
  for (auto &t : plan->tasks)
    if (t.dev_id == rank) rt.trt[t.index].members = plan->member_computes[t.index];
  // last-use item of each slot occupant (for reuse gating)
  auto w_release = [&](int ti) -> int {
    TaskInfo &t = plan->tasks[ti];
    if (t.type == HM_TASK_F) return rt.trt[ti].members.back();
    // B task: its U task's W swap-out (or U compute)
    int u = ti + 1;
    int last = rt.trt[u].members.back();
    for (size_t i = 0; i < plan->items.size(); ++i) {
      auto &r = plan->items[i].rec;
      if (r.task == u && !r.is_compute && r.stage == 2 && r.tensor == HM_W) last = (int)i;
    }
    return last;
  };
  auto k_release = [&](int ui) -> int {
    int last = rt.trt[ui].members.back();
    for (size_t i = 0; i < plan->items.size(); ++i) {
      auto &r = plan->items[i].rec;
      if (r.task == ui && !r.is_compute && r.stage == 2 && r.tensor == HM_K) last = (int)i;
    }
    return last;
  };
  std::vector<int> w_prev(NW, -1), dw_prev(NDW, -1), k_prev(NK, -1), st_prev(NST, -1);
  std::map<int, int> w_wait, dw_wait, k_wait, st_wait;  // task -> item to wait (end) before reuse
  // wrap-around: the first occupants wait on the last occupants of the previous iteration
  std::vector<int> order;
  for (int pass = 0; pass < 2; ++pass)
    for (int ti : mine) {
      TaskRt &tr = rt.trt[ti];
      TaskInfo &t = plan->tasks[ti];
      if (t.type != HM_TASK_U) {
        if (w_prev[tr.w_slot] >= 0 && pass == 1) w_wait[ti] = w_release(w_prev[tr.w_slot]);
        w_prev[tr.w_slot] = ti;
        if (t.type == HM_TASK_B) {
          // (bf16 payloads: the U task's W swap-out reads the planes from the dW slot)
          if (dw_prev[tr.dw_slot] >= 0 && pass == 1)
            dw_wait[ti] = rt.w_planar ? w_release(dw_prev[tr.dw_slot]) : rt.trt[dw_prev[tr.dw_slot] + 1].members.back();
          dw_prev[tr.dw_slot] = ti;
          if (tr.stash_slot >= 0) {
            if (st_prev[tr.stash_slot] >= 0 && pass == 1) st_wait[ti] = rt.trt[st_prev[tr.stash_slot]].members.back();
            st_prev[tr.stash_slot] = ti;
          }
        }
      } else {
        if (k_prev[tr.k_slot] >= 0 && pass == 1) k_wait[ti] = k_release(k_prev[tr.k_slot]);
        k_prev[tr.k_slot] = ti;
      }
    }
  int u_ord = 0;  // my U tasks in plan order (the same sequence on every DP rank)
  for (size_t i = 0; i < plan->items.size(); ++i) {
    const hm_item &r = plan->items[i].rec;
    if (r.gpu != rank) continue;
    Action a;
    a.item = (int)i;
    a.task = r.task;
    a.member = r.member;
    for (auto &dp : plan->items[i].deps) {
      if (plan->items[dp.first].rec.gpu == rank) a.waits.push_back(dp);
      else a.rwaits.push_back({dp.first, 0});  // produced on another GPU this iteration
    }
    TaskInfo &t = plan->tasks[r.task];
    TaskRt &tr = rt.trt[r.task];
    if (r.is_compute) {
      if (t.type == HM_TASK_U) {
        if (rt.comm || rt.ipc_reduce) {  // (a 1-rank communicator still runs the collective: the N=1 test of this path)
          // sum the pack's gradient over the data-parallel ranks on the comm
          // stream; overlaps the next backward task on the compute stream
          Action ar;
          ar.kind = 5;
          ar.stream = rt.s_comm;
          ar.task = r.task;
          TaskRt &bt = rt.trt[tr.b_task];
          ar.waits.push_back({bt.members.back(), false});
          ar.dst = rt.slots.dw[bt.dw_slot];
          ar.count = rt.dp_shard ? tr.sh_chunk : tr.params;  // reduce-scatter: per-rank receive count
          ar.pack_lo = t.lo;
          ar.pack_ord = u_ord++;
          rt.dw_off[t.lo] = reinterpret_cast<uint8_t *>(ar.dst) - rt.pool;
          cudaEvent_t e;
          HM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          rt.ar_events.push_back(e);
          ar.done = e;
          a.wait_events.push_back(e);
          rt.actions.push_back(std::move(ar));
        }
        a.kind = 1;
        a.stream = rt.s_update;
      } else {
        a.kind = 0;
        a.stream = rt.s_compute;
        if (r.member == 0 && dw_wait.count(r.task)) a.waits.push_back({dw_wait[r.task], false});
      }
    } else if (r.stage == 0) {
      a.kind = 2;
      a.stream = rt.s_h2d;
      a.bytes = r.nbytes;
      if (r.channel == HM_CPU_GPU_SWAP && r.tensor == HM_W && rt.w_planar) {
        // per layer: hi plane -> the bf16 operand slot; forward: the lo plane of
        // the fp32 prefix -> staging; backward: the whole lo plane -> the dW
        // slot (joined into fp32 W before dW is zeroed)
        const uint8_t *hb = reinterpret_cast<const uint8_t *>(rt.w_host);
        int64_t expect = 0, soff = 0;
        for (int L = t.lo; L <= t.hi; ++L) {
          const int64_t o = rt.w_off[L] - rt.w_off[t.lo], P = rt.lay[L].size, f = rt.lay[L].f32n;
          const uint8_t *hL = hb + 4 * rt.w_off[L];
          a.segs.push_back({reinterpret_cast<uint8_t *>(rt.slots.wsh[tr.w_slot]) + 2 * o, hL, 2 * P});
          if (t.type == HM_TASK_F) {
            if (f) a.segs.push_back({reinterpret_cast<uint8_t *>(rt.slots.wlo[tr.w_slot]) + 2 * soff, hL + 2 * P, 2 * f});
            soff += f;
            expect += 2 * P + 2 * f;
          } else {
            a.segs.push_back({reinterpret_cast<uint8_t *>(rt.slots.dw[tr.dw_slot]) + 4 * o, hL + 2 * P, 2 * P});
            expect += 4 * P;
          }
        }
        if (r.nbytes != expect)
          return fail(HM_ERR_INTERNAL, "bf16-payload W swap-in size disagrees with the plan (load it with w_f bytes)");
        if (w_wait.count(r.task)) a.waits.push_back({w_wait[r.task], false});
        if (t.type == HM_TASK_B && dw_wait.count(r.task)) a.waits.push_back({dw_wait[r.task], false});
      } else if (r.channel == HM_CPU_GPU_SWAP && r.tensor == HM_W) {
        a.src = rt.w_host + rt.w_off[t.lo];
        a.dst = rt.slots.w[tr.w_slot];
        if (r.nbytes != tr.params * 4) return fail(HM_ERR_INTERNAL, "W swap-in size disagrees with the model layout");
        if (w_wait.count(r.task)) a.waits.push_back({w_wait[r.task], false});
      } else if (r.channel == HM_CPU_GPU_SWAP && r.tensor == HM_K) {
        const int64_t off = rt.dp_shard ? tr.sh_off : 0, len = rt.dp_shard ? tr.sh_len : tr.params;
        a.src = rt.k_host + 2 * (rt.w_off[t.lo] + off);
        a.dst = rt.slots.k[tr.k_slot];
        if (r.nbytes != len * 8) return fail(HM_ERR_INTERNAL, "K swap-in size disagrees with the model layout");
        if (k_wait.count(r.task)) a.waits.push_back({k_wait[r.task], false});
      } else if (r.channel == HM_PEER2PEER) {
        // pull the producer's output over NVLink into this task's receive buffer
        a.kind = 6;
        a.stream = rt.s_p2p_in;
        const int64_t per = bnd(rt, r.tensor == HM_X ? r.layer : r.layer + 1);
        const int64_t off = r.peer_member >= 0 ? tr.s0[r.member] * per : 0;
        const int64_t expect = r.peer_member >= 0 ? (int64_t)t.group[r.member] * per : (int64_t)minibatch * per;
        if (r.nbytes != expect) return fail(HM_ERR_INTERNAL, "peer hand-off size disagrees with the activation layout");
        if (!tr.in_buf) return fail(HM_ERR_INTERNAL, "peer hand-off without a receive buffer");
        a.dst = reinterpret_cast<uint8_t *>(tr.in_buf) + off;
        a.peer_rank = plan->tasks[r.peer_task].dev_id;
        a.peer_task = r.peer_task;
        a.peer_off = off;
      } else if (r.channel == HM_MESSAGE_PASSING && r.tensor == HM_SX) {
        if (!rt.stash_host_off.count(r.layer)) return fail(HM_ERR_INTERNAL, "stash-in of an unknown head");
        a.src = stash_base + rt.stash_host_off[r.layer];
        a.dst = rt.slots.stash_in[tr.stash_slot];
        if (r.nbytes != stash_bytes[r.layer]) return fail(HM_ERR_INTERNAL, "stash-in size disagrees with x(L)");
        if (st_wait.count(r.task)) a.waits.push_back({st_wait[r.task], false});
      } else {
        return fail(HM_ERR_VALIDATION, "unsupported input transfer in plan");
      }
    } else {
      a.kind = 3;
      a.stream = rt.s_d2h;
      a.bytes = r.nbytes;
      if (r.channel == HM_CPU_GPU_SWAP && r.tensor == HM_W) {
        TaskRt &bt = rt.trt[tr.b_task];
        // bf16 payloads: the U task left the [hi | lo] planes of each layer in the dW slot
        const int64_t off = rt.dp_shard ? tr.sh_off : 0, len = rt.dp_shard ? tr.sh_len : tr.params;
        a.src = rt.w_planar ? static_cast<const void *>(rt.slots.dw[bt.dw_slot]) : rt.slots.w[bt.w_slot] + off;
        a.dst = rt.w_host + rt.w_off[t.lo] + off;
        if (!rt.w_planar && r.nbytes != len * 4) return fail(HM_ERR_INTERNAL, "W swap-out size disagrees with the model layout");
      } else if (r.channel == HM_CPU_GPU_SWAP && r.tensor == HM_K) {
        const int64_t off = rt.dp_shard ? tr.sh_off : 0, len = rt.dp_shard ? tr.sh_len : tr.params;
        a.src = rt.slots.k[tr.k_slot];
        a.dst = rt.k_host + 2 * (rt.w_off[t.lo] + off);
        if (r.nbytes != len * 8) return fail(HM_ERR_INTERNAL, "K swap-out size disagrees with the model layout");
      } else if (r.channel == HM_MESSAGE_PASSING && r.tensor == HM_SX) {
        const int64_t per = bnd(rt, r.layer);
        const int64_t boff = tr.s0[r.member] * per;
        a.src = rt.stash_dev.at(r.layer) + boff;
        a.dst = stash_base + rt.stash_host_off[r.layer] + boff;
        if (r.nbytes != (int64_t)t.group[r.member] * per) return fail(HM_ERR_INTERNAL, "stash-out size disagrees");
      } else {
        return fail(HM_ERR_VALIDATION, "unsupported output transfer in plan");
      }
    }
    rt.actions.push_back(std::move(a));
  }
  // ---- cross-iteration dependencies (pipelined steps) --------------------------
  // Iteration i+1 may start while iteration i's last swap-outs drain; these
  // waits keep every host / device buffer hand-off across the boundary exact.
  auto overlaps = [&](int t1, int t2) {
    auto &a = plan->tasks[t1];
    auto &b = plan->tasks[t2];
    return a.lo <= b.hi && b.lo <= a.hi;
  };
  std::vector<int> w_out, k_out, sx_in, p2p_in;
  std::map<std::pair<int, int>, int> sx_out;  // (layer, member) -> item (the F task's rank)
  for (size_t i = 0; i < plan->items.size(); ++i) {
    const hm_item &r = plan->items[i].rec;
    if (r.is_compute) continue;
    if (r.stage == 2 && r.tensor == HM_W) w_out.push_back((int)i);
    if (r.stage == 2 && r.tensor == HM_K) k_out.push_back((int)i);
    if (r.stage == 0 && r.tensor == HM_SX) sx_in.push_back((int)i);
    if (r.stage == 2 && r.tensor == HM_SX && r.gpu == rank) sx_out[{r.layer, r.member}] = (int)i;
    if (r.channel == HM_PEER2PEER) p2p_in.push_back((int)i);
  }
  auto xdep = [&](Action &a, int item) {
    if (plan->items[item].rec.gpu == rank) a.xwaits.push_back(item);
    else a.rwaits.push_back({item, 1});
  };
  // host W / K / stash regions: another rank's transfers touch the same bytes
  // only when the arenas are one shared segment (Harmony-PP across processes);
  // Harmony-DP ranks with their own replicas never wait on each other here
  auto xdep_host = [&](Action &a, int item) {
    if (plan->items[item].rec.gpu == rank || rt.shared_arena) xdep(a, item);
  };
  // sharded update: each rank's K shard and its stash are its own regions
  auto xdep_k = [&](Action &a, int item) {
    if (plan->items[item].rec.gpu == rank || !rt.dp_shard) xdep_host(a, item);
  };
  for (auto &a : rt.actions) {
    if (a.item < 0) continue;
    const hm_item &r = plan->items[a.item].rec;
    if (a.kind == 2 && r.tensor == HM_W)  // host W region rewritten by last iteration's swap-out
      for (int o : w_out)
        if (overlaps(plan->items[o].rec.task, r.task)) xdep_host(a, o);
    if (a.kind == 2 && r.tensor == HM_K)
      for (int o : k_out)
        if (overlaps(plan->items[o].rec.task, r.task)) xdep_k(a, o);
    if (a.kind == 3 && r.tensor == HM_SX)  // host stash region still read by last iteration's stash-in
      for (int o : sx_in)
        if (plan->items[o].rec.layer == r.layer) xdep_k(a, o);
    if (a.kind == 0 && plan->tasks[r.task].type == HM_TASK_F)
      for (int L : rt.trt[r.task].stash_heads) {
        auto it = sx_out.find({L, r.member});
        if (it != sx_out.end()) xdep(a, it->second);
      }
    if (a.kind == 0 && rt.trt[r.task].out_buf)  // peers still copying last iteration's output
      for (int o : p2p_in)
        if (plan->items[o].rec.peer_task == r.task) xdep(a, o);
    if (a.kind == 6)  // my receive buffer is read by last iteration's compute of this task
      xdep(a, rt.trt[r.task].members.back());
  }
  rt.counters[7] = 0;  // cross-rank (device-counter) waits per iteration
  for (auto &a : rt.actions) rt.counters[7] += (int64_t)a.rwaits.size();
  // W leaves before K: the next iteration's forward needs W first
  for (size_t i = 0; i + 1 < rt.actions.size(); ++i) {
    Action &x = rt.actions[i], &y = rt.actions[i + 1];
    if (x.kind == 3 && y.kind == 3 && x.task == y.task && x.item >= 0 && y.item >= 0 &&
        plan->items[x.item].rec.tensor == HM_K && plan->items[y.item].rec.tensor == HM_W)
      std::swap(x, y);
  }
  return HM_OK;
}

// Drop the loaded plan and everything derived from it (actions, events,
// captured graphs, peer mappings); the device pool is kept for reuse.
static void unload_plan(hm_runtime &rt) {
  cudaDeviceSynchronize();
  for (auto &g : rt.graph_exec)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  rt.actions.clear();
  rt.trt.clear();
  for (auto &e : rt.ar_events) cudaEventDestroy(e);
  rt.ar_events.clear();
  for (auto *v : {&rt.ev_start, &rt.ev_end, &rt.ev_tstart, &rt.ev_tend})
    for (auto &e : *v)
      if (e) {
        cudaEventDestroy(e);
        e = nullptr;
      }
  rt.ev_start.clear();
  rt.ev_end.clear();
  rt.ev_tstart.clear();
  rt.ev_tend.clear();
  rt.ev_live.clear();
  for (size_t i = 0; i < rt.peer_pool.size(); ++i)
    if (rt.peer_pool[i] && (int)i != rt.rank) cudaIpcCloseMemHandle(rt.peer_pool[i]);
  rt.peer_pool.clear();
  rt.peer_out_off.clear();
  rt.peer_sig_off.clear();
  rt.peer_dw_off.clear();
  rt.ledger.clear();
  rt.trace.clear();
  rt.iterations = 0;
  rt.plan = nullptr;
}

// Harmony-DP gradient sum of one pack over CUDA IPC (hm_runtime_init_ipc_reduce):
//   publish "my gradient is complete" (ready counter of the U task), wait for
//   every peer's, sum all ranks' gradients in rank order into ar_tmp (reads
//   the peers' dW slots through their mapped pools), publish "done reading",
//   wait until every peer has read mine, then overwrite my dW with the sum.
//   Everything is enqueued on the comm stream with device-side waits.
static int ipc_grad_sum(hm_runtime &rt, const Action &a) {
  if (!memops().wait || !memops().write) return fail(HM_ERR_DEVICE, "stream memory operations unavailable");
  if (rt.nranks > 8) return fail(HM_ERR_VALIDATION, "IPC gradient sum: at most 8 ranks");
  // (ready, read) counters of this pack: indexed by its rank among the U
  // tasks, which is the same on every Harmony-DP rank
  const int64_t base = (int64_t)rt.plan->items.size() + 2 * (int64_t)a.pack_ord;
  auto counter = [&](int rank, int64_t idx) -> CUdeviceptr {
    return reinterpret_cast<CUdeviceptr>(rt.peer_pool[rank] + rt.peer_sig_off[rank]) + 4 * (CUdeviceptr)idx;
  };
  const float *src[8] = {nullptr};
  for (int p = 0; p < rt.nranks; ++p) {
    if (p >= (int)rt.peer_pool.size() || !rt.peer_pool[p])
      return fail(HM_ERR_VALIDATION, "IPC gradient sum: rank " + std::to_string(p) + " not imported");
    if (p == rt.rank) {
      src[p] = static_cast<const float *>(a.dst);
      continue;
    }
    auto it = rt.peer_dw_off[p].find(a.pack_lo);
    if (it == rt.peer_dw_off[p].end()) return fail(HM_ERR_INTERNAL, "peer exported no gradient buffer for this pack");
    src[p] = reinterpret_cast<const float *>(rt.peer_pool[p] + it->second);
  }
  const cuuint32_t step = (cuuint32_t)rt.step;
  auto publish = [&](int64_t idx) -> int {
    if (memops().write(a.stream, counter(rt.rank, idx), step, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return fail(HM_ERR_DEVICE, "cuStreamWriteValue32 failed");
    return HM_OK;
  };
  auto await_all = [&](int64_t idx) -> int {
    for (int p = 0; p < rt.nranks; ++p)
      if (p != rt.rank && memops().wait(a.stream, counter(p, idx), step, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(HM_ERR_DEVICE, "cuStreamWaitValue32 failed");
    return HM_OK;
  };
  // sharded update: only this rank's shard of the sum is needed
  int64_t off = 0, len = a.count;
  if (rt.dp_shard) {
    off = rt.trt[a.task].sh_off;
    len = rt.trt[a.task].sh_len;
    for (int p = 0; p < rt.nranks; ++p) src[p] += off;
  }
  HM_TRY(publish(base));
  HM_TRY(await_all(base));
  if (len > 0) HM_TRY(layers::sum_ranks(src, rt.nranks, rt.ar_tmp, len, a.stream));
  HM_TRY(publish(base + 1));
  HM_TRY(await_all(base + 1));
  if (len > 0)
    HM_CUDA(cudaMemcpyAsync(static_cast<float *>(a.dst) + off, rt.ar_tmp, len * 4, cudaMemcpyDeviceToDevice, a.stream));
  return HM_OK;
}

static int join_streams(hm_runtime &rt) {
  cudaStream_t others[] = {rt.s_h2d, rt.s_d2h, rt.s_update, rt.s_comm};
  for (size_t i = 0; i < 4; ++i) {
    HM_CUDA(cudaEventRecord(rt.ev_join[i], others[i]));
    HM_CUDA(cudaStreamWaitEvent(rt.s_compute, rt.ev_join[i], 0));
  }
  return HM_OK;
}

// Enqueue one iteration's body on the runtime's streams.  With `capture`,
// the enqueue is being recorded into a CUDA graph: dependency events stay
// capture-internal, timing events become external event-record nodes, and
// waits on the previous iteration's events are dropped (an iteration only
// starts after the previous one completed).
static int enqueue_body(hm_runtime &rt, bool capture, bool pipelined, int64_t &h2d, int64_t &d2h, int64_t &coll) {
  cudaStream_t sc = rt.s_compute;
  auto rec_time = [&](cudaEvent_t e, cudaStream_t s) -> cudaError_t {
    return capture ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
  };
  HM_CUDA(cudaMemsetAsync(rt.loss_cur, 0, sizeof(double), sc));
  cudaStream_t others[] = {rt.s_h2d, rt.s_d2h, rt.s_update, rt.s_comm};
  if (!pipelined) {
    HM_CUDA(cudaEventRecord(rt.ev_fork, sc));
    for (cudaStream_t o : others) HM_CUDA(cudaStreamWaitEvent(o, rt.ev_fork, 0));
  }
  static const bool serialize = getenv("HM_SERIALIZE") && getenv("HM_SERIALIZE")[0] == '1';
  for (Action &a0 : rt.actions) {
    Action tmp;
    if (serialize) {  // diagnostics: every action on the compute stream, in plan order
      tmp = a0;
      tmp.stream = sc;
    }
    Action &a = serialize ? tmp : a0;
    // waits on the previous iteration: dropped inside a capture (iterations are
    // serialised around graph launches) and when that event's last record
    // happened inside a graph capture (the previous iteration has completed)
    if (!capture)
      for (int x : a.xwaits)
        if (rt.ev_live[x]) HM_CUDA(cudaStreamWaitEvent(a.stream, rt.ev_end[x], 0));
    for (auto &w : a.waits) {
      const bool prev_iter = a.item >= 0 && w.first > a.item;
      if (prev_iter && (capture || !rt.ev_live[w.first])) continue;
      HM_CUDA(cudaStreamWaitEvent(a.stream, w.second ? rt.ev_start[w.first] : rt.ev_end[w.first], 0));
    }
    for (cudaEvent_t e : a.wait_events) HM_CUDA(cudaStreamWaitEvent(a.stream, e, 0));
    for (auto &rw : a.rwaits) {  // produced on another GPU: wait for its device-side counter
      const int64_t want = rt.step - rw.second;
      if (want < 1) continue;
      const int peer = rt.plan->items[rw.first].rec.gpu;
      if (peer >= (int)rt.peer_pool.size() || !rt.peer_pool[peer])
        return fail(HM_ERR_VALIDATION, "peer " + std::to_string(peer) + " not imported (hm_runtime_ipc_import)");
      const CUdeviceptr flag =
          reinterpret_cast<CUdeviceptr>(rt.peer_pool[peer] + rt.peer_sig_off[peer]) + 4 * (CUdeviceptr)rw.first;
      if (!memops().wait) return fail(HM_ERR_DEVICE, "cuStreamWaitValue32 unavailable");
      if (memops().wait(a.stream, flag, (cuuint32_t)want, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(HM_ERR_DEVICE, "cuStreamWaitValue32 failed");
    }
    if (a.kind == 5) {
      if (rt.ipc_reduce) {
        HM_TRY(ipc_grad_sum(rt, a));
      } else if (rt.dp_shard) {  // in place: rank g receives the sum of chunk g
        float *buf = static_cast<float *>(a.dst);
        ncclResult_t nr = nccl().reduce_scatter(buf, buf + (int64_t)rt.rank * a.count, (size_t)a.count, ncclFloat32,
                                                ncclSum, rt.comm, a.stream);
        if (nr != ncclSuccess) return fail(HM_ERR_DEVICE, std::string("ncclReduceScatter: ") + nccl().error_string(nr));
      } else {
        ncclResult_t nr = nccl().all_reduce(a.dst, a.dst, (size_t)a.count, ncclFloat32, ncclSum, rt.comm, a.stream);
        if (nr != ncclSuccess) return fail(HM_ERR_DEVICE, std::string("ncclAllReduce: ") + nccl().error_string(nr));
      }
      HM_CUDA(cudaEventRecord(a.done, a.stream));
      coll += rt.dp_shard ? (rt.nranks - 1) * a.count * 4 : 2 * (rt.nranks - 1) * a.count * 4 / rt.nranks;
      continue;
    }
    HM_CUDA(cudaEventRecord(rt.ev_start[a.item], a.stream));
    if (capture) HM_CUDA(rec_time(rt.ev_tstart[a.item], a.stream));
    switch (a.kind) {
      case 0:
        HM_TRY(run_member(rt, a.task, a.member));
        break;
      case 1: {
        TaskRt &tr = rt.trt[a.task];
        TaskRt &bt = rt.trt[tr.b_task];
        if (rt.dp_shard) {  // this rank's shard only (K slot holds just the shard)
          if (tr.sh_len > 0)
            HM_TRY(adam_launch(rt.slots.w[bt.w_slot] + tr.sh_off, rt.slots.dw[bt.dw_slot] + tr.sh_off,
                               rt.slots.k[tr.k_slot], tr.sh_len, rt.m.lr, rt.m.beta1, rt.m.beta2, rt.m.eps, rt.step,
                               1.0f, a.stream));
        } else if (capture)  // step-dependent scalars read from device memory at replay
          HM_TRY(adam_launch_dev(rt.slots.w[bt.w_slot], rt.slots.dw[bt.dw_slot], rt.slots.k[tr.k_slot], tr.params,
                                 rt.m.beta1, rt.m.beta2, rt.m.eps, rt.adam_dev, 1.0f, a.stream));
        else
          HM_TRY(adam_launch(rt.slots.w[bt.w_slot], rt.slots.dw[bt.dw_slot], rt.slots.k[tr.k_slot], tr.params,
                             rt.m.lr, rt.m.beta1, rt.m.beta2, rt.m.eps, rt.step, 1.0f, a.stream));
        if (rt.w_planar) {  // updated W -> [hi | lo] planes per layer in the (consumed) dW slot, for the swap-out
          const TaskInfo &ut = rt.plan->tasks[a.task];
          for (int L = ut.lo; L <= ut.hi; ++L) {
            const int64_t o = rt.w_off[L] - rt.w_off[ut.lo], P = rt.lay[L].size;
            uint16_t *hi = reinterpret_cast<uint16_t *>(rt.slots.dw[bt.dw_slot] + o);
            HM_TRY(layers::w_split(rt.slots.w[bt.w_slot] + o, hi, hi + P, P, a.stream));
          }
        }
        break;
      }
      case 2:
        if (a.segs.empty()) HM_CUDA(cudaMemcpyAsync(a.dst, a.src, a.bytes, cudaMemcpyHostToDevice, a.stream));
        for (auto &g : a.segs) HM_CUDA(cudaMemcpyAsync(g.dst, g.src, g.bytes, cudaMemcpyHostToDevice, a.stream));
        h2d += a.bytes;
        break;
      case 3:
        HM_CUDA(cudaMemcpyAsync(a.dst, a.src, a.bytes, cudaMemcpyDeviceToHost, a.stream));
        d2h += a.bytes;
        break;
      case 6: {
        if (a.peer_rank >= (int)rt.peer_pool.size() || !rt.peer_pool[a.peer_rank])
          return fail(HM_ERR_VALIDATION, "peer buffer not imported");
        auto it = rt.peer_out_off[a.peer_rank].find(a.peer_task);
        if (it == rt.peer_out_off[a.peer_rank].end()) return fail(HM_ERR_INTERNAL, "peer has no source buffer");
        const uint8_t *src = rt.peer_pool[a.peer_rank] + it->second + a.peer_off;
        HM_CUDA(cudaMemcpyAsync(a.dst, src, a.bytes, cudaMemcpyDeviceToDevice, a.stream));
        rt.p2p_bytes += a.bytes;
        break;
      }
      default:
        return fail(HM_ERR_INTERNAL, "bad action");
    }
    HM_CUDA(cudaEventRecord(rt.ev_end[a.item], a.stream));
    // publish completion of this item for the peers (value = iteration): every
    // item under Harmony-PP, the W swap-outs under the sharded DP update
    if (rt.p2p_mode || (rt.dp_shard && a.kind == 3 && rt.plan->items[a.item].rec.tensor == HM_W)) {
      if (!memops().write) return fail(HM_ERR_DEVICE, "cuStreamWriteValue32 unavailable");
      if (memops().write(a.stream, reinterpret_cast<CUdeviceptr>(rt.sig) + 4 * (CUdeviceptr)a.item,
                         (cuuint32_t)rt.step, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return fail(HM_ERR_DEVICE, "cuStreamWriteValue32 failed");
    }
    if (capture) HM_CUDA(rec_time(rt.ev_tend[a.item], a.stream));
    rt.ev_live[a.item] = capture ? 0 : 1;
  }
  if (!pipelined) HM_TRY(join_streams(rt));
  return HM_OK;
}

static int run_iteration(hm_runtime &rt, const int32_t *tokens, const int32_t *labels, int is_device, double *loss) {
  if (!rt.plan) return fail(HM_ERR_VALIDATION, "no plan loaded");
  HM_CUDA(cudaSetDevice(rt.device));
  const int64_t launches0 = launch_counter().load();
  rt.step += 1;
  cudaStream_t sc = rt.s_compute;
  const int64_t tb = (int64_t)rt.minibatch * bnd(rt, 0);                    // tokens / images
  const int64_t lb = (int64_t)rt.minibatch * labels_per_sample(rt) * 4;  // labels
  rt.loss_cur = rt.loss_dev;
  // Adam bias corrections for this step live in device memory so a captured
  // graph replays correctly: {lr / (1 - b1^t), 1 / sqrt(1 - b2^t)}
  rt.adam_host[0] = (float)(rt.m.lr / (1.0 - std::pow((double)rt.m.beta1, rt.step)));
  rt.adam_host[1] = (float)(1.0 / std::sqrt(1.0 - std::pow((double)rt.m.beta2, rt.step)));
  HM_CUDA(cudaEventRecord(rt.ev_iter0, sc));
  HM_CUDA(cudaMemcpyAsync(rt.adam_dev, rt.adam_host, 2 * sizeof(float), cudaMemcpyHostToDevice, sc));
  HM_CUDA(cudaMemcpyAsync(rt.tokens, tokens, tb, is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, sc));
  HM_CUDA(cudaMemcpyAsync(rt.labels, labels, lb, is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, sc));
  int64_t h2d = 0, d2h = 0, coll = 0;
  const int gi = rt.profiling ? 1 : 0;
  const bool use_graph = rt.use_graph && !rt.p2p_mode && !rt.ipc_reduce && !rt.dp_shard && rt.iterations >= 1;
  if (use_graph) {
    if (!rt.graph_exec[gi]) {
      // record the iteration once (with or without per-kernel timing events)
      if (gi == 1) {  // the timing events recorded here are replayed by graph [1] only
        rt.prof.reset();
        rt.prof.capture = true;
      }
      profiler() = rt.profiling ? &rt.prof : nullptr;
      if (rt.profiling) {
        rt.gemm_shapes.clear();
        gemm::shape_log() = &rt.gemm_shapes;
      }
      const int64_t l0 = launch_counter().load();
      HM_CUDA(cudaStreamBeginCapture(sc, cudaStreamCaptureModeRelaxed));
      int rc = enqueue_body(rt, true, false, h2d, d2h, coll);
      gemm::shape_log() = nullptr;
      cudaGraph_t g = nullptr;
      cudaError_t ce = cudaStreamEndCapture(sc, &g);
      profiler() = nullptr;
      rt.prof.capture = false;
      if (rc != HM_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (ce != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("graph capture: ") + cudaGetErrorString(ce));
      HM_CUDA(cudaGraphInstantiate(&rt.graph_exec[gi], g, 0));
      cudaGraphDestroy(g);
      rt.graph_launches[gi] = launch_counter().load() - l0;
      rt.graph_bytes[gi][0] = h2d;
      rt.graph_bytes[gi][1] = d2h;
      rt.graph_bytes[gi][2] = coll;
      launch_counter().fetch_sub(rt.graph_launches[gi]);  // counted when replayed
    }
    if (gi == 1) HM_CUDA(rt.prof.clear_spans(sc));
    HM_CUDA(cudaGraphLaunch(rt.graph_exec[gi], sc));
    count_launch(rt.graph_launches[gi]);
    h2d = rt.graph_bytes[gi][0];
    d2h = rt.graph_bytes[gi][1];
    coll = rt.graph_bytes[gi][2];
  } else {
    rt.prof.reset();
    if (rt.profiling) HM_CUDA(rt.prof.clear_spans(sc));
    profiler() = rt.profiling ? &rt.prof : nullptr;
    if (rt.profiling) {
      rt.gemm_shapes.clear();
      gemm::shape_log() = &rt.gemm_shapes;
    }
    int rc = enqueue_body(rt, false, false, h2d, d2h, coll);
    gemm::shape_log() = nullptr;
    profiler() = nullptr;
    HM_TRY(rc);
  }
  double loss_sum = 0;
  HM_CUDA(cudaMemcpyAsync(&loss_sum, rt.loss_dev, sizeof(double), cudaMemcpyDeviceToHost, sc));
  HM_CUDA(cudaEventRecord(rt.ev_iter1, sc));
  HM_CUDA(cudaEventSynchronize(rt.ev_iter1));
  rt.iterations += 1;
  if (loss) *loss = loss_sum / (double)rt.global_tokens;
  // measured ledger and trace
  rt.ledger.clear();
  rt.trace.clear();
  for (Action &a : rt.actions) {
    if (a.item < 0) continue;
    hm_item rec = rt.plan->items[a.item].rec;
    float t0 = 0, t1 = 0;
    cudaEvent_t es = use_graph ? rt.ev_tstart[a.item] : rt.ev_start[a.item];
    cudaEvent_t ee = use_graph ? rt.ev_tend[a.item] : rt.ev_end[a.item];
    HM_CUDA(cudaEventElapsedTime(&t0, rt.ev_iter0, es));
    HM_CUDA(cudaEventElapsedTime(&t1, rt.ev_iter0, ee));
    rec.start_ns = (int64_t)((double)t0 * 1e6);
    rec.end_ns = (int64_t)((double)t1 * 1e6);
    rec.duration_ns = rec.end_ns - rec.start_ns;
    (rec.is_compute ? rt.trace : rt.ledger).push_back(rec);
  }
  float it_ms = 0;
  HM_CUDA(cudaEventElapsedTime(&it_ms, rt.ev_iter0, rt.ev_iter1));
  if (rt.profiling) {
    rt.klaunch.clear();
    std::vector<unsigned long long> spans;
    if (rt.prof.spans) {
      spans.resize(std::min(rt.prof.recs.size(), RtProfiler::kSpanCap) * 2);
      HM_CUDA(cudaMemcpy(spans.data(), rt.prof.spans, spans.size() * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost));
    }
    for (size_t i = 0; i < rt.prof.recs.size(); ++i) {
      auto &p = rt.prof.recs[i];
      if (!p.e1) continue;
      float ms = 0;
      HM_CUDA(cudaEventElapsedTime(&ms, p.e0, p.e1));
      double span_ms = 0;  // kernel-only device time (GEMM launches record it)
      if (2 * i + 1 < spans.size() && spans[2 * i] && spans[2 * i + 1])
        span_ms = (double)(spans[2 * i + 1] - ~spans[2 * i]) * 1e-6;
      rt.klaunch.insert(rt.klaunch.end(), {(double)p.cls, p.flops, p.bytes, (double)ms, span_ms});
      rt.kstats[p.cls][0] += ms;
      rt.kstats[p.cls][1] += p.flops;
      rt.kstats[p.cls][2] += p.bytes;
      rt.kstats[p.cls][3] += 1;
    }
  }
  rt.counters[0] = launch_counter().load() - launches0;
  rt.counters[1] = (int64_t)((double)it_ms * 1e6);
  rt.counters[2] = rt.pool_bytes;
  rt.counters[3] = h2d;
  rt.counters[4] = d2h;
  rt.counters[5] = rt.p2p_bytes;
  rt.counters[6] = coll;
  rt.p2p_bytes = 0;
  return HM_OK;
}

// `n` back-to-back iterations with cross-iteration overlap: iteration i+1's
// swap-ins start as soon as the buffers they need are free (e.g. while
// iteration i's last K swap-out drains).  Eager enqueue; one sync at the end.
static int run_steps(hm_runtime &rt, int n, const int32_t *tokens, const int32_t *labels, int is_device,
                     double *losses, int64_t *total_ns) {
  if (!rt.plan) return fail(HM_ERR_VALIDATION, "no plan loaded");
  if (n < 1 || n > 64) return fail(HM_ERR_VALIDATION, "run_steps: 1 <= n <= 64");
  HM_CUDA(cudaSetDevice(rt.device));
  const int64_t launches0 = launch_counter().load();
  cudaStream_t sc = rt.s_compute;
  const int64_t tb = (int64_t)rt.minibatch * bnd(rt, 0);
  const int64_t lb = (int64_t)rt.minibatch * labels_per_sample(rt) * 4;
  int64_t h2d = 0, d2h = 0, coll = 0;
  HM_CUDA(cudaEventRecord(rt.ev_first, sc));
  cudaStream_t others[] = {rt.s_h2d, rt.s_d2h, rt.s_update, rt.s_comm};
  for (cudaStream_t o : others) HM_CUDA(cudaStreamWaitEvent(o, rt.ev_first, 0));
  for (int i = 0; i < n; ++i) {
    rt.step += 1;
    rt.loss_cur = rt.loss_dev + i;
    if (i == n - 1) HM_CUDA(cudaEventRecord(rt.ev_iter0, sc));
    HM_CUDA(cudaMemcpyAsync(rt.tokens, tokens, tb, is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, sc));
    HM_CUDA(cudaMemcpyAsync(rt.labels, labels, lb, is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, sc));
    HM_TRY(enqueue_body(rt, false, true, h2d, d2h, coll));
  }
  HM_TRY(join_streams(rt));
  HM_CUDA(cudaMemcpyAsync(rt.loss_host, rt.loss_dev, n * sizeof(double), cudaMemcpyDeviceToHost, sc));
  HM_CUDA(cudaEventRecord(rt.ev_iter1, sc));
  HM_CUDA(cudaEventSynchronize(rt.ev_iter1));
  rt.iterations += n;
  for (int i = 0; i < n; ++i)
    if (losses) losses[i] = rt.loss_host[i] / (double)rt.global_tokens;
  float ms = 0;
  HM_CUDA(cudaEventElapsedTime(&ms, rt.ev_first, rt.ev_iter1));
  if (total_ns) *total_ns = (int64_t)((double)ms * 1e6);
  // measured ledger / trace of the last iteration (relative to its start)
  rt.ledger.clear();
  rt.trace.clear();
  for (Action &a : rt.actions) {
    if (a.item < 0) continue;
    hm_item rec = rt.plan->items[a.item].rec;
    float t0 = 0, t1 = 0;
    HM_CUDA(cudaEventElapsedTime(&t0, rt.ev_iter0, rt.ev_start[a.item]));
    HM_CUDA(cudaEventElapsedTime(&t1, rt.ev_iter0, rt.ev_end[a.item]));
    rec.start_ns = (int64_t)((double)t0 * 1e6);
    rec.end_ns = (int64_t)((double)t1 * 1e6);
    rec.duration_ns = rec.end_ns - rec.start_ns;
    (rec.is_compute ? rt.trace : rt.ledger).push_back(rec);
  }
  float it_ms = 0;
  HM_CUDA(cudaEventElapsedTime(&it_ms, rt.ev_iter0, rt.ev_iter1));
  rt.counters[0] = launch_counter().load() - launches0;
  rt.counters[1] = (int64_t)((double)it_ms * 1e6);
  rt.counters[2] = rt.pool_bytes;
  rt.counters[3] = h2d;
  rt.counters[4] = d2h;
  rt.counters[5] = rt.p2p_bytes / n;
  rt.counters[6] = coll;
  rt.p2p_bytes = 0;
  return HM_OK;
}

}  // namespace hm

namespace hm {
// NUMA node of the GPU's PCIe function (sysfs), -1 if unknown
static int gpu_numa_node(int device) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
  std::string b(bus);
  for (auto &c : b) c = (char)tolower(c);
  std::vector<std::string> names = {b};
  const size_t colon = b.find(':');
  if (colon == 8) names.push_back(b.substr(4));  // 8-digit PCI domain -> sysfs' 4 digits
  for (auto &n : names) {
    FILE *f = fopen(("/sys/bus/pci/devices/" + n + "/numa_node").c_str(), "r");
    if (!f) continue;
    int node = -1;
    if (fscanf(f, "%d", &node) != 1) node = -1;
    fclose(f);
    return node;
  }
  return -1;
}

// Pinned host arena of `bytes`: an anonymous mapping with a preferred-node
// memory policy (pages are faulted in by the pinning, on that node), huge
// pages advised, registered with CUDA.  Zero-filled.
static void *numa_pinned_alloc(int64_t bytes, int node) {
  void *p = mmap(nullptr, (size_t)bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return nullptr;
  madvise(p, (size_t)bytes, MADV_HUGEPAGE);
  if (node >= 0 && node < 1024) {
    unsigned long mask[16] = {0};
    mask[node / 64] = 1UL << (node % 64);
    const int kMpolPreferred = 1;
    syscall(SYS_mbind, p, (unsigned long)bytes, kMpolPreferred, mask, 1024UL, 0U);  // best effort
  }
  if (cudaHostRegister(p, (size_t)bytes, cudaHostRegisterPortable) != cudaSuccess) {
    munmap(p, (size_t)bytes);
    return nullptr;
  }
  return p;
}
static void numa_pinned_free(void *p, int64_t bytes) {
  if (!p) return;
  cudaHostUnregister(p);
  munmap(p, (size_t)bytes);
}

// streams, events and the pinned W / K arenas (shared by both model families)
static hm_runtime *finish_create(std::unique_ptr<hm_runtime> rt, int32_t *status) {
  auto bad = [&](int code, const std::string &msg) -> hm_runtime * {
    hm::set_last_error(msg);
    if (status) *status = code;
    return nullptr;
  };
  cudaStream_t *ss[] = {&rt->s_compute, &rt->s_h2d,     &rt->s_d2h,    &rt->s_update,
                        &rt->s_p2p_in,  &rt->s_p2p_out, &rt->s_comm};
  for (auto p : ss)
    if (cudaStreamCreateWithFlags(p, cudaStreamNonBlocking) != cudaSuccess) return bad(HM_ERR_DEVICE, "stream create");
  cudaEventCreate(&rt->ev_iter0);
  cudaEventCreate(&rt->ev_iter1);
  cudaEventCreateWithFlags(&rt->ev_fork, cudaEventDisableTiming);
  for (auto &e : rt->ev_join) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (cudaHostAlloc(&rt->adam_host, 64, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(&rt->loss_host, 64 * sizeof(double), cudaHostAllocDefault) != cudaSuccess)
    return bad(HM_ERR_DEVICE, "pinned alloc");
  cudaEventCreate(&rt->ev_first);
  rt->numa_node = gpu_numa_node(rt->device);
  rt->w_map_bytes = align_up(std::max<int64_t>(rt->total_params * 4, 4096), 1 << 21);
  rt->k_map_bytes = align_up(std::max<int64_t>(rt->total_params * 8, 4096), 1 << 21);
  rt->w_host = static_cast<float *>(numa_pinned_alloc(rt->w_map_bytes, rt->numa_node));
  rt->k_host = static_cast<float *>(numa_pinned_alloc(rt->k_map_bytes, rt->numa_node));  // zero: Adam state at step 0
  if (!rt->w_host || !rt->k_host) {
    numa_pinned_free(rt->w_host, rt->w_map_bytes);
    numa_pinned_free(rt->k_host, rt->k_map_bytes);
    rt->w_host = rt->k_host = nullptr;
    return bad(HM_ERR_DEVICE, "pinned host arena allocation failed (" + std::to_string(rt->total_params * 12) + " B)");
  }
  if (status) *status = HM_OK;
  return rt.release();
}
}  // namespace hm

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

hm_runtime *hm_runtime_create(int32_t device, const hm_model *model, int64_t alpha_bytes, int32_t *status) {
  auto bad = [&](int code, const std::string &msg) -> hm_runtime * {
    hm::set_last_error(msg);
    if (status) *status = code;
    return nullptr;
  };
  if (!model) return bad(HM_ERR_VALIDATION, "null model");
  if (model->d_model % model->n_head) return bad(HM_ERR_VALIDATION, "d_model % n_head != 0");
  const int dh = model->d_model / model->n_head;
  if (dh != 64 && dh != 128) return bad(HM_ERR_VALIDATION, "head_dim must be 64 or 128");
  if (model->seq_len % 64 || model->d_model % 64) return bad(HM_ERR_VALIDATION, "seq_len and d_model must be multiples of 64");
  if (model->vocab_padded % 8 || model->vocab_padded < model->vocab) return bad(HM_ERR_VALIDATION, "bad padded vocab");
  if (model->math_mode != 0 && model->math_mode != 1)
    return bad(HM_ERR_VALIDATION, "math_mode: 0 = bf16 operands, 1 = fp32 operands (parity mode)");
  if (cudaSetDevice(device) != cudaSuccess) return bad(HM_ERR_DEVICE, "cudaSetDevice failed");
  auto rt = std::make_unique<hm_runtime>();
  rt->device = device;
  rt->m = *model;
  rt->alpha = alpha_bytes;
  rt->R = model->n_layer;
  rt->S = model->seq_len;
  rt->H = model->n_head;
  rt->DH = dh;
  rt->V = model->vocab;
  rt->Vp = model->vocab_padded;
  rt->precise = model->math_mode == 1;
  rt->w_off.assign(rt->R + 1, 0);
  for (int L = 0; L < rt->R; ++L) {
    rt->lay.push_back(hm::make_layout(*rt, L));
    rt->w_off[L + 1] = rt->w_off[L] + rt->lay.back().size;
  }
  rt->total_params = rt->w_off[rt->R];
  return hm::finish_create(std::move(rt), status);
}

hm_runtime *hm_runtime_create_cnn(int32_t device, const hm_cnn_model *model, int64_t alpha_bytes, int32_t *status) {
  auto bad = [&](int code, const std::string &msg) -> hm_runtime * {
    hm::set_last_error(msg);
    if (status) *status = code;
    return nullptr;
  };
  if (!model || !model->layers || model->n_layer < 1) return bad(HM_ERR_VALIDATION, "null or empty CNN model");
  const int R = model->n_layer;
  if (model->classes < 1 || model->classes_padded % 64 || model->classes_padded < model->classes)
    return bad(HM_ERR_VALIDATION, "classes_padded must be a multiple of 64 and >= classes");
  for (int L = 0; L < R; ++L) {
    const hm_cnn_layer &c = model->layers[L];
    const std::string at = "CNN layer " + std::to_string(L) + ": ";
    if ((c.type == HM_CNN_HEAD) != (L == R - 1)) return bad(HM_ERR_VALIDATION, at + "the head must be the last layer");
    if (c.type < HM_CNN_CONV || c.type > HM_CNN_RES2) return bad(HM_ERR_VALIDATION, at + "unknown type");
    if (c.h < 1 || c.w < 1 || c.cin % 64 || c.cin < 64 || (c.type != HM_CNN_HEAD && (c.cout % 64 || c.cout < 64)))
      return bad(HM_ERR_VALIDATION, at + "channels must be positive multiples of 64");
    if (c.type == HM_CNN_DOWN && (c.h % 2 || c.w % 2)) return bad(HM_ERR_VALIDATION, at + "pooling needs even h, w");
    if ((c.type == HM_CNN_RES || c.type == HM_CNN_RES2) && c.cin != c.cout)
      return bad(HM_ERR_VALIDATION, at + "residual blocks keep the width");
    if ((c.type == HM_CNN_RES2) != (c.skip >= 0)) return bad(HM_ERR_VALIDATION, at + "only res2 layers have a skip");
    if (c.type == HM_CNN_RES2) {
      if (c.skip >= L - 1) return bad(HM_ERR_VALIDATION, at + "the skip source must precede the block");
      const hm_cnn_layer &sc = model->layers[c.skip];
      const int sh = sc.type == HM_CNN_DOWN ? sc.h / 2 : sc.h, sw = sc.type == HM_CNN_DOWN ? sc.w / 2 : sc.w;
      if (sc.type == HM_CNN_HEAD || sc.cout != c.cout || sh != c.h || sw != c.w)
        return bad(HM_ERR_VALIDATION, at + "skip source shape differs from the block output");
    }
    if (L + 1 < R) {
      const hm_cnn_layer &n = model->layers[L + 1];
      const int oh = c.type == HM_CNN_DOWN ? c.h / 2 : c.h, ow = c.type == HM_CNN_DOWN ? c.w / 2 : c.w;
      if (n.cin != c.cout || n.h != oh || n.w != ow)
        return bad(HM_ERR_VALIDATION, at + "output shape does not match the next layer's input");
    }
  }
  if (cudaSetDevice(device) != cudaSuccess) return bad(HM_ERR_DEVICE, "cudaSetDevice failed");
  auto rt = std::make_unique<hm_runtime>();
  rt->device = device;
  rt->family = HM_FAMILY_CNN;
  rt->m.n_layer = R;
  rt->m.lr = model->lr;
  rt->m.beta1 = model->beta1;
  rt->m.beta2 = model->beta2;
  rt->m.eps = model->eps;
  rt->alpha = alpha_bytes;
  rt->R = R;
  rt->S = 1;
  rt->classes = model->classes;
  rt->classes_p = model->classes_padded;
  rt->cnn.assign(model->layers, model->layers + R);
  rt->w_off.assign(R + 1, 0);
  for (int L = 0; L < R; ++L) {
    rt->cnn_lay.push_back(hm::cnn_layout(*rt, L));
    rt->w_off[L + 1] = rt->w_off[L] + rt->cnn_lay.back().size;
  }
  rt->total_params = rt->w_off[R];
  return hm::finish_create(std::move(rt), status);
}



void *hm_runtime_arena(hm_runtime *rt, int32_t kind, int64_t *bytes) {
  if (!rt) return nullptr;
  if (kind == HM_ARENA_W) {
    if (bytes) *bytes = rt->total_params * 4;
    return rt->w_host;
  }
  if (kind == HM_ARENA_K) {
    if (bytes) *bytes = rt->total_params * 8;
    return rt->k_host;
  }
  if (bytes) *bytes = rt->stash_host_bytes;
  return rt->stash_host;
}

int hm_runtime_layer_offsets(const hm_runtime *rt, int64_t *w_off, int32_t cap) {
  if (!rt || cap < rt->R + 1) return hm::fail(HM_ERR_VALIDATION, "layer offsets buffer too small");
  for (int i = 0; i <= rt->R; ++i) w_off[i] = rt->w_off[i];
  return rt->R + 1;
}

int hm_runtime_load_plan(hm_runtime *rt, hm_plan *plan, int32_t rank, int32_t minibatch) {
  if (!rt || !plan) return hm::fail(HM_ERR_VALIDATION, "null argument");
  if (cudaSetDevice(rt->device) != cudaSuccess) return hm::fail(HM_ERR_DEVICE, "cudaSetDevice");
  if (minibatch < 1) return hm::fail(HM_ERR_VALIDATION, "minibatch must be >= 1");
  // global tokens = minibatch of the whole job: sum over ranks' F groups of task 0 of each rank
  int64_t global = 0;
  std::map<int, int64_t> per_rank;
  for (auto &t : plan->p->tasks)
    if (t.type == HM_TASK_F && (t.lo == 0)) {
      int64_t s = 0;
      for (int u : t.group) s += u;
      per_rank[t.dev_id] += s;
    }
  for (auto &kv : per_rank) global += kv.second;
  // The previous plan's device state does not survive a (re)load: any failure
  // below leaves the runtime with NO plan (run calls then fail with "no plan
  // loaded"), never with a half-built one that points at freed buffers.  Peer
  // pool mappings are dropped too: the pool is reallocated, so every rank
  // must export / import again after loading.
  hm::unload_plan(*rt);
  rt->global_tokens = global * hm::labels_per_sample(*rt);
  const int rc = hm::load_plan(*rt, plan->p, rank, minibatch);
  if (rc != HM_OK) hm::unload_plan(*rt);
  return rc;
}

int hm_runtime_run_iteration(hm_runtime *rt, const int32_t *tokens, const int32_t *labels, int32_t is_device,
                             double *loss_out) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  return hm::run_iteration(*rt, tokens, labels, is_device, loss_out);
}

int hm_runtime_run_steps(hm_runtime *rt, int32_t n, const int32_t *tokens, const int32_t *labels, int32_t is_device,
                         double *losses, int64_t *total_ns) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  return hm::run_steps(*rt, n, tokens, labels, is_device, losses, total_ns);
}

int32_t hm_runtime_ledger_count(const hm_runtime *rt) { return rt ? (int32_t)rt->ledger.size() : 0; }
int hm_runtime_ledger(const hm_runtime *rt, hm_item *out, int32_t cap) {
  if (!rt || cap < (int32_t)rt->ledger.size()) return hm::fail(HM_ERR_VALIDATION, "ledger buffer too small");
  std::copy(rt->ledger.begin(), rt->ledger.end(), out);
  return (int)rt->ledger.size();
}
int32_t hm_runtime_trace_count(const hm_runtime *rt) { return rt ? (int32_t)rt->trace.size() : 0; }
int hm_runtime_trace(const hm_runtime *rt, hm_item *out, int32_t cap) {
  if (!rt || cap < (int32_t)rt->trace.size()) return hm::fail(HM_ERR_VALIDATION, "trace buffer too small");
  std::copy(rt->trace.begin(), rt->trace.end(), out);
  return (int)rt->trace.size();
}
int hm_runtime_counters(const hm_runtime *rt, int64_t *out, int32_t cap) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  const int n = cap < 8 ? cap : 8;
  for (int i = 0; i < n; ++i) out[i] = rt->counters[i];
  return n;
}

int hm_runtime_debug_read(const hm_runtime *rt, int32_t which, int64_t offset, int64_t bytes, void *host) {
  if (!rt || !host || offset < 0 || bytes < 0) return hm::fail(HM_ERR_VALIDATION, "debug_read: bad arguments");
  const uint8_t *base = which == 0 ? rt->shared_store : which == 1 ? rt->work_store : nullptr;
  if (!base) return hm::fail(HM_ERR_VALIDATION, "debug_read: which = 0 (shared store) | 1 (work store)");
  HM_CUDA(cudaDeviceSynchronize());
  HM_CUDA(cudaMemcpy(host, base + offset, bytes, cudaMemcpyDeviceToHost));
  return HM_OK;
}

int hm_nccl_unique_id(const char *nccl_path, uint8_t *out) {
  std::string err;
  if (!hm::nccl().load(nccl_path, err)) return hm::fail(HM_ERR_DEVICE, err);
  ncclUniqueId id;
  ncclResult_t r = hm::nccl().get_unique_id(&id);
  if (r != ncclSuccess) return hm::fail(HM_ERR_DEVICE, std::string("ncclGetUniqueId: ") + hm::nccl().error_string(r));
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return HM_OK;
}

int hm_runtime_init_comm(hm_runtime *rt, const char *nccl_path, const uint8_t *id, int32_t nranks, int32_t rank) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  std::string err;
  if (!hm::nccl().load(nccl_path, err)) return hm::fail(HM_ERR_DEVICE, err);
  if (cudaSetDevice(rt->device) != cudaSuccess) return hm::fail(HM_ERR_DEVICE, "cudaSetDevice");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclResult_t r = hm::nccl().comm_init_rank(&rt->comm, nranks, uid, rank);
  if (r != ncclSuccess) return hm::fail(HM_ERR_DEVICE, std::string("ncclCommInitRank: ") + hm::nccl().error_string(r));
  rt->nranks = nranks;
  return HM_OK;
}

int hm_runtime_init_ipc_reduce(hm_runtime *rt, int32_t nranks, int32_t rank) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  if (rt->comm) return hm::fail(HM_ERR_VALIDATION, "an NCCL communicator is already attached");
  if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks)
    return hm::fail(HM_ERR_VALIDATION, "IPC gradient sum: 1 <= nranks <= 8, 0 <= rank < nranks");
  if (rt->plan) return hm::fail(HM_ERR_VALIDATION, "call before hm_runtime_load_plan");
  rt->ipc_reduce = true;
  rt->nranks = nranks;
  return HM_OK;
}

int hm_runtime_share_arenas(hm_runtime *rt, const char *shm_name, int32_t create, int64_t stash_bytes) {
  if (!rt || !shm_name || !*shm_name) return hm::fail(HM_ERR_VALIDATION, "shared arena needs a name");
  if (rt->shared_arena) return hm::fail(HM_ERR_VALIDATION, "arenas already shared");
  const int64_t wb = hm::align_up(rt->total_params * 4, 1 << 21), kb = hm::align_up(rt->total_params * 8, 1 << 21);
  const int64_t sb = hm::align_up(std::max<int64_t>(stash_bytes, 4096), 1 << 21);
  const int64_t total = wb + kb + sb;
  std::string name = shm_name[0] == '/' ? shm_name : std::string("/") + shm_name;
  int fd = shm_open(name.c_str(), O_RDWR | (create ? O_CREAT | O_EXCL : 0), 0600);
  if (fd < 0) return hm::fail(HM_ERR_DEVICE, "shm_open(" + name + ") failed");
  if (create && ftruncate(fd, total) != 0) {
    close(fd);
    shm_unlink(name.c_str());
    return hm::fail(HM_ERR_DEVICE, "ftruncate of the shared arena failed");
  }
  void *p = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return hm::fail(HM_ERR_DEVICE, "mmap of the shared arena failed");
  if (cudaHostRegister(p, total, cudaHostRegisterPortable) != cudaSuccess) {
    munmap(p, total);
    return hm::fail(HM_ERR_DEVICE, "cudaHostRegister of the shared arena failed");
  }
  hm::numa_pinned_free(rt->w_host, rt->w_map_bytes);
  hm::numa_pinned_free(rt->k_host, rt->k_map_bytes);
  rt->w_host = rt->k_host = nullptr;
  if (rt->stash_host) cudaFreeHost(rt->stash_host);
  uint8_t *base = static_cast<uint8_t *>(p);
  rt->w_host = reinterpret_cast<float *>(base);
  rt->k_host = reinterpret_cast<float *>(base + wb);
  rt->stash_host = base + wb + kb;
  rt->stash_host_bytes = sb;
  rt->shared_arena = true;
  rt->shared_owner = create != 0;
  rt->shm_name = name;
  rt->shm_ptr = p;
  rt->shm_bytes = total;
  return HM_OK;
}

int hm_runtime_ipc_export(hm_runtime *rt, uint8_t *buf, int32_t cap) {
  if (!rt || !rt->pool) return hm::fail(HM_ERR_VALIDATION, "load a plan before exporting");
  std::vector<uint8_t> out;
  auto put = [&](const void *p, size_t n) {
    const uint8_t *b = static_cast<const uint8_t *>(p);
    out.insert(out.end(), b, b + n);
  };
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, rt->pool) != cudaSuccess) return hm::fail(HM_ERR_DEVICE, "cudaIpcGetMemHandle failed");
  const uint32_t magic = 0x484d3250;  // "HM2P"
  const int32_t rank = rt->rank, n = (int32_t)rt->out_off.size();
  put(&magic, 4);
  put(&rank, 4);
  put(&h, sizeof(h));
  put(&rt->sig_off, 8);
  put(&n, 4);
  for (auto &kv : rt->out_off) {
    const int32_t task = kv.first;
    put(&task, 4);
    put(&kv.second, 8);
  }
  const int32_t m = (int32_t)rt->dw_off.size();  // gradient buffers read by the IPC gradient sum
  put(&m, 4);
  for (auto &kv : rt->dw_off) {
    const int32_t task = kv.first;
    put(&task, 4);
    put(&kv.second, 8);
  }
  if ((int32_t)out.size() > cap) return hm::fail(HM_ERR_VALIDATION, "ipc buffer too small");
  std::memcpy(buf, out.data(), out.size());
  return (int)out.size();
}

int hm_runtime_ipc_import(hm_runtime *rt, const uint8_t *buf, int32_t len) {
  if (!rt || !buf || len < 0) return hm::fail(HM_ERR_VALIDATION, "bad ipc blob");
  if (!rt->plan) return hm::fail(HM_ERR_VALIDATION, "load a plan before importing peers");
  size_t o = 0;
  bool ok = true;
  auto get = [&](void *p, size_t n) {  // bounds-checked read of the blob
    if (!ok || o + n > (size_t)len) {
      ok = false;
      return;
    }
    std::memcpy(p, buf + o, n);
    o += n;
  };
  uint32_t magic = 0;
  int32_t peer = -1, n = -1;
  cudaIpcMemHandle_t h;
  int64_t sig_off = -1;
  get(&magic, 4);
  if (!ok || magic != 0x484d3250) return hm::fail(HM_ERR_VALIDATION, "bad ipc blob magic");
  get(&peer, 4);
  get(&h, sizeof(h));
  get(&sig_off, 8);
  get(&n, 4);
  if (!ok) return hm::fail(HM_ERR_VALIDATION, "truncated ipc blob header");
  if (peer < 0 || peer > 4096) return hm::fail(HM_ERR_VALIDATION, "bad peer rank");
  if (n < 0 || (size_t)n * 12 + 4 > (size_t)len - o) return hm::fail(HM_ERR_VALIDATION, "ipc blob length disagrees with its entry count");
  std::map<int, int64_t> offs, dwo;
  for (int i = 0; i < n; ++i) {
    int32_t task;
    int64_t off;
    get(&task, 4);
    get(&off, 8);
    if (!ok || off < 0) return hm::fail(HM_ERR_VALIDATION, "bad ipc blob entry");
    offs[task] = off;
  }
  int32_t m = -1;
  get(&m, 4);
  if (!ok || m < 0 || (size_t)m * 12 != (size_t)len - o) return hm::fail(HM_ERR_VALIDATION, "ipc blob length disagrees with its gradient entry count");
  for (int i = 0; i < m; ++i) {
    int32_t task;
    int64_t off;
    get(&task, 4);
    get(&off, 8);
    if (!ok || off < 0) return hm::fail(HM_ERR_VALIDATION, "bad ipc blob gradient entry");
    dwo[task] = off;
  }
  if (sig_off < 0) return hm::fail(HM_ERR_VALIDATION, "bad ipc blob signal offset");
  if ((int)rt->peer_pool.size() <= peer) {
    rt->peer_pool.resize(peer + 1, nullptr);
    rt->peer_out_off.resize(peer + 1);
    rt->peer_sig_off.resize(peer + 1, 0);
    rt->peer_dw_off.resize(peer + 1);
  }
  rt->peer_dw_off[peer] = std::move(dwo);
  if (peer == rt->rank) {
    rt->peer_out_off[peer] = std::move(offs);
    rt->peer_sig_off[peer] = sig_off;
    rt->peer_pool[peer] = rt->pool;
    return HM_OK;
  }
  if (cudaSetDevice(rt->device) != cudaSuccess) return hm::fail(HM_ERR_DEVICE, "cudaSetDevice");
  if (rt->peer_pool[peer]) {  // re-import: close the previous mapping first
    cudaIpcCloseMemHandle(rt->peer_pool[peer]);
    rt->peer_pool[peer] = nullptr;
  }
  void *p = nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return hm::fail(HM_ERR_DEVICE, "cudaIpcOpenMemHandle failed for rank " + std::to_string(peer));
  rt->peer_out_off[peer] = std::move(offs);
  rt->peer_sig_off[peer] = sig_off;
  rt->peer_pool[peer] = static_cast<uint8_t *>(p);
  return HM_OK;
}

int hm_runtime_get_step(const hm_runtime *rt) { return rt ? rt->step : -1; }

int hm_runtime_numa_node(const hm_runtime *rt) { return rt ? rt->numa_node : -1; }

int hm_runtime_set_w_payload(hm_runtime *rt, int32_t mode) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  if (mode != 0 && mode != 1) return hm::fail(HM_ERR_VALIDATION, "w payload: 0 = fp32 (reference), 1 = bf16 planes");
  if (rt->plan) return hm::fail(HM_ERR_VALIDATION, "set the W payload before loading a plan");
  if (mode == 1 && rt->family != HM_FAMILY_GPT)
    return hm::fail(HM_ERR_VALIDATION, "bf16 W payloads are implemented for the transformer family");
  if (mode == 1 && rt->precise)
    return hm::fail(HM_ERR_VALIDATION, "bf16 W payloads feed bf16 GEMM operands: not with math_mode 1 (fp32 operands)");
  rt->w_planar = mode == 1;
  return HM_OK;
}

int hm_runtime_set_step(hm_runtime *rt, int32_t step) {
  if (!rt || step < 0) return hm::fail(HM_ERR_VALIDATION, "bad step");
  rt->step = step;
  return HM_OK;
}

int hm_runtime_set_graph(hm_runtime *rt, int32_t enable) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  rt->use_graph = enable != 0;
  return HM_OK;
}

int hm_runtime_set_profiling(hm_runtime *rt, int32_t enable) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  rt->profiling = enable != 0;
  for (auto &row : rt->kstats)
    for (double &v : row) v = 0;
  return HM_OK;
}

int hm_runtime_kernel_stats(const hm_runtime *rt, double *out, int32_t cap) {
  if (!rt || cap < hm::KC_COUNT * 4) return hm::fail(HM_ERR_VALIDATION, "kernel stats buffer too small");
  for (int c = 0; c < hm::KC_COUNT; ++c)
    for (int j = 0; j < 4; ++j) out[c * 4 + j] = rt->kstats[c][j];
  return hm::KC_COUNT;
}

int hm_runtime_kernel_launches(const hm_runtime *rt, double *out, int32_t cap) {
  int n = (int)(rt->klaunch.size() / 5);
  if (out)
    for (int i = 0; i < n && i < cap; ++i)
      for (int j = 0; j < 5; ++j) out[5 * i + j] = rt->klaunch[5 * i + j];
  return n;
}

int hm_runtime_gemm_shapes(const hm_runtime *rt, int64_t *out, int32_t cap) {
  if (!rt) return hm::fail(HM_ERR_VALIDATION, "null runtime");
  const int n = (int)(rt->gemm_shapes.size() / 7);
  if (out)
    for (int i = 0; i < n && i < cap; ++i)
      for (int j = 0; j < 7; ++j) out[7 * i + j] = rt->gemm_shapes[7 * i + j];
  return n;
}

void hm_runtime_free(hm_runtime *rt) {
  if (!rt) return;
  cudaSetDevice(rt->device);
  cudaDeviceSynchronize();
  for (auto &e : rt->ev_start) if (e) cudaEventDestroy(e);
  for (auto &e : rt->ev_end) if (e) cudaEventDestroy(e);
  for (auto &e : rt->ev_tstart) if (e) cudaEventDestroy(e);
  for (auto &e : rt->ev_tend) if (e) cudaEventDestroy(e);
  for (auto &g : rt->graph_exec) if (g) cudaGraphExecDestroy(g);
  if (rt->ev_fork) cudaEventDestroy(rt->ev_fork);
  for (auto &e : rt->ev_join) if (e) cudaEventDestroy(e);
  if (rt->adam_host) cudaFreeHost(rt->adam_host);
  if (rt->loss_host) cudaFreeHost(rt->loss_host);
  if (rt->ev_first) cudaEventDestroy(rt->ev_first);
  if (rt->ev_iter0) cudaEventDestroy(rt->ev_iter0);
  if (rt->ev_iter1) cudaEventDestroy(rt->ev_iter1);
  for (auto &e : rt->ar_events) cudaEventDestroy(e);
  if (rt->comm) hm::nccl().comm_destroy(rt->comm);
  if (rt->pool) cudaFree(rt->pool);
  for (size_t i = 0; i < rt->peer_pool.size(); ++i)
    if (rt->peer_pool[i] && (int)i != rt->rank) cudaIpcCloseMemHandle(rt->peer_pool[i]);
  if (rt->shared_arena) {
    cudaHostUnregister(rt->shm_ptr);
    munmap(rt->shm_ptr, rt->shm_bytes);
    if (rt->shared_owner) shm_unlink(rt->shm_name.c_str());
  } else {
    hm::numa_pinned_free(rt->w_host, rt->w_map_bytes);
    hm::numa_pinned_free(rt->k_host, rt->k_map_bytes);
    if (rt->stash_host) cudaFreeHost(rt->stash_host);
  }
  if (rt->stash_priv) cudaFreeHost(rt->stash_priv);
  cudaStream_t ss[] = {rt->s_compute, rt->s_h2d, rt->s_d2h, rt->s_update, rt->s_p2p_in, rt->s_p2p_out, rt->s_comm};
  for (auto s : ss) if (s) cudaStreamDestroy(s);
  delete rt;
}

}  // extern "C"
