/*
 * harmony_b200.h -- C ABI of libharmony_b200.so, the B200-native runtime of
 * Harmony's swap-aware layer-pack training (arXiv 2202.01306).
 *
 * The reference (`wrapsched`, pure Python) has no FFI; its boundary is three
 * Python calls.  Each entry point below names the reference interface it
 * replaces (paths relative to /root/reference/pkg/src/wrapsched/):
 *
 *   hm_plan_*      <- simulator._build_items / simulator._run / simulate
 *                     (simulator.py:150-336, 347-375, 378-434): the swap plan,
 *                     the per-task swap-byte ledger and the event-driven
 *                     estimate, built from the lowered task graph of
 *                     taskgraph.generate_task_graph (taskgraph.py:211-236).
 *   hm_runtime_*   <- no reference code: the runtime the paper describes in
 *                     PAPER.md:572-586 and the reference only models.  Its
 *                     ledger equals hm_plan's by construction (it executes it).
 *   hm_k_*         <- no reference code: the sm_100a kernels of F/B/U tasks,
 *                     exported individually so they are testable alone.
 *
 * Conventions: plain C types only, sizes in bytes (int64), times in ns.
 * Every function returns an int status (HM_OK = 0, negative = error) unless
 * documented otherwise; the message of the last error on the calling thread
 * is available from hm_last_error().  Status codes map onto the reference's
 * exception classes (errors.py:4-73) in paper_2202_01306_b200/errors.py.
 */
#ifndef HARMONY_B200_H
#define HARMONY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define HM_OK 0
#define HM_ERR_VALIDATION (-1)      /* ValidationError                       */
#define HM_ERR_CAPACITY (-2)        /* CapacityViolationError (alpha)        */
#define HM_ERR_DEADLOCK (-3)        /* DeadlockError                         */
#define HM_ERR_DEVICE (-4)          /* CUDA / NCCL failure (WrapschedError)  */
#define HM_ERR_MISSING_PROFILE (-5) /* MissingProfileError                   */
#define HM_ERR_INTERNAL (-6)        /* invariant violation                   */
#define HM_ERR_PROFILE_RANGE (-7)   /* ProfileRangeError                     */
#define HM_ERR_LAYER_TOO_LARGE (-8) /* LayerTooLargeError (packing)          */
#define HM_ERR_UNPACKABLE (-9)      /* UnpackableError (packing)             */

/* ---- enums shared with the Python lowering (taskgraph.py:61-71, core.py:44-54) */
enum hm_tensor { HM_X = 0, HM_Y = 1, HM_DX = 2, HM_DY = 3, HM_W = 4, HM_DW = 5, HM_K = 6, HM_SX = 7 };
enum hm_channel { HM_CPU_GPU_SWAP = 0, HM_PEER2PEER = 1, HM_MESSAGE_PASSING = 2, HM_SHARED_MEMORY = 3 };
enum hm_task_type { HM_TASK_F = 0, HM_TASK_B = 1, HM_TASK_U = 2 };
enum hm_device_kind { HM_DEV_GPU = 0, HM_DEV_CPU = 1 };
/* Resources of the estimator (simulator.py:3-10): id = kind * gpu_count + gpu,
 * the two host root links use gpu = 0. */
enum hm_resource_kind {
  HM_RES_COMPUTE = 0, HM_RES_SWAP_IN = 1, HM_RES_SWAP_OUT = 2, HM_RES_P2P_IN = 3,
  HM_RES_P2P_OUT = 4, HM_RES_UPDATE = 5, HM_RES_ROOT_OUT = 6, HM_RES_ROOT_IN = 7
};

/* ---- lowered task graph (one flat table; taskgraph.py:91-106) ------------ */
typedef struct {
  int32_t tensor;    /* hm_tensor                                          */
  int32_t layer;     /* dict key of Task.inputs/outputs[tensor]            */
  int32_t channel;   /* hm_channel                                         */
  int32_t peer_task; /* Channel.src_task (inputs) / dst_task (outputs), -1  */
  int32_t src_layer; /* Channel.src_layer (relay payload), -1 if none       */
} hm_entry;

typedef struct {
  int32_t index, type, lo, hi, dev_kind, dev_id, recompute;
  int32_t group_off, group_len; /* slice of the groups[] array            */
  int32_t in_off, in_len;       /* slice of entries[], insertion order     */
  int32_t out_off, out_len;
} hm_task;

typedef struct {
  int32_t gpu_count;
  int32_t cpu_offload_update;
  int64_t pcie_bandwidth;      /* bytes/s per direction per GPU link     */
  int64_t root_link_bandwidth; /* shared host uplink                     */
  int64_t p2p_bandwidth;       /* 0 = pcie_bandwidth (reference model)   */
  int64_t update_cpu_rate;
  const int32_t *p2p_group_of; /* [gpu_count] switch-group id per GPU    */
  /* Harmony-DP fast mode (not the reference ledger): the U
   * task on GPU g updates only shard g of its pack -- parameters
   * [g*c, min(P, (g+1)*c)) with c = 64*ceil(P / (64 N)) -- so its K-in,
   * K-out and W-out rows carry that shard (8, 8 and 4 bytes per parameter)
   * and its update time scales by the shard's share.  The gradient is
   * reduce-scattered instead of all-reduced; W and K live in ONE host arena
   * all ranks share.  0 = the reference (every rank updates a replica). */
  int32_t dp_sharded_update;
} hm_machine;

/* Integer profile tables, row-major [layer][u] with u = 0..u_top (u = 0 is
 * unused).  -1 = no model (MissingProfileError if touched), -2 = above the
 * fitted u_max (ProfileRangeError if touched).  t_u is indexed [layer][1]. */
typedef struct {
  int32_t layers, u_top;
  const int64_t *x, *y;      /* [layers*(u_top+1)] */
  const int64_t *w, *dw, *k; /* [layers]           */
  const int64_t *t_f, *t_b, *t_u; /* [layers*(u_top+1)] or NULL if no times */
  const int64_t *w_f;             /* [layers] W bytes a FORWARD task moves (bf16
                                     swap-payload mode), or NULL = w (reference) */
} hm_profile;

/* One work item of the plan (simulator.py:86-108 `_Item`, extended with the
 * addressing fields the runtime needs: layer, peer task, peer member). */
typedef struct {
  int32_t task, stage, member, seq; /* key (task, stage 0 in/1 compute/2 out, member, seq) */
  int32_t is_compute;
  int32_t tensor, channel;          /* -1 for compute items                 */
  int32_t gpu;                      /* device index of the owning task      */
  int32_t layer;                    /* stash/p2p layer key, -1 otherwise    */
  int32_t peer_task, peer_member;   /* producer (inputs) or consumer (MP out) */
  int32_t n_res, res[4];            /* resource ids (hm_resource_kind*N+gpu) */
  int64_t nbytes;
  int64_t duration_ns;
  int64_t start_ns, end_ns;         /* filled by hm_plan_simulate           */
} hm_item;

typedef struct hm_plan hm_plan;

/* Build the swap plan of a lowered graph (restates simulator._build_items). */
hm_plan *hm_plan_build(const hm_task *tasks, int32_t n_tasks, const int32_t *groups,
                       const hm_entry *entries, const hm_machine *machine,
                       const hm_profile *profile, int32_t *status);
/* Layer-pack decomposition of layers [0, count) (paper Algorithm 2;
 * replaces packing.balanced_time_pack / greedy_maxpack_baseline,
 * pkg/src/wrapsched/packing.py:67-186).  mode 0 = balanced time, 1 = greedy.
 * time / mem: per-layer pass time (ns) and memory (bytes) at the microbatch;
 * ckpt: per-layer bytes a FORWARD pack adds for its checkpointed input
 * (x(first, u)), NULL for backward packs.  Out: the first layer of each pack
 * (in/out *n_packs = capacity / count).  HM_ERR_LAYER_TOO_LARGE sets
 * *bad_layer; HM_ERR_UNPACKABLE when no pack count fits alpha. */
int hm_pack_layers(int32_t mode, int32_t count, const int64_t *time, const int64_t *mem, const int64_t *ckpt,
                   int64_t alpha, int32_t *first_layer, int32_t *n_packs, int32_t *bad_layer);
/* Run the FIFO event loop (simulator._run); returns status, fills start/end. */
int hm_plan_simulate(hm_plan *plan, int64_t *makespan_ns);
int32_t hm_plan_item_count(const hm_plan *plan);
int hm_plan_items(const hm_plan *plan, hm_item *out, int32_t cap);
/* Dependency edges (dep item -> item; at_start = dep's start gates item). */
int32_t hm_plan_edge_count(const hm_plan *plan);
int hm_plan_edges(const hm_plan *plan, int32_t *dep, int32_t *item, int32_t *at_start, int32_t cap);
void hm_plan_free(hm_plan *plan);

const char *hm_last_error(void);
const char *hm_version(void);
/* Kernels launched by this library so far (all streams, all threads). */
int64_t hm_launch_count(void);

/* ---- runtime -------------------------------------------
 * One runtime per process and GPU (torchrun launches one process per GPU).
 * It owns: pinned host arenas (W, K, stash), one device pool capped at alpha,
 * the streams compute / swap_in / swap_out / p2p_in / p2p_out / update, and
 * the sm_100a kernels.  hm_runtime_run_iteration executes every item of the
 * loaded plan that belongs to this rank's GPU and records the ledger. */
typedef struct {
  int32_t n_layer;    /* R: chain layers (embedding fused into 0, head into R-1) */
  int32_t d_model, n_head, seq_len, vocab, vocab_padded;
  int32_t causal;     /* 1 = GPT, 0 = BERT-style full attention             */
  int32_t math_mode;  /* 0 = bf16 tensor-core operands, fp32 accumulate (throughput
                       *     mode; tolerance stated separately);
                       * 1 = fp32 operands (parity mode): every activation kept in
                       *     fp32, GEMMs as three-plane bf16 split products on the
                       *     same tcgen05 kernel (fp32-level accuracy), fp32 SIMT
                       *     attention / LayerNorm forward / cross-entropy       */
  double lr, beta1, beta2, eps; /* double: 1-beta computed exactly as torch does */
} hm_model;

typedef struct hm_runtime hm_runtime;

/* Deep-CNN layer chain (BASELINE config c5, VGG / ResNet-style packs).  Each
 * chain layer is one of: 0 conv (3x3 conv + bias + ReLU), 1 down (conv + ReLU,
 * then 2x2 average pool), 2 res (basic residual block relu(x + conv(relu(conv
 * x)))), 3 head (global average pool + fully connected + cross-entropy).
 * h, w, cin = the layer's input; activations NHWC bf16; channels % 64 == 0
 * (the image enters layer 0 zero-padded to 64 channels); one label per sample. */
enum { HM_FAMILY_GPT = 0, HM_FAMILY_CNN = 1 };
enum { HM_CNN_CONV = 0, HM_CNN_DOWN = 1, HM_CNN_RES = 2, HM_CNN_HEAD = 3, HM_CNN_RES2 = 4 };
/* type 4 res2: relu(conv(x) + bias + skip) with skip = the output of layer
 * `skip` (a residual block at convolution granularity; the skip edge may cross
 * pack boundaries and travels through device-resident relay stores). */
typedef struct {
  int32_t type, cin, cout, h, w;
  int32_t skip; /* res2: source layer of the skip input; -1 otherwise */
} hm_cnn_layer;
typedef struct {
  int32_t n_layer;
  const hm_cnn_layer *layers;
  int32_t classes, classes_padded;
  double lr, beta1, beta2, eps;
} hm_cnn_model;

enum hm_arena { HM_ARENA_W = 0, HM_ARENA_K = 1, HM_ARENA_STASH = 2 };

hm_runtime *hm_runtime_create(int32_t device, const hm_model *model, int64_t alpha_bytes,
                              int32_t *status);
/* Pinned host arena owned by the runtime; returns its host pointer. */
hm_runtime *hm_runtime_create_cnn(int32_t device, const hm_cnn_model *model, int64_t alpha_bytes,
                                  int32_t *status);
void *hm_runtime_arena(hm_runtime *rt, int32_t kind, int64_t *bytes);
/* Per-layer parameter offsets (in floats) of the W arena; K uses 2x. */
int hm_runtime_layer_offsets(const hm_runtime *rt, int64_t *w_off, int32_t cap);
int hm_runtime_load_plan(hm_runtime *rt, hm_plan *plan, int32_t rank, int32_t minibatch);
/* tokens/labels: [minibatch, seq_len] int32, host (pinned or pageable) or
 * device pointers (is_device = 1).  loss_out: mean token cross-entropy. */
int hm_runtime_run_iteration(hm_runtime *rt, const int32_t *tokens, const int32_t *labels,
                             int32_t is_device, double *loss_out);
/* n (1..64) back-to-back iterations on the same batch with cross-iteration
 * overlap (iteration i+1's swap-ins start while iteration i's last swap-outs
 * drain; every buffer hand-off across the boundary is event-ordered).
 * losses[n] per iteration; total_ns = device time of all n iterations. */
int hm_runtime_run_steps(hm_runtime *rt, int32_t n, const int32_t *tokens, const int32_t *labels,
                         int32_t is_device, double *losses, int64_t *total_ns);
int32_t hm_runtime_ledger_count(const hm_runtime *rt);
/* Executed transfer rows of the last iteration, in execution order; the
 * start/end fields hold measured CUDA-event times relative to iteration start. */
int hm_runtime_ledger(const hm_runtime *rt, hm_item *out, int32_t cap);
/* Measured compute items (same hm_item layout) of the last iteration. */
int32_t hm_runtime_trace_count(const hm_runtime *rt);
int hm_runtime_trace(const hm_runtime *rt, hm_item *out, int32_t cap);
/* Counters of the last iteration: [0] kernels launched, [1] iteration ns,
 * [2] device bytes in use (peak), [3] H2D bytes, [4] D2H bytes, [5] P2P bytes,
 * [6] NCCL all-reduce bytes per GPU (ring volume 2(N-1)/N x |dW|). */
int hm_runtime_counters(const hm_runtime *rt, int64_t *out, int32_t cap);
/* Diagnostics: copy `bytes` at `offset` of the shared-pack activation store
 * (which = 0) or the recompute work store (1) to host memory (synchronous). */
int hm_runtime_debug_read(const hm_runtime *rt, int32_t which, int64_t offset, int64_t bytes, void *host);
/* Harmony-DP: NCCL (dlopen'ed from nccl_path, NULL = default search) unique
 * id on one rank (128 bytes), then every rank joins the communicator.  With
 * nranks > 1, hm_runtime_load_plan inserts one all-reduce (sum) of each
 * pack's gradient buffer between its B task and its U task, on a comm stream
 * that overlaps the next B task. */
int hm_nccl_unique_id(const char *nccl_path, uint8_t *out);
int hm_runtime_init_comm(hm_runtime *rt, const char *nccl_path, const uint8_t *id, int32_t nranks,
                         int32_t rank);
/* Harmony-DP with several processes on ONE GPU (tests; NCCL cannot put two
 * ranks on one device): the per-pack gradient sum runs over CUDA IPC instead
 * of NCCL -- every rank sums all ranks' gradient buffers in rank order (the
 * same bits everywhere), ordered by device-side counters.  Call before
 * load_plan; after it, every rank exports / imports its IPC blob as for PP. */
int hm_runtime_init_ipc_reduce(hm_runtime *rt, int32_t nranks, int32_t rank);
/* Harmony-PP across processes (one per GPU): W, K and stash arenas live in
 * one POSIX shared-memory segment registered as pinned memory in every rank
 * (rank 0 creates it, then the others attach).  Call before load_plan. */
int hm_runtime_share_arenas(hm_runtime *rt, const char *shm_name, int32_t create, int64_t stash_bytes);
/* After load_plan: export this rank's device pool (CUDA IPC handle), the
 * offsets of its peer-visible source buffers and of its per-item completion
 * counters; every rank imports every peer's blob.  Cross-GPU hand-offs are
 * then pulled with cudaMemcpyAsync over NVLink and ordered by device-side
 * waits on the producer's counters (cuStreamWaitValue32). */
int hm_runtime_ipc_export(hm_runtime *rt, uint8_t *buf, int32_t cap);
int hm_runtime_ipc_import(hm_runtime *rt, const uint8_t *buf, int32_t len);
/* Optimizer step counter (Adam bias correction); checkpoint / resume of the
 * host arenas restores it together with W and K. */
int hm_runtime_get_step(const hm_runtime *rt);
/* NUMA node the W / K host arenas were placed on (the GPU's, from sysfs;
 * -1 = unknown, default policy). */
int hm_runtime_numa_node(const hm_runtime *rt);
int hm_runtime_set_step(hm_runtime *rt, int32_t step);
/* W swap payload, before hm_runtime_load_plan: 0 = fp32 (the reference's
 * ledger), 1 = bf16 planes (SURVEY 8f4b fast mode: the host W arena holds each
 * layer as [bf16 hi plane | 16-bit lo plane]; forward tasks move the hi plane
 * plus the lo plane of the fp32-read prefix; the plan must be built with
 * hm_profile.w_f).  Transformer family only. */
int hm_runtime_set_w_payload(hm_runtime *rt, int32_t mode);
/* Record each iteration into a CUDA graph after the first (default on) and
 * replay it: one launch per iteration instead of thousands. */
int hm_runtime_set_graph(hm_runtime *rt, int32_t enable);
/* Per-launch CUDA-event timing of the runtime's kernels (resets the stats). */
int hm_runtime_set_profiling(hm_runtime *rt, int32_t enable);
/* Accumulated stats since profiling was enabled, 7 classes x {ms, flops,
 * bytes, launches}: 0 GEMM, 1 attention fwd, 2 attention bwd, 3 LayerNorm,
 * 4 cross-entropy, 5 Adam, 6 other (cast, embedding, bias grad). */
int hm_runtime_kernel_stats(const hm_runtime *rt, double *out, int32_t cap);
/* Per-launch records of the last profiled iteration, {class, flops, bytes,
 * event ms, device-clock ms} each (the device-clock span -- first CTA start
 * to last CTA end on %globaltimer -- is recorded by GEMM launches only);
 * returns the number of launches (copies at most cap). */
int hm_runtime_kernel_launches(const hm_runtime *rt, double *out, int32_t cap);
/* GEMM calls of the last profiled iteration, 7 fields each {m, n, k, a_major,
 * b_major, epilogue, has_bias}, in launch order; returns the count. */
int hm_runtime_gemm_shapes(const hm_runtime *rt, int64_t *out, int32_t cap);
void hm_runtime_free(hm_runtime *rt);

/* ---- kernels, testable alone (raw device pointers, a cudaStream_t) -------- */
/* Fused Adam over one pack: W, m, v updated in place from g; K holds (m, v)
 * interleaved per parameter.  step >= 1.  Reads 16 B/param, writes 12 B/param. */
int hm_k_adam(float *w, const float *g, float *k, int64_t n, double lr, double beta1,
              double beta2, double eps, int32_t step, float grad_scale, void *stream);
/* C[M,N] (+)= A . B^T with bf16 operands, fp32 accumulate (tcgen05 + TMEM + TMA).
 * a_major/b_major: 0 = K-major (reduction dim contiguous), 1 = MN-major.
 * epilogue: see hm_gemm_epilogue. */
enum hm_gemm_epilogue {
  HM_EPI_STORE_BF16 = 0,      /* D = acc (+bias) -> bf16                     */
  HM_EPI_STORE_F32 = 1,       /* D = acc (+bias) -> fp32                     */
  HM_EPI_ACC_F32 = 2,         /* D += acc (fp32, TMA reduce-add; split-K ok)  */
  HM_EPI_RESID_F32 = 3,       /* D = R + acc + bias -> fp32 (R may alias D)  */
  HM_EPI_GELU_BF16 = 4,       /* P = acc + bias (bf16), D = gelu(P) (bf16)   */
  HM_EPI_DGELU_BF16 = 5,      /* D = acc * gelu'(P) -> bf16                  */
  HM_EPI_RELU_BF16 = 6,       /* D = relu(acc + bias) -> bf16                */
  HM_EPI_RESID_RELU_BF16 = 7, /* D = relu(acc + bias + R), R bf16 -> bf16    */
  HM_EPI_DRELU_BF16 = 8,      /* D = acc * (P > 0), P bf16 -> bf16           */
  HM_EPI_ADD_BF16 = 9         /* D = acc + R, R bf16 -> bf16                 */
};
int hm_k_gemm(const void *a, const void *b, void *d, int64_t m, int64_t n, int64_t k,
              int64_t lda, int64_t ldb, int64_t ldd, int32_t a_major, int32_t b_major,
              int32_t epilogue, const float *bias, const void *aux, int64_t ld_aux,
              int32_t batch, int64_t stride_a, int64_t stride_b, int64_t stride_d,
              void *stream);

/* 3x3 convolution, stride 1, zero padding 1, NHWC bf16 activations, weights
 * W[Cout][3][3][Cin] bf16 (= [Cout, 9*Cin], K-major), as implicit GEMM on
 * tcgen05: the activation operand is gathered by TMA im2col loads (one
 * 64-channel slice of one filter tap per k-block), never materialised.
 * Cin and Cout must be multiples of 64.
 *   fwd:   y[N*H*W, Cout]  = im2col(x) . W^T            (epilogue: any bf16 one)
 *   dgrad: dx[N*H*W, Cin]  = im2col(dy) . flip(W)       (epilogue: STORE/DRELU/ADD bf16)
 *   wgrad: dw[Cout, 9*Cin] += dy^T . im2col(x)          (fp32 TMA reduce-add, split-K) */
int hm_k_conv_fwd(const void *x, const void *w, void *y, int32_t n, int32_t h, int32_t wd, int32_t cin,
                  int32_t cout, int32_t epilogue, const float *bias, const void *aux, void *stream);
int hm_k_conv_dgrad(const void *dy, const void *w, void *dx, int32_t n, int32_t h, int32_t wd, int32_t cin,
                    int32_t cout, int32_t epilogue, const void *aux, void *stream);
int hm_k_conv_wgrad(const void *dy, const void *x, float *dw, int32_t n, int32_t h, int32_t wd, int32_t cin,
                    int32_t cout, void *stream);

/* Deep-CNN layer pieces (NHWC bf16): dz = dy * (y > 0); 2x2 average pool
 * and its backward fused with the producing conv's ReLU mask; global average
 * pool [nb, P, c] -> [nb, c] and its backward (fp32 gradient in). */
int hm_k_relu_bwd(const void *dy, const void *y, void *dz, int64_t n, void *stream);
int hm_k_pool2_fwd(const void *a, void *y, int32_t n, int32_t h, int32_t w, int32_t c, void *stream);
int hm_k_pool2_relu_bwd(const void *dy, const void *a, void *dz, int32_t n, int32_t h, int32_t w, int32_t c,
                        void *stream);
int hm_k_gap_fwd(const void *x, void *pooled, int32_t nb, int32_t P, int32_t c, void *stream);
int hm_k_gap_bwd(const float *dp, void *dx, int32_t nb, int32_t P, int32_t c, void *stream);
/* out = a + b (bf16, n % 8 == 0): the skip gradient joining the trunk gradient */
int hm_k_add_bf16(const void *a, const void *b, void *out, int64_t n, void *stream);

/* Tile configuration the GEMM picks for an (m, n, k, epilogue, B major) problem:
 * bn = output tile width (128 | 192 | 256; 192 single-CTA only), cta_pair = 1 (128-row tile on one SM) or
 * 2 (256-row tile on a CTA pair, tcgen05.mma.cta_group::2), splits = split-K
 * factor (ACC_F32 only; partial sums meet in a TMA reduce-add), 0 = stream-K
 * (ACC_F32 only: each persistent CTA pair runs an equal share of the
 * tiles x k-blocks sequence, tiles cut between CTAs summed by the same reduce-add). */
int hm_k_gemm_tile(int64_t m, int64_t n, int64_t k, int32_t epilogue, int32_t b_major, int32_t *bn,
                   int32_t *cta_pair, int32_t *splits);
/* Force a tile configuration for every later GEMM of the process (0 = auto;
 * splits = -1 forces stream-K for ACC_F32); for tests and tuning (same as
 * HM_GEMM_BN / HM_GEMM_CG / HM_GEMM_SPLITK). */
int hm_k_gemm_set_tile(int32_t bn, int32_t cta_pair, int32_t splits);
/* The GEMM's own per-launch time (us) for one shape {m, n, k, a_major,
 * b_major, epilogue, has_bias}: a CUDA graph of `reps` back-to-back launches
 * on rotating random operand sets (inputs not L2-resident), timed with CUDA
 * events around whole graph replays. */
int hm_k_gemm_replay(const int64_t *shape, int32_t reps, void *stream, double *us_per_launch);

/* Fused attention over qkv [batch*seq, 3*heads*head_dim] bf16 (q|k|v thirds).
 * out [batch*seq, heads*head_dim] bf16; lse [batch*seq, heads] fp32 (log2).
 * head_dim 64 or 128; seq multiple of 64; causal 1 = GPT mask. */
int hm_k_attn_fwd(const void *qkv, void *out, float *lse, int32_t batch, int32_t seq, int32_t heads,
                  int32_t head_dim, int32_t causal, void *stream);
/* Same forward on tcgen05 tensor cores (head_dim 64 or 128, seq % 128 == 0);
 * hm_k_attn_fwd / hm_k_attn_bwd and the runtime use it whenever the shape
 * allows. */
int hm_k_attn_fwd_tc(const void *qkv, void *out, float *lse, int32_t batch, int32_t seq, int32_t heads,
                     int32_t head_dim, int32_t causal, void *stream);
/* Backward: writes dq|dk|dv into dqkv (same layout as qkv).  Scratch:
 * dvec [batch*seq*heads] fp32, dq_acc [batch*seq, heads*head_dim] fp32. */
int hm_k_attn_bwd(const void *qkv, const void *out, const void *dout, const float *lse, float *dvec,
                  float *dq_acc, void *dqkv, int32_t batch, int32_t seq, int32_t heads, int32_t head_dim,
                  int32_t causal, void *stream);
/* fp32 -> bf16 cast of n elements. */
int hm_k_cast_bf16(const float *src, void *dst, int64_t n, void *stream);
/* Weight planes (bf16 swap payloads): hi = bf16 nearest with ties toward zero
 * (the runtime's bf16 GEMM operand of a weight in both payload modes), lo = the
 * low 16 bits; join(hi, lo) restores the fp32 bits exactly. */
int hm_k_cast_w_bf16(const float *src, void *dst, int64_t n, void *stream);
int hm_k_w_split(const float *w, void *hi, void *lo, int64_t n, void *stream);
int hm_k_w_join(const void *hi, const void *lo, float *w, int64_t n, void *stream);
/* Token + position embedding: out[b*seq+p] = wte[tokens[b*seq+p]] + wpe[p] (fp32). */
int hm_k_embed_fwd(const int32_t *tokens, const float *wte, const float *wpe, float *out, int32_t batch,
                   int32_t seq, int32_t d, void *stream);
/* dwte[tokens[r]] += dx[r]; dwpe[p] += sum_b dx[b*seq+p]. */
int hm_k_embed_bwd(const int32_t *tokens, const float *dx, float *dwte, float *dwpe, int32_t batch,
                   int32_t seq, int32_t d, void *stream);
/* y = bf16(LN(x) * g + b), eps 1e-5; mean/rstd [rows] saved for backward. */
int hm_k_layernorm_fwd(const float *x, const float *g, const float *b, void *y, float *mean, float *rstd,
                       int64_t rows, int32_t d, void *stream);
/* out = LN_bwd(dy) + resid (resid may be NULL or alias out); optional bf16
 * copy of out; dg += sum dy*xhat, db += sum dy. */
int hm_k_layernorm_bwd(const float *dy, const float *x, const float *mean, const float *rstd,
                       const float *g, const float *resid, float *out, void *out_bf16, float *dg,
                       float *db, int64_t rows, int32_t d, void *stream);
/* Softmax cross-entropy over vocab columns [0, vocab) of fp32 logits with row
 * pitch ld; dlogits (bf16, same pitch) = (softmax - onehot) * scale, padding
 * columns zeroed; loss_sum (fp64) += sum of per-row CE. */
int hm_k_cross_entropy(const float *logits, const int32_t *labels, int64_t rows, int64_t ld,
                       int32_t vocab, void *dlogits, double *loss_sum, float scale, void *stream);
/* db[n] += sum_r dy[r, n] (dy bf16 if is_bf16 else fp32, row pitch ld). */
int hm_k_bias_grad(const void *dy, int32_t is_bf16, float *db, int64_t rows, int32_t n, int64_t ld,
                   void *stream);

/* ---- fp32-operand parity mode (math_mode 1; kernels/precise.cu) ----------- */
/* C = A . B^T with fp32 operands: each split into three bf16 planes
 * (x = x0 + x1 + x2) in scratch_a / scratch_b (>= 3 x the operand's
 * elements, rounded up to 8, each), the six plane products with i + j <= 2
 * summed in fp32 by the tcgen05 GEMM.  Arguments as hm_k_gemm (batch 1);
 * the bf16 epilogues write fp32; RESID / GELU / DGELU go through acc
 * (>= m x n fp32 elements) and an elementwise pass (exact tanh GELU). */
int hm_k_gemm_precise(const float *a, const float *b, void *d, int64_t m, int64_t n, int64_t k,
                      int64_t lda, int64_t ldb, int64_t ldd, int32_t a_major, int32_t b_major,
                      int32_t epilogue, const float *bias, void *aux, int64_t ld_aux, void *scratch_a,
                      int64_t scratch_a_elems, void *scratch_b, int64_t scratch_b_elems, float *acc,
                      int64_t acc_elems, void *stream);
/* fp32 attention (layouts as hm_k_attn_fwd; lse is the natural log here). */
int hm_k_attn_fwd_f32(const float *qkv, float *out, float *lse, int32_t batch, int32_t seq, int32_t heads,
                      int32_t head_dim, int32_t causal, void *stream);
int hm_k_attn_bwd_f32(const float *qkv, const float *out, const float *dout, const float *lse, float *dvec,
                      float *dqkv, int32_t batch, int32_t seq, int32_t heads, int32_t head_dim,
                      int32_t causal, void *stream);
/* LayerNorm forward with fp32 output; cross-entropy with fp32 dlogits. */
int hm_k_layernorm_fwd_f32(const float *x, const float *g, const float *b, float *y, float *mean,
                           float *rstd, int64_t rows, int32_t d, void *stream);
int hm_k_cross_entropy_f32(const float *logits, const int32_t *labels, int64_t rows, int64_t ld,
                           int32_t vocab, float *dlogits, double *loss_sum, float scale, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HARMONY_B200_H */
