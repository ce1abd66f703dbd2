// attention_fwd64.cu -- flash-attention forward for head_dim 64 (GPT-2 XL,
// BERT-Large) on the 5th-gen tensor cores, built around the two limits the
// head_dim-64 shape hits first: the MUFU exp2 rate (16384 ex2 per 128 x 128
// tile against 512 cycles of MMA) and the softmax's wait on the tensor pipe.
//
// Persistent: one CTA per SM walks (sample-head, query-tile pair) items,
// causal pairs heaviest first, dealt in snake order; every ring / buffer
// parity follows running counters across items, the next item's Q pair is
// double-buffered, and its first S MMAs are issued while the current item's
// last tiles are still in the softmax (16 x 1024 x 25 heads: 114.6 vs 138.6 us
// for one CTA per pair).
//   warp 0      TMA: Q pairs, then K_j / V_j into a 4-stage ring
//   warp 1      PV MMA issuer, warp 2 S MMA issuer
//   warps 4-7   softmax of tile 0, warps 8-11 of tile 1 (one thread per
//               query row = TMEM lane)
// TMEM (512 columns): three rotating 128-column S buffers + O_0, O_1 (64
// columns each).  S buffers are handed out in the order the S tiles are
// computed (S_0(0), S_1(0), S_0(1), S_1(1), ...), so S for the next step of
// a tile is computed while its softmax still works on the current one: the
// MMA warp issues PV(n) and then S(n + 3) into the buffer PV(n) has just
// consumed (tcgen05.mma executes in issue order).  The softmax therefore
// never waits for its own PV + S round trip, only for the tensor pipe's
// throughput.
//
// Softmax per tile: the whole S row (128 fp32) is read with four
// tcgen05.ld.x32 and one wait, masked on the causal
// diagonal (the softmax warpgroups raise their register budget to 216 with
// setmaxnreg, the TMA / MMA warpgroup drops to 72: three warps share each
// SMSP's 16K registers), reduced with 3-input max, exponentiated with packed f32x2 FMA /
// add (half the FP32 issue slots) and ex2.approx, and written back as bf16
// pairs into the S buffer's own columns, where the PV MMA reads it as its A
// operand straight from TMEM.  O stays in TMEM; it is rescaled in place only
// when a row max grows by more than 2^8 (lazy rescale, exact in O / l).
//
// Measured balance (HM_ATTN_TRACE clock64 trace, tools/probes/attn_mma_probe):
// a position (one tile's 128 x 128 block) holds 542 cycles of MMAs (PV 8 x
// 128x64x16 from TMEM: 366; S 4 x 128x128x16: 256), but tcgen05.mma issue
// blocks at the execution rate, a try_wait on an already completed mbarrier
// costs ~150 cycles while the SS MMAs saturate shared memory and a commit
// ~45, so one issuing thread left the pipe idle for its own waits (~1300
// cycles per position).  Hence two issuing threads (PV / S) on two SM
// sub-partitions, descriptors as precomputed 32-bit words, one K-block wait
// per step and counters without divisions.  The softmax then bounds it: 128
// ex2 + 64 bf16x2 conversions per row on the XU pipe with both tiles' warps on
// each SMSP; one exponent pair in eight goes to the FMA pipe (ex2_poly2).
// O leaves each tile as one TMA store from SW128 staging, and the kernel is
// launched with programmatic dependent launch (set-up overlaps the previous
// kernel's tail).
//
// Output conventions as attention.cu: o [tokens, d] bf16, lse [tokens, H]
// in the log2 domain.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "../runtime/common.hpp"
#include "pdl.cuh"
#include "sm100.cuh"

namespace hm {
namespace attn_fwd64 {

using namespace sm100;

constexpr int DH = 64, BQ = 128, BKV = 128;
constexpr int kStages = 4;               // K / V ring (a power of two)
constexpr int kSBuf = 3;                 // rotating S / P buffers in TMEM
constexpr uint32_t kTile = BQ * DH * 2;  // 128 rows x 128 B: one SW128 atom column, 16 KB
constexpr int kThreads = 384;
constexpr float kRescaleLog2 = 8.f;      // lazy-rescale threshold (log2 units)
constexpr uint32_t C_O = kSBuf * BKV;    // O_t at columns [384 + 64 t, 448 + 64 t)
constexpr size_t kSmem = 1024 + 4 * kTile /*Q pair x 2 items*/ + 2 * kStages * kTile /*K, V*/ + 2 * kTile /*O staging*/ + 256;
static_assert(C_O + 2 * DH == 512, "TMEM budget");

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// packed fp32 pairs (sm_100 FFMA2 / FADD2 / FMUL2: one issue slot for two lanes' worth)
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.ftz.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.ftz.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.ftz.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// 2^x for a pair of x <= 0 on the FMA / ALU pipes instead of the XU (MUFU)
// pipe the softmax is bound by: x = j + f with j = rint(x) by magic-number
// rounding and f in [-0.5, 0.5]; 2^f from a degree-3 polynomial (relative
// error 7.5e-5, a fortieth of bf16's rounding step); j added into the
// exponent field.  x is clamped at -120 (masked keys: 2^-120, not 0).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -120.f);
  x.y = fmaxf(x.y, -120.f);
  const float2 y = add2(x, make_float2(12582912.f, 12582912.f));  // 1.5 * 2^23: rint(x) in the low bits
  const float2 j = add2(y, make_float2(-12582912.f, -12582912.f));
  const float2 f = fma2(j, make_float2(-1.f, -1.f), x);
  float2 q = fma2(make_float2(0.05517165f, 0.05517165f), f, make_float2(0.24261093f, 0.24261093f));
  q = fma2(q, f, make_float2(0.69326096f, 0.69326096f));
  q = fma2(q, f, make_float2(0.99992808f, 0.99992808f));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(y.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(y.y) << 23)));
}
// generic-proxy shared-memory writes -> visible to the TMA (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// the r-th item of CTA c of G (snake order over a heaviest-first list)
__device__ __forceinline__ int item_of(int r, int c, int G) { return r * G + ((r & 1) ? G - 1 - c : c); }

// One item = the query-tile pair (2 pr, 2 pr + 1) of one (sample, head), and
// the global bases of its running counters.  Positions n = 0 .. npos - 1
// order its S / PV MMAs: S_0(0), S_1(0), S_0(1), S_1(1), ... then the longer
// tile alone.
struct Item {
  bool valid;
  int r, b, h, pr, nkv0, nkv1, mn, tlast, npos;
  int kvb, pb, g0, g1;  // first global K/V block, position, tile-0 and tile-1 step
  __device__ void at(int n, int &t, int &j) const {
    if (n < 2 * mn) {
      t = n & 1;
      j = n >> 1;
    } else {
      t = tlast;
      j = mn + (n - 2 * mn);
    }
  }
};

template <bool CAUSAL>
__device__ __forceinline__ Item make_item(int r, int c, int G, int S, int H, int BH, int kvb, int pb, int g0, int g1) {
  Item it;
  const int nq = S / BQ, npair = (nq + 1) >> 1, n_items = npair * BH;
  const int i = item_of(r, c, G);
  it.valid = i < n_items;
  it.r = r;
  int bh;
  if (CAUSAL) {  // heaviest pairs first
    it.pr = npair - 1 - i / BH;
    bh = i % BH;
  } else {
    it.pr = i % npair;
    bh = i / npair;
  }
  it.b = bh / H;
  it.h = bh % H;
  const int qb0 = 2 * it.pr;
  const bool has1 = qb0 + 1 < nq;
  it.nkv0 = CAUSAL ? qb0 + 1 : S / BKV;
  it.nkv1 = has1 ? (CAUSAL ? qb0 + 2 : S / BKV) : 0;
  it.mn = it.nkv0 < it.nkv1 ? it.nkv0 : it.nkv1;
  it.tlast = it.nkv1 >= it.nkv0 ? 1 : 0;
  it.npos = it.nkv0 + it.nkv1;
  it.kvb = kvb;
  it.pb = pb;
  it.g0 = g0;
  it.g1 = g1;
  return it;
}

template <bool CAUSAL, int EMU>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo, float *__restrict__ lse,
               int S, int H, int BH, float scale_log2, unsigned long long *trace) {
  extern __shared__ uint8_t smem_raw[];
  // diagnostics (HM_ATTN_TRACE=1), 512 words per CTA: globaltimer at [0] entry,
  // [1] setup done, [62] exit; clock64 at [2] setup, [61] exit, [4 + 4 k + 2 t]
  // tile t's first S of item k, [+1] its epilogue done, [64 + 96 t + 2 k] tile
  // t's k-th S ready, [+1] its P handed over, and for the issuing threads at
  // position n < 60: [256 + 4 n] P(n) ready, [+1] PV(n) issued, [+2] S(n)'s
  // inputs ready, [+3] S(n) issued
  unsigned long long *tr = trace ? trace + 512 * blockIdx.x : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sQ = smem;                  // [2 items][2 tiles]
  uint8_t *sK = sQ + 4 * kTile;        // [kStages]
  uint8_t *sV = sK + kStages * kTile;  // [kStages]
  uint8_t *sO = sV + kStages * kTile;  // [tile]: the item's O, SW128 rows, for one TMA store
  uint64_t *bar = reinterpret_cast<uint64_t *>(sO + 2 * kTile);
  uint64_t *q_full = bar, *q_empty = bar + 2;                   // [item parity]
  uint64_t *kv_full = bar + 4, *kv_empty = kv_full + kStages;  // [stage]
  uint64_t *s_full = kv_empty + kStages;                       // [S buffer]
  uint64_t *p_full = s_full + kSBuf;                           // [tile][step parity]
  uint64_t *o_done = p_full + 4;                               // [tile]: the item's last PV_t
  uint64_t *pv_done = o_done + 2;                              // [S buffer]: PV read its P
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(pv_done + kSBuf);

  const int G = gridDim.x, c = blockIdx.x;
  const int d = H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto next_item = [&](const Item &it) {
    return make_item<CAUSAL>(it.r + 1, c, G, S, H, BH, it.kvb + (it.nkv0 > it.nkv1 ? it.nkv0 : it.nkv1),
                             it.pb + it.npos, it.g0 + it.nkv0, it.g1 + it.nkv1);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&o_done[i], 1);
    }
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < kSBuf; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&p_full[i], 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the set-up above overlapped the previous
  // kernel's tail; nothing global is read or written before it has completed
  griddep_wait();
  if (tr && threadIdx.x == 0) {
    tr[1] = globaltimer();
    tr[2] = clock64();
  }

  if (warp < 4) {
    reg_dealloc<72>();  // 3 x 168 per SMSP at launch = 72 + 2 x 216
    if (warp == 0 && lane == 0) {
      auto load_q = [&](const Item &q) {
        const int qp = q.r & 1, row0 = q.b * S;
        mbar_wait(&q_empty[qp], ((q.r >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[qp], (q.nkv1 > 0 ? 2 : 1) * kTile);
        tma_load_2d(sQ + (2 * qp) * kTile, &tm, &q_full[qp], q.h * DH, row0 + 2 * q.pr * BQ);
        if (q.nkv1 > 0) tma_load_2d(sQ + (2 * qp + 1) * kTile, &tm, &q_full[qp], q.h * DH, row0 + (2 * q.pr + 1) * BQ);
      };
      Item it = make_item<CAUSAL>(0, c, G, S, H, BH, 0, 0, 0, 0);
      if (it.valid) load_q(it);
      for (; it.valid; it = next_item(it)) {
        const int row0 = it.b * S;
        const int nall = it.nkv0 > it.nkv1 ? it.nkv0 : it.nkv1;
        // the next item's Q pair goes out while this item's K / V still stream
        // (a whole ring ahead of its first S), once the ring guarantees the
        // item before this one has issued its last S (which frees that buffer)
        const int j_q = nall - 1 < kStages ? nall - 1 : kStages;
        for (int j = 0; j < nall; ++j) {
          const int kb = it.kvb + j, st = kb & (kStages - 1);
          mbar_wait(&kv_empty[st], ((kb / kStages) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], 2 * kTile);
          tma_load_2d(sK + st * kTile, &tm, &kv_full[st], d + it.h * DH, row0 + j * BKV);
          tma_load_2d(sV + st * kTile, &tm, &kv_full[st], 2 * d + it.h * DH, row0 + j * BKV);
          if (j == j_q) {
            const Item nx = next_item(it);
            if (nx.valid) load_q(nx);
          }
        }
      }
    } else if ((warp == 1 || warp == 2) && lane == 0) {
      // Two issuing threads on two SM sub-partitions: warp 1 issues the PVs,
      // warp 2 the S MMAs.  tcgen05.mma issue blocks at the execution rate and
      // every mbarrier round trip costs ~150 cycles while the SS MMAs saturate
      // shared memory, so one thread doing both left the tensor pipe idle for
      // its waits and commits (~1300 cycles per 622 of MMAs); two threads wait
      // while the other issues.  S(m) overwrites the P that PV(m - 3) reads, and
      // MMAs of different threads are not ordered: the S thread waits for PV(m
      // - 3) to COMPLETE (pv_done), which also lets a softmax rescale wait on
      // S(prev + 3) for PV(prev).
      constexpr uint32_t idesc_s = idesc_bf16_f32(BQ, BKV, 0, 0);  // Q K-major, K K-major
      constexpr uint32_t idesc_o = idesc_bf16_f32(BQ, DH, 0, 1);   // P (TMEM), V MN-major
      // descriptor low words of buffer 0 (a buffer adds kTile >> 4, a K step of
      // Q / K 32 B >> 4 = 2, of V 2048 B >> 4 = 128); all share one high word
      const uint32_t d_hi = (uint32_t)(umma_desc_sw128(0, 0, 1024) >> 32);
      if (warp == 2) {
        const uint32_t q_lo0 = (uint32_t)umma_desc_sw128(smem_u32(sQ), 16, 1024);
        const uint32_t k_lo0 = (uint32_t)umma_desc_sw128(smem_u32(sK), 16, 1024);
        Item sit = make_item<CAUSAL>(0, c, G, S, H, BH, 0, 0, 0, 0);
        int s_loc = 0, s_buf = 0, kv_ready = -1, tail = 0;
        for (int m = 0;; ++m) {
          if (s_loc >= sit.npos) {
            do {
              sit = next_item(sit);
            } while (sit.valid && sit.npos == 0);
            s_loc = 0;
          }
          if (m >= kSBuf) {  // PV(m - 3) has read this buffer's P
            mbar_wait(&pv_done[s_buf], ((m - kSBuf) / kSBuf) & 1);
            tc_fence_after();
          }
          if (!sit.valid) {  // past the last item: kSBuf empty commits keep s_full's
            mma_commit(&s_full[s_buf]);  // phases in step with the positions a rescale names
            s_buf = s_buf == kSBuf - 1 ? 0 : s_buf + 1;
            if (++tail == kSBuf) break;
            continue;
          }
          const int qp = sit.r & 1;
          if (s_loc == 0) mbar_wait(&q_full[qp], (sit.r >> 1) & 1);
          int t, j;
          sit.at(s_loc, t, j);
          const int kb = sit.kvb + j;
          if (kb > kv_ready) {  // both tiles' S of a step read the same K block: one wait
            mbar_wait(&kv_full[kb & (kStages - 1)], (kb / kStages) & 1);
            kv_ready = kb;
          }
          tc_fence_after();
          if (tr && m < 60) tr[258 + 4 * m] = clock64();
          const uint32_t q_lo = q_lo0 + (uint32_t)(2 * qp + t) * (kTile >> 4);
          const uint32_t k_lo = k_lo0 + (uint32_t)(kb & (kStages - 1)) * (kTile >> 4);
          const uint32_t d_s = tmem + s_buf * BKV;
          mma_bf16_lohi(d_s, q_lo, k_lo, d_hi, idesc_s, 0u);
#pragma unroll
          for (int kk = 1; kk < DH / 16; ++kk) mma_bf16_lohi(d_s, q_lo + 2 * kk, k_lo + 2 * kk, d_hi, idesc_s, 1u);
          mma_commit(&s_full[s_buf]);
          if (s_loc == sit.npos - 1) mma_commit(&q_empty[qp]);  // the item's last Q K^T: its Q pair is free
          if (tr && m < 60) tr[259 + 4 * m] = clock64();
          s_buf = s_buf == kSBuf - 1 ? 0 : s_buf + 1;
          ++s_loc;
        }
      } else {
        const uint32_t v_lo0 = (uint32_t)umma_desc_sw128(smem_u32(sV), kTile, 1024);
        int pv_buf = 0, gc0 = 0, gc1 = 0;  // PV position % kSBuf; steps of tile 0 / 1 so far
        for (Item it = make_item<CAUSAL>(0, c, G, S, H, BH, 0, 0, 0, 0); it.valid; it = next_item(it)) {
          for (int n = 0; n < it.npos; ++n) {
            int t, j;
            it.at(n, t, j);
            const int gs = t ? gc1++ : gc0++, kb = it.kvb + j, P = it.pb + n;
            mbar_wait(&p_full[2 * t + (gs & 1)], (gs >> 1) & 1);  // P_t(j) in S buffer pv_buf (and O_t rescaled)
            tc_fence_after();
            if (tr && P < 60) tr[256 + 4 * P] = clock64();
            const uint32_t v_lo = v_lo0 + (uint32_t)(kb & (kStages - 1)) * (kTile >> 4);
            const uint32_t p_tm = tmem + pv_buf * BKV, d_o = tmem + C_O + t * DH;
            mma_bf16_ts_lohi(d_o, p_tm, v_lo, d_hi, idesc_o, j > 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 1; kk < BKV / 16; ++kk) mma_bf16_ts_lohi(d_o, p_tm + kk * 8, v_lo + kk * 128, d_hi, idesc_o, 1u);
            if (tr && P < 60) tr[257 + 4 * P] = clock64();
            mma_commit(&pv_done[pv_buf]);
            if (j == (t == 0 ? it.nkv0 : it.nkv1) - 1) mma_commit(&o_done[t]);  // O_t of this item final
            // last use of K_j / V_j: the S MMAs that read K_j completed before
            // their softmax handed over the P this PV reads
            if (t == 1 || j >= it.mn) mma_commit(&kv_empty[kb & (kStages - 1)]);
            pv_buf = pv_buf == kSBuf - 1 ? 0 : pv_buf + 1;
          }
        }
      }
    }
  } else {
    reg_alloc<216>();
    const int t = (warp >> 2) - 1;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;  // query row inside the tile == TMEM lane
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    const uint32_t o_addr = tmem + lane_addr + C_O + t * DH;
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    int done = 0;  // items this tile has finished (o_done parity)
    const bool rec = tr && q4 == 0 && lane == 0;
    int ks = 0;  // trace: steps this tile has run
    for (Item it = make_item<CAUSAL>(0, c, G, S, H, BH, 0, 0, 0, 0); it.valid; it = next_item(it)) {
      const int nkv = t == 0 ? it.nkv0 : it.nkv1;
      if (nkv == 0) continue;
      const int qb = 2 * it.pr + t, row0 = it.b * S, g_base = t == 0 ? it.g0 : it.g1;
      float m = -INFINITY, l = 0.f;  // m: the max the exponents are taken against (log2 domain)
      for (int j = 0; j < nkv; ++j) {
        const int n = it.pb + (j < it.mn ? 2 * j + t : 2 * it.mn + (j - it.mn));  // global position
        const int gs = g_base + j;                                                // global step of this tile
        const int buf = n % kSBuf;
        const uint32_t s_addr = tmem + lane_addr + buf * BKV;
        mbar_wait(&s_full[buf], (n / kSBuf) & 1);
        tc_fence_after();
        if (rec && j == 0 && it.r < 14) tr[4 + 4 * it.r + 2 * t] = clock64();
        if (rec && ks < 48) tr[64 + 96 * t + 2 * ks] = clock64();
        uint32_t v[BKV];
#pragma unroll
        for (int q = 0; q < BKV / 32; ++q)
          tmem_ld_32x32b_x32(s_addr + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * q));
        tmem_ld_wait();
        if (CAUSAL && j == qb) {  // diagonal tile: keys after the query are masked
#pragma unroll
          for (int cc = 0; cc < BKV; ++cc)
            if (cc > r) v[cc] = 0xff800000u;  // -inf
        }
        float mx[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) mx[e] = fmaxf(__uint_as_float(v[e]), __uint_as_float(v[4 + e]));
#pragma unroll
        for (int cc = 8; cc < BKV; cc += 8) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            mx[e] = fmaxf(mx[e], fmaxf(__uint_as_float(v[cc + e]), __uint_as_float(v[cc + 4 + e])));
        }
        const float m_row = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
        float alpha = 1.f;
        if (m_row > m + kRescaleLog2) {  // first tile (m = -inf) always lands here
          alpha = ex2(m - m_row);
          m = m_row;
        }
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {  // warp-uniform: tcgen05.ld / st are .sync.aligned
          // wait for PV_t(j - 1): S(prev + 3) is issued only once PV(prev) has
          // completed, so its completion covers it.  Its buffer cannot have
          // cycled again: the next S into it follows PV(n + 1), which follows
          // this thread's P(n).
          const int jp = j - 1;
          const int need = it.pb + (jp < it.mn ? 2 * jp + t : 2 * it.mn + (jp - it.mn)) + kSBuf;
          mbar_wait(&s_full[need % kSBuf], (need / kSBuf) & 1);
          tc_fence_after();
          const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
          for (int c0 = 0; c0 < DH; c0 += 32) {
            uint32_t ov[32];
            tmem_ld_32x32b_x32(o_addr + c0, ov);
            tmem_ld_wait();
#pragma unroll
            for (int cc = 0; cc < 32; cc += 2) {
              const float2 o2 = mul2(make_float2(__uint_as_float(ov[cc]), __uint_as_float(ov[cc + 1])), a2);
              ov[cc] = __float_as_uint(o2.x);
              ov[cc + 1] = __float_as_uint(o2.y);
            }
            tmem_st_32x32b_x32(o_addr + c0, ov);
          }
        }
        const float2 nm2 = make_float2(-m, -m);
        float2 rs[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c0 = 0; c0 < BKV; c0 += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int cc = 0; cc < 32; cc += 2) {
            const float2 x = fma2(make_float2(__uint_as_float(v[c0 + cc]), __uint_as_float(v[c0 + cc + 1])), sc2, nm2);
            // EMU > 0: one exponent pair in EMU on the FMA pipe (the XU pipe bounds the softmax)
            const float2 p = (EMU > 0 && (cc >> 1) % (EMU > 0 ? EMU : 1) == (EMU > 0 ? EMU : 1) - 1)
                                 ? ex2_poly2(x)
                                 : make_float2(ex2(x.x), ex2(x.y));
            rs[(cc >> 1) & 1] = add2(rs[(cc >> 1) & 1], p);
            pk[cc >> 1] = bf16x2(p.x, p.y);
          }
          // keys c0..c0+31 -> P columns c0/2..c0/2+15 (every S column already read)
          tmem_st_32x32b_x16(s_addr + (c0 >> 1), pk);
        }
        tmem_st_wait();
        l = l * alpha + ((rs[0].x + rs[0].y) + (rs[1].x + rs[1].y));
        tc_fence_before();
        mbar_arrive(&p_full[2 * t + (gs & 1)]);
        if (rec && ks < 48) tr[65 + 96 * t + 2 * ks] = clock64();
        ++ks;
      }
      // epilogue: O / l and lse once the item's last PV_t has completed; the
      // next item's first PV_t overwrites O only after this thread's next P
      mbar_wait(&o_done[t], done & 1);
      ++done;
      tc_fence_after();
      const float inv = 1.f / l;
      // O leaves as one TMA store per tile from SW128 staging (query rows are d
      // apart in `out`: 16-B stores from every thread throttle the LSU)
      const bool leader = q4 == 0 && lane == 0;
      if (leader) bulk_wait_read0();  // this tile's previous store has read the staging
      asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
      uint8_t *srow = sO + t * kTile + r * 128;
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t ov[32];
        tmem_ld_32x32b_x32(o_addr + c0, ov);
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 32; cc += 8) {
          uint4 w;
          w.x = bf16x2(__uint_as_float(ov[cc]) * inv, __uint_as_float(ov[cc + 1]) * inv);
          w.y = bf16x2(__uint_as_float(ov[cc + 2]) * inv, __uint_as_float(ov[cc + 3]) * inv);
          w.z = bf16x2(__uint_as_float(ov[cc + 4]) * inv, __uint_as_float(ov[cc + 5]) * inv);
          w.w = bf16x2(__uint_as_float(ov[cc + 6]) * inv, __uint_as_float(ov[cc + 7]) * inv);
          *reinterpret_cast<uint4 *>(srow + ((((c0 + cc) >> 3) ^ (r & 7)) << 4)) = w;
        }
      }
      fence_async_smem();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
      if (leader) {
        tma_store_2d(&tmo, sO + t * kTile, it.h * DH, row0 + qb * BQ);
        bulk_commit();
      }
      lse[(int64_t)(row0 + qb * BQ + r) * H + it.h] = m + log2f(l);
      if (rec && it.r < 14) tr[5 + 4 * it.r + 2 * t] = clock64();
      tc_fence_before();
    }
    if (q4 == 0 && lane == 0) bulk_wait0();  // the last O store has left shared memory
  }
  tc_fence_before();
  __syncthreads();
  if (tr && threadIdx.x == 0) {
    tr[61] = clock64();
    tr[62] = globaltimer();
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

bool supported(int S, int DHx) { return DHx == DH && S % BQ == 0; }

int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  const int d = H * DH;
  CUtensorMap tm;  // qkv [B*S, 3d] bf16, {64, 128} boxes, 128-B swizzle
  cuuint64_t dims[2] = {(cuuint64_t)3 * d, (cuuint64_t)B * S};
  cuuint64_t strides[1] = {(cuuint64_t)3 * d * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(qkv), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(HM_ERR_DEVICE, "attention (head_dim 64) tensor map encode failed");
  CUtensorMap tmo;  // out [B*S, d] bf16, {64, 128} boxes, 128-B swizzle (TMA-stored O tiles)
  {
    cuuint64_t odims[2] = {(cuuint64_t)d, (cuuint64_t)B * S};
    cuuint64_t ostrides[1] = {(cuuint64_t)d * 2};
    if (fn(&tmo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, o, odims, ostrides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(HM_ERR_DEVICE, "attention (head_dim 64) output tensor map encode failed");
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  ProfScope ps(KC_ATTN_FWD, s, 4.0 * B * (double)S * S * H * DH * (causal ? 0.5 : 1.0), (double)B * S * H * DH * 2 * 4);
  static bool attr[2] = {false, false};
  // one exponent pair in eight on the FMA pipe (HM_ATTN_EMU=0: all on the XU
  // pipe): 4 x 1024 x 25 causal 36.3 -> 35.4 us, 8 x 512 x 16 22.8 -> 21.8;
  // one in four measured the same, one in two slower (profiles/r02_attn_emu_ab.jsonl)
  static const bool emu = !(getenv("HM_ATTN_EMU") && atoi(getenv("HM_ATTN_EMU")) == 0);
  auto k = causal ? (emu ? fwd_kernel<true, 8> : fwd_kernel<true, 0>) : (emu ? fwd_kernel<false, 8> : fwd_kernel<false, 0>);
  if (!attr[causal ? 1 : 0]) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr[causal ? 1 : 0] = true;
  }
  const int npair = (S / BQ + 1) / 2;
  const int sms = current_sm_count();
  const int items = npair * B * H;
  const int grid = items < sms ? items : sms;
  static const bool tracing = getenv("HM_ATTN_TRACE") && getenv("HM_ATTN_TRACE")[0] == '1';
  static unsigned long long *tbuf = nullptr;
  if (tracing && !tbuf) HM_CUDA(cudaMalloc(&tbuf, 512 * 1024 * sizeof(unsigned long long)));
  if (tracing) HM_CUDA(cudaMemsetAsync(tbuf, 0, 512 * grid * sizeof(unsigned long long), s));
  HM_CUDA(launch_pdl(k, dim3(grid), dim3(kThreads), kSmem, s, tm, tmo, lse, S, H, B * H, scale_log2,
                     tracing ? tbuf : nullptr));
  if (tracing) {  // one JSON line per launch: every CTA's timestamps, ns after the earliest entry
    std::vector<unsigned long long> h(512 * grid);
    HM_CUDA(cudaStreamSynchronize(s));
    HM_CUDA(cudaMemcpy(h.data(), tbuf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ULL;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[512 * c]);
    fprintf(stderr, "{\"attn_fwd64_trace\": {\"B\": %d, \"S\": %d, \"H\": %d, \"cta\": [", B, S, H);
    for (int c = 0; c < grid; ++c) {
      fprintf(stderr, "%s[", c ? ", " : "");
      for (int n = 0; n < 512; ++n) {  // [0], [1], [62]: ns after the earliest entry; the rest raw clock64
        const unsigned long long x = h[512 * c + n];
        fprintf(stderr, "%s%lld", n ? ", " : "",
                !x ? -1LL : (n == 0 || n == 1 || n == 62) ? (long long)(x - t0) : (long long)x);
      }
      fprintf(stderr, "]");
    }
    fprintf(stderr, "]}}\n");
  }
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

}  // namespace attn_fwd64
}  // namespace hm
