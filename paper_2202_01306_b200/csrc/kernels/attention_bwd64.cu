// attention_bwd64.cu -- flash-attention backward for head_dim 64 on the 5th-gen
// tensor cores, pipelined over 64-query sub-blocks (HM_ATTN_BWD=s; measured
// within 3% of attention_tc.cu's 128-query kernel, which stays the default:
// see attention.cu).
//
// The 128-query dataflow of attention_tc.cu is bounded by its
// single shared-memory P^T / dS^T buffer: the softmax of block n+1 may write
// only after dV / dK / dQ(n) have read block n's (3800 cycles per block where
// the MMAs need ~1300, HM_ATTN_TRACE).  Here every CTA (persistent, heaviest
// causal key blocks first, snake order as in attention_tc.cu) walks 64-query
// sub-blocks j of its 128-key block, and the two softmax warpgroups take the
// even and the odd sub-blocks:
//
//   S^T_j  = K Q_j^T,  dP^T_j = V dO_j^T     TMEM buffer j & 1 (64 + 64 columns)
//   P^T_j  = exp2(S^T_j c - lse),  dS^T_j = P^T_j (dP^T_j - D)
//            -> bf16 pairs written back into the buffer's own columns, and
//               dS^T_j also into shared memory (half j & 1 of the pair buffer)
//   dV    += P^T_j dO_j,  dK += dS^T_j Q_j   (A operands straight from TMEM)
//   dQ_p   = dS_p K       per pair p = (2p, 2p+1): M = 128 queries, TMEM
//                         double-buffered, drained by both warpgroups one pair
//                         later, one TMA reduce-add per warpgroup half
//
// TMEM: S/dP buffers [0, 256), dV [256, 320), dK [320, 384), dQ x2 [384, 512).
// S^T_{j+2} reuses buffer j & 1 and is issued right after dV / dK(j), which
// read P^T_j / dS^T_j from it first (tcgen05.mma executes in issue order), so
// a warpgroup's next sub-block is computed while it still works on the
// current one, and the two warpgroups keep the tensor pipe fed alternately.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <mutex>

#include "../runtime/common.hpp"
#include "sm100.cuh"

namespace hm {
namespace attn_bwd64 {

using namespace sm100;

constexpr int DH = 64, BKV = 128, SQ = 64;
constexpr int kQStages = 3;
constexpr uint32_t kKV = BKV * 128;         // 128 keys x 64 dims bf16: 16 KB
constexpr uint32_t kSub = SQ * 128;         // 64 queries x 64 dims bf16: 8 KB
constexpr uint32_t kDS = 2 * BKV * 128;     // dS^T of a pair: [query half][128 keys][64 queries]: 32 KB
constexpr uint32_t kDQ = BKV * 32 * 4;      // one warpgroup's dQ half: 128 queries x 32 fp32: 16 KB
constexpr int kThreads = 384;
constexpr uint32_t C_DV = 256, C_DK = 320, C_DQ = 384;
constexpr size_t kSmem = 1024 + 2 * kKV + 2 * kQStages * kSub + 2 * kDS + 2 * kDQ + 2 * 2 * 128 * 4 + 256;
static_assert(kSmem <= 232448, "shared memory");

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// the r-th item of CTA c of G (snake order over a heaviest-first list)
__device__ __forceinline__ int item_of(int r, int c, int G) { return r * G + ((r & 1) ? G - 1 - c : c); }

template <bool CAUSAL>
__global__ void __launch_bounds__(kThreads, 1)
    bwd_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
               const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
               const float *__restrict__ lse, const float *__restrict__ dvec, __nv_bfloat16 *__restrict__ dqkv, int S,
               int H, int BH, float scale_log2, float scale, unsigned long long *trace) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sK = smem;
  uint8_t *sV = sK + kKV;
  uint8_t *sQ = sV + kKV;                    // [kQStages]
  uint8_t *sdO = sQ + kQStages * kSub;       // [kQStages]
  uint8_t *sDS = sdO + kQStages * kSub;      // [2 pair buffers]
  uint8_t *sDQ = sDS + 2 * kDS;              // [2 warpgroups]
  float *sLD = reinterpret_cast<float *>(sDQ + 2 * kDQ);  // [2 wg][2 stages][lse 64 | D 64]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sLD + 2 * 2 * 128);
  uint64_t *kv_full = bar, *kv_empty = bar + 1;
  uint64_t *q_full = bar + 2, *q_empty = q_full + kQStages;  // [kQStages]
  uint64_t *s_full = q_empty + kQStages;                     // [wg]
  uint64_t *p_full = s_full + 2;                             // [wg]
  uint64_t *ds_empty = p_full + 2;                           // [pair buffer]
  uint64_t *dq_full = ds_empty + 2, *dq_empty = dq_full + 2;  // [dQ buffer]
  uint64_t *acc_full = dq_empty + 2, *acc_empty = acc_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 1);

  const int nkb = S / BKV, n_items = nkb * BH;
  const int G = gridDim.x, c = blockIdx.x;
  const int d = H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto decode = [&](int i, int &kb, int &b, int &h) {
    int bh;
    if (CAUSAL) {  // key block 0 first: it sees every query
      kb = i / BH;
      bh = i % BH;
    } else {
      kb = i % nkb;
      bh = i / nkb;
    }
    b = bh / H;
    h = bh % H;
  };
  auto nsub_of = [&](int kb) { return (S - (CAUSAL ? kb * BKV : 0)) / SQ; };  // even: S % 128 == 0
  // diagnostics (HM_ATTN_TRACE=1): clock64 at phase boundaries of CTA 0's first
  // 64 sub-blocks, trace[event * 64 + sub-block]
  auto mark = [&](int ev, int nn) {
    if (trace && c == 0 && nn < 64) trace[ev * 64 + nn] = clock64();
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&ds_empty[i], 1);
      mbar_init(&dq_full[i], 1);
      mbar_init(&dq_empty[i], 256);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 256);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    reg_dealloc<72>();  // 3 x 168 registers per SMSP at launch = 72 + 2 x 216
    if (warp == 0 && lane == 0) {
      int g = 0;  // running sub-block counter
      for (int r = 0, i; (i = item_of(r, c, G)) < n_items; ++r) {
        int kb, b, h;
        decode(i, kb, b, h);
        const int row0 = b * S, q0 = CAUSAL ? kb * BKV : 0, nsub = nsub_of(kb);
        mbar_wait(kv_empty, (r & 1) ^ 1);  // every MMA of the previous item has read K / V
        mbar_expect_tx(kv_full, 2 * kKV);
        tma_load_2d(sK, &tm_kv, kv_full, d + h * DH, row0 + kb * BKV);
        tma_load_2d(sV, &tm_kv, kv_full, 2 * d + h * DH, row0 + kb * BKV);
        for (int j = 0; j < nsub; ++j, ++g) {
          const int st = g % kQStages;
          mbar_wait(&q_empty[st], ((g / kQStages) & 1) ^ 1);
          mbar_expect_tx(&q_full[st], 2 * kSub);
          tma_load_2d(sQ + st * kSub, &tm_q, &q_full[st], h * DH, row0 + q0 + j * SQ);
          tma_load_2d(sdO + st * kSub, &tm_do, &q_full[st], h * DH, row0 + q0 + j * SQ);
        }
      }
    } else if (warp == 1 && lane == 0) {
      constexpr uint32_t id_st = idesc_bf16_f32(BKV, SQ, 0, 0);   // S^T, dP^T: K-major x K-major, N = 64
      constexpr uint32_t id_acc = idesc_bf16_f32(BKV, DH, 0, 1);  // dV, dK: A (TMEM), B MN-major
      constexpr uint32_t id_dq = idesc_bf16_f32(BKV, DH, 1, 1);   // dQ: A = dS MN-major, B = K MN-major
      const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
      // S^T / dP^T of running sub-block gg into TMEM buffer gg & 1
      auto issue_s = [&](int gg) {
        const int st = gg % kQStages, w = gg & 1;
        mbar_wait(&q_full[st], (gg / kQStages) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ + st * kSub), do_base = smem_u32(sdO + st * kSub);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          mma_bf16(tmem + w * 128, umma_desc_sw128(k_base + kk * 32, 16, 1024),
                   umma_desc_sw128(q_base + kk * 32, 16, 1024), id_st, kk > 0);
          mma_bf16(tmem + w * 128 + 64, umma_desc_sw128(v_base + kk * 32, 16, 1024),
                   umma_desc_sw128(do_base + kk * 32, 16, 1024), id_st, kk > 0);
        }
        mma_commit(&s_full[w]);
        mark(0, gg);
      };
      int g = 0;
      for (int r = 0, i; (i = item_of(r, c, G)) < n_items; ++r) {
        int kb, b, h;
        decode(i, kb, b, h);
        const int nsub = nsub_of(kb);
        mbar_wait(kv_full, r & 1);
        issue_s(g);
        issue_s(g + 1);
        for (int j = 0; j < nsub; ++j) {
          const int gg = g + j, w = gg & 1, st = gg % kQStages;
          mbar_wait(&p_full[w], (gg >> 1) & 1);  // P^T / dS^T of sub-block gg in TMEM (and dS^T in smem)
          mark(1, gg);
          if (j == 0) mbar_wait(acc_empty, (r & 1) ^ 1);  // the previous item's dV / dK drained
          tc_fence_after();
          const uint32_t q_base = smem_u32(sQ + st * kSub), do_base = smem_u32(sdO + st * kSub);
#pragma unroll
          for (int kk = 0; kk < SQ / 16; ++kk) {  // reduction over the sub-block's 64 queries
            const uint32_t acc = (j > 0 || kk > 0) ? 1u : 0u;
            mma_bf16_ts(tmem + C_DV, tmem + w * 128 + kk * 8, umma_desc_sw128(do_base + kk * 2048, kSub, 1024),
                        id_acc, acc);
            mma_bf16_ts(tmem + C_DK, tmem + w * 128 + 64 + kk * 8, umma_desc_sw128(q_base + kk * 2048, kSub, 1024),
                        id_acc, acc);
          }
          mma_commit(&q_empty[st]);
          if (j & 1) {  // pair complete: dQ_p = dS_p K (128 queries)
            const int pg = gg >> 1, qb = pg & 1;
            mbar_wait(&dq_empty[qb], ((pg >> 1) & 1) ^ 1);  // dQ of pair pg - 2 drained
            tc_fence_after();
            const uint32_t ds_base = smem_u32(sDS + qb * kDS);
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk)  // reduction over the 128 keys
              mma_bf16(tmem + C_DQ + qb * 64, umma_desc_sw128(ds_base + kk * 2048, BKV * 128, 1024),
                       umma_desc_sw128(k_base + kk * 2048, kKV, 1024), id_dq, kk > 0);
            mma_commit(&dq_full[qb]);
            mma_commit(&ds_empty[qb]);
            mark(2, gg);
          }
          // S^T(gg + 2) reuses buffer w: dV / dK(gg) above read P^T / dS^T from it first
          if (j + 2 < nsub) issue_s(gg + 2);
        }
        mma_commit(acc_full);
        mma_commit(kv_empty);
        g += nsub;
      }
    }
  } else {
    reg_alloc<216>();
    const int w = (warp >> 2) - 1;  // warpgroup: even (0) / odd (1) sub-blocks
    const int q4 = warp & 3;
    const int rr = q4 * 32 + lane;  // key row (S^T, dP^T, dV, dK) / query row of a pair (dQ) == TMEM lane
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    const uint32_t s_addr = tmem + lane_addr + w * 128;
    float *ld_base = sLD + w * 256;  // [2 stages][lse 64 | D 64]
    uint8_t *dq_stage = sDQ + w * kDQ;
    // dQ of pair pg (query rows qrow .. qrow + 127, head hh): this warpgroup's 32
    // columns TMEM -> SW128 stage -> one TMA reduce-add
    auto dq_out = [&](int pg, int qrow, int hh) {
      const int qb = pg & 1;
      mbar_wait(&dq_full[qb], (pg >> 1) & 1);
      tc_fence_after();
      uint32_t q[32];
      tmem_ld_32x32b_x32(tmem + lane_addr + C_DQ + qb * 64 + w * 32, q);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&dq_empty[qb]);
      if (rr == 0) bulk_wait_read0();  // the previous reduce has read the stage
      named_sync(3 + w, 128);
      uint8_t *row = dq_stage + rr * 128;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        *reinterpret_cast<float4 *>(row + ((jj ^ (rr & 7)) << 4)) =
            make_float4(__uint_as_float(q[4 * jj]) * scale, __uint_as_float(q[4 * jj + 1]) * scale,
                        __uint_as_float(q[4 * jj + 2]) * scale, __uint_as_float(q[4 * jj + 3]) * scale);
      fence_async_smem();
      named_sync(3 + w, 128);
      if (rr == 0) {
        tma_reduce_add_2d(&tm_dq, dq_stage, hh * DH + 32 * w, qrow);
        bulk_commit();
      }
    };
    int g = 0;
    int prev_pg = -1, prev_qrow = 0, prev_h = 0;
    for (int r = 0, it; (it = item_of(r, c, G)) < n_items; ++r) {
      int kb, b, h;
      decode(it, kb, b, h);
      const int row0 = b * S, q0 = CAUSAL ? kb * BKV : 0, nsub = nsub_of(kb);
      const int key = kb * BKV + rr;
      // lse (threads 0-63) / D (64-127) of this warpgroup's next sub-block, one ahead
      auto ld_src = [&](int j) {
        return rr < SQ ? lse[(int64_t)(row0 + q0 + j * SQ + rr) * H + h]
                       : dvec[(int64_t)(row0 + q0 + j * SQ + rr - SQ) * H + h];
      };
      float x_next = ld_src(w);
      for (int j = w; j < nsub; j += 2) {
        const int gg = g + j, pg = gg >> 1;  // pg: this warpgroup's running sub-block count == pair index
        float *lds = ld_base + (pg & 1) * 128;
        lds[rr] = x_next;
        if (j + 2 < nsub) x_next = ld_src(j + 2);
        named_sync(1 + w, 128);
        mbar_wait(&s_full[w], pg & 1);
        if (rr == 0) mark(3, gg);
        tc_fence_after();
        uint32_t sv[SQ], dp[SQ];
        tmem_ld_32x32b_x32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(sv));
        tmem_ld_32x32b_x32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
        tmem_ld_32x32b_x32(s_addr + 64, *reinterpret_cast<uint32_t(*)[32]>(dp));
        tmem_ld_32x32b_x32(s_addr + 96, *reinterpret_cast<uint32_t(*)[32]>(dp + 32));
        tmem_ld_wait();
        const int qs = q0 + j * SQ;  // first query of the sub-block
        const bool diag = CAUSAL && qs < kb * BKV + BKV;
        uint32_t pk[SQ / 2], dk[SQ / 2];
#pragma unroll
        for (int cq = 0; cq < SQ; cq += 4) {
          const float4 L4 = *reinterpret_cast<const float4 *>(lds + cq);
          const float4 D4 = *reinterpret_cast<const float4 *>(lds + SQ + cq);
          const float lq[4] = {L4.x, L4.y, L4.z, L4.w}, dq4[4] = {D4.x, D4.y, D4.z, D4.w};
          float p[4], gr[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            p[k] = ex2(fmaf(__uint_as_float(sv[cq + k]), scale_log2, -lq[k]));
            if (diag && qs + cq + k < key) p[k] = 0.f;  // query < key: masked
            gr[k] = p[k] * (__uint_as_float(dp[cq + k]) - dq4[k]);
          }
          pk[cq >> 1] = bf16x2(p[0], p[1]);
          pk[(cq >> 1) + 1] = bf16x2(p[2], p[3]);
          dk[cq >> 1] = bf16x2(gr[0], gr[1]);
          dk[(cq >> 1) + 1] = bf16x2(gr[2], gr[3]);
        }
        // P^T / dS^T into the buffer's own columns (A operands of dV / dK)
        tmem_st_32x32b_x32(s_addr, pk);
        tmem_st_32x32b_x32(s_addr + 64, dk);
        // dS^T into half w of the pair's shared-memory buffer (A operand of dQ)
        if (rr == 0) mark(4, gg);
        mbar_wait(&ds_empty[pg & 1], ((pg >> 1) & 1) ^ 1);  // dQ of pair pg - 2 has read it
        if (rr == 0) mark(5, gg);
        uint8_t *dsrow = sDS + (pg & 1) * kDS + w * (BKV * 128) + rr * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          *reinterpret_cast<uint4 *>(dsrow + ((ch ^ (rr & 7)) << 4)) =
              make_uint4(dk[4 * ch], dk[4 * ch + 1], dk[4 * ch + 2], dk[4 * ch + 3]);
        tmem_st_wait();
        fence_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full[w]);
        if (rr == 0) mark(6, gg);
        // the previous pair's dQ: complete by now or soon, drained off the critical path
        if (prev_pg >= 0) dq_out(prev_pg, prev_qrow, prev_h);
        if (rr == 0) mark(7, gg);
        prev_pg = pg;
        prev_qrow = row0 + q0 + (j & ~1) * SQ;
        prev_h = h;
      }
      // dV (warpgroup 0) or dK (warpgroup 1) of this key block
      mbar_wait(acc_full, r & 1);
      tc_fence_after();
      uint32_t acc[DH];
      tmem_ld_32x32b_x32(tmem + lane_addr + (w == 0 ? C_DV : C_DK), *reinterpret_cast<uint32_t(*)[32]>(acc));
      tmem_ld_32x32b_x32(tmem + lane_addr + (w == 0 ? C_DV : C_DK) + 32, *reinterpret_cast<uint32_t(*)[32]>(acc + 32));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(acc_empty);  // the next item's first dV / dK MMAs may overwrite
      const int64_t ldq = 3 * (int64_t)d;
      __nv_bfloat16 *orow = dqkv + (int64_t)(row0 + kb * BKV + rr) * ldq + (w == 0 ? 2 * d : d) + h * DH;
      const float osc = w == 0 ? 1.f : scale;
#pragma unroll
      for (int cc = 0; cc < DH; cc += 8) {
        uint4 v;
        v.x = bf16x2(__uint_as_float(acc[cc]) * osc, __uint_as_float(acc[cc + 1]) * osc);
        v.y = bf16x2(__uint_as_float(acc[cc + 2]) * osc, __uint_as_float(acc[cc + 3]) * osc);
        v.z = bf16x2(__uint_as_float(acc[cc + 4]) * osc, __uint_as_float(acc[cc + 5]) * osc);
        v.w = bf16x2(__uint_as_float(acc[cc + 6]) * osc, __uint_as_float(acc[cc + 7]) * osc);
        *reinterpret_cast<uint4 *>(orow + cc) = v;
      }
      g += nsub;
    }
    if (prev_pg >= 0) dq_out(prev_pg, prev_qrow, prev_h);
    if (rr == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
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

// [rows, inner] with a row pitch in bytes, {box0, box1} boxes
static int make_map(CUtensorMap *tm, const void *base, CUtensorMapDataType dt, int64_t inner, int64_t rows,
                    int64_t pitch_bytes, uint32_t box0, uint32_t box1) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  if (fn(tm, dt, 2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return fail(HM_ERR_DEVICE, "attention backward (head_dim 64) tensor map encode failed");
  return HM_OK;
}

bool supported(int S, int DHx) { return DHx == DH && S % BKV == 0; }

// dq_acc must be zeroed by the caller; it receives scale * dS K (fp32)
int backward_main(const void *qkv, const void *dout, const float *lse, const float *dvec, float *dq_acc, void *dqkv,
                  int B, int S, int H, int causal, cudaStream_t s) {
  const int d = H * DH;
  CUtensorMap tkv, tq, tdo, tdq;
  const auto bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  HM_TRY(make_map(&tkv, qkv, bf, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2, 64, BKV));
  HM_TRY(make_map(&tq, qkv, bf, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2, 64, SQ));
  HM_TRY(make_map(&tdo, dout, bf, d, (int64_t)B * S, (int64_t)d * 2, 64, SQ));
  HM_TRY(make_map(&tdq, dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, d, (int64_t)B * S, (int64_t)d * 4, 32, BKV));
  static bool attr[2] = {false, false};
  auto k = causal ? bwd_kernel<true> : bwd_kernel<false>;
  if (!attr[causal ? 1 : 0]) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr[causal ? 1 : 0] = true;
  }
  const int sms = current_sm_count();
  const int items = (S / BKV) * B * H;
  const float scale = 1.f / sqrtf((float)DH);
  static const bool tracing = getenv("HM_ATTN_TRACE") && getenv("HM_ATTN_TRACE")[0] == '1';
  static unsigned long long *tbuf = nullptr;
  if (tracing && !tbuf) {
    HM_CUDA(cudaMalloc(&tbuf, 8 * 64 * sizeof(unsigned long long)));
    HM_CUDA(cudaMemset(tbuf, 0, 8 * 64 * sizeof(unsigned long long)));
  }
  k<<<dim3(items < sms ? items : sms), kThreads, kSmem, s>>>(tkv, tq, tdo, tdq, lse, dvec,
                                                             static_cast<__nv_bfloat16 *>(dqkv), S, H, B * H,
                                                             1.4426950408889634f * scale, scale,
                                                             tracing ? tbuf : nullptr);
  if (tracing) {  // CTA 0's phase timestamps (cycles from its first S^T issue) to stderr
    unsigned long long hbuf[8 * 64];
    HM_CUDA(cudaStreamSynchronize(s));
    HM_CUDA(cudaMemcpy(hbuf, tbuf, sizeof hbuf, cudaMemcpyDeviceToHost));
    fprintf(stderr, "{\"attn_bwd64_trace\": [");
    for (int e = 0; e < 8; ++e) {
      fprintf(stderr, "%s[", e ? ", " : "");
      for (int n = 0; n < 64; ++n)
        fprintf(stderr, "%s%lld", n ? ", " : "", hbuf[e * 64 + n] ? (long long)(hbuf[e * 64 + n] - hbuf[0]) : 0LL);
      fprintf(stderr, "]");
    }
    fprintf(stderr, "]}\n");
  }
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

}  // namespace attn_bwd64
}  // namespace hm
