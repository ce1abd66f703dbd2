// attention_tc128.cu -- flash attention for head_dim 128 (the >HBM GPT shapes:
// d = 8192, 64 heads) on the 5th-gen tensor cores.  attention_tc.cu covers
// head_dim 64; at 128 the head-dim-64 dataflow no longer fits (O held in
// registers would need 128 more per thread, the backward's five accumulators
// 640 TMEM columns), so both kernels here are laid out differently.
//
// Forward (fwd_kernel: one CTA per pair of 128-query tiles, heaviest causal
// pairs first):
//   warp 0      TMA: both Q tiles once, then K_j / V_j (128 keys x 128 dims,
//               two 64-column SW128 boxes each) into a 2-stage ring shared by
//               the two query tiles
//   warp 1      MMA issuer.  Per tile t: S_t = Q_t K_j^T (128x128x128) into
//               TMEM, O_t += P_t V_j (128x128x128) with P_t read straight from
//               TMEM (bf16 pairs packed into S_t's own columns).  The two
//               tiles ping-pong: S_1 / PV_0 run while softmax 0 / 1 work.
//   warps 4-7   softmax of tile 0, warps 8-11 of tile 1, one thread per query
//               row (TMEM lane).  O stays in TMEM; it is rescaled in place
//               only when a row max grows by more than 2^8 (lazy rescale: the
//               P values stay <= 256, exact in the final O / l).
//   TMEM: tile t owns columns [256 t, 256 t + 128) for S / P and
//   [256 t + 128, 256 t + 256) for O -- all 512.
//
// Backward (bwd_kernel: one CTA per (sample, head, 128-key block), looping
// over 64-query sub-blocks):
//   S^T  = K Q^T,  dP^T = V dO^T       (128 keys x 64 queries each)
//   P^T  = exp2(S^T c - lse),  dS^T = P^T (dP^T - D)   (bf16 -> smem)
//   dV  += P^T dO,  dK += dS^T Q       (128 keys x 128 dims, TMEM-resident)
//   dQ^T = K^T dS^T                    (128 dims x 64 queries, double-buffered)
// dQ is produced transposed (head dims on the TMEM lanes) so that with the
// 64-query sub-block all five accumulators fit in 512 columns:
// S^T 64 | dP^T 64 | dV 128 | dK 128 | dQ^T 2 x 64.  The softmax warps stage
// dQ (scaled) row-major in shared memory and one TMA reduce-add per sub-block
// adds it into the fp32 dq_acc (converted to bf16 by attention.cu's dq_convert).
//
// Outputs match attention.cu's conventions: o [tokens, d] bf16, lse
// [tokens, H] in the log2 domain, dqkv [tokens, 3d] bf16.
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>
#include <type_traits>

#include "../runtime/common.hpp"
#include "pdl.cuh"
#include "sm100.cuh"

namespace hm {
namespace attn_tc128 {

using namespace sm100;

constexpr int DH = 128, BQ = 128, BKV = 128, SUBQ = 64;
constexpr uint32_t kAtom = 128 * 128;      // 128 rows x 128 B (64 head dims) SW128 box: 16 KB
constexpr uint32_t kTile = 2 * kAtom;      // 128 rows x 128 head dims: 32 KB
constexpr uint32_t kSubAtom = SUBQ * 128;  // 64 rows x 128 B: 8 KB
constexpr uint32_t kSubTile = 2 * kSubAtom;
constexpr uint32_t kPT = BKV * 128;        // P^T / dS^T: 128 keys x 64 queries bf16: 16 KB
constexpr uint32_t kDqStage = SUBQ * DH * 4;  // dQ of one sub-block, fp32 row-major: 32 KB
constexpr int kThreads = 384;              // TMA, MMA, TMEM-alloc, idle, 2 x 4 softmax warps
constexpr float kRescaleLog2 = 8.f;        // lazy-rescale threshold (log2 units)

template <int HD>
constexpr size_t fwd_smem() { return 1024 + 6 * (size_t)HD * 256 /*Q x2 tiles, K x2, V x2*/ + 256; }
constexpr size_t kFwdSmem = fwd_smem<128>();
constexpr size_t kBwdSmem = 1024 + 2 * kTile /*K, V*/ + 4 * kSubTile /*Q, dO x2*/ + 2 * kPT /*P^T, dS^T*/ +
                            kDqStage + 2 * 2 * SUBQ * 4 /*lse, D x2*/ + 512;
static_assert(kFwdSmem <= 232448 && kBwdSmem <= 232448, "shared memory");

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------------
// forward (HD = 128; HD = 64 is the same dataflow with one SW128 atom per
// tile and O in 64 TMEM columns -- selectable for head_dim 64 with
// HM_ATTN_FWD=t, see attention_tc.cu)
// ---------------------------------------------------------------------------
template <int HD, bool CAUSAL>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo, float *__restrict__ lse,
               int S, int H, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  constexpr uint32_t TILE = HD * 256;  // 128 rows x HD head dims bf16 (HD / 64 SW128 atoms)
  constexpr int DH = HD;
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sQ = smem;              // [2 tiles]
  uint8_t *sK = sQ + 2 * TILE;    // [2 stages]
  uint8_t *sV = sK + 2 * TILE;    // [2 stages]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sV + 2 * TILE);
  uint64_t *q_full = bar;
  uint64_t *kv_full = bar + 1, *kv_empty = bar + 3;
  uint64_t *s_full = bar + 5, *p_full = bar + 7, *o_full = bar + 9;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 11);

  const int nq = S / BQ, npair = (nq + 1) >> 1;
  // blockIdx.x (fastest in launch order) walks the heads, blockIdx.y the
  // pairs: every head's heaviest causal pair launches before any lighter one
  const int pr = CAUSAL ? npair - 1 - (int)blockIdx.y : (int)blockIdx.y;
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int qb0 = 2 * pr;
  const bool has1 = qb0 + 1 < nq;
  const int nkv0 = CAUSAL ? qb0 + 1 : S / BKV;
  const int nkv1 = has1 ? (CAUSAL ? qb0 + 2 : S / BKV) : 0;
  const int nkv_all = nkv0 > nkv1 ? nkv0 : nkv1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = b * S;
  constexpr uint32_t C_S = 0, C_O = 128;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // programmatic dependent launch: set-up above overlapped the previous kernel

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, (has1 ? 2 : 1) * TILE);
      for (int t = 0; t < (has1 ? 2 : 1); ++t)
        for (int a = 0; a < DH / 64; ++a)
          tma_load_2d(sQ + t * TILE + a * kAtom, &tm, q_full, h * DH + 64 * a, row0 + (qb0 + t) * BQ);
      for (int j = 0; j < nkv_all; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * TILE);
        for (int a = 0; a < DH / 64; ++a) {
          tma_load_2d(sK + st * TILE + a * kAtom, &tm, &kv_full[st], d + h * DH + 64 * a, row0 + j * BKV);
          tma_load_2d(sV + st * TILE + a * kAtom, &tm, &kv_full[st], 2 * d + h * DH + 64 * a, row0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(BQ, BKV, 0, 0);  // Q K-major, K K-major
      constexpr uint32_t idesc_o = idesc_bf16_f32(BQ, DH, 0, 1);   // P (TMEM), V MN-major
      const int nkv[2] = {nkv0, nkv1};
      mbar_wait(q_full, 0);
      auto issue_s = [&](int t, int j) {
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ + t * TILE), k_base = smem_u32(sK + (j & 1) * TILE);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_bf16(tmem + t * 256 + C_S, umma_desc_sw128(q_base + off, 16, 1024),
                   umma_desc_sw128(k_base + off, 16, 1024), idesc_s, kk > 0);
        }
        mma_commit(&s_full[t]);
      };
      auto issue_o = [&](int t, int j) {
        mbar_wait(&p_full[t], j & 1);  // P_t(j) packed and O_t rescaled
        tc_fence_after();
        const uint32_t v_base = smem_u32(sV + (j & 1) * TILE);
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_bf16_ts(tmem + t * 256 + C_O, tmem + t * 256 + C_S + kk * 8,
                      umma_desc_sw128(v_base + kk * 2048, kAtom, 1024), idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&o_full[t]);
      };
      mbar_wait(&kv_full[0], 0);
      for (int t = 0; t < 2; ++t)
        if (nkv[t] > 0) issue_s(t, 0);
      for (int j = 0; j < nkv_all; ++j) {
        bool next_ready = false;
        for (int t = 0; t < 2; ++t) {
          if (j >= nkv[t]) continue;
          issue_o(t, j);
          // S_t(j+1) overwrites P_t(j) in TMEM: tcgen05.mma executes in
          // issue order, so PV_t(j) has read it by then
          if (j + 1 < nkv[t]) {
            if (!next_ready) {
              mbar_wait(&kv_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
              next_ready = true;
            }
            issue_s(t, j + 1);
          }
        }
        mma_commit(&kv_empty[j & 1]);
      }
    }
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;
    const int nkv = t == 0 ? nkv0 : nkv1;
    if (nkv > 0) {
      const int q4 = warp & 3;
      const int r = q4 * 32 + lane;  // query row inside the tile == TMEM lane
      const int qb = qb0 + t;
      const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
      const uint32_t s_addr = tmem + lane_addr + t * 256 + C_S, o_addr = tmem + lane_addr + t * 256 + C_O;
      float m = -INFINITY, l = 0.f;  // m: the max the exponents are taken against (log2 domain)
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&s_full[t], j & 1);
        tc_fence_after();
        const bool diag = CAUSAL && j == qb;
        float mx = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < BKV; c0 += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(s_addr + c0, v);
          tmem_ld_wait();
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float x = (diag && c0 + c > r) ? -INFINITY : __uint_as_float(v[c]);
            m4[c & 3] = fmaxf(m4[c & 3], x);
          }
          mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
        }
        const float m_row = mx * scale_log2;
        float alpha = 1.f;
        if (m_row > m + kRescaleLog2) {  // first tile (m = -inf) always lands here
          alpha = ex2(m - m_row);
          m = m_row;
        }
        if (j > 0) {
          // PV_t(j-1) completed before S_t(j) (in-order MMAs): O_t is final for j-1
          mbar_wait(&o_full[t], (j - 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {  // warp-uniform: tcgen05.ld / st are .sync.aligned
#pragma unroll
            for (int c0 = 0; c0 < DH; c0 += 32) {
              uint32_t ov[32];
              tmem_ld_32x32b_x32(o_addr + c0, ov);
              tmem_ld_wait();
#pragma unroll
              for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha);
              tmem_st_32x32b_x32(o_addr + c0, ov);
            }
          }
        }
        float rs4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c0 = 0; c0 < BKV; c0 += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(s_addr + c0, v);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            float p0 = ex2(fmaf(__uint_as_float(v[c]), scale_log2, -m));
            float p1 = ex2(fmaf(__uint_as_float(v[c + 1]), scale_log2, -m));
            if (diag && c0 + c > r) p0 = 0.f;
            if (diag && c0 + c + 1 > r) p1 = 0.f;
            rs4[(c >> 1) & 3] += p0 + p1;
            __nv_bfloat162 tb = __floats2bfloat162_rn(p0, p1);
            pk[c >> 1] = *reinterpret_cast<uint32_t *>(&tb);
          }
          // keys c0..c0+31 -> P columns c0/2..c0/2+15 (S columns already read)
          tmem_st_32x32b_x16(s_addr + (c0 >> 1), pk);
        }
        tmem_st_wait();
        l = l * alpha + ((rs4[0] + rs4[1]) + (rs4[2] + rs4[3]));
        tc_fence_before();
        mbar_arrive(&p_full[t]);
      }
      mbar_wait(&o_full[t], (nkv - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      // O leaves as TMA stores (one per 64 head dims) from this tile's Q
      // buffer, free once its last PV has completed (every S MMA of the tile
      // was issued before it): rows are d apart in `out`, and 16-B stores from
      // every thread throttle the LSU
      uint8_t *srow = sQ + t * TILE + r * 128;
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t ov[32];
        tmem_ld_32x32b_x32(o_addr + c0, ov);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          uint4 w;
          uint32_t *wp = reinterpret_cast<uint32_t *>(&w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 tb = __floats2bfloat162_rn(__uint_as_float(ov[c + 2 * e]) * inv,
                                                      __uint_as_float(ov[c + 2 * e + 1]) * inv);
            wp[e] = *reinterpret_cast<uint32_t *>(&tb);
          }
          const int col = c0 + c;
          *reinterpret_cast<uint4 *>(srow + (col >> 6) * kAtom + ((((col & 63) >> 3) ^ (r & 7)) << 4)) = w;
        }
      }
      fence_async_smem();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
      if (q4 == 0 && lane == 0) {
#pragma unroll
        for (int a = 0; a < DH / 64; ++a) tma_store_2d(&tmo, sQ + t * TILE + a * kAtom, h * DH + 64 * a, row0 + qb * BQ);
        bulk_commit();
        bulk_wait0();  // shared memory is released when the CTA exits
      }
      lse[(int64_t)(row0 + qb * BQ + r) * H + h] = m + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
template <bool CAUSAL>
__global__ void __launch_bounds__(kThreads, 1)
    bwd_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
               const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
               const __grid_constant__ CUtensorMap tm_dkv, const float *__restrict__ lse,
               const float *__restrict__ dvec, int S, int H, float scale_log2, float scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sK = smem;
  uint8_t *sV = sK + kTile;
  uint8_t *sQ = sV + kTile;            // [2] stages of 64 queries
  uint8_t *sdO = sQ + 2 * kSubTile;    // [2] stages
  uint8_t *sP = sdO + 2 * kSubTile;    // P^T  [128 keys x 64 queries]
  uint8_t *sdS = sP + kPT;             // dS^T
  float *sDQ = reinterpret_cast<float *>(sdS + kPT);  // [64 queries][128 dims] fp32
  float *sL = sDQ + SUBQ * DH;         // [2][64] lse
  float *sD = sL + 2 * SUBQ;           // [2][64] D
  uint64_t *bar = reinterpret_cast<uint64_t *>(sD + 2 * SUBQ);
  uint64_t *kv_full = bar;
  uint64_t *q_full = bar + 1, *q_empty = bar + 3;
  uint64_t *st_full = bar + 5, *st_empty = bar + 6;
  uint64_t *p_full = bar + 7, *p_empty = bar + 8;
  uint64_t *dq_empty = bar + 11, *acc_full = bar + 13;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 14);

  const int nq = S / SUBQ;
  const int kb = blockIdx.y;  // heads fastest: the heavy causal key blocks (small kb) launch first
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int q_begin = CAUSAL ? kb * (BKV / SUBQ) : 0;
  const int count = nq - q_begin;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = b * S;
  constexpr uint32_t C_ST = 0, C_DP = 64, C_DV = 128, C_DK = 256, C_DQ = 384;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&dq_empty[i], 256);
    }
    mbar_init(st_full, 1);
    mbar_init(st_empty, 256);
    mbar_init(p_full, 256);
    mbar_init(p_empty, 1);
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // programmatic dependent launch: set-up above overlapped the previous kernel

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * kTile);
      for (int a = 0; a < 2; ++a) {
        tma_load_2d(sK + a * kAtom, &tm_kv, kv_full, d + h * DH + 64 * a, row0 + kb * BKV);
        tma_load_2d(sV + a * kAtom, &tm_kv, kv_full, 2 * d + h * DH + 64 * a, row0 + kb * BKV);
      }
      for (int i = q_begin, n = 0; i < nq; ++i, ++n) {
        const int st = n & 1;
        mbar_wait(&q_empty[st], ((n >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[st], 2 * kSubTile);
        for (int a = 0; a < 2; ++a) {
          tma_load_2d(sQ + st * kSubTile + a * kSubAtom, &tm_q, &q_full[st], h * DH + 64 * a, row0 + i * SUBQ);
          tma_load_2d(sdO + st * kSubTile + a * kSubAtom, &tm_do, &q_full[st], h * DH + 64 * a, row0 + i * SUBQ);
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // two issuing threads (see attention_fwd64.cu / attention_tc.cu): warp 2
    // issues S^T / dP^T, warp 1 the gradient MMAs; the softmax orders them
    if (lane == 0) {
      constexpr uint32_t id_st = idesc_bf16_f32(BKV, SUBQ, 0, 0);  // S^T, dP^T: K-major x K-major
      constexpr uint32_t id_acc = idesc_bf16_f32(BKV, DH, 0, 1);   // dV, dK: A K-major, B MN-major
      constexpr uint32_t id_dq = idesc_bf16_f32(DH, SUBQ, 1, 1);   // dQ^T: A = K^T MN-major, B = dS^T MN-major
      mbar_wait(kv_full, 0);
      const uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);
      const uint32_t p_base = smem_u32(sP), ds_base = smem_u32(sdS);
      auto issue_st = [&](int n) {
        const int st = n & 1;
        mbar_wait(&q_full[st], (n >> 1) & 1);
        mbar_wait(st_empty, (n & 1) ^ 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ + st * kSubTile), do_base = smem_u32(sdO + st * kSubTile);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {  // reduction over the head dims
          const uint32_t a_off = (kk >> 2) * kAtom + (kk & 3) * 32;
          const uint32_t b_off = (kk >> 2) * kSubAtom + (kk & 3) * 32;
          mma_bf16(tmem + C_ST, umma_desc_sw128(k_base + a_off, 16, 1024), umma_desc_sw128(q_base + b_off, 16, 1024),
                   id_st, kk > 0);
          mma_bf16(tmem + C_DP, umma_desc_sw128(v_base + a_off, 16, 1024), umma_desc_sw128(do_base + b_off, 16, 1024),
                   id_st, kk > 0);
        }
        mma_commit(st_full);
      };
      if (warp == 2) {
        for (int n = 0; n < count; ++n) issue_st(n);
      } else {
        for (int n = 0; n < count; ++n) {
          const int st = n & 1;
          const uint32_t ph = n & 1;
          const uint32_t q_base = smem_u32(sQ + st * kSubTile), do_base = smem_u32(sdO + st * kSubTile);
          mbar_wait(p_full, ph);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < SUBQ / 16; ++kk) {  // reduction over the 64 queries
            const uint32_t acc = (n > 0 || kk > 0) ? 1u : 0u;
            mma_bf16(tmem + C_DV, umma_desc_sw128(p_base + kk * 32, 16, 1024),
                     umma_desc_sw128(do_base + kk * 2048, kSubAtom, 1024), id_acc, acc);
            mma_bf16(tmem + C_DK, umma_desc_sw128(ds_base + kk * 32, 16, 1024),
                     umma_desc_sw128(q_base + kk * 2048, kSubAtom, 1024), id_acc, acc);
          }
          const int qb = n & 1;
          mbar_wait(&dq_empty[qb], ((n >> 1) & 1) ^ 1);  // dQ^T of sub-block n-2 has left this buffer
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)  // reduction over the 128 keys
            mma_bf16(tmem + C_DQ + qb * SUBQ, umma_desc_sw128(k_base + kk * 2048, kAtom, 1024),
                     umma_desc_sw128(ds_base + kk * 2048, kPT, 1024), id_dq, kk > 0);
          // one commit publishes dQ^T(n) and frees sub-block n's Q / dO stage
          // (S^T / dP^T(n), the other thread's readers, completed before p_full(n))
          mma_commit(&q_empty[st]);
          mma_commit(p_empty);
        }
        mma_commit(acc_full);
      }
    }
  } else if (warp >= 4) {
    // two warpgroups on the same TMEM lanes: warpgroup wg owns queries
    // [32 wg, 32 wg + 32) of every sub-block, and dV (wg 0) or dK (wg 1) at the end
    const int wg = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;  // key row (S^T, dP^T, dV, dK) / head dim (dQ^T) == TMEM lane
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    const float *src = wg == 0 ? lse : dvec;
    float *dst = wg == 0 ? sL : sD;
    float x_next = r < SUBQ ? src[(int64_t)(row0 + q_begin * SUBQ + r) * H + h] : 0.f;
    // dQ^T of sub-block nn (query sub-block qblk): TMEM -> smem [query][dim]
    // (consecutive lanes write consecutive words: conflict-free) -> one TMA
    // reduce-add of the 64 x 128 fp32 tile
    auto dq_out = [&](int qblk, int nn) {
      const int qb = nn & 1;
      mbar_wait(&q_empty[qb], (nn >> 1) & 1);  // sub-block nn's gradient MMAs (dQ^T included) retired
      tc_fence_after();
      uint32_t q[32];
      tmem_ld_32x32b_x32(tmem + lane_addr + C_DQ + qb * SUBQ + wg * 32, q);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&dq_empty[qb]);
      if (wg == 0 && r == 0) bulk_wait_read0();  // the previous reduce has read the stage
      asm volatile("bar.sync 2, 256;" ::: "memory");
#pragma unroll
      for (int c = 0; c < 32; ++c) sDQ[(wg * 32 + c) * DH + r] = __uint_as_float(q[c]) * scale;
      fence_async_smem();
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (wg == 0 && r == 0) {
        tma_reduce_add_2d(&tm_dq, sDQ, h * DH, row0 + qblk * SUBQ);
        bulk_commit();
      }
    };
    uint8_t *prow = sP + r * 128;
    uint8_t *dsrow = sdS + r * 128;
    const int key = kb * BKV + r;
    for (int i = q_begin, n = 0; i < nq; ++i, ++n) {
      const int st = n & 1;
      const uint32_t ph = n & 1;
      if (r < SUBQ) {
        dst[st * SUBQ + r] = x_next;
        if (i + 1 < nq) x_next = src[(int64_t)(row0 + (i + 1) * SUBQ + r) * H + h];
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mbar_wait(st_full, ph);
      tc_fence_after();
      // sub-blocks that straddle the diagonal (queries < this key are masked)
      const bool diag = CAUSAL && i * SUBQ < (kb + 1) * BKV;
      const float *Ls = sL + st * SUBQ;
      const float *Ds = sD + st * SUBQ;
      uint32_t sv[32], dp[32];
      tmem_ld_32x32b_x32(tmem + lane_addr + C_ST + wg * 32, sv);
      tmem_ld_32x32b_x32(tmem + lane_addr + C_DP + wg * 32, dp);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(st_empty);  // S^T / dP^T read: the next sub-block's MMAs may overwrite
      uint32_t pk[16], dk[16];
      auto elementwise = [&](auto diag_tag) {
        constexpr bool DIAG = decltype(diag_tag)::value;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          const int qi = wg * 32 + c;
          const float4 L4 = *reinterpret_cast<const float4 *>(Ls + qi);
          const float4 D4 = *reinterpret_cast<const float4 *>(Ds + qi);
          const float lq[4] = {L4.x, L4.y, L4.z, L4.w}, dq4[4] = {D4.x, D4.y, D4.z, D4.w};
          float p[4], g[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            p[k] = ex2(fmaf(__uint_as_float(sv[c + k]), scale_log2, -lq[k]));
            if (DIAG && i * SUBQ + qi + k < key) p[k] = 0.f;  // query < key: masked
            g[k] = p[k] * (__uint_as_float(dp[c + k]) - dq4[k]);
          }
          __nv_bfloat162 tp0 = __floats2bfloat162_rn(p[0], p[1]), tp1 = __floats2bfloat162_rn(p[2], p[3]);
          __nv_bfloat162 td0 = __floats2bfloat162_rn(g[0], g[1]), td1 = __floats2bfloat162_rn(g[2], g[3]);
          pk[c >> 1] = *reinterpret_cast<uint32_t *>(&tp0);
          pk[(c >> 1) + 1] = *reinterpret_cast<uint32_t *>(&tp1);
          dk[c >> 1] = *reinterpret_cast<uint32_t *>(&td0);
          dk[(c >> 1) + 1] = *reinterpret_cast<uint32_t *>(&td1);
        }
      };
      if (diag) elementwise(std::true_type{});
      else elementwise(std::false_type{});
      mbar_wait(p_empty, ph ^ 1);  // the previous sub-block's MMAs have consumed P^T / dS^T
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t off = (((wg * 4) + ch) ^ (r & 7)) << 4;
        *reinterpret_cast<uint4 *>(prow + off) = make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
        *reinterpret_cast<uint4 *>(dsrow + off) = make_uint4(dk[4 * ch], dk[4 * ch + 1], dk[4 * ch + 2], dk[4 * ch + 3]);
      }
      fence_async_smem();
      mbar_arrive(p_full);
      // the previous sub-block's dQ^T: drained while this sub-block's gradient MMAs run
      if (n > 0) dq_out(i - 1, n - 1);
    }
    dq_out(nq - 1, count - 1);
    if (wg == 0 && r == 0) bulk_wait0();
    mbar_wait(acc_full, 0);
    tc_fence_after();
    // dV (warpgroup 0) / dK (warpgroup 1) staged in SW128 atoms in the (spent)
    // V / K buffers and stored by TMA: rows are 3d apart in dqkv, and 16-B
    // stores from every thread throttle the LSU at the end of every CTA
    const float osc = wg == 0 ? 1.f : scale;
    const uint32_t acc_addr = tmem + lane_addr + (wg == 0 ? C_DV : C_DK);
    uint8_t *stage = wg == 0 ? sV : sK;
    uint8_t *srow = stage + r * 128;
#pragma unroll
    for (int c0 = 0; c0 < DH; c0 += 32) {
      uint32_t acc[32];
      tmem_ld_32x32b_x32(acc_addr + c0, acc);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        uint4 w;
        uint32_t *pw = reinterpret_cast<uint32_t *>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 a = __floats2bfloat162_rn(__uint_as_float(acc[c + 2 * e]) * osc,
                                                   __uint_as_float(acc[c + 2 * e + 1]) * osc);
          pw[e] = *reinterpret_cast<uint32_t *>(&a);
        }
        const int col = c0 + c;
        *reinterpret_cast<uint4 *>(srow + (col >> 6) * kAtom + ((((col & 63) >> 3) ^ (r & 7)) << 4)) = w;
      }
    }
    fence_async_smem();
    asm volatile("bar.sync %0, 128;" ::"r"(3 + wg) : "memory");
    if (r == 0) {
#pragma unroll
      for (int a = 0; a < DH / 64; ++a)
        tma_store_2d(&tm_dkv, stage + a * kAtom, (wg == 0 ? 2 * d : d) + h * DH + 64 * a, row0 + kb * BKV);
      bulk_commit();
      bulk_wait0();  // shared memory is released when the CTA exits
    }
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

// bf16 [rows, inner] (row pitch in bytes), {64, box_rows} boxes, 128-B swizzle
static int make_map(CUtensorMap *tm, const void *base, int64_t inner, int64_t rows, int64_t pitch_bytes,
                    uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  if (fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(HM_ERR_DEVICE, "attention (head_dim 128) tensor map encode failed");
  return HM_OK;
}

bool supported(int S, int DHx) { return DHx == DH && S % BQ == 0; }

template <int HD>
static int forward_hd(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s) {
  const int d = H * HD;
  CUtensorMap tm;
  HM_TRY(make_map(&tm, qkv, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2, 128));
  CUtensorMap tmo;  // out [B*S, d] bf16, {64, 128} SW128 boxes (TMA-stored O)
  HM_TRY(make_map(&tmo, o, d, (int64_t)B * S, (int64_t)d * 2, 128));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  ProfScope ps(KC_ATTN_FWD, s, 4.0 * B * (double)S * S * H * HD * (causal ? 0.5 : 1.0), (double)B * S * H * HD * 2 * 4);
  static bool attr[2] = {false, false};
  auto k = causal ? fwd_kernel<HD, true> : fwd_kernel<HD, false>;
  if (!attr[causal ? 1 : 0]) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem<HD>()));
    attr[causal ? 1 : 0] = true;
  }
  const int npair = (S / BQ + 1) / 2;
  HM_CUDA(launch_pdl(k, dim3(B * H, npair), dim3(kThreads), fwd_smem<HD>(), s, tm, tmo, lse, S, H, scale_log2));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s) {
  return forward_hd<128>(qkv, o, lse, B, S, H, causal, s);
}

// head_dim 64 through the same kernel (attention_tc.cu dispatches it on HM_ATTN_FWD=t)
int forward64(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s) {
  return forward_hd<64>(qkv, o, lse, B, S, H, causal, s);
}

// dq_acc must be zeroed by the caller; it receives scale * dS K (fp32)
int backward_main(const void *qkv, const void *dout, const float *lse, const float *dvec, float *dq_acc, void *dqkv,
                  int B, int S, int H, int causal, cudaStream_t s) {
  const int d = H * DH;
  CUtensorMap tkv, tq, tdo, tdq;
  HM_TRY(make_map(&tkv, qkv, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2, BKV));
  HM_TRY(make_map(&tq, qkv, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2, SUBQ));
  HM_TRY(make_map(&tdo, dout, d, (int64_t)B * S, (int64_t)d * 2, SUBQ));
  CUtensorMap tdkv;  // dqkv [B*S, 3d] bf16, {64, 128} SW128 boxes: TMA-stored dK / dV
  HM_TRY(make_map(&tdkv, dqkv, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2, BKV));
  {  // dq_acc [B*S, d] fp32, {128, 64} boxes, no swizzle (row-major smem stage)
    EncodeFn fn = encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)B * S};
    cuuint64_t strides[1] = {(cuuint64_t)d * 4};
    cuuint32_t box[2] = {DH, SUBQ};
    cuuint32_t estr[2] = {1, 1};
    if (!fn || fn(&tdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq_acc, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(HM_ERR_DEVICE, "attention (head_dim 128) dQ tensor map encode failed");
  }
  static bool attr[2] = {false, false};
  auto k = causal ? bwd_kernel<true> : bwd_kernel<false>;
  if (!attr[causal ? 1 : 0]) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem));
    attr[causal ? 1 : 0] = true;
  }
  const float scale = 1.f / sqrtf((float)DH);
  HM_CUDA(launch_pdl(k, dim3(B * H, S / BKV), dim3(kThreads), kBwdSmem, s, tkv, tq, tdo, tdq, tdkv, lse, dvec, S, H,
                     1.4426950408889634f * scale, scale));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

}  // namespace attn_tc128
}  // namespace hm
