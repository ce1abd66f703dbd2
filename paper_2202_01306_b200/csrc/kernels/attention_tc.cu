// attention_tc.cu -- flash attention (head_dim 64) on the 5th-gen tensor cores:
// the backward, and the persistent query-block-pair forward (HM_ATTN_FWD=q;
// the default forward is attention_fwd64.cu).
//
// fwd2p_kernel (one CTA per SM walking a list of query-block pairs):
//   warp 0      TMA: the pair's Q tiles (double-buffered per item), then
//               K_j / V_j tiles (128 keys) into a 2-stage ring
//   warp 1      MMA issuer: S = Q K_j^T (128x128x64) into TMEM per tile,
//               O = P V_j (128x64x128) into TMEM per tile
//   warps 4-11  two softmax warpgroups (one per query tile), one thread per
//               query row (TMEM lane): the S row from TMEM, online max /
//               exp2 / sum in registers, P (bf16) into 128B-swizzled smem as
//               the PV MMA's A operand, O accumulated in registers one tile
//               behind with the running rescale
// Backward: bwd_kernel (one CTA per 128-key block, two softmax warpgroups, dQ
// by TMA reduce-add).
// Output o [tokens, d] bf16 and lse [tokens, H] (log2 domain) exactly as the
// mma.sync kernel (attention.cu), which stays the fallback for sequence
// lengths that are not a multiple of 128 (head_dim 128: attention_tc128.cu).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <mutex>
#include <type_traits>

#include "../runtime/common.hpp"
#include "pdl.cuh"
#include "sm100.cuh"

namespace hm {
namespace attn_fwd64 {  // attention_fwd64.cu
int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s);
}  // namespace attn_fwd64
namespace attn_tc128 {  // attention_tc128.cu
bool supported(int S, int DH);
int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s);
int forward64(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s);
}  // namespace attn_tc128
namespace attn_tc {

using namespace sm100;

constexpr int BQ = 128, BKV = 128, DH = 64;
constexpr int kThreads2 = 384;  // TMA, MMA, TMEM-alloc, idle, 2 x 4 softmax / elementwise warps
constexpr uint32_t kTileBytes = BKV * DH * 2;  // 16 KB: 128 rows x 128 B
constexpr uint32_t kPBytes = BQ * BKV * 2;     // 32 KB: two 64-key swizzle atoms

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }


// ---------------------------------------------------------------------------
// forward, persistent with two query tiles per item: softmax warpgroups A and
// B share every K/V tile, and the MMA thread interleaves them (S_A(j+1) is
// issued while softmax B works on S_B(j) and vice versa).  An item is the query-block pair
// (2p, 2p+1) of one (sample, head): under causal masking the two tiles sweep
// 2p+1 and 2p+2 K/V tiles, so the pair stays balanced, and the item list is
// ordered heaviest first, so the persistent CTAs finish together.  The causal
// mask is a separate instantiation of the tile body (only the diagonal tile
// pays for it).  Q is double-buffered per item.
// ---------------------------------------------------------------------------
constexpr size_t kSmem2P = 1024 + 4 * kTileBytes /*Q pair x2*/ + 4 * kTileBytes /*K, V x2*/ + 2 * kPBytes + 512;

template <bool CAUSAL>
__global__ void __launch_bounds__(kThreads2, 1)
    fwd2p_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16 *__restrict__ out, float *__restrict__ lse,
                 int S, int H, int BH, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared address space (STS / LDS, not generic ST / LD)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sQ = smem;                   // [2 items][2 tiles]
  uint8_t *sK = sQ + 4 * kTileBytes;    // [2] stages
  uint8_t *sV = sK + 2 * kTileBytes;    // [2] stages
  uint8_t *sP = sV + 2 * kTileBytes;    // [2] tiles
  uint64_t *bar = reinterpret_cast<uint64_t *>(sP + 2 * kPBytes);
  uint64_t *q_full = bar, *q_empty = bar + 2;        // [item stage]
  uint64_t *kv_full = bar + 4, *kv_empty = bar + 6;  // [kv stage]
  uint64_t *s_full = bar + 8, *s_empty = bar + 10;   // [tile]
  uint64_t *p_full = bar + 12, *p_empty = bar + 14;  // [tile]
  uint64_t *o_full = bar + 16, *o_empty = bar + 18;  // [tile]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 20);

  const int nq = S / BQ, np = nq / 2, n_items = np * BH;
  const int d = H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t C_S = 0, C_O = 2 * BKV;  // TMEM: S_A, S_B | O_A, O_B
  auto item = [&](int i, int &bh, int &p) {
    if (CAUSAL) {
      p = np - 1 - i / BH;
      bh = i % BH;
    } else {
      p = i % np;
      bh = i / np;
    }
  };
  auto nkv_of = [&](int qb) { return CAUSAL ? qb + 1 : nq; };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 128);
      mbar_init(&p_full[i], 128);
      mbar_init(&p_empty[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, it = 0;
      for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++it) {
        int bh, p;
        item(i, bh, p);
        const int b = bh / H, h = bh % H, row0 = b * S;
        const int qs = it & 1;
        mbar_wait(&q_empty[qs], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[qs], 2 * kTileBytes);
        tma_load_2d(sQ + (2 * qs) * kTileBytes, &tm, &q_full[qs], h * DH, row0 + (2 * p) * BQ);
        tma_load_2d(sQ + (2 * qs + 1) * kTileBytes, &tm, &q_full[qs], h * DH, row0 + (2 * p + 1) * BQ);
        const int nkv = nkv_of(2 * p + 1);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int st = g & 1;
          mbar_wait(&kv_empty[st], ((g >> 1) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], 2 * kTileBytes);
          tma_load_2d(sK + st * kTileBytes, &tm, &kv_full[st], d + h * DH, row0 + j * BKV);
          tma_load_2d(sV + st * kTileBytes, &tm, &kv_full[st], 2 * d + h * DH, row0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(BQ, BKV, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_f32(BQ, DH, 0, 1);
      int g0 = 0, it = 0;
      int cs[2] = {0, 0}, cp[2] = {0, 0};  // S issues / PV issues per tile
      for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++it) {
        int bh, p;
        item(i, bh, p);
        const int nkv_a = nkv_of(2 * p), nkv_b = nkv_of(2 * p + 1);
        const int qs = it & 1;
        mbar_wait(&q_full[qs], (it >> 1) & 1);
        auto issue_s = [&](int t, int j) {  // S_t(j) = Q_t K_j^T
          const int gj = g0 + j, st = gj & 1;
          if (t == 0) mbar_wait(&kv_full[st], (gj >> 1) & 1);
          mbar_wait(&s_empty[t], (cs[t] & 1) ^ 1);
          tc_fence_after();
          const uint32_t q_base = smem_u32(sQ + (2 * qs + t) * kTileBytes), k_base = smem_u32(sK + st * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            mma_bf16(tmem + C_S + t * BKV, umma_desc_sw128(q_base + kk * 32, 16, 1024),
                     umma_desc_sw128(k_base + kk * 32, 16, 1024), idesc_s, kk > 0);
          mma_commit(&s_full[t]);
          ++cs[t];
        };
        auto issue_pv = [&](int t, int j) {  // O_t(j) = P_t(j) V_j
          const int st = (g0 + j) & 1;
          mbar_wait(&p_full[t], cp[t] & 1);
          mbar_wait(&o_empty[t], (cp[t] & 1) ^ 1);
          tc_fence_after();
          const uint32_t p_base = smem_u32(sP + t * kPBytes), v_base = smem_u32(sV + st * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            mma_bf16(tmem + C_O + t * DH, umma_desc_sw128(p_base + (kk >> 2) * (BQ * 128) + (kk & 3) * 32, 16, 1024),
                     umma_desc_sw128(v_base + kk * 2048, BKV * 128, 1024), idesc_o, kk > 0);
          mma_commit(&o_full[t]);
          mma_commit(&p_empty[t]);
          ++cp[t];
        };
        issue_s(0, 0);
        issue_s(1, 0);
        for (int j = 0; j < nkv_b; ++j) {
          if (j < nkv_a) {
            issue_pv(0, j);
            if (j + 1 < nkv_a) issue_s(0, j + 1);
          }
          issue_pv(1, j);
          mma_commit(&kv_empty[(g0 + j) & 1]);
          if (j + 1 < nkv_b) {
            if (!(j + 1 < nkv_a)) mbar_wait(&kv_full[(g0 + j + 1) & 1], ((g0 + j + 1) >> 1) & 1);
            issue_s(1, j + 1);
          }
        }
        mma_commit(&q_empty[qs]);  // every Q K^T of this item issued: Q pair free once they retire
        g0 += nkv_b;
      }
    }
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;  // query tile: 0 = A (2p), 1 = B (2p+1)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const uint32_t s_addr = tmem + lane_addr + C_S + t * BKV;
    int n = 0;  // tiles this warpgroup has processed (buffer parities)
    for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
      int bh, p;
      item(i, bh, p);
      const int b = bh / H, h = bh % H, row0 = b * S;
      const int qb = 2 * p + t;
      const int nkv = nkv_of(qb);
      float o[DH];
#pragma unroll
      for (int c = 0; c < DH; ++c) o[c] = 0.f;
      float m = -INFINITY, l = 0.f, alpha_prev = 1.f;
      auto add_o = [&](int nn, float alpha) {
        mbar_wait(&o_full[t], nn & 1);
        tc_fence_after();
        uint32_t v[DH];
#pragma unroll
        for (int c0 = 0; c0 < DH; c0 += 32)
          tmem_ld_32x32b_x32(tmem + lane_addr + C_O + t * DH + c0, *reinterpret_cast<uint32_t(*)[32]>(v + c0));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&o_empty[t]);
#pragma unroll
        for (int c = 0; c < DH; ++c) o[c] = o[c] * alpha + __uint_as_float(v[c]);
      };
      // one K/V tile: row max (pass 1), exp / row sum / bf16 P (pass 2), the S
      // row read from TMEM in CH-column pieces (CH / 32 loads in flight per wait)
      auto tile = [&](auto diag_tag) -> float {
        constexpr bool DIAG = decltype(diag_tag)::value;
        // 64-column halves (1135 vs 1220 ns per tile at s = 1024, full attention);
        // the masked diagonal tile reads 32-column quarters
        constexpr int CH = DIAG ? 32 : 64;
        float mx = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < BKV; c0 += CH) {
          uint32_t v[CH];
#pragma unroll
          for (int q0 = 0; q0 < CH; q0 += 32)
            tmem_ld_32x32b_x32(s_addr + c0 + q0, *reinterpret_cast<uint32_t(*)[32]>(v + q0));
          tmem_ld_wait();
          float m8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) m8[e] = -INFINITY;
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            const float x = (DIAG && c0 + c > r) ? -INFINITY : __uint_as_float(v[c]);
            m8[c & 7] = fmaxf(m8[c & 7], x);
          }
          mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                                fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))));
        }
        const float m_new = fmaxf(m, mx * scale_log2);
        const float alpha = ex2(m - m_new);
        m = m_new;
        mbar_wait(&p_empty[t], (n & 1) ^ 1);
        uint8_t *prow = sP + t * kPBytes + r * 128;
        float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c0 = 0; c0 < BKV; c0 += CH) {
          uint32_t v[CH];
#pragma unroll
          for (int q0 = 0; q0 < CH; q0 += 32)
            tmem_ld_32x32b_x32(s_addr + c0 + q0, *reinterpret_cast<uint32_t(*)[32]>(v + q0));
          tmem_ld_wait();
          uint32_t pk[CH / 2];
#pragma unroll
          for (int c = 0; c < CH; c += 2) {
            float p0 = ex2(fmaf(__uint_as_float(v[c]), scale_log2, -m_new));
            float p1 = ex2(fmaf(__uint_as_float(v[c + 1]), scale_log2, -m_new));
            if (DIAG && c0 + c > r) p0 = 0.f;
            if (DIAG && c0 + c + 1 > r) p1 = 0.f;
            rs8[(c >> 1) & 7] += p0 + p1;
            __nv_bfloat162 tb = __floats2bfloat162_rn(p0, p1);
            pk[c >> 1] = *reinterpret_cast<uint32_t *>(&tb);
          }
          uint8_t *atom_row = prow + (c0 >> 6) * (BQ * 128);  // 64-key swizzle atoms
#pragma unroll
          for (int ch = 0; ch < CH / 8; ++ch) {
            const int chunk = ((c0 & 63) >> 3) + ch;
            *reinterpret_cast<uint4 *>(atom_row + ((chunk ^ (r & 7)) << 4)) =
                make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
          }
        }
        tc_fence_before();
        mbar_arrive(&s_empty[t]);
        fence_async_smem();
        mbar_arrive(&p_full[t]);
        const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
        l = l * alpha + rs;
        return alpha;
      };
      // unmasked tiles in the loop; under causal masking the diagonal tile
      // (always the last, j = qb) runs after it with its own instantiation
      const int nfull = CAUSAL ? nkv - 1 : nkv;
      for (int j = 0; j < nfull; ++j, ++n) {
        mbar_wait(&s_full[t], n & 1);
        tc_fence_after();
        const float alpha = tile(std::false_type{});
        if (j > 0) add_o(n - 1, alpha_prev);
        alpha_prev = alpha;
      }
      if (CAUSAL) {
        mbar_wait(&s_full[t], n & 1);
        tc_fence_after();
        const float alpha = tile(std::true_type{});
        if (nfull > 0) add_o(n - 1, alpha_prev);
        alpha_prev = alpha;
        ++n;
      }
      add_o(n - 1, alpha_prev);
      const float inv = 1.f / l;
      __nv_bfloat16 *orow = out + (int64_t)(row0 + qb * BQ + r) * d + h * DH;
#pragma unroll
      for (int c = 0; c < DH; c += 8) {
        uint4 w;
        uint32_t *wp = reinterpret_cast<uint32_t *>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 tb = __floats2bfloat162_rn(o[c + 2 * e] * inv, o[c + 2 * e + 1] * inv);
          wp[e] = *reinterpret_cast<uint32_t *>(&tb);
        }
        *reinterpret_cast<uint4 *>(orow + c) = w;
      }
      lse[(int64_t)(row0 + qb * BQ + r) * H + h] = m + log2f(l);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

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


// ---------------------------------------------------------------------------
// backward (FA2 dataflow on tcgen05), persistent: one CTA per SM walks a list
// of (sample-head, 128-key block) items, looping over the query blocks that
// attend to each key block:
//   S^T  = K Q^T        dP^T = V dO^T          (TMEM, 128 keys x 128 queries)
//   P^T  = exp2(S^T * c - lse)   dS^T = P^T * (dP^T - D)   (bf16 -> smem)
//   dV  += P^T dO       dK  += dS^T Q          (TMEM accumulators)
//   dQ_i = dS K  -> one TMA reduce-add per block into dq_acc (scaled fp32),
//                   converted by dq_convert
// Causal items are listed heaviest first (key block 0 sees every query
// block) and dealt to the CTAs in a snake order (round r: CTA c takes item
// r G + c for even r, r G + G - 1 - c for odd r), so the CTAs finish
// together; TMEM allocation and barrier set-up are paid once per SM.  Every
// ring / buffer parity follows one running block counter across items; the
// next item's first S^T / dP^T only waits for its own K / V, and its first
// dV / dK MMAs for the previous item's accumulators to have been drained.
// ---------------------------------------------------------------------------
constexpr uint32_t kDqStage = BQ * DH * 4;  // 32 KB: dQ tile (fp32) staged for the TMA reduce-add
// no alignment slack: the dynamic shared-memory base of a kernel without static
// shared memory is 1024-B aligned on sm_100 (tools/probes/smem_base_probe.cu;
// the kernel traps if not), and K / V x2 + Q / dO x2 + dS^T x2 fill 227 KB
constexpr size_t kSmemBwd = 4 * kTileBytes /*K,V x2*/ + 4 * kTileBytes /*Q,dO x2*/ + 2 * kPBytes /*dS^T x2*/ +
                            kDqStage +
                            2 * 2 * BQ * 4 /*lse,D x2*/ + 512;

// the r-th item of CTA c of G (snake order over a heaviest-first list)
__device__ __forceinline__ int bwd_item(int r, int c, int G) { return r * G + ((r & 1) ? G - 1 - c : c); }

template <bool CAUSAL>
__global__ void __launch_bounds__(kThreads2, 1)
    bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dkv,
               const float *__restrict__ lse, const float *__restrict__ dvec, float *__restrict__ dq_acc,
               __nv_bfloat16 *__restrict__ dqkv, int S, int H, int BH, float scale_log2, float scale,
               unsigned long long *trace) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared address space (STS / LDS, not generic ST / LD)
  if (smem_u32(smem_raw) & 1023u) __trap();  // kSmemBwd has no alignment slack (see there)
  uint8_t *smem = smem_raw;
  uint8_t *sK = smem;                     // [2] items
  uint8_t *sV = sK + 2 * kTileBytes;      // [2] items
  uint8_t *sQ = sV + 2 * kTileBytes;      // [2] stages
  uint8_t *sdO = sQ + 2 * kTileBytes;     // [2] stages
  uint8_t *sdS = sdO + 2 * kTileBytes;    // dS^T [2 blocks][128 keys x 128 queries] (P^T lives in TMEM)
  uint8_t *sDQ = sdS + 2 * kPBytes;       // dQ stage: 2 x [128 rows x 32 fp32] SW128 chunks
  float *sL = reinterpret_cast<float *>(sDQ + kDqStage);  // [2][128] lse
  float *sD = sL + 2 * BQ;                               // [2][128] D
  uint64_t *bar = reinterpret_cast<uint64_t *>(sD + 2 * BQ);
  uint64_t *kv_full = bar + 14, *kv_empty = bar + 16;  // [item parity]: K / V double-buffered across items
  // q_empty[b]: block n's gradient MMAs retired (n & 1 == b) -- frees its Q / dO
  // stage and dS^T buffer and publishes dQ(n)
  uint64_t *q_full = bar + 2, *q_empty = bar + 4;
  uint64_t *st_full = bar + 6, *st_empty = bar + 7;
  uint64_t *p_full = bar + 8, *pt_free = bar + 9;  // P^T (TMEM) + dS^T (smem) written / P^T read by dV
  uint64_t *dq_empty = bar + 11;
  uint64_t *acc_full = bar + 12, *acc_empty = bar + 13;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 18);

  const int nq = S / BQ, nkb = S / BKV, n_items = nkb * BH;
  const int G = gridDim.x, c = blockIdx.x;
  const int d = H * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto decode = [&](int i, int &kb, int &b, int &h) {
    int bh;
    if (CAUSAL) {  // key block 0 first: it sees every query block
      kb = i / BH;
      bh = i % BH;
    } else {
      kb = i % nkb;
      bh = i / nkb;
    }
    b = bh / H;
    h = bh % H;
  };
  // TMEM columns
  constexpr uint32_t C_ST = 0, C_DP = 128, C_DV = 256, C_DK = 320, C_DQ = 384, C_PT = 448;
  // diagnostics (HM_ATTN_TRACE=1): clock64 at the phase boundaries of CTA 0's
  // first 64 blocks, trace[event * 64 + block]
  auto mark = [&](int ev, int nn) {
    if (trace && c == 0 && nn < 64) trace[ev * 64 + nn] = clock64();
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    tma_prefetch(&tm_dkv);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(st_full, 1);
    mbar_init(st_empty, 256);
    mbar_init(p_full, 256);
    mbar_init(pt_free, 1);
    mbar_init(dq_empty, 256);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 256);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the set-up above overlapped the previous
  // kernel's tail (dvec); nothing global is read or written before it completed
  griddep_wait();

  if (warp == 0) {
    if (lane == 0) {
      int n = 0;  // running query-block counter (Q / dO stage parities)
      for (int r = 0, i; (i = bwd_item(r, c, G)) < n_items; ++r) {
        int kb, b, h;
        decode(i, kb, b, h);
        const int row0 = b * S;
        // K / V of item r in buffer r & 1: loaded while item r - 1 still runs,
        // so the next item's first S^T / dP^T and elementwise pass overlap the
        // current item's last gradient MMAs
        const int ks = r & 1;
        mbar_wait(&kv_empty[ks], ((r >> 1) & 1) ^ 1);  // every MMA of item r - 2 has read this buffer
        mbar_expect_tx(&kv_full[ks], 2 * kTileBytes);
        tma_load_2d(sK + ks * kTileBytes, &tm_qkv, &kv_full[ks], d + h * DH, row0 + kb * BKV);
        tma_load_2d(sV + ks * kTileBytes, &tm_qkv, &kv_full[ks], 2 * d + h * DH, row0 + kb * BKV);
        for (int qi = CAUSAL ? kb : 0; qi < nq; ++qi, ++n) {
          const int st = n & 1;
          mbar_wait(&q_empty[st], ((n >> 1) & 1) ^ 1);
          mbar_expect_tx(&q_full[st], 2 * kTileBytes);
          tma_load_2d(sQ + st * kTileBytes, &tm_qkv, &q_full[st], h * DH, row0 + qi * BQ);
          tma_load_2d(sdO + st * kTileBytes, &tm_do, &q_full[st], h * DH, row0 + qi * BQ);
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // Two issuing threads on two SM sub-partitions: warp 2 issues S^T / dP^T,
    // warp 1 the gradient MMAs (dV, dK, dQ).  tcgen05.mma issue blocks at the
    // execution rate and each mbarrier round trip costs ~150 cycles, so one
    // thread issuing everything idled the pipe through its own waits.  The two
    // streams touch disjoint TMEM / shared memory except through the softmax
    // (st_full -> softmax -> p_full), which orders them.
    if (lane == 0) {
      constexpr uint32_t id_kk = idesc_bf16_f32(128, 128, 0, 0);   // S^T, dP^T: K-major x K-major
      constexpr uint32_t id_kmn = idesc_bf16_f32(128, DH, 0, 1);   // dV, dK: A K-major, B MN-major
      constexpr uint32_t id_mnmn = idesc_bf16_f32(128, DH, 1, 1);  // dQ: A MN-major (dS), B MN-major (K)
      uint32_t k_base = smem_u32(sK), v_base = smem_u32(sV);  // this item's K / V buffer
      const uint32_t ds_buf0 = smem_u32(sdS);
      // S^T = K Q^T and dP^T = V dO^T of running block n (TMEM C_ST / C_DP)
      auto issue_st = [&](int n) {
        const int st = n & 1;
        mbar_wait(&q_full[st], (n >> 1) & 1);
        mbar_wait(st_empty, (n & 1) ^ 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ + st * kTileBytes), do_base = smem_u32(sdO + st * kTileBytes);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          mma_bf16(tmem + C_ST, umma_desc_sw128(k_base + kk * 32, 16, 1024),
                   umma_desc_sw128(q_base + kk * 32, 16, 1024), id_kk, kk > 0);
          mma_bf16(tmem + C_DP, umma_desc_sw128(v_base + kk * 32, 16, 1024),
                   umma_desc_sw128(do_base + kk * 32, 16, 1024), id_kk, kk > 0);
        }
        mma_commit(st_full);
        mark(0, n);
      };
      int n = 0;
      if (warp == 2) {
        for (int r = 0, i; (i = bwd_item(r, c, G)) < n_items; ++r) {
          int kb, b, h;
          decode(i, kb, b, h);
          const int count = nq - (CAUSAL ? kb : 0);
          mbar_wait(&kv_full[r & 1], (r >> 1) & 1);
          k_base = smem_u32(sK + (r & 1) * kTileBytes);
          v_base = smem_u32(sV + (r & 1) * kTileBytes);
          // block n+1's S^T / dP^T go in as soon as the softmax warps have read
          // block n's (st_empty, inside issue_st), while block n's gradient MMAs
          // are still queued from the other thread
          for (int blk = 0; blk < count; ++blk, ++n) issue_st(n);
        }
      } else {
        for (int r = 0, i; (i = bwd_item(r, c, G)) < n_items; ++r) {
          int kb, b, h;
          decode(i, kb, b, h);
          const int count = nq - (CAUSAL ? kb : 0);
          mbar_wait(&kv_full[r & 1], (r >> 1) & 1);  // dQ reads K
          k_base = smem_u32(sK + (r & 1) * kTileBytes);
          for (int blk = 0; blk < count; ++blk, ++n) {
            const int st = n & 1;
            const uint32_t ph = n & 1;
            // P^T lives in TMEM (the dV MMA's A operand) and dS^T is double-
            // buffered in shared memory, so softmax n+1 waits only for dV(n).
            // What bounds a block is shared-memory bandwidth: the SS MMAs read
            // ~160 KB per block (128 B / clock feeds a 128x64x16 SS MMA exactly,
            // so these N = 64 MMAs run at 48 cycles alone), plus the TMA, dS^T
            // and dQ-stage traffic: ~2300 of the ~3800 cycles per block, and the
            // trace shows the MMAs at ~120 cycles each (profiles/r02_attn_bwd_trace_pt_tmem.log).
            const uint32_t q_base = smem_u32(sQ + st * kTileBytes), do_base = smem_u32(sdO + st * kTileBytes);
            const uint32_t ds_base = ds_buf0 + (n & 1) * kPBytes;
            mbar_wait(p_full, ph);
            mark(1, n);
            if (blk == 0) mbar_wait(acc_empty, (r & 1) ^ 1);  // the previous item's dV / dK drained
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < BQ / 16; ++kk)  // dV += P^T dO, P^T from TMEM (16 queries = 8 columns)
              mma_bf16_ts(tmem + C_DV, tmem + C_PT + kk * 8, umma_desc_sw128(do_base + kk * 2048, BQ * 128, 1024),
                          id_kmn, (blk > 0 || kk > 0) ? 1u : 0u);
            mma_commit(pt_free);  // P^T read: the next block's softmax may overwrite it
#pragma unroll
            for (int kk = 0; kk < BQ / 16; ++kk) {  // dK += dS^T Q, reduction over the 128 queries
              const uint32_t a_off = (kk >> 2) * (BKV * 128) + (kk & 3) * 32;
              mma_bf16(tmem + C_DK, umma_desc_sw128(ds_base + a_off, 16, 1024),
                       umma_desc_sw128(q_base + kk * 2048, BQ * 128, 1024), id_kmn, (blk > 0 || kk > 0) ? 1u : 0u);
            }
            mbar_wait(dq_empty, ph ^ 1);  // the previous block's dQ has left TMEM
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk)  // reduction over the 128 keys
              mma_bf16(tmem + C_DQ, umma_desc_sw128(ds_base + kk * 2048, BKV * 128, 1024),
                       umma_desc_sw128(k_base + kk * 2048, BKV * 128, 1024), id_mnmn, kk > 0);
            // one commit frees block n's Q / dO stage (producer; S^T / dP^T(n),
            // the other thread's readers of Q / dO, completed before p_full(n)),
            // its dS^T buffer (softmax, block n + 2) and publishes dQ(n)
            // (softmax): every commit and wait idles the issuing thread (~45 /
            // ~150 cycles, see attention_fwd64.cu)
            mma_commit(&q_empty[st]);
            mark(2, n);
          }
          mma_commit(acc_full);
          mma_commit(&kv_empty[r & 1]);
        }
      }
    }
  } else if (warp >= 4) {
    // two softmax warpgroups on the same TMEM lanes (key rows): warpgroup wg
    // owns queries [64 wg, 64 wg + 64) of every block, half of dQ's columns,
    // and dV (wg 0) or dK (wg 1) at the end of an item -- two warps per SM
    // sub-partition hide each other's MUFU / TMEM / shared-memory latencies
    const int wg = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int rr = q4 * 32 + lane;  // key row (S^T, dP^T, dV, dK) / query row (dQ) == TMEM lane
    const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
    // lse (wg 0) and D (wg 1) of the query blocks (tiny, strided: plain
    // loads), fetched one block ahead so their latency hides behind the
    // previous block's work
    const float *src = wg == 0 ? lse : dvec;
    float *dst = wg == 0 ? sL : sD;
    // dQ of running block nn (query block qblk of the item at row0 / head h):
    // TMEM -> one TMA reduce-add of the whole 128 x 64 fp32 tile (in L2)
    // instead of 8192 scalar atomics, staged in SW128 rows (conflict-free
    // writes); each warpgroup drains 32 columns
    auto dq_out = [&](int qrow, int hh, int nn) {
      mbar_wait(&q_empty[nn & 1], (nn >> 1) & 1);  // block nn's gradient MMAs (dQ included) retired
      tc_fence_after();
      uint32_t q[32];
      tmem_ld_32x32b_x32(tmem + lane_addr + C_DQ + wg * 32, q);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(dq_empty);
      if (wg == 0 && rr == 0) bulk_wait_read0();  // the previous block's reduce has read the stage
      asm volatile("bar.sync 2, 256;" ::: "memory");
      uint8_t *chunk = sDQ + wg * (BQ * 128) + rr * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4 *>(chunk + ((j ^ (rr & 7)) << 4)) =
            make_float4(__uint_as_float(q[4 * j]) * scale, __uint_as_float(q[4 * j + 1]) * scale,
                        __uint_as_float(q[4 * j + 2]) * scale, __uint_as_float(q[4 * j + 3]) * scale);
      fence_async_smem();
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (wg == 0 && rr == 0) {
#pragma unroll
        for (int cc = 0; cc < DH / 32; ++cc)
          tma_reduce_add_2d(&tm_dq, sDQ + cc * (BQ * 128), hh * DH + 32 * cc, qrow);
        bulk_commit();
      }
    };
    const int hq = wg;
    uint8_t *dsrow0 = sdS + rr * 128 + hq * (BKV * 128);  // + (block & 1) * kPBytes
    const uint32_t pt_addr = tmem + lane_addr + C_PT + hq * 32;  // this warpgroup's P^T columns
    int n = 0;
    int prev_qrow = 0, prev_h = 0;  // the block whose dQ is drained next
    int pend_r = -1, pend_row = 0, pend_h = 0;  // the item whose dV / dK are still in TMEM
    // dV (warpgroup 0) or dK (warpgroup 1) of item pend_r: TMEM -> registers,
    // release the accumulators, then bf16 rows to global
    auto drain_acc = [&]() {
      if (pend_r < 0) return;
      mbar_wait(acc_full, pend_r & 1);
      tc_fence_after();
      uint32_t acc[DH];
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32)
        tmem_ld_32x32b_x32(tmem + lane_addr + (wg == 0 ? C_DV : C_DK) + c0,
                           *reinterpret_cast<uint32_t(*)[32]>(acc + c0));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(acc_empty);  // the next item's first dV / dK MMAs may overwrite
      // this warpgroup's 128 x 64 bf16 tile, staged in SW128 rows in its half of
      // the dQ stage, leaves as one TMA store: dqkv rows are 3d apart, and 16-B
      // stores from every thread cost ~3000 cycles of LSU time per item
      if (wg == 0 && rr == 0) bulk_wait_read0();  // the last dQ reduce-add has read the stage
      asm volatile("bar.sync 2, 256;" ::: "memory");
      uint8_t *trow = sDQ + wg * (BQ * 128) + rr * 128;
      const float osc = wg == 0 ? 1.f : scale;
#pragma unroll
      for (int j = 0; j < DH / 8; ++j) {
        uint4 w;
        uint32_t *pw = reinterpret_cast<uint32_t *>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 a2 = __floats2bfloat162_rn(__uint_as_float(acc[8 * j + 2 * e]) * osc,
                                                    __uint_as_float(acc[8 * j + 2 * e + 1]) * osc);
          pw[e] = *reinterpret_cast<uint32_t *>(&a2);
        }
        *reinterpret_cast<uint4 *>(trow + ((j ^ (rr & 7)) << 4)) = w;
      }
      fence_async_smem();
      asm volatile("bar.sync 2, 256;" ::: "memory");
      if (wg == 0 && rr == 0) {
        tma_store_2d(&tm_dkv, sDQ, 2 * d + pend_h * DH, pend_row);         // dV
        tma_store_2d(&tm_dkv, sDQ + BQ * 128, d + pend_h * DH, pend_row);  // dK
        bulk_commit();
      }
      pend_r = -1;
    };
    for (int r = 0, it; (it = bwd_item(r, c, G)) < n_items; ++r) {
      int kb, b, h;
      decode(it, kb, b, h);
      const int row0 = b * S;
      const int q_begin = CAUSAL ? kb : 0;
      float x_next = src[(int64_t)(row0 + q_begin * BQ + rr) * H + h];
      for (int i = q_begin; i < nq; ++i, ++n) {
        const int st = n & 1;
        const uint32_t ph = n & 1;
        dst[st * BQ + rr] = x_next;
        if (i + 1 < nq) x_next = src[(int64_t)(row0 + (i + 1) * BQ + rr) * H + h];
        asm volatile("bar.sync 1, 256;" ::: "memory");
        mbar_wait(st_full, ph);
        if (wg == 0 && rr == 0) mark(3, n);
        tc_fence_after();
        const bool diag = CAUSAL && i == kb;
        const float *Ls = sL + st * BQ;
        const float *Ds = sD + st * BQ;
        // this warpgroup's 64 queries in two 32-column chunks; the first chunk is
        // computed before waiting for dV(n - 1) to release P^T (TMEM) and dK / dQ
        // (n - 2) the dS^T buffer, so those waits overlap it
        uint8_t *dsrow = dsrow0 + (n & 1) * kPBytes;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t sv[32], dp[32];
          tmem_ld_32x32b_x32(tmem + lane_addr + C_ST + hq * 64 + c0, sv);
          tmem_ld_32x32b_x32(tmem + lane_addr + C_DP + hq * 64 + c0, dp);
          tmem_ld_wait();
          if (c0 == 32) {
            tc_fence_before();
            mbar_arrive(st_empty);  // S^T / dP^T fully read: the next block's MMAs may overwrite
          }
          uint32_t pk[16], dk[16];
          // the causal mask is a separate instantiation: only the diagonal block pays for it
          auto elementwise = [&](auto diag_tag) {
            constexpr bool DIAG = decltype(diag_tag)::value;
#pragma unroll
            for (int cq = 0; cq < 32; cq += 4) {
              const int qi = hq * 64 + c0 + cq;
              // lse / D of four queries per 16-B shared-memory load (broadcast)
              const float4 L4 = *reinterpret_cast<const float4 *>(Ls + qi);
              const float4 D4 = *reinterpret_cast<const float4 *>(Ds + qi);
              const float lq[4] = {L4.x, L4.y, L4.z, L4.w}, dq4[4] = {D4.x, D4.y, D4.z, D4.w};
              float p[4], g[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                p[k] = ex2(fmaf(__uint_as_float(sv[cq + k]), scale_log2, -lq[k]));
                if (DIAG && qi + k < rr) p[k] = 0.f;  // query < key: masked
                g[k] = p[k] * (__uint_as_float(dp[cq + k]) - dq4[k]);
              }
              __nv_bfloat162 tp0 = __floats2bfloat162_rn(p[0], p[1]), tp1 = __floats2bfloat162_rn(p[2], p[3]);
              __nv_bfloat162 td0 = __floats2bfloat162_rn(g[0], g[1]), td1 = __floats2bfloat162_rn(g[2], g[3]);
              pk[cq >> 1] = *reinterpret_cast<uint32_t *>(&tp0);
              pk[(cq >> 1) + 1] = *reinterpret_cast<uint32_t *>(&tp1);
              dk[cq >> 1] = *reinterpret_cast<uint32_t *>(&td0);
              dk[(cq >> 1) + 1] = *reinterpret_cast<uint32_t *>(&td1);
            }
          };
          if (diag) elementwise(std::true_type{});
          else elementwise(std::false_type{});
          if (c0 == 0) {
            mbar_wait(&q_empty[n & 1], ((n >> 1) & 1) ^ 1);  // dK / dQ(n - 2) have read this dS^T buffer
            mbar_wait(pt_free, ph ^ 1);                       // dV(n - 1) has read P^T
            tc_fence_after();
            if (wg == 0 && rr == 0) mark(4, n);
          }
          tmem_st_32x32b_x16(pt_addr + (c0 >> 1), pk);  // queries c0..c0+31 -> 16 bf16-pair columns
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            const uint32_t off = (((c0 >> 3) + ch) ^ (rr & 7)) << 4;
            *reinterpret_cast<uint4 *>(dsrow + off) = make_uint4(dk[4 * ch], dk[4 * ch + 1], dk[4 * ch + 2], dk[4 * ch + 3]);
          }
        }
        tmem_st_wait();
        fence_async_smem();
        tc_fence_before();
        mbar_arrive(p_full);
        if (rr == 0) mark(wg == 0 ? 5 : 7, n);
        drain_acc();  // the previous item's dV / dK (first block of an item only)
        // the previous block's dQ: drained while this block's gradient MMAs run
        // (dQ(n) cannot start before this drain releases the TMEM columns)
        if (n > 0) dq_out(prev_qrow, prev_h, n - 1);
        if (wg == 0 && rr == 0) mark(6, n);
        prev_qrow = row0 + i * BQ;
        prev_h = h;
      }
      // this item's dV / dK are drained after the next item's first block has
      // been handed to the MMAs (below), so that block's elementwise pass
      // overlaps this item's last gradient MMAs
      pend_r = r;
      pend_row = row0 + kb * BKV;
      pend_h = h;
    }
    drain_acc();
    if (n > 0) dq_out(prev_qrow, prev_h, n - 1);
    if (wg == 0 && rr == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

static int make_map(CUtensorMap *tm, const void *base, int64_t inner, int64_t rows, int64_t pitch_bytes) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  if (fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(HM_ERR_DEVICE, "attention tensor map encode failed");
  return HM_OK;
}

int backward_main(const void *qkv, const void *dout, const float *lse, const float *dvec, float *dq_acc, void *dqkv,
                  int B, int S, int H, int causal, cudaStream_t s) {
  const int d = H * DH;
  CUtensorMap tq, td;
  HM_TRY(make_map(&tq, qkv, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2));
  HM_TRY(make_map(&td, dout, d, (int64_t)B * S, (int64_t)d * 2));
  CUtensorMap tdkv;  // dqkv [B*S, 3d] bf16, {64, 128} boxes: dK / dV tiles leave by TMA store
  HM_TRY(make_map(&tdkv, dqkv, 3 * (int64_t)d, (int64_t)B * S, 3 * (int64_t)d * 2));
  CUtensorMap tdq;  // dq_acc [B*S, d] fp32, {32, 128} boxes in SW128 (the reduce-add target)
  {
    EncodeFn fn = encode_fn();
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)B * S};
    cuuint64_t strides[1] = {(cuuint64_t)d * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t estr[2] = {1, 1};
    if (!fn || fn(&tdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq_acc, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(HM_ERR_DEVICE, "attention dQ tensor map encode failed");
  }
  static bool attr[2] = {false, false};
  auto k = causal ? bwd_kernel<true> : bwd_kernel<false>;
  if (!attr[causal ? 1 : 0]) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBwd));
    attr[causal ? 1 : 0] = true;
  }
  const float scale = 1.f / sqrtf((float)DH);
  const int sms = current_sm_count();
  const int items = (S / BKV) * B * H;
  // HM_ATTN_TRACE=1 (diagnostics): CTA 0's phase timestamps, printed to stderr
  static const bool tracing = getenv("HM_ATTN_TRACE") && getenv("HM_ATTN_TRACE")[0] == '1';
  static unsigned long long *tbuf = nullptr;
  if (tracing && !tbuf) {
    HM_CUDA(cudaMalloc(&tbuf, 8 * 64 * sizeof(unsigned long long)));
    HM_CUDA(cudaMemset(tbuf, 0, 8 * 64 * sizeof(unsigned long long)));
  }
  HM_CUDA(launch_pdl(k, dim3(items < sms ? items : sms), dim3(kThreads2), kSmemBwd, s, tq, td, tdq, tdkv, lse, dvec,
                     dq_acc, static_cast<__nv_bfloat16 *>(dqkv), S, H, B * H, 1.4426950408889634f * scale, scale,
                     tracing ? tbuf : nullptr));
  if (tracing) {
    unsigned long long h[8 * 64];
    HM_CUDA(cudaStreamSynchronize(s));
    HM_CUDA(cudaMemcpy(h, tbuf, sizeof h, cudaMemcpyDeviceToHost));
    fprintf(stderr, "{\"attn_bwd_trace\": [");
    for (int e = 0; e < 8; ++e) {
      fprintf(stderr, "%s[", e ? ", " : "");
      for (int n = 0; n < 64; ++n) fprintf(stderr, "%s%llu", n ? ", " : "", h[e * 64 + n] ? h[e * 64 + n] - h[0] : 0ULL);
      fprintf(stderr, "]");
    }
    fprintf(stderr, "]}\n");
  }
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

// true if the tensor-core path handles this shape (else use the mma.sync kernel)
bool supported(int S, int DHx) { return DHx == DH && S % BQ == 0; }

int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s) {
  // HM_ATTN_FWD: unset = attention_fwd64.cu (rotating S buffers in TMEM, whole-row
  // softmax in registers); q = the persistent query-block-pair kernel below (the
  // round-1 default, S % 256 == 0); t = attention_tc128.cu's dataflow at head_dim 64
  static const char *mode_env = getenv("HM_ATTN_FWD");
  static const char mode = mode_env ? mode_env[0] : 'd';
  if (mode == 't') return attn_tc128::forward64(qkv, o, lse, B, S, H, causal, s);
  if (mode != 'q' || S % (2 * BQ) != 0) return attn_fwd64::forward(qkv, o, lse, B, S, H, causal, s);
  EncodeFn fn = encode_fn();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  const int d = H * DH;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)3 * d, (cuuint64_t)B * S};
  cuuint64_t strides[1] = {(cuuint64_t)3 * d * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(qkv), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(HM_ERR_DEVICE, "attention tensor map encode failed");
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  ProfScope ps(KC_ATTN_FWD, s, 4.0 * B * (double)S * S * H * DH * (causal ? 0.5 : 1.0), (double)B * S * H * DH * 2 * 4);
  static bool attrq[2] = {false, false};
  const int sms_q = current_sm_count();
  auto kq = causal ? fwd2p_kernel<true> : fwd2p_kernel<false>;
  if (!attrq[causal ? 1 : 0]) {
    HM_CUDA(cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem2P));
    attrq[causal ? 1 : 0] = true;
  }
  const int items = (S / (2 * BQ)) * B * H;
  kq<<<dim3(items < sms_q ? items : sms_q), kThreads2, kSmem2P, s>>>(tm, static_cast<__nv_bfloat16 *>(o), lse, S, H,
                                                                    B * H, scale_log2);
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

}  // namespace attn_tc
}  // namespace hm


extern "C" int hm_k_attn_fwd_tc(const void *qkv, void *out, float *lse, int32_t batch, int32_t seq, int32_t heads,
                                int32_t head_dim, int32_t causal, void *stream) {
  if (hm::attn_tc128::supported(seq, head_dim))
    return hm::attn_tc128::forward(qkv, out, lse, batch, seq, heads, causal, static_cast<cudaStream_t>(stream));
  if (!hm::attn_tc::supported(seq, head_dim))
    return hm::fail(HM_ERR_VALIDATION, "tcgen05 attention needs head_dim 64 or 128 and seq % 128 == 0");
  return hm::attn_tc::forward(qkv, out, lse, batch, seq, heads, causal, static_cast<cudaStream_t>(stream));
}
