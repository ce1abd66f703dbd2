// attention_fwd64.cu -- flash-attention forward for head_dim 64 (GPT-2 XL,
// BERT-Large) on the 5th-gen tensor cores, built around the two limits the
// head_dim-64 shape hits first: the MUFU exp2 rate (16384 ex2 per 128 x 128
// tile against 512 cycles of MMA) and the softmax's wait on the tensor pipe.
//
// One CTA per pair of 128-query tiles (heaviest causal pairs first):
//   warp 0      TMA: both Q tiles once, then K_j / V_j into a 3-stage ring
//   warp 1      TMEM allocation, MMA issuer
//   warps 4-7   softmax of tile 0, warps 8-11 of tile 1 (one thread per
//               query row; warp w reads TMEM lanes 32 (w % 4) .. + 31)
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
// Output conventions as attention.cu: o [tokens, d] bf16, lse [tokens, H]
// in the log2 domain.
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>

#include "../runtime/common.hpp"
#include "sm100.cuh"

namespace hm {
namespace attn_fwd64 {

using namespace sm100;

constexpr int DH = 64, BQ = 128, BKV = 128;
constexpr int kStages = 3;               // K / V ring
constexpr int kSBuf = 3;                 // rotating S / P buffers in TMEM
constexpr uint32_t kTile = BQ * DH * 2;  // 128 rows x 128 B: one SW128 atom column, 16 KB
constexpr int kThreads = 384;
constexpr float kRescaleLog2 = 8.f;      // lazy-rescale threshold (log2 units)
constexpr uint32_t C_O = kSBuf * BKV;    // O_t at columns [384 + 64 t, 448 + 64 t)
constexpr size_t kSmem = 1024 + 2 * kTile /*Q pair*/ + 2 * kStages * kTile /*K, V*/ + 256;
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

template <bool CAUSAL>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16 *__restrict__ out, float *__restrict__ lse,
               int S, int H, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sQ = smem;                  // [2 tiles]
  uint8_t *sK = sQ + 2 * kTile;        // [kStages]
  uint8_t *sV = sK + kStages * kTile;  // [kStages]
  uint64_t *bar = reinterpret_cast<uint64_t *>(sV + kStages * kTile);
  uint64_t *q_full = bar;
  uint64_t *kv_full = bar + 1, *kv_empty = bar + 1 + kStages;
  uint64_t *s_full = bar + 1 + 2 * kStages;       // [kSBuf]
  uint64_t *p_full = s_full + kSBuf;              // [tile]
  uint64_t *o_full = p_full + 2;                  // [tile]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_full + 2);

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
  const int mn = nkv0 < nkv1 ? nkv0 : nkv1, nall = nkv0 > nkv1 ? nkv0 : nkv1, npos = nkv0 + nkv1;
  const int tlast = nkv1 >= nkv0 ? 1 : 0;  // the tile that runs alone past step mn
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = b * S;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < kSBuf; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    reg_dealloc<72>();  // 3 x 168 per SMSP at launch = 72 + 2 x 216
    if (warp == 0 && lane == 0) {
      mbar_expect_tx(q_full, (has1 ? 2 : 1) * kTile);
      tma_load_2d(sQ, &tm, q_full, h * DH, row0 + qb0 * BQ);
      if (has1) tma_load_2d(sQ + kTile, &tm, q_full, h * DH, row0 + (qb0 + 1) * BQ);
      for (int j = 0; j < nall; ++j) {
        const int st = j % kStages;
        mbar_wait(&kv_empty[st], ((j / kStages) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * kTile);
        tma_load_2d(sK + st * kTile, &tm, &kv_full[st], d + h * DH, row0 + j * BKV);
        tma_load_2d(sV + st * kTile, &tm, &kv_full[st], 2 * d + h * DH, row0 + j * BKV);
      }
    } else if (warp == 1 && lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(BQ, BKV, 0, 0);  // Q K-major, K K-major
      constexpr uint32_t idesc_o = idesc_bf16_f32(BQ, DH, 0, 1);   // P (TMEM), V MN-major
      // position n of the S / PV sequence -> (tile, step)
      auto at = [&](int n, int &t, int &j) {
        if (n < 2 * mn) {
          t = n & 1;
          j = n >> 1;
        } else {
          t = tlast;
          j = mn + (n - 2 * mn);
        }
      };
      mbar_wait(q_full, 0);
      auto issue_s = [&](int n) {
        int t, j;
        at(n, t, j);
        const int st = j % kStages;
        mbar_wait(&kv_full[st], (j / kStages) & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sQ + t * kTile), k_base = smem_u32(sK + st * kTile);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          mma_bf16(tmem + (n % kSBuf) * BKV, umma_desc_sw128(q_base + kk * 32, 16, 1024),
                   umma_desc_sw128(k_base + kk * 32, 16, 1024), idesc_s, kk > 0);
        mma_commit(&s_full[n % kSBuf]);
      };
      for (int n = 0; n < kSBuf && n < npos; ++n) issue_s(n);
      for (int n = 0; n < npos; ++n) {
        int t, j;
        at(n, t, j);
        mbar_wait(&p_full[t], j & 1);  // P_t(j) written into S buffer n % 3 (and O_t rescaled)
        tc_fence_after();
        const uint32_t v_base = smem_u32(sV + (j % kStages) * kTile);
        const uint32_t p_tm = tmem + (n % kSBuf) * BKV;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_bf16_ts(tmem + C_O + t * DH, p_tm + kk * 8, umma_desc_sw128(v_base + kk * 2048, kTile, 1024), idesc_o,
                      (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&o_full[t]);
        if (t == 1 || j >= mn) mma_commit(&kv_empty[j % kStages]);  // last use of K_j / V_j
        // S(n + 3) overwrites P(n) in TMEM: issued after PV(n), which reads it first
        if (n + kSBuf < npos) issue_s(n + kSBuf);
      }
    }
  } else {
    reg_alloc<216>();
    const int t = (warp >> 2) - 1;
    const int nkv = t == 0 ? nkv0 : nkv1;
    if (nkv > 0) {
      const int q4 = warp & 3;
      const int r = q4 * 32 + lane;  // query row inside the tile == TMEM lane
      const int qb = qb0 + t;
      const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
      const uint32_t o_addr = tmem + lane_addr + C_O + t * DH;
      const float2 sc2 = make_float2(scale_log2, scale_log2);
      float m = -INFINITY, l = 0.f;  // m: the max the exponents are taken against (log2 domain)
      for (int j = 0; j < nkv; ++j) {
        const int n = j < mn ? 2 * j + t : 2 * mn + (j - mn);
        const int buf = n % kSBuf;
        const uint32_t s_addr = tmem + lane_addr + buf * BKV;
        mbar_wait(&s_full[buf], (n / kSBuf) & 1);
        tc_fence_after();
        uint32_t v[BKV];
#pragma unroll
        for (int q = 0; q < BKV / 32; ++q)
          tmem_ld_32x32b_x32(s_addr + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * q));
        tmem_ld_wait();
        if (CAUSAL && j == qb) {  // diagonal tile: keys after the query are masked
#pragma unroll
          for (int c = 0; c < BKV; ++c)
            if (c > r) v[c] = 0xff800000u;  // -inf
        }
        float mx[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) mx[e] = fmaxf(__uint_as_float(v[e]), __uint_as_float(v[4 + e]));
#pragma unroll
        for (int c = 8; c < BKV; c += 8) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            mx[e] = fmaxf(mx[e], fmaxf(__uint_as_float(v[c + e]), __uint_as_float(v[c + 4 + e])));
        }
        const float m_row = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
        float alpha = 1.f;
        if (m_row > m + kRescaleLog2) {  // first tile (m = -inf) always lands here
          alpha = ex2(m - m_row);
          m = m_row;
        }
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {  // warp-uniform: tcgen05.ld / st are .sync.aligned
          // PV_t(j - 2) is complete (S(n) was issued after it); wait for PV_t(j - 1)
          mbar_wait(&o_full[t], (j - 1) & 1);
          tc_fence_after();
          const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
          for (int c0 = 0; c0 < DH; c0 += 32) {
            uint32_t ov[32];
            tmem_ld_32x32b_x32(o_addr + c0, ov);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
              const float2 o2 = mul2(make_float2(__uint_as_float(ov[c]), __uint_as_float(ov[c + 1])), a2);
              ov[c] = __float_as_uint(o2.x);
              ov[c + 1] = __float_as_uint(o2.y);
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
          for (int c = 0; c < 32; c += 2) {
            const float2 x = fma2(make_float2(__uint_as_float(v[c0 + c]), __uint_as_float(v[c0 + c + 1])), sc2, nm2);
            const float2 p = make_float2(ex2(x.x), ex2(x.y));
            rs[(c >> 1) & 1] = add2(rs[(c >> 1) & 1], p);
            pk[c >> 1] = bf16x2(p.x, p.y);
          }
          // keys c0..c0+31 -> P columns c0/2..c0/2+15 (every S column already read)
          tmem_st_32x32b_x16(s_addr + (c0 >> 1), pk);
        }
        tmem_st_wait();
        l = l * alpha + ((rs[0].x + rs[0].y) + (rs[1].x + rs[1].y));
        tc_fence_before();
        mbar_arrive(&p_full[t]);
      }
      mbar_wait(&o_full[t], (nkv - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      __nv_bfloat16 *orow = out + (int64_t)(row0 + qb * BQ + r) * d + h * DH;
#pragma unroll
      for (int c0 = 0; c0 < DH; c0 += 32) {
        uint32_t ov[32];
        tmem_ld_32x32b_x32(o_addr + c0, ov);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          uint4 w;
          w.x = bf16x2(__uint_as_float(ov[c]) * inv, __uint_as_float(ov[c + 1]) * inv);
          w.y = bf16x2(__uint_as_float(ov[c + 2]) * inv, __uint_as_float(ov[c + 3]) * inv);
          w.z = bf16x2(__uint_as_float(ov[c + 4]) * inv, __uint_as_float(ov[c + 5]) * inv);
          w.w = bf16x2(__uint_as_float(ov[c + 6]) * inv, __uint_as_float(ov[c + 7]) * inv);
          *reinterpret_cast<uint4 *>(orow + c0 + c) = w;
        }
      }
      lse[(int64_t)(row0 + qb * BQ + r) * H + h] = m + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
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
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  ProfScope ps(KC_ATTN_FWD, s, 4.0 * B * (double)S * S * H * DH * (causal ? 0.5 : 1.0), (double)B * S * H * DH * 2 * 4);
  static bool attr[2] = {false, false};
  auto k = causal ? fwd_kernel<true> : fwd_kernel<false>;
  if (!attr[causal ? 1 : 0]) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    attr[causal ? 1 : 0] = true;
  }
  const int npair = (S / BQ + 1) / 2;
  k<<<dim3(B * H, npair), kThreads, kSmem, s>>>(tm, static_cast<__nv_bfloat16 *>(o), lse, S, H, scale_log2);
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

}  // namespace attn_fwd64
}  // namespace hm
