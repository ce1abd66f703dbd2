// attention.cu -- fused (flash-style) multi-head attention, forward and
// backward, for the transformer blocks of a layer pack.
//
// Layout: qkv [tokens, 3d] bf16 (q | k | v, head-major inside each third),
// o / do [tokens, d] bf16, lse [tokens, H] fp32 (log2 domain).  Scores never
// touch HBM: per (sample, head, 64-query block) the kernel streams 64-key K/V
// tiles through shared memory (cp.async double buffer), keeps the online
// softmax in registers and accumulates O in registers.
//
// Round-1 implementation: warp-level mma.sync m16n8k16 (bf16 -> fp32) with
// ldmatrix fragments.  Attention is ~5-10% of a block's FLOPs at the BASELINE
// shapes (4sd vs 24d^2, halved by the causal mask); the tcgen05 version is a
// later-round item.
#include <cuda_bf16.h>

#include <cstdlib>
#include <string>

#include "../runtime/common.hpp"
#include "pdl.cuh"

namespace hm {
namespace attn_tc {
bool supported(int S, int DH);
int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s);
int backward_main(const void *qkv, const void *dout, const float *lse, const float *dvec, float *dq_acc, void *dqkv,
                  int B, int S, int H, int causal, cudaStream_t s);
}  // namespace attn_tc
namespace attn_bwd64 {  // head_dim 64 backward over 64-query sub-blocks (attention_bwd64.cu)
int backward_main(const void *qkv, const void *dout, const float *lse, const float *dvec, float *dq_acc, void *dqkv,
                  int B, int S, int H, int causal, cudaStream_t s);
}  // namespace attn_bwd64
namespace attn_tc128 {  // head_dim 128 (attention_tc128.cu)
bool supported(int S, int DH);
int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int causal, cudaStream_t s);
int backward_main(const void *qkv, const void *dout, const float *lse, const float *dvec, float *dq_acc, void *dqkv,
                  int B, int S, int H, int causal, cudaStream_t s);
}  // namespace attn_tc128
namespace attn {

constexpr int BQ = 64, BKV = 64, THREADS = 128;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

// Copy a [64 rows x DH] bf16 tile (global row pitch `ld` elements) into smem
// with row pitch DH+8.
template <int DH>
__device__ __forceinline__ void load_tile(__nv_bfloat16 *s, const __nv_bfloat16 *g, int64_t ld) {
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < 64 * CH; i += THREADS) {
    const int r = i / CH, c = i % CH;
    cp_async16(s + r * (DH + 8) + c * 8, g + (int64_t)r * ld + c * 8);
  }
}

// A fragments (16 rows x 16 cols) from a row-major smem tile.
template <int LD>
__device__ __forceinline__ void lda_frag(uint32_t (&a)[4], const __nv_bfloat16 *s, int row0, int col0) {
  const int lane = threadIdx.x & 31;
  const int mi = lane >> 3, ri = lane & 7;
  ldsm_x4(a, s + (row0 + ri + (mi & 1) * 8) * LD + col0 + (mi >> 1) * 8);
}
// B fragments for two n-blocks from storage [n][k] (row-major, k contiguous).
template <int LD>
__device__ __forceinline__ void ldb_nk(uint32_t (&b)[4], const __nv_bfloat16 *s, int n0, int k0) {
  const int lane = threadIdx.x & 31;
  const int mi = lane >> 3, ri = lane & 7;
  ldsm_x4(b, s + (n0 + ri + (mi >> 1) * 8) * LD + k0 + (mi & 1) * 8);
}
// B fragments for two n-blocks from storage [k][n] (row-major, n contiguous).
template <int LD>
__device__ __forceinline__ void ldb_kn(uint32_t (&b)[4], const __nv_bfloat16 *s, int k0, int n0) {
  const int lane = threadIdx.x & 31;
  const int mi = lane >> 3, ri = lane & 7;
  ldsm_x4_t(b, s + (k0 + ri + (mi & 1) * 8) * LD + n0 + (mi >> 1) * 8);
}

template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(THREADS) fwd_kernel(const __nv_bfloat16 *__restrict__ qkv,
                                                      __nv_bfloat16 *__restrict__ out, float *__restrict__ lse,
                                                      int S, int H, float scale_log2) {
  constexpr int LD = DH + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16 *sQ = reinterpret_cast<__nv_bfloat16 *>(smem_raw);
  __nv_bfloat16 *sK = sQ + 64 * LD;       // [2][64][LD]
  __nv_bfloat16 *sV = sK + 2 * 64 * LD;   // [2][64][LD]
  const int nq = S / BQ;
  const int qb = CAUSAL ? nq - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int64_t ld = 3 * (int64_t)d;
  const __nv_bfloat16 *base = qkv + (int64_t)b * S * ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;

  load_tile<DH>(sQ, base + (int64_t)qb * BQ * ld + h * DH, ld);
  load_tile<DH>(sK, base + d + h * DH, ld);
  load_tile<DH>(sV, base + 2 * d + h * DH, ld);
  cp_commit();
  const int nk = CAUSAL ? qb + 1 : nq;

  uint32_t qf[DH / 16][4];
  float o[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int kb = 0; kb < nk; ++kb) {
    const int st = kb & 1;
    if (kb + 1 < nk) {
      load_tile<DH>(sK + (st ^ 1) * 64 * LD, base + (int64_t)(kb + 1) * BKV * ld + d + h * DH, ld);
      load_tile<DH>(sV + (st ^ 1) * 64 * LD, base + (int64_t)(kb + 1) * BKV * ld + 2 * d + h * DH, ld);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kc = 0; kc < DH / 16; ++kc) lda_frag<LD>(qf[kc], sQ, warp * 16, kc * 16);
    }
    const __nv_bfloat16 *k_s = sK + st * 64 * LD;
    const __nv_bfloat16 *v_s = sV + st * 64 * LD;
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < DH / 16; ++kc) {
#pragma unroll
      for (int nb2 = 0; nb2 < 4; ++nb2) {
        uint32_t bf[4];
        ldb_nk<LD>(bf, k_s, nb2 * 16, kc * 16);
        mma16816(s[2 * nb2], qf[kc], bf[0], bf[1]);
        mma16816(s[2 * nb2 + 1], qf[kc], bf[2], bf[3]);
      }
    }
    const bool diag = CAUSAL && kb == qb;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[j][e] * scale_log2;
        if (diag) {
          const int key = 8 * j + 2 * t + (e & 1);
          const int qry = warp * 16 + g + (e >= 2 ? 8 : 0);
          if (key > qry) v = -INFINITY;
        }
        s[j][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float a0 = exp2f(m0 - mn0), a1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s[j][0] = exp2f(s[j][0] - mn0);
      s[j][1] = exp2f(s[j][1] - mn0);
      s[j][2] = exp2f(s[j][2] - mn1);
      s[j][3] = exp2f(s[j][3] - mn1);
      rs0 += s[j][0] + s[j][1];
      rs1 += s[j][2] + s[j][3];
    }
    l0 = l0 * a0 + rs0;
    l1 = l1 * a1 + rs1;
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
      o[j][0] *= a0; o[j][1] *= a0;
      o[j][2] *= a1; o[j][3] *= a1;
    }
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      uint32_t pa[4] = {pack_bf16(s[2 * kc][0], s[2 * kc][1]), pack_bf16(s[2 * kc][2], s[2 * kc][3]),
                        pack_bf16(s[2 * kc + 1][0], s[2 * kc + 1][1]), pack_bf16(s[2 * kc + 1][2], s[2 * kc + 1][3])};
#pragma unroll
      for (int nb2 = 0; nb2 < DH / 16; ++nb2) {
        uint32_t bf[4];
        ldb_kn<LD>(bf, v_s, kc * 16, nb2 * 16);
        mma16816(o[2 * nb2], pa, bf[0], bf[1]);
        mma16816(o[2 * nb2 + 1], pa, bf[2], bf[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffff, l0, 1);
  l0 += __shfl_xor_sync(0xffffffff, l0, 2);
  l1 += __shfl_xor_sync(0xffffffff, l1, 1);
  l1 += __shfl_xor_sync(0xffffffff, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  const int64_t row0 = (int64_t)b * S + qb * BQ + warp * 16 + g;
  __nv_bfloat16 *o0 = out + row0 * d + h * DH;
  __nv_bfloat16 *o1 = o0 + 8 * (int64_t)d;
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) {
    *reinterpret_cast<uint32_t *>(o0 + 8 * j + 2 * t) = pack_bf16(o[j][0] * i0, o[j][1] * i0);
    *reinterpret_cast<uint32_t *>(o1 + 8 * j + 2 * t) = pack_bf16(o[j][2] * i1, o[j][3] * i1);
  }
  if (t == 0) {
    lse[row0 * H + h] = m0 + log2f(l0);
    lse[(row0 + 8) * H + h] = m1 + log2f(l1);
  }
}

// D[token, h] = sum_c dO * O  (the softmax-backward row term)
// D[token, head] = sum_k dO * O over the head's DH values: one thread per
// (token, head) row of DH bf16 (DH * 2 bytes = DH / 8 16-B loads of each input,
// all in flight); consecutive threads read consecutive rows (coalesced).
template <int DH>
// D = rowsum(dO * O) per (token, head), and the dQ accumulator of that (token,
// head) zeroed in the same pass (it receives reduce-adds next).  DH / 8
// threads per (token, head), one 16-B load of O and of dO each: a warp reads
// 32 x 16 B contiguous (one thread per (token, head) touched a 128-B stride).
__global__ void dvec_kernel(const __nv_bfloat16 *__restrict__ o, const __nv_bfloat16 *__restrict__ dout,
                            float *__restrict__ dvec, float *__restrict__ dq_acc, int64_t rows, int H) {
  pdl_wait();
  constexpr int TPR = DH / 8;  // threads per (token, head)
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t w = t / TPR;
  const int part = (int)(t % TPR);
  const bool live = w < rows * H;
  float acc = 0.f;
  if (live) {
    const uint4 va = reinterpret_cast<const uint4 *>(o + w * DH)[part];
    const uint4 vc = reinterpret_cast<const uint4 *>(dout + w * DH)[part];
    const __nv_bfloat162 *x = reinterpret_cast<const __nv_bfloat162 *>(&va);
    const __nv_bfloat162 *y = reinterpret_cast<const __nv_bfloat162 *>(&vc);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fx = __bfloat1622float2(x[j]), fy = __bfloat1622float2(y[j]);
      acc = fmaf(fx.x, fy.x, fmaf(fx.y, fy.y, acc));
    }
    float4 *z = reinterpret_cast<float4 *>(dq_acc + w * DH) + 2 * part;
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int m = TPR / 2; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (live && part == 0) dvec[w] = acc;
}

template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(THREADS) bwd_kernel(const __nv_bfloat16 *__restrict__ qkv,
                                                      const __nv_bfloat16 *__restrict__ dout,
                                                      const float *__restrict__ lse, const float *__restrict__ dvec,
                                                      float *__restrict__ dq_acc, __nv_bfloat16 *__restrict__ dqkv,
                                                      int S, int H, float scale_log2, float scale) {
  constexpr int LD = DH + 8;
  constexpr int LDS = 64 + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16 *sK = reinterpret_cast<__nv_bfloat16 *>(smem_raw);
  __nv_bfloat16 *sV = sK + 64 * LD;
  __nv_bfloat16 *sQ = sV + 64 * LD;
  __nv_bfloat16 *sdO = sQ + 64 * LD;
  __nv_bfloat16 *sdS = sdO + 64 * LD;  // [64 queries][LDS]
  float *sL = reinterpret_cast<float *>(sdS + 64 * LDS);
  float *sD = sL + 64;
  const int nq = S / BQ;
  const int kb = blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int64_t ld = 3 * (int64_t)d;
  const __nv_bfloat16 *base = qkv + (int64_t)b * S * ld;
  const __nv_bfloat16 *dbase = dout + (int64_t)b * S * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;

  load_tile<DH>(sK, base + (int64_t)kb * BKV * ld + d + h * DH, ld);
  load_tile<DH>(sV, base + (int64_t)kb * BKV * ld + 2 * d + h * DH, ld);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  uint32_t kf[DH / 16][4], vf[DH / 16][4];
#pragma unroll
  for (int kc = 0; kc < DH / 16; ++kc) {
    lda_frag<LD>(kf[kc], sK, warp * 16, kc * 16);
    lda_frag<LD>(vf[kc], sV, warp * 16, kc * 16);
  }
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[j][e] = dv[j][e] = 0.f;

  for (int qb = CAUSAL ? kb : 0; qb < nq; ++qb) {
    load_tile<DH>(sQ, base + (int64_t)qb * BQ * ld + h * DH, ld);
    load_tile<DH>(sdO, dbase + (int64_t)qb * BQ * d + h * DH, d);
    cp_commit();
    if (threadIdx.x < 64) {
      const int64_t row = (int64_t)b * S + qb * BQ + threadIdx.x;
      sL[threadIdx.x] = lse[row * H + h];
      sD[threadIdx.x] = dvec[row * H + h];
    }
    cp_wait<0>();
    __syncthreads();
    // S^T[16 keys x 64 queries] = K Q^T
    float st[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) st[j][0] = st[j][1] = st[j][2] = st[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < DH / 16; ++kc)
#pragma unroll
      for (int nb2 = 0; nb2 < 4; ++nb2) {
        uint32_t bf[4];
        ldb_nk<LD>(bf, sQ, nb2 * 16, kc * 16);
        mma16816(st[2 * nb2], kf[kc], bf[0], bf[1]);
        mma16816(st[2 * nb2 + 1], kf[kc], bf[2], bf[3]);
      }
    const bool diag = CAUSAL && qb == kb;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qry = 8 * j + 2 * t + (e & 1);
        const int key = warp * 16 + g + (e >= 2 ? 8 : 0);
        float p = exp2f(st[j][e] * scale_log2 - sL[qry]);
        if (diag && qry < key) p = 0.f;
        st[j][e] = p;  // P^T
      }
    // dV += P^T dO
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      uint32_t pa[4] = {pack_bf16(st[2 * kc][0], st[2 * kc][1]), pack_bf16(st[2 * kc][2], st[2 * kc][3]),
                        pack_bf16(st[2 * kc + 1][0], st[2 * kc + 1][1]),
                        pack_bf16(st[2 * kc + 1][2], st[2 * kc + 1][3])};
#pragma unroll
      for (int nb2 = 0; nb2 < DH / 16; ++nb2) {
        uint32_t bf[4];
        ldb_kn<LD>(bf, sdO, kc * 16, nb2 * 16);
        mma16816(dv[2 * nb2], pa, bf[0], bf[1]);
        mma16816(dv[2 * nb2 + 1], pa, bf[2], bf[3]);
      }
    }
    // dP^T = V dO^T
    float dp[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < DH / 16; ++kc)
#pragma unroll
      for (int nb2 = 0; nb2 < 4; ++nb2) {
        uint32_t bf[4];
        ldb_nk<LD>(bf, sdO, nb2 * 16, kc * 16);
        mma16816(dp[2 * nb2], vf[kc], bf[0], bf[1]);
        mma16816(dp[2 * nb2 + 1], vf[kc], bf[2], bf[3]);
      }
    // dS^T = P^T * (dP^T - D)
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qry = 8 * j + 2 * t + (e & 1);
        dp[j][e] = st[j][e] * (dp[j][e] - sD[qry]);
      }
    // dK += dS^T Q ; stash dS (as [query][key]) for dQ
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      uint32_t pa[4] = {pack_bf16(dp[2 * kc][0], dp[2 * kc][1]), pack_bf16(dp[2 * kc][2], dp[2 * kc][3]),
                        pack_bf16(dp[2 * kc + 1][0], dp[2 * kc + 1][1]),
                        pack_bf16(dp[2 * kc + 1][2], dp[2 * kc + 1][3])};
#pragma unroll
      for (int nb2 = 0; nb2 < DH / 16; ++nb2) {
        uint32_t bf[4];
        ldb_kn<LD>(bf, sQ, kc * 16, nb2 * 16);
        mma16816(dk[2 * nb2], pa, bf[0], bf[1]);
        mma16816(dk[2 * nb2 + 1], pa, bf[2], bf[3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qry = 8 * j + 2 * t + (e & 1);
        const int key = warp * 16 + g + (e >= 2 ? 8 : 0);
        sdS[qry * LDS + key] = __float2bfloat16_rn(dp[j][e]);
      }
    __syncthreads();
    // dQ[16 queries of this warp x DH] += dS K   (reduction over the 64 keys)
    float dq[DH / 8][4];
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      uint32_t af[4];
      lda_frag<LDS>(af, sdS, warp * 16, kc * 16);
#pragma unroll
      for (int nb2 = 0; nb2 < DH / 16; ++nb2) {
        uint32_t bf[4];
        ldb_kn<LD>(bf, sK, kc * 16, nb2 * 16);
        mma16816(dq[2 * nb2], af, bf[0], bf[1]);
        mma16816(dq[2 * nb2 + 1], af, bf[2], bf[3]);
      }
    }
    const int64_t q0 = (int64_t)b * S + qb * BQ + warp * 16 + g;
    float *dq0 = dq_acc + q0 * d + h * DH;
    float *dq1 = dq0 + 8 * (int64_t)d;
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
      atomicAdd(dq0 + 8 * j + 2 * t, dq[j][0]);
      atomicAdd(dq0 + 8 * j + 2 * t + 1, dq[j][1]);
      atomicAdd(dq1 + 8 * j + 2 * t, dq[j][2]);
      atomicAdd(dq1 + 8 * j + 2 * t + 1, dq[j][3]);
    }
    __syncthreads();
  }
  const int64_t k0 = (int64_t)b * S + kb * BKV + warp * 16 + g;
  __nv_bfloat16 *dk0 = dqkv + k0 * ld + d + h * DH;
  __nv_bfloat16 *dv0 = dqkv + k0 * ld + 2 * d + h * DH;
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) {
    *reinterpret_cast<uint32_t *>(dk0 + 8 * j + 2 * t) = pack_bf16(dk[j][0] * scale, dk[j][1] * scale);
    *reinterpret_cast<uint32_t *>(dk0 + 8 * ld + 8 * j + 2 * t) = pack_bf16(dk[j][2] * scale, dk[j][3] * scale);
    *reinterpret_cast<uint32_t *>(dv0 + 8 * j + 2 * t) = pack_bf16(dv[j][0], dv[j][1]);
    *reinterpret_cast<uint32_t *>(dv0 + 8 * ld + 8 * j + 2 * t) = pack_bf16(dv[j][2], dv[j][3]);
  }
}

// dQ (fp32 accumulator [rows, d]) -> the Q third of dqkv [rows, 3d] as bf16,
// four values per thread (float4 in, bf16x4 out); d % 4 == 0.
__global__ void dq_convert(const float *__restrict__ dq_acc, __nv_bfloat16 *__restrict__ dqkv, int64_t rows, int d,
                           float scale) {
  pdl_wait();
  const uint32_t d4 = (uint32_t)(d / 4);
  const int64_t n4 = rows * d4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d4;
    const int64_t c = 4 * (i - r * d4);
    const float4 v = reinterpret_cast<const float4 *>(dq_acc)[i];
    __nv_bfloat162 p0 = __floats2bfloat162_rn(v.x * scale, v.y * scale), p1 = __floats2bfloat162_rn(v.z * scale, v.w * scale);
    *reinterpret_cast<uint2 *>(dqkv + r * 3 * (int64_t)d + c) =
        make_uint2(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1));
  }
}

template <int DH>
static size_t fwd_smem() { return (size_t)5 * 64 * (DH + 8) * 2; }
template <int DH>
static size_t bwd_smem() { return (size_t)4 * 64 * (DH + 8) * 2 + 64 * 72 * 2 + 2 * 64 * 4; }

template <int DH, bool CAUSAL>
static int fwd_launch(const __nv_bfloat16 *qkv, __nv_bfloat16 *o, float *lse, int B, int S, int H, cudaStream_t s) {
  static bool attr = false;
  auto k = fwd_kernel<DH, CAUSAL>;
  if (!attr) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem<DH>()));
    attr = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  const double fl = 4.0 * B * (double)S * S * H * DH * (CAUSAL ? 0.5 : 1.0);
  ProfScope ps(KC_ATTN_FWD, s, fl, (double)B * S * H * DH * 2 * 4);
  k<<<dim3(S / BQ, B * H), THREADS, fwd_smem<DH>(), s>>>(qkv, o, lse, S, H, scale_log2);
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

template <int DH, bool CAUSAL>
static int bwd_launch(const __nv_bfloat16 *qkv, const __nv_bfloat16 *o, const __nv_bfloat16 *dout, const float *lse,
                      float *dvec, float *dq_acc, __nv_bfloat16 *dqkv, int B, int S, int H, cudaStream_t s) {
  static bool attr = false;
  auto k = bwd_kernel<DH, CAUSAL>;
  if (!attr) {
    HM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd_smem<DH>()));
    attr = true;
  }
  const int64_t rows = (int64_t)B * S;
  const int d = H * DH;
  ProfScope ps(KC_ATTN_BWD, s, 10.0 * B * (double)S * S * H * DH * (CAUSAL ? 0.5 : 1.0), (double)rows * d * 2 * 8);
  const int64_t threads = rows * H * (DH / 8);
  HM_CUDA(launch_pdl(dvec_kernel<DH>, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s, o, dout, dvec, dq_acc,
                     rows, H));
  const float scale = 1.f / sqrtf((float)DH);
  // The tcgen05 backward (attention_tc.cu: TMEM accumulators, dQ as one TMA
  // reduce-add per query block) is the default where it applies (head_dim 64,
  // seq % 128 == 0): 1.4-1.5x this mma.sync kernel on B200.  HM_ATTN_BWD=mma
  // forces the mma.sync kernel.
  // head_dim 64: the 128-query kernel of attention_tc.cu; HM_ATTN_BWD=s selects
  // attention_bwd64.cu (64-query sub-blocks, alternating softmax warpgroups,
  // P^T / dS^T from TMEM): equal within 3% (104 vs 107 us at 4 x 1024 x 25
  // heads, 417 vs 403 at 16 x 1024, profiles/r02_attn_perf_bwd64_ab.jsonl) --
  // both wait on the tensor pipe, which runs the N = 64 MMAs at 45-48 cycles
  // alone (32 ideal, profiles/r02_mma_probe.jsonl) and at ~90 next to the
  // softmax warps' TMEM and shared-memory traffic (HM_ATTN_TRACE)
  static const bool use_tc = [] {
    const char *e = getenv("HM_ATTN_BWD");
    return !(e && std::string(e) == "mma");
  }();
  static const bool bwd_s = [] {
    const char *e = getenv("HM_ATTN_BWD");
    return e && std::string(e) == "s";
  }();
  if (use_tc && (attn_tc::supported(S, DH) || attn_tc128::supported(S, DH))) {
    // tcgen05 main kernel; it folds the softmax scale into dq_acc
    if (DH == 64 && bwd_s)
      HM_TRY(attn_bwd64::backward_main(qkv, dout, lse, dvec, dq_acc, dqkv, B, S, H, CAUSAL ? 1 : 0, s));
    else if (DH == 64)
      HM_TRY(attn_tc::backward_main(qkv, dout, lse, dvec, dq_acc, dqkv, B, S, H, CAUSAL ? 1 : 0, s));
    else HM_TRY(attn_tc128::backward_main(qkv, dout, lse, dvec, dq_acc, dqkv, B, S, H, CAUSAL ? 1 : 0, s));
    HM_CUDA(launch_pdl(dq_convert, dim3(1184), dim3(256), 0, s, (const float *)dq_acc, dqkv, rows, d, 1.f));
  } else {
    k<<<dim3(S / BKV, B * H), THREADS, bwd_smem<DH>(), s>>>(qkv, dout, lse, dvec, dq_acc, dqkv, S, H,
                                                             1.4426950408889634f * scale, scale);
    HM_CUDA(launch_pdl(dq_convert, dim3(1184), dim3(256), 0, s, (const float *)dq_acc, dqkv, rows, d, scale));
  }
  count_launch(3);
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int DH, int causal, cudaStream_t s) {
  if (S % 64) return fail(HM_ERR_VALIDATION, "attention: seq_len must be a multiple of 64");
  static const bool force_mma = [] {
    const char *e = getenv("HM_ATTN");
    return e && std::string(e) == "mma";
  }();
  if (!force_mma && attn_tc::supported(S, DH)) return attn_tc::forward(qkv, o, lse, B, S, H, causal, s);
  if (!force_mma && attn_tc128::supported(S, DH)) return attn_tc128::forward(qkv, o, lse, B, S, H, causal, s);
  auto q = static_cast<const __nv_bfloat16 *>(qkv);
  auto out = static_cast<__nv_bfloat16 *>(o);
  if (DH == 64) return causal ? fwd_launch<64, true>(q, out, lse, B, S, H, s) : fwd_launch<64, false>(q, out, lse, B, S, H, s);
  if (DH == 128)
    return causal ? fwd_launch<128, true>(q, out, lse, B, S, H, s) : fwd_launch<128, false>(q, out, lse, B, S, H, s);
  return fail(HM_ERR_VALIDATION, "attention: head_dim must be 64 or 128");
}

int backward(const void *qkv, const void *o, const void *dout, const float *lse, float *dvec, float *dq_acc,
             void *dqkv, int B, int S, int H, int DH, int causal, cudaStream_t s) {
  if (S % 64) return fail(HM_ERR_VALIDATION, "attention: seq_len must be a multiple of 64");
  auto q = static_cast<const __nv_bfloat16 *>(qkv);
  auto oo = static_cast<const __nv_bfloat16 *>(o);
  auto dO = static_cast<const __nv_bfloat16 *>(dout);
  auto dst = static_cast<__nv_bfloat16 *>(dqkv);
  if (DH == 64)
    return causal ? bwd_launch<64, true>(q, oo, dO, lse, dvec, dq_acc, dst, B, S, H, s)
                  : bwd_launch<64, false>(q, oo, dO, lse, dvec, dq_acc, dst, B, S, H, s);
  if (DH == 128)
    return causal ? bwd_launch<128, true>(q, oo, dO, lse, dvec, dq_acc, dst, B, S, H, s)
                  : bwd_launch<128, false>(q, oo, dO, lse, dvec, dq_acc, dst, B, S, H, s);
  return fail(HM_ERR_VALIDATION, "attention: head_dim must be 64 or 128");
}

}  // namespace attn
}  // namespace hm

extern "C" int hm_k_attn_fwd(const void *qkv, void *out, float *lse, int32_t batch, int32_t seq, int32_t heads,
                             int32_t head_dim, int32_t causal, void *stream) {
  return hm::attn::forward(qkv, out, lse, batch, seq, heads, head_dim, causal, static_cast<cudaStream_t>(stream));
}

extern "C" int hm_k_attn_bwd(const void *qkv, const void *out, const void *dout, const float *lse, float *dvec,
                             float *dq_acc, void *dqkv, int32_t batch, int32_t seq, int32_t heads, int32_t head_dim,
                             int32_t causal, void *stream) {
  return hm::attn::backward(qkv, out, dout, lse, dvec, dq_acc, dqkv, batch, seq, heads, head_dim, causal,
                            static_cast<cudaStream_t>(stream));
}
