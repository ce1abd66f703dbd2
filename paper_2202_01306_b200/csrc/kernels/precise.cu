// precise.cu -- the fp32-operand parity mode of the transformer layer pack
// (hm_model.math_mode = 1; BASELINE.json north_star: "loss and weights after
// K steps within 1e-3 relative in fp32-accumulate mode, with the bf16
// tolerance stated separately").
//
// Every activation the default mode keeps as a bf16 GEMM operand is kept in
// fp32 here, and every GEMM runs on the same tcgen05 kernel with each fp32
// operand split into three bf16 planes, x = x0 + x1 + x2 (x0 = bf16(x),
// x1 = bf16(x - x0), x2 = bf16(x - x0 - x1): 24 significant bits).  The
// product keeps the six plane products with i + j <= 2, summed in fp32
// (TMEM accumulators, then TMA reduce-adds), smallest first; the dropped
// terms are below 2^-24 relative -- fp32-level accuracy with tensor cores.
// Attention, LayerNorm forward and cross-entropy get fp32 SIMT kernels with
// full-precision expf / tanhf / sqrtf; the rest of the pack (LayerNorm
// backward, bias gradients, embedding, Adam) is fp32 in both modes.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "../runtime/common.hpp"
#include "../runtime/kernels_api.hpp"
#include "pdl.cuh"

namespace hm {
namespace prec {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
  return v;
}

static unsigned blocks_for(int64_t n, int per) { return (unsigned)std::min<int64_t>((n + per - 1) / per, 148 * 32); }

// ---- three-plane split ----------------------------------------------------------
__global__ void split3_kernel(const float *__restrict__ x, bf16 *__restrict__ p, int64_t n, int64_t plane) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const bf16 a = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(a);  // exact
    const bf16 b = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(b);  // exact
    p[i] = a;
    p[plane + i] = b;
    p[2 * plane + i] = __float2bfloat16_rn(r2);
  }
}

int split3(const float *x, void *planes, int64_t n, int64_t plane, cudaStream_t s) {
  if (n <= 0) return HM_OK;
  ProfScope ps(KC_MISC, s, 0, 10.0 * n);
  HM_CUDA(launch_pdl(split3_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, s, x, static_cast<bf16 *>(planes), n,
                     plane));
  count_launch();
  return HM_OK;
}

// ---- GEMM epilogues applied after the split-product sum --------------------------
enum { PE_RESID = 0, PE_GELU = 1, PE_DGELU = 2 };

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float dgelu_tanh(float x) {  // torch's tanh-approximation backward
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanhf(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

__global__ void epilogue_kernel(int kind, const float *__restrict__ acc, int64_t M, int N, const float *bias,
                                float *aux, int64_t ld_aux, float *d, int64_t ldd) {
  pdl_wait();
  const int64_t n = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N;
    const int c = (int)(i - r * N);
    const float a = acc[i] + (bias ? bias[c] : 0.f);
    if (kind == PE_RESID) {
      d[r * ldd + c] = aux[r * ld_aux + c] + a;
    } else if (kind == PE_GELU) {
      aux[r * ld_aux + c] = a;
      d[r * ldd + c] = gelu_tanh(a);
    } else {
      d[r * ldd + c] = acc[i] * dgelu_tanh(aux[r * ld_aux + c]);
    }
  }
}

// C = A . B^T with fp32 operands through the bf16 tensor-core GEMM (see the
// header comment).  Same argument meaning as gemm::run; the bf16 epilogues
// write fp32 here.  `sa` / `sb` hold three planes of the largest A / B operand,
// `c32` an M x N fp32 accumulator for the fused epilogues.
int gemm(const float *A, const float *B, void *D, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
         int64_t ldd, int a_mn, int b_mn, int epi, const float *bias, void *aux, int64_t ld_aux, cudaStream_t s,
         void *sa, int64_t sa_elems, void *sb, int64_t sb_elems, float *c32, int64_t c32_elems) {
  const int64_t na = (a_mn ? K - 1 : M - 1) * lda + (a_mn ? M : K);
  const int64_t nb = (b_mn ? K - 1 : N - 1) * ldb + (b_mn ? N : K);
  const int64_t pa = (na + 7) / 8 * 8, pb = (nb + 7) / 8 * 8;  // 16-B aligned planes
  if (3 * pa > sa_elems || 3 * pb > sb_elems) return fail(HM_ERR_INTERNAL, "precise gemm: split scratch too small");
  HM_TRY(split3(A, sa, na, pa, s));
  HM_TRY(split3(B, sb, nb, pb, s));
  const bool fused = epi == HM_EPI_RESID_F32 || epi == HM_EPI_GELU_BF16 || epi == HM_EPI_DGELU_BF16;
  if (!fused && epi != HM_EPI_STORE_BF16 && epi != HM_EPI_STORE_F32 && epi != HM_EPI_ACC_F32)
    return fail(HM_ERR_VALIDATION, "precise gemm: unsupported epilogue");
  if (fused && M * N > c32_elems) return fail(HM_ERR_INTERNAL, "precise gemm: accumulator scratch too small");
  void *tgt = fused ? static_cast<void *>(c32) : D;
  const int64_t ldt = fused ? N : ldd;
  const bf16 *a = static_cast<const bf16 *>(sa), *b = static_cast<const bf16 *>(sb);
  static const int order[6][2] = {{2, 0}, {0, 2}, {1, 1}, {1, 0}, {0, 1}, {0, 0}};  // smallest terms first
  // the accumulating passes (all but the smallest, first term) sum K in
  // chunks of at most 16 k-blocks (1024) in TMEM, the chunks in fp32 by the
  // reduce-add: the tensor core's long-chain accumulation error, not the bf16
  // planes, bounds this mode's accuracy otherwise
  struct KCap {
    int prev;
    KCap() : prev(gemm::max_kblocks_per_split()) { gemm::max_kblocks_per_split() = 16; }
    ~KCap() { gemm::max_kblocks_per_split() = prev; }
  } kcap;
  for (int t = 0; t < 6; ++t) {
    const int i = order[t][0], j = order[t][1];
    const bool first = t == 0 && epi != HM_EPI_ACC_F32;
    const int e = first ? HM_EPI_STORE_F32 : HM_EPI_ACC_F32;
    HM_TRY(gemm::run(a + i * pa, b + j * pb, tgt, M, N, K, lda, ldb, ldt, a_mn, b_mn, e,
                     first && !fused ? bias : nullptr, nullptr, 0, s, 0));
  }
  if (!fused) return HM_OK;
  const int kind = epi == HM_EPI_RESID_F32 ? PE_RESID : epi == HM_EPI_GELU_BF16 ? PE_GELU : PE_DGELU;
  ProfScope ps(KC_MISC, s, 0, 12.0 * M * N);
  HM_CUDA(launch_pdl(epilogue_kernel, dim3(blocks_for(M * N, 256)), dim3(256), 0, s, kind, (const float *)c32, M,
                     (int)N, kind == PE_DGELU ? nullptr : bias, static_cast<float *>(aux), ld_aux,
                     static_cast<float *>(D), ldd));
  count_launch();
  return HM_OK;
}

// ---- LayerNorm forward, fp32 out ------------------------------------------------
__global__ void ln_fwd_kernel(const float *__restrict__ x, const float *__restrict__ g, const float *__restrict__ b,
                              float *__restrict__ y, float *__restrict__ mean, float *__restrict__ rstd, int64_t rows,
                              int d) {
  pdl_wait();
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float *xr = x + r * d;
  float s = 0.f;
  for (int i = lane; i < d; i += 32) s += xr[i];
  const float mu = warp_sum(s) / d;
  float q = 0.f;
  for (int i = lane; i < d; i += 32) q += (xr[i] - mu) * (xr[i] - mu);
  const float rs = 1.f / sqrtf(warp_sum(q) / d + 1e-5f);
  for (int i = lane; i < d; i += 32) y[r * d + i] = (xr[i] - mu) * rs * g[i] + b[i];
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

int ln_fwd(const float *x, const float *g, const float *b, float *y, float *mean, float *rstd, int64_t rows, int d,
           cudaStream_t s) {
  ProfScope ps(KC_LAYERNORM, s, 0, 8.0 * rows * d);
  HM_CUDA(launch_pdl(ln_fwd_kernel, dim3((unsigned)((rows * 32 + 255) / 256)), dim3(256), 0, s, x, g, b, y, mean,
                     rstd, rows, d));
  count_launch();
  return HM_OK;
}

// ---- softmax cross-entropy, fp32 dlogits ----------------------------------------
__global__ void __launch_bounds__(512) ce_kernel(const float *__restrict__ logits, const int32_t *__restrict__ labels,
                                                 int64_t ldl, int V, float *__restrict__ dlog, double *loss_sum,
                                                 float scale) {
  pdl_wait();
  const int64_t r = blockIdx.x;
  const float *row = logits + r * ldl;
  __shared__ float red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float m = -INFINITY;
  for (int i = threadIdx.x; i < V; i += blockDim.x) m = fmaxf(m, row[i]);
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < nw; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float s = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) s += expf(row[i] - m);
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = 0.f;
  for (int w = 0; w < nw; ++w) s += red[w];
  const int lab = labels[r];
  const float inv = 1.f / s;
  for (int i = threadIdx.x; i < ldl; i += blockDim.x)
    dlog[r * ldl + i] = i < V ? (expf(row[i] - m) * inv - (i == lab ? 1.f : 0.f)) * scale : 0.f;
  if (threadIdx.x == 0) atomicAdd(loss_sum, (double)m + log((double)s) - (double)row[lab]);
}

int cross_entropy(const float *logits, const int32_t *labels, int64_t rows, int64_t ldl, int V, float *dlogits,
                  double *loss_sum, float scale, cudaStream_t s) {
  ProfScope ps(KC_XENT, s, 0, 8.0 * rows * ldl);
  HM_CUDA(launch_pdl(ce_kernel, dim3((unsigned)rows), dim3(512), 0, s, logits, labels, ldl, V, dlogits, loss_sum,
                     scale));
  count_launch();
  return HM_OK;
}

// ---- attention, fp32 SIMT --------------------------------------------------------
// qkv [B*S, 3*H*DH] fp32 (q | k | v thirds), o [B*S, H*DH], lse [B*S, H]
// (natural log of the row's sum of exp(q.k * scale)).  A block owns 32 rows of
// one (batch, head); 8 warps x 4 rows; key / value tiles of 32 rows are staged
// in shared memory (padded rows: lane j reads row j conflict-free).  A lane
// owns DH/32 output columns.  Online softmax in fp32 with expf.
constexpr int T32 = 32;

template <int DH>
__global__ void __launch_bounds__(256) attn_fwd_kernel(const float *__restrict__ qkv, float *__restrict__ o,
                                                       float *__restrict__ lse, int S, int H, int causal, float scale) {
  pdl_wait();
  extern __shared__ float sm[];
  float *Qs = sm;                        // [32][DH]
  float *Ks = Qs + T32 * DH;             // [32][DH+1]
  float *Vs = Ks + T32 * (DH + 1);       // [32][DH]
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ld = 3LL * H * DH;
  const float *base = qkv + (int64_t)b * S * ld;
  for (int i = threadIdx.x; i < T32 * DH; i += blockDim.x) {
    const int r = i / DH, c = i % DH;
    Qs[i] = base[(int64_t)(qt * T32 + r) * ld + h * DH + c];
  }
  constexpr int E = DH / 32;
  float m[4], l[4], acc[4][E];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[r][e] = 0.f;
  }
  const int nkt = causal ? qt + 1 : S / T32;
  for (int kt = 0; kt < nkt; ++kt) {
    __syncthreads();
    for (int i = threadIdx.x; i < T32 * DH; i += blockDim.x) {
      const int r = i / DH, c = i % DH;
      const float *row = base + (int64_t)(kt * T32 + r) * ld;
      Ks[r * (DH + 1) + c] = row[H * DH + h * DH + c];
      Vs[r * DH + c] = row[2 * H * DH + h * DH + c];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qi = warp * 4 + r, qg = qt * T32 + qi, kg = kt * T32 + lane;
      float sc = 0.f;
#pragma unroll 16
      for (int c = 0; c < DH; ++c) sc = fmaf(Qs[qi * DH + c], Ks[lane * (DH + 1) + c], sc);
      sc *= scale;
      if (causal && kg > qg) sc = -INFINITY;
      const float mn = fmaxf(m[r], warp_max(sc));
      const float p = sc == -INFINITY ? 0.f : expf(sc - mn);
      const float corr = m[r] == -INFINITY ? 0.f : expf(m[r] - mn);
      l[r] = l[r] * corr + warp_sum(p);
      m[r] = mn;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[r][e] *= corr;
      for (int j = 0; j < T32; ++j) {
        const float pj = __shfl_sync(0xffffffff, p, j);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[r][e] = fmaf(pj, Vs[j * DH + lane + 32 * e], acc[r][e]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = (int64_t)b * S + qt * T32 + warp * 4 + r;
    const float inv = 1.f / l[r];
#pragma unroll
    for (int e = 0; e < E; ++e) o[row * H * DH + h * DH + lane + 32 * e] = acc[r][e] * inv;
    if (lane == 0) lse[row * H + h] = m[r] + logf(l[r]);
  }
}

// dvec[row, h] = sum_c dO[row, h*DH + c] * O[row, h*DH + c]
__global__ void attn_dvec_kernel(const float *__restrict__ o, const float *__restrict__ dout, float *__restrict__ dvec,
                                 int64_t rows, int H, int DH) {
  pdl_wait();
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows * H) return;
  const int64_t r = w / H;
  const int h = (int)(w - r * H);
  float s = 0.f;
  for (int c = lane; c < DH; c += 32) s += o[r * H * DH + h * DH + c] * dout[r * H * DH + h * DH + c];
  s = warp_sum(s);
  if (lane == 0) dvec[w] = s;
}

// dQ: a block owns 32 query rows (8 warps x 4), loops over key tiles; lane j = key j.
template <int DH>
__global__ void __launch_bounds__(256) attn_dq_kernel(const float *__restrict__ qkv, const float *__restrict__ dout,
                                                      const float *__restrict__ lse, const float *__restrict__ dvec,
                                                      float *__restrict__ dqkv, int S, int H, int causal,
                                                      float scale) {
  pdl_wait();
  extern __shared__ float sm[];
  float *Qs = sm;                     // [32][DH]
  float *Os = Qs + T32 * DH;          // [32][DH]  dO rows
  float *Ks = Os + T32 * DH;          // [32][DH+1]
  float *Vs = Ks + T32 * (DH + 1);    // [32][DH+1]
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ld = 3LL * H * DH, ldo = (int64_t)H * DH;
  const float *base = qkv + (int64_t)b * S * ld;
  for (int i = threadIdx.x; i < T32 * DH; i += blockDim.x) {
    const int r = i / DH, c = i % DH;
    const int64_t row = (int64_t)qt * T32 + r;
    Qs[i] = base[row * ld + h * DH + c];
    Os[i] = dout[((int64_t)b * S + row) * ldo + h * DH + c];
  }
  constexpr int E = DH / 32;
  float dq[4][E], ls[4], dv[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = (int64_t)b * S + qt * T32 + warp * 4 + r;
    ls[r] = lse[row * H + h];
    dv[r] = dvec[row * H + h];
#pragma unroll
    for (int e = 0; e < E; ++e) dq[r][e] = 0.f;
  }
  const int nkt = causal ? qt + 1 : S / T32;
  for (int kt = 0; kt < nkt; ++kt) {
    __syncthreads();
    for (int i = threadIdx.x; i < T32 * DH; i += blockDim.x) {
      const int r = i / DH, c = i % DH;
      const float *row = base + (int64_t)(kt * T32 + r) * ld;
      Ks[r * (DH + 1) + c] = row[H * DH + h * DH + c];
      Vs[r * (DH + 1) + c] = row[2 * H * DH + h * DH + c];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qi = warp * 4 + r, qg = qt * T32 + qi, kg = kt * T32 + lane;
      float sc = 0.f, dp = 0.f;
#pragma unroll 16
      for (int c = 0; c < DH; ++c) {
        sc = fmaf(Qs[qi * DH + c], Ks[lane * (DH + 1) + c], sc);
        dp = fmaf(Os[qi * DH + c], Vs[lane * (DH + 1) + c], dp);
      }
      const float p = (causal && kg > qg) ? 0.f : expf(sc * scale - ls[r]);
      const float ds = p * (dp - dv[r]) * scale;
      for (int j = 0; j < T32; ++j) {
        const float dsj = __shfl_sync(0xffffffff, ds, j);
#pragma unroll
        for (int e = 0; e < E; ++e) dq[r][e] = fmaf(dsj, Ks[j * (DH + 1) + lane + 32 * e], dq[r][e]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = (int64_t)b * S + qt * T32 + warp * 4 + r;
#pragma unroll
    for (int e = 0; e < E; ++e) dqkv[row * ld + h * DH + lane + 32 * e] = dq[r][e];
  }
}

// dK, dV: a block owns 32 key rows (8 warps x 4), loops over query tiles; lane i = query i.
template <int DH>
__global__ void __launch_bounds__(256) attn_dkv_kernel(const float *__restrict__ qkv, const float *__restrict__ dout,
                                                       const float *__restrict__ lse, const float *__restrict__ dvec,
                                                       float *__restrict__ dqkv, int S, int H, int causal,
                                                       float scale) {
  pdl_wait();
  extern __shared__ float sm[];
  float *Ks = sm;                     // [32][DH]  own keys
  float *Vs = Ks + T32 * DH;          // [32][DH]
  float *Qs = Vs + T32 * DH;          // [32][DH+1]
  float *Os = Qs + T32 * (DH + 1);    // [32][DH+1]
  float *Ls = Os + T32 * (DH + 1);    // [32] lse
  float *Dv = Ls + T32;               // [32] dvec
  const int kt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ld = 3LL * H * DH, ldo = (int64_t)H * DH;
  const float *base = qkv + (int64_t)b * S * ld;
  for (int i = threadIdx.x; i < T32 * DH; i += blockDim.x) {
    const int r = i / DH, c = i % DH;
    const float *row = base + (int64_t)(kt * T32 + r) * ld;
    Ks[i] = row[H * DH + h * DH + c];
    Vs[i] = row[2 * H * DH + h * DH + c];
  }
  constexpr int E = DH / 32;
  float dk[4][E], dvv[4][E];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int e = 0; e < E; ++e) dk[r][e] = dvv[r][e] = 0.f;
  const int q0 = causal ? kt : 0;
  for (int qt = q0; qt < S / T32; ++qt) {
    __syncthreads();
    for (int i = threadIdx.x; i < T32 * DH; i += blockDim.x) {
      const int r = i / DH, c = i % DH;
      const int64_t row = (int64_t)qt * T32 + r;
      Qs[r * (DH + 1) + c] = base[row * ld + h * DH + c];
      Os[r * (DH + 1) + c] = dout[((int64_t)b * S + row) * ldo + h * DH + c];
    }
    if (threadIdx.x < T32) {
      const int64_t row = (int64_t)b * S + qt * T32 + threadIdx.x;
      Ls[threadIdx.x] = lse[row * H + h];
      Dv[threadIdx.x] = dvec[row * H + h];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int kj = warp * 4 + r, kg = kt * T32 + kj, qg = qt * T32 + lane;
      float sc = 0.f, dp = 0.f;
#pragma unroll 16
      for (int c = 0; c < DH; ++c) {
        sc = fmaf(Qs[lane * (DH + 1) + c], Ks[kj * DH + c], sc);
        dp = fmaf(Os[lane * (DH + 1) + c], Vs[kj * DH + c], dp);
      }
      const float p = (causal && kg > qg) ? 0.f : expf(sc * scale - Ls[lane]);
      const float ds = p * (dp - Dv[lane]) * scale;
      for (int i = 0; i < T32; ++i) {
        const float pi = __shfl_sync(0xffffffff, p, i), dsi = __shfl_sync(0xffffffff, ds, i);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          dvv[r][e] = fmaf(pi, Os[i * (DH + 1) + lane + 32 * e], dvv[r][e]);
          dk[r][e] = fmaf(dsi, Qs[i * (DH + 1) + lane + 32 * e], dk[r][e]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = (int64_t)b * S + kt * T32 + warp * 4 + r;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      dqkv[row * ld + H * DH + h * DH + lane + 32 * e] = dk[r][e];
      dqkv[row * ld + 2 * H * DH + h * DH + lane + 32 * e] = dvv[r][e];
    }
  }
}

template <typename K>
static cudaError_t launch_big(K kernel, dim3 grid, size_t smem, cudaStream_t s, const float *a, const float *b,
                              const float *c, const float *d, float *e, int S, int H, int causal, float scale) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl(kernel, grid, dim3(256), smem, s, a, b, c, d, e, S, H, causal, scale);
}

int attn_forward(const float *qkv, float *o, float *lse, int B, int S, int H, int DH, int causal, cudaStream_t s) {
  if (S % T32) return fail(HM_ERR_VALIDATION, "precise attention: seq_len must be a multiple of 32");
  ProfScope ps(KC_ATTN_FWD, s, 4.0 * B * H * (double)S * S * DH * (causal ? 0.5 : 1.0), 0);
  const dim3 grid(S / T32, H, B);
  const float scale = 1.f / sqrtf((float)DH);
  const size_t smem = (size_t)T32 * (3 * DH + 1) * 4;
  cudaError_t e;
  if (DH == 64) {
    cudaFuncSetAttribute(attn_fwd_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = launch_pdl(attn_fwd_kernel<64>, grid, dim3(256), smem, s, qkv, o, lse, S, H, causal, scale);
  } else if (DH == 128) {
    cudaFuncSetAttribute(attn_fwd_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = launch_pdl(attn_fwd_kernel<128>, grid, dim3(256), smem, s, qkv, o, lse, S, H, causal, scale);
  } else {
    return fail(HM_ERR_VALIDATION, "precise attention: head_dim must be 64 or 128");
  }
  HM_CUDA(e);
  count_launch();
  return HM_OK;
}

int attn_backward(const float *qkv, const float *o, const float *dout, const float *lse, float *dvec, float *dqkv,
                  int B, int S, int H, int DH, int causal, cudaStream_t s) {
  if (S % T32) return fail(HM_ERR_VALIDATION, "precise attention: seq_len must be a multiple of 32");
  if (DH != 64 && DH != 128) return fail(HM_ERR_VALIDATION, "precise attention: head_dim must be 64 or 128");
  ProfScope ps(KC_ATTN_BWD, s, 10.0 * B * H * (double)S * S * DH * (causal ? 0.5 : 1.0), 0);
  const int64_t rows = (int64_t)B * S;
  HM_CUDA(launch_pdl(attn_dvec_kernel, dim3((unsigned)((rows * H * 32 + 255) / 256)), dim3(256), 0, s, o, dout, dvec,
                     rows, H, DH));
  count_launch();
  const dim3 grid(S / T32, H, B);
  const float scale = 1.f / sqrtf((float)DH);
  const size_t smem_q = (size_t)T32 * (4 * DH + 2) * 4, smem_kv = (size_t)T32 * (4 * DH + 4) * 4;
  if (DH == 64) {
    HM_CUDA(launch_big(attn_dq_kernel<64>, grid, smem_q, s, qkv, dout, lse, dvec, dqkv, S, H, causal, scale));
    HM_CUDA(launch_big(attn_dkv_kernel<64>, grid, smem_kv, s, qkv, dout, lse, dvec, dqkv, S, H, causal, scale));
  } else {
    HM_CUDA(launch_big(attn_dq_kernel<128>, grid, smem_q, s, qkv, dout, lse, dvec, dqkv, S, H, causal, scale));
    HM_CUDA(launch_big(attn_dkv_kernel<128>, grid, smem_kv, s, qkv, dout, lse, dvec, dqkv, S, H, causal, scale));
  }
  count_launch(2);
  return HM_OK;
}

}  // namespace prec
}  // namespace hm

extern "C" int hm_k_gemm_precise(const float *a, const float *b, void *d, int64_t m, int64_t n, int64_t k,
                                 int64_t lda, int64_t ldb, int64_t ldd, int32_t a_major, int32_t b_major,
                                 int32_t epilogue, const float *bias, void *aux, int64_t ld_aux, void *scratch_a,
                                 int64_t scratch_a_elems, void *scratch_b, int64_t scratch_b_elems, float *acc,
                                 int64_t acc_elems, void *stream) {
  return hm::prec::gemm(a, b, d, m, n, k, lda, ldb, ldd, a_major, b_major, epilogue, bias, aux, ld_aux,
                        static_cast<cudaStream_t>(stream), scratch_a, scratch_a_elems, scratch_b, scratch_b_elems,
                        acc, acc_elems);
}

extern "C" int hm_k_attn_fwd_f32(const float *qkv, float *out, float *lse, int32_t batch, int32_t seq, int32_t heads,
                                 int32_t head_dim, int32_t causal, void *stream) {
  return hm::prec::attn_forward(qkv, out, lse, batch, seq, heads, head_dim, causal, static_cast<cudaStream_t>(stream));
}

extern "C" int hm_k_attn_bwd_f32(const float *qkv, const float *out, const float *dout, const float *lse, float *dvec,
                                 float *dqkv, int32_t batch, int32_t seq, int32_t heads, int32_t head_dim,
                                 int32_t causal, void *stream) {
  return hm::prec::attn_backward(qkv, out, dout, lse, dvec, dqkv, batch, seq, heads, head_dim, causal,
                                 static_cast<cudaStream_t>(stream));
}

extern "C" int hm_k_layernorm_fwd_f32(const float *x, const float *g, const float *b, float *y, float *mean,
                                      float *rstd, int64_t rows, int32_t d, void *stream) {
  return hm::prec::ln_fwd(x, g, b, y, mean, rstd, rows, d, static_cast<cudaStream_t>(stream));
}

extern "C" int hm_k_cross_entropy_f32(const float *logits, const int32_t *labels, int64_t rows, int64_t ld,
                                      int32_t vocab, float *dlogits, double *loss_sum, float scale, void *stream) {
  return hm::prec::cross_entropy(logits, labels, rows, ld, vocab, dlogits, loss_sum, scale,
                                 static_cast<cudaStream_t>(stream));
}
