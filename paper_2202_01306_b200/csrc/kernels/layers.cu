// layers.cu -- the bandwidth-bound kernels of a transformer layer pack:
// weight cast, embedding fwd/bwd, LayerNorm fwd/bwd, softmax cross-entropy
// fwd+bwd, bias gradients.  All are HBM-bound row/column kernels: one warp
// per row, 16-byte vector accesses, fp32 math.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "../runtime/common.hpp"
#include "pdl.cuh"

namespace hm {
namespace layers {

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

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ---- fp32 -> bf16 cast (pack weights after swap-in; dY before GEMMs) --------
__global__ void cast_kernel(const float4 *__restrict__ src, uint2 *__restrict__ dst, int64_t n4) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = src[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    dst[i] = make_uint2(*reinterpret_cast<uint32_t *>(&a), *reinterpret_cast<uint32_t *>(&b));
  }
}
__global__ void cast_tail(const float *src, __nv_bfloat16 *dst, int64_t begin, int64_t n) {
  pdl_wait();
  int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = __float2bfloat16_rn(src[i]);
}

int cast_f32_bf16(const float *src, void *dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return HM_OK;
  ProfScope ps(KC_MISC, s, 0, 6.0 * n);
  const int64_t n4 = ((uintptr_t)src & 15) || ((uintptr_t)dst & 7) ? 0 : n / 4;
  if (n4) {
    int64_t blocks = (n4 + 255) / 256;
    if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
    HM_CUDA(launch_pdl(cast_kernel, dim3((unsigned)blocks), dim3(256), 0, s, reinterpret_cast<const float4 *>(src), reinterpret_cast<uint2 *>(dst), n4));
    count_launch();
  }
  if (n4 * 4 < n) {
    const int64_t rest = n - n4 * 4;
    HM_CUDA(launch_pdl(cast_tail, dim3((unsigned)((rest + 255) / 256)), dim3(256), 0, s, src, static_cast<__nv_bfloat16 *>(dst), n4 * 4, n));
    count_launch();
  }
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

// ---- weight planes (bf16 swap-payload mode) ---------------------------------------
// An fp32 weight w splits exactly into hi = bf16(w) rounded to nearest with
// ties toward zero magnitude -- (bits + 0x7FFF) >> 16 -- and lo = the low 16
// bits of w: bits = (hi << 16) + d with d = lo if lo <= 0x8000, else lo - 0x10000
// (d in [-0x7FFF, 0x8000]).  hi is the GEMM operand itself, so a forward task
// that only needs bf16 weights moves half the bytes; cast_w_bf16 (the
// reference-payload path) produces the same hi, so both modes compute
// bit-identically.
__device__ __forceinline__ uint32_t w_hi(uint32_t u) { return (u + 0x7FFFu) >> 16; }
__device__ __forceinline__ uint32_t w_join1(uint32_t hi, uint32_t lo) {
  return (hi << 16) + (lo <= 0x8000u ? lo : lo - 0x10000u);
}

__global__ void cast_w_kernel(const uint4 *__restrict__ src, uint2 *__restrict__ dst, int64_t n4) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    dst[i] = make_uint2(w_hi(v.x) | (w_hi(v.y) << 16), w_hi(v.z) | (w_hi(v.w) << 16));
  }
}

__global__ void w_join_kernel(const uint16_t *__restrict__ hi, const uint16_t *__restrict__ lo, uint32_t *__restrict__ w,
                              int64_t n) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = w_join1(hi[i], lo[i]);
}

__global__ void w_split_kernel(const uint32_t *__restrict__ w, uint16_t *__restrict__ hi, uint16_t *__restrict__ lo,
                               int64_t n) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = w[i];
    hi[i] = (uint16_t)w_hi(u);
    lo[i] = (uint16_t)(u & 0xFFFFu);
  }
}

static unsigned elem_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > (int64_t)sm_count() * 16) b = (int64_t)sm_count() * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

int cast_w_bf16(const float *src, void *dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return HM_OK;
  if (n % 4 || ((uintptr_t)src & 15) || ((uintptr_t)dst & 7))  // weight slots are 256-B aligned, packs n % 8 == 0
    return fail(HM_ERR_VALIDATION, "cast_w_bf16: weights must be 16-B aligned, n % 4 == 0");
  ProfScope ps(KC_MISC, s, 0, 6.0 * n);
  HM_CUDA(launch_pdl(cast_w_kernel, dim3(elem_blocks(n / 4)), dim3(256), 0, s, reinterpret_cast<const uint4 *>(src),
                     static_cast<uint2 *>(dst), n / 4));
  count_launch();
  return HM_OK;
}

int w_join(const void *hi, const void *lo, float *w, int64_t n, cudaStream_t s) {
  if (n <= 0) return HM_OK;
  ProfScope ps(KC_MISC, s, 0, 8.0 * n);
  HM_CUDA(launch_pdl(w_join_kernel, dim3(elem_blocks(n)), dim3(256), 0, s, static_cast<const uint16_t *>(hi),
                     static_cast<const uint16_t *>(lo), reinterpret_cast<uint32_t *>(w), n));
  count_launch();
  return HM_OK;
}

int w_split(const float *w, void *hi, void *lo, int64_t n, cudaStream_t s) {
  if (n <= 0) return HM_OK;
  ProfScope ps(KC_MISC, s, 0, 8.0 * n);
  HM_CUDA(launch_pdl(w_split_kernel, dim3(elem_blocks(n)), dim3(256), 0, s, reinterpret_cast<const uint32_t *>(w),
                     static_cast<uint16_t *>(hi), static_cast<uint16_t *>(lo), n));
  count_launch();
  return HM_OK;
}

// ---- embedding -----------------------------------------------------------------
__global__ void embed_fwd_kernel(const int32_t *__restrict__ tok, const float *__restrict__ wte,
                                 const float *__restrict__ wpe, float *__restrict__ out, int64_t rows, int S, int d) {
  pdl_wait();
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float4 *a = reinterpret_cast<const float4 *>(wte + (int64_t)tok[r] * d);
  const float4 *b = reinterpret_cast<const float4 *>(wpe + (int64_t)(r % S) * d);
  float4 *o = reinterpret_cast<float4 *>(out + r * d);
  for (int i = lane; i < d / 4; i += 32) {
    float4 x = a[i], y = b[i];
    o[i] = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
  }
}
// dwte[tok] += dx (atomic; tokens repeat), one warp per row
__global__ void embed_bwd_tok_kernel(const int32_t *__restrict__ tok, const float *__restrict__ dx,
                                     float *__restrict__ dwte, int64_t rows, int d) {
  pdl_wait();
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float *dst = dwte + (int64_t)tok[r] * d;
  const float *src = dx + r * d;
  for (int i = lane; i < d; i += 32) atomicAdd(dst + i, src[i]);
}
// dwpe[p] += sum_b dx[b*S + p] (deterministic, no atomics)
__global__ void embed_bwd_pos_kernel(const float *__restrict__ dx, float *__restrict__ dwpe, int B, int S, int d) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)S * d) return;
  float acc = 0.f;
  for (int b = 0; b < B; ++b) acc += dx[(int64_t)b * S * d + i];
  dwpe[i] += acc;
}

int embed_fwd(const int32_t *tok, const float *wte, const float *wpe, float *out, int B, int S, int d, cudaStream_t s) {
  const int64_t rows = (int64_t)B * S;
  ProfScope ps(KC_MISC, s, 0, 12.0 * rows * d);
  HM_CUDA(launch_pdl(embed_fwd_kernel, dim3((unsigned)((rows * 32 + 255) / 256)), dim3(256), 0, s, tok, wte, wpe, out, rows, S, d));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}
int embed_bwd(const int32_t *tok, const float *dx, float *dwte, float *dwpe, int B, int S, int d, cudaStream_t s) {
  const int64_t rows = (int64_t)B * S;
  ProfScope ps(KC_MISC, s, 0, 16.0 * rows * d);
  HM_CUDA(launch_pdl(embed_bwd_tok_kernel, dim3((unsigned)((rows * 32 + 255) / 256)), dim3(256), 0, s, tok, dx, dwte, rows, d));
  embed_bwd_pos_kernel<<<(unsigned)(((int64_t)S * d + 255) / 256), 256, 0, s>>>(dx, dwpe, B, S, d);
  count_launch(2);
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

// ---- LayerNorm forward: fp32 x -> bf16 y (GEMM operand), mean/rstd saved ---------
__global__ void ln_fwd_kernel(const float *__restrict__ x, const float *__restrict__ gam, const float *__restrict__ bet,
                              __nv_bfloat16 *__restrict__ y, float *__restrict__ mean, float *__restrict__ rstd,
                              int64_t rows, int d, float eps) {
  pdl_wait();
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
  const int n4 = d / 4;
  float s = 0.f;
  for (int i = lane; i < n4; i += 32) {
    float4 v = xr[i];
    s += v.x + v.y + v.z + v.w;
  }
  const float mu = warp_sum(s) / d;
  float q = 0.f;
  for (int i = lane; i < n4; i += 32) {
    float4 v = xr[i];
    q += (v.x - mu) * (v.x - mu) + (v.y - mu) * (v.y - mu) + (v.z - mu) * (v.z - mu) + (v.w - mu) * (v.w - mu);
  }
  const float rs = rsqrtf(warp_sum(q) / d + eps);
  uint2 *yr = reinterpret_cast<uint2 *>(y + r * d);
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  const float4 *b4 = reinterpret_cast<const float4 *>(bet);
  for (int i = lane; i < n4; i += 32) {
    float4 v = xr[i], gg = g4[i], bb = b4[i];
    __nv_bfloat162 a = __floats2bfloat162_rn((v.x - mu) * rs * gg.x + bb.x, (v.y - mu) * rs * gg.y + bb.y);
    __nv_bfloat162 c = __floats2bfloat162_rn((v.z - mu) * rs * gg.z + bb.z, (v.w - mu) * rs * gg.w + bb.w);
    yr[i] = make_uint2(*reinterpret_cast<uint32_t *>(&a), *reinterpret_cast<uint32_t *>(&c));
  }
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

// Row-in-registers variant (d <= 128 * NV4): x is read from HBM exactly once
// (all NV4 float4 loads of a lane issued together), mean and variance come
// from the registers, and gamma / beta are L2-resident.
template <int NV4>
__global__ void __launch_bounds__(256) ln_fwd_reg_kernel(const float *__restrict__ x, const float *__restrict__ gam,
                                                         const float *__restrict__ bet, __nv_bfloat16 *__restrict__ y,
                                                         float *__restrict__ mean, float *__restrict__ rstd,
                                                         int64_t rows, int d, float eps) {
  pdl_wait();
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
  const int n4 = d / 4;
  float4 v[NV4];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = lane + 32 * k;
    v[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int k = 0; k < NV4; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  const float mu = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k)
    if (lane + 32 * k < n4) {
      const float a = v[k].x - mu, b = v[k].y - mu, c = v[k].z - mu, e = v[k].w - mu;
      q += (a * a + b * b) + (c * c + e * e);
    }
  const float rs = rsqrtf(warp_sum(q) / d + eps);
  uint2 *yr = reinterpret_cast<uint2 *>(y + r * d);
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  const float4 *b4 = reinterpret_cast<const float4 *>(bet);
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = lane + 32 * k;
    if (i < n4) {
      const float4 gg = __ldg(g4 + i), bb = __ldg(b4 + i);
      __nv_bfloat162 a = __floats2bfloat162_rn((v[k].x - mu) * rs * gg.x + bb.x, (v[k].y - mu) * rs * gg.y + bb.y);
      __nv_bfloat162 c = __floats2bfloat162_rn((v[k].z - mu) * rs * gg.z + bb.z, (v[k].w - mu) * rs * gg.w + bb.w);
      yr[i] = make_uint2(*reinterpret_cast<uint32_t *>(&a), *reinterpret_cast<uint32_t *>(&c));
    }
  }
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

// Rows of 1024 < d <= 2048 (GPT-2 XL's 1600): two warps per row, four rows per
// 256-thread block, half the row's float4 per lane (the one-warp kernel holds
// 13 float4 per lane at d = 1600 and keeps fewer rows in flight); mean and
// variance combine across the pair under a named barrier.
template <int NV4>
__global__ void __launch_bounds__(256) ln_fwd_pair_kernel(const float *__restrict__ x, const float *__restrict__ gam,
                                                          const float *__restrict__ bet, __nv_bfloat16 *__restrict__ y,
                                                          float *__restrict__ mean, float *__restrict__ rstd,
                                                          int64_t rows, int d, float eps) {
  pdl_wait();
  __shared__ float red[2][4][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = warp >> 1, wi = warp & 1;
  const int64_t r = (int64_t)blockIdx.x * 4 + grp;
  if (r >= rows) return;  // both warps of the row leave together
  const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
  const int n4 = d / 4;
  float4 v[NV4];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = wi * 32 + lane + 64 * k;
    v[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int k = 0; k < NV4; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  s = warp_sum(s);
  if (lane == 0) red[0][grp][wi] = s;
  asm volatile("bar.sync %0, 64;" ::"r"(1 + grp) : "memory");
  const float mu = (red[0][grp][0] + red[0][grp][1]) / d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k)
    if (wi * 32 + lane + 64 * k < n4) {
      const float a = v[k].x - mu, b = v[k].y - mu, c = v[k].z - mu, e = v[k].w - mu;
      q += (a * a + b * b) + (c * c + e * e);
    }
  q = warp_sum(q);
  if (lane == 0) red[1][grp][wi] = q;
  asm volatile("bar.sync %0, 64;" ::"r"(1 + grp) : "memory");
  const float rs = rsqrtf((red[1][grp][0] + red[1][grp][1]) / d + eps);
  uint2 *yr = reinterpret_cast<uint2 *>(y + r * d);
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  const float4 *b4 = reinterpret_cast<const float4 *>(bet);
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = wi * 32 + lane + 64 * k;
    if (i < n4) {
      const float4 gg = __ldg(g4 + i), bb = __ldg(b4 + i);
      __nv_bfloat162 a = __floats2bfloat162_rn((v[k].x - mu) * rs * gg.x + bb.x, (v[k].y - mu) * rs * gg.y + bb.y);
      __nv_bfloat162 c = __floats2bfloat162_rn((v[k].z - mu) * rs * gg.z + bb.z, (v[k].w - mu) * rs * gg.w + bb.w);
      yr[i] = make_uint2(*reinterpret_cast<uint32_t *>(&a), *reinterpret_cast<uint32_t *>(&c));
    }
  }
  if (lane == 0 && wi == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

// Wide rows (d > 2048, e.g. 8192): one 256-thread block per row, the row in
// registers (NV4 float4 per thread, all loads in flight), mean and variance by
// two block reductions -- one HBM read of x instead of three L2 passes.
template <int NV4>
__global__ void __launch_bounds__(256) ln_fwd_wide_kernel(const float *__restrict__ x, const float *__restrict__ gam,
                                                          const float *__restrict__ bet, __nv_bfloat16 *__restrict__ y,
                                                          float *__restrict__ mean, float *__restrict__ rstd,
                                                          int64_t rows, int d, float eps) {
  pdl_wait();
  __shared__ float red[2][8];
  const int64_t r = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
  const int n4 = d / 4;
  float4 v[NV4];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = t + 256 * k;
    v[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int k = 0; k < NV4; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  s = warp_sum(s);
  if (lane == 0) red[0][warp] = s;
  __syncthreads();
  s = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[0][w];
  const float mu = s / d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k)
    if (t + 256 * k < n4) {
      const float a = v[k].x - mu, b = v[k].y - mu, c = v[k].z - mu, e = v[k].w - mu;
      q += (a * a + b * b) + (c * c + e * e);
    }
  q = warp_sum(q);
  if (lane == 0) red[1][warp] = q;
  __syncthreads();
  q = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) q += red[1][w];
  const float rs = rsqrtf(q / d + eps);
  uint2 *yr = reinterpret_cast<uint2 *>(y + r * d);
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  const float4 *b4 = reinterpret_cast<const float4 *>(bet);
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = t + 256 * k;
    if (i < n4) {
      const float4 gg = __ldg(g4 + i), bb = __ldg(b4 + i);
      __nv_bfloat162 a = __floats2bfloat162_rn((v[k].x - mu) * rs * gg.x + bb.x, (v[k].y - mu) * rs * gg.y + bb.y);
      __nv_bfloat162 c = __floats2bfloat162_rn((v[k].z - mu) * rs * gg.z + bb.z, (v[k].w - mu) * rs * gg.w + bb.w);
      yr[i] = make_uint2(*reinterpret_cast<uint32_t *>(&a), *reinterpret_cast<uint32_t *>(&c));
    }
  }
  if (t == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

int ln_fwd(const float *x, const float *g, const float *b, void *y, float *mean, float *rstd, int64_t rows, int d,
           cudaStream_t s) {
  if (d % 4) return fail(HM_ERR_VALIDATION, "layernorm: d must be a multiple of 4");
  ProfScope ps(KC_LAYERNORM, s, 0, 6.0 * rows * d);
  static const int impl = getenv("HM_LN_FWD") ? atoi(getenv("HM_LN_FWD")) : 1;  // 0 = three-pass kernel
  if (impl) {
    const dim3 grid((unsigned)((rows * 32 + 255) / 256)), block(256);
    auto yy = static_cast<__nv_bfloat16 *>(y);
    const int nv4 = (d / 4 + 31) / 32;
    cudaError_t e = cudaErrorInvalidValue;
    if (d > 1024 && d <= 2048) {  // two warps per row (4096 x 1600: see profiles/r02_ln_perf*)
      const dim3 grid2((unsigned)((rows + 3) / 4));
      const int p4 = (d / 4 + 63) / 64;
      HM_CUDA(launch_pdl(p4 <= 7 ? ln_fwd_pair_kernel<7> : ln_fwd_pair_kernel<8>, grid2, block, 0, s, x, g, b, yy, mean,
                         rstd, rows, d, 1e-5f));
      count_launch();
      return HM_OK;
    }
    if (nv4 <= 4) e = launch_pdl(ln_fwd_reg_kernel<4>, grid, block, 0, s, x, g, b, yy, mean, rstd, rows, d, 1e-5f);
    else if (nv4 <= 8) e = launch_pdl(ln_fwd_reg_kernel<8>, grid, block, 0, s, x, g, b, yy, mean, rstd, rows, d, 1e-5f);
    else if (nv4 <= 13) e = launch_pdl(ln_fwd_reg_kernel<13>, grid, block, 0, s, x, g, b, yy, mean, rstd, rows, d, 1e-5f);
    else if (nv4 <= 16) e = launch_pdl(ln_fwd_reg_kernel<16>, grid, block, 0, s, x, g, b, yy, mean, rstd, rows, d, 1e-5f);
    if (nv4 <= 16) {
      HM_CUDA(e);
      count_launch();
      return HM_OK;
    }
    const int w4 = (d / 4 + 255) / 256;  // float4 per thread, one block per row
    if (w4 <= 8) {
      HM_CUDA(launch_pdl(w4 <= 4 ? ln_fwd_wide_kernel<4> : ln_fwd_wide_kernel<8>, dim3((unsigned)rows), dim3(256), 0,
                         s, x, g, b, yy, mean, rstd, rows, d, 1e-5f));
      count_launch();
      return HM_OK;
    }
  }
  HM_CUDA(launch_pdl(ln_fwd_kernel, dim3((unsigned)((rows * 32 + 255) / 256)), dim3(256), 0, s, x, g, b, static_cast<__nv_bfloat16 *>(y), mean,
                                                                    rstd, rows, d, 1e-5f));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

// ---- LayerNorm backward -------------------------------------------------------------
// dx = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)),  dxhat = dy * gamma
// out = dx + resid (resid may alias out or be null); optional bf16 copy of out;
// dgamma += sum dy*xhat, dbeta += sum dy (block partials in smem, then atomics).
__global__ void ln_bwd_kernel(const float *__restrict__ dy, const float *__restrict__ x, const float *__restrict__ mean,
                              const float *__restrict__ rstd, const float *__restrict__ gam, const float *resid,
                              float *out, __nv_bfloat16 *__restrict__ out_bf, float *__restrict__ dgam,
                              float *__restrict__ dbet, int64_t rows, int d, int rows_per_block) {
  pdl_wait();
  extern __shared__ float sacc[];  // [2*d]
  for (int i = threadIdx.x; i < 2 * d; i += blockDim.x) sacc[i] = 0.f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r_end = min(rows, r_begin + rows_per_block);
  const int n4 = d / 4;
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  for (int64_t r = r_begin + warp; r < r_end; r += nw) {
    const float4 *dyr = reinterpret_cast<const float4 *>(dy + r * d);
    const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
    const float mu = mean[r], rs = rstd[r];
    float c1 = 0.f, c2 = 0.f;
    for (int i = lane; i < n4; i += 32) {
      float4 a = dyr[i], v = xr[i], gg = g4[i];
      float h0 = (v.x - mu) * rs, h1 = (v.y - mu) * rs, h2 = (v.z - mu) * rs, h3 = (v.w - mu) * rs;
      float e0 = a.x * gg.x, e1 = a.y * gg.y, e2 = a.z * gg.z, e3 = a.w * gg.w;
      c1 += e0 + e1 + e2 + e3;
      c2 += e0 * h0 + e1 * h1 + e2 * h2 + e3 * h3;
      atomicAdd(&sacc[4 * i], a.x * h0);
      atomicAdd(&sacc[4 * i + 1], a.y * h1);
      atomicAdd(&sacc[4 * i + 2], a.z * h2);
      atomicAdd(&sacc[4 * i + 3], a.w * h3);
      atomicAdd(&sacc[d + 4 * i], a.x);
      atomicAdd(&sacc[d + 4 * i + 1], a.y);
      atomicAdd(&sacc[d + 4 * i + 2], a.z);
      atomicAdd(&sacc[d + 4 * i + 3], a.w);
    }
    c1 = warp_sum(c1) / d;
    c2 = warp_sum(c2) / d;
    float4 *outr = reinterpret_cast<float4 *>(out + r * d);
    const float4 *rr = resid ? reinterpret_cast<const float4 *>(resid + r * d) : nullptr;
    uint2 *ob = out_bf ? reinterpret_cast<uint2 *>(out_bf + r * d) : nullptr;
    for (int i = lane; i < n4; i += 32) {
      float4 a = dyr[i], v = xr[i], gg = g4[i];
      float4 o;
      o.x = rs * (a.x * gg.x - c1 - (v.x - mu) * rs * c2);
      o.y = rs * (a.y * gg.y - c1 - (v.y - mu) * rs * c2);
      o.z = rs * (a.z * gg.z - c1 - (v.z - mu) * rs * c2);
      o.w = rs * (a.w * gg.w - c1 - (v.w - mu) * rs * c2);
      if (rr) {
        float4 q = rr[i];
        o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
      }
      outr[i] = o;
      if (ob) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(o.x, o.y), p1 = __floats2bfloat162_rn(o.z, o.w);
        ob[i] = make_uint2(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    atomicAdd(&dgam[i], sacc[i]);
    atomicAdd(&dbet[i], sacc[d + i]);
  }
}

// Default LayerNorm backward: one warp per row, WARPS warps per block.  Each
// warp keeps PRIVATE dgamma/dbeta partials in shared memory (its lanes own
// fixed float4 columns, so plain read-modify-writes, no atomics: shared-memory
// float atomics compile to CAS spin loops on sm_100a), the block sums its warps'
// partials once and adds them to global memory (one atomic per column per
// block).  The second pass re-reads dy / x from L1 / L2.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    ln_bwd_warp_kernel(const float *__restrict__ dy, const float *__restrict__ x, const float *__restrict__ mean,
                       const float *__restrict__ rstd, const float *__restrict__ gam, const float *resid, float *out,
                       __nv_bfloat16 *__restrict__ out_bf, float *__restrict__ dgam, float *__restrict__ dbet,
                       int64_t rows, int d, int rows_per_block) {
  pdl_wait();
  extern __shared__ float4 spart4[];  // [WARPS][2][d / 4]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n4 = d / 4;
  float4 *pg = spart4 + (size_t)warp * 2 * n4;
  float4 *pb = pg + n4;
  for (int i = lane; i < n4; i += 32) pg[i] = pb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r_end = min(rows, r_begin + rows_per_block);
  for (int64_t r = r_begin + warp; r < r_end; r += WARPS) {
    const float4 *dyr = reinterpret_cast<const float4 *>(dy + r * d);
    const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
    const float mu = mean[r], rs = rstd[r];
    float c1 = 0.f, c2 = 0.f;
#pragma unroll 4
    for (int i = lane; i < n4; i += 32) {
      const float4 a = dyr[i], v = xr[i], gg = g4[i];
      const float h0 = (v.x - mu) * rs, h1 = (v.y - mu) * rs, h2 = (v.z - mu) * rs, h3 = (v.w - mu) * rs;
      const float e0 = a.x * gg.x, e1 = a.y * gg.y, e2 = a.z * gg.z, e3 = a.w * gg.w;
      c1 += (e0 + e1) + (e2 + e3);
      c2 += (e0 * h0 + e1 * h1) + (e2 * h2 + e3 * h3);
      float4 q = pg[i];
      q.x += a.x * h0; q.y += a.y * h1; q.z += a.z * h2; q.w += a.w * h3;
      pg[i] = q;
      float4 t = pb[i];
      t.x += a.x; t.y += a.y; t.z += a.z; t.w += a.w;
      pb[i] = t;
    }
    c1 = warp_sum(c1) / d;
    c2 = warp_sum(c2) / d;
    float4 *outr = reinterpret_cast<float4 *>(out + r * d);
    const float4 *rr = resid ? reinterpret_cast<const float4 *>(resid + r * d) : nullptr;
    uint2 *ob = out_bf ? reinterpret_cast<uint2 *>(out_bf + r * d) : nullptr;
#pragma unroll 4
    for (int i = lane; i < n4; i += 32) {
      const float4 a = dyr[i], v = xr[i], gg = g4[i];
      float4 o;
      o.x = rs * (a.x * gg.x - c1 - (v.x - mu) * rs * c2);
      o.y = rs * (a.y * gg.y - c1 - (v.y - mu) * rs * c2);
      o.z = rs * (a.z * gg.z - c1 - (v.z - mu) * rs * c2);
      o.w = rs * (a.w * gg.w - c1 - (v.w - mu) * rs * c2);
      if (rr) {
        const float4 q = rr[i];
        o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
      }
      outr[i] = o;
      if (ob) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(o.x, o.y), p1 = __floats2bfloat162_rn(o.z, o.w);
        ob[i] = make_uint2(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1));
      }
    }
  }
  __syncthreads();
  const float *sp = reinterpret_cast<const float *>(spart4);
  for (int c = threadIdx.x; c < d; c += WARPS * 32) {
    float sg = 0.f, sb = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      sg += sp[(size_t)w * 2 * d + c];
      sb += sp[(size_t)w * 2 * d + d + c];
    }
    atomicAdd(&dgam[c], sg);
    atomicAdd(&dbet[c], sb);
  }
}

// Register-resident variant of ln_bwd_warp_kernel (d <= 1024): each lane loads
// its NV4 float4 columns of dy and x once, all loads in flight together, and
// computes dx from registers -- one HBM read of each row instead of a second
// pass through L2.
template <int NV4, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    ln_bwd_rowreg_kernel(const float *__restrict__ dy, const float *__restrict__ x, const float *__restrict__ mean,
                         const float *__restrict__ rstd, const float *__restrict__ gam, const float *resid, float *out,
                         __nv_bfloat16 *__restrict__ out_bf, float *__restrict__ dgam, float *__restrict__ dbet,
                         int64_t rows, int d, int rows_per_block) {
  pdl_wait();
  extern __shared__ float4 spart4[];  // [WARPS][2][d / 4]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n4 = d / 4;
  float4 *pg = spart4 + (size_t)warp * 2 * n4;
  float4 *pb = pg + n4;
  for (int i = lane; i < n4; i += 32) pg[i] = pb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r_end = min(rows, r_begin + rows_per_block);
  for (int64_t r = r_begin + warp; r < r_end; r += WARPS) {
    const float4 *dyr = reinterpret_cast<const float4 *>(dy + r * d);
    const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
    float4 a[NV4], v[NV4];
#pragma unroll
    for (int k = 0; k < NV4; ++k) {
      const int i = lane + 32 * k;
      if (i < n4) {
        a[k] = dyr[i];
        v[k] = xr[i];
      }
    }
    const float mu = mean[r], rs = rstd[r];
    float c1 = 0.f, c2 = 0.f;
#pragma unroll
    for (int k = 0; k < NV4; ++k) {
      const int i = lane + 32 * k;
      if (i < n4) {
        const float4 gg = g4[i];
        v[k].x = (v[k].x - mu) * rs; v[k].y = (v[k].y - mu) * rs;  // v := xhat
        v[k].z = (v[k].z - mu) * rs; v[k].w = (v[k].w - mu) * rs;
        const float e0 = a[k].x * gg.x, e1 = a[k].y * gg.y, e2 = a[k].z * gg.z, e3 = a[k].w * gg.w;
        c1 += (e0 + e1) + (e2 + e3);
        c2 += (e0 * v[k].x + e1 * v[k].y) + (e2 * v[k].z + e3 * v[k].w);
        float4 q = pg[i];
        q.x += a[k].x * v[k].x; q.y += a[k].y * v[k].y; q.z += a[k].z * v[k].z; q.w += a[k].w * v[k].w;
        pg[i] = q;
        float4 t = pb[i];
        t.x += a[k].x; t.y += a[k].y; t.z += a[k].z; t.w += a[k].w;
        pb[i] = t;
      }
    }
    c1 = warp_sum(c1) / d;
    c2 = warp_sum(c2) / d;
    float4 *outr = reinterpret_cast<float4 *>(out + r * d);
    const float4 *rr = resid ? reinterpret_cast<const float4 *>(resid + r * d) : nullptr;
    uint2 *ob = out_bf ? reinterpret_cast<uint2 *>(out_bf + r * d) : nullptr;
#pragma unroll
    for (int k = 0; k < NV4; ++k) {
      const int i = lane + 32 * k;
      if (i < n4) {
        const float4 gg = g4[i];
        float4 o;
        o.x = rs * (a[k].x * gg.x - c1 - v[k].x * c2);
        o.y = rs * (a[k].y * gg.y - c1 - v[k].y * c2);
        o.z = rs * (a[k].z * gg.z - c1 - v[k].z * c2);
        o.w = rs * (a[k].w * gg.w - c1 - v[k].w * c2);
        if (rr) {
          const float4 q = rr[i];
          o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
        }
        outr[i] = o;
        if (ob) {
          __nv_bfloat162 p0 = __floats2bfloat162_rn(o.x, o.y), p1 = __floats2bfloat162_rn(o.z, o.w);
          ob[i] = make_uint2(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1));
        }
      }
    }
  }
  __syncthreads();
  const float *sp = reinterpret_cast<const float *>(spart4);
  for (int c = threadIdx.x; c < d; c += WARPS * 32) {
    float sg = 0.f, sb = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      sg += sp[(size_t)w * 2 * d + c];
      sb += sp[(size_t)w * 2 * d + d + c];
    }
    atomicAdd(&dgam[c], sg);
    atomicAdd(&dbet[c], sb);
  }
}

template <int NV4>
static int ln_bwd_rowreg(const float *dy, const float *x, const float *mean, const float *rstd, const float *g,
                         const float *resid, float *out, void *out_bf, float *dg, float *db, int64_t rows, int d,
                         cudaStream_t s) {
  constexpr int kWarps = 4;
  const size_t smem = (size_t)kWarps * 2 * d * sizeof(float);
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    HM_CUDA(cudaFuncSetAttribute(ln_bwd_rowreg_kernel<NV4, kWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_smem = smem;
  }
  const int per_sm = std::max<int>(1, std::min<int>(4, (int)((200 * 1024) / smem)));
  int64_t blocks = (int64_t)sm_count() * per_sm;
  int rpb = (int)((rows + blocks - 1) / blocks);
  if (rpb < kWarps) rpb = kWarps;
  blocks = (rows + rpb - 1) / rpb;
  HM_CUDA(launch_pdl(ln_bwd_rowreg_kernel<NV4, kWarps>, dim3((unsigned)blocks), dim3(kWarps * 32), smem, s, dy, x,
                     mean, rstd, g, resid, out, static_cast<__nv_bfloat16 *>(out_bf), dg, db, rows, d, rpb));
  count_launch();
  return HM_OK;
}

// Register-resident rows wider than one warp can hold (d > 1024): a row is
// split over WPR warps (lane l of warp w of the row group owns float4 columns
// 32 w + l, + 32 WPR, ...), so dy and x are read from HBM exactly once with
// all loads in flight; the row statistics c1 / c2 combine across the group's
// warps through shared memory under a named barrier, and dgamma / dbeta
// accumulate in registers over every row the group visits (fixed columns per
// lane), folded per block in shared memory and added to global memory once
// per column per block.
template <int NV4, int WARPS, int WPR>
__global__ void __launch_bounds__(WARPS * 32)
    ln_bwd_wide_kernel(const float *__restrict__ dy, const float *__restrict__ x, const float *__restrict__ mean,
                       const float *__restrict__ rstd, const float *__restrict__ gam, const float *resid, float *out,
                       __nv_bfloat16 *__restrict__ out_bf, float *__restrict__ dgam, float *__restrict__ dbet,
                       int64_t rows, int d, int rows_per_block) {
  constexpr int G = WARPS / WPR;  // row groups per block
  pdl_wait();
  extern __shared__ float sred[];  // [2][G][WPR][2] row statistics, then [G][2][d] dgamma / dbeta partials
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / WPR, wi = warp % WPR;
  const int n4 = d / 4;
  const float4 *g4 = reinterpret_cast<const float4 *>(gam);
  float4 gg[NV4], accg[NV4], accb[NV4];
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = wi * 32 + lane + 32 * WPR * k;
    gg[k] = i < n4 ? g4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    accg[k] = accb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r_end = min(rows, r_begin + rows_per_block);
  int par = 0;
  for (int64_t r = r_begin + grp; r < r_end; r += G, par ^= 1) {
    const float4 *dyr = reinterpret_cast<const float4 *>(dy + r * d);
    const float4 *xr = reinterpret_cast<const float4 *>(x + r * d);
    const float4 *rr = resid ? reinterpret_cast<const float4 *>(resid + r * d) : nullptr;
    // dy, x and the residual all in flight before the first use (the residual
    // would otherwise be a second dependent HBM round trip after the barrier)
    float4 a[NV4], v[NV4], q[NV4];
#pragma unroll
    for (int k = 0; k < NV4; ++k) {
      const int i = wi * 32 + lane + 32 * WPR * k;
      if (i < n4) {
        a[k] = dyr[i];
        v[k] = xr[i];
        q[k] = rr ? rr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        a[k] = v[k] = q[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    const float mu = mean[r], rs = rstd[r];
    float c1 = 0.f, c2 = 0.f;
#pragma unroll
    for (int k = 0; k < NV4; ++k) {
      v[k].x = (v[k].x - mu) * rs; v[k].y = (v[k].y - mu) * rs;  // v := xhat (0 past the row end: a = 0 there)
      v[k].z = (v[k].z - mu) * rs; v[k].w = (v[k].w - mu) * rs;
      const float e0 = a[k].x * gg[k].x, e1 = a[k].y * gg[k].y, e2 = a[k].z * gg[k].z, e3 = a[k].w * gg[k].w;
      c1 += (e0 + e1) + (e2 + e3);
      c2 += (e0 * v[k].x + e1 * v[k].y) + (e2 * v[k].z + e3 * v[k].w);
      accg[k].x += a[k].x * v[k].x; accg[k].y += a[k].y * v[k].y;
      accg[k].z += a[k].z * v[k].z; accg[k].w += a[k].w * v[k].w;
      accb[k].x += a[k].x; accb[k].y += a[k].y; accb[k].z += a[k].z; accb[k].w += a[k].w;
    }
    c1 = warp_sum(c1);
    c2 = warp_sum(c2);
    float *red = sred + ((par * G + grp) * WPR) * 2;
    if (lane == 0) {
      red[2 * wi] = c1;
      red[2 * wi + 1] = c2;
    }
    // the row group's warps only (double-buffered by row parity: the next row's
    // writes go to the other buffer, the one after waits behind this barrier)
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(WPR * 32) : "memory");
    c1 = 0.f;
    c2 = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) {
      c1 += red[2 * w];
      c2 += red[2 * w + 1];
    }
    c1 /= d;
    c2 /= d;
    float4 *outr = reinterpret_cast<float4 *>(out + r * d);
    uint2 *ob = out_bf ? reinterpret_cast<uint2 *>(out_bf + r * d) : nullptr;
#pragma unroll
    for (int k = 0; k < NV4; ++k) {
      const int i = wi * 32 + lane + 32 * WPR * k;
      if (i < n4) {
        float4 o;
        o.x = rs * (a[k].x * gg[k].x - c1 - v[k].x * c2) + q[k].x;
        o.y = rs * (a[k].y * gg[k].y - c1 - v[k].y * c2) + q[k].y;
        o.z = rs * (a[k].z * gg[k].z - c1 - v[k].z * c2) + q[k].z;
        o.w = rs * (a[k].w * gg[k].w - c1 - v[k].w * c2) + q[k].w;
        outr[i] = o;
        if (ob) {
          __nv_bfloat162 p0 = __floats2bfloat162_rn(o.x, o.y), p1 = __floats2bfloat162_rn(o.z, o.w);
          ob[i] = make_uint2(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1));
        }
      }
    }
  }
  __syncthreads();
  float4 *part = reinterpret_cast<float4 *>(sred + 4 * G * WPR);  // [G][2][n4] float4
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int i = wi * 32 + lane + 32 * WPR * k;
    if (i < n4) {
      part[(size_t)(grp * 2) * n4 + i] = accg[k];
      part[(size_t)(grp * 2 + 1) * n4 + i] = accb[k];
    }
  }
  __syncthreads();
  const float *pf = reinterpret_cast<const float *>(part);
  for (int c = threadIdx.x; c < d; c += WARPS * 32) {
    float sg = 0.f, sb = 0.f;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      sg += pf[(size_t)(q * 2) * d + c];
      sb += pf[(size_t)(q * 2 + 1) * d + c];
    }
    atomicAdd(&dgam[c], sg);
    atomicAdd(&dbet[c], sb);
  }
}

template <int NV4, int WARPS, int WPR>
static int ln_bwd_wide(const float *dy, const float *x, const float *mean, const float *rstd, const float *g,
                       const float *resid, float *out, void *out_bf, float *dg, float *db, int64_t rows, int d,
                       cudaStream_t s) {
  constexpr int G = WARPS / WPR;
  const size_t smem = (size_t)4 * G * WPR * sizeof(float) + (size_t)G * 2 * d * sizeof(float) + 16;
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    HM_CUDA(cudaFuncSetAttribute(ln_bwd_wide_kernel<NV4, WARPS, WPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_smem = smem;
  }
  const int per_sm = std::max<int>(1, std::min<int>(4, (int)((200 * 1024) / smem)));
  int64_t blocks = (int64_t)sm_count() * per_sm;
  int rpb = (int)((rows + blocks - 1) / blocks);
  if (rpb < G) rpb = G;
  blocks = (rows + rpb - 1) / rpb;
  HM_CUDA(launch_pdl(ln_bwd_wide_kernel<NV4, WARPS, WPR>, dim3((unsigned)blocks), dim3(WARPS * 32), smem, s, dy, x,
                     mean, rstd, g, resid, out, static_cast<__nv_bfloat16 *>(out_bf), dg, db, rows, d, rpb));
  count_launch();
  return HM_OK;
}

int ln_bwd(const float *dy, const float *x, const float *mean, const float *rstd, const float *g, const float *resid,
           float *out, void *out_bf, float *dg, float *db, int64_t rows, int d, cudaStream_t s) {
  if (d % 4) return fail(HM_ERR_VALIDATION, "layernorm: d must be a multiple of 4");
  static const bool use_smem_atomic = [] {
    const char *e = getenv("HM_LN_BWD");
    return e && e[0] == 'a';
  }();
  static const bool use_two_pass = [] {
    const char *e = getenv("HM_LN_BWD");
    return e && e[0] == 'w';
  }();
  // Rows in registers: one warp per row up to d = 1024 (4096 x 1024: 17.9 vs 22.0
  // us for the shared-atomic kernel), 2 / 8 warps per row up to d = 8192 (4096 x
  // 1600: 26.0 vs 31.9 us for the two-pass kernel; 4096 x 8192: 98 vs 183 us,
  // profiles/r02_ln_perf*.jsonl).  HM_LN_BWD=w forces the two-pass kernel (dy / x
  // re-read from L2), a the shared-atomic one (also the fallback above d = 8192).
  if (!use_smem_atomic && !use_two_pass && d <= 1024) {
    ProfScope ps(KC_LAYERNORM, s, 0, (resid ? 16.0 : 12.0) * rows * d + (out_bf ? 2.0 * rows * d : 0));
    const int nv4 = (d / 4 + 31) / 32;
    if (nv4 <= 2) return ln_bwd_rowreg<2>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
    if (nv4 <= 4) return ln_bwd_rowreg<4>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
    return ln_bwd_rowreg<8>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
  }
  // wider rows (d > 1024) split over 2 (d <= 2048) or 8 (d <= 8192) warps, still
  // register-resident: one HBM read of dy / x
  static const bool use_wide = [] {
    const char *e = getenv("HM_LN_BWD");
    return !(e && e[0] == 'w');
  }();
  if (use_wide && !use_smem_atomic && d % 4 == 0 && d <= 8192) {
    ProfScope ps(KC_LAYERNORM, s, 0, (resid ? 16.0 : 12.0) * rows * d + (out_bf ? 2.0 * rows * d : 0));
    const int n4 = d / 4;
    if (d <= 2048) {
      if (n4 <= 64 * 4) return ln_bwd_wide<4, 8, 2>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
      if (n4 <= 64 * 7) return ln_bwd_wide<7, 8, 2>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
      return ln_bwd_wide<8, 8, 2>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
    }
    if (n4 <= 256 * 4) return ln_bwd_wide<4, 8, 8>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
    return ln_bwd_wide<8, 8, 8>(dy, x, mean, rstd, g, resid, out, out_bf, dg, db, rows, d, s);
  }
  if (!use_smem_atomic && (size_t)4 * 2 * d * sizeof(float) <= 160 * 1024) {  // 4 warps' private partials
    constexpr int kWarps = 4;
    const size_t smem = (size_t)kWarps * 2 * d * sizeof(float);
    static size_t attr_smem = 0;
    if (smem > attr_smem) {
      HM_CUDA(cudaFuncSetAttribute(ln_bwd_warp_kernel<kWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_smem = smem;
    }
    ProfScope ps(KC_LAYERNORM, s, 0, (resid ? 16.0 : 12.0) * rows * d + (out_bf ? 2.0 * rows * d : 0));
    const int per_sm = std::max<int>(1, std::min<int>(8, (int)((200 * 1024) / smem)));
    int64_t blocks = (int64_t)sm_count() * per_sm;
    int rpb = (int)((rows + blocks - 1) / blocks);
    if (rpb < kWarps) rpb = kWarps;
    blocks = (rows + rpb - 1) / rpb;
    HM_CUDA(launch_pdl(ln_bwd_warp_kernel<kWarps>, dim3((unsigned)blocks), dim3(kWarps * 32), smem, s, dy, x, mean,
                       rstd, g, resid, out, static_cast<__nv_bfloat16 *>(out_bf), dg, db, rows, d, rpb));
    count_launch();
    return HM_OK;
  }
  const size_t smem = 2 * (size_t)d * sizeof(float);
  static bool attr = false;
  if (!attr) {
    HM_CUDA(cudaFuncSetAttribute(ln_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  ProfScope ps(KC_LAYERNORM, s, 0, (resid ? 16.0 : 12.0) * rows * d + (out_bf ? 2.0 * rows * d : 0));
  int64_t blocks = sm_count() * 2;
  int rpb = (int)((rows + blocks - 1) / blocks);
  if (rpb < 8) rpb = 8;
  blocks = (rows + rpb - 1) / rpb;
  HM_CUDA(launch_pdl(ln_bwd_kernel, dim3((unsigned)blocks), dim3(512), smem, s, dy, x, mean, rstd, g, resid, out,
                                                    static_cast<__nv_bfloat16 *>(out_bf), dg, db, rows, d, rpb));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

// ---- softmax cross-entropy over the (padded) vocabulary -----------------------------
// logits fp32 [rows, ldl], valid columns [0, V); loss_sum += sum_r CE_r (double);
// dlogits bf16 [rows, ldl] = (softmax - onehot) * scale, zero in the padding.
// One block per row.  Pass 1: online (max, sum of exp) over float4 chunks,
// one rescale per 4 logits.  Pass 2 (row re-read, mostly from L2): softmax
// minus one-hot, scaled, written as bf16x4.  exp via exp2 of log2e-scaled
// values.  ldl % 4 == 0 and 16-B aligned rows (the padded vocabulary).
__device__ __forceinline__ void ce_merge(float &m, float &s, float mo, float so) {
  const float mn = fmaxf(m, mo);
  s = (m == -INFINITY ? 0.f : s * exp2f(m - mn)) + (mo == -INFINITY ? 0.f : so * exp2f(mo - mn));
  m = mn;
}

__global__ void __launch_bounds__(512) ce_kernel(const float *__restrict__ logits, const int32_t *__restrict__ labels,
                                                 int64_t ldl, int V, __nv_bfloat16 *__restrict__ dlog, double *loss_sum,
                                                 float scale) {
  pdl_wait();
  constexpr float kL2E = 1.4426950408889634f;
  const int64_t r = blockIdx.x;
  const float *row = logits + r * ldl;
  const float4 *row4 = reinterpret_cast<const float4 *>(row);
  __shared__ float red_m[32], red_s[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int V4 = V >> 2;  // whole float4 chunks inside the vocabulary
  float m = -INFINITY, s = 0.f;  // in log2 units: m = max(x * log2e)
#pragma unroll 4
  for (int i = threadIdx.x; i < V4; i += blockDim.x) {
    const float4 v = row4[i];
    const float a = v.x * kL2E, b = v.y * kL2E, c = v.z * kL2E, e = v.w * kL2E;
    const float mn = fmaxf(fmaxf(m, fmaxf(a, b)), fmaxf(c, e));
    s = (m == -INFINITY ? 0.f : s * exp2f(m - mn)) + ((exp2f(a - mn) + exp2f(b - mn)) + (exp2f(c - mn) + exp2f(e - mn)));
    m = mn;
  }
  for (int i = 4 * V4 + threadIdx.x; i < V; i += blockDim.x) ce_merge(m, s, row[i] * kL2E, 1.f);
#pragma unroll
  for (int o = 16; o; o >>= 1) ce_merge(m, s, __shfl_xor_sync(0xffffffff, m, o), __shfl_xor_sync(0xffffffff, s, o));
  if (lane == 0) {
    red_m[warp] = m;
    red_s[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < nw ? red_m[lane] : -INFINITY;
    s = lane < nw ? red_s[lane] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) ce_merge(m, s, __shfl_xor_sync(0xffffffff, m, o), __shfl_xor_sync(0xffffffff, s, o));
    if (lane == 0) {
      red_m[0] = m;
      red_s[0] = s;
    }
  }
  __syncthreads();
  m = red_m[0];
  s = red_s[0];
  const int lab = labels[r];
  const float inv = 1.f / s;
  uint2 *drow = reinterpret_cast<uint2 *>(dlog + r * ldl);
  const int L4 = (int)(ldl >> 2);
#pragma unroll 4
  for (int i = threadIdx.x; i < L4; i += blockDim.x) {
    const float4 v = row4[i];
    const int c0 = 4 * i;
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (c0 + k < V) g[k] = (exp2f(x[k] * kL2E - m) * inv - (c0 + k == lab ? 1.f : 0.f)) * scale;
    __nv_bfloat162 p0 = __floats2bfloat162_rn(g[0], g[1]), p1 = __floats2bfloat162_rn(g[2], g[3]);
    drow[i] = make_uint2(*reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1));
  }
  // loss = ln(sum e^x) - x_label = (m + log2 s) ln 2 - x_label
  if (threadIdx.x == 0) atomicAdd(loss_sum, (double)((m + log2f(s)) * 0.6931471805599453f - row[lab]));
}

int cross_entropy(const float *logits, const int32_t *labels, int64_t rows, int64_t ldl, int V, void *dlogits,
                  double *loss_sum, float scale, cudaStream_t s) {
  ProfScope ps(KC_XENT, s, 0, 6.0 * rows * ldl);
  if ((ldl & 3) || ((uintptr_t)logits & 15) || ((uintptr_t)dlogits & 7))
    return fail(HM_ERR_VALIDATION, "cross_entropy: rows must be 16-B aligned, ldl % 4 == 0");
  HM_CUDA(launch_pdl(ce_kernel, dim3((unsigned)rows), dim3(512), 0, s, logits, labels, ldl, V, static_cast<__nv_bfloat16 *>(dlogits), loss_sum,
                                            scale));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

// ---- bias gradient: db[n] += sum_r dy[r, n] ------------------------------------------
// Column sums of dy [rows, n] (leading dimension ld) into db.  A block is cx
// column threads x (256 / cx) row lanes (cx = 8, 16 or 32: narrow convolution
// biases get more row lanes): each thread owns 8 consecutive columns (one 16-B
// load per row for bf16, two for fp32) and every ry-th row of the block's row
// range, four rows in flight; the row lanes meet in shared memory and each
// block adds one partial per column (few atomics per address).
template <typename T>
__global__ void __launch_bounds__(256) bias_grad_kernel(const T *__restrict__ dy, float *__restrict__ db, int64_t rows,
                                                        int n, int64_t ld, int rows_per_block, int cx) {
  pdl_wait();
  __shared__ float part[256 * 8];
  const int ry = 256 / cx;
  const int tx = threadIdx.x % cx, ty = threadIdx.x / cx;
  const int col = (blockIdx.x * cx + tx) * 8;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (col < n) {
    auto add_row = [&](int64_t r) {
      if constexpr (sizeof(T) == 2) {
        const uint4 v = *reinterpret_cast<const uint4 *>(dy + r * ld + col);
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h[k]);
          a[2 * k] += f.x;
          a[2 * k + 1] += f.y;
        }
      } else {
        const float4 v0 = *reinterpret_cast<const float4 *>(dy + r * ld + col);
        const float4 v1 = *reinterpret_cast<const float4 *>(dy + r * ld + col + 4);
        a[0] += v0.x; a[1] += v0.y; a[2] += v0.z; a[3] += v0.w;
        a[4] += v1.x; a[5] += v1.y; a[6] += v1.z; a[7] += v1.w;
      }
    };
    int64_t r = r0 + ty;
    for (; r + 3 * ry < r1; r += 4 * ry) {
#pragma unroll
      for (int k = 0; k < 4; ++k) add_row(r + (int64_t)ry * k);
    }
    for (; r < r1; r += ry) add_row(r);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) part[ty * (cx * 8) + tx * 8 + k] = a[k];
  __syncthreads();
  const int c = threadIdx.x;  // the block's cx * 8 columns
  const int gc = blockIdx.x * cx * 8 + c;
  if (c < cx * 8 && gc < n) {
    float t = 0.f;
    for (int y = 0; y < ry; ++y) t += part[y * (cx * 8) + c];
    atomicAdd(db + gc, t);
  }
}

// (n % 8 != 0 or unaligned rows: two columns per thread)
template <typename T>
__global__ void bias_grad2_kernel(const T *__restrict__ dy, float *__restrict__ db, int64_t rows, int n, int64_t ld,
                                  int rows_per_block) {
  pdl_wait();
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (col >= n) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float a0 = 0.f, a1 = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    if constexpr (sizeof(T) == 2) {
      float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(dy + r * ld + col));
      a0 += v.x;
      a1 += v.y;
    } else {
      float2 v = *reinterpret_cast<const float2 *>(dy + r * ld + col);
      a0 += v.x;
      a1 += v.y;
    }
  }
  atomicAdd(db + col, a0);
  atomicAdd(db + col + 1, a1);
}

// ---- gradient sum over ranks (IPC test backend of the Harmony-DP all-reduce) ---------
struct RankSrcs {
  const float *p[8];
};
__global__ void sum_ranks_kernel(RankSrcs src, int n, float *__restrict__ out, int64_t count) {
  pdl_wait();
  const int64_t n4 = count / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4 *>(src.p[0])[i];
    for (int r = 1; r < n; ++r) {
      const float4 v = reinterpret_cast<const float4 *>(src.p[r])[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4 *>(out)[i] = acc;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = src.p[0][i];
    for (int r = 1; r < n; ++r) acc += src.p[r][i];
    out[i] = acc;
  }
}

int sum_ranks(const float *const *src, int n, float *out, int64_t count, cudaStream_t s) {
  if (n < 1 || n > 8) return fail(HM_ERR_VALIDATION, "sum_ranks: 1..8 sources");
  RankSrcs rs{};
  for (int r = 0; r < n; ++r) {
    if ((uintptr_t)src[r] & 15) return fail(HM_ERR_VALIDATION, "sum_ranks: sources must be 16-B aligned");
    rs.p[r] = src[r];
  }
  ProfScope ps(KC_MISC, s, 0, 4.0 * (n + 1) * count);
  const unsigned grid = (unsigned)std::min<int64_t>((count / 4 + 255) / 256 + 1, (int64_t)sm_count() * 8);
  HM_CUDA(launch_pdl(sum_ranks_kernel, dim3(grid), dim3(256), 0, s, rs, n, out, count));
  count_launch();
  return HM_OK;
}

int bias_grad(const void *dy, int is_bf16, float *db, int64_t rows, int n, int64_t ld, cudaStream_t s) {
  if (n % 2) return fail(HM_ERR_VALIDATION, "bias_grad: n must be even");
  ProfScope ps(KC_MISC, s, 0, (is_bf16 ? 2.0 : 4.0) * rows * n);
  const int esz = is_bf16 ? 2 : 4;
  const bool wide = n % 8 == 0 && (ld * esz) % 16 == 0 && ((uintptr_t)dy & 15) == 0;
  int gx, threads;
  int64_t gy;
  int cx = 32;
  if (wide) {  // cx column threads (8 columns each) x 256 / cx row lanes per block, ~4 blocks per SM
    while (cx > 8 && cx / 2 * 8 >= n) cx /= 2;
    threads = 256;
    gx = (n + cx * 8 - 1) / (cx * 8);
    gy = ((int64_t)sm_count() * 4 + gx - 1) / gx;
  } else {
    threads = 128;
    gx = (n / 2 + threads - 1) / threads;
    gy = ((int64_t)sm_count() * 8 + gx - 1) / gx;
  }
  int rpb = (int)((rows + gy - 1) / gy);
  if (rpb < 32) rpb = 32;
  gy = (rows + rpb - 1) / rpb;
  const dim3 grid(gx, (unsigned)gy);
  if (is_bf16) {
    if (wide)
      HM_CUDA(launch_pdl(bias_grad_kernel<__nv_bfloat16>, grid, dim3(threads), 0, s,
                         static_cast<const __nv_bfloat16 *>(dy), db, rows, n, ld, rpb, cx));
    else
      HM_CUDA(launch_pdl(bias_grad2_kernel<__nv_bfloat16>, grid, dim3(threads), 0, s,
                         static_cast<const __nv_bfloat16 *>(dy), db, rows, n, ld, rpb));
  } else {
    if (wide)
      HM_CUDA(launch_pdl(bias_grad_kernel<float>, grid, dim3(threads), 0, s, static_cast<const float *>(dy), db, rows,
                         n, ld, rpb, cx));
    else
      HM_CUDA(launch_pdl(bias_grad2_kernel<float>, grid, dim3(threads), 0, s, static_cast<const float *>(dy), db, rows,
                         n, ld, rpb));
  }
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

}  // namespace layers
}  // namespace hm

using namespace hm::layers;

extern "C" {
int hm_k_cast_bf16(const float *src, void *dst, int64_t n, void *stream) {
  return cast_f32_bf16(src, dst, n, static_cast<cudaStream_t>(stream));
}
int hm_k_cast_w_bf16(const float *src, void *dst, int64_t n, void *stream) {
  return cast_w_bf16(src, dst, n, static_cast<cudaStream_t>(stream));
}
int hm_k_w_split(const float *w, void *hi, void *lo, int64_t n, void *stream) {
  return w_split(w, hi, lo, n, static_cast<cudaStream_t>(stream));
}
int hm_k_w_join(const void *hi, const void *lo, float *w, int64_t n, void *stream) {
  return w_join(hi, lo, w, n, static_cast<cudaStream_t>(stream));
}
int hm_k_embed_fwd(const int32_t *tokens, const float *wte, const float *wpe, float *out, int32_t batch, int32_t seq,
                   int32_t d, void *stream) {
  return embed_fwd(tokens, wte, wpe, out, batch, seq, d, static_cast<cudaStream_t>(stream));
}
int hm_k_embed_bwd(const int32_t *tokens, const float *dx, float *dwte, float *dwpe, int32_t batch, int32_t seq,
                   int32_t d, void *stream) {
  return embed_bwd(tokens, dx, dwte, dwpe, batch, seq, d, static_cast<cudaStream_t>(stream));
}
int hm_k_layernorm_fwd(const float *x, const float *g, const float *b, void *y, float *mean, float *rstd, int64_t rows,
                       int32_t d, void *stream) {
  return ln_fwd(x, g, b, y, mean, rstd, rows, d, static_cast<cudaStream_t>(stream));
}
int hm_k_layernorm_bwd(const float *dy, const float *x, const float *mean, const float *rstd, const float *g,
                       const float *resid, float *out, void *out_bf16, float *dg, float *db, int64_t rows, int32_t d,
                       void *stream) {
  return ln_bwd(dy, x, mean, rstd, g, resid, out, out_bf16, dg, db, rows, d, static_cast<cudaStream_t>(stream));
}
int hm_k_cross_entropy(const float *logits, const int32_t *labels, int64_t rows, int64_t ld, int32_t vocab,
                       void *dlogits, double *loss_sum, float scale, void *stream) {
  return cross_entropy(logits, labels, rows, ld, vocab, dlogits, loss_sum, scale, static_cast<cudaStream_t>(stream));
}
int hm_k_bias_grad(const void *dy, int32_t is_bf16, float *db, int64_t rows, int32_t n, int64_t ld, void *stream) {
  return bias_grad(dy, is_bf16, db, rows, n, ld, static_cast<cudaStream_t>(stream));
}
}
