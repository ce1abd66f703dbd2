// cnn.cu -- the HBM-bound pieces of the deep-CNN layer packs (BASELINE config
// c5): ReLU backward, 2x2 average pooling, global average pooling.  The
// convolutions themselves are implicit GEMMs on tcgen05 (gemm.cu, MODE 1-3).
// Activations are NHWC bf16; every kernel moves 16 B (8 channels) per thread
// per access and grid-strides over a grid sized to the SM count.
#include <cuda_bf16.h>

#include "../runtime/common.hpp"
#include "pdl.cuh"

namespace hm {
namespace cnn {

using bf16 = __nv_bfloat16;

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

static unsigned grid_for(int64_t n8) {
  int64_t g = (n8 + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 16;
  return (unsigned)(g < cap ? (g > 0 ? g : 1) : cap);
}

__device__ __forceinline__ void unpack8(const uint4 &u, float (&f)[8]) {
  const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(p[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162 *p = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// dz = dy * (y > 0)
__global__ void relu_bwd_kernel(const uint4 *__restrict__ dy, const uint4 *__restrict__ y, uint4 *__restrict__ dz,
                                int64_t n8) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float g[8], v[8];
    unpack8(dy[i], g);
    unpack8(y[i], v);
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = v[j] > 0.f ? g[j] : 0.f;
    dz[i] = pack8(g);
  }
}

// out = a + b
__global__ void add_kernel(const uint4 *__restrict__ a, const uint4 *__restrict__ b, uint4 *__restrict__ out,
                           int64_t n8) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float x[8], y[8];
    unpack8(a[i], x);
    unpack8(b[i], y);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] += y[j];
    out[i] = pack8(x);
  }
}

// y[n, h/2, w/2, c] = mean of the 2x2 window of a[n, h, w, c]; one thread per 8 channels of one output pixel
__global__ void pool2_fwd_kernel(const bf16 *__restrict__ a, bf16 *__restrict__ y, int n, int h, int w, int c) {
  pdl_wait();
  const int ho = h / 2, wo = w / 2, c8 = c / 8;
  const int64_t total = (int64_t)n * ho * wo * c8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cc = (int)(i % c8);
    int64_t p = i / c8;
    const int x = (int)(p % wo);
    p /= wo;
    const int yy = (int)(p % ho);
    const int64_t b = p / ho;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int64_t src = (((b * h + 2 * yy + dy) * w) + 2 * x + dx) * c + cc * 8;
        float f[8];
        unpack8(*reinterpret_cast<const uint4 *>(a + src), f);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += f[j];
      }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] *= 0.25f;
    *reinterpret_cast<uint4 *>(y + (i / c8) * c + cc * 8) = pack8(acc);
  }
}

// dz[n, h, w, c] = dy[n, h/2, w/2, c] / 4 * (a > 0): average-pool backward fused with
// the ReLU mask of the convolution that produced a
__global__ void pool2_relu_bwd_kernel(const bf16 *__restrict__ dy, const bf16 *__restrict__ a, bf16 *__restrict__ dz,
                                      int n, int h, int w, int c) {
  pdl_wait();
  const int ho = h / 2, wo = w / 2, c8 = c / 8;
  const int64_t total = (int64_t)n * h * w * c8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cc = (int)(i % c8);
    int64_t p = i / c8;
    const int x = (int)(p % w);
    p /= w;
    const int yy = (int)(p % h);
    const int64_t b = p / h;
    float g[8], v[8];
    unpack8(*reinterpret_cast<const uint4 *>(dy + (((b * ho + yy / 2) * wo) + x / 2) * c + cc * 8), g);
    unpack8(*reinterpret_cast<const uint4 *>(a + (i / c8) * c + cc * 8), v);
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = v[j] > 0.f ? 0.25f * g[j] : 0.f;
    *reinterpret_cast<uint4 *>(dz + (i / c8) * c + cc * 8) = pack8(g);
  }
}

// pooled[b, c] = mean over p of x[b, p, c]; block per (sample, 8*256-channel slab), fp32 sums
__global__ void gap_fwd_kernel(const bf16 *__restrict__ x, bf16 *__restrict__ pooled, int P, int c) {
  pdl_wait();
  const int b = blockIdx.y;
  const int c8 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c8 * 8 >= c) return;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bf16 *src = x + (int64_t)b * P * c + c8 * 8;
  for (int p = 0; p < P; ++p) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4 *>(src + (int64_t)p * c), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += f[j];
  }
  const float inv = 1.f / (float)P;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] *= inv;
  *reinterpret_cast<uint4 *>(pooled + (int64_t)b * c + c8 * 8) = pack8(acc);
}

// dx[b, p, c] = dpooled[b, c] / P
__global__ void gap_bwd_kernel(const float *__restrict__ dp, bf16 *__restrict__ dx, int nb, int P, int c) {
  pdl_wait();
  const int c8n = c / 8;
  const int64_t total = (int64_t)nb * P * c8n;
  const float inv = 1.f / (float)P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cc = (int)(i % c8n);
    const int64_t b = i / c8n / P;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = dp[b * c + cc * 8 + j] * inv;
    reinterpret_cast<uint4 *>(dx)[i] = pack8(f);
  }
}

int relu_bwd(const void *dy, const void *y, void *dz, int64_t n, cudaStream_t s) {
  if (n % 8) return fail(HM_ERR_VALIDATION, "relu_bwd: n must be a multiple of 8");
  ProfScope ps(KC_MISC, s, 0, 6.0 * n);
  HM_CUDA(launch_pdl(relu_bwd_kernel, dim3(grid_for(n / 8)), dim3(256), 0, s, static_cast<const uint4 *>(dy), static_cast<const uint4 *>(y),
                                                 static_cast<uint4 *>(dz), n / 8));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

int add_bf16(const void *a, const void *b, void *out, int64_t n, cudaStream_t s) {
  if (n % 8) return fail(HM_ERR_VALIDATION, "add_bf16: n must be a multiple of 8");
  ProfScope ps(KC_MISC, s, 0, 6.0 * n);
  HM_CUDA(launch_pdl(add_kernel, dim3(grid_for(n / 8)), dim3(256), 0, s, static_cast<const uint4 *>(a),
                     static_cast<const uint4 *>(b), static_cast<uint4 *>(out), n / 8));
  count_launch();
  return HM_OK;
}

int pool2_fwd(const void *a, void *y, int n, int h, int w, int c, cudaStream_t s) {
  if (h % 2 || w % 2 || c % 8) return fail(HM_ERR_VALIDATION, "pool2: even h, w and c % 8 == 0");
  ProfScope ps(KC_MISC, s, 0, 2.5 * n * h * w * (double)c);
  HM_CUDA(launch_pdl(pool2_fwd_kernel, dim3(grid_for((int64_t)n * h * w * c / 32)), dim3(256), 0, s, static_cast<const bf16 *>(a),
                                                                         static_cast<bf16 *>(y), n, h, w, c));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

int pool2_relu_bwd(const void *dy, const void *a, void *dz, int n, int h, int w, int c, cudaStream_t s) {
  if (h % 2 || w % 2 || c % 8) return fail(HM_ERR_VALIDATION, "pool2: even h, w and c % 8 == 0");
  ProfScope ps(KC_MISC, s, 0, 4.5 * n * h * w * (double)c);
  HM_CUDA(launch_pdl(pool2_relu_bwd_kernel, dim3(grid_for((int64_t)n * h * w * c / 8)), dim3(256), 0, s, 
      static_cast<const bf16 *>(dy), static_cast<const bf16 *>(a), static_cast<bf16 *>(dz), n, h, w, c));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

int gap_fwd(const void *x, void *pooled, int nb, int P, int c, cudaStream_t s) {
  if (c % 8) return fail(HM_ERR_VALIDATION, "gap: c % 8 == 0");
  ProfScope ps(KC_MISC, s, 0, 2.0 * nb * (double)P * c);
  const int c8 = c / 8, threads = c8 < 128 ? c8 : 128;
  HM_CUDA(launch_pdl(gap_fwd_kernel, dim3(dim3((c8 + threads - 1) / threads, nb)), dim3(threads), 0, s, static_cast<const bf16 *>(x),
                                                                          static_cast<bf16 *>(pooled), P, c));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

int gap_bwd(const float *dp, void *dx, int nb, int P, int c, cudaStream_t s) {
  if (c % 8) return fail(HM_ERR_VALIDATION, "gap: c % 8 == 0");
  ProfScope ps(KC_MISC, s, 0, 2.0 * nb * (double)P * c);
  HM_CUDA(launch_pdl(gap_bwd_kernel, dim3(grid_for((int64_t)nb * P * c / 8)), dim3(256), 0, s, dp, static_cast<bf16 *>(dx), nb, P, c));
  count_launch();
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

}  // namespace cnn
}  // namespace hm

extern "C" {
int hm_k_relu_bwd(const void *dy, const void *y, void *dz, int64_t n, void *stream) {
  return hm::cnn::relu_bwd(dy, y, dz, n, static_cast<cudaStream_t>(stream));
}
int hm_k_pool2_fwd(const void *a, void *y, int32_t n, int32_t h, int32_t w, int32_t c, void *stream) {
  return hm::cnn::pool2_fwd(a, y, n, h, w, c, static_cast<cudaStream_t>(stream));
}
int hm_k_pool2_relu_bwd(const void *dy, const void *a, void *dz, int32_t n, int32_t h, int32_t w, int32_t c,
                        void *stream) {
  return hm::cnn::pool2_relu_bwd(dy, a, dz, n, h, w, c, static_cast<cudaStream_t>(stream));
}
int hm_k_gap_fwd(const void *x, void *pooled, int32_t nb, int32_t P, int32_t c, void *stream) {
  return hm::cnn::gap_fwd(x, pooled, nb, P, c, static_cast<cudaStream_t>(stream));
}
int hm_k_add_bf16(const void *a, const void *b, void *out, int64_t n, void *stream) {
  return hm::cnn::add_bf16(a, b, out, n, static_cast<cudaStream_t>(stream));
}
int hm_k_gap_bwd(const float *dp, void *dx, int32_t nb, int32_t P, int32_t c, void *stream) {
  return hm::cnn::gap_bwd(dp, dx, nb, P, c, static_cast<cudaStream_t>(stream));
}
}
