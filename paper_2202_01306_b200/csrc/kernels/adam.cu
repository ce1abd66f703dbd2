// adam.cu -- the UPD task's fused Adam (paper §3.3 jit-update).
//
// One pass over a pack: reads W, g, m, v (16 B/param), writes W, m, v
// (12 B/param) -- HBM-bound, 28 B/param algorithmic traffic.  K holds (m, v)
// interleaved per parameter so a pack's optimizer state is one contiguous
// range of the host K arena (one swap-in row, one swap-out row).
// Update rule and operation order follow torch.optim.Adam (no weight decay):
//   m = m + (1-b1)(g - m) ;  v = b2 v + (1-b2) g^2
//   w -= (lr / (1-b1^t)) * m / (sqrt(v) / sqrt(1-b2^t) + eps)
#include <cmath>
#include "../runtime/common.hpp"

namespace hm {

__global__ void __launch_bounds__(256) adam_kernel(float4 *__restrict__ w, const float4 *__restrict__ g,
                                                   float4 *__restrict__ k, int64_t n4, float lr_t, float omb1,
                                                   float b2, float omb2, float inv_sqrt_bc2, float eps, float gscale,
                                                   const float *__restrict__ sc) {
  if (sc) {  // step-dependent scalars from device memory (graph replay)
    lr_t = sc[0];
    inv_sqrt_bc2 = sc[1];
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 wi = w[i];
    const float4 gi = g[i];
    float4 k0 = k[2 * i], k1 = k[2 * i + 1];  // (m0 v0 m1 v1) (m2 v2 m3 v3)
    float gg[4] = {gi.x * gscale, gi.y * gscale, gi.z * gscale, gi.w * gscale};
    float m[4] = {k0.x, k0.z, k1.x, k1.z};
    float v[4] = {k0.y, k0.w, k1.y, k1.w};
    float ww[4] = {wi.x, wi.y, wi.z, wi.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m[j] = m[j] + omb1 * (gg[j] - m[j]);  // torch lerp form
      v[j] = b2 * v[j] + omb2 * gg[j] * gg[j];
      const float denom = sqrtf(v[j]) * inv_sqrt_bc2 + eps;
      ww[j] -= lr_t * (m[j] / denom);
    }
    w[i] = make_float4(ww[0], ww[1], ww[2], ww[3]);
    k[2 * i] = make_float4(m[0], v[0], m[1], v[1]);
    k[2 * i + 1] = make_float4(m[2], v[2], m[3], v[3]);
  }
}

__global__ void adam_tail(float *w, const float *g, float *k, int64_t begin, int64_t n, float lr_t, float omb1,
                          float b2, float omb2, float inv_sqrt_bc2, float eps, float gscale, const float *sc) {
  if (sc) {
    lr_t = sc[0];
    inv_sqrt_bc2 = sc[1];
  }
  int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float gi = g[i] * gscale;
  float m = k[2 * i] + omb1 * (gi - k[2 * i]);
  float v = b2 * k[2 * i + 1] + omb2 * gi * gi;
  w[i] -= lr_t * (m / (sqrtf(v) * inv_sqrt_bc2 + eps));
  k[2 * i] = m;
  k[2 * i + 1] = v;
}

static int adam_impl(float *w, const float *g, float *k, int64_t n, float lr_t, double b1, double b2, double eps,
                     float isb, const float *sc, float gscale, cudaStream_t s) {
  if (n <= 0) return HM_OK;
  if (((uintptr_t)w | (uintptr_t)g | (uintptr_t)k) & 15) return fail(HM_ERR_VALIDATION, "adam: 16B alignment");
  const int64_t n4 = n / 4;
  // 1 - beta in double, as torch.optim.Adam does (1 - 0.999f in float is off by 1.3e-5)
  const float omb1 = (float)(1.0 - b1), omb2 = (float)(1.0 - b2);
  ProfScope ps(KC_ADAM, s, 0, 28.0 * n);
  if (n4) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (n4 + 255) / 256;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    adam_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<float4 *>(w), reinterpret_cast<const float4 *>(g),
                                                 reinterpret_cast<float4 *>(k), n4, lr_t, omb1, (float)b2, omb2, isb, (float)eps, gscale, sc);
    count_launch();
  }
  if (n4 * 4 < n) {
    adam_tail<<<1, 32, 0, s>>>(w, g, k, n4 * 4, n, lr_t, omb1, (float)b2, omb2, isb, (float)eps, gscale, sc);
    count_launch();
  }
  HM_CUDA(cudaGetLastError());
  return HM_OK;
}

int adam_launch(float *w, const float *g, float *k, int64_t n, double lr, double b1, double b2, double eps, int step,
                float gscale, cudaStream_t s) {
  if (step < 1) return fail(HM_ERR_VALIDATION, "adam: step must be >= 1");
  const double bc1 = 1.0 - std::pow(b1, step);
  const double bc2 = 1.0 - std::pow(b2, step);
  return adam_impl(w, g, k, n, (float)(lr / bc1), b1, b2, eps, (float)(1.0 / std::sqrt(bc2)), nullptr, gscale, s);
}

// Same update with {lr/(1-b1^t), 1/sqrt(1-b2^t)} read from device memory.
int adam_launch_dev(float *w, const float *g, float *k, int64_t n, double b1, double b2, double eps, const float *scalars,
                    float gscale, cudaStream_t s) {
  return adam_impl(w, g, k, n, 0.f, b1, b2, eps, 0.f, scalars, gscale, s);
}

}  // namespace hm

extern "C" int hm_k_adam(float *w, const float *g, float *k, int64_t n, double lr, double beta1, double beta2,
                         double eps, int32_t step, float grad_scale, void *stream) {
  return hm::adam_launch(w, g, k, n, lr, beta1, beta2, eps, step, grad_scale, static_cast<cudaStream_t>(stream));
}
