// Throughput probe of the special-function (XU) pipe on sm_100a: ex2.approx,
// cvt.rn.bf16x2.f32 and a degree-3 polynomial exp2 on the FMA pipe.  One
// launch per op, 148 x 8 CTAs of 128 threads (independent chains, 8 per
// thread), clock64 per SM.  Prints lanes/clk/SM for each op.
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t cvt2(float a, float b) {
  uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float ex2_poly(float x) {
  // 2^x = 2^floor(x) * p(frac), p degree 3 (minimax on [0,1))
  x = fmaxf(x, -127.f);
  const float fl = floorf(x);
  const float f = x - fl;
  float p = fmaf(f, 0.0555041086648216f, 0.2402264923172690f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)fl << 23));
}

__device__ __forceinline__ float ex2_poly2(float x) {
  // round-to-nearest by the 1.5 * 2^23 magic add (FADD, not FRND), f in [-0.5, 0.5]
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.0558755f, 0.2401397f);
  p = fmaf(p, f, 0.6931472f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int OP>
__global__ void probe(float *out, long long *cyc, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = ex2(a[i]);
      else if (OP == 1) acc += cvt2(a[i], a[(i + 1) & 7]), a[i] += 1e-7f;
      else if (OP == 2) a[i] = ex2_poly(a[i]);
      else if (OP == 3) { a[i] = (i & 1) ? ex2_poly(a[i]) : ex2(a[i]); }
      else if (OP == 4) a[i] = ex2_poly2(a[i]);
      else a[i] = (i & 3) == 3 ? ex2_poly2(a[i]) : ex2(a[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int per_sm = 8, threads = 128, iters = 4096;
  float *out; long long *cyc;
  cudaMalloc(&out, sms * per_sm * threads * 4); cudaMalloc(&cyc, sms * per_sm * 8);
  const char *names[] = {"ex2.approx", "cvt.rn.bf16x2 (per pair)", "poly exp2 (FMA pipe)", "half ex2 / half poly", "poly exp2, magic-add rounding", "3/4 ex2 + 1/4 magic poly"};
  for (int op = 0; op < 6; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (op == 0) probe<0><<<sms * per_sm, threads>>>(out, cyc, iters);
      if (op == 1) probe<1><<<sms * per_sm, threads>>>(out, cyc, iters);
      if (op == 2) probe<2><<<sms * per_sm, threads>>>(out, cyc, iters);
      if (op == 3) probe<3><<<sms * per_sm, threads>>>(out, cyc, iters);
      if (op == 4) probe<4><<<sms * per_sm, threads>>>(out, cyc, iters);
      if (op == 5) probe<5><<<sms * per_sm, threads>>>(out, cyc, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long h[2048]; cudaMemcpy(h, cyc, sms * per_sm * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < sms * per_sm; ++i) avg += h[i]; avg /= sms * per_sm;
      // all per_sm CTAs co-resident: ops per SM / cycles of one CTA's window
      const double ops = (double)per_sm * threads * iters * 8;
      if (rep) printf("{\"op\": \"%s\", \"lanes_per_clk_per_sm\": %.2f, \"ms\": %.3f, \"ghz_est\": %.3f}\n", names[op],
                      ops / avg, ms, avg / (ms * 1e6));
    }
  }
  return 0;
}
