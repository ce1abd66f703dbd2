// TMEM read bandwidth probe (sm_100a): W warpgroups of one CTA per SM each
// read their 128 lanes x 128 columns (64 KB fp32, an attention S tile) with
// tcgen05.ld.32x32b.x32, N rounds; loads per wait = 1, 2 or 4.  Prints
// bytes / clk / SM.  Also the tcgen05.st rate (x16).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../../paper_2202_01306_b200/csrc/kernels/sm100.cuh"
using namespace hm::sm100;

template <int PER_WAIT, bool STORE>
__global__ void __launch_bounds__(384, 1) probe(float *out, long long *cyc, int rounds, int nwg) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  float acc = 0.f;
  long long t0 = clock64();
  const int wg = warp >> 2;
  if (wg < nwg) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + wg * 128;
    for (int r = 0; r < rounds; ++r) {
      if (STORE) {
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = r + i;
#pragma unroll
        for (int c = 0; c < 128; c += 16) tmem_st_32x32b_x16(base + c, v);
        tmem_st_wait();
      } else {
#pragma unroll
        for (int c0 = 0; c0 < 128; c0 += 32 * PER_WAIT) {
          uint32_t v[32 * PER_WAIT];
#pragma unroll
          for (int q = 0; q < PER_WAIT; ++q) tmem_ld_32x32b_x32(base + c0 + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * q));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32 * PER_WAIT; ++i) acc += __uint_as_float(v[i]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int P, bool S>
void run(int sms, float *out, long long *cyc, int nwg, const char *name) {
  const int rounds = 2000;
  long long h[1024];
  for (int rep = 0; rep < 2; ++rep) {
    probe<P, S><<<sms, 384>>>(out, cyc, rounds, nwg);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  const double bytes = (double)nwg * 128 * 128 * 4 * rounds;
  printf("{\"op\": \"%s\", \"warpgroups\": %d, \"bytes_per_clk_per_sm\": %.1f, \"clk_per_64KB_tile\": %.0f, \"err\": \"%s\"}\n",
         name, nwg, bytes / avg, avg / (nwg * (double)rounds), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out; long long *cyc;
  cudaMalloc(&out, sms * 384 * 4); cudaMalloc(&cyc, sms * 8);
  for (int nwg = 1; nwg <= 2; ++nwg) {
    run<1, false>(sms, out, cyc, nwg, "ld x32, 1 per wait");
    run<2, false>(sms, out, cyc, nwg, "ld x32, 2 per wait");
    run<4, false>(sms, out, cyc, nwg, "ld x32, 4 per wait");
    run<1, true>(sms, out, cyc, nwg, "st x16");
  }
  return 0;
}
