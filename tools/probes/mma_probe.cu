// tcgen05.mma issue / execution rate probe (sm_100a): one CTA per SM, one
// thread issues R MMAs of a given shape back to back (descriptors
// precomputed), commits, waits; cycles per MMA.  SS = both operands from
// shared memory, TS = A from TMEM.  Also the same loop with the descriptors
// rebuilt per MMA from addresses (the kernels' pattern).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../../paper_2202_01306_b200/csrc/kernels/sm100.cuh"
using namespace hm::sm100;

template <int N, bool TS, bool REBUILD>
__global__ void __launch_bounds__(128, 1) probe(long long *out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint64_t da = umma_desc_sw128(a, 16, 1024), db = umma_desc_sw128(b, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS) {
          const uint64_t dbk = REBUILD ? umma_desc_sw128(b + kk * 32, 16, 1024) : db + (uint64_t)(kk * 2);
          mma_bf16_ts(tmem + 256, tmem + kk * 8, dbk, idesc, 1u);
        } else {
          const uint64_t dak = REBUILD ? umma_desc_sw128(a + kk * 32, 16, 1024) : da + (uint64_t)(kk * 2);
          const uint64_t dbk = REBUILD ? umma_desc_sw128(b + kk * 32, 16, 1024) : db + (uint64_t)(kk * 2);
          mma_bf16(tmem + 256, dak, dbk, idesc, 1u);
        }
      }
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS, bool REBUILD>
void run(long long *d, const char *name) {
  const int reps = 2000;
  cudaFuncSetAttribute(probe<N, TS, REBUILD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  for (int i = 0; i < 2; ++i) probe<N, TS, REBUILD><<<148, 128, 65 * 1024>>>(d, reps);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = reps * 4.0;
  printf("{\"mma\": \"%s\", \"issue_cyc_per_mma\": %.1f, \"total_cyc_per_mma\": %.1f, \"ideal_cyc\": %.1f, \"err\": \"%s\"}\n",
         name, h[0] / n, h[1] / n, 128.0 * N * 16 / 4096.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long *d;
  cudaMalloc(&d, 64);
  run<64, false, false>(d, "128x64x16 SS");
  run<128, false, false>(d, "128x128x16 SS");
  run<256, false, false>(d, "128x256x16 SS");
  run<64, true, false>(d, "128x64x16 TS");
  run<128, true, false>(d, "128x128x16 TS");
  run<64, false, true>(d, "128x64x16 SS, descriptors rebuilt per MMA");
  run<64, true, true>(d, "128x64x16 TS, descriptors rebuilt per MMA");
  return 0;
}
