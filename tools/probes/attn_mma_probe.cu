// Issue-rate probe of the head_dim-64 attention forward's MMA stream
// (sm_100a): one thread per SM issues "positions" of PV (8 x 128x64x16, A = P
// from TMEM, B = V MN-major) + S (4 x 128x128x16 SS) the way
// attention_fwd64.cu does, with variants that isolate each ingredient.
// Prints cycles per position.
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include "../../paper_2202_01306_b200/csrc/kernels/sm100.cuh"
using namespace hm::sm100;

// VARIANT: 0 PV + S as the kernel (S(n+3) into the buffer PV(n) read), 3 commits
//          1 PV only   2 S only   3 as 0 without commits   4 as 0, S into a
//          buffer PV does not read   5 as 0, B of PV K-major   6 as 0 with
//          an mbarrier try_wait per position (already complete)   7 PV + S
//          + one completed try_wait, no commits   8 as 7 with test_wait   9 as 6
//          with the wait between PV and S   10 as 7 with the wait between the
//          4th and 5th PV MMA
template <int VARIANT>
__global__ void __launch_bounds__(128, 1) probe(long long *out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar[4];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    if (VARIANT >= 6) mbar_arrive(&bar[3]);  // completes phase 0
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, 0, 0);
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, 64, 0, VARIANT == 5 ? 0 : 1);
    const uint32_t d_hi = (uint32_t)(umma_desc_sw128(0, 0, 1024) >> 32);
    const uint32_t q_lo = (uint32_t)umma_desc_sw128(smem_u32(smem), 16, 1024);
    const uint32_t k_lo = (uint32_t)umma_desc_sw128(smem_u32(smem + 16384), 16, 1024);
    const uint32_t v_lo = (uint32_t)umma_desc_sw128(smem_u32(smem + 32768), 16384, 1024);
    int buf = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t p_tm = tmem + buf * 128, d_o = tmem + 384 + (r & 1) * 64;
      if (VARIANT != 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          mma_bf16_ts_lohi(d_o, p_tm + kk * 8, v_lo + (VARIANT == 5 ? kk * 2 : kk * 128), d_hi, idesc_o, 1u);
          if (VARIANT == 10 && kk == 3) mbar_wait(&bar[3], 0);
        }
      }
      if (VARIANT == 7 || VARIANT == 9) mbar_wait(&bar[3], 0);
      if (VARIANT == 11) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar[3])) : "memory");
      }
      if (VARIANT == 12) {  // plain shared-memory read of the barrier word (phase bit 63)
        uint64_t w;
        do {
          asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(w) : "r"(smem_u32(&bar[3])) : "memory");
        } while (!(w >> 63) && false);
        if (w == 0x1234) out[5] = w;
      }
      if (VARIANT == 8) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar[3])) : "memory");
      }
      if (VARIANT == 0 || VARIANT == 4 || VARIANT == 5 || VARIANT == 6 || VARIANT == 9) {
        mma_commit(&bar[0]);
        mma_commit(&bar[1]);
      }
      if (VARIANT == 6) mbar_wait(&bar[3], 0);
      if (VARIANT != 1) {
        const uint32_t d_s = tmem + (VARIANT == 4 ? ((buf + 1) % 3) : buf) * 128;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_lohi(d_s, q_lo + 2 * kk, k_lo + 2 * kk, d_hi, idesc_s, kk > 0);
      }
      if (VARIANT == 0 || VARIANT == 4 || VARIANT == 5 || VARIANT == 6 || VARIANT == 9) mma_commit(&bar[2]);
      buf = buf == 2 ? 0 : buf + 1;
    }
    long long t1 = clock64();
    mma_commit(&bar[3]);
    mbar_wait(&bar[3], VARIANT >= 6 ? 1 : 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int V>
void run(long long *d, const char *name) {
  const int reps = 1000;
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  for (int i = 0; i < 2; ++i) probe<V><<<148, 128, 65 * 1024>>>(d, reps);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("{\"variant\": \"%s\", \"issue_cyc_per_position\": %.1f, \"total_cyc_per_position\": %.1f, \"err\": \"%s\"}\n",
         name, h[0] / (double)reps, h[1] / (double)reps, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long *d;
  cudaMalloc(&d, 64);
  run<0>(d, "PV(8, TS, V MN-major) + S(4, SS) into the buffer PV read, 3 commits");
  run<1>(d, "PV only");
  run<2>(d, "S only");
  run<3>(d, "PV + S, no commits");
  run<4>(d, "PV + S, S into another buffer");
  run<5>(d, "PV + S, V K-major");
  run<6>(d, "PV + S + commits + one completed mbarrier wait");
  run<7>(d, "PV + S + one completed try_wait, no commits");
  run<8>(d, "PV + S + one completed test_wait, no commits");
  run<9>(d, "PV + commits + completed try_wait + S + commit (wait before S)");
  run<10>(d, "PV(4) + completed try_wait + PV(4) + S, no commits");
  run<11>(d, "PV + S + one completed try_wait.relaxed, no commits");
  run<12>(d, "PV + S + one ld.volatile.shared of the barrier word, no commits");
  return 0;
}
