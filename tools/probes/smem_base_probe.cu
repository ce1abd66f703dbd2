#include <cstdio>
#include <cstdint>
__global__ void k(unsigned *out) {
  extern __shared__ uint8_t smem_raw[];
  unsigned a = (unsigned)__cvta_generic_to_shared(smem_raw);
  if (threadIdx.x == 0) out[blockIdx.x] = a;
}
int main() {
  unsigned *d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  k<<<4, 384, 232448>>>(d);
  unsigned h[4]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("dyn smem base: %u %u %u %u (err %s)\n", h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
}
