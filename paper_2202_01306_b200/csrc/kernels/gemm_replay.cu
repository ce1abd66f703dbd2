// gemm_replay.cu -- the GEMM's own per-launch time for one problem shape.
//
// The bench's dominant-kernel roofline: the shapes a training iteration
// launches (logged by gemm::run while the runtime profiles an iteration) are
// replayed here, each as a CUDA graph of back-to-back launches of the same
// kernel configuration (programmatic dependent launch between them, as in the
// step), timed with CUDA events around whole graph launches -- so the
// per-launch figure holds no event nodes, host launch gaps or neighbouring
// kernels.  Operands are random bf16 in [-1, 1); several operand sets rotate
// so the replayed launches do not find their inputs in L2 (126 MB).
#include <cuda_bf16.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../runtime/common.hpp"
#include "../runtime/kernels_api.hpp"

namespace hm {
namespace gemm {

__global__ void fill_random_bf16(__nv_bfloat16 *p, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 16;
    x *= 0x7feb352d;
    x ^= x >> 15;
    x *= 0x846ca68b;
    x ^= x >> 16;
    p[i] = __float2bfloat16((float)(x >> 8) * (2.0f / 16777216.0f) - 1.0f);
  }
}

static int replay(const int64_t *shape, int reps, cudaStream_t caller, double *us) {
  const int64_t M = shape[0], N = shape[1], K = shape[2];
  const int a_mn = (int)shape[3], b_mn = (int)shape[4], epi = (int)shape[5], has_bias = (int)shape[6];
  if (M <= 0 || N <= 0 || K <= 0 || reps < 1) return fail(HM_ERR_VALIDATION, "gemm replay: bad shape");
  const bool f32 = epi == HM_EPI_STORE_F32 || epi == HM_EPI_ACC_F32 || epi == HM_EPI_RESID_F32;
  const int64_t a_el = M * K, b_el = N * K, d_by = M * N * (f32 ? 4 : 2);
  const int64_t aux_by = (epi == HM_EPI_RESID_F32 ? 4 : 2) * M * N;
  const bool need_aux = epi == HM_EPI_RESID_F32 || epi == HM_EPI_GELU_BF16 || epi == HM_EPI_DGELU_BF16 ||
                        epi == HM_EPI_RESID_RELU_BF16 || epi == HM_EPI_DRELU_BF16 || epi == HM_EPI_ADD_BF16;
  const int64_t set_by = 2 * (a_el + b_el) + d_by + (need_aux ? aux_by : 0);
  const int sets = (int)std::max<int64_t>(1, std::min<int64_t>(8, (256LL << 20) / std::max<int64_t>(set_by, 1) + 1));
  // a private non-blocking stream: the caller's may be the legacy default
  // stream, which cannot be captured into a graph
  (void)caller;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
    return fail(HM_ERR_DEVICE, "gemm replay: stream create");
  std::vector<void *> bufs;
  auto alloc = [&](int64_t bytes) -> void * {
    void *p = nullptr;
    if (cudaMalloc(&p, (size_t)std::max<int64_t>(bytes, 256)) != cudaSuccess) return nullptr;
    bufs.push_back(p);
    return p;
  };
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    for (void *p : bufs) cudaFree(p);
    cudaStreamDestroy(s);
  };
  struct Set { void *a, *b, *d, *aux; };
  std::vector<Set> S(sets);
  float *bias = nullptr;
  if (has_bias) {
    bias = static_cast<float *>(alloc(N * 4));
    if (!bias) return cleanup(), fail(HM_ERR_DEVICE, "gemm replay: out of memory");
    cudaMemsetAsync(bias, 0, N * 4, s);
  }
  for (int i = 0; i < sets; ++i) {
    S[i].a = alloc(a_el * 2);
    S[i].b = alloc(b_el * 2);
    S[i].d = alloc(d_by);
    S[i].aux = need_aux ? alloc(aux_by) : nullptr;
    if (!S[i].a || !S[i].b || !S[i].d || (need_aux && !S[i].aux))
      return cleanup(), fail(HM_ERR_DEVICE, "gemm replay: out of memory");
    fill_random_bf16<<<1184, 256, 0, s>>>(static_cast<__nv_bfloat16 *>(S[i].a), a_el, 17u * i + 1);
    fill_random_bf16<<<1184, 256, 0, s>>>(static_cast<__nv_bfloat16 *>(S[i].b), b_el, 31u * i + 7);
    cudaMemsetAsync(S[i].d, 0, d_by, s);
    if (S[i].aux) cudaMemsetAsync(S[i].aux, 0, aux_by, s);
  }
  // same leading dimensions as the runtime's dense operands
  const int64_t lda = a_mn ? M : K, ldb = b_mn ? N : K, ldd = N;
  auto one = [&](int i) {
    const Set &x = S[i % sets];
    return run(x.a, x.b, x.d, M, N, K, lda, ldb, ldd, a_mn, b_mn, epi, bias, x.aux, N, s, 0);
  };
  int rc = one(0);  // warm: tensor maps, smem attribute
  if (rc != HM_OK) return cleanup(), rc;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  cudaStreamSynchronize(s);
  cudaError_t be = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (be != cudaSuccess) return cleanup(), fail(HM_ERR_DEVICE, std::string("gemm replay: capture: ") + cudaGetErrorString(be));
  const int64_t launches0 = launch_counter().load();
  for (int r = 0; r < reps && rc == HM_OK; ++r) rc = one(r);
  cudaError_t ce = cudaStreamEndCapture(s, &g);
  launch_counter().fetch_sub(launch_counter().load() - launches0);
  if (rc != HM_OK || ce != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return cleanup(), rc != HM_OK ? rc : fail(HM_ERR_DEVICE, "gemm replay: end capture");
  }
  ce = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return cleanup(), fail(HM_ERR_DEVICE, "gemm replay: instantiate");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaGraphLaunch(ge, s);  // warm-up replay
  const int outer = 3;
  cudaEventRecord(e0, s);
  for (int o = 0; o < outer; ++o) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  ce = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(ge);
  cleanup();
  if (ce != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("gemm replay: ") + cudaGetErrorString(ce));
  *us = 1000.0 * ms / ((double)outer * reps);
  return HM_OK;
}

}  // namespace gemm
}  // namespace hm

extern "C" int hm_k_gemm_replay(const int64_t *shape, int32_t reps, void *stream, double *us_per_launch) {
  if (!shape || !us_per_launch) return hm::fail(HM_ERR_VALIDATION, "gemm replay: null argument");
  return hm::gemm::replay(shape, reps, static_cast<cudaStream_t>(stream), us_per_launch);
}
