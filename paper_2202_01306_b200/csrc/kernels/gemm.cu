// gemm.cu -- tcgen05 GEMM for the F/B/U compute of a layer pack (sm_100a).
//
//   D[M,N] (op)= A[M,K] . B[N,K]^T        bf16 operands, fp32 accumulate
//
// Used for every dense contraction of a transformer block:
//   forward  Y  = X  . W^T   A = X  (K-major), B = W [out,in] (K-major)
//   dgrad    dX = dY . W     A = dY (K-major), B = W [out,in] (MN-major)
//   wgrad    dW += dY^T . X  A = dY (MN-major), B = X (MN-major), fp32 accumulate
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0   TMA producer: A/B tiles -> SW128 smem ring (kStages deep)
//   warp 1   MMA issuer: one elected thread issues tcgen05.mma 128xBNx16,
//            accumulator double-buffered in TMEM (2 x BN fp32 columns)
//   warp 2   TMEM allocator
//   warps 4-11 epilogue (two per TMEM lane quadrant, each draining half the
//            columns): tcgen05.ld 32 lanes x 32 columns per warp, fused
//            bias / residual / GELU / dGELU / fp32 accumulate, vector stores
// The epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <map>

#include "../runtime/common.hpp"
#include "sm100.cuh"

namespace hm {
namespace gemm {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SW128 atom row
constexpr int kGroupM = 8;
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quadrant, each draining half the columns
constexpr int kThreads = 128 + 32 * kEpiWarps;

struct Args {
  int32_t M, N, K, num_m, num_n, num_k;
  void *d;
  int64_t ldd;
  const float *bias;
  void *aux;
  int64_t ld_aux;
  int32_t epi;
};

template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr uint32_t kABytes = BM * BK * 2;
  static constexpr uint32_t kBBytes = BN * BK * 2;
  static constexpr uint32_t kTmemCols = 2 * BN >= 512 ? 512 : (2 * BN >= 256 ? 256 : 128);
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBBytes) + 256;
};

__device__ __forceinline__ void tile_coord(int t, int num_m, int num_n, int &mb, int &nb) {
  const int per_group = kGroupM * num_n;
  const int g = t / per_group;
  const int first = g * kGroupM;
  const int gsize = min(num_m - first, kGroupM);
  const int r = t % per_group;
  mb = first + r % gsize;
  nb = r / gsize;
}

__device__ __forceinline__ float gelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float dgelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanhf(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

// Operands the epilogue reads from global memory for one 32-column chunk,
// fetched before the TMEM load so the two latencies overlap.
struct EpiPre {
  float4 f[8];  // residual / accumulate source (fp32)
  uint4 b[4];   // pre-activation (bf16) for dGELU
};

__device__ __forceinline__ void epilogue_prefetch(const Args &a, int row, int col0, EpiPre &p) {
  if (a.epi == HM_EPI_ACC_F32 || a.epi == HM_EPI_RESID_F32) {
    const float *src = a.epi == HM_EPI_ACC_F32
                           ? reinterpret_cast<const float *>(a.d) + (int64_t)row * a.ldd + col0
                           : reinterpret_cast<const float *>(a.aux) + (int64_t)row * a.ld_aux + col0;
#pragma unroll
    for (int j = 0; j < 8; ++j) p.f[j] = reinterpret_cast<const float4 *>(src)[j];
  } else if (a.epi == HM_EPI_DGELU_BF16) {
    const __nv_bfloat16 *aux = reinterpret_cast<const __nv_bfloat16 *>(a.aux) + (int64_t)row * a.ld_aux + col0;
#pragma unroll
    for (int j = 0; j < 4; ++j) p.b[j] = reinterpret_cast<const uint4 *>(aux)[j];
  }
}

// Apply the epilogue to 32 consecutive columns [col0, col0+32) of one row.
// `pre` holds the chunk's global operands when the chunk is full.
__device__ __forceinline__ void epilogue_row(const Args &a, int row, int col0, float (&v)[32], const EpiPre &pre) {
  const int N = a.N;
  const bool full = col0 + 32 <= N;
  if (a.bias && a.epi != HM_EPI_ACC_F32 && a.epi != HM_EPI_DGELU_BF16) {
    if (full) {
      const float4 *b4 = reinterpret_cast<const float4 *>(a.bias + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 b = __ldg(b4 + j);
        v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) v[j] += a.bias[col0 + j];
    }
  }
  switch (a.epi) {
    case HM_EPI_STORE_F32:
    case HM_EPI_ACC_F32:
    case HM_EPI_RESID_F32: {
      float *dst = reinterpret_cast<float *>(a.d) + (int64_t)row * a.ldd + col0;
      const float *src = nullptr;
      if (a.epi == HM_EPI_ACC_F32) src = dst;
      if (a.epi == HM_EPI_RESID_F32) src = reinterpret_cast<const float *>(a.aux) + (int64_t)row * a.ld_aux + col0;
      if (full) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          if (src) {
            const float4 s = pre.f[j];
            o.x += s.x; o.y += s.y; o.z += s.z; o.w += s.w;
          }
          reinterpret_cast<float4 *>(dst)[j] = o;
        }
      } else {
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) dst[j] = v[j] + (src ? src[j] : 0.f);
      }
      break;
    }
    case HM_EPI_STORE_BF16:
    case HM_EPI_GELU_BF16:
    case HM_EPI_DGELU_BF16: {
      __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(a.d) + (int64_t)row * a.ldd + col0;
      __nv_bfloat16 *aux = a.aux ? reinterpret_cast<__nv_bfloat16 *>(a.aux) + (int64_t)row * a.ld_aux + col0 : nullptr;
      if (a.epi == HM_EPI_DGELU_BF16) {
        if (full) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 p = pre.b[j];
            const __nv_bfloat162 *p2 = reinterpret_cast<const __nv_bfloat162 *>(&p);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float2 f = __bfloat1622float2(p2[e]);
              v[8 * j + 2 * e] *= dgelu_f(f.x);
              v[8 * j + 2 * e + 1] *= dgelu_f(f.y);
            }
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (col0 + j < N) v[j] *= dgelu_f(__bfloat162float(aux[j]));
        }
      } else if (a.epi == HM_EPI_GELU_BF16) {
        // store the pre-activation, then activate
        if (full) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 p;
            __nv_bfloat162 *p2 = reinterpret_cast<__nv_bfloat162 *>(&p);
#pragma unroll
            for (int e = 0; e < 4; ++e) p2[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
            reinterpret_cast<uint4 *>(aux)[j] = p;
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (col0 + j < N) aux[j] = __float2bfloat16_rn(v[j]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
      }
      if (full) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 p;
          __nv_bfloat162 *p2 = reinterpret_cast<__nv_bfloat162 *>(&p);
#pragma unroll
          for (int e = 0; e < 4; ++e) p2[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
          reinterpret_cast<uint4 *>(dst)[j] = p;
        }
      } else {
        for (int j = 0; j < 32; ++j)
          if (col0 + j < N) dst[j] = __float2bfloat16_rn(v[j]);
      }
      break;
    }
    default:
      break;
  }
}

template <int BN, int A_MN, int B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Args args) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * C::kABytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + C::kStages * C::kBBytes);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int ntiles = args.num_m * args.num_n;

  if (warp == 0) {
    if (lane == 0) {
      // programmatic dependent launch: everything above (barrier init, TMEM
      // alloc, descriptor prefetch) overlapped the previous kernel's tail;
      // global operands are read only after it has fully completed
      griddep_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int mb, nb;
        tile_coord(t, args.num_m, args.num_n, mb, nb);
        for (int kb = 0; kb < args.num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::kABytes + C::kBBytes);
          uint8_t *a_dst = sA + stage * C::kABytes;
          uint8_t *b_dst = sB + stage * C::kBBytes;
          if (!A_MN) {
            tma_load_2d(a_dst, &tmA, &full[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_2d(a_dst + c * (BK * 128), &tmA, &full[stage], mb * BM + c * 64, kb * BK);
          }
          if (!B_MN) {
            tma_load_2d(b_dst, &tmB, &full[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d(b_dst + c * (BK * 128), &tmB, &full[stage], nb * BN + c * 64, kb * BK);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t use = (uint32_t)(local >> 1);
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < args.num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * C::kABytes);
          const uint32_t b_base = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 16 elements = 32 B inside the swizzle atom.
            // MN-major: advance 16 K-rows = 16 x 128 B.
            const uint64_t da = A_MN ? umma_desc_sw128(a_base + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t db = B_MN ? umma_desc_sw128(b_base + k * 2048, BK * 128, 1024)
                                     : umma_desc_sw128(b_base + k * 32, 16, 1024);
            mma_bf16(d_tmem, da, db, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          mma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
      griddep_launch_dependents();  // only epilogues remain: let the next kernel set up
    }
  } else if (warp >= 4) {
    const int q = warp & 3;              // a warp may only touch TMEM lanes 32*(warp%4)..+31
    const int half = (warp - 4) >> 2;    // which half of the tile's columns
    constexpr int kChunks = BN / 32 / (kEpiWarps / 4);
    griddep_wait();  // epilogue reads / writes global memory of the previous kernel's outputs
    int local = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      int mb, nb;
      tile_coord(t, args.num_m, args.num_n, mb, nb);
      const int acc = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const int row = mb * BM + q * 32 + (int)lane;
#pragma unroll 1
      for (int c = half * kChunks; c < (half + 1) * kChunks; ++c) {
        const int col0 = nb * BN + c * 32;
        if (col0 >= args.N) break;
        EpiPre pre;
        if (row < args.M && col0 + 32 <= args.N) epilogue_prefetch(args, row, col0, pre);
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (row < args.M) epilogue_row(args, row, col0, v, pre);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps (cached), launch
// ---------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2D bf16 map: inner dim d0 (contiguous), outer d1, row pitch in bytes, box {64, box1}, SW128.
static int make_map(CUtensorMap *out, const void *ptr, uint64_t d0, uint64_t d1, uint64_t pitch_bytes,
                    uint32_t box1) {
  using Key = std::tuple<const void *, uint64_t, uint64_t, uint64_t, uint32_t>;
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  Key key{ptr, d0, d1, pitch_bytes, box1};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return HM_OK;
    }
  }
  EncodeFn fn = encode_fn();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {64, box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *out;
  return HM_OK;
}

static int num_sms();

// Tile width (measured on B200, profiles/r01_kernel_perf_bn.jsonl): the
// 128x256 tile wins almost everywhere; the narrower tile only pays off for
// short reductions (K <= 2048) with fewer than two waves of wide tiles, where
// per-tile fill/drain dominates.
static int pick_bn(int64_t M, int64_t N, int64_t K) {
  const int64_t sms = num_sms();
  const int64_t tiles256 = ((M + BM - 1) / BM) * ((N + 255) / 256);
  return (tiles256 < 2 * sms && K <= 2048) ? 128 : 256;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int A_MN, int B_MN>
static int launch(const CUtensorMap &ta, const CUtensorMap &tb, const Args &a, cudaStream_t s) {
  using C = Cfg<BN>;
  static bool attr = false;
  auto kern = gemm_kernel<BN, A_MN, B_MN>;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    if (e != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("gemm smem attr: ") + cudaGetErrorString(e));
    attr = true;
  }
  const int ntiles = a.num_m * a.num_n;
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  const bool f32 = a.epi == HM_EPI_STORE_F32 || a.epi == HM_EPI_ACC_F32 || a.epi == HM_EPI_RESID_F32;
  const double io = (double)a.M * a.N * (f32 ? 4 : 2) * (a.epi == HM_EPI_ACC_F32 || a.epi >= HM_EPI_RESID_F32 ? 2 : 1);
  ProfScope ps(KC_GEMM, s, 2.0 * a.M * a.N * a.K, 2.0 * ((double)a.M * a.K + (double)a.N * a.K) + io);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, ta, tb, a);
  if (le != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("gemm launch: ") + cudaGetErrorString(le));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("gemm launch: ") + cudaGetErrorString(e));
  count_launch();
  return HM_OK;
}

int run(const void *A, const void *B, void *D, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
        int64_t ldd, int a_mn, int b_mn, int epi, const float *bias, void *aux, int64_t ld_aux,
        cudaStream_t stream, int force_bn) {
  if (M <= 0 || N <= 0 || K <= 0) return fail(HM_ERR_VALIDATION, "gemm: empty problem");
  if ((lda * 2) % 16 || (ldb * 2) % 16) return fail(HM_ERR_VALIDATION, "gemm: operand pitch must be 16B aligned");
  if (((uintptr_t)A | (uintptr_t)B) & 15) return fail(HM_ERR_VALIDATION, "gemm: operands must be 16B aligned");
  const bool f32out = epi == HM_EPI_STORE_F32 || epi == HM_EPI_ACC_F32 || epi == HM_EPI_RESID_F32;
  if ((ldd * (f32out ? 4 : 2)) % 16 || ((uintptr_t)D & 15))
    return fail(HM_ERR_VALIDATION, "gemm: output must be 16B aligned with 16B pitch");
  if ((epi == HM_EPI_RESID_F32 || epi == HM_EPI_GELU_BF16 || epi == HM_EPI_DGELU_BF16) && !aux)
    return fail(HM_ERR_VALIDATION, "gemm: epilogue needs an aux tensor");
  if (aux && ((ld_aux * (epi == HM_EPI_RESID_F32 ? 4 : 2)) % 16 || ((uintptr_t)aux & 15)))
    return fail(HM_ERR_VALIDATION, "gemm: aux must be 16B aligned with 16B pitch");
  static const int env_bn = [] {
    const char *e = getenv("HM_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  int bn = force_bn ? force_bn : env_bn ? env_bn : pick_bn(M, N, K);
  Args a{};
  a.M = (int)M; a.N = (int)N; a.K = (int)K;
  a.num_m = (int)((M + BM - 1) / BM);
  a.num_n = (int)((N + bn - 1) / bn);
  a.num_k = (int)((K + BK - 1) / BK);
  a.d = D; a.ldd = ldd; a.bias = bias; a.aux = aux; a.ld_aux = ld_aux; a.epi = epi;
  CUtensorMap ta, tb;
  int rc = a_mn ? make_map(&ta, A, M, K, lda * 2, 64) : make_map(&ta, A, K, M, lda * 2, BM);
  if (rc) return rc;
  rc = b_mn ? make_map(&tb, B, N, K, ldb * 2, 64) : make_map(&tb, B, K, N, ldb * 2, bn);
  if (rc) return rc;
  const int key = (bn == 256 ? 4 : 0) | (a_mn ? 2 : 0) | (b_mn ? 1 : 0);
  switch (key) {
    case 0: return launch<128, 0, 0>(ta, tb, a, stream);
    case 1: return launch<128, 0, 1>(ta, tb, a, stream);
    case 2: return launch<128, 1, 0>(ta, tb, a, stream);
    case 3: return launch<128, 1, 1>(ta, tb, a, stream);
    case 4: return launch<256, 0, 0>(ta, tb, a, stream);
    case 5: return launch<256, 0, 1>(ta, tb, a, stream);
    case 6: return launch<256, 1, 0>(ta, tb, a, stream);
    default: return launch<256, 1, 1>(ta, tb, a, stream);
  }
}

}  // namespace gemm
}  // namespace hm

extern "C" int hm_k_gemm(const void *a, const void *b, void *d, int64_t m, int64_t n, int64_t k, int64_t lda,
                         int64_t ldb, int64_t ldd, int32_t a_major, int32_t b_major, int32_t epilogue,
                         const float *bias, const void *aux, int64_t ld_aux, int32_t batch, int64_t stride_a,
                         int64_t stride_b, int64_t stride_d, void *stream) {
  if (batch < 1) return hm::fail(HM_ERR_VALIDATION, "gemm: batch must be >= 1");
  for (int32_t i = 0; i < batch; ++i) {
    int rc = hm::gemm::run(static_cast<const __nv_bfloat16 *>(a) + i * stride_a,
                           static_cast<const __nv_bfloat16 *>(b) + i * stride_b,
                           static_cast<char *>(d) + i * stride_d * (epilogue == HM_EPI_STORE_BF16 ||
                                                                            epilogue >= HM_EPI_GELU_BF16
                                                                        ? 2
                                                                        : 4),
                           m, n, k, lda, ldb, ldd, a_major, b_major, epilogue, bias, const_cast<void *>(aux),
                           ld_aux, static_cast<cudaStream_t>(stream), 0);
    if (rc) return rc;
  }
  return HM_OK;
}
