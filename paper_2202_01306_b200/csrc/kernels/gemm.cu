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

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <vector>
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
  int32_t splits;  // split-K factor (ACC_F32 only: partial sums meet in the TMA reduce-add)
  int32_t streamk;  // 1: stream-K (ACC_F32 only): every CTA (pair) takes an equal run of the
                    // tiles x k-blocks sequence; a tile cut between two runs is summed by
                    // the reduce-add like a split
  // implicit-GEMM 3x3 convolution (MODE 1-3): image H x W of the im2col
  // operand, its 64-channel blocks, and (dgrad) the output-channel blocks
  int32_t cv_h, cv_w, cv_cb, cv_cbo;
  unsigned long long *span;  // profiling: {~first start, last end} globaltimer (null = off)
  void *d;
  int64_t ldd;
  const float *bias;
  void *aux;
  int64_t ld_aux;
  int32_t epi;
};

// CG = CTAs per tile: 1 (128 x BN tile, one SM) or 2 (a CTA pair on one TPC
// computes a 256 x BN tile with tcgen05.mma.cta_group::2: each CTA stages its
// own 128 rows of A and HALF of B's BN rows, so per-SM operand traffic per
// FLOP drops by a third at BN = 256).
template <int BN, int CG, int B_MN = 0>
struct Cfg {
  static constexpr int kBRows = BN / CG;  // B rows staged per CTA
  // MN-major B is staged in 64-column swizzle atoms: a 96-row half (BN = 192
  // pair) takes two atoms, the second half-used (its other 32 columns belong
  // to the peer CTA and are loaded but never read)
  static constexpr int kBChunks = (kBRows + 63) / 64;
  static constexpr uint32_t kABytes = BM * BK * 2;
  static constexpr uint32_t kBBytes = B_MN ? kBChunks * 64 * BK * 2 : kBRows * BK * 2;
  static constexpr int kStages = (int)((196608u) / (kABytes + kBBytes)) > 8 ? 8 : (int)(196608u / (kABytes + kBBytes));
  static constexpr uint32_t kTmemCols = 2 * BN > 256 ? 512 : (2 * BN > 128 ? 256 : 128);  // pow2 >= 2 BN
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBBytes) + kEpiWarps * 4096 + 256;
};

// The work units a persistent CTA (pair) `slot` of `nslots` visits, in order:
// (tile, k-block range).  Classic: units (tile, split) round robin.  Stream-K:
// the contiguous run [slot * T / nslots, (slot + 1) * T / nslots) of the
// T = tiles x num_k k-block sequence, cut at tile boundaries.
struct UnitIter {
  int64_t g, g_end;  // stream-K cursor / end, or classic unit index / unit count
  int step;
  __device__ UnitIter(const Args &a, int slot, int nslots) {
    const int64_t tiles = (int64_t)a.num_m * a.num_n;
    if (a.streamk) {
      const int64_t T = tiles * a.num_k;
      g = slot * T / nslots;
      g_end = (slot + 1) * T / nslots;
      step = 0;
    } else {
      g = slot;
      g_end = tiles * a.splits;
      step = nslots;
    }
  }
  __device__ bool next(const Args &a, int &tile, int &kb0, int &kb1) {
    if (g >= g_end) return false;
    if (a.streamk) {
      tile = (int)(g / a.num_k);
      kb0 = (int)(g - (int64_t)tile * a.num_k);
      kb1 = (int)min((int64_t)a.num_k, kb0 + (g_end - g));
      g += kb1 - kb0;
    } else {
      tile = (int)(g / a.splits);
      const int sp = (int)(g - (int64_t)tile * a.splits);
      kb0 = (int)((int64_t)sp * a.num_k / a.splits);
      kb1 = (int)((int64_t)(sp + 1) * a.num_k / a.splits);
      g += step;
    }
    return true;
  }
};

// grouped raster: kGroupM row-tiles sweep the column tiles together (L2 reuse of B)
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
  return 0.5f * x * (1.f + tanh_approx(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float dgelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanh_approx(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

// Epilogue staging: each epilogue warp owns a 4 KB shared-memory buffer that
// holds one 32-row x 32-column chunk of the tile.  fp32 chunks are 128 B rows
// in the TMA SWIZZLE_128B layout, bf16 chunks 64 B rows in SWIZZLE_64B, so the
// thread-per-row writes out of tcgen05.ld are bank-conflict free and the chunk
// leaves (and source operands arrive) as one coalesced TMA bulk tensor copy.
constexpr int kEpiBuf = 4096;

__device__ __forceinline__ uint32_t sw128_off(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }
__device__ __forceinline__ uint32_t sw64_off(int r, int j) { return r * 64 + ((j ^ ((r >> 1) & 3)) << 4); }

// Sources read back through TMA before the epilogue math: the residual
// (RESID_F32) and the pre-activation (DGELU_BF16).  ACC_F32 reads nothing: its
// chunk leaves as a TMA reduce-add, which also makes split-K free of fix-ups.
__device__ __forceinline__ bool epi_src_f32(int epi) { return epi == HM_EPI_RESID_F32; }
__host__ __device__ __forceinline__ bool epi_src_bf16(int epi) {
  return epi == HM_EPI_DGELU_BF16 || epi == HM_EPI_RESID_RELU_BF16 || epi == HM_EPI_DRELU_BF16 ||
         epi == HM_EPI_ADD_BF16;
}
__host__ __device__ __forceinline__ bool epi_takes_bias(int epi) {
  return epi != HM_EPI_ACC_F32 && epi != HM_EPI_DGELU_BF16 && epi != HM_EPI_DRELU_BF16 && epi != HM_EPI_ADD_BF16;
}

// Apply the epilogue to one row's 32 columns [col0, col0+32) held in v and
// write the result(s) into the warp's staging buffer (row r = lane).
__device__ __forceinline__ void epilogue_chunk(const Args &a, int col0, float (&v)[32], uint8_t *buf, int r) {
  const int N = a.N;
  if (a.bias && epi_takes_bias(a.epi)) {
    if (col0 + 32 <= N) {
      const float4 *b4 = reinterpret_cast<const float4 *>(a.bias + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 b = __ldg(b4 + j);
        v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < N) v[j] += __ldg(a.bias + col0 + j);
    }
  }
  switch (a.epi) {
    case HM_EPI_STORE_F32:
    case HM_EPI_ACC_F32:
    case HM_EPI_RESID_F32: {
      const bool src = a.epi == HM_EPI_RESID_F32;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 *p = reinterpret_cast<float4 *>(buf + sw128_off(r, j));
        float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        if (src) {
          const float4 s = *p;
          o.x += s.x; o.y += s.y; o.z += s.z; o.w += s.w;
        }
        *p = o;
      }
      break;
    }
    case HM_EPI_STORE_BF16:
    case HM_EPI_GELU_BF16:
    case HM_EPI_DGELU_BF16:
    case HM_EPI_RELU_BF16:
    case HM_EPI_RESID_RELU_BF16:
    case HM_EPI_DRELU_BF16:
    case HM_EPI_ADD_BF16: {
      uint8_t *out = buf;
      if (a.epi == HM_EPI_RESID_RELU_BF16 || a.epi == HM_EPI_DRELU_BF16 || a.epi == HM_EPI_ADD_BF16) {
        // bf16 source chunk (residual or post-activation) landed in buf
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 p = *reinterpret_cast<const uint4 *>(buf + sw64_off(r, j));
          const __nv_bfloat162 *p2 = reinterpret_cast<const __nv_bfloat162 *>(&p);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(p2[e]);
            float &v0 = v[8 * j + 2 * e], &v1 = v[8 * j + 2 * e + 1];
            if (a.epi == HM_EPI_DRELU_BF16) {
              v0 = f.x > 0.f ? v0 : 0.f;
              v1 = f.y > 0.f ? v1 : 0.f;
            } else {
              v0 += f.x;
              v1 += f.y;
            }
          }
        }
      }
      if (a.epi == HM_EPI_RELU_BF16 || a.epi == HM_EPI_RESID_RELU_BF16) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
      }
      if (a.epi == HM_EPI_DGELU_BF16) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 p = *reinterpret_cast<const uint4 *>(buf + sw64_off(r, j));
          const __nv_bfloat162 *p2 = reinterpret_cast<const __nv_bfloat162 *>(&p);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 f = __bfloat1622float2(p2[e]);
            v[8 * j + 2 * e] *= dgelu_f(f.x);
            v[8 * j + 2 * e + 1] *= dgelu_f(f.y);
          }
        }
      } else if (a.epi == HM_EPI_GELU_BF16) {
        // pre-activation -> first half of the buffer, activation -> second half
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 p;
          __nv_bfloat162 *p2 = reinterpret_cast<__nv_bfloat162 *>(&p);
#pragma unroll
          for (int e = 0; e < 4; ++e) p2[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
          *reinterpret_cast<uint4 *>(buf + sw64_off(r, j)) = p;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
        out = buf + kEpiBuf / 2;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 p;
        __nv_bfloat162 *p2 = reinterpret_cast<__nv_bfloat162 *>(&p);
#pragma unroll
        for (int e = 0; e < 4; ++e) p2[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
        *reinterpret_cast<uint4 *>(out + sw64_off(r, j)) = p;
      }
      break;
    }
    default:
      break;
  }
}

// MODE: 0 plain GEMM (2-D tensor maps)
//       1 conv fwd   A = im2col(x): one k-block = 64 channels of one filter tap
//       2 conv dgrad A = im2col(dy), B = W[Cout][9][Cin] through a 3-D map with
//                    the tap flipped (dx = correlation of dy with the rotated W)
//       3 conv wgrad B = im2col(x) in 64-pixel x 64-channel MN-major chunks
template <int BN, int A_MN, int B_MN, int CG, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX, Args args) {
  using C = Cfg<BN, CG, B_MN>;
  constexpr int kTileM = BM * CG;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared address space (STS / LDS, not generic ST / LD)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * C::kABytes;
  uint8_t *sEpi = sB + C::kStages * C::kBBytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sEpi + kEpiWarps * kEpiBuf);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;
  uint64_t *tempty = tfull + 2;
  uint64_t *ebar = tempty + 2;  // one per epilogue warp: source chunk landed
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(ebar + kEpiWarps);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // 0 = pair leader (issues the MMAs)
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmD);
    tma_prefetch(&tmX);
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CG * kEpiWarps);  // one arrival per epilogue warp of every CTA of the tile
    }
    for (int i = 0; i < kEpiWarps; ++i) mbar_init(&ebar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if (CG == 2)
      tmem_alloc_pair<C::kTmemCols>(tmem_slot);
    else
      tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int slot = blockIdx.x / CG, nslots = gridDim.x / CG;  // persistent CTA (pair) index

  if (warp == 0) {
    if (lane == 0) {
      // programmatic dependent launch: everything above (barrier init, TMEM
      // alloc, descriptor prefetch) overlapped the previous kernel's tail;
      // global operands are read only after it has fully completed
      griddep_wait();
      if (args.span) atomicMax(&args.span[0], ~globaltimer());
      int stage = 0;
      uint32_t phase = 0;
      UnitIter it(args, slot, nslots);
      int tile, kb0, kb1;
      while (it.next(args, tile, kb0, kb1)) {
        int mb, nb;
        tile_coord(tile, args.num_m, args.num_n, mb, nb);
        const int m0 = mb * kTileM + (int)rank * BM;           // this CTA's A rows
        const int n0 = nb * BN + (int)rank * C::kBRows;        // this CTA's B rows
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint32_t bar_addr = smem_u32(&full[stage]);
          if (leader) mbar_expect_tx(&full[stage], CG * (C::kABytes + C::kBBytes));
          if (CG == 2) bar_addr = mapa_shared(bar_addr, 0);
          uint8_t *a_dst = sA + stage * C::kABytes;
          uint8_t *b_dst = sB + stage * C::kBBytes;
          auto load = [&](uint8_t *dst, const CUtensorMap *m, int c0, int c1) {
            if (CG == 2)
              tma_load_2d_pair(dst, m, bar_addr, c0, c1);
            else
              tma_load_2d(dst, m, &full[stage], c0, c1);
          };
          // im2col gather of 64 channels [c0, c0+64) of filter tap `tap` for the
          // pixels starting at flat NHW index p (base pixel = p - (1, 1))
          auto load_im2col = [&](uint8_t *dst, const CUtensorMap *m, int c0, int tap, int p) {
            const int hw = args.cv_h * args.cv_w;
            const int n = p / hw, rem = p - n * hw, h = rem / args.cv_w, w = rem - h * args.cv_w;
            const uint16_t r = (uint16_t)(tap / 3), s = (uint16_t)(tap - 3 * (tap / 3));
            if (CG == 2)
              tma_load_im2col_pair(dst, m, bar_addr, c0, w - 1, h - 1, n, s, r);
            else
              tma_load_im2col(dst, m, &full[stage], c0, w - 1, h - 1, n, s, r);
          };
          if (MODE == 1 || MODE == 2) {
            const int tap = kb / args.cv_cb;
            load_im2col(a_dst, &tmA, (kb - tap * args.cv_cb) * 64, tap, m0);
          } else if (!A_MN) {
            load(a_dst, &tmA, kb * BK, m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) load(a_dst + c * (BK * 128), &tmA, m0 + c * 64, kb * BK);
          }
          if (MODE == 2) {
            // K = (tap', co): 64 output channels of tap' against the flipped tap
            const int tap = kb / args.cv_cbo, co0 = (kb - tap * args.cv_cbo) * 64;
#pragma unroll
            for (int c = 0; c < C::kBRows / 64; ++c) {
              if (CG == 2)
                tma_load_3d_pair(b_dst + c * (BK * 128), &tmB, bar_addr, n0 + c * 64, 8 - tap, co0);
              else
                tma_load_3d(b_dst + c * (BK * 128), &tmB, &full[stage], n0 + c * 64, 8 - tap, co0);
            }
          } else if (MODE == 3) {
            // N = (tap, ci): each 64-column chunk is one tap's 64-channel block
#pragma unroll
            for (int c = 0; c < C::kBRows / 64; ++c) {
              const int nbk = (n0 >> 6) + c, tap = nbk / args.cv_cb;
              load_im2col(b_dst + c * (BK * 128), &tmB, (nbk - tap * args.cv_cb) * 64, tap, kb * BK);
            }
          } else if (!B_MN) {
            load(b_dst, &tmB, kb * BK, n0);
          } else {
#pragma unroll
            for (int c = 0; c < C::kBChunks; ++c) load(b_dst + c * (BK * 128), &tmB, n0 + c * 64, kb * BK);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // every CTA must trigger (or exit) before the dependent grid may launch:
      // the pair follower has no MMA thread, so its producer signals here
      if (CG == 2 && !leader) griddep_launch_dependents();
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(kTileM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      UnitIter it(args, slot, nslots);
      int tile, kb0, kb1;
      for (; it.next(args, tile, kb0, kb1); ++local) {
        const int acc = local & 1;
        const uint32_t use = (uint32_t)(local >> 1);
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
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
            const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
            if (CG == 2)
              mma_bf16_pair(d_tmem, da, db, idesc, accum);
            else
              mma_bf16(d_tmem, da, db, idesc, accum);
          }
          if (CG == 2)
            mma_commit_pair(&empty[stage], 0x3);
          else
            mma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2)
          mma_commit_pair(&tfull[acc], 0x3);
        else
          mma_commit(&tfull[acc]);
      }
      griddep_launch_dependents();  // only epilogues remain: let the next kernel set up
    }
  } else if (warp >= 4) {
    const int q = warp & 3;              // a warp may only touch TMEM lanes 32*(warp%4)..+31
    const int half = (warp - 4) >> 2;    // which half of the tile's columns
    constexpr int kChunks = BN / 32 / (kEpiWarps / 4);
    uint8_t *buf = sEpi + (warp - 4) * kEpiBuf;
    uint64_t *bar = &ebar[warp - 4];
    uint32_t bphase = 0;
    const int epi = args.epi;
    const bool src_f32 = epi_src_f32(epi);
    const bool has_src = src_f32 || epi_src_bf16(epi);
    const CUtensorMap *tsrc = &tmX;
    griddep_wait();  // epilogue reads / writes global memory of the previous kernel's outputs
    int local = 0;
    UnitIter it(args, slot, nslots);
    int tile, kb0_, kb1_;
    for (; it.next(args, tile, kb0_, kb1_); ++local) {
      int mb, nb;
      tile_coord(tile, args.num_m, args.num_n, mb, nb);
      const int acc = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      const int row0 = mb * kTileM + (int)rank * BM + q * 32;
      const int c_first = half * kChunks;
      // free the staging buffer and start the chunk's source-operand load
      auto prep = [&](int c) {
        if (lane == 0) {
          bulk_wait_read0();
          if (has_src) {
            mbar_expect_tx(bar, src_f32 ? 4096u : 2048u);
            tma_load_2d(buf, tsrc, bar, nb * BN + c * 32, row0);
          }
        }
        __syncwarp();
      };
      if (nb * BN + c_first * 32 < args.N) prep(c_first);  // overlaps the wait for the accumulator
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = c_first; c < c_first + kChunks; ++c) {
        const int col0 = nb * BN + c * 32;
        if (col0 >= args.N) break;
        if (c != c_first) prep(c);
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (has_src) {
          mbar_wait(bar, bphase);
          bphase ^= 1;
        }
        epilogue_chunk(args, col0, v, buf, (int)lane);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (epi == HM_EPI_GELU_BF16) {
            tma_store_2d(&tmX, buf, col0, row0);
            tma_store_2d(&tmD, buf + kEpiBuf / 2, col0, row0);
          } else if (epi == HM_EPI_ACC_F32) {
            tma_reduce_add_2d(&tmD, buf, col0, row0);
          } else {
            tma_store_2d(&tmD, buf, col0, row0);
          }
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2)
          mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        else
          mbar_arrive(&tempty[acc]);
      }
    }
    if (lane == 0) bulk_wait0();  // stores complete before the CTA (and its smem) retires
  }
  if (CG == 2) {
    tc_fence_before();
    cluster_sync();  // no remote arrive may target a CTA that has left; TMEM freed by both
  } else {
    __syncthreads();
  }
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_pair<C::kTmemCols>(tmem_base);
    else
      tmem_dealloc<C::kTmemCols>(tmem_base);
  }
  if (args.span && threadIdx.x == 0) atomicMax(&args.span[1], globaltimer());
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

// 2D map: inner dim d0 (contiguous), outer d1, row pitch in bytes, box {box0, box1}.
// Operand maps are bf16 {64, rows} SW128 (one 128-B swizzle atom per row);
// epilogue maps are {32, 32} chunks: fp32 SW128 (128-B rows), bf16 SW64 (64-B rows).
static int make_map(CUtensorMap *out, const void *ptr, uint64_t d0, uint64_t d1, uint64_t pitch_bytes,
                    uint32_t box1, bool f32 = false, uint32_t box0 = 64) {
  using Key = std::tuple<const void *, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t, bool>;
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  Key key{ptr, d0, d1, pitch_bytes, box1, box0, f32};
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
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  const uint32_t row_bytes = box0 * (f32 ? 4 : 2);
  const CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  CUresult r = fn(out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void *>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *out;
  return HM_OK;
}

static int num_sms();

struct TileCfg {
  int bn, cg, splits, streamk;
};

static int env_int(const char *name) {
  const char *e = getenv(name);
  return e ? atoi(e) : 0;
}

// Tile shape, CTA pairing and split-K from a wave-quantisation cost model:
//   time = waves x (k-blocks per unit + ~4 k-blocks of fill / epilogue tail) x t_kb
// where a unit is a (128*cg) x bn output tile (or one of its k-splits), waves =
// ceil(units / (SMs / cg)), and t_kb is the time of one 64-deep k-block of a
// unit relative to the MMA bound: bn / 256 / eff(cg, bn).  eff is the
// fraction of tensor peak each shape sustains on long-K problems, measured on
// B200 (profiles/r01_gemm_tile_sweep.jsonl: 8192^3 runs at 1550 TFLOP/s on
// 256x256 pair tiles, 1382 on 128x256, < 1000 on 128-wide tiles; operand
// traffic per SM per MMA cycle 64 / 96 / 96-128 B).  Split-K only for ACC_F32
// (partials meet in the TMA reduce-add).  HM_GEMM_BN / HM_GEMM_CG /
// HM_GEMM_SPLITK force a choice.
static int g_force_bn = env_int("HM_GEMM_BN"), g_force_cg = env_int("HM_GEMM_CG"),
           g_force_s = env_int("HM_GEMM_SPLITK");
// stream-K for ACC_F32: 1 = always, -1 = when the cost model prefers it, unset / 0 =
// never (hm_k_gemm_set_tile splits = -1 also forces it).  Off by default: on the
// GPT-2 XL weight-gradient shapes it measured 2-9% slower than the split-K units
// the model picks (profiles/r02_gemm_streamk_ab.jsonl): every CTA pair touches 3-4
// tile segments, each paying a pipeline fill and a full-tile reduce-add epilogue.
static const int g_streamk = getenv("HM_GEMM_STREAMK") ? atoi(getenv("HM_GEMM_STREAMK")) : 0;
// 128 x 192 single-CTA tiles (fit 1600-wide outputs in 9 column tiles)
static const bool g_tile192 = getenv("HM_GEMM_192") ? atoi(getenv("HM_GEMM_192")) != 0 : true;
static const double g_eff192 = getenv("HM_GEMM_EFF192") ? atof(getenv("HM_GEMM_EFF192")) : 0.70;
// 256 x 192 pair tiles (an MN-major B half of 96 rows is staged as two
// 64-column atoms, a third more B traffic: g_eff192pm)
static const double g_eff192p = getenv("HM_GEMM_EFF192P") ? atof(getenv("HM_GEMM_EFF192P")) : 0.80;
static const double g_eff192pm = getenv("HM_GEMM_EFF192PM") ? atof(getenv("HM_GEMM_EFF192PM")) : 0.78;

int &max_kblocks_per_split() {
  static int v = 0;
  return v;
}

static TileCfg pick_tile(int64_t M, int64_t N, int64_t K, int epi, bool allow192 = true, bool b_mn = false) {
  const int env_bn = g_force_bn, env_cg = g_force_cg, env_s = g_force_s > 0 ? g_force_s : 0;
  const bool acc = epi == HM_EPI_ACC_F32;
  // accuracy cap (fp32-operand mode): the tensor core's fp32 accumulation over a
  // long K chain loses ~1e-5 relative at K = 6400 vs ~2e-6 in three splits
  // summed by the reduce-add (profiles/r02_gemm_split_accuracy.jsonl)
  const int64_t kcap = acc ? max_kblocks_per_split() : 0;
  const bool force_sk = acc && (g_force_s == -1 || g_streamk == 1), allow_sk = acc && !env_s && g_streamk != 0;
  const int64_t sms = num_sms();
  const int64_t num_k = (K + BK - 1) / BK;
  TileCfg best{256, 1, 1, 0};
  double best_t = 1e300;
  for (int cg = 1; cg <= 2; ++cg) {
    if (env_cg && cg != env_cg) continue;
    for (int bn : {128, 192, 256}) {
      if (env_bn && bn != env_bn) continue;
      if (bn == 192 && (!g_tile192 || !allow192)) continue;
      // pair tiles lose more when B is MN-major (dgrad / wgrad: 64-wide B chunks per k-block)
      const double eff = bn == 128   ? 0.55
                         : bn == 192 ? (cg == 1 ? g_eff192 : (b_mn ? g_eff192pm : g_eff192p))
                                     : (cg == 1 ? 0.80 : (b_mn ? 0.86 : 0.93));
      const double t_kb = bn / 256.0 / eff;
      const int64_t tiles = ((M + BM * cg - 1) / (BM * cg)) * ((N + bn - 1) / bn);
      const int64_t slots = sms / cg;
      const int64_t num_k_tot = (K + BK - 1) / BK;
      const int s_min = kcap > 0 ? (int)std::min<int64_t>(32, (num_k_tot + kcap - 1) / kcap) : 1;
      for (int s = 1; s <= (acc ? 32 : 1); ++s) {
        if (env_s && s != env_s) continue;
        if (s < s_min && !env_s) continue;
        if (s > 1 && num_k / s < 8 && s > s_min) break;
        const double waves = (double)((tiles * s + slots - 1) / slots);
        const double t = waves * ((double)num_k / s + 4.0) * t_kb * (s > 1 ? 1.03 : 1.0);
        if (t < best_t && !force_sk) {
          best_t = t;
          best = TileCfg{bn, cg, s, 0};
        }
      }
      // stream-K (reduce-add epilogue only): every slot runs ceil(tiles x num_k / slots)
      // k-blocks, paying the fill / epilogue tail once per tile segment it touches
      if (allow_sk || force_sk) {
        const int64_t per = (tiles * num_k + slots - 1) / slots;
        const int64_t segs = std::min<int64_t>(tiles, (per + num_k - 1) / num_k + 1);
        const double t = ((double)per + 4.0 * (double)segs) * t_kb * 1.02;
        if (t < best_t || (force_sk && !best.streamk)) {
          best_t = t;
          best = TileCfg{bn, cg, 1, 1};
        }
      }
    }
  }
  return best;
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

template <int BN, int A_MN, int B_MN, int CG, int MODE = 0>
static int launch(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &td, const CUtensorMap &tx,
                  const Args &a, cudaStream_t s) {
  using C = Cfg<BN, CG, B_MN>;
  static bool attr = false;
  auto kern = gemm_kernel<BN, A_MN, B_MN, CG, MODE>;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    if (e != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("gemm smem attr: ") + cudaGetErrorString(e));
    attr = true;
  }
  const int units = a.streamk ? a.num_m * a.num_n * a.num_k : a.num_m * a.num_n * a.splits;
  const int grid = CG * std::min(units, num_sms() / CG);
  const bool f32 = a.epi == HM_EPI_STORE_F32 || a.epi == HM_EPI_ACC_F32 || a.epi == HM_EPI_RESID_F32;
  const double io = (double)a.M * a.N * (f32 ? 4 : 2) * (a.epi == HM_EPI_ACC_F32 || a.epi >= HM_EPI_RESID_F32 ? 2 : 1);
  ProfScope ps(KC_GEMM, s, 2.0 * a.M * a.N * a.K, 2.0 * ((double)a.M * a.K + (double)a.N * a.K) + io);
  Args args = a;
  args.span = profiler() ? profiler()->span_slot() : nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = CG;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  static const bool pdl = !(getenv("HM_GEMM_PDL") && getenv("HM_GEMM_PDL")[0] == '0');
  attrs[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = CG > 1 ? 2 : 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, ta, tb, td, tx, args);
  if (le != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("gemm launch: ") + cudaGetErrorString(le));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HM_ERR_DEVICE, std::string("gemm launch: ") + cudaGetErrorString(e));
  count_launch();
  return HM_OK;
}

std::vector<int64_t> *&shape_log() {
  static std::vector<int64_t> *log = nullptr;
  return log;
}

int run(const void *A, const void *B, void *D, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
        int64_t ldd, int a_mn, int b_mn, int epi, const float *bias, void *aux, int64_t ld_aux,
        cudaStream_t stream, int force_bn) {
  if (M <= 0 || N <= 0 || K <= 0) return fail(HM_ERR_VALIDATION, "gemm: empty problem");
  if (shape_log()) shape_log()->insert(shape_log()->end(), {M, N, K, a_mn, b_mn, epi, bias ? 1 : 0});
  if (epi < HM_EPI_STORE_BF16 || epi > HM_EPI_ADD_BF16) return fail(HM_ERR_VALIDATION, "gemm: unknown epilogue");
  if ((lda * 2) % 16 || (ldb * 2) % 16) return fail(HM_ERR_VALIDATION, "gemm: operand pitch must be 16B aligned");
  if (((uintptr_t)A | (uintptr_t)B) & 15) return fail(HM_ERR_VALIDATION, "gemm: operands must be 16B aligned");
  const bool f32out = epi == HM_EPI_STORE_F32 || epi == HM_EPI_ACC_F32 || epi == HM_EPI_RESID_F32;
  if ((ldd * (f32out ? 4 : 2)) % 16 || ((uintptr_t)D & 15))
    return fail(HM_ERR_VALIDATION, "gemm: output must be 16B aligned with 16B pitch");
  if ((epi == HM_EPI_RESID_F32 || epi == HM_EPI_GELU_BF16 || epi_src_bf16(epi)) && !aux)
    return fail(HM_ERR_VALIDATION, "gemm: epilogue needs an aux tensor");
  if (aux && ((ld_aux * (epi == HM_EPI_RESID_F32 ? 4 : 2)) % 16 || ((uintptr_t)aux & 15)))
    return fail(HM_ERR_VALIDATION, "gemm: aux must be 16B aligned with 16B pitch");
  TileCfg tc = pick_tile(M, N, K, epi, true, b_mn != 0);
  if (force_bn) tc.bn = force_bn;
  const int bn = tc.bn;
  Args a{};
  a.M = (int)M; a.N = (int)N; a.K = (int)K;
  a.num_m = (int)((M + BM * tc.cg - 1) / (BM * tc.cg));
  a.num_n = (int)((N + bn - 1) / bn);
  a.num_k = (int)((K + BK - 1) / BK);
  a.splits = tc.splits;
  a.streamk = tc.streamk;
  a.d = D; a.ldd = ldd; a.bias = bias; a.aux = aux; a.ld_aux = ld_aux; a.epi = epi;
  CUtensorMap ta, tb, td, tx;
  int rc = a_mn ? make_map(&ta, A, M, K, lda * 2, 64) : make_map(&ta, A, K, M, lda * 2, BM);
  if (rc) return rc;
  rc = b_mn ? make_map(&tb, B, N, K, ldb * 2, 64) : make_map(&tb, B, K, N, ldb * 2, bn / tc.cg);
  if (rc) return rc;
  rc = make_map(&td, D, N, M, ldd * (f32out ? 4 : 2), 32, f32out, 32);
  if (rc) return rc;
  if (aux) {
    const bool aux_f32 = epi == HM_EPI_RESID_F32;
    rc = make_map(&tx, aux, N, M, ld_aux * (aux_f32 ? 4 : 2), 32, aux_f32, 32);
    if (rc) return rc;
  } else {
    tx = td;
  }
  if (bn == 192 && tc.cg == 2) {
    switch ((a_mn ? 2 : 0) | (b_mn ? 1 : 0)) {
      case 0: return launch<192, 0, 0, 2>(ta, tb, td, tx, a, stream);
      case 1: return launch<192, 0, 1, 2>(ta, tb, td, tx, a, stream);
      case 2: return launch<192, 1, 0, 2>(ta, tb, td, tx, a, stream);
      default: return launch<192, 1, 1, 2>(ta, tb, td, tx, a, stream);
    }
  }
  if (bn == 192) {
    switch ((a_mn ? 2 : 0) | (b_mn ? 1 : 0)) {
      case 0: return launch<192, 0, 0, 1>(ta, tb, td, tx, a, stream);
      case 1: return launch<192, 0, 1, 1>(ta, tb, td, tx, a, stream);
      case 2: return launch<192, 1, 0, 1>(ta, tb, td, tx, a, stream);
      default: return launch<192, 1, 1, 1>(ta, tb, td, tx, a, stream);
    }
  }
  const int key = (tc.cg == 2 ? 8 : 0) | (bn == 256 ? 4 : 0) | (a_mn ? 2 : 0) | (b_mn ? 1 : 0);
  switch (key) {
    case 0: return launch<128, 0, 0, 1>(ta, tb, td, tx, a, stream);
    case 1: return launch<128, 0, 1, 1>(ta, tb, td, tx, a, stream);
    case 2: return launch<128, 1, 0, 1>(ta, tb, td, tx, a, stream);
    case 3: return launch<128, 1, 1, 1>(ta, tb, td, tx, a, stream);
    case 4: return launch<256, 0, 0, 1>(ta, tb, td, tx, a, stream);
    case 5: return launch<256, 0, 1, 1>(ta, tb, td, tx, a, stream);
    case 6: return launch<256, 1, 0, 1>(ta, tb, td, tx, a, stream);
    case 7: return launch<256, 1, 1, 1>(ta, tb, td, tx, a, stream);
    case 8: return launch<128, 0, 0, 2>(ta, tb, td, tx, a, stream);
    case 9: return launch<128, 0, 1, 2>(ta, tb, td, tx, a, stream);
    case 10: return launch<128, 1, 0, 2>(ta, tb, td, tx, a, stream);
    case 11: return launch<128, 1, 1, 2>(ta, tb, td, tx, a, stream);
    case 12: return launch<256, 0, 0, 2>(ta, tb, td, tx, a, stream);
    case 13: return launch<256, 0, 1, 2>(ta, tb, td, tx, a, stream);
    case 14: return launch<256, 1, 0, 2>(ta, tb, td, tx, a, stream);
    default: return launch<256, 1, 1, 2>(ta, tb, td, tx, a, stream);
  }
}

// ---- implicit-GEMM 3x3 convolution -------------------------------------------------
// im2col map over an NHWC bf16 activation [n, h, w, c]: base pixels range over
// [-1, dim-1) in W and H (zero padding 1, output size = input size), one
// 64-channel slice per request, `pixels` (128 or 64) pixels per request.
static int make_im2col_map(CUtensorMap *out, const void *ptr, int n, int h, int w, int c, uint32_t pixels) {
  using Key = std::tuple<const void *, int, int, int, int, uint32_t>;
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  Key key{ptr, n, h, w, c, pixels};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return HM_OK;
    }
  }
  using Im2colFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const int *, const int *, cuuint32_t, cuuint32_t,
                                const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Im2colFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<Im2colFn>(p);
    return (Im2colFn) nullptr;
  }();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeIm2col unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)w * c * 2, (cuuint64_t)h * w * c * 2};
  int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, lower, upper, 64,
                  pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 1024) cache.clear();
  cache[key] = *out;
  return HM_OK;
}

// W[cout][9][cin] bf16 as a 3-D map {cin, 9, cout}, box {64, 1, 64}: one tap's
// 64 x 64 (cout x cin) block, cin contiguous (an MN-major B chunk for dgrad).
static int make_filter_map(CUtensorMap *out, const void *ptr, int cin, int cout) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(HM_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)cin, 9, (cuuint64_t)cout};
  cuuint64_t strides[2] = {(cuuint64_t)cin * 2, (cuuint64_t)cin * 9 * 2};
  cuuint32_t box[3] = {64, 1, 64};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HM_ERR_DEVICE, "filter tensor map failed (" + std::to_string((int)r) + ")");
  return HM_OK;
}

template <int MODE, int A_MN, int B_MN>
static int launch_conv(const TileCfg &tc, const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &td,
                       const CUtensorMap &tx, const Args &a, cudaStream_t s) {
  const int key = (tc.cg == 2 ? 2 : 0) | (tc.bn == 256 ? 1 : 0);
  switch (key) {
    case 0: return launch<128, A_MN, B_MN, 1, MODE>(ta, tb, td, tx, a, s);
    case 1: return launch<256, A_MN, B_MN, 1, MODE>(ta, tb, td, tx, a, s);
    case 2: return launch<128, A_MN, B_MN, 2, MODE>(ta, tb, td, tx, a, s);
    default: return launch<256, A_MN, B_MN, 2, MODE>(ta, tb, td, tx, a, s);
  }
}

// mode 1 fwd, 2 dgrad, 3 wgrad (see the kernel's MODE comment)
int run_conv(int mode, const void *act, const void *wt, void *out, int n, int h, int w, int cin, int cout, int epi,
             const float *bias, const void *aux, cudaStream_t stream) {
  if (n <= 0 || h <= 0 || w <= 0 || cin <= 0 || cout <= 0) return fail(HM_ERR_VALIDATION, "conv: empty problem");
  if (cin % 64 || cout % 64) return fail(HM_ERR_VALIDATION, "conv: channels must be multiples of 64");
  if (((uintptr_t)act | (uintptr_t)wt | (uintptr_t)out | (uintptr_t)aux) & 15)
    return fail(HM_ERR_VALIDATION, "conv: tensors must be 16B aligned");
  const int64_t P = (int64_t)n * h * w;
  if (P >= (int64_t)1 << 31) return fail(HM_ERR_VALIDATION, "conv: too many pixels");
  int64_t M, N, K;
  if (mode == 1) { M = P; N = cout; K = 9LL * cin; }
  else if (mode == 2) { M = P; N = cin; K = 9LL * cout; }
  else { M = cout; N = 9LL * cin; K = P; epi = HM_EPI_ACC_F32; }
  if (mode != 3 && (epi == HM_EPI_STORE_F32 || epi == HM_EPI_ACC_F32 || epi == HM_EPI_RESID_F32 ||
                    epi == HM_EPI_GELU_BF16))
    return fail(HM_ERR_VALIDATION, "conv: fwd/dgrad epilogues are the bf16 ones");
  if (epi_src_bf16(epi) && !aux) return fail(HM_ERR_VALIDATION, "conv: epilogue needs an aux tensor");
  TileCfg tc = pick_tile(M, N, K, epi, /*allow192=*/false, mode != 1);  // conv kernels come in 128 / 256 widths
  Args a{};
  a.M = (int)M; a.N = (int)N; a.K = (int)K;
  a.num_m = (int)((M + BM * tc.cg - 1) / (BM * tc.cg));
  a.num_n = (int)((N + tc.bn - 1) / tc.bn);
  a.num_k = (int)((K + BK - 1) / BK);
  a.splits = tc.splits;
  a.streamk = tc.streamk;
  a.d = out; a.ldd = N; a.bias = bias; a.aux = const_cast<void *>(aux); a.ld_aux = N; a.epi = epi;
  a.cv_h = h; a.cv_w = w; a.cv_cb = (mode == 2 ? cout : cin) / 64; a.cv_cbo = cout / 64;
  const bool f32out = mode == 3;
  CUtensorMap ta, tb, td, tx;
  int rc;
  if (mode == 1 || mode == 2) {
    rc = make_im2col_map(&ta, act, n, h, w, mode == 1 ? cin : cout, BM);
    if (rc) return rc;
    rc = mode == 1 ? make_map(&tb, wt, 9ULL * cin, cout, 9ULL * cin * 2, tc.bn / tc.cg) : make_filter_map(&tb, wt, cin, cout);
  } else {
    rc = make_map(&ta, act, cout, P, (uint64_t)cout * 2, 64);  // dy [P, cout] read MN-major
    if (rc) return rc;
    rc = make_im2col_map(&tb, wt, n, h, w, cin, BK);  // here `wt` is the activation x
  }
  if (rc) return rc;
  rc = make_map(&td, out, N, M, N * (f32out ? 4 : 2), 32, f32out, 32);
  if (rc) return rc;
  if (aux) {
    rc = make_map(&tx, aux, N, M, N * 2, 32, false, 32);
    if (rc) return rc;
  } else {
    tx = td;
  }
  if (mode == 1) return launch_conv<1, 0, 0>(tc, ta, tb, td, tx, a, stream);
  if (mode == 2) return launch_conv<2, 0, 1>(tc, ta, tb, td, tx, a, stream);
  return launch_conv<3, 1, 1>(tc, ta, tb, td, tx, a, stream);
}

}  // namespace gemm
}  // namespace hm

extern "C" int hm_k_conv_fwd(const void *x, const void *w, void *y, int32_t n, int32_t h, int32_t wd, int32_t cin,
                             int32_t cout, int32_t epilogue, const float *bias, const void *aux, void *stream) {
  return hm::gemm::run_conv(1, x, w, y, n, h, wd, cin, cout, epilogue, bias, aux, static_cast<cudaStream_t>(stream));
}
extern "C" int hm_k_conv_dgrad(const void *dy, const void *w, void *dx, int32_t n, int32_t h, int32_t wd, int32_t cin,
                               int32_t cout, int32_t epilogue, const void *aux, void *stream) {
  return hm::gemm::run_conv(2, dy, w, dx, n, h, wd, cin, cout, epilogue, nullptr, aux,
                            static_cast<cudaStream_t>(stream));
}
extern "C" int hm_k_conv_wgrad(const void *dy, const void *x, float *dw, int32_t n, int32_t h, int32_t wd, int32_t cin,
                               int32_t cout, void *stream) {
  return hm::gemm::run_conv(3, dy, x, dw, n, h, wd, cin, cout, HM_EPI_ACC_F32, nullptr, nullptr,
                            static_cast<cudaStream_t>(stream));
}

extern "C" int hm_k_gemm_set_tile(int32_t bn, int32_t cta_pair, int32_t splits) {
  if ((bn && bn != 128 && bn != 192 && bn != 256) || (cta_pair && cta_pair != 1 && cta_pair != 2) || splits < -1 ||
      splits > 32)
    return hm::fail(HM_ERR_VALIDATION,
                    "gemm tile override: bn in {0,128,192,256}, cta_pair in {0,1,2}, splits in [-1,32] (-1 = stream-K)");
  hm::gemm::g_force_bn = bn;
  hm::gemm::g_force_cg = cta_pair;
  hm::gemm::g_force_s = splits;
  return HM_OK;
}

extern "C" int hm_k_gemm_tile(int64_t m, int64_t n, int64_t k, int32_t epilogue, int32_t b_major, int32_t *bn,
                              int32_t *cta_pair, int32_t *splits) {
  const hm::gemm::TileCfg t = hm::gemm::pick_tile(m, n, k, epilogue, true, b_major != 0);
  *bn = t.bn;
  *cta_pair = t.cg;
  *splits = t.streamk ? 0 : t.splits;
  return HM_OK;
}

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
