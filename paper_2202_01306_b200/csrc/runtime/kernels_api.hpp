// kernels_api.hpp -- internal C++ entry points of the kernels (csrc/kernels/*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace hm {
int adam_launch_dev(float *w, const float *g, float *k, int64_t n, double b1, double b2, double eps,
                    const float *scalars, float gscale, cudaStream_t s);
int adam_launch(float *w, const float *g, float *k, int64_t n, double lr, double b1, double b2, double eps, int step,
                float gscale, cudaStream_t s);
namespace gemm {
int run(const void *A, const void *B, void *D, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldd,
        int a_mn, int b_mn, int epi, const float *bias, void *aux, int64_t ld_aux, cudaStream_t stream, int force_bn);
// when set, every gemm::run call appends {M, N, K, a_mn, b_mn, epi, has_bias}
std::vector<int64_t> *&shape_log();
// > 0: accumulating (ACC_F32) GEMMs split K so that no split sums more than
// this many 64-deep k-blocks in TMEM (the fp32-operand mode's accuracy knob)
int &max_kblocks_per_split();
}
namespace attn {
int forward(const void *qkv, void *o, float *lse, int B, int S, int H, int DH, int causal, cudaStream_t s);
int backward(const void *qkv, const void *o, const void *dout, const float *lse, float *dvec, float *dq_acc,
             void *dqkv, int B, int S, int H, int DH, int causal, cudaStream_t s);
}
namespace layers {
int cast_f32_bf16(const float *src, void *dst, int64_t n, cudaStream_t s);
// weight planes: hi = bf16 nearest, ties toward zero; lo = low 16 bits (exact split)
int cast_w_bf16(const float *src, void *dst, int64_t n, cudaStream_t s);
int w_join(const void *hi, const void *lo, float *w, int64_t n, cudaStream_t s);
int w_split(const float *w, void *hi, void *lo, int64_t n, cudaStream_t s);
int embed_fwd(const int32_t *tok, const float *wte, const float *wpe, float *out, int B, int S, int d, cudaStream_t s);
int embed_bwd(const int32_t *tok, const float *dx, float *dwte, float *dwpe, int B, int S, int d, cudaStream_t s);
int ln_fwd(const float *x, const float *g, const float *b, void *y, float *mean, float *rstd, int64_t rows, int d,
           cudaStream_t s);
int ln_bwd(const float *dy, const float *x, const float *mean, const float *rstd, const float *g, const float *resid,
           float *out, void *out_bf, float *dg, float *db, int64_t rows, int d, cudaStream_t s);
int cross_entropy(const float *logits, const int32_t *labels, int64_t rows, int64_t ldl, int V, void *dlogits,
                  double *loss_sum, float scale, cudaStream_t s);
int bias_grad(const void *dy, int is_bf16, float *db, int64_t rows, int n, int64_t ld, cudaStream_t s);
// out[i] = src[0][i] + src[1][i] + ... (n <= 8 sources, summed in that order)
int sum_ranks(const float *const *src, int n, float *out, int64_t count, cudaStream_t s);
}  // namespace layers
// fp32-operand parity mode (kernels/precise.cu): three-plane bf16 split GEMMs,
// fp32 SIMT attention / LayerNorm forward / cross-entropy
namespace prec {
int split3(const float *x, void *planes, int64_t n, int64_t plane, cudaStream_t s);
int gemm(const float *A, const float *B, void *D, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
         int64_t ldd, int a_mn, int b_mn, int epi, const float *bias, void *aux, int64_t ld_aux, cudaStream_t s,
         void *sa, int64_t sa_elems, void *sb, int64_t sb_elems, float *c32, int64_t c32_elems);
int ln_fwd(const float *x, const float *g, const float *b, float *y, float *mean, float *rstd, int64_t rows, int d,
           cudaStream_t s);
int cross_entropy(const float *logits, const int32_t *labels, int64_t rows, int64_t ldl, int V, float *dlogits,
                  double *loss_sum, float scale, cudaStream_t s);
int attn_forward(const float *qkv, float *o, float *lse, int B, int S, int H, int DH, int causal, cudaStream_t s);
int attn_backward(const float *qkv, const float *o, const float *dout, const float *lse, float *dvec, float *dqkv,
                  int B, int S, int H, int DH, int causal, cudaStream_t s);
}  // namespace prec
namespace gemm {
int run_conv(int mode, const void *act, const void *wt, void *out, int n, int h, int w, int cin, int cout, int epi,
             const float *bias, const void *aux, cudaStream_t stream);
}
namespace cnn {
int relu_bwd(const void *dy, const void *y, void *dz, int64_t n, cudaStream_t s);
int pool2_fwd(const void *a, void *y, int n, int h, int w, int c, cudaStream_t s);
int pool2_relu_bwd(const void *dy, const void *a, void *dz, int n, int h, int w, int c, cudaStream_t s);
int gap_fwd(const void *x, void *pooled, int nb, int P, int c, cudaStream_t s);
int gap_bwd(const float *dp, void *dx, int nb, int P, int c, cudaStream_t s);
int add_bf16(const void *a, const void *b, void *out, int64_t n, cudaStream_t s);
}  // namespace cnn
}  // namespace hm
