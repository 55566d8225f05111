// C ABI of the Dense GEMMs (include/sgb200.h: sg_gemm).
#include <cuda_runtime.h>

#include "common.h"
#include "gemm.h"

namespace sg {
int ctx_num_sms(sg_ctx* ctx);
int ctx_compute_sms(sg_ctx* ctx);
int ctx_activate(sg_ctx* ctx);
}  // namespace sg

using namespace sg;

extern "C" int sg_gemm(sg_ctx* ctx, const sg_gemm_desc* d, void* stream) {
  SG_NVTX("sg_gemm");
  if (!ctx || !d) return fail(SG_EINVAL, "null argument");
  if (d->M < 0 || d->N < 0 || d->K < 0 || d->M > (1ll << 31) - 1 || d->N > (1ll << 31) - 1 ||
      d->K > (1ll << 31) - 1)
    return fail(SG_EINVAL, "gemm: bad extents");
  if (d->M == 0 || d->N == 0) return SG_OK;
  if (d->epilogue < SG_EPI_STORE || d->epilogue > SG_EPI_BIAS_MSE) return fail(SG_EINVAL, "gemm: bad epilogue");
  if (d->epilogue == SG_EPI_BIAS_MSE &&
      (d->precision != SG_PREC_BF16 || !d->aux || !d->out2_lp || !d->loss_part || d->act != SG_ACT_IDENTITY ||
       d->out_lp || d->batch > 1))
    return fail(SG_EINVAL, "gemm: BIAS_MSE needs BF16, identity, targets in aux, out2_lp and loss_part, no out_lp");
  if (d->epilogue == SG_EPI_BIAS_ACT_SEED &&
      (!d->aux || !d->out2_lp || d->batch > 1 ||
       !((d->precision == SG_PREC_BF16 && d->out_lp && !d->out) ||
         (d->precision == SG_PREC_TF32 && d->out && !d->out_lp))))
    return fail(SG_EINVAL, "gemm: BIAS_ACT_SEED needs the seed in aux and out2_lp, with BF16 out_lp (no fp32 out) "
                           "or TF32 out (fp32 h and out2)");
  if (d->act < SG_ACT_IDENTITY || d->act > SG_ACT_RELU) return fail(SG_EINVAL, "gemm: bad activation");
  if (d->epilogue == SG_EPI_ACT_GRAD && !d->aux) return fail(SG_EINVAL, "gemm: ACT_GRAD needs aux");
  const long long batch = d->batch < 1 ? 1 : d->batch;
  if (batch > 65535) return fail(SG_EINVAL, "gemm: at most 65535 batch entries");
  if (batch > 1 && (d->stride_a < 0 || d->stride_b < 0 || d->stride_out < 0 || d->stride_lp < 0))
    return fail(SG_EINVAL, "gemm: negative batch stride");
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (d->precision == SG_PREC_BF16 || d->precision == SG_PREC_TF32) {
    const bool tf32 = d->precision == SG_PREC_TF32;
    if (d->K == 0) return fail(SG_EINVAL, "gemm: K must be positive");
    if (tf32 && d->out_lp) return fail(SG_EINVAL, "gemm: out_lp is a BF16-precision output");
    GemmArgs g{};
    gemm_args_from_desc(ctx, d, g);
    return launch_gemm_tc(g, tf32, ctx_compute_sms(ctx), st);
  }
  if (d->precision == SG_PREC_STRICT_FP32 || d->precision == SG_PREC_STRICT_FP64) {
    if (d->out_lp) return fail(SG_EINVAL, "gemm: out_lp is a BF16-precision output");
    strict::StrictArgs g{(int)d->M, (int)d->N, (int)d->K, d->A, d->lda, d->a_mn_major != 0,
                         d->B, d->ldb, d->b_mn_major != 0, d->epilogue, d->act, ctx_domain_word(ctx), d->bias, d->aux,
                         d->ld_aux, d->out_pre, d->ld_pre, d->out, d->ld_out, (int)batch, d->stride_a,
                         d->stride_b, d->stride_out};
    return launch_gemm_strict(g, d->precision == SG_PREC_STRICT_FP64, st);
  }
  return fail(SG_EINVAL, "gemm: unknown precision");
}

namespace sg {
void gemm_args_from_desc(sg_ctx* ctx, const sg_gemm_desc* d, GemmArgs& g) {
  const bool tf32 = d->precision == SG_PREC_TF32;
  const long long batch = d->batch < 1 ? 1 : d->batch;
  g.M = (int)d->M;
  g.N = (int)d->N;
  g.K = (int)d->K;
  g.A = d->A;
  g.lda = d->lda;
  g.a_mn = d->a_mn_major != 0;
  g.B = d->B;
  g.ldb = d->ldb;
  g.b_mn = d->b_mn_major != 0;
  g.epi.mode = d->epilogue;
  g.epi.act = d->act;
  g.epi.bias = (const float*)d->bias;
  g.epi.aux = tf32 ? nullptr : (const __nv_bfloat16*)d->aux;
  g.epi.aux_f32 = tf32 ? (const float*)d->aux : nullptr;
  g.epi.ld_aux = d->ld_aux;
  g.epi.out_pre = (float*)d->out_pre;
  g.epi.ld_pre = d->ld_pre;
  g.epi.out_f32 = (float*)d->out;
  g.epi.ld_f32 = d->ld_out;
  g.epi.out_bf16 = (__nv_bfloat16*)d->out_lp;
  g.epi.ld_bf16 = d->ld_lp;
  g.epi.colsum = d->colsum;
  g.epi.ld_colsum = d->ld_colsum;
  g.epi.dom = ctx_domain_word(ctx);
  if (d->epilogue == SG_EPI_BIAS_MSE) {
    g.epi.aux = nullptr;  // the targets travel in aux (fp32)
    g.epi.seed = (const float*)d->aux;
    g.epi.ld_seed = d->ld_aux;
    g.epi.out2_bf16 = (__nv_bfloat16*)d->out2_lp;
    g.epi.ld_out2 = d->ld_out2;
    g.epi.loss_part = d->loss_part;
    g.epi.loss_scale = (float)d->loss_scale;
  }
  if (d->epilogue == SG_EPI_BIAS_ACT_SEED) {
    g.epi.aux = nullptr;  // the seed travels in aux: fp32, read per row in the epilogue
    g.epi.aux_f32 = nullptr;
    g.epi.seed = (const float*)d->aux;
    g.epi.ld_seed = d->ld_aux;
    if (tf32) g.epi.out2_f32 = (float*)d->out2_lp;  // TF32: h and dz in fp32
    else g.epi.out2_bf16 = (__nv_bfloat16*)d->out2_lp;
    g.epi.ld_out2 = d->ld_out2;
  }
  g.split_part = d->split_part;
  g.split_part_elems = d->split_part_elems;
  g.batch = (int)batch;
  g.sa = d->stride_a;
  g.sb = d->stride_b;
  g.so_f32 = d->stride_out;
  g.so_lp = d->stride_lp;
}
}  // namespace sg

extern "C" int sg_gemm_splits(sg_ctx* ctx, const sg_gemm_desc* d, int32_t* splits, int64_t* ld_part) {
  if (!ctx || !d || !splits || !ld_part) return fail(SG_EINVAL, "null argument");
  *splits = 1;
  *ld_part = (d->N + 3) / 4 * 4;
  if (d->precision != SG_PREC_BF16 && d->precision != SG_PREC_TF32) return SG_OK;  // strict GEMMs never split
  if (d->M <= 0 || d->N <= 0 || d->K <= 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  GemmArgs g{};
  gemm_args_from_desc(ctx, d, g);
  int s = 1;
  long long ld = 0;
  plan_gemm_splits(g, d->precision == SG_PREC_TF32, ctx_compute_sms(ctx), &s, &ld);
  *splits = s;
  *ld_part = ld;
  return SG_OK;
}

extern "C" int sg_splitk_reduce_multi(sg_ctx* ctx, int32_t n, const float* const* parts, const int32_t* splits,
                                      const int64_t* M, const int64_t* N, const int64_t* ld_part,
                                      float* const* outs, const int64_t* ld_out, void* stream) {
  SG_NVTX("sg_splitk_reduce_multi");
  if (!ctx || n < 0 || (n && (!parts || !splits || !M || !N || !ld_part || !outs || !ld_out)))
    return fail(SG_EINVAL, "null argument");
  if (n == 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  return splitk_reduce_multi(n, parts, splits, M, N, ld_part, outs, ld_out, (cudaStream_t)stream);
}
