// C ABI of one Dense layer (include/sgb200.h: sg_dense_forward / sg_dense_backward).
//
// The layer of nn_train.py:189-196 (wt = transpose(W); z = matmul(h, wt);
// zb = add(z, b); h' = act(zb)) and its pullback (rules.py:45-46 add,
// 82-94 activations, 113-115 matmul, 123-124 transpose), each composed from
// the GEMM / reduction kernels in one call: the forward is ONE GEMM with the
// bias + activation epilogue; the pullback is dW = dZ^T X (both operands
// MN-major, no transposes), db = colsum(dZ) (finalising partial sums when a
// producer kernel fused stage 1), dX = dZ W with the lower layer's act'
// fused into the epilogue.
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.h"
#include "gemm.h"

namespace sg {
int ctx_activate(sg_ctx* ctx);
int ctx_compute_sms(sg_ctx* ctx);
int colsum_partials(const void* x, int dtype, long long ld, long long M, long long N, float* part, long long ldp,
                    cudaStream_t st);
}  // namespace sg

using namespace sg;

namespace {

int act_dtype(int precision) {
  switch (precision) {
    case SG_PREC_BF16: return SG_BF16;
    case SG_PREC_TF32:
    case SG_PREC_STRICT_FP32: return SG_F32;
    case SG_PREC_STRICT_FP64: return SG_F64;
    default: return -1;
  }
}

bool tensor_core(int precision) { return precision == SG_PREC_BF16 || precision == SG_PREC_TF32; }

int check_desc(const sg_dense_desc* d) {
  if (!d || !d->X || !d->W) return fail(SG_EINVAL, "dense: null X or W");
  if (d->batch < 0 || d->fan_in <= 0 || d->fan_out <= 0) return fail(SG_EINVAL, "dense: bad extents");
  if (act_dtype(d->precision) < 0) return fail(SG_EINVAL, "dense: unknown precision");
  if (d->act < SG_ACT_IDENTITY || d->act > SG_ACT_RELU) return fail(SG_EINVAL, "dense: bad activation");
  if (d->ldx < d->fan_in || d->ldw < d->fan_in) return fail(SG_EINVAL, "dense: leading dimension below fan_in");
  return SG_OK;
}

}  // namespace

extern "C" {

int sg_dense_forward(sg_ctx* ctx, const sg_dense_desc* d, void* H, int64_t ldh, void* H_f32, int64_t ld_hf, void* Z,
                     int64_t ldz, void* stream) {
  SG_NVTX("sg_dense_forward");
  if (!ctx) return fail(SG_EINVAL, "null argument");
  if (int rc = check_desc(d)) return rc;
  if (d->batch == 0) return SG_OK;
  const bool bf16 = d->precision == SG_PREC_BF16;
  if (H_f32 && !bf16) return fail(SG_EINVAL, "dense: H_f32 is a BF16-precision output");
  sg_gemm_desc g{};
  g.M = d->batch;
  g.N = d->fan_out;
  g.K = d->fan_in;
  g.A = d->X;
  g.lda = d->ldx;
  g.B = d->W;
  g.ldb = d->ldw;
  g.precision = d->precision;
  g.epilogue = SG_EPI_BIAS_ACT;
  g.act = d->act;
  g.bias = d->b;
  g.out_pre = Z;
  g.ld_pre = ldz;
  if (bf16) {
    g.out_lp = H;
    g.ld_lp = ldh;
    g.out = H_f32;
    g.ld_out = ld_hf;
  } else {
    g.out = H;
    g.ld_out = ldh;
  }
  return sg_gemm(ctx, &g, stream);
}

int sg_dense_backward(sg_ctx* ctx, const sg_dense_desc* d, const sg_dense_grad* gr, void* stream) {
  SG_NVTX("sg_dense_backward");
  if (!ctx || !gr) return fail(SG_EINVAL, "null argument");
  if (int rc = check_desc(d)) return rc;
  if (!gr->dZ || !gr->dW || !gr->db) return fail(SG_EINVAL, "dense: dZ, dW and db are required");
  if (gr->act_prev < SG_ACT_IDENTITY || gr->act_prev > SG_ACT_RELU) return fail(SG_EINVAL, "dense: bad act_prev");
  const int adt = act_dtype(d->precision);
  const bool tc = tensor_core(d->precision);
  if (!tc && (gr->colsum_in || gr->colsum_out))
    return fail(SG_EINVAL, "dense: partial column sums are a tensor-core-precision feature");
  if (gr->dX && d->precision == SG_PREC_BF16 && gr->dx_dtype != SG_BF16 && gr->dx_dtype != SG_F32)
    return fail(SG_EINVAL, "dense: BF16 dX must be bf16 or f32");
  if (gr->dX && d->precision != SG_PREC_BF16 && gr->dx_dtype != adt)
    return fail(SG_EINVAL, "dense: dX dtype must be the activation dtype");
  if (d->batch == 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;

  // dW = dZ^T . X   (rules.py:113-115 second cotangent, then _transpose :123-124)
  sg_gemm_desc g{};
  g.M = d->fan_out;
  g.N = d->fan_in;
  g.K = d->batch;
  g.A = gr->dZ;
  g.lda = gr->ld_dz;
  g.a_mn_major = 1;
  g.B = d->X;
  g.ldb = d->ldx;
  g.b_mn_major = 1;
  g.precision = d->precision;
  g.epilogue = SG_EPI_STORE;
  g.out = gr->dW;
  g.ld_out = gr->ld_dw;
  // db = reduce_like(dZ, (fan_out,))   (rules.py:45-46)
  const long long G = (d->batch + 31) / 32;
  // db finalised as the dW GEMM's tail job (SGB200_DENSE_FUSED_DB=1): one
  // launch fewer per layer but measured slower (c5 step +0.1..0.15 ms: the
  // tail runs after every CTA's tiles); default: its own full-width launch.
  static const bool fused_db = [] {
    const char* e = std::getenv("SGB200_DENSE_FUSED_DB");
    return e && e[0] == '1';
  }();
  if (tc && gr->colsum_in && fused_db) {
    // the dW GEMM finalises db from the producer-fused partial sums as its
    // tail job (one launch for dW and db; k_colsum_finalize's arithmetic)
    if (d->fan_in <= 0 || g.K <= 0) return fail(SG_EINVAL, "dense: empty dW");
    GemmArgs ga{};
    gemm_args_from_desc(ctx, &g, ga);
    ga.fin.part = gr->colsum_in;
    ga.fin.G = G;
    ga.fin.ld = gr->ld_colsum_in;
    ga.fin.N = d->fan_out;
    ga.fin.out = (float*)gr->db;
    if ((rc = launch_gemm_tc(ga, d->precision == SG_PREC_TF32, ctx_compute_sms(ctx), st))) return rc;
  } else if ((rc = sg_gemm(ctx, &g, stream))) {
    return rc;
  }
  if (!tc) {
    if ((rc = sg_colsum_strict(ctx, gr->dZ, adt, gr->ld_dz, d->batch, d->fan_out, gr->db, stream))) return rc;
  } else if (gr->colsum_in) {
    if (!fused_db &&
        (rc = sg_colsum_finalize(ctx, gr->colsum_in, G, gr->ld_colsum_in, d->fan_out, (float*)gr->db, stream)))
      return rc;
  } else {
    const long long ldp = (d->fan_out + 3) / 4 * 4;
    float* part = nullptr;
    SG_CUDA_TRY(cudaMallocAsync((void**)&part, (size_t)G * ldp * sizeof(float), st));
    rc = colsum_partials(gr->dZ, adt, gr->ld_dz, d->batch, d->fan_out, part, ldp, st);
    if (!rc) rc = sg_colsum_finalize(ctx, part, G, ldp, d->fan_out, (float*)gr->db, stream);
    SG_CUDA_TRY(cudaFreeAsync(part, st));
    if (rc) return rc;
  }

  // dX = dZ . W  [.* act_prev'(X)]   (rules.py:113-115 first cotangent, :82-94)
  if (gr->dX) {
    sg_gemm_desc x{};
    x.M = d->batch;
    x.N = d->fan_in;
    x.K = d->fan_out;
    x.A = gr->dZ;
    x.lda = gr->ld_dz;
    x.B = d->W;
    x.ldb = d->ldw;
    x.b_mn_major = 1;
    x.precision = d->precision;
    x.epilogue = gr->act_prev == SG_ACT_IDENTITY ? SG_EPI_STORE : SG_EPI_ACT_GRAD;
    x.act = gr->act_prev;
    x.aux = d->X;
    x.ld_aux = d->ldx;
    if (d->precision == SG_PREC_BF16 && gr->dx_dtype == SG_BF16) {
      x.out_lp = gr->dX;
      x.ld_lp = gr->ld_dx;
    } else {
      x.out = gr->dX;
      x.ld_out = gr->ld_dx;
    }
    x.colsum = gr->colsum_out;
    x.ld_colsum = gr->ld_colsum_out;
    if ((rc = sg_gemm(ctx, &x, stream))) return rc;
  }
  return SG_OK;
}

}  // extern "C"
