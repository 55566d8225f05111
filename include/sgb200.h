/* sgb200 — C ABI of the B200 hot path for the ssagrad reference
 * (arXiv 1811.01457 "Flux" reproduction, /root/reference/pkg/src/ssagrad).
 *
 * Every entry point takes plain pointers and sizes; no torch types cross
 * this boundary.  Device pointers are CUDA device addresses, `stream` is a
 * cudaStream_t (CUstream) or NULL for the legacy default stream.  The
 * caller owns and allocates every input and output buffer; the library
 * never frees caller memory (reference DenseTensor values are immutable
 * and every op returns a fresh tensor, SPEC.md:195 / tensor.py:29-47).
 *
 * Status codes (mirroring the reference's Python exceptions):
 *   SG_OK            0
 *   SG_EDOMAIN       1  DomainError / EvalError   (tensor.py:25-26, interp.py:26-35)
 *   SG_EINVAL        2  ValueError (shapes, arguments)    (tensor.py:118-119, 358-359)
 *   SG_ECUDA         3  CUDA / NVRTC failure
 *   SG_ENCCL         4  collective (NCCL) failure
 * sg_last_error() returns the message of the last failing call on this thread.
 */
#ifndef SGB200_H
#define SGB200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SG_API __attribute__((visibility("default")))
#else
#define SG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_EDOMAIN 1
#define SG_EINVAL 2
#define SG_ECUDA 3
#define SG_ENCCL 4

/* element types */
#define SG_F32 0
#define SG_F64 1
#define SG_BF16 2

#define SG_MAX_DIMS 8

/* A C-contiguous row-major tensor, or (ndim == 0) an f64 scalar by value.
 * Replaces the reference runtime value `DenseTensor | float`
 * (tensor.py:29-47; scalars are plain Python floats, interp.py:3-13). */
typedef struct sg_tensor {
  void* ptr;
  int32_t dtype;
  int32_t ndim;
  int64_t shape[SG_MAX_DIMS];
  double scalar;
} sg_tensor;

typedef struct sg_ctx sg_ctx;
typedef struct sg_kernel sg_kernel;

/* ---------------------------------------------------------------- context */
SG_API int sg_version(void);
SG_API int sg_create(int device, sg_ctx** out);
SG_API int sg_destroy(sg_ctx* ctx);
/* Copies the last error message of the calling thread into buf (NUL-terminated). */
SG_API int sg_last_error(char* buf, size_t n);

/* ------------------------------------------------------- fused broadcast
 * Replaces the per-element interpreter of `fused_map` / `fused_pack`
 * (interp.py:322-352, Machine.dispatch "fused_map"/"fused_pack" at
 * interp.py:264-267) and the public API `fused_map_with_partials` /
 * `fused_map_pullback` (forward_ad.py:194-235).
 *
 * sg_ew_compile registers the CUDA C++ lowering of one scalar IR function
 * (device functions `sg_entry_p` / `sg_entry_d` produced by the host-side
 * codegen) under `key`; variants for each broadcast pattern are JIT
 * compiled with NVRTC for sm_100a on first use and cached.  k = number of
 * sub-function arguments (<= 16), dtype = SG_F32 or SG_F64. */
SG_API int sg_ew_compile(sg_ctx* ctx, const char* user_src, const char* key, int k, int dtype,
                  sg_kernel** out);
/* y = f.(args...) with trailing-aligned broadcasting (tensor.py:108-121). */
SG_API int sg_ew_forward(sg_ctx* ctx, sg_kernel* kern, int k, const sg_tensor* args, sg_tensor* y,
                  void* stream);
/* argbars[i] = reduce_like(ybar .* d f/d arg_i, type(arg_i))  — the fused
 * adjoint (rules.py:177-185 + tensor.py:327-345).  y may be NULL (no primal
 * output) or receive the primal.  For an f64-scalar arg (ndim 0) the
 * cotangent is written as one element of argbars[i].ptr (dtype of y).  */
SG_API int sg_ew_grad(sg_ctx* ctx, sg_kernel* kern, int k, const sg_tensor* args, const sg_tensor* ybar,
               sg_tensor* y, sg_tensor* argbars, void* stream);
/* pack = [primal, d f/d arg_0, ...], shape (1+k, *out_shape): `fused_pack`. */
SG_API int sg_ew_pack(sg_ctx* ctx, sg_kernel* kern, int k, const sg_tensor* args, sg_tensor* pack,
               void* stream);
/* Synchronises `stream`, reads and clears the context's device error word.
 * Returns SG_EDOMAIN and fills (*element, *site) when an element failed
 * (lowest flat element index wins); SG_OK otherwise. */
SG_API int sg_ew_check(sg_ctx* ctx, void* stream, int64_t* element, int32_t* site);
/* Per-element step budget for sub-functions with loops (interp.py:23,113-122). */
SG_API int sg_ew_set_step_limit(sg_ctx* ctx, int64_t limit);
/* NVRTC-compiles one variant without touching a GPU (build checks on CPU
 * hosts): kinds[i] in {0 full, 1 row, 2 col, 3 one-element, 4 by-value}. */
SG_API int sg_ew_compile_only(const char* user_src, int k, int dtype, const int* kinds, int vec, int bdx,
                              int bdy, size_t* cubin_bytes);
/* Number of NVRTC variants compiled so far (introspection / tests). */
SG_API int sg_ew_variant_count(sg_kernel* kern);

/* ------------------------------------------------------------ Dense GEMM
 * D[M,N] = sum_k A[m,k] B[n,k] with a fused epilogue: the Dense layer's
 * `matmul(h, transpose(W))` + `add` + activation (nn_train.py:189-210,
 * tensor.py:351-361) and its adjoints (rules.py:45-46, 82-94, 113-115, 123-124).
 * A is [M][lda] (K-major) or, with a_mn_major, [K][lda] (MN-major); same for
 * B with N.  So X.W^T, dZ.W and dZ^T.X all run without transposes.
 *
 * precision:
 *   SG_PREC_BF16         A,B bf16 -> tcgen05 tensor cores (TMA + TMEM), fp32
 *                        accumulate; lda/ldb multiples of 8, 16-byte aligned.
 *   SG_PREC_STRICT_FP32  A,B f32 -> CUDA cores, ascending-k fold with every
 *                        product and sum rounded (no FMA): bit-exact with the
 *                        reference kernel's order restated in fp32.
 *   SG_PREC_STRICT_FP64  same in f64: bit-exact with the unmodified reference.
 *   SG_PREC_TF32         A,B f32 -> tcgen05 kind::tf32 (operands rounded to
 *                        TF32 by the tensor cores, fp32 accumulate); lda/ldb
 *                        multiples of 4, 16-byte aligned; aux is f32.
 * epilogue (per output element, v = the dot product):
 *   SG_EPI_STORE     out = v
 *   SG_EPI_BIAS_ACT  out_pre = v + bias[n];  out = act(v + bias[n])
 *   SG_EPI_ACT_GRAD  out = v * act'(aux[m][n])   (act' from the saved output h:
 *                    sigmoid h(1-h), tanh 1-h^2, relu [h>0]; rules.py:82-94)
 * Outputs: `out` (f32; f64 for STRICT_FP64), optional `out_lp` bf16 copy
 * (BF16 precision only), optional `out_pre`.  Null pointers are skipped. */
#define SG_PREC_BF16 0
#define SG_PREC_STRICT_FP32 1
#define SG_PREC_STRICT_FP64 2
#define SG_PREC_TF32 3

#define SG_EPI_STORE 0
#define SG_EPI_BIAS_ACT 1
#define SG_EPI_ACT_GRAD 2
/* BIAS_ACT with a known cotangent of the activation (a value-and-pullback
 * call, reverse_ad.py:633-663 `grad` with seeds): out_lp = act(z + b) (bf16,
 * the saved activation) and, in the same epilogue, out2_lp = seed .* act'(h)
 * with h that bf16 activation (rules.py:82-94), column sums of it into colsum;
 * seed is fp32 [M][ld_seed] passed in `aux`/`ld_aux`.  BF16 precision, no
 * fp32 `out`; replaces a separate act' pass over the seed. */
#define SG_EPI_BIAS_ACT_SEED 3
/* The MSE loss of a linear top layer in its own epilogue (training step,
 * loss = scale * sum (z - y)^2, z = x W^T + b): reads the
 * targets y (fp32, in `aux`/`ld_aux`), writes dz = 2 (z - y) scale as bf16 to
 * out2_lp (+ its column sums into colsum) and per-(32-row group, 32-column
 * chunk) partial losses to loss_part[group * ceil(N/32) + chunk] (f64, summed
 * in a fixed order by sg_sum_f64); z itself is written only if `out` is given.
 * BF16 precision, identity activation; `colsum` ld = ld_colsum. */
#define SG_EPI_BIAS_MSE 4

#define SG_ACT_IDENTITY 0
#define SG_ACT_SIGMOID 1
#define SG_ACT_TANH 2
#define SG_ACT_RELU 3

typedef struct sg_gemm_desc {
  int64_t M, N, K;
  const void* A;
  int64_t lda;
  int32_t a_mn_major;
  const void* B;
  int64_t ldb;
  int32_t b_mn_major;
  int32_t precision;
  int32_t epilogue;
  int32_t act;
  const void* bias;
  const void* aux;
  int64_t ld_aux;
  void* out_pre;
  int64_t ld_pre;
  void* out;
  int64_t ld_out;
  void* out_lp;
  int64_t ld_lp;
  /* optional fp32 column sums of the result per 32-row group, [ceil(M/32)][ld_colsum]
   * (BF16 precision): the bias gradient's first reduction stage, see sg_colsum_finalize */
  float* colsum;
  int64_t ld_colsum;
  /* batched GEMM (the reference's bmm, tensor.py:364-369, one per lane):
   * batch >= 1 independent problems, operands/outputs `stride_*` elements
   * apart (out_lp uses stride_lp).  batch 0 is treated as 1.  Batched calls
   * take the STORE / BIAS_ACT epilogues (bias shared) without colsum/out_pre. */
  int64_t batch;
  int64_t stride_a, stride_b, stride_out, stride_lp;
  void* out2_lp; /* BIAS_ACT_SEED: [M][ld_out2] seed .* act'(h) -- bf16 (h in out_lp) for BF16,
                  * fp32 (h in out) for TF32; BIAS_MSE: dz (bf16) */
  int64_t ld_out2;
  double* loss_part; /* BIAS_MSE: [ceil(M/32)][ceil(N/32)] partial losses */
  double loss_scale; /* BIAS_MSE: scale (1 / global batch) */
  /* deferred split-K (optional): when the launcher splits K (a STORE GEMM whose
   * output tiles cannot fill the GPU, e.g. dW of a narrow layer), the fp32
   * partials [splits][M][ld] (see sg_gemm_splits) are written here and NOT
   * reduced: the caller reduces them later with sg_splitk_reduce_multi (several
   * GEMMs in one launch).  Ignored when the GEMM does not split. */
  float* split_part;
  int64_t split_part_elems; /* capacity of split_part in floats */
} sg_gemm_desc;

SG_API int sg_gemm(sg_ctx* ctx, const sg_gemm_desc* desc, void* stream);
/* The split-K factor sg_gemm picks for desc (1: no split) and the partials'
 * row pitch ld (floats): a deferred split needs splits * M * ld floats. */
SG_API int sg_gemm_splits(sg_ctx* ctx, const sg_gemm_desc* desc, int32_t* splits, int64_t* ld_part);
/* out_i[m][n] = sum_s part_i[s][m][n], s ascending (sg_gemm's own split-K
 * reduce, bit-identical) for n deferred split-K GEMMs in one launch. */
SG_API int sg_splitk_reduce_multi(sg_ctx* ctx, int32_t n, const float* const* parts, const int32_t* splits,
                                  const int64_t* M, const int64_t* N, const int64_t* ld_part, float* const* outs,
                                  const int64_t* ld_out, void* stream);

/* ------------------------------------------------ Dense step, memory-bound
 * dz = ybar .* act'(h)  (rules.py:82-94 with the saved output h, reference
 * operation order), optionally a second copy dz2 in another dtype and the
 * per-32-row column sums (bias-gradient stage 1).  dtypes: SG_F32/F64/BF16. */
SG_API int sg_act_grad(sg_ctx* ctx, const void* ybar, int32_t ybar_dtype, int64_t ld_y, const void* h,
                       int32_t h_dtype, int64_t ld_h, int64_t M, int64_t N, int32_t act, void* dz,
                       int32_t dz_dtype, int64_t ld_dz, void* dz2, int32_t dz2_dtype, int64_t ld_dz2,
                       float* colsum, int64_t ld_colsum, void* stream);
/* out[n] = sum_g part[g][n] (fixed order, fp64 accumulation): bias-gradient stage 2. */
SG_API int sg_colsum_finalize(sg_ctx* ctx, const float* part, int64_t G, int64_t ld_part, int64_t N, float* out,
                              void* stream);
/* The same for n bias gradients in one launch (parts[i] [G[i]][ld_part[i]] -> outs[i][N[i]]). */
SG_API int sg_colsum_finalize_multi(sg_ctx* ctx, int32_t n, const float* const* parts, const int64_t* G,
                                    const int64_t* ld_part, const int64_t* N, float* const* outs, void* stream);
/* reduce_to((M,N) -> (N,)) in the reference's exact order (sequential ascending
 * row fold, tensor.py:287-292, 337-338), f32/f64: STRICT precision bias gradients. */
SG_API int sg_colsum_strict(sg_ctx* ctx, const void* x, int32_t dtype, int64_t ld, int64_t M, int64_t N,
                            void* out, void* stream);

#define SG_LOSS_SOFTMAX_XENT 0
#define SG_LOSS_MSE 1
#define SG_LOSS_BCE 2
/* Fused loss forward + gradient over logits z [M][N] and targets y:
 *   SOFTMAX_XENT: loss = -scale * sum y log softmax(z);  dz = (p * rowsum(y) - y) * scale
 *                 (the c1 loss IR: exp / reduce_sum(axis=1) / div / log / mul, scale = 1/n)
 *   MSE:          loss = scale * sum (z - y)^2;           dz = 2 (z - y) * scale
 *   BCE:          one-logit head + clamped mean BCE (nn_train.py:209-227):
 *                 p = sigmoid(z) clamped to [1e-7, 1-1e-7];
 *                 loss = -scale * sum y log p + (1-y) log(1-p);  dz = 0 where clamped
 * `loss` (device f64) receives the total; loss_part is scratch of n_part doubles
 * (>= ceil(N/32)*ceil(M/32) for MSE and BCE; ceil(M/32) for softmax).  Under data
 * parallelism scale = 1/global_batch so shard gradients sum to the full one. */
SG_API int sg_loss(sg_ctx* ctx, int32_t kind, const void* z, int32_t dtype, int64_t ld_z, const void* y,
                   int64_t ld_y, int64_t M, int64_t N, double scale, double* loss, double* loss_part,
                   int64_t n_part, void* dz, int32_t dz_dtype, int64_t ld_dz, void* dz2, int32_t dz2_dtype,
                   int64_t ld_dz2, float* colsum, int64_t ld_colsum, void* stream);
/* *out = sum of part[0..n) in a fixed order (f64): the partial losses of BIAS_MSE. */
SG_API int sg_sum_f64(sg_ctx* ctx, const double* part, int64_t n, double* out, void* stream);
/* params -= lr * grads over the flat parameter buffer (nn_train.py:365-372);
 * optional bf16 shadow copy of the updated parameters for the next GEMMs. */
SG_API int sg_sgd(sg_ctx* ctx, void* params, const void* grads, int32_t dtype, int64_t n, double lr,
                  void* shadow_bf16, void* stream);
SG_API int sg_cast(sg_ctx* ctx, const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t n,
                   void* stream);
/* 2-D cast / copy of a [rows][cols] block between row-strided buffers (the
 * minibatch load of a training step: fp32 host-layout rows -> the bf16
 * activation rows the first GEMM reads through TMA). */
SG_API int sg_cast_2d(sg_ctx* ctx, const void* src, int32_t src_dtype, int64_t ld_src, void* dst, int32_t dst_dtype,
                      int64_t ld_dst, int64_t rows, int64_t cols, void* stream);

/* ------------------------------------------------ persistent GEMM chains
 * A sequence of BF16 GEMMs (each an sg_gemm_desc: the Dense forward, dX and
 * dW products of nn_train.py:189-196 / rules.py:113-115 with their fused
 * epilogues) run by ONE persistent launch of CTA pairs.  A problem may depend
 * on earlier ones; its 256 x 256 output tiles then wait only for the rows
 * they read:
 *   SG_DEP_ROWS   A is K-major and is the earlier problem's output: a tile
 *                 waits for the producer's tiles of its 256-row block;
 *   SG_DEP_KROWS  A is MN-major over the earlier problem's output rows (dW =
 *                 dZ^T X): a K-split waits for the row blocks in its K range;
 *   SG_DEP_ALL    every tile of the earlier problem.
 * splits > 1 runs a STORE / fp32-output problem as K-splits finished inside
 * the kernel in ascending split order.  Results are bit-identical to issuing
 * the same sg_gemm calls one by one.  Buffers are bound at creation: a chain
 * is a plan (tensor maps, schedule, counters) replayed by sg_chain_run. */
#define SG_DEP_ROWS 1
#define SG_DEP_KROWS 2
#define SG_DEP_ALL 3
typedef struct sg_chain_problem {
  sg_gemm_desc gemm;
  int32_t splits;
  int32_t n_deps;       /* 0..2 */
  int32_t dep_kind[2];  /* SG_DEP_* */
  int32_t dep_on[2];    /* index of an earlier problem */
} sg_chain_problem;
typedef struct sg_chain sg_chain;
SG_API int sg_chain_create(sg_ctx* ctx, const sg_chain_problem* problems, int32_t n, sg_chain** out);
SG_API int sg_chain_run(sg_chain* chain, void* stream);
SG_API int sg_chain_info(const sg_chain* chain, int32_t* units, int32_t* ctas, double* est_us);
SG_API int sg_chain_destroy(sg_chain* chain);

/* ------------------------------------------------ Dense-path domain errors
 * The reference raises where its float64 ops are undefined: math.exp
 * overflow (an uncaught OverflowError from scalar_sigmoid / exp,
 * tensor.py:214-215, 245-250), division by zero (DomainError, tensor.py:
 * 197-205) and log of p <= 0 (DomainError, tensor.py:230-233), the latter two
 * wrapped into EvalError by run_blocks (interp.py:117-119).  The Dense-path
 * kernels compute numerically stable values (max-subtracted log-sum-exp) and,
 * beside them, evaluate the reference's conditions on the float64 widening of
 * the same values, OR-ing these bits into a per-context device word:
 *   sigmoid activation / BCE head:  z < -709.782712893384   -> EXP_OVERFLOW
 *   softmax cross-entropy:          z >  709.782712893384   -> EXP_OVERFLOW
 *                                   row sum of exp(z) == 0  -> DIV_ZERO
 *                                   exp(z_j) / sum == 0     -> LOG_NONPOS
 * sg_domain_check synchronises `stream`, returns the bits in *flags (and
 * clears them); SG_EDOMAIN when any is set. */
#define SG_DOM_EXP_OVERFLOW 1
#define SG_DOM_DIV_ZERO 2
#define SG_DOM_LOG_NONPOS 4
SG_API int sg_domain_check(sg_ctx* ctx, void* stream, int32_t* flags);

/* ------------------------------------------------ small-chain training step
 * The whole step of a small Dense chain -- forward (nn_train.py:189-210), loss
 * + seed, pullback (rules.py:45-46, 82-94, 113-124) and SGD (nn_train.py:
 * 365-372) -- in ONE cooperative launch, fp32 on the CUDA cores (c1: MLP
 * 784-32-10 at batch 128 is latency-bound: 13 MFLOP per step).  Parameters use
 * the flat [W0, b0, W1, b1, ...] layout of the Dense-chain engine: W_l at
 * P + w_off[l], rows of ldw[l] >= fan_in, b_l at P + b_off[l]; G (same layout)
 * receives the gradients, P is updated in place, and the optional bf16 shadow
 * S mirrors the new P.  Losses: SG_LOSS_SOFTMAX_XENT, SG_LOSS_MSE (as sg_loss);
 * `loss` (device f64) receives the total.  Limits: 1..4 layers, widths <= 1024,
 * batch <= 512, batch x width working sets that fit in shared memory.
 * `scratch` (device, >= sg_mlp_small_scratch_bytes) must be zeroed once
 * before the first step (it holds the grid barrier). */
#define SG_MLP_SMALL_MAXL 4
typedef struct sg_mlp_small_desc {
  int32_t L;                          /* layers */
  int32_t sizes[SG_MLP_SMALL_MAXL + 1];
  int32_t act[SG_MLP_SMALL_MAXL];     /* SG_ACT_* per layer */
  int64_t w_off[SG_MLP_SMALL_MAXL], b_off[SG_MLP_SMALL_MAXL], ldw[SG_MLP_SMALL_MAXL];
  int32_t loss;                       /* SG_LOSS_SOFTMAX_XENT or SG_LOSS_MSE */
  int32_t B;                          /* minibatch rows */
  double scale;                       /* loss scale (1/batch) */
  double lr;
} sg_mlp_small_desc;
SG_API int sg_mlp_small_scratch_bytes(const sg_mlp_small_desc* d, int64_t* bytes);
SG_API int sg_mlp_small_step(sg_ctx* ctx, const sg_mlp_small_desc* d, float* P, float* G, void* S_bf16,
                             const float* X, int64_t ldx, const float* Y, int64_t ldy, float* Z, int64_t ldz,
                             double* loss, void* scratch, int64_t scratch_bytes, void* stream);

/* ------------------------------------------------------ Dense layer
 * One Dense layer as the reference builds it (nn_train.py:189-210:
 * transpose(W) / matmul / add / activation) and its pullback (rules.py:45-46,
 * 82-94, 113-124), composed from the kernels above in one call each.
 * Operand dtype = the precision's activation dtype: bf16 (SG_PREC_BF16),
 * f32 (SG_PREC_TF32, SG_PREC_STRICT_FP32), f64 (SG_PREC_STRICT_FP64). */
typedef struct sg_dense_desc {
  int64_t batch, fan_in, fan_out;
  int32_t precision; /* SG_PREC_* */
  int32_t act;       /* SG_ACT_* of this layer */
  const void* X;     /* layer input [batch][ldx] */
  int64_t ldx;
  const void* W; /* [fan_out][ldw] (bf16 copy for BF16) */
  int64_t ldw;
  const void* b; /* [fan_out] f32 (f64 for STRICT_FP64) */
} sg_dense_desc;

/* H = act(X W^T + b) in the activation dtype (NULL to skip); H_f32: optional
 * f32 copy (BF16 only, e.g. the logits a loss reads); Z: optional
 * pre-activation z + b (f32 / f64). */
SG_API int sg_dense_forward(sg_ctx* ctx, const sg_dense_desc* d, void* H, int64_t ldh, void* H_f32, int64_t ld_hf,
                            void* Z, int64_t ldz, void* stream);

typedef struct sg_dense_grad {
  const void* dZ; /* dL/d(z + b) [batch][ld_dz], activation dtype (sg_act_grad / sg_loss make it) */
  int64_t ld_dz;
  const float* colsum_in; /* optional per-32-row partial column sums of dZ (BF16/TF32), else computed */
  int64_t ld_colsum_in;
  int32_t act_prev; /* SG_ACT_* of the layer below: dX = (dZ W) .* act_prev'(X) -- its dZ.
                       SG_ACT_IDENTITY: plain dX = dZ W */
  void* dX;         /* optional [batch][ld_dx] (NULL: first layer, dX not needed) */
  int64_t ld_dx;
  int32_t dx_dtype; /* SG_BF16 or SG_F32 for BF16; the activation dtype otherwise */
  float* colsum_out; /* optional partial column sums of dX (BF16/TF32); may alias colsum_in:
                        db is finalised before dX is computed */
  int64_t ld_colsum_out;
  void* dW; /* [fan_out][ld_dw] f32 (f64 for STRICT_FP64) */
  int64_t ld_dw;
  void* db; /* [fan_out] f32 (f64) */
} sg_dense_grad;

/* dW = dZ^T X, db = colsum(dZ), dX = dZ W [.* act_prev'(X)]; in that order. */
SG_API int sg_dense_backward(sg_ctx* ctx, const sg_dense_desc* d, const sg_dense_grad* g, void* stream);

/* ------------------------------------------- data parallelism (NCCL)
 * minibatch rows sharded over ranks (one process per GPU),
 * losses scaled by the global 1/B, and the flat gradient buffer (order
 * [W0, b0, W1, b1, ...], nn_train.py:99-103) all-reduced (SUM) in per-layer
 * buckets.  The communicator owns a comm stream: sg_dp_allreduce forks from
 * the caller's stream (event), reduces on the comm stream, and sg_dp_wait
 * joins it back -- stream-ordered and CUDA-graph capturable.  NCCL is
 * resolved at run time (dlopen libnccl.so.2); sg_dp_available() says
 * whether it was found.  The 128-byte unique id from rank 0's
 * sg_dp_unique_id reaches the other ranks over the host's rendezvous. */
typedef struct sg_dp sg_dp;
SG_API int sg_dp_available(void);
SG_API int sg_dp_unique_id(uint8_t* out, size_t n);
SG_API int sg_dp_init(sg_ctx* ctx, const uint8_t* unique_id, size_t n, int rank, int world, sg_dp** out);
SG_API int sg_dp_allreduce(sg_dp* dp, void* buf, int64_t n, int32_t dtype, void* stream);
SG_API int sg_dp_wait(sg_dp* dp, void* stream);
SG_API int sg_dp_finalize(sg_dp* dp);

/* out = reduce_to(a .* b, out_shape); b may be NULL.  The contraction of
 * `fused_map_pullback` (forward_ad.py:232-235) and `reduce_to`
 * (tensor.py:327-345) on the device; fp64 accumulation, fixed order. */
SG_API int sg_reduce_to(sg_ctx* ctx, const sg_tensor* a, const sg_tensor* b, sg_tensor* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SGB200_H */
