// Dense-layer GEMM interfaces shared by the tensor-core and strict kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/sgb200.h"

namespace sg {

// Epilogue of one GEMM tile row (see include/sgb200.h for the modes).
struct GemmEpilogue {
  int mode;                    // SG_EPI_STORE / SG_EPI_BIAS_ACT / SG_EPI_ACT_GRAD
  int act;                     // SG_ACT_*
  const float* bias;           // [N]                                (BIAS_ACT)
  const __nv_bfloat16* aux;    // saved activation h [M][ld_aux]     (ACT_GRAD, BF16 precision)
  const float* aux_f32;        // same, fp32                         (ACT_GRAD, TF32 precision)
  long long ld_aux;
  float* out_pre;              // optional fp32 z+b before activation (BIAS_ACT)
  long long ld_pre;
  float* out_f32;              // optional fp32 result
  long long ld_f32;
  __nv_bfloat16* out_bf16;     // optional bf16 result
  long long ld_bf16;
  float* colsum;               // optional column sums of the result per 32-row group:
  long long ld_colsum;         //   colsum[(m / 32)][n], [ceil(M/32)][ld_colsum]
  unsigned* dom = nullptr;     // domain flags (SG_DOM_*): sigmoid pre-activations that overflow the reference
  const float* seed = nullptr; // BIAS_ACT_SEED: cotangent of the activation, fp32 [M][ld_seed]
  long long ld_seed = 0;
  __nv_bfloat16* out2_bf16 = nullptr;  // BIAS_ACT_SEED: seed .* act'(h); BIAS_MSE: dz; bf16 [M][ld_out2]
  float* out2_f32 = nullptr;           // BIAS_ACT_SEED in TF32: seed .* act'(h), fp32 [M][ld_out2]
  long long ld_out2 = 0;
  double* loss_part = nullptr;          // BIAS_MSE: [ceil(M/32)][ceil(N/32)] partial losses
  float loss_scale = 0.0f;
};

// Column sums of a 32x32 block held one row per lane (v[i] = column i):
// a 31-shuffle transpose-reduce leaves column L's sum in lane L, summed in a
// fixed order (deterministic).  v is destroyed.
// (the adds in packed fp32x2 pairs -- FADD2, the same roundings -- unless
// SG_EPI_SCALAR_MATH)
__device__ __forceinline__ void warp_colsum_store(float (&v)[32], float* dst, int lane, int n) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#if !defined(SG_EPI_SCALAR_MATH) || !SG_EPI_SCALAR_MATH
    if (s >= 2) {
#pragma unroll
      for (int i = 0; i < s; i += 2) {
        const float r0 = __shfl_xor_sync(0xffffffffu, upper ? v[i] : v[i + s], s);
        const float r1 = __shfl_xor_sync(0xffffffffu, upper ? v[i + 1] : v[i + 1 + s], s);
        const float2 k = make_float2(upper ? v[i + s] : v[i], upper ? v[i + 1 + s] : v[i + 1]);
        const float2 r = __fadd2_rn(k, make_float2(r0, r1));
        v[i] = r.x, v[i + 1] = r.y;
      }
      continue;
    }
#endif
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  if (lane < n) dst[lane] = v[0];
}

// Optional bias-gradient finalize a GEMM runs as its tail job:
// out[j] = sum_g part[g][j], g < G, j < N (k_colsum_finalize's arithmetic).
struct FinalizeJob {
  const float* part = nullptr;
  long long G = 0, ld = 0, N = 0;
  float* out = nullptr;
};

struct GemmArgs {
  int M, N, K;
  const void* A;  // bf16, or fp32 with tf32 (operands read as TF32 by the tensor cores)
  long long lda;
  bool a_mn;  // A stored [K][M] (MN-major) instead of [M][K]
  const void* B;
  long long ldb;
  bool b_mn;  // B stored [K][N] instead of [N][K]
  GemmEpilogue epi;
  int batch = 1;             // independent GEMMs (bmm lanes)
  long long sa = 0, sb = 0;  // operand batch strides (elements)
  long long so_f32 = 0, so_lp = 0;  // output batch strides (elements)
  FinalizeJob fin;            // run after the tiles (CTA-pair kernels) or as its own launch
  float* split_part = nullptr;  // deferred split-K: partials land here, the caller reduces them
  long long split_part_elems = 0;
};

int launch_gemm_tc(const GemmArgs& g, bool tf32, int num_sms, cudaStream_t st);
void plan_gemm_splits(const GemmArgs& g, bool tf32, int num_sms, int* splits, long long* ld_part);
int splitk_reduce_multi(int n, const float* const* parts, const int32_t* S, const int64_t* M, const int64_t* N,
                        const int64_t* ld_part, float* const* outs, const int64_t* ld_out, cudaStream_t st);
// sg_gemm_desc -> GemmArgs of the tensor-core kernels (validated by sg_gemm)
void gemm_args_from_desc(sg_ctx* ctx, const sg_gemm_desc* d, GemmArgs& g);
int colsum_finalize_launch(const float* part, long long G, long long ld, long long N, float* out, int num_sms,
                           cudaStream_t st);

namespace strict {
struct StrictArgs {
  int M, N, K;
  const void* A;
  long long lda;
  bool a_mn;
  const void* B;
  long long ldb;
  bool b_mn;
  int mode, act;
  unsigned* dom;
  const void* bias;
  const void* aux;
  long long ld_aux;
  void* out_pre;
  long long ld_pre;
  void* out;
  long long ld_out;
  int batch = 1;  // blockIdx.z: independent GEMMs with these element strides
  long long sa = 0, sb = 0, so = 0;
};
}  // namespace strict
int launch_gemm_strict(const strict::StrictArgs& g, bool f64, cudaStream_t st);

// ----------------------------------------------------- epilogue row helpers
// One thread owns one output row segment of up to 32 consecutive columns.
__device__ __forceinline__ void store_row_f32(float* dst, const float (&v)[32], int n) {
  if (n == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < n) dst[i] = v[i];
  }
}

__device__ __forceinline__ void store_row_bf16(__nv_bfloat16* dst, const float (&v)[32], int n) {
  if (n == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
#pragma unroll
    for (int i = 0; i < 16; i += 4)
      *reinterpret_cast<uint4*>(dst + 2 * i) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < n) dst[i] = __float2bfloat16_rn(v[i]);
  }
}

__device__ __forceinline__ void load_row_f32(const float* src, float (&v)[32], int n) {
  if (n == 32 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(src + i));
      v[i] = f.x, v[i + 1] = f.y, v[i + 2] = f.z, v[i + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i < n ? __ldg(src + i) : 0.0f;
  }
}
__device__ __forceinline__ void load_row_bf16(const __nv_bfloat16* src, float (&v)[32], int n) {
  if (n == 32 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint4 w = __ldg(reinterpret_cast<const uint4*>(src + i));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        v[i + 2 * j] = f.x;
        v[i + 2 * j + 1] = f.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i < n ? __bfloat162float(src[i]) : 0.0f;
  }
}

}  // namespace sg
