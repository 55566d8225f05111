// K9: strict-order GEMM on CUDA cores (STRICT_FP32 / STRICT_FP64 precision).
//
// Every output is the reference's fold (tensor.py:351-361):
//   C[i,j] = ((a_i0*b_0j) + a_i1*b_1j) + ... ascending in k,
// each product and each sum rounded separately (__fmul_rn/__fadd_rn, so no
// FMA contraction).  In fp64 this is bit-identical to the unmodified
// reference; in fp32 to the fp32 restatement in oracle/csrc/strict_gemm.c.
// Tiling only changes *when* a term is added, never the order per output.
#include <cuda_runtime.h>

#include "common.h"
#include "gemm.h"

namespace sg {
namespace strict {

constexpr int TM = 64, TN = 64, TK = 16;

template <class T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <class T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

template <class T>
__device__ __forceinline__ T act_fwd(T z, int act) {
  switch (act) {
    case SG_ACT_SIGMOID: return (T)1 / ((T)1 + exp(-z));  // tensor.py:214-215
    case SG_ACT_TANH: return tanh(z);
    case SG_ACT_RELU: return z > (T)0 ? z : (T)0;
    default: return z;
  }
}
template <class T>
__device__ __forceinline__ T act_grad(T h, int act) {  // rules.py:82-94 operation order
  switch (act) {
    case SG_ACT_SIGMOID: return mul_rn(h, add_rn((T)1, -h));
    case SG_ACT_TANH: return add_rn((T)1, -mul_rn(h, h));
    case SG_ACT_RELU: return h > (T)0 ? (T)1 : (T)0;
    default: return (T)1;
  }
}

template <class T>
__global__ void __launch_bounds__(256) strict_gemm_kernel(const StrictArgs g) {
  __shared__ T As[TK][TM + 1];
  __shared__ T Bs[TK][TN + 1];
  const long long bz = blockIdx.z;  // batch entry (bmm lane, tensor.py:364-369)
  const T* A = reinterpret_cast<const T*>(g.A) + bz * g.sa;
  const T* B = reinterpret_cast<const T*>(g.B) + bz * g.sb;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tid = threadIdx.x;
  const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = (T)-0.0;  // -0 + p == p exactly: fold starts at the first product
  for (int k0 = 0; k0 < g.K; k0 += TK) {
    for (int e = tid; e < TK * TM; e += 256) {
      const int kk = g.a_mn ? e / TM : e % TK, mm = g.a_mn ? e % TM : e / TK;
      const int m = m0 + mm, k = k0 + kk;
      T v = (T)0;
      if (m < g.M && k < g.K) v = g.a_mn ? A[(long long)k * g.lda + m] : A[(long long)m * g.lda + k];
      As[kk][mm] = v;
    }
    for (int e = tid; e < TK * TN; e += 256) {
      const int kk = g.b_mn ? e / TN : e % TK, nn = g.b_mn ? e % TN : e / TK;
      const int n = n0 + nn, k = k0 + kk;
      T v = (T)0;
      if (n < g.N && k < g.K) v = g.b_mn ? B[(long long)k * g.ldb + n] : B[(long long)n * g.ldb + k];
      Bs[kk][nn] = v;
    }
    __syncthreads();
    const int kmax = min(TK, g.K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tm + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = add_rn(acc[i][j], mul_rn(a[i], b[j]));
    }
    __syncthreads();
  }
  T* out = g.out ? reinterpret_cast<T*>(g.out) + bz * g.so : nullptr;
  const T* bias = reinterpret_cast<const T*>(g.bias);
  const T* aux = reinterpret_cast<const T*>(g.aux);
  T* pre = reinterpret_cast<T*>(g.out_pre);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + tm + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tn + j;
      if (n >= g.N) continue;
      T v = acc[i][j];
      if (g.K == 0) v = (T)0;
      if (g.mode == SG_EPI_BIAS_ACT) {
        if (bias) v = add_rn(v, bias[n]);  // add(z, b): tensor.py:179-182
        if (pre) pre[(long long)m * g.ld_pre + n] = v;
        // scalar_sigmoid's math.exp(-z) raises OverflowError (tensor.py:214-215)
        if (g.act == SG_ACT_SIGMOID && (double)v < -EXP_MAX_ARG && g.dom)
          atomicOr(g.dom, (unsigned)SG_DOM_EXP_OVERFLOW);
        v = act_fwd(v, g.act);
      } else if (g.mode == SG_EPI_ACT_GRAD) {
        v = mul_rn(v, act_grad(aux[(long long)m * g.ld_aux + n], g.act));
      }
      if (out) out[(long long)m * g.ld_out + n] = v;
    }
  }
}

}  // namespace strict

int launch_gemm_strict(const strict::StrictArgs& g, bool f64, cudaStream_t st) {
  dim3 grid((g.N + strict::TN - 1) / strict::TN, (g.M + strict::TM - 1) / strict::TM, g.batch);
  if (grid.y > 65535 || g.batch > 65535 || g.batch < 1) return fail(SG_EINVAL, "strict GEMM: M or batch too large");
  if (g.batch > 1 && (g.out_pre || g.mode == SG_EPI_ACT_GRAD))
    return fail(SG_EINVAL, "strict GEMM: batched GEMMs take the STORE / BIAS_ACT epilogues without out_pre");
  if (f64)
    strict::strict_gemm_kernel<double><<<grid, 256, 0, st>>>(g);
  else
    strict::strict_gemm_kernel<float><<<grid, 256, 0, st>>>(g);
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

}  // namespace sg
