// Memory-bound kernels of the Dense training step (K6 bias-grad, K7 loss, K8 SGD).
//
// Reference: loss IR composed from exp/reduce_sum/div/log/mul (SURVEY §8(d)
// c1) or sub/mul/reduce_sum (MSE, c4/c5); bias gradient `reduce_like`
// column sums (rules.py:45-46, tensor.py:327-345); SGD `p - lr*g`
// (nn_train.py:365-372).  All reductions are deterministic (fixed order);
// fp64 accumulation for fp32 data.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>
#include <string>

#include "common.h"
#include "gemm.h"

// Programmatic dependent launch for the step's memory-bound kernels (launched
// through pdl_launch): wait until the previous grid in the stream completed
// (its writes visible) before touching memory; signal the next grid once this
// block's work is issued, so its launch and prologue overlap our tail.
#define SG_GRID_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define SG_GRID_TRIGGER() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

namespace sg {
template <class... KArgs, class... Args>
cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  // opt-in (SGB200_PDL=1): measured neutral to slightly slower on the
  // graph-replayed c4/c5 steps (the fused broadcast kernels keep theirs: +2.5 %)
  static const bool pdl = [] {
    const char* e = std::getenv("SGB200_PDL");
    return e && e[0] == '1';
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace sg

namespace sg {
namespace dk {

template <class T> __device__ __forceinline__ T ld_as(const void* p, int dtype, long long i);
template <> __device__ __forceinline__ float ld_as<float>(const void* p, int dtype, long long i) {
  if (dtype == SG_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  if (dtype == SG_F64) return (float)reinterpret_cast<const double*>(p)[i];
  return reinterpret_cast<const float*>(p)[i];
}
template <> __device__ __forceinline__ double ld_as<double>(const void* p, int dtype, long long i) {
  if (dtype == SG_BF16) return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  if (dtype == SG_F64) return reinterpret_cast<const double*>(p)[i];
  return (double)reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void st_as(void* p, int dtype, long long i, double v) {
  if (dtype == SG_BF16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn((float)v);
  else if (dtype == SG_F64) reinterpret_cast<double*>(p)[i] = v;
  else reinterpret_cast<float*>(p)[i] = (float)v;
}

template <class T>
__device__ __forceinline__ T act_grad_h(T h, int act) {  // rules.py:82-94, derivative from the output
  switch (act) {
    case SG_ACT_SIGMOID: return h * ((T)1 - h);
    case SG_ACT_TANH: return (T)1 - h * h;
    case SG_ACT_RELU: return h > (T)0 ? (T)1 : (T)0;
    default: return (T)1;
  }
}

// --- dZ = ybar .* act'(h); lane = column, warp walks 32 rows, column sums per 32-row group
template <class T>
__global__ void __launch_bounds__(256) k_act_grad(const void* ybar, int yd, long long ldy, const void* h, int hd,
                                                  long long ldh, long long M, long long N, int act, void* dz,
                                                  int dzd, long long lddz, void* dz2, int dz2d, long long lddz2,
                                                  float* colsum, long long ldc) {
  SG_GRID_WAIT();
  const long long c = blockIdx.x * 32ll + threadIdx.x;
  const long long g = blockIdx.y * 8ll + threadIdx.y;  // 32-row group
  const long long r0 = g * 32;
  if (r0 >= M) return;
  T acc = (T)0;
  if (c < N) {
    const long long r1 = r0 + 32 < M ? r0 + 32 : M;
    for (long long r = r0; r < r1; ++r) {
      const T yb = ld_as<T>(ybar, yd, r * ldy + c);
      const T hv = ld_as<T>(h, hd, r * ldh + c);
      const T v = yb * act_grad_h(hv, act);  // mul(ybar, act') (rules.py:87-89)
      st_as(dz, dzd, r * lddz + c, (double)v);
      if (dz2) st_as(dz2, dz2d, r * lddz2 + c, (double)v);
      acc += v;
    }
    if (colsum) colsum[g * ldc + c] = (float)acc;
  }
  SG_GRID_TRIGGER();
}

// --- vectorised fast paths (fp32 seed/logits, bf16 activations and dZ):
// thread = 8 consecutive columns, block = 2048 columns x one 32-row group;
// all global traffic is 16-byte loads/stores, column sums stay in registers.
struct V8 {
  float v[8];
};
__device__ __forceinline__ V8 ld8_f32(const float* p) {
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p));
  const float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
  return V8{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
}
__device__ __forceinline__ V8 ld8_bf16(const __nv_bfloat16* p) {
  const uint4 w = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
  V8 r;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __bfloat1622float2(h[j]);
    r.v[2 * j] = f.x;
    r.v[2 * j + 1] = f.y;
  }
  return r;
}
__device__ __forceinline__ void st8_bf16(__nv_bfloat16* p, const V8& x) {
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x.v[2 * j], x.v[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ void st8_f32(float* p, const V8& x) {
  reinterpret_cast<float4*>(p)[0] = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(x.v[4], x.v[5], x.v[6], x.v[7]);
}

__device__ __forceinline__ V8 ld8(const float* p) { return ld8_f32(p); }
__device__ __forceinline__ V8 ld8(const __nv_bfloat16* p) { return ld8_bf16(p); }
__device__ __forceinline__ void st8(float* p, const V8& v) { st8_f32(p, v); }
__device__ __forceinline__ void st8(__nv_bfloat16* p, const V8& v) { st8_bf16(p, v); }

// HT/DT: bf16 (BF16 tensor-core chain) or float (TF32 chain)
// Block (64, 4): 512 columns (8 per thread) x one 32-row group, each ty a
// quarter of the group's rows; the quarters' column sums are combined in
// shared memory in a fixed order (one partial row per group).  Four times
// the threads of a one-thread-per-32-rows layout: small batches still fill
// the machine.
__device__ __forceinline__ void quarter_colsum(float (&acc)[8], float* colsum, long long ldc, long long g,
                                               long long c, bool ok) {
  __shared__ float part[4][64][9];
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int j = 0; j < 8; ++j) part[ty][tx][j] = acc[j];
  __syncthreads();
  if (ty == 0 && ok && colsum) {
    V8 o;
#pragma unroll
    for (int j = 0; j < 8; ++j) o.v[j] = ((part[0][tx][j] + part[1][tx][j]) + part[2][tx][j]) + part[3][tx][j];
    st8_f32(colsum + g * ldc + c, o);
  }
}

// 8 rows per thread, all loads in flight (#pragma unroll 8: c3 48.5 us vs 51.5 with 4)
template <class HT, class DT>
__global__ void __launch_bounds__(256) k_act_grad_v8(const float* ybar, long long ldy, const HT* h,
                                                     long long ldh, long long M, long long N, int act,
                                                     DT* dz, long long lddz, float* colsum,
                                                     long long ldc) {
  SG_GRID_WAIT();
  const long long c = (blockIdx.x * 64ll + threadIdx.x) * 8;
  const bool ok = c < N;
  const long long g = blockIdx.y, r0 = g * 32 + threadIdx.y * 8;
  const long long r1 = r0 + 8 < M ? r0 + 8 : M;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (ok) {
#pragma unroll 8
    for (long long r = r0; r < r1; ++r) {
      const V8 yb = ld8_f32(ybar + r * ldy + c);
      const V8 hv = ld8(h + r * ldh + c);
      V8 o;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o.v[j] = yb.v[j] * act_grad_h(hv.v[j], act);
        acc[j] += o.v[j];
      }
      st8(dz + r * lddz + c, o);
    }
  }
  quarter_colsum(acc, colsum, ldc, g, c, ok);
  SG_GRID_TRIGGER();
}

template <class DT>
__global__ void __launch_bounds__(256) k_mse_v8(const float* z, long long ldz, const float* y, long long ldy,
                                                long long M, long long N, float scale, DT* dz,
                                                long long lddz, float* colsum, long long ldc, double* loss_part) {
  SG_GRID_WAIT();
  // block (64, 4) as k_act_grad_v8
  // Loss partials: one per 32 x 32 block, [row group][column block], with the
  // arithmetic of the fused BIAS_MSE GEMM epilogue (gemm_tc_dev.cuh epi_chunk):
  // per row, fp32 sums of 8 columns folded left to right, then the warp
  // butterfly's tree over the 32 rows -- so the separate loss kernel and the
  // fused one give bit-identical losses.
  __shared__ float rs[32][65];  // per-row sums of 8 columns [row in group][8-column group]
  const long long c = (blockIdx.x * 64ll + threadIdx.x) * 8;
  const bool ok = c < N;
  const long long g = blockIdx.y, r0 = g * 32 + threadIdx.y * 8;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
  for (int k = 0; k < 8; ++k) {
    const long long r = r0 + k;
    float l = 0.0f;
    if (ok && r < M) {
      const V8 zv = ld8_f32(z + r * ldz + c);
      const V8 yv = ld8_f32(y + r * ldy + c);
      V8 o;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = zv.v[j] - yv.v[j];
        l += d * d;
        o.v[j] = d * scale + d * scale;
        acc[j] += o.v[j];
      }
      st8(dz + r * lddz + c, o);
    }
    rs[threadIdx.y * 8 + k][threadIdx.x] = l;
  }
  quarter_colsum(acc, colsum, ldc, g, c, ok);
  __syncthreads();
  const int tid = threadIdx.y * 64 + threadIdx.x;
  const long long n0 = blockIdx.x * 512ll + tid * 32;
  if (tid < 16 && n0 < N) {
    float lr[32];
#pragma unroll
    for (int i = 0; i < 32; ++i)
      lr[i] = ((rs[i][4 * tid] + rs[i][4 * tid + 1]) + rs[i][4 * tid + 2]) + rs[i][4 * tid + 3];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < o; ++i) lr[i] = lr[i] + lr[i + o];
    loss_part[g * ((N + 31) / 32) + n0 / 32] = (double)lr[0] * (double)scale;
  }
  SG_GRID_TRIGGER();
}

// --- out[n] = sum_g part[g][n], fixed order, fp64 accumulation
// 8 columns (one 32-byte sector) x 32 row groups per block: many blocks even
// for narrow layers, each thread folds g = ty, ty+32, ... then a fixed fold over ty.
// Block = 32 columns x 32 threads; thread ty folds the 128 slices ty, ty+32,
// ty+64, ty+96 (slice s: row groups g = s, s+128, ..., ascending), then a
// fixed tree over the 128 slices -- the order of a 128-thread-per-column
// fold, with coalesced 128-byte rows and a quarter of the blocks of one.
__device__ __forceinline__ void colsum_finalize_block(const float* part, long long G, long long ldp, long long N,
                                                      float* out, long long j0) {
  constexpr int RG = 128;  // slices per column
  __shared__ double red[RG][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const long long j = j0 + tx;
#pragma unroll
  for (int i = 0; i < RG / 32; ++i) {
    double acc = 0.0;
    if (j < N) {
#pragma unroll 4
      for (long long g = ty + 32 * i; g < G; g += RG) acc += (double)part[g * ldp + j];
    }
    red[ty + 32 * i][tx] = acc;
  }
  __syncthreads();
  for (int s = RG / 2; s > 0; s >>= 1) {  // fixed-order tree over the slices
    for (int r = ty; r < s; r += 32) red[r][tx] += red[r + s][tx];
    __syncthreads();
  }
  if (ty == 0 && j < N) out[j] = (float)red[0][tx];
}
__global__ void __launch_bounds__(1024) k_colsum_finalize(const float* part, long long G, long long ldp, long long N,
                                                          float* out) {
  SG_GRID_WAIT();
  colsum_finalize_block(part, G, ldp, N, out, blockIdx.x * 32ll);
  SG_GRID_TRIGGER();
}

// The same finalize for several bias gradients in one launch (blockIdx.y =
// job): the chained backward pass finalises every layer's db at once.
constexpr int MAX_COLSUM_JOBS = 32;
struct ColsumJobs {
  const float* part[MAX_COLSUM_JOBS];
  float* out[MAX_COLSUM_JOBS];
  long long G[MAX_COLSUM_JOBS], ldp[MAX_COLSUM_JOBS], N[MAX_COLSUM_JOBS];
};
__global__ void __launch_bounds__(1024) k_colsum_finalize_multi(const __grid_constant__ ColsumJobs jobs) {
  SG_GRID_WAIT();
  const int b = blockIdx.y;
  if (blockIdx.x * 32ll < jobs.N[b])  // block-uniform
    colsum_finalize_block(jobs.part[b], jobs.G[b], jobs.ldp[b], jobs.N[b], jobs.out[b], blockIdx.x * 32ll);
  SG_GRID_TRIGGER();
}

// --- reduce_to over rows in the reference's order: sequential ascending fold
//     (tensor.py:287-292, 337-338) — STRICT precision bias gradients
template <class T>
__global__ void k_colsum_strict(const T* x, long long ld, long long M, long long N, T* out) {
  SG_GRID_WAIT();
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= N) return;
  T acc = x[j];
  for (long long r = 1; r < M; ++r) acc = acc + x[r * ld + j];
  out[j] = acc;
  SG_GRID_TRIGGER();
}

// --- per-32-row column sums of x (bias-gradient stage 1 when no producer fused it)
template <class T>
__global__ void __launch_bounds__(256) k_colsum_part(const T* x, long long ld, long long M, long long N, float* part,
                                                     long long ldp) {
  SG_GRID_WAIT();
  const long long c = blockIdx.x * 256ll + threadIdx.x;
  if (c >= N) return;
  const long long g = blockIdx.y, r0 = g * 32, r1 = r0 + 32 < M ? r0 + 32 : M;
  float acc = 0.0f;
  for (long long r = r0; r < r1; ++r) acc += (float)x[r * ld + c];
  part[g * ldp + c] = acc;
  SG_GRID_TRIGGER();
}

// --- losses.  Per-block loss partial sums (fixed order) -> loss_part[block]
// MSE: loss = sum((z-y)^2) * scale; dz = d*scale + d*scale (rules.py:53-58 on mul(d,d))
template <class T>
__global__ void __launch_bounds__(256) k_mse(const T* z, long long ldz, const T* y, long long ldy, long long M,
                                             long long N, T scale, void* dz, int dzd, long long lddz, void* dz2,
                                             int dz2d, long long lddz2, float* colsum, long long ldc,
                                             double* loss_part) {
  SG_GRID_WAIT();
  __shared__ double red[256];
  const long long c = blockIdx.x * 32ll + threadIdx.x;
  const long long g = blockIdx.y * 8ll + threadIdx.y;
  const long long r0 = g * 32;
  double lsum = 0.0;
  if (r0 < M && c < N) {
    T acc = (T)0;
    const long long r1 = r0 + 32 < M ? r0 + 32 : M;
    for (long long r = r0; r < r1; ++r) {
      const T d = z[r * ldz + c] - y[r * ldy + c];
      lsum += (double)d * (double)d;
      const T v = d * scale + d * scale;
      st_as(dz, dzd, r * lddz + c, (double)v);
      if (dz2) st_as(dz2, dz2d, r * lddz2 + c, (double)v);
      acc += v;
    }
    if (colsum) colsum[g * ldc + c] = (float)acc;
  }
  const int tid = threadIdx.y * 32 + threadIdx.x;
  red[tid] = lsum;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  if (tid == 0) loss_part[blockIdx.y * gridDim.x + blockIdx.x] = red[0] * (double)scale;
  SG_GRID_TRIGGER();
}

// clamped binary cross-entropy on logits (nn_train.py:209-227):
//   p = sigmoid(z); p2 = clamp(p, lo, hi) via lt/select + gt/select;
//   loss = -scale * sum(y log p2 + (1-y) log(1-p2));
//   dz = [p kept] * (-(g(1-y))/(1-p2) + (g y)/p2) * (p (1-p)),  g = -scale
// (pullback order: rules.py mul/log/sub, select passes only kept entries, sigmoid).
// Evaluated in f64 whatever the logit dtype: the clamp bounds 1e-7 / 1-1e-7
// are not representable in f32 (1-1e-7 rounds to 1-2^-23, and log(1-p)
// of a saturated prediction would move by 0.18), and the head is one column.
template <class T>
__global__ void __launch_bounds__(256) k_bce(const T* z, long long ldz, const T* y, long long ldy, long long M,
                                             long long N, T scale, void* dz, int dzd, long long lddz, void* dz2,
                                             int dz2d, long long lddz2, float* colsum, long long ldc,
                                             double* loss_part, unsigned* dom) {
  SG_GRID_WAIT();
  __shared__ double red[256];
  const long long c = blockIdx.x * 32ll + threadIdx.x;
  const long long g = blockIdx.y * 8ll + threadIdx.y;
  const long long r0 = g * 32;
  const double lo = 1e-7, hi = 1.0 - 1e-7, one = 1.0;
  bool ovf = false;
  double lsum = 0.0;
  if (r0 < M && c < N) {
    double acc = 0.0;
    const long long r1 = r0 + 32 < M ? r0 + 32 : M;
    for (long long r = r0; r < r1; ++r) {
      const double zz = (double)z[r * ldz + c], yy = (double)y[r * ldy + c];
      ovf |= zz < -EXP_MAX_ARG;  // scalar_sigmoid: math.exp(-z) overflows (tensor.py:214-215)
      const double p = one / (one + exp(-zz));
      const bool under = p < lo;
      const double p1 = under ? lo : p;
      const bool over = p1 > hi;
      const double p2 = over ? hi : p1;
      const double yn = one - yy, pn = one - p2;
      lsum += yy * log(p2) + yn * log(pn);
      const double gs = -(double)scale;
      const double pbar = (under || over) ? 0.0 : -((gs * yn) / pn) + (gs * yy) / p2;
      const double v = pbar * (p * (one - p));
      st_as(dz, dzd, r * lddz + c, v);
      if (dz2) st_as(dz2, dz2d, r * lddz2 + c, v);
      acc += v;
    }
    if (colsum) colsum[g * ldc + c] = (float)acc;
  }
  if (ovf && dom) atomicOr(dom, (unsigned)SG_DOM_EXP_OVERFLOW);
  const int tid = threadIdx.y * 32 + threadIdx.x;
  red[tid] = lsum;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  if (tid == 0) loss_part[blockIdx.y * gridDim.x + blockIdx.x] = red[0] * -(double)scale;
  SG_GRID_TRIGGER();
}

// The c1 loss IR's float64 domain conditions for one softmax row, checked
// beside the stable evaluation (see SG_DOM_* in include/sgb200.h):
// exp(z) overflow (OverflowError), row sum == 0 (div: DomainError) and
// exp(z_j)/sum == 0 (log: DomainError), evaluated exactly only for rows
// with an extreme logit (|z| > 700); warp-collective, lanes own columns
// lane + 32t of the row.
template <class T, int MAXT>
__device__ __forceinline__ void softmax_row_domain(const T (&zc)[MAXT], int nt, long long N, int lane, T mx,
                                                   unsigned* dom) {
  T mn = (T)INFINITY;
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
    if (t < nt && lane + 32 * t < N) mn = min(mn, zc[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (!dom || ((double)mx <= 700.0 && (double)mn >= -700.0)) return;  // warp-uniform
  if ((double)mx > EXP_MAX_ARG) {
    if (lane == 0) atomicOr(dom, (unsigned)SG_DOM_EXP_OVERFLOW);
    return;
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
    if (t < nt && lane + 32 * t < N) s += exp((double)zc[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (s == 0.0) {
    if (lane == 0) atomicOr(dom, (unsigned)SG_DOM_DIV_ZERO);
    return;
  }
  bool zero = false;
#pragma unroll
  for (int t = 0; t < MAXT; ++t)
    if (t < nt && lane + 32 * t < N) zero |= !(exp((double)zc[t]) / s > 0.0) && !isnan((double)zc[t]);
  if (__any_sync(0xffffffffu, zero) && lane == 0) atomicOr(dom, (unsigned)SG_DOM_LOG_NONPOS);
}

// softmax cross-entropy for narrow heads (N <= 128): one warp per row, a
// 32-warp block per 32-row group, so every row's dependent chain (max ->
// exp-sum -> log -> probabilities) runs concurrently; the group's column sums
// and loss are reduced through shared memory in a fixed order.
template <class T>
__global__ void __launch_bounds__(1024) k_softmax_xent_rows(const T* z, long long ldz, const T* y, long long ldy,
                                                            long long M, long long N, T scale, void* dz, int dzd,
                                                            long long lddz, void* dz2, int dz2d, long long lddz2,
                                                            float* colsum, long long ldc, double* loss_part,
                                                            unsigned* dom) {
  SG_GRID_WAIT();
  __shared__ float cs[32][129];
  __shared__ double red[32];
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const long long r = blockIdx.x * 32ll + w;
  const int nt = (int)((N + 31) / 32);  // <= 4
  double l = 0.0;
  T zc[4], yc[4];
  if (r < M) {
    T mx = -INFINITY;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const long long c = lane + 32ll * t;
      const bool ok = t < nt && c < N;
      zc[t] = ok ? z[r * ldz + c] : (T)-INFINITY;
      yc[t] = ok ? y[r * ldy + c] : (T)0;
      mx = max(mx, zc[t]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    T se = 0, sy = 0, syz = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t < nt && lane + 32 * t < N) {
        const T d = zc[t] - mx;
        se += exp(d);
        sy += yc[t];
        syz += yc[t] * d;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      se += __shfl_xor_sync(0xffffffffu, se, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
      syz += __shfl_xor_sync(0xffffffffu, syz, o);
    }
    softmax_row_domain<T, 4>(zc, nt, N, lane, mx, dom);
    const T lse = log(se);
    l = (double)(sy * lse - syz);  // -sum y (z - mx - lse)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const long long c = lane + 32ll * t;
      if (t < nt && c < N) {
        const T v = (exp(zc[t] - mx - lse) * sy - yc[t]) * scale;
        st_as(dz, dzd, r * lddz + c, (double)v);
        if (dz2) st_as(dz2, dz2d, r * lddz2 + c, (double)v);
        cs[w][c] = (float)v;
      }
    }
  } else {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (lane + 32 * t < 129) cs[w][lane + 32 * t] = 0.0f;
  }
  if (lane == 0) red[w] = l;
  __syncthreads();
  if (colsum) {
    for (int c = threadIdx.x; c < N; c += 1024) {
      float acc = 0.0f;
      for (int i = 0; i < 32; ++i) acc += cs[i][c];  // fixed order over the group's rows
      colsum[blockIdx.x * ldc + c] = acc;
    }
  }
  if (threadIdx.x == 0) {
    double s2 = 0.0;
    for (int i = 0; i < 32; ++i) s2 += red[i];
    loss_part[blockIdx.x] = s2 * (double)scale;
  }
  SG_GRID_TRIGGER();
}

// softmax cross-entropy, warp per row (N <= 1024):
//   loss_row = -sum_j y_j log p_j ; dz = (p * sum_j y_j - y) * scale  (scale = 1/n)
// Lanes own columns lane + 32t; each warp walks 32 consecutive rows so the
// column sums for the bias gradient stay in registers.
template <class T>
__global__ void __launch_bounds__(256) k_softmax_xent(const T* z, long long ldz, const T* y, long long ldy,
                                                      long long M, long long N, T scale, void* dz, int dzd,
                                                      long long lddz, void* dz2, int dz2d, long long lddz2,
                                                      float* colsum, long long ldc, double* loss_part,
                                                      unsigned* dom) {
  SG_GRID_WAIT();
  __shared__ double red[8];
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const long long g = blockIdx.x * 8ll + w;  // 32-row group
  const long long r0 = g * 32;
  constexpr int MAXT = 32;                   // N <= 1024
  T csum[MAXT];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) csum[t] = (T)0;
  const int nt = (int)((N + 31) / 32);
  double lsum = 0.0;
  if (r0 < M) {
    const long long r1 = r0 + 32 < M ? r0 + 32 : M;
    for (long long r = r0; r < r1; ++r) {
      T mx = -INFINITY;
      for (int t = 0; t < nt; ++t) {
        const long long c = lane + 32ll * t;
        if (c < N) mx = max(mx, z[r * ldz + c]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      T se = 0, sy = 0, syz = 0;
      for (int t = 0; t < nt; ++t) {
        const long long c = lane + 32ll * t;
        if (c < N) {
          const T zc = z[r * ldz + c] - mx;
          const T yc = y[r * ldy + c];
          se += exp(zc);
          sy += yc;
          syz += yc * zc;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        se += __shfl_xor_sync(0xffffffffu, se, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        syz += __shfl_xor_sync(0xffffffffu, syz, o);
      }
      {
        T zr[MAXT];
#pragma unroll
        for (int t = 0; t < MAXT; ++t) {
          const long long c = lane + 32ll * t;
          zr[t] = (t < nt && c < N) ? z[r * ldz + c] : (T)0;
        }
        softmax_row_domain<T, MAXT>(zr, nt, N, lane, mx, dom);
      }
      const T lse = log(se);
      if (lane == 0) lsum += (double)(sy * lse - syz);  // -sum y (z - mx - lse)
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        const long long c = lane + 32ll * t;
        if (t < nt && c < N) {
          const T p = exp(z[r * ldz + c] - mx - lse);
          const T v = (p * sy - y[r * ldy + c]) * scale;
          st_as(dz, dzd, r * lddz + c, (double)v);
          if (dz2) st_as(dz2, dz2d, r * lddz2 + c, (double)v);
          csum[t] += v;
        }
      }
    }
    if (colsum) {
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        const long long c = lane + 32ll * t;
        if (t < nt && c < N) colsum[g * ldc + c] = (float)csum[t];
      }
    }
  }
  if (lane == 0) red[w] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int i = 0; i < 8; ++i) s += red[i];
    loss_part[blockIdx.x] = s * (double)scale;
  }
  SG_GRID_TRIGGER();
}

// one block of 1024 threads, loads unrolled 8 deep: the c5 loss has 32 K
// partials (a 256-thread loop took 14 us); fixed order
__global__ void __launch_bounds__(1024) k_sum_loss(const double* part, long long n, double* out) {
  SG_GRID_WAIT();
  __shared__ double red[1024];
  double acc = 0.0;
#pragma unroll 8
  for (long long i = threadIdx.x; i < n; i += 1024) acc += part[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
  SG_GRID_TRIGGER();
}

// --- SGD over the flat parameter buffer + bf16 shadow copy for the next GEMMs
template <class T>
__global__ void k_sgd(T* p, const T* g, long long n, T lr, __nv_bfloat16* shadow) {
  SG_GRID_WAIT();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const T v = p[i] - lr * g[i];
    p[i] = v;
    if (shadow) shadow[i] = __float2bfloat16_rn((float)v);
  }
  SG_GRID_TRIGGER();
}
__global__ void k_sgd_vec(float4* p, const float4* g, long long n4, float lr, uint2* shadow) {
  SG_GRID_WAIT();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 v = p[i];
    const float4 d = __ldcs(g + i);
    v.x -= lr * d.x;
    v.y -= lr * d.y;
    v.z -= lr * d.z;
    v.w -= lr * d.w;
    p[i] = v;
    if (shadow) {
      __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
      shadow[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    }
  }
  SG_GRID_TRIGGER();
}

__global__ void k_cast(const void* src, int sd, void* dst, int dd, long long n) {
  SG_GRID_WAIT();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    st_as(dst, dd, i, ld_as<double>(src, sd, i));
  SG_GRID_TRIGGER();
}

// 2-D cast of a row-strided block; fp32 -> bf16 (the minibatch load) with
// 8-element vectors: two streaming float4 loads -> one 16-byte store.
// Blocks walk rows (grid-stride), threads the 8-column vectors of a row.
__global__ void k_cast2d_f32_bf16(const float* __restrict__ src, long long lds, __nv_bfloat16* __restrict__ dst,
                                  long long ldd, long long rows, long long vecs) {
  SG_GRID_WAIT();
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const float4* s4 = reinterpret_cast<const float4*>(src + r * lds);
    uint4* d4 = reinterpret_cast<uint4*>(dst + r * ldd);
    for (long long v = threadIdx.x; v < vecs; v += blockDim.x) {
      const float4 a = __ldcs(s4 + 2 * v), b = __ldcs(s4 + 2 * v + 1);
      __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(b.x, b.y), h3 = __floats2bfloat162_rn(b.z, b.w);
      d4[v] = make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                         *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
    }
  }
  SG_GRID_TRIGGER();
}
__global__ void k_cast2d(const void* src, int sd, long long lds, void* dst, int dd, long long ldd, long long rows,
                         long long cols) {
  SG_GRID_WAIT();
  for (long long r = blockIdx.x; r < rows; r += gridDim.x)
    for (long long c = threadIdx.x; c < cols; c += blockDim.x)
      st_as(dst, dd, r * ldd + c, ld_as<double>(src, sd, r * lds + c));
  SG_GRID_TRIGGER();
}

}  // namespace dk

int ctx_num_sms(sg_ctx* ctx);
int ctx_activate(sg_ctx* ctx);

}  // namespace sg

using namespace sg;

namespace {
inline unsigned cap_grid(long long n, int block, long long cap) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}
inline bool fdt(int d) { return d == SG_F32 || d == SG_F64; }
}  // namespace

namespace sg {
int colsum_finalize_launch(const float* part, long long G, long long ld, long long N, float* out, int,
                           cudaStream_t st) {
  if (N <= 0) return SG_OK;
  SG_CUDA_TRY(pdl_launch(dk::k_colsum_finalize, dim3((unsigned)((N + 31) / 32)), dim3(1024), 0, st, part, G, ld, N, out));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}
// stage 1 of a bias gradient for an already materialised dZ (bf16 / f32)
int colsum_partials(const void* x, int dtype, long long ld, long long M, long long N, float* part, long long ldp,
                    cudaStream_t st) {
  const dim3 grid((unsigned)((N + 255) / 256), (unsigned)((M + 31) / 32));
  if (grid.y > 65535) return fail(SG_EINVAL, "colsum: M too large");
  if (dtype == SG_BF16)
    SG_CUDA_TRY(pdl_launch(dk::k_colsum_part<__nv_bfloat16>, dim3(grid), dim3(256), 0, st, (const __nv_bfloat16*)x, ld, M, N, part, ldp));
  else if (dtype == SG_F32)
    SG_CUDA_TRY(pdl_launch(dk::k_colsum_part<float>, dim3(grid), dim3(256), 0, st, (const float*)x, ld, M, N, part, ldp));
  else
    return fail(SG_EINVAL, "colsum: bf16/f32 only");
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}
}  // namespace sg

extern "C" {

int sg_act_grad(sg_ctx* ctx, const void* ybar, int32_t ybar_dtype, int64_t ld_y, const void* h, int32_t h_dtype,
                int64_t ld_h, int64_t M, int64_t N, int32_t act, void* dz, int32_t dz_dtype, int64_t ld_dz,
                void* dz2, int32_t dz2_dtype, int64_t ld_dz2, float* colsum, int64_t ld_colsum, void* stream) {
  SG_NVTX("sg_act_grad");
  if (!ctx || !ybar || !h || !dz) return fail(SG_EINVAL, "null argument");
  if (M <= 0 || N <= 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (ybar_dtype == SG_F32 && (h_dtype == SG_BF16 || h_dtype == SG_F32) && h_dtype == dz_dtype && !dz2 &&
      N % 8 == 0 && ld_y % 8 == 0 && ld_h % 8 == 0 && ld_dz % 8 == 0 && a16(ybar) && a16(h) && a16(dz) &&
      (!colsum || (a16(colsum) && ld_colsum % 4 == 0)) && (M + 31) / 32 <= 65535) {
    dim3 g8((unsigned)((N + 511) / 512), (unsigned)((M + 31) / 32));
    if (h_dtype == SG_BF16)
      SG_CUDA_TRY(pdl_launch(dk::k_act_grad_v8<__nv_bfloat16, __nv_bfloat16>, dim3(g8), dim3(dim3(64, 4)), 0, (cudaStream_t)stream, (const float*)ybar, ld_y, (const __nv_bfloat16*)h,
                                                              ld_h, M, N, act, (__nv_bfloat16*)dz, ld_dz, colsum,
                                                              ld_colsum));
    else
      SG_CUDA_TRY(pdl_launch(dk::k_act_grad_v8<float, float>, dim3(g8), dim3(dim3(64, 4)), 0, (cudaStream_t)stream, (const float*)ybar, ld_y, (const float*)h, ld_h, M,
                                                              N, act, (float*)dz, ld_dz, colsum, ld_colsum));
    SG_CUDA_TRY(cudaGetLastError());
    return SG_OK;
  }
  dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 255) / 256));
  if (grid.y > 65535) return fail(SG_EINVAL, "act_grad: M too large");
  const bool f64 = ybar_dtype == SG_F64;
  if (f64)
    SG_CUDA_TRY(pdl_launch(dk::k_act_grad<double>, dim3(grid), dim3(dim3(32, 8)), 0, (cudaStream_t)stream, 
        ybar, ybar_dtype, ld_y, h, h_dtype, ld_h, M, N, act, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2, colsum,
        ld_colsum));
  else
    SG_CUDA_TRY(pdl_launch(dk::k_act_grad<float>, dim3(grid), dim3(dim3(32, 8)), 0, (cudaStream_t)stream, 
        ybar, ybar_dtype, ld_y, h, h_dtype, ld_h, M, N, act, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2, colsum,
        ld_colsum));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_colsum_finalize(sg_ctx* ctx, const float* part, int64_t G, int64_t ld_part, int64_t N, float* out,
                       void* stream) {
  SG_NVTX("sg_colsum_finalize");
  if (!ctx || !part || !out) return fail(SG_EINVAL, "null argument");
  if (N <= 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  SG_CUDA_TRY(pdl_launch(dk::k_colsum_finalize, dim3((unsigned)((N + 31) / 32)), dim3(1024), 0, (cudaStream_t)stream, part, G, ld_part, N,
                                                                                             out));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_colsum_finalize_multi(sg_ctx* ctx, int32_t n, const float* const* parts, const int64_t* G,
                             const int64_t* ld_part, const int64_t* N, float* const* outs, void* stream) {
  SG_NVTX("sg_colsum_finalize_multi");
  if (!ctx || n < 0 || (n && (!parts || !G || !ld_part || !N || !outs))) return fail(SG_EINVAL, "null argument");
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  for (int b0 = 0; b0 < n; b0 += dk::MAX_COLSUM_JOBS) {
    dk::ColsumJobs jobs{};
    const int nb = std::min(n - b0, dk::MAX_COLSUM_JOBS);
    long long nmax = 1;
    for (int i = 0; i < nb; ++i) {
      if (!parts[b0 + i] || !outs[b0 + i] || G[b0 + i] < 0 || N[b0 + i] < 0 || ld_part[b0 + i] < N[b0 + i])
        return fail(SG_EINVAL, "colsum_finalize_multi: bad job " + std::to_string(b0 + i));
      jobs.part[i] = parts[b0 + i];
      jobs.out[i] = outs[b0 + i];
      jobs.G[i] = G[b0 + i];
      jobs.ldp[i] = ld_part[b0 + i];
      jobs.N[i] = N[b0 + i];
      nmax = std::max(nmax, (long long)N[b0 + i]);
    }
    SG_CUDA_TRY(pdl_launch(dk::k_colsum_finalize_multi, dim3(dim3((unsigned)((nmax + 31) / 32), (unsigned)nb)), dim3(1024), 0, (cudaStream_t)stream, 
        jobs));
    SG_CUDA_TRY(cudaGetLastError());
  }
  return SG_OK;
}

int sg_colsum_strict(sg_ctx* ctx, const void* x, int32_t dtype, int64_t ld, int64_t M, int64_t N, void* out,
                     void* stream) {
  SG_NVTX("sg_colsum_strict");
  if (!ctx || !x || !out) return fail(SG_EINVAL, "null argument");
  if (!fdt(dtype)) return fail(SG_EINVAL, "colsum_strict: f32/f64 only");
  if (M <= 0 || N <= 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  if (dtype == SG_F64)
    SG_CUDA_TRY(pdl_launch(dk::k_colsum_strict<double>, dim3(cap_grid(N, 128, 1 << 20)), dim3(128), 0, (cudaStream_t)stream, 
        (const double*)x, ld, M, N, (double*)out));
  else
    SG_CUDA_TRY(pdl_launch(dk::k_colsum_strict<float>, dim3(cap_grid(N, 128, 1 << 20)), dim3(128), 0, (cudaStream_t)stream, 
        (const float*)x, ld, M, N, (float*)out));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_loss(sg_ctx* ctx, int32_t kind, const void* z, int32_t dtype, int64_t ld_z, const void* y, int64_t ld_y,
            int64_t M, int64_t N, double scale, double* loss, double* loss_part, int64_t n_part, void* dz,
            int32_t dz_dtype, int64_t ld_dz, void* dz2, int32_t dz2_dtype, int64_t ld_dz2, float* colsum,
            int64_t ld_colsum, void* stream) {
  SG_NVTX("sg_loss");
  if (!ctx || !z || !y || !dz || !loss || !loss_part) return fail(SG_EINVAL, "null argument");
  if (!fdt(dtype)) return fail(SG_EINVAL, "loss: logits must be f32/f64");
  if (M <= 0 || N <= 0) return fail(SG_EINVAL, "loss: empty batch");
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned* dom = ctx_domain_word(ctx);
  long long blocks = 0;
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (kind == SG_LOSS_MSE && dtype == SG_F32 && (dz_dtype == SG_BF16 || dz_dtype == SG_F32) && !dz2 &&
      N % 8 == 0 && ld_z % 8 == 0 &&
      ld_y % 8 == 0 && ld_dz % 8 == 0 && a16(z) && a16(y) && a16(dz) &&
      (!colsum || (a16(colsum) && ld_colsum % 4 == 0)) && (M + 31) / 32 <= 65535) {
    dim3 g8((unsigned)((N + 511) / 512), (unsigned)((M + 31) / 32));
    blocks = ((M + 31) / 32) * ((N + 31) / 32);  // one partial per 32 x 32 block (k_mse_v8)
    if (blocks > n_part) return fail(SG_EINVAL, "loss: loss_part too small");
    if (dz_dtype == SG_BF16)
      SG_CUDA_TRY(pdl_launch(dk::k_mse_v8<__nv_bfloat16>, dim3(g8), dim3(dim3(64, 4)), 0, st, (const float*)z, ld_z, (const float*)y, ld_y, M, N, (float)scale,
                                       (__nv_bfloat16*)dz, ld_dz, colsum, ld_colsum, loss_part));
    else
      SG_CUDA_TRY(pdl_launch(dk::k_mse_v8<float>, dim3(g8), dim3(dim3(64, 4)), 0, st, (const float*)z, ld_z, (const float*)y, ld_y, M, N, (float)scale,
                                               (float*)dz, ld_dz, colsum, ld_colsum, loss_part));
  } else if (kind == SG_LOSS_MSE) {
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 255) / 256));
    if (grid.y > 65535) return fail(SG_EINVAL, "loss: M too large");
    blocks = (long long)grid.x * grid.y;
    if (blocks > n_part) return fail(SG_EINVAL, "loss: loss_part too small");
    if (dtype == SG_F64)
      SG_CUDA_TRY(pdl_launch(dk::k_mse<double>, dim3(grid), dim3(dim3(32, 8)), 0, st, (const double*)z, ld_z, (const double*)y, ld_y, M, N,
                                                       scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2, colsum,
                                                       ld_colsum, loss_part));
    else
      SG_CUDA_TRY(pdl_launch(dk::k_mse<float>, dim3(grid), dim3(dim3(32, 8)), 0, st, (const float*)z, ld_z, (const float*)y, ld_y, M, N,
                                                      (float)scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2,
                                                      colsum, ld_colsum, loss_part));
  } else if (kind == SG_LOSS_BCE) {
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 255) / 256));
    if (grid.y > 65535) return fail(SG_EINVAL, "loss: M too large");
    blocks = (long long)grid.x * grid.y;
    if (blocks > n_part) return fail(SG_EINVAL, "loss: loss_part too small");
    if (dtype == SG_F64)
      SG_CUDA_TRY(pdl_launch(dk::k_bce<double>, dim3(grid), dim3(dim3(32, 8)), 0, st, (const double*)z, ld_z, (const double*)y, ld_y, M, N,
                                                       scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2, colsum,
                                                       ld_colsum, loss_part, dom));
    else
      SG_CUDA_TRY(pdl_launch(dk::k_bce<float>, dim3(grid), dim3(dim3(32, 8)), 0, st, (const float*)z, ld_z, (const float*)y, ld_y, M, N,
                                                      (float)scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2,
                                                      colsum, ld_colsum, loss_part, dom));
  } else if (kind == SG_LOSS_SOFTMAX_XENT && N <= 128) {
    blocks = (M + 31) / 32;
    if (blocks > n_part) return fail(SG_EINVAL, "loss: loss_part too small");
    if (dtype == SG_F64)
      SG_CUDA_TRY(pdl_launch(dk::k_softmax_xent_rows<double>, dim3((unsigned)blocks), dim3(1024), 0, st, 
          (const double*)z, ld_z, (const double*)y, ld_y, M, N, scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2,
          colsum, ld_colsum, loss_part, dom));
    else
      SG_CUDA_TRY(pdl_launch(dk::k_softmax_xent_rows<float>, dim3((unsigned)blocks), dim3(1024), 0, st, 
          (const float*)z, ld_z, (const float*)y, ld_y, M, N, (float)scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype,
          ld_dz2, colsum, ld_colsum, loss_part, dom));
  } else if (kind == SG_LOSS_SOFTMAX_XENT) {
    if (N > 1024) return fail(SG_EINVAL, "softmax_xent: at most 1024 classes");
    blocks = (M + 255) / 256;
    if (blocks > n_part) return fail(SG_EINVAL, "loss: loss_part too small");
    if (dtype == SG_F64)
      SG_CUDA_TRY(pdl_launch(dk::k_softmax_xent<double>, dim3((unsigned)blocks), dim3(256), 0, st, 
          (const double*)z, ld_z, (const double*)y, ld_y, M, N, scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype, ld_dz2,
          colsum, ld_colsum, loss_part, dom));
    else
      SG_CUDA_TRY(pdl_launch(dk::k_softmax_xent<float>, dim3((unsigned)blocks), dim3(256), 0, st, 
          (const float*)z, ld_z, (const float*)y, ld_y, M, N, (float)scale, dz, dz_dtype, ld_dz, dz2, dz2_dtype,
          ld_dz2, colsum, ld_colsum, loss_part, dom));
  } else {
    return fail(SG_EINVAL, "loss: unknown kind");
  }
  SG_CUDA_TRY(cudaGetLastError());
  SG_CUDA_TRY(pdl_launch(dk::k_sum_loss, dim3(1), dim3(1024), 0, st, loss_part, blocks, loss));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_sgd(sg_ctx* ctx, void* params, const void* grads, int32_t dtype, int64_t n, double lr, void* shadow_bf16,
           void* stream) {
  SG_NVTX("sg_sgd");
  if (!ctx || !params || !grads) return fail(SG_EINVAL, "null argument");
  if (!fdt(dtype)) return fail(SG_EINVAL, "sgd: f32/f64 parameters");
  if (n <= 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long cap = (long long)ctx_num_sms(ctx) * 8;
  const bool vec = dtype == SG_F32 && n % 4 == 0 && ((uintptr_t)params % 16) == 0 &&
                   ((uintptr_t)grads % 16) == 0 && (!shadow_bf16 || ((uintptr_t)shadow_bf16 % 8) == 0);
  if (vec)
    SG_CUDA_TRY(pdl_launch(dk::k_sgd_vec, dim3(cap_grid(n / 4, 256, cap)), dim3(256), 0, st, (float4*)params, (const float4*)grads, n / 4,
                                                              (float)lr, (uint2*)shadow_bf16));
  else if (dtype == SG_F32)
    SG_CUDA_TRY(pdl_launch(dk::k_sgd<float>, dim3(cap_grid(n, 256, cap)), dim3(256), 0, st, (float*)params, (const float*)grads, n, (float)lr,
                                                             (__nv_bfloat16*)shadow_bf16));
  else
    SG_CUDA_TRY(pdl_launch(dk::k_sgd<double>, dim3(cap_grid(n, 256, cap)), dim3(256), 0, st, (double*)params, (const double*)grads, n, lr,
                                                              (__nv_bfloat16*)shadow_bf16));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_cast(sg_ctx* ctx, const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t n, void* stream) {
  SG_NVTX("sg_cast");
  if (!ctx || !src || !dst) return fail(SG_EINVAL, "null argument");
  if (n <= 0) return SG_OK;
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  SG_CUDA_TRY(pdl_launch(dk::k_cast, dim3(cap_grid(n, 256, (long long)ctx_num_sms(ctx) * 16)), dim3(256), 0, (cudaStream_t)stream, 
      src, src_dtype, dst, dst_dtype, n));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_cast_2d(sg_ctx* ctx, const void* src, int32_t src_dtype, int64_t ld_src, void* dst, int32_t dst_dtype,
               int64_t ld_dst, int64_t rows, int64_t cols, void* stream) {
  SG_NVTX("sg_cast_2d");
  if (!ctx || !src || !dst) return fail(SG_EINVAL, "null argument");
  if (rows <= 0 || cols <= 0) return SG_OK;
  if (ld_src < cols || ld_dst < cols) return fail(SG_EINVAL, "cast_2d: leading dimension smaller than the row");
  if (src_dtype < SG_F32 || src_dtype > SG_BF16 || dst_dtype < SG_F32 || dst_dtype > SG_BF16)
    return fail(SG_EINVAL, "cast_2d: dtypes are f32 / f64 / bf16");
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = (unsigned)std::min<long long>(rows, (long long)ctx_num_sms(ctx) * 16);
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (src_dtype == SG_F32 && dst_dtype == SG_BF16 && cols % 8 == 0 && ld_src % 4 == 0 && ld_dst % 8 == 0 &&
      a16(src) && a16(dst)) {
    const long long vecs = cols / 8;
    const int block = vecs >= 256 ? 256 : (int)((vecs + 31) / 32 * 32);
    SG_CUDA_TRY(pdl_launch(dk::k_cast2d_f32_bf16, dim3(grid), dim3(block), 0, st, (const float*)src, ld_src, (__nv_bfloat16*)dst, ld_dst, rows,
                                                   vecs));
  } else {
    const int block = cols >= 256 ? 256 : (int)((cols + 31) / 32 * 32);
    SG_CUDA_TRY(pdl_launch(dk::k_cast2d, dim3(grid), dim3(block), 0, st, src, src_dtype, ld_src, dst, dst_dtype, ld_dst, rows, cols));
  }
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_sum_f64(sg_ctx* ctx, const double* part, int64_t n, double* out, void* stream) {
  SG_NVTX("sg_sum_f64");
  if (!ctx || !part || !out) return fail(SG_EINVAL, "null argument");
  if (n <= 0) return fail(SG_EINVAL, "sum_f64: empty");
  int rc = ctx_activate(ctx);
  if (rc) return rc;
  SG_CUDA_TRY(pdl_launch(dk::k_sum_loss, dim3(1), dim3(1024), 0, (cudaStream_t)stream, part, (long long)n, out));
  return SG_OK;
}

}  // extern "C"
