// Precompiled reduction / broadcast helpers used around the fused kernels.
//
//  * sum of fp64 partials written by the fused gradient kernel, in a fixed
//    order (deterministic, like the reference's sequential cumsum folds,
//    tensor.py:287-345 — the order differs, the result is reproducible);
//  * generic broadcast materialisation for patterns that do not collapse
//    to the 2-D fast path;
//  * generic reduce_to(a .* b) for `fused_map_pullback` (forward_ad.py:226-235).
#include <cuda_runtime.h>

#include "common.h"
#include <algorithm>
#include <cstdlib>

#include "reduce_kernels.h"

namespace sg {

namespace {

// out[j] = sum_g part[g*N + j]: 32 columns x 32 row-groups per block (many
// independent loads in flight per column strip); each thread folds
// g = ty, ty+32, ... ascending, then a fixed fold over ty.
template <class T>
__global__ void __launch_bounds__(1024) k_sum_cols(const double* __restrict__ part, long long G, long long N,
                                                   T* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the partials come from the previous grid (PDL launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ double red[32][33];
  const long long j = blockIdx.x * 32ll + threadIdx.x;
  double acc = 0.0;
  if (j < N) {
#pragma unroll 4
    for (long long g = threadIdx.y; g < G; g += 32) acc += part[g * N + j];
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && j < N) {
    double s = red[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 32; ++y) s += red[y][threadIdx.x];
    out[j] = (T)s;
  }
}

// k_sum_cols for several jobs (blockIdx.y): identical arithmetic per column.
template <class T>
__global__ void __launch_bounds__(1024) k_sum_cols_multi(const __grid_constant__ SumJobs jobs) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ double red[32][33];
  const int b = blockIdx.y;
  const long long N = jobs.N[b], G = jobs.G[b];
  if (blockIdx.x * 32ll >= N) return;  // block-uniform
  const double* __restrict__ part = jobs.part[b];
  const long long j = blockIdx.x * 32ll + threadIdx.x;
  double acc = 0.0;
  if (j < N) {
#pragma unroll 4
    for (long long g = threadIdx.y; g < G; g += 32) acc += part[g * N + j];
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && j < N) {
    double s = red[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 32; ++y) s += red[y][threadIdx.x];
    reinterpret_cast<T*>(jobs.out[b])[j] = (T)s;
  }
}

// One block per output column; strided partial sums then a fixed tree.
template <class T>
__global__ void __launch_bounds__(256) k_sum_block(const double* __restrict__ part, long long G, long long N,
                                                   T* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ double red[256];
  for (long long j = blockIdx.x; j < N; j += gridDim.x) {
    double acc = 0.0;
    for (long long g = threadIdx.x; g < G; g += 256) acc += part[g * N + j];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = (T)red[0];
    __syncthreads();
  }
}

template <class T>
__global__ void k_expand(const T* __restrict__ in, T* __restrict__ out, long long n, DimMap m) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    long long rem = e, off = 0;
    for (int d = m.nd - 1; d >= 0; --d) {
      long long q = rem / m.ext[d];
      long long cd = rem - q * m.ext[d];
      rem = q;
      off += cd * m.stride[d];
    }
    out[e] = in[off];
  }
}

// out[o] = sum_j a[off(o,j)] * b[off(o,j)], block per output
template <class T>
__global__ void __launch_bounds__(256) k_reduce_block(const T* __restrict__ a, const T* __restrict__ b,
                                                      T* __restrict__ out, long long n_out, long long n_red,
                                                      DimMap kept, DimMap red_map) {
  __shared__ double red[256];
  for (long long o = blockIdx.x; o < n_out; o += gridDim.x) {
    long long rem = o, base = 0;
    for (int d = kept.nd - 1; d >= 0; --d) {
      long long q = rem / kept.ext[d];
      base += (rem - q * kept.ext[d]) * kept.stride[d];
      rem = q;
    }
    double acc = 0.0;
    for (long long j = threadIdx.x; j < n_red; j += 256) {
      long long r2 = j, off = base;
      for (int d = red_map.nd - 1; d >= 0; --d) {
        long long q = r2 / red_map.ext[d];
        off += (r2 - q * red_map.ext[d]) * red_map.stride[d];
        r2 = q;
      }
      double v = (double)a[off];
      if (b) v *= (double)b[off];
      acc += v;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[o] = (T)red[0];
    __syncthreads();
  }
}

// thread per output, sequential ascending fold (small reduction extents)
template <class T>
__global__ void k_reduce_thread(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                                long long n_out, long long n_red, DimMap kept, DimMap red_map) {
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < n_out;
       o += (long long)gridDim.x * blockDim.x) {
    long long rem = o, base = 0;
    for (int d = kept.nd - 1; d >= 0; --d) {
      long long q = rem / kept.ext[d];
      base += (rem - q * kept.ext[d]) * kept.stride[d];
      rem = q;
    }
    double acc = 0.0;
    for (long long j = 0; j < n_red; ++j) {
      long long r2 = j, off = base;
      for (int d = red_map.nd - 1; d >= 0; --d) {
        long long q = r2 / red_map.ext[d];
        off += (r2 - q * red_map.ext[d]) * red_map.stride[d];
        r2 = q;
      }
      double v = (double)a[off];
      if (b) v *= (double)b[off];
      acc += v;
    }
    out[o] = (T)acc;
  }
}

inline int grid_for(long long n, int block, int cap) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

template <class Kern, class... Args>
static cudaError_t launch_pdl_ew(Kern kern, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  static const bool pdl = [] {
    const char* e = std::getenv("SGB200_EW_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

int launch_sum_partials(const double* part, long long G, long long N, void* out, int dtype,
                        cudaStream_t s) {
  const bool blockwise = N < 256 && G >= 256;
  const dim3 gb(grid_for(N, 1, 4096)), gc((unsigned)((N + 31) / 32));
  if (dtype == SG_F32) {
    if (blockwise)
      SG_CUDA_TRY(launch_pdl_ew(k_sum_block<float>, gb, dim3(256), s, part, G, N, (float*)out));
    else
      SG_CUDA_TRY(launch_pdl_ew(k_sum_cols<float>, gc, dim3(32, 32), s, part, G, N, (float*)out));
  } else {
    if (blockwise)
      SG_CUDA_TRY(launch_pdl_ew(k_sum_block<double>, gb, dim3(256), s, part, G, N, (double*)out));
    else
      SG_CUDA_TRY(launch_pdl_ew(k_sum_cols<double>, gc, dim3(32, 32), s, part, G, N, (double*)out));
  }
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int launch_sum_partials_multi(const SumJobs& jobs, int dtype, cudaStream_t s) {
  SumJobs cols;
  long long nmax = 1;
  for (int i = 0; i < jobs.n; ++i) {
    if (jobs.N[i] < 256 && jobs.G[i] >= 256) {  // full-reduction shape: the blockwise kernel
      if (int rc = launch_sum_partials(jobs.part[i], jobs.G[i], jobs.N[i], jobs.out[i], dtype, s)) return rc;
      continue;
    }
    cols.part[cols.n] = jobs.part[i];
    cols.out[cols.n] = jobs.out[i];
    cols.G[cols.n] = jobs.G[i];
    cols.N[cols.n] = jobs.N[i];
    nmax = std::max(nmax, jobs.N[i]);
    ++cols.n;
  }
  if (cols.n == 0) return SG_OK;
  const dim3 grid((unsigned)((nmax + 31) / 32), (unsigned)cols.n);
  if (dtype == SG_F32) SG_CUDA_TRY(launch_pdl_ew(k_sum_cols_multi<float>, grid, dim3(32, 32), s, cols));
  else SG_CUDA_TRY(launch_pdl_ew(k_sum_cols_multi<double>, grid, dim3(32, 32), s, cols));
  return SG_OK;
}

int launch_expand(const void* in, void* out, long long n, const DimMap& m, int dtype, cudaStream_t s) {
  if (dtype == SG_F32)
    k_expand<float><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>((const float*)in, (float*)out, n, m);
  else
    k_expand<double><<<grid_for(n, 256, 148 * 16), 256, 0, s>>>((const double*)in, (double*)out, n, m);
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int launch_reduce(const void* a, const void* b, void* out, long long n_out, long long n_red,
                  const DimMap& kept, const DimMap& red, int dtype, cudaStream_t s) {
  const bool per_thread = n_red <= 64;
  if (dtype == SG_F32) {
    if (per_thread)
      k_reduce_thread<float><<<grid_for(n_out, 256, 148 * 16), 256, 0, s>>>(
          (const float*)a, (const float*)b, (float*)out, n_out, n_red, kept, red);
    else
      k_reduce_block<float><<<grid_for(n_out, 1, 148 * 16), 256, 0, s>>>(
          (const float*)a, (const float*)b, (float*)out, n_out, n_red, kept, red);
  } else {
    if (per_thread)
      k_reduce_thread<double><<<grid_for(n_out, 256, 148 * 16), 256, 0, s>>>(
          (const double*)a, (const double*)b, (double*)out, n_out, n_red, kept, red);
    else
      k_reduce_block<double><<<grid_for(n_out, 1, 148 * 16), 256, 0, s>>>(
          (const double*)a, (const double*)b, (double*)out, n_out, n_red, kept, red);
  }
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

}  // namespace sg
