#pragma once
#include <cuda_runtime.h>

namespace sg {

// Mixed-radix index map: coordinates over `ext` (row-major, last fastest)
// contribute coord * stride to an element offset.
struct DimMap {
  int nd;
  long long ext[8];
  long long stride[8];
};

int launch_sum_partials(const double* part, long long G, long long N, void* out, int dtype,
                        cudaStream_t s);
// Several partial-sum finalizations in as few launches as possible (one for
// all column-strip jobs, blockIdx.y = job); the same arithmetic per job.
constexpr int SUM_JOBS_MAX = 16;
struct SumJobs {
  int n = 0;
  const double* part[SUM_JOBS_MAX];
  void* out[SUM_JOBS_MAX];
  long long G[SUM_JOBS_MAX], N[SUM_JOBS_MAX];
};
int launch_sum_partials_multi(const SumJobs& jobs, int dtype, cudaStream_t s);
int launch_expand(const void* in, void* out, long long n, const DimMap& m, int dtype, cudaStream_t s);
int launch_reduce(const void* a, const void* b, void* out, long long n_out, long long n_red,
                  const DimMap& kept, const DimMap& red, int dtype, cudaStream_t s);

}  // namespace sg
