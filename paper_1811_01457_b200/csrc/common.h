// Shared host-side helpers of the sgb200 runtime.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/sgb200.h"

namespace sg {

// NVTX range over one C-ABI call (ranges for nsys / ncu --nvtx
// filtering).  NVTX3 is header-only: without an attached tool the push/pop
// are a null-check each.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define SG_NVTX(name) ::sg::NvtxRange sg_nvtx_range_(name)

// Last error message of the calling thread (sg_last_error).
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

inline int cuda_fail(cudaError_t e, const char* what) {
  return fail(SG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
// Driver API entry points, resolved through cudart (no link-time libcuda
// dependency, so the library also loads on hosts without a GPU driver).
struct Driver {
  CUresult (*moduleLoadData)(CUmodule*, const void*);
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*);
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, CUstream, void**, void**);
  CUresult (*getErrorString)(CUresult, const char**);
  CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int);
  CUresult (*launchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**);  // optional (PDL)
};
// Returns nullptr (and sets the error) if the driver cannot be reached.
const Driver* driver();

inline int cu_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  if (const Driver* d = driver()) d->getErrorString(r, &s);
  return fail(SG_ECUDA, std::string(what) + ": " + (s ? s : "unknown driver error"));
}

// Function attributes (cudaFuncSetAttribute) are per device: `mask` keeps one
// bit per device on which the caller already set them.  True the first time
// on the current device.
inline bool first_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const uint64_t bit = 1ull << (dev & 63);
  return !(mask.fetch_or(bit) & bit);
}

// Device word of the Dense-path domain flags (SG_DOM_*, sg_domain_check).
unsigned* ctx_domain_word(sg_ctx* ctx);
// The reference's float64 thresholds (CPython math.exp / glibc): exp(x) is
// finite for x <= EXP_MAX_ARG and raises OverflowError above it.
constexpr double EXP_MAX_ARG = 709.782712893384;
// fp32 form of "(double)z < -EXP_MAX_ARG": the largest float below -EXP_MAX_ARG
constexpr float SIGMOID_OVF_F32 = -709.78271484375f;

inline size_t dtype_size(int dt) { return dt == SG_F64 ? 8 : (dt == SG_F32 ? 4 : 2); }

inline long long numel(const sg_tensor& t) {
  long long n = 1;
  for (int i = 0; i < t.ndim; ++i) n *= t.shape[i];
  return n;
}

}  // namespace sg

#define SG_CUDA_TRY(expr)                                          \
  do {                                                             \
    cudaError_t e_ = (expr);                                       \
    if (e_ != cudaSuccess) return ::sg::cuda_fail(e_, #expr);      \
  } while (0)

#define SG_CU_TRY(expr)                                            \
  do {                                                             \
    CUresult r_ = (expr);                                          \
    if (r_ != CUDA_SUCCESS) return ::sg::cu_fail(r_, #expr);       \
  } while (0)
