// sgb200 runtime: contexts, NVRTC variant cache and the fused-broadcast
// entry points of include/sgb200.h.
//
// The reference interprets a scalar IR function per element (interp.py:
// 322-352).  Here the host codegen hands us CUDA C++ for that function;
// for every broadcast pattern we instantiate the kernel skeleton
// (ew_skeleton.cuh) with NVRTC for sm_100a, cache the module, and launch
// it on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <memory>
#include <atomic>
#include <mutex>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <unistd.h>
#include <unordered_map>
#include <vector>

#include "common.h"
#include "ew_embed.h"
#include "reduce_kernels.h"
#include "sg_ew_params.h"

namespace sg {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

const Driver* driver() {
  static Driver d;
  static int state = 0;  // 0 unresolved, 1 ok, 2 failed
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (state == 0) {
    auto get = [](const char* name, void** fp) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fp, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fp;
    };
    bool ok = get("cuModuleLoadData", (void**)&d.moduleLoadData) &&
              get("cuModuleGetFunction", (void**)&d.moduleGetFunction) &&
              get("cuLaunchKernel", (void**)&d.launchKernel) &&
              get("cuGetErrorString", (void**)&d.getErrorString) &&
              get("cuFuncSetAttribute", (void**)&d.funcSetAttribute);
    if (!get("cuLaunchKernelEx", (void**)&d.launchKernelEx)) d.launchKernelEx = nullptr;
    state = ok ? 1 : 2;
  }
  if (state != 1) {
    set_error("CUDA driver entry points unavailable (no GPU driver?)");
    return nullptr;
  }
  return &d;
}

}  // namespace sg

using namespace sg;

struct sg_ctx {
  int device = 0;
  int num_sms = 148;
  std::atomic<int> sm_reserve{0};  // SMs left to concurrent collectives: max over live communicators
  std::vector<int> reserves;       // one entry per live communicator (sg_dp_init / sg_dp_finalize)
  unsigned long long* d_err = nullptr;
  unsigned* d_dom = nullptr;       // Dense-path domain flags (SG_DOM_*)
  long long step_limit = 2000000;  // interp.py:23 DEFAULT_STEP_LIMIT
  std::mutex mu;
};

namespace {

struct Variant {
  CUmodule mod = nullptr;
  CUfunction fwd = nullptr, grad = nullptr, pack = nullptr;
};

}  // namespace

struct sg_kernel {
  sg_ctx* ctx = nullptr;
  std::string src, key;
  int k = 0;
  int dtype = SG_F32;
  std::mutex mu;
  std::unordered_map<std::string, Variant> variants;
};

namespace {

std::string cache_dir() {
  const char* env = std::getenv("SGB200_CACHE");
  if (env && *env) return env;
  const char* home = std::getenv("HOME");
  return std::string(home ? home : "/tmp") + "/.cache/sgb200";
}

bool read_file(const std::string& path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return !out.empty();
}

void write_file(const std::string& path, const std::string& data) {
  std::string dir = cache_dir();
  std::string acc;
  for (size_t i = 0; i < dir.size(); ++i) {  // mkdir -p
    acc.push_back(dir[i]);
    if (dir[i] == '/' || i + 1 == dir.size()) mkdir(acc.c_str(), 0755);
  }
  std::string tmp = path + ".tmp" + std::to_string((long long)getpid());
  std::ofstream f(tmp, std::ios::binary);
  f.write(data.data(), (std::streamsize)data.size());
  f.close();
  std::rename(tmp.c_str(), path.c_str());
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

struct Shape2D {
  long long R = 1, C = 1;
  int kinds[SG_MAXK];
  bool expand[SG_MAXK];  // operand must be materialised at full shape first
};

// Capture-safe (no synchronising calls): the primary context was
// initialised once in sg_create, cudaSetDevice makes it current again.
int ensure_context(sg_ctx* ctx) {
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && cur == ctx->device) return SG_OK;
  SG_CUDA_TRY(cudaSetDevice(ctx->device));
  return SG_OK;
}

}  // namespace

namespace sg {
int ctx_num_sms(sg_ctx* ctx) { return ctx->num_sms; }
// SMs the persistent GEMMs may occupy: all of them, minus what an active
// data-parallel communicator reserves so its all-reduce kernels can run
// beside the backward GEMMs (a 1-CTA/SM persistent GEMM with ~227 KB of
// shared memory leaves no room for an NCCL CTA on the SMs it holds).
int ctx_compute_sms(sg_ctx* ctx) {
  const int n = ctx->num_sms - ctx->sm_reserve.load();
  return n < 2 ? 2 : (n & ~1);
}
// A communicator adds its reserve on init (delta > 0) and removes it on
// finalize (delta < 0).  The effective reserve is the MAX over the live
// communicators, not their sum: several trainers in one process share the
// same free SMs for their collectives, so a leaked or concurrent
// communicator never shrinks the GEMM grids further.
void ctx_add_sm_reserve(sg_ctx* ctx, int delta) {
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (delta > 0) {
    ctx->reserves.push_back(delta);
  } else if (delta < 0) {
    auto it = std::find(ctx->reserves.begin(), ctx->reserves.end(), -delta);
    if (it != ctx->reserves.end()) ctx->reserves.erase(it);
  }
  int m = 0;
  for (int r : ctx->reserves) m = std::max(m, r);
  ctx->sm_reserve = m;
}
int ctx_activate(sg_ctx* ctx) { return ensure_context(ctx); }
unsigned* ctx_domain_word(sg_ctx* ctx) { return ctx->d_dom; }
}  // namespace sg

namespace {

// Output shape of the broadcast (tensor.py:108-121): trailing alignment.
int broadcast_shape(int k, const sg_tensor* args, std::vector<long long>& out) {
  out.clear();
  for (int i = 0; i < k; ++i) {
    const sg_tensor& a = args[i];
    if (a.ndim == 0) continue;
    if (a.ndim < 0 || a.ndim > SG_MAX_DIMS) return fail(SG_EINVAL, "bad tensor rank");
    std::vector<long long> s(a.shape, a.shape + a.ndim);
    size_t n = std::max(out.size(), s.size());
    std::vector<long long> r(n);
    for (size_t j = 1; j <= n; ++j) {
      long long da = j <= out.size() ? out[out.size() - j] : 1;
      long long db = j <= s.size() ? s[s.size() - j] : 1;
      if (da != db && da != 1 && db != 1) {
        std::ostringstream m;
        m << "shapes do not broadcast (operand " << i << ")";
        return fail(SG_EINVAL, m.str());
      }
      r[n - j] = std::max(da, db);
    }
    out = r;
  }
  // Every operand must then expand to the result (tensor.py:124-132
  // can_expand, raised by bcast_to from interp.py's _spread_flat): the
  // reference's max() rule makes a zero extent against 1 (or against the
  // scalar start) a result extent of 1, which a zero-extent operand cannot
  // fill -- the reference raises ValueError for any empty tensor operand.
  for (int i = 0; i < k; ++i) {
    const sg_tensor& a = args[i];
    if (a.ndim == 0) continue;
    for (int j = 1; j <= a.ndim; ++j) {
      const long long d = a.shape[a.ndim - j];
      if (d != out[out.size() - j] && d != 1) {
        std::ostringstream m;
        m << "cannot broadcast operand " << i << " (extent " << d << ") to the result extent "
          << out[out.size() - j];
        return fail(SG_EINVAL, m.str());
      }
    }
  }
  return SG_OK;
}

// Collapse the broadcast to out[R][C] with one kind per operand.
// A 1-D problem (every operand full-shaped or a single element) has no
// preferred 2-D shape: fold it into rows of a wide power-of-two width so the
// kernels get their usual long per-thread row walks (scalar cotangents then
// accumulate in registers over many rows instead of one block reduction per
// 1024 elements).
void fold_rows(Shape2D& s) {
  if (s.R != 1 || s.C < (1ll << 16)) return;
  for (long long w = 4096; w >= 256; w >>= 1)
    if (s.C % w == 0) {
      s.R = s.C / w;
      s.C = w;
      return;
    }
}

long long elems(const std::vector<long long>& shape) {
  long long n = 1;
  for (long long d : shape) n *= d;
  return n;
}

void canonicalise(int k, const sg_tensor* args, const std::vector<long long>& out, Shape2D& s) {
  const int n = (int)out.size();
  for (int i = 0; i < k; ++i) s.expand[i] = false;
  auto bmask = [&](int d) {
    unsigned m = 0;
    for (int i = 0; i < k; ++i) {
      const sg_tensor& a = args[i];
      if (a.ndim == 0) continue;
      int pd = d - (n - a.ndim);
      long long e = pd >= 0 ? a.shape[pd] : 1;
      if (e == 1) m |= 1u << i;
    }
    return m;
  };
  struct G { unsigned mask; long long ext; };
  std::vector<G> groups;
  for (int d = 0; d < n; ++d) {
    if (out[d] == 1) continue;
    unsigned m = bmask(d);
    if (!groups.empty() && groups.back().mask == m)
      groups.back().ext *= out[d];
    else
      groups.push_back({m, out[d]});
  }
  if (groups.size() > 2) {
    // not 2-D: materialise every partially broadcast operand, then all
    // tensor operands are either full-shaped or single elements
    unsigned full_mask = 0;
    for (int i = 0; i < k; ++i) {
      if (args[i].ndim == 0) continue;
      if (numel(args[i]) == 1) continue;
      bool full = true;
      for (auto& g : groups) full = full && !(g.mask & (1u << i));
      if (!full) s.expand[i] = true;
    }
    (void)full_mask;
    long long total = 1;
    for (auto& g : groups) total *= g.ext;
    s.R = 1;
    s.C = total;
    for (int i = 0; i < k; ++i) {
      if (args[i].ndim == 0) s.kinds[i] = SG_SVAL;
      else if (numel(args[i]) == 1) s.kinds[i] = SG_SPTR;
      else s.kinds[i] = SG_FULL;
    }
    fold_rows(s);
    return;
  }
  if (groups.empty()) groups.push_back({0u, 1});
  if (groups.size() == 1) {
    s.R = 1;
    s.C = groups[0].ext;
    for (int i = 0; i < k; ++i) {
      if (args[i].ndim == 0) s.kinds[i] = SG_SVAL;
      else if (groups[0].mask & (1u << i)) s.kinds[i] = SG_SPTR;
      else s.kinds[i] = SG_FULL;
    }
    fold_rows(s);
    return;
  }
  s.R = groups[0].ext;
  s.C = groups[1].ext;
  for (int i = 0; i < k; ++i) {
    if (args[i].ndim == 0) {
      s.kinds[i] = SG_SVAL;
      continue;
    }
    bool br = groups[0].mask & (1u << i), bc = groups[1].mask & (1u << i);
    if (!br && !bc) s.kinds[i] = SG_FULL;
    else if (br && !bc) s.kinds[i] = SG_ROW;
    else if (!br && bc) s.kinds[i] = SG_COL;
    else s.kinds[i] = SG_SPTR;
  }
}

// DimMap from the output shape to an operand's elements (stride 0 where broadcast).
DimMap operand_map(const sg_tensor& a, const std::vector<long long>& out) {
  DimMap m{};
  const int n = (int)out.size();
  m.nd = n;
  long long st = 1;
  for (int d = n - 1; d >= 0; --d) {
    int pd = d - (n - a.ndim);
    long long e = pd >= 0 ? a.shape[pd] : 1;
    m.ext[d] = out[d];
    m.stride[d] = (e == 1) ? 0 : st;
    st *= e;
  }
  return m;
}

struct Launch {
  int vec, bdx, bdy;
  unsigned gx, gy;
  long long rpb;
  int rowmode = 0;  // gradient kernel: one warp per row (COL operands, no ROW operands)
  int flat = 0;     // forward kernel: flat address-order walk (SG_FLAT)
};

long long env_ll(const char* name, long long dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoll(e) : dflt;
}

// Blocks per SM the grid is sized for (an upper bound: at most one row per
// thread-row).  Tuned on B200 (tools/ew_sweep*.sh, c2 shape): the forward
// kernel streams best with many short-lived blocks (64/SM: ~27 rows each);
// the gradient kernel amortises its fp64 partial-sum rows over long spans
// (6/SM, 85-register budget, SG_GRAD_MINB 3, up to 4 rows in flight).
Launch plan(const sg_ctx* ctx, const Shape2D& s, int dtype, const sg_tensor* args, int k,
            const void* const* extra_ptrs, int n_extra, long long per_sm = 8, long long max_bdx = 256) {
  Launch L;
  const int esz = dtype == SG_F64 ? 8 : 4;
  int vec = 16 / esz;
  auto aligned = [&](const void* p) { return ((uintptr_t)p % 16) == 0; };
  bool ok = (s.C % vec) == 0;
  for (int i = 0; i < k && ok; ++i)
    if (args[i].ndim > 0 && !s.expand[i] && (s.kinds[i] == SG_FULL || s.kinds[i] == SG_ROW))
      ok = aligned(args[i].ptr);
  for (int i = 0; i < n_extra && ok; ++i)
    if (extra_ptrs[i]) ok = aligned(extra_ptrs[i]);
  if (!ok) vec = 1;
  L.vec = vec;
  long long cv = (s.C + vec - 1) / vec;
  int bdx = 1;
  if (max_bdx < 1 || max_bdx > 256) max_bdx = 256;
  while (bdx < cv && bdx < max_bdx) bdx <<= 1;
  L.bdx = bdx;
  L.bdy = 256 / bdx;
  long long gx = (cv + bdx - 1) / bdx;
  L.gx = (unsigned)gx;
  long long target = (long long)ctx->num_sms * per_sm;
  long long gy = std::max<long long>(1, std::min<long long>((s.R + L.bdy - 1) / L.bdy,
                                                             (target + gx - 1) / gx));
  gy = std::min<long long>(gy, 65535);
  L.rpb = (s.R + gy - 1) / gy;
  L.gy = (unsigned)((s.R + L.rpb - 1) / L.rpb);
  if (L.gy == 0) L.gy = 1;
  return L;
}

std::string variant_key(int k, const int* kinds, const Launch& L) {
  std::ostringstream key;
  key << "v" << L.vec << "x" << L.bdx << "y" << L.bdy << (L.rowmode ? "r" : "") << (L.flat ? "f" : "") << "k";
  for (int i = 0; i < k; ++i) key << kinds[i];
  return key.str();
}

std::string build_source(const std::string& user, const std::string& tag, int k, int dtype,
                         const int* kinds, const Launch& L) {
  std::ostringstream src;
  src << "// sgb200 fused kernel " << tag << "\n";
  if (dtype == SG_F64) src << "typedef double T;\n#define SG_T_IS_DOUBLE 1\n";
  else src << "typedef float T;\n";
  src << "#define SG_K " << k << "\n#define SG_KT " << std::max(1, k) << "\n";
  src << "#define SG_VEC " << L.vec << "\n#define SG_BDX " << L.bdx << "\n#define SG_BDY " << L.bdy << "\n";
  bool has_col = false;
  for (int i = 0; i < k; ++i) has_col |= kinds[i] == SG_COL;
  bool has_row = false;
  for (int i = 0; i < k; ++i) has_row |= kinds[i] == SG_ROW;
  src << "#define SG_HAS_COL " << (has_col ? 1 : 0) << "\n#define SG_HAS_ROW " << (has_row ? 1 : 0) << "\n";
  src << "#define SG_ROWMODE " << L.rowmode << "\n";
  src << "#define SG_FLAT " << L.flat << "\n";
  // tuning overrides, e.g. SGB200_EW_DEFINES="#define SG_UNROLL 8"
  if (const char* extra = std::getenv("SGB200_EW_DEFINES")) src << extra << "\n";
  // gradient kernel: 3 blocks per SM (85-register budget) and as many rows in
  // flight as x/ybar-style row loads fit: 32 registers of row data per
  // thread (c2: x + ybar, float4 -> 4 rows; measured on B200, tools/ew_sweep8.sh)
  {
    int nfull = 0;
    for (int i = 0; i < k; ++i) nfull += kinds[i] == SG_FULL;
    const int words = (nfull + 1) * L.vec * (dtype == SG_F64 ? 2 : 1);  // 32-bit registers per row
    const bool f64 = dtype == SG_F64;  // f64 measured best at the earlier 4 blocks/SM, 3 rows
    const int rows = f64 ? 3 : std::max(1, std::min(4, 32 / std::max(1, words)));
    src << "#ifndef SG_GRAD_MINB\n#define SG_GRAD_MINB " << (f64 ? 4 : 3) << "\n#endif\n";
    src << "#ifndef SG_GUNROLL\n#define SG_GUNROLL " << rows << "\n#endif\n";
  }
  src << "#define SG_KINDS {";
  for (int i = 0; i < std::max(1, k); ++i) src << (i ? "," : "") << (i < k ? kinds[i] : 0);
  src << "}\n";
  src << kSgEwParamsSrc << "\n";
  // the user code needs D/T/sg_exp from the skeleton prelude: split the
  // skeleton at the marker so helpers precede the user functions and the
  // kernels follow them
  std::string skel = kSgEwSkeletonSrc;
  const std::string marker = "static __device__ const int sg_kinds";
  size_t cut = skel.find(marker);
  src << skel.substr(0, cut) << "\n" << user << "\n" << skel.substr(cut);
  return src.str();
}

int nvrtc_compile(const std::string& full, std::string& cubin) {
  const uint64_t h = fnv1a(full);
  char hbuf[32];
  std::snprintf(hbuf, sizeof hbuf, "%016llx", (unsigned long long)h);
  const std::string cpath = cache_dir() + "/ew_" + hbuf + ".cubin";
  if (read_file(cpath, cubin)) return SG_OK;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, full.c_str(), "sg_fused.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return fail(SG_ECUDA, "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-lineinfo", "--std=c++17",
                        "-DSG_NVRTC=1", "-diag-suppress=177,550"};
  nvrtcResult rc = nvrtcCompileProgram(prog, 6, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    return fail(SG_ECUDA, "NVRTC compile failed:\n" + log);
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin.resize(n);
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  write_file(cpath, cubin);
  return SG_OK;
}

int compile_variant(sg_kernel* kern, const Shape2D& s, const Launch& L, Variant** out) {
  const std::string key = variant_key(kern->k, s.kinds, L);
  std::lock_guard<std::mutex> g(kern->mu);
  auto it = kern->variants.find(key);
  if (it != kern->variants.end()) {
    *out = &it->second;
    return SG_OK;
  }
  std::string cubin;
  int rc = nvrtc_compile(build_source(kern->src, kern->key + " " + key, kern->k, kern->dtype, s.kinds, L),
                         cubin);
  if (rc) return rc;
  Variant v;
  if ((rc = ensure_context(kern->ctx))) return rc;
  const Driver* drv = driver();
  if (!drv) return SG_ECUDA;
  SG_CU_TRY(drv->moduleLoadData(&v.mod, cubin.data()));
  SG_CU_TRY(drv->moduleGetFunction(&v.fwd, v.mod, "sg_ew_forward"));
  SG_CU_TRY(drv->moduleGetFunction(&v.grad, v.mod, "sg_ew_grad"));
  SG_CU_TRY(drv->moduleGetFunction(&v.pack, v.mod, "sg_ew_pack"));
  auto res = kern->variants.emplace(key, v);
  *out = &res.first->second;
  return SG_OK;
}

int check_args(sg_kernel* kern, int k, const sg_tensor* args) {
  if (!kern) return fail(SG_EINVAL, "null kernel");
  if (k != kern->k) {
    std::ostringstream m;
    m << "kernel takes " << kern->k << " arguments, got " << k;
    return fail(SG_EINVAL, m.str());
  }
  for (int i = 0; i < k; ++i) {
    if (args[i].ndim > 0 && args[i].dtype != kern->dtype)
      return fail(SG_EINVAL, "operand dtype does not match the kernel dtype");
    if (args[i].ndim > 0 && !args[i].ptr && numel(args[i]) > 0) return fail(SG_EINVAL, "null operand");
  }
  return SG_OK;
}

int check_out(const sg_tensor* t, const std::vector<long long>& shape, int dtype, const char* what,
              int lead = -1) {
  std::vector<long long> want = shape;
  if (lead >= 0) want.insert(want.begin(), lead);
  long long n = 1;
  for (long long d : want) n *= d;
  if (!t || t->dtype != dtype) return fail(SG_EINVAL, std::string(what) + ": dtype mismatch");
  // same extents in the same order (size-1 axes aside): a transposed or
  // reshaped buffer with the right element count is still an error
  std::vector<long long> got, exp;
  for (int i = 0; i < t->ndim; ++i)
    if (t->shape[i] != 1) got.push_back(t->shape[i]);
  for (long long d : want)
    if (d != 1) exp.push_back(d);
  if (numel(*t) != n || got != exp) return fail(SG_EINVAL, std::string(what) + ": shape mismatch");
  if (!t->ptr && n) return fail(SG_EINVAL, std::string(what) + ": null pointer");
  return SG_OK;
}

// Operands that do not fit the 2-D pattern are materialised into temporaries.
// Temporaries (expanded operands, partial sums) are stream-ordered
// allocations owned here: freed on every path out of a call, the early
// error returns included.
struct Prepared {
  SgEwParams p;
  std::vector<void*> temps;
  cudaStream_t st = nullptr;
  Prepared() = default;
  Prepared(const Prepared&) = delete;
  Prepared& operator=(const Prepared&) = delete;
  ~Prepared() {
    for (void* t : temps) cudaFreeAsync(t, st);
  }
};

int prepare(sg_kernel* kern, int k, const sg_tensor* args, const std::vector<long long>& out,
            const Shape2D& s, cudaStream_t st, Prepared& pr) {
  std::memset(&pr.p, 0, sizeof pr.p);
  pr.st = st;
  long long total = 1;
  for (long long d : out) total *= d;
  for (int i = 0; i < k; ++i) {
    pr.p.sval[i] = args[i].scalar;
    pr.p.in[i] = args[i].ptr;
    if (s.expand[i]) {
      void* tmp = nullptr;
      SG_CUDA_TRY(cudaMallocAsync(&tmp, (size_t)total * dtype_size(kern->dtype), st));
      pr.temps.push_back(tmp);
      int rc = launch_expand(args[i].ptr, tmp, total, operand_map(args[i], out), kern->dtype, st);
      if (rc) return rc;
      pr.p.in[i] = tmp;
    }
  }
  pr.p.R = s.R;
  pr.p.C = s.C;
  pr.p.c_log2 = -1;
  if (s.C > 0 && (s.C & (s.C - 1)) == 0)
    for (int b = 0; b < 63; ++b)
      if ((1ll << b) == s.C) pr.p.c_log2 = b;
  pr.p.err = kern->ctx->d_err;
  pr.p.step_limit = kern->ctx->step_limit;
  return SG_OK;
}

int release(Prepared& pr, cudaStream_t st) {
  for (void* t : pr.temps) SG_CUDA_TRY(cudaFreeAsync(t, st));
  pr.temps.clear();
  return SG_OK;
}

int launch(CUfunction f, const Launch& L, SgEwParams& p, cudaStream_t st) {
  p.rows_per_block = L.rpb;
  void* params[] = {&p};
  const Driver* drv = driver();
  if (!drv) return SG_ECUDA;
  // programmatic dependent launch: the kernel's prologue and launch overlap the
  // previous grid's tail (its griddepcontrol.wait orders the memory accesses)
  static const bool pdl = [] {
    const char* e = std::getenv("SGB200_EW_PDL");
    return !(e && e[0] == '0');
  }();
  if (pdl && drv->launchKernelEx) {
    CUlaunchConfig cfg = {};
    cfg.gridDimX = L.gx;
    cfg.gridDimY = L.gy;
    cfg.gridDimZ = 1;
    cfg.blockDimX = L.bdx;
    cfg.blockDimY = L.bdy;
    cfg.blockDimZ = 1;
    cfg.sharedMemBytes = 0;
    cfg.hStream = (CUstream)st;
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SG_CU_TRY(drv->launchKernelEx(&cfg, f, params, nullptr));
    return SG_OK;
  }
  SG_CU_TRY(drv->launchKernel(f, L.gx, L.gy, 1, L.bdx, L.bdy, 1, 0, (CUstream)st, params, nullptr));
  return SG_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int sg_version(void) { return 1; }

int sg_last_error(char* buf, size_t n) {
  if (!buf || n == 0) return SG_EINVAL;
  std::snprintf(buf, n, "%s", sg::g_last_error.c_str());
  return SG_OK;
}

int sg_create(int device, sg_ctx** out) {
  if (!out) return fail(SG_EINVAL, "null output");
  auto* ctx = new sg_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) {
    delete ctx;
    return fail(SG_ECUDA, "cannot initialise the CUDA primary context");
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&ctx->d_err, sizeof(unsigned long long)) != cudaSuccess) {
    delete ctx;
    return fail(SG_ECUDA, "cudaMalloc(error word) failed");
  }
  cudaMemset(ctx->d_err, 0xff, sizeof(unsigned long long));
  if (cudaMalloc(&ctx->d_dom, sizeof(unsigned)) != cudaSuccess) {
    cudaFree(ctx->d_err);
    delete ctx;
    return fail(SG_ECUDA, "cudaMalloc(domain word) failed");
  }
  cudaMemset(ctx->d_dom, 0, sizeof(unsigned));
  // keep stream-ordered temporaries cached in the pool between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaDeviceSynchronize();
  *out = ctx;
  return SG_OK;
}

int sg_destroy(sg_ctx* ctx) {
  if (!ctx) return SG_OK;
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->d_dom) cudaFree(ctx->d_dom);
  delete ctx;
  return SG_OK;
}

int sg_ew_set_step_limit(sg_ctx* ctx, int64_t limit) {
  if (!ctx) return fail(SG_EINVAL, "null ctx");
  ctx->step_limit = limit;
  return SG_OK;
}

int sg_ew_compile(sg_ctx* ctx, const char* user_src, const char* key, int k, int dtype,
                  sg_kernel** out) {
  SG_NVTX("sg_ew_compile");
  if (!ctx || !user_src || !out) return fail(SG_EINVAL, "null argument");
  if (k < 0 || k > SG_MAXK) return fail(SG_EINVAL, "fused_map supports at most 16 operands");
  if (dtype != SG_F32 && dtype != SG_F64) return fail(SG_EINVAL, "fused kernels compute in f32 or f64");
  auto* kern = new sg_kernel();
  kern->ctx = ctx;
  kern->src = user_src;
  kern->key = key ? key : "";
  kern->k = k;
  kern->dtype = dtype;
  *out = kern;
  return SG_OK;
}

int sg_ew_variant_count(sg_kernel* kern) { return kern ? (int)kern->variants.size() : 0; }

int sg_ew_compile_only(const char* user_src, int k, int dtype, const int* kinds, int vec, int bdx,
                       int bdy, size_t* cubin_bytes) {
  if (!user_src || (k && !kinds)) return fail(SG_EINVAL, "null argument");
  if (k < 0 || k > SG_MAXK) return fail(SG_EINVAL, "fused_map supports at most 16 operands");
  Launch L{vec, bdx, bdy, 1, 1, 1};
  std::string cubin;
  int rc = nvrtc_compile(build_source(user_src, "compile-only", k, dtype, kinds, L), cubin);
  if (rc) return rc;
  if (cubin_bytes) *cubin_bytes = cubin.size();
  if (const char* path = std::getenv("SGB200_CUBIN_OUT")) {  // inspection hook (cuobjdump)
    if (FILE* f = std::fopen(path, "wb")) {
      std::fwrite(cubin.data(), 1, cubin.size(), f);
      std::fclose(f);
    }
  }
  return SG_OK;
}

int sg_ew_forward(sg_ctx* ctx, sg_kernel* kern, int k, const sg_tensor* args, sg_tensor* y, void* stream) {
  SG_NVTX("sg_ew_forward");
  int rc = check_args(kern, k, args);
  if (rc) return rc;
  std::vector<long long> out;
  if ((rc = broadcast_shape(k, args, out))) return rc;
  if ((rc = check_out(y, out, kern->dtype, "y"))) return rc;
  if (elems(out) == 0) return SG_OK;  // an empty broadcast: nothing to compute
  Shape2D s;
  canonicalise(k, args, out, s);
  const void* extra[] = {y->ptr};
  Launch L = plan(ctx, s, kern->dtype, args, k, extra, 1, env_ll("SGB200_EW_FWD_BLOCKS_PER_SM", 64),
                  env_ll("SGB200_EW_FWD_BDX", 256));
  if (env_ll("SGB200_EW_FLAT", 0)) {  // flat address-order walk
    const long long nvec = s.R * s.C / L.vec;
    const long long per_block = 256ll * 4;  // 256 threads x SG_UNROLL (4) vectors
    L.flat = 1;
    L.bdx = 256;
    L.bdy = 1;
    L.gx = (unsigned)((nvec + per_block - 1) / per_block);
    L.gy = 1;
    L.rpb = 0;
  }
  Variant* v = nullptr;
  if ((rc = compile_variant(kern, s, L, &v))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  Prepared pr;
  if ((rc = prepare(kern, k, args, out, s, st, pr))) return rc;
  pr.p.out = y->ptr;
  if ((rc = launch(v->fwd, L, pr.p, st))) return rc;
  return release(pr, st);
}

int sg_ew_pack(sg_ctx* ctx, sg_kernel* kern, int k, const sg_tensor* args, sg_tensor* pack, void* stream) {
  SG_NVTX("sg_ew_pack");
  int rc = check_args(kern, k, args);
  if (rc) return rc;
  std::vector<long long> out;
  if ((rc = broadcast_shape(k, args, out))) return rc;
  if ((rc = check_out(pack, out, kern->dtype, "pack", 1 + k))) return rc;
  if (elems(out) == 0) return SG_OK;
  Shape2D s;
  canonicalise(k, args, out, s);
  const void* extra[] = {pack->ptr};
  Launch L = plan(ctx, s, kern->dtype, args, k, extra, 1);
  Variant* v = nullptr;
  if ((rc = compile_variant(kern, s, L, &v))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  Prepared pr;
  if ((rc = prepare(kern, k, args, out, s, st, pr))) return rc;
  pr.p.pack = pack->ptr;
  if ((rc = launch(v->pack, L, pr.p, st))) return rc;
  return release(pr, st);
}

int sg_ew_grad(sg_ctx* ctx, sg_kernel* kern, int k, const sg_tensor* args, const sg_tensor* ybar,
               sg_tensor* y, sg_tensor* argbars, void* stream) {
  SG_NVTX("sg_ew_grad");
  int rc = check_args(kern, k, args);
  if (rc) return rc;
  std::vector<long long> out;
  if ((rc = broadcast_shape(k, args, out))) return rc;
  if ((rc = check_out(ybar, out, kern->dtype, "ybar"))) return rc;
  if (y && y->ptr && (rc = check_out(y, out, kern->dtype, "y"))) return rc;
  for (int i = 0; i < k; ++i) {
    long long want = args[i].ndim == 0 ? 1 : numel(args[i]);
    if (argbars[i].dtype != kern->dtype || numel(argbars[i]) != want || (!argbars[i].ptr && want))
      return fail(SG_EINVAL, "argbar " + std::to_string(i) + " does not match its operand");
  }
  if (elems(out) == 0) {
    // an empty broadcast: every cotangent is a sum of zero terms (reduce_like,
    // rules.py:302-311 / tensor.py:327-345) -- zeros
    for (int i = 0; i < k; ++i) {
      const long long want = args[i].ndim == 0 ? 1 : numel(args[i]);
      if (want) SG_CUDA_TRY(cudaMemsetAsync(argbars[i].ptr, 0, (size_t)want * dtype_size(kern->dtype),
                                            (cudaStream_t)stream));
    }
    return SG_OK;
  }
  Shape2D s;
  canonicalise(k, args, out, s);
  std::vector<const void*> extra = {ybar->ptr, y ? y->ptr : nullptr};
  for (int i = 0; i < k; ++i) extra.push_back(s.kinds[i] == SG_FULL ? argbars[i].ptr : nullptr);
  Launch L = plan(ctx, s, kern->dtype, args, k, extra.data(), (int)extra.size(),
                  env_ll("SGB200_EW_GRAD_BLOCKS_PER_SM", kern->dtype == SG_F64 ? 8 : 6),
                  env_ll("SGB200_EW_GRAD_BDX", 256));
  // COL operands without ROW operands: warps own rows and walk the columns, so
  // each row's cotangent is one register accumulation + one warp reduction
  // (instead of a shuffle tree per 128 elements) and is written final.
  bool has_col = false, has_row = false;
  for (int i = 0; i < k; ++i) {
    has_col |= s.kinds[i] == SG_COL;
    has_row |= s.kinds[i] == SG_ROW;
  }
  if (has_col && !has_row && s.C >= 32ll * L.vec && env_ll("SGB200_EW_ROWMODE", 1)) {
    L.rowmode = 1;
    L.bdx = 256;
    L.bdy = 1;
    L.gx = 1;
    const long long warps = (s.R + 7) / 8;
    L.gy = (unsigned)std::max<long long>(1, std::min<long long>(
        {warps, (long long)ctx->num_sms * env_ll("SGB200_EW_ROWMODE_BLOCKS_PER_SM", 8), 65535ll}));
    L.rpb = 0;
  }
  Variant* v = nullptr;
  if ((rc = compile_variant(kern, s, L, &v))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  Prepared pr;
  if ((rc = prepare(kern, k, args, out, s, st, pr))) return rc;
  pr.p.ybar = ybar->ptr;
  pr.p.out = y ? y->ptr : nullptr;
  long long total = s.R * s.C;
  const long long G_row = (long long)L.gy * L.bdy;
  const long long G_col = L.rowmode ? 1 : (long long)L.gx * L.bdx / std::min(32, L.bdx);
  const long long G_blk = (long long)L.gx * L.gy;
  for (int i = 0; i < k; ++i) {
    const int kind = s.kinds[i];
    if (kind == SG_FULL) {
      // an expanded operand's full cotangent lands in a temporary, then reduce_to
      if (s.expand[i]) {
        void* tmp = nullptr;
        SG_CUDA_TRY(cudaMallocAsync(&tmp, (size_t)total * dtype_size(kern->dtype), st));
        pr.temps.push_back(tmp);
        pr.p.xbar[i] = tmp;
      } else {
        pr.p.xbar[i] = argbars[i].ptr;
      }
      continue;
    }
    long long n = kind == SG_ROW ? G_row * s.C : kind == SG_COL ? G_col * s.R : G_blk;
    double* pp = nullptr;
    SG_CUDA_TRY(cudaMallocAsync((void**)&pp, (size_t)n * sizeof(double), st));
    pr.temps.push_back(pp);
    pr.p.part[i] = pp;
  }
  if ((rc = launch(v->grad, L, pr.p, st))) return rc;
  SumJobs jobs;
  for (int i = 0; i < k; ++i) {
    const int kind = s.kinds[i];
    if (kind == SG_FULL) {
      if (s.expand[i]) {
        // reduce the full-shape cotangent to the operand's own shape
        DimMap kept{}, red{};
        const int n = (int)out.size();
        long long st_in = 1;
        std::vector<long long> stride(n);
        for (int d = n - 1; d >= 0; --d) {
          stride[d] = st_in;
          st_in *= out[d];
        }
        long long n_out = 1, n_red = 1;
        for (int d = 0; d < n; ++d) {
          int pd = d - (n - args[i].ndim);
          long long e = pd >= 0 ? args[i].shape[pd] : 1;
          if (e == out[d]) {
            kept.ext[kept.nd] = out[d];
            kept.stride[kept.nd++] = stride[d];
            n_out *= out[d];
          } else {
            red.ext[red.nd] = out[d];
            red.stride[red.nd++] = stride[d];
            n_red *= out[d];
          }
        }
        if ((rc = launch_reduce(pr.p.xbar[i], nullptr, argbars[i].ptr, n_out, n_red, kept, red,
                                kern->dtype, st)))
          return rc;
      }
      continue;
    }
    long long G = kind == SG_ROW ? G_row : kind == SG_COL ? G_col : G_blk;
    long long N = kind == SG_ROW ? s.C : kind == SG_COL ? s.R : 1;
    if (jobs.n == SUM_JOBS_MAX) {
      if ((rc = launch_sum_partials_multi(jobs, kern->dtype, st))) return rc;
      jobs.n = 0;
    }
    jobs.part[jobs.n] = pr.p.part[i];
    jobs.out[jobs.n] = argbars[i].ptr;
    jobs.G[jobs.n] = G;
    jobs.N[jobs.n] = N;
    ++jobs.n;
  }
  // every broadcast operand's cotangent finalised in one launch
  if (jobs.n && (rc = launch_sum_partials_multi(jobs, kern->dtype, st))) return rc;
  return release(pr, st);
}

int sg_ew_check(sg_ctx* ctx, void* stream, int64_t* element, int32_t* site) {
  if (!ctx) return fail(SG_EINVAL, "null ctx");
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA_TRY(cudaStreamSynchronize(st));
  unsigned long long w = ~0ull;
  SG_CUDA_TRY(cudaMemcpy(&w, ctx->d_err, sizeof w, cudaMemcpyDeviceToHost));
  if (w == ~0ull) return SG_OK;
  SG_CUDA_TRY(cudaMemset(ctx->d_err, 0xff, sizeof(unsigned long long)));
  if (element) *element = (int64_t)(w >> 24);
  if (site) *site = (int32_t)(w & 0xffffff);
  return fail(SG_EDOMAIN, "element " + std::to_string((long long)(w >> 24)) + " failed at site " +
                              std::to_string((long long)(w & 0xffffff)));
}

int sg_domain_check(sg_ctx* ctx, void* stream, int32_t* flags) {
  if (!ctx) return fail(SG_EINVAL, "null ctx");
  if (int rc = ensure_context(ctx)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  SG_CUDA_TRY(cudaStreamSynchronize(st));
  unsigned w = 0;
  SG_CUDA_TRY(cudaMemcpy(&w, ctx->d_dom, sizeof w, cudaMemcpyDeviceToHost));
  if (flags) *flags = (int32_t)w;
  if (!w) return SG_OK;
  SG_CUDA_TRY(cudaMemset(ctx->d_dom, 0, sizeof(unsigned)));
  if (w & SG_DOM_EXP_OVERFLOW) return fail(SG_EDOMAIN, "math range error");
  if (w & SG_DOM_DIV_ZERO) return fail(SG_EDOMAIN, "division by zero");
  return fail(SG_EDOMAIN, "log of non-positive value 0.0");
}

int sg_reduce_to(sg_ctx* ctx, const sg_tensor* a, const sg_tensor* b, sg_tensor* out, void* stream) {
  SG_NVTX("sg_reduce_to");
  if (!ctx || !a || !out) return fail(SG_EINVAL, "null argument");
  if (a->dtype != SG_F32 && a->dtype != SG_F64) return fail(SG_EINVAL, "reduce_to computes in f32/f64");
  if (b && (b->dtype != a->dtype || b->ndim != a->ndim)) return fail(SG_EINVAL, "b must match a");
  if (b)
    for (int d = 0; d < a->ndim; ++d)
      if (b->shape[d] != a->shape[d]) return fail(SG_EINVAL, "b must match a");
  if (out->dtype != a->dtype) return fail(SG_EINVAL, "out dtype must match a");
  const int n = a->ndim;
  if (out->ndim > n) return fail(SG_EINVAL, "target rank exceeds source rank");
  // can_expand(out, a) (tensor.py:124-131)
  for (int j = 1; j <= out->ndim; ++j) {
    long long t = out->shape[out->ndim - j], s = a->shape[n - j];
    if (t != s && t != 1) return fail(SG_EINVAL, "target shape does not expand to the source");
  }
  DimMap kept{}, red{};
  long long stride = 1;
  std::vector<long long> strides(n);
  for (int d = n - 1; d >= 0; --d) {
    strides[d] = stride;
    stride *= a->shape[d];
  }
  long long n_out = 1, n_red = 1;
  for (int d = 0; d < n; ++d) {
    int pd = d - (n - out->ndim);
    long long t = pd >= 0 ? out->shape[pd] : 1;
    if (t == a->shape[d] && t != 1) {
      kept.ext[kept.nd] = a->shape[d];
      kept.stride[kept.nd++] = strides[d];
      n_out *= a->shape[d];
    } else if (a->shape[d] != 1) {
      red.ext[red.nd] = a->shape[d];
      red.stride[red.nd++] = strides[d];
      n_red *= a->shape[d];
    }
  }
  int rc = ensure_context(ctx);
  if (rc) return rc;
  return launch_reduce(a->ptr, b ? b->ptr : nullptr, out->ptr, n_out, n_red, kept, red, a->dtype,
                       (cudaStream_t)stream);
}

}  // extern "C"
