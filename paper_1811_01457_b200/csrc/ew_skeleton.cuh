// Programmatic dependent launch (the runtime launches these kernels with
// programmatic stream serialisation): wait until the previous grid in the
// stream has completed and its memory is visible, then let the next grid's
// CTAs launch as soon as ours leave room (they wait in their own
// griddepcontrol.wait).  Both are no-ops without the launch attribute.
#define SG_PDL_BEGIN()                                        \
  do {                                                        \
    asm volatile("griddepcontrol.wait;" ::: "memory");        \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)
#define SG_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

// Fused elementwise kernel skeleton (K1 forward, K2 gradient, pack).
//
// Compiled at run time by NVRTC together with the code generated from the
// user's scalar IR function (codegen.py).  The host prepends:
//   typedef float|double T;  #define SG_K <k>  #define SG_KT max(k,1)
//   #define SG_VEC <1|2|4>   #define SG_KINDS {kind0, kind1, ...}
//   #define SG_BDX/SG_BDY    (block shape, threads along C / along R)
// and this file's kernels are instantiated for that combination.
//
// Layout: canonical 2-D grid out[R][C]; thread (tx, ty) of block (bx, by)
// owns SG_VEC consecutive columns c = (bx*SG_BDX + tx)*SG_VEC and walks rows
// r = by*rows_per_block + ty, ... with stride SG_BDY.  A thread therefore
// keeps the same columns for its whole life, which is what lets the
// gradient kernel accumulate broadcast-axis sums (ROW operands, e.g. the
// bias vector) in fp64 registers and write one deterministic partial per
// (row-thread, column); COL operands (shape (R,1)) are reduced across the
// columns of a row with warp shuffles.
//
// Reference semantics: element e of the output is f(args[e']) for the
// trailing-aligned broadcast of interp.py:322-332; the gradient writes
// reduce_like(ybar * d f/d arg_i, type_i) (forward_ad.py:226-235,
// rules.py:177-185) without materialising the (1+K)-row pack.

#ifndef SG_UNROLL
#define SG_UNROLL 4   // rows in flight per thread, forward
#endif
#ifndef SG_GUNROLL
#define SG_GUNROLL 3  // rows in flight per thread, gradient (the runtime sets it from the operand kinds)
#endif
#ifndef SG_RUNROLL
#define SG_RUNROLL 2  // column chunks in flight per lane, gradient row mode
#endif
#ifndef SG_GRAD_MINB
#define SG_GRAD_MINB 3  // blocks per SM the gradient kernel's register budget is sized for
#endif

struct D { T p; T t[SG_KT]; };

#if defined(SG_T_IS_DOUBLE)
__device__ __forceinline__ T sg_exp(T x) { return exp(x); }
__device__ __forceinline__ T sg_log(T x) { return log(x); }
__device__ __forceinline__ T sg_tanh(T x) { return tanh(x); }
#else
__device__ __forceinline__ T sg_exp(T x) { return expf(x); }
__device__ __forceinline__ T sg_log(T x) { return logf(x); }
__device__ __forceinline__ T sg_tanh(T x) { return tanhf(x); }
#endif

// ---- vector access helpers (SG_VEC * sizeof(T) is 4, 8 or 16 bytes)
#if defined(SG_T_IS_DOUBLE)
#if SG_VEC == 2
typedef double2 SgRaw;
#else
typedef double SgRaw;
#endif
#else
#if SG_VEC == 4
typedef float4 SgRaw;
#elif SG_VEC == 2
typedef float2 SgRaw;
#else
typedef float SgRaw;
#endif
#endif

struct __align__(sizeof(SgRaw)) VT { T v[SG_VEC]; };

__device__ __forceinline__ VT sg_from_raw(const SgRaw& w) {
  static_assert(sizeof(SgRaw) == sizeof(VT), "vector width");
  return *reinterpret_cast<const VT*>(&w);
}
__device__ __forceinline__ SgRaw sg_to_raw(const VT& v) { return *reinterpret_cast<const SgRaw*>(&v); }
// operands read once per element.  Plain loads measured faster than
// evict-first (.cs) ones on B200 (+2-3% on K2); stores stay evict-first.
#ifndef SG_LD_CS
#define SG_LD_CS 0
#endif
#ifndef SG_ST_CS
#define SG_ST_CS 1
#endif
__device__ __forceinline__ VT sg_ldv_stream(const T* p) {
#if SG_LD_CS
  return sg_from_raw(__ldcs(reinterpret_cast<const SgRaw*>(p)));
#else
  return sg_from_raw(*reinterpret_cast<const SgRaw*>(p));
#endif
}
// broadcast vectors (bias-like, re-read by every row): cached loads
__device__ __forceinline__ VT sg_ldv(const T* p) {
  return sg_from_raw(__ldg(reinterpret_cast<const SgRaw*>(p)));
}
__device__ __forceinline__ void sg_stv(T* p, const VT& v) {
#if SG_ST_CS
  __stcs(reinterpret_cast<SgRaw*>(p), sg_to_raw(v));
#else
  *reinterpret_cast<SgRaw*>(p) = sg_to_raw(v);
#endif
}

__device__ __forceinline__ void sg_publish_error(unsigned long long* err, long long elem, int site) {
  unsigned long long w = ((unsigned long long)elem << 24) | (unsigned long long)(site & 0xffffff);
  atomicMin(err, w);
}

static __device__ const int sg_kinds[SG_KT] = SG_KINDS;

// Row-invariant operands (ROW vectors, one-element tensors, by-value scalars)
// are loaded once per thread: a thread keeps its columns for its lifetime.
__device__ __forceinline__ void sg_load_invariant(const SgEwParams& p, long long c, T (&inv)[SG_KT][SG_VEC]) {
#pragma unroll
  for (int i = 0; i < SG_K; ++i) {
    const int kind = sg_kinds[i];
    const T* base = reinterpret_cast<const T*>(p.in[i]);
    if (kind == SG_ROW) {
      VT v = sg_ldv(base + c);
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) inv[i][j] = v.v[j];
    } else if (kind == SG_SPTR || kind == SG_SVAL) {
      const T s = kind == SG_SPTR ? base[0] : (T)p.sval[i];
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) inv[i][j] = s;
    }
  }
}

// Per-row operands (FULL rows, COL scalars) for row r; invariants copied in.
__device__ __forceinline__ void sg_load_row(const SgEwParams& p, long long r, long long c,
                                            const T (&inv)[SG_KT][SG_VEC], T (&x)[SG_KT][SG_VEC]) {
#pragma unroll
  for (int i = 0; i < SG_K; ++i) {
    const int kind = sg_kinds[i];
    const T* base = reinterpret_cast<const T*>(p.in[i]);
    if (kind == SG_FULL) {
      VT v = sg_ldv_stream(base + r * p.C + c);
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) x[i][j] = v.v[j];
    } else if (kind == SG_COL) {
      const T s = __ldg(base + r);
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) x[i][j] = s;
    } else {
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) x[i][j] = inv[i][j];
    }
  }
}

__device__ __forceinline__ long long sg_row_begin(const SgEwParams& p, long long by) {
  return by * p.rows_per_block;
}
__device__ __forceinline__ long long sg_row_end(const SgEwParams& p, long long by) {
  long long e = (by + 1) * p.rows_per_block;
  return e < p.R ? e : p.R;
}
// Row walk of thread (by, ty): r = base + it * stride, it in [0, n).
// SG_ROW_IL 0 (default): each block owns the contiguous span [r0, r1);
// 1: rows interleaved over the whole grid (base = by*BDY + ty, stride =
// gy*BDY).  Measured on B200 (tools/ew_sweep4.sh): contiguous spans stream
// faster for both kernels once the forward grid is large.
#ifndef SG_ROW_IL
#define SG_ROW_IL 0
#endif
struct SgRows {
  long long base, stride, n;
};
__device__ __forceinline__ SgRows sg_rows(const SgEwParams& p, int ty, long long by) {
  SgRows w;
#if SG_ROW_IL
  w.base = by * SG_BDY + ty;
  w.stride = (long long)gridDim.y * SG_BDY;
  w.n = p.R > w.base ? (p.R - w.base + w.stride - 1) / w.stride : 0;
#else
  const long long r0 = sg_row_begin(p, by), r1 = sg_row_end(p, by);
  w.base = r0 + ty;
  w.stride = SG_BDY;
  w.n = r1 > w.base ? (r1 - w.base + SG_BDY - 1) / SG_BDY : 0;
#endif
  return w;
}
// SG_GRAD_REV 1: the gradient kernel walks the row spans last-to-first, to
// start on the rows the forward kernel finished with (still in L2).  Measured
// 1.5 % SLOWER in the c2 step on B200 (tools/c2_ab.sh; the forward's dirty
// output lines are written back under it), so off by default.
#ifndef SG_GRAD_REV
#define SG_GRAD_REV 0
#endif
__device__ __forceinline__ long long sg_grad_span() {
  return SG_GRAD_REV ? (long long)(gridDim.y - 1 - blockIdx.y) : (long long)blockIdx.y;
}

__device__ __forceinline__ void sg_primal_row(const SgEwParams& p, long long r, long long c,
                                              const T (&x)[SG_KT][SG_VEC], T* out) {
  VT y;
#pragma unroll
  for (int j = 0; j < SG_VEC; ++j) {
    T a[SG_KT];
#pragma unroll
    for (int i = 0; i < SG_KT; ++i) a[i] = (i < SG_K) ? x[i][j] : (T)0;
    int err = 0;
    long long steps = p.step_limit;
    sg_entry_p(a, y.v[j], err, steps);
    if (err) sg_publish_error(p.err, r * p.C + c + j, err);
  }
  sg_stv(out + r * p.C + c, y);
}

// --------------------------------------------------------------- K1: forward
#ifndef SG_FLAT
#define SG_FLAT 0
#endif
#if SG_FLAT
// Flat walk (torch-like): each block covers 256 * SG_UNROLL consecutive
// vectors of the output, so the whole grid sweeps memory in address order;
// broadcast operands are re-read per vector (L1 hits).
__device__ __forceinline__ void sg_load_elem(const SgEwParams& p, long long r, long long c, T (&x)[SG_KT][SG_VEC]) {
#pragma unroll
  for (int i = 0; i < SG_K; ++i) {
    const int kind = sg_kinds[i];
    const T* base = reinterpret_cast<const T*>(p.in[i]);
    if (kind == SG_FULL || kind == SG_ROW) {
      const VT v = kind == SG_FULL ? sg_ldv_stream(base + r * p.C + c) : sg_ldv(base + c);
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) x[i][j] = v.v[j];
    } else {
      const T s = kind == SG_COL ? __ldg(base + r) : (kind == SG_SPTR ? base[0] : (T)p.sval[i]);
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) x[i][j] = s;
    }
  }
}
extern "C" __global__ void __launch_bounds__(256)
sg_ew_forward(const SgEwParams p) {
  SG_PDL_WAIT();  // multi-wave grid: no early trigger
  const long long nvec = p.R * p.C / SG_VEC;
  const long long v0 = (long long)blockIdx.x * (256 * SG_UNROLL) + threadIdx.x;
  T* out = reinterpret_cast<T*>(p.out);
  T xs[SG_UNROLL][SG_KT][SG_VEC];
  long long rr[SG_UNROLL], cc[SG_UNROLL];
#pragma unroll
  for (int u = 0; u < SG_UNROLL; ++u) {
    const long long e = (v0 + u * 256) * SG_VEC;
    rr[u] = p.c_log2 >= 0 ? e >> p.c_log2 : e / p.C;
    cc[u] = e - rr[u] * p.C;
    if (v0 + u * 256 < nvec) sg_load_elem(p, rr[u], cc[u], xs[u]);
  }
#pragma unroll
  for (int u = 0; u < SG_UNROLL; ++u)
    if (v0 + u * 256 < nvec) sg_primal_row(p, rr[u], cc[u], xs[u], out);
}
#else
// SG_FWD_MINB: optional blocks-per-SM register budget (default: none, the
// compiler's choice -- an explicit 1 relaxes it to more registers)
#ifdef SG_FWD_MINB
extern "C" __global__ void __launch_bounds__(SG_BDX * SG_BDY, SG_FWD_MINB)
#else
extern "C" __global__ void __launch_bounds__(SG_BDX * SG_BDY)
#endif
sg_ew_forward(const SgEwParams p) {
  SG_PDL_BEGIN();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long c = ((long long)blockIdx.x * SG_BDX + tx) * SG_VEC;
  if (c >= p.C) return;
  const SgRows w = sg_rows(p, ty, blockIdx.y);
  const long long n = w.n;
  T* out = reinterpret_cast<T*>(p.out);
  T inv[SG_KT][SG_VEC];
  sg_load_invariant(p, c, inv);
  long long it = 0;
  for (; it + SG_UNROLL <= n; it += SG_UNROLL) {  // full chunks: all loads issued first
    T xs[SG_UNROLL][SG_KT][SG_VEC];
#pragma unroll
    for (int u = 0; u < SG_UNROLL; ++u) sg_load_row(p, w.base + (it + u) * w.stride, c, inv, xs[u]);
#pragma unroll
    for (int u = 0; u < SG_UNROLL; ++u) sg_primal_row(p, w.base + (it + u) * w.stride, c, xs[u], out);
  }
  for (; it < n; ++it) {
    T xs[SG_KT][SG_VEC];
    const long long r = w.base + it * w.stride;
    sg_load_row(p, r, c, inv, xs);
    sg_primal_row(p, r, c, xs, out);
  }
}

#endif

// ------------------------------------------------------ K2: fused gradient
// Recomputes the duals from the inputs, writes xbar for full operands and
// fp64 partial sums for broadcast operands.  Partial layouts:
//   SG_ROW:              part[(by*SG_BDY + ty) * C + c]      (G_row = gy*SG_BDY rows)
//   SG_COL:              part[g * R + r], g = lane-group column id
//   SG_SPTR / SG_SVAL:   part[by * gx + bx]                  (block partial)
// SG_ROW_SMEM 1 (default): the per-column fp64 sums of ROW operands live in
// shared memory (this thread's own slots) instead of registers -- frees 16
// registers under the 64-register budget for a third row of loads in flight
// (+2 % on c2, +9 % for cheaper sub-functions; tools/ew_sweep5.sh).
#ifndef SG_ROW_SMEM
#define SG_ROW_SMEM 1
#endif
#if !SG_HAS_ROW
#undef SG_ROW_SMEM
#define SG_ROW_SMEM 0
#endif
struct SgGradAcc {
#if SG_ROW_SMEM
  double* srow;               // srow[(i * SG_VEC + j) * SG_BDX * SG_BDY]
#else
  double row[SG_KT][SG_VEC];  // ROW operands: per-column sums over my rows
#endif
  double s[SG_KT];            // scalar operands
};
#if SG_ROW_SMEM
#define SG_ACC_ROW(acc, i, j) (acc).srow[((i) * SG_VEC + (j)) * (SG_BDX * SG_BDY)]
#else
#define SG_ACC_ROW(acc, i, j) (acc).row[i][j]
#endif

// One row: duals, ybar contraction, xbar stores.  Contributions to ROW and
// scalar operands are added into pre[i][j] (type T, registers) and flushed
// into the fp64 sums by sg_flush_pre once per group of SG_GUNROLL rows: one
// fp64 conversion + shared-memory update per group instead of per element.
// (f32: the group sum adds at most (SG_GUNROLL-1) * 2^-24 * sum|terms| of
// error, far inside the 1e-6 * sum|terms| tolerance.)  Returns the per-row
// sums for COL operands in colsum.
__device__ __forceinline__ void sg_grad_row(const SgEwParams& p, long long r, long long c,
                                            const T (&x)[SG_KT][SG_VEC], const VT& yb, T (&pre)[SG_KT][SG_VEC],
                                            double (&colsum)[SG_KT]) {
  VT y, g[SG_KT];
#pragma unroll
  for (int j = 0; j < SG_VEC; ++j) {
    T a[SG_KT], d[SG_KT];
#pragma unroll
    for (int i = 0; i < SG_KT; ++i) a[i] = (i < SG_K) ? x[i][j] : (T)0;
    int err = 0;
    long long steps = p.step_limit;
    sg_entry_d(a, y.v[j], d, err, steps);
    if (err) sg_publish_error(p.err, r * p.C + c + j, err);
#pragma unroll
    for (int i = 0; i < SG_K; ++i) {
      const T contrib = yb.v[j] * d[i];  // ybar .* partial_i (forward_ad.py:233)
      const int kind = sg_kinds[i];
      if (kind == SG_FULL) g[i].v[j] = contrib;
      else if (kind == SG_COL) colsum[i] += (double)contrib;
      else pre[i][j] += contrib;
    }
  }
  if (p.out) sg_stv(reinterpret_cast<T*>(p.out) + r * p.C + c, y);
#pragma unroll
  for (int i = 0; i < SG_K; ++i)
    if (sg_kinds[i] == SG_FULL) sg_stv(reinterpret_cast<T*>(p.xbar[i]) + r * p.C + c, g[i]);
}

__device__ __forceinline__ void sg_zero_pre(T (&pre)[SG_KT][SG_VEC]) {
#pragma unroll
  for (int i = 0; i < SG_KT; ++i)
#pragma unroll
    for (int j = 0; j < SG_VEC; ++j) pre[i][j] = (T)0;
}

__device__ __forceinline__ void sg_flush_pre(SgGradAcc& acc, T (&pre)[SG_KT][SG_VEC]) {
#pragma unroll
  for (int i = 0; i < SG_K; ++i) {
    const int kind = sg_kinds[i];
    if (kind == SG_ROW) {
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) SG_ACC_ROW(acc, i, j) += (double)pre[i][j];
    } else if (kind == SG_SPTR || kind == SG_SVAL) {
#pragma unroll
      for (int j = 0; j < SG_VEC; ++j) acc.s[i] += (double)pre[i][j];
    }
  }
  sg_zero_pre(pre);
}

extern "C" __global__ void __launch_bounds__(SG_BDX * SG_BDY, SG_GRAD_MINB)
sg_ew_grad(const SgEwParams p) {
  SG_PDL_BEGIN();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long c = ((long long)blockIdx.x * SG_BDX + tx) * SG_VEC;
  const bool active = c < p.C;
  const SgRows w = sg_rows(p, ty, sg_grad_span());
  const T* ybar = reinterpret_cast<const T*>(p.ybar);

  SgGradAcc acc;
#if SG_ROW_SMEM
  __shared__ double sg_srow[SG_KT * SG_VEC * SG_BDX * SG_BDY];
  acc.srow = sg_srow + ty * SG_BDX + tx;
#endif
#pragma unroll
  for (int i = 0; i < SG_KT; ++i) {
    acc.s[i] = 0.0;
#pragma unroll
    for (int j = 0; j < SG_VEC; ++j) SG_ACC_ROW(acc, i, j) = 0.0;
  }
  T pre[SG_KT][SG_VEC];
  sg_zero_pre(pre);
  T inv[SG_KT][SG_VEC];
  if (active || SG_ROWMODE) sg_load_invariant(p, SG_ROWMODE ? 0 : c, inv);  // row mode: scalars only

#if SG_ROWMODE
  // one warp per row, lanes walk the columns: COL cotangents accumulate in a
  // register over the whole row, one warp reduction per row, written final
  // (part[i][r], a single partial group).  ROW operands never take this path.
  {
    const int lane = tx % 32, wib = tx / 32;
    const int warps = (SG_BDX * SG_BDY) / 32;
    const long long rstride = (long long)gridDim.y * warps;
    constexpr long long CSTEP = 32ll * SG_VEC;
    for (long long r = (long long)blockIdx.y * warps + wib; r < p.R; r += rstride) {
      double colsum[SG_KT];
#pragma unroll
      for (int i = 0; i < SG_KT; ++i) colsum[i] = 0.0;
      long long c0 = (long long)lane * SG_VEC;
      for (; c0 + (SG_RUNROLL - 1) * CSTEP < p.C; c0 += SG_RUNROLL * CSTEP) {
        T xs[SG_RUNROLL][SG_KT][SG_VEC];
        VT yb[SG_RUNROLL];
#pragma unroll
        for (int u = 0; u < SG_RUNROLL; ++u) {
          sg_load_row(p, r, c0 + u * CSTEP, inv, xs[u]);
          yb[u] = sg_ldv_stream(ybar + r * p.C + c0 + u * CSTEP);
        }
#pragma unroll
        for (int u = 0; u < SG_RUNROLL; ++u) sg_grad_row(p, r, c0 + u * CSTEP, xs[u], yb[u], pre, colsum);
        sg_flush_pre(acc, pre);
      }
      for (; c0 < p.C; c0 += CSTEP) {
        T xs[SG_KT][SG_VEC];
        sg_load_row(p, r, c0, inv, xs);
        const VT yb = sg_ldv_stream(ybar + r * p.C + c0);
        sg_grad_row(p, r, c0, xs, yb, pre, colsum);
        sg_flush_pre(acc, pre);
      }
#pragma unroll
      for (int i = 0; i < SG_K; ++i) {
        if (sg_kinds[i] != SG_COL) continue;
        double sum = colsum[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off);
        if (lane == 0) p.part[i][r] = sum;
      }
    }
  }
#elif !SG_HAS_COL
  // no cross-thread work per row: full chunks with all loads issued first
  if (active) {
    const long long n = w.n;
    double colsum[SG_KT];
    long long it = 0;
    for (; it + SG_GUNROLL <= n; it += SG_GUNROLL) {
      T xs[SG_GUNROLL][SG_KT][SG_VEC];
      VT yb[SG_GUNROLL];
#pragma unroll
      for (int u = 0; u < SG_GUNROLL; ++u) {
        const long long r = w.base + (it + u) * w.stride;
        sg_load_row(p, r, c, inv, xs[u]);
        yb[u] = sg_ldv_stream(ybar + r * p.C + c);
      }
#pragma unroll
      for (int u = 0; u < SG_GUNROLL; ++u)
        sg_grad_row(p, w.base + (it + u) * w.stride, c, xs[u], yb[u], pre, colsum);
      sg_flush_pre(acc, pre);
    }
    for (; it < n; ++it) {
      const long long r = w.base + it * w.stride;
      T xs[SG_KT][SG_VEC];
      sg_load_row(p, r, c, inv, xs);
      VT yb = sg_ldv_stream(ybar + r * p.C + c);
      sg_grad_row(p, r, c, xs, yb, pre, colsum);
    }
    sg_flush_pre(acc, pre);
  }
#else
  // COL operands reduce across the lanes sharing a row: every lane of a
  // group must take the same trip count, so walk the block's row span
  constexpr int kGroup = SG_BDX >= 32 ? 32 : SG_BDX;
  // the block-uniform trip count: the longest walk of any ty in the block
  const long long rows_span = sg_rows(p, 0, sg_grad_span()).n;
  const long long gi = ((long long)blockIdx.x * SG_BDX + tx) / kGroup;
  // SG_GUNROLL rows per trip: every row's loads are issued before the first
  // row is computed (the trip count stays block-uniform for the shuffles)
  for (long long it = 0; it < rows_span; it += SG_GUNROLL) {
    T xs[SG_GUNROLL][SG_KT][SG_VEC];
    VT yb[SG_GUNROLL];
#pragma unroll
    for (int u = 0; u < SG_GUNROLL; ++u) {
      const long long r = w.base + (it + u) * w.stride;
      if (active && it + u < w.n) {
        sg_load_row(p, r, c, inv, xs[u]);
        yb[u] = sg_ldv_stream(ybar + r * p.C + c);
      }
    }
#pragma unroll
    for (int u = 0; u < SG_GUNROLL; ++u) {
      if (it + u >= rows_span) break;  // block-uniform
      const long long r = w.base + (it + u) * w.stride;
      const bool live = active && it + u < w.n;
      double colsum[SG_KT];
#pragma unroll
      for (int i = 0; i < SG_KT; ++i) colsum[i] = 0.0;
      if (live) sg_grad_row(p, r, c, xs[u], yb[u], pre, colsum);
#pragma unroll
      for (int i = 0; i < SG_K; ++i) {
        if (sg_kinds[i] != SG_COL) continue;
        double sum = colsum[i];
#pragma unroll
        for (int off = kGroup / 2; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off, kGroup);
        if (live && (tx % kGroup) == 0) p.part[i][gi * p.R + r] = sum;
      }
    }
    sg_flush_pre(acc, pre);
  }
#endif
  // ROW partials: one row of partials per row-thread
#pragma unroll
  for (int i = 0; i < SG_K; ++i) {
    if (sg_kinds[i] != SG_ROW || !active) continue;
    const long long gi = (long long)blockIdx.y * SG_BDY + ty;
#pragma unroll
    for (int j = 0; j < SG_VEC; ++j) p.part[i][gi * p.C + c + j] = SG_ACC_ROW(acc, i, j);
  }
  // scalar partials: block tree reduction in a fixed order
  __shared__ double red[SG_BDX * SG_BDY];
  const int tid = ty * SG_BDX + tx;
#pragma unroll
  for (int i = 0; i < SG_K; ++i) {
    if (sg_kinds[i] != SG_SPTR && sg_kinds[i] != SG_SVAL) continue;
    red[tid] = (active || SG_ROWMODE) ? acc.s[i] : 0.0;
    __syncthreads();
    for (int s = (SG_BDX * SG_BDY) / 2; s > 0; s >>= 1) {
      if (tid < s) red[tid] += red[tid + s];
      __syncthreads();
    }
    if (tid == 0) p.part[i][(long long)blockIdx.y * gridDim.x + blockIdx.x] = red[0];
    __syncthreads();
  }
}

// ------------------------------------------------------------------- pack
// fused_pack layout of interp.py:334-352: pack[0] = primal, pack[1+i] = d f/d arg_i.
extern "C" __global__ void __launch_bounds__(SG_BDX * SG_BDY)
sg_ew_pack(const SgEwParams p) {
  SG_PDL_BEGIN();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long c = ((long long)blockIdx.x * SG_BDX + tx) * SG_VEC;
  if (c >= p.C) return;
  const SgRows w = sg_rows(p, ty, blockIdx.y);
  const long long plane = p.R * p.C;
  T* pk = reinterpret_cast<T*>(p.pack);
  T inv[SG_KT][SG_VEC];
  sg_load_invariant(p, c, inv);
  for (long long it = 0; it < w.n; ++it) {
    const long long r = w.base + it * w.stride;
    T xs[SG_KT][SG_VEC];
    sg_load_row(p, r, c, inv, xs);
    VT y, g[SG_KT];
#pragma unroll
    for (int j = 0; j < SG_VEC; ++j) {
      T a[SG_KT], d[SG_KT];
#pragma unroll
      for (int i = 0; i < SG_KT; ++i) a[i] = (i < SG_K) ? xs[i][j] : (T)0;
      int err = 0;
      long long steps = p.step_limit;
      sg_entry_d(a, y.v[j], d, err, steps);
      if (err) sg_publish_error(p.err, r * p.C + c + j, err);
#pragma unroll
      for (int i = 0; i < SG_KT; ++i) g[i].v[j] = d[i];
    }
    sg_stv(pk + r * p.C + c, y);
#pragma unroll
    for (int i = 0; i < SG_K; ++i) sg_stv(pk + (long long)(1 + i) * plane + r * p.C + c, g[i]);
  }
}
