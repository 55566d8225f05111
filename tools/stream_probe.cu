// Streaming-pattern probe for the fused gradient kernel (K2) at the c2 size:
// 2 reads + 1 write of 2^28 fp32 (x, ybar -> xbar), with and without the
// per-column fp64 sums the ROW operands need.  Compares the access orders:
//   flat   : torch-like, one short block per 4096-element slab, linear sweep
//   span   : K2's layout (4 column groups x gy row spans, contiguous spans)
//   ilv    : persistent grid, row chunks interleaved over the grid (global sweep)
//   bulk   : persistent grid, cp.async.bulk (TMA 1-D) ring in shared memory
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe tools/stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr long long R = 1 << 16, C = 1 << 12;

__device__ __forceinline__ float dsig(float a, float x, float b, float yb, float& da, float& db) {
  float s = a * x + b;
  float y = 1.f / (1.f + __expf(-s));
  float d = y * (1.f - y) * yb;
  da = d * x;
  db = d;
  return d * a;
}

// ---------------- flat: torch-like
template <int U>
__global__ void __launch_bounds__(256) k_flat(const float4* x, const float4* yb, float4* xb, long long n4) {
  long long base = (long long)blockIdx.x * 256 * U + threadIdx.x;
  float4 xv[U], yv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    long long i = base + u * 256;
    if (i < n4) { xv[u] = x[i]; yv[u] = yb[i]; }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    long long i = base + u * 256;
    if (i < n4) {
      float da, db;
      float4 o;
      o.x = dsig(0.5f, xv[u].x, 0.1f, yv[u].x, da, db);
      o.y = dsig(0.5f, xv[u].y, 0.1f, yv[u].y, da, db);
      o.z = dsig(0.5f, xv[u].z, 0.1f, yv[u].z, da, db);
      o.w = dsig(0.5f, xv[u].w, 0.1f, yv[u].w, da, db);
      __stcs(xb + i, o);
    }
  }
}

// ---------------- row walkers with optional fp64 column sums (ROW a, b)
// MODE 0: contiguous spans of rpb rows per blockIdx.y; MODE 1: rows interleaved (stride gy)
// ACC 0: none, 1: fp64 smem sums per element, 2: fp32 sums over the U rows then fp64 smem
// ACC 3: fp32 Kahan sums in registers over the block's rows (no shared memory)
// MERGE > 0: the last of MERGE consecutive row blocks sums their partial rows
// (fixed order) into one group partial; the partials stay in L2.
template <int MODE, int ACC, int U, int MERGE = 0>
__global__ void __launch_bounds__(256, 4) k_rows(const float* x, const float* yb, float* xb, const float* a,
                                                 const float* b, double* part, long long rpb,
                                                 unsigned* cnt = nullptr, double* part2 = nullptr) {
  __shared__ double sacc[2 * 4 * 256];
  const int tx = threadIdx.x;
  const long long c = ((long long)blockIdx.x * 256 + tx) * 4;
  long long r0, stride, n;
  if (MODE == 0) {
    r0 = blockIdx.y * rpb;
    long long r1 = r0 + rpb < R ? r0 + rpb : R;
    stride = 1;
    n = r1 - r0;
  } else {
    r0 = blockIdx.y;
    stride = gridDim.y;
    n = (R - r0 + stride - 1) / stride;
  }
  const float4 av = *reinterpret_cast<const float4*>(a + c);
  const float4 bv = *reinterpret_cast<const float4*>(b + c);
  double* s = sacc + tx;
  if (ACC) for (int q = 0; q < 8; ++q) s[q * 256] = 0.0;
  float ks[8], kc[8];
  for (int q = 0; q < 8; ++q) ks[q] = kc[q] = 0.f;
  long long it = 0;
  for (; it + U <= n; it += U) {
    float4 xv[U], yv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long off = (r0 + (it + u) * stride) * C + c;
      xv[u] = *reinterpret_cast<const float4*>(x + off);
      yv[u] = *reinterpret_cast<const float4*>(yb + off);
    }
    float fa[4] = {0, 0, 0, 0}, fb[4] = {0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long off = (r0 + (it + u) * stride) * C + c;
      float4 o;
      float da[4], db[4];
      o.x = dsig(av.x, xv[u].x, bv.x, yv[u].x, da[0], db[0]);
      o.y = dsig(av.y, xv[u].y, bv.y, yv[u].y, da[1], db[1]);
      o.z = dsig(av.z, xv[u].z, bv.z, yv[u].z, da[2], db[2]);
      o.w = dsig(av.w, xv[u].w, bv.w, yv[u].w, da[3], db[3]);
      __stcs(reinterpret_cast<float4*>(xb + off), o);
      if (ACC == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          s[j * 256] += (double)da[j];
          s[(4 + j) * 256] += (double)db[j];
        }
      } else if (ACC == 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) { fa[j] += da[j]; fb[j] += db[j]; }
      } else if (ACC == 3) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float v = j < 4 ? da[j] : db[j - 4];
          float yk = v - kc[j];
          float t = ks[j] + yk;
          kc[j] = (t - ks[j]) - yk;
          ks[j] = t;
        }
      }
    }
    if (ACC == 2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s[j * 256] += (double)fa[j];
        s[(4 + j) * 256] += (double)fb[j];
      }
    }
  }
  for (; it < n; ++it) {
    long long off = (r0 + it * stride) * C + c;
    float4 xv = *reinterpret_cast<const float4*>(x + off);
    float4 yv = *reinterpret_cast<const float4*>(yb + off);
    float4 o;
    float da[4], db[4];
    o.x = dsig(av.x, xv.x, bv.x, yv.x, da[0], db[0]);
    o.y = dsig(av.y, xv.y, bv.y, yv.y, da[1], db[1]);
    o.z = dsig(av.z, xv.z, bv.z, yv.z, da[2], db[2]);
    o.w = dsig(av.w, xv.w, bv.w, yv.w, da[3], db[3]);
    __stcs(reinterpret_cast<float4*>(xb + off), o);
    if (ACC)
      for (int j = 0; j < 4; ++j) { s[j * 256] += (double)da[j]; s[(4 + j) * 256] += (double)db[j]; }
  }
  if (ACC == 3)
    for (int q = 0; q < 8; ++q) s[q * 256] += (double)ks[q] - (double)kc[q];
  if (ACC) {
    long long g = blockIdx.y;
    for (int j = 0; j < 4; ++j) {
      part[g * C + c + j] = s[j * 256];
      part[(gridDim.y + g) * C + c + j] = s[(4 + j) * 256];
    }
  }
  if (MERGE > 0) {
    __shared__ unsigned last;
    __threadfence();
    __syncthreads();
    const unsigned grp = blockIdx.y / MERGE;
    if (threadIdx.x == 0) {
      unsigned* ctr = cnt + blockIdx.x * 4096 + grp;
      const unsigned want = min((unsigned)MERGE, gridDim.y - grp * MERGE);
      last = atomicAdd(ctr, 1u) == want - 1;
      if (last) *ctr = 0;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      const unsigned g0 = grp * MERGE, g1 = min(g0 + MERGE, gridDim.y);
      for (int j = 0; j < 4; ++j) {
        double sa = 0, sb = 0;
        for (unsigned g = g0; g < g1; ++g) {
          sa += __ldcg(part + g * C + c + j);
          sb += __ldcg(part + (gridDim.y + g) * C + c + j);
        }
        part2[grp * C + c + j] = sa;
        part2[(4096 + grp) * C + c + j] = sb;
      }
    }
  }
}

// ---------------- bulk: cp.async.bulk ring, 1 producer thread, 8 consumer warps
// A work item is RB rows x 1024 columns (4 KB per row) of x and ybar; items are
// interleaved over the persistent grid.
constexpr int RB = 2, ST = 4;
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(ph));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

template <int ACC>
__global__ void __launch_bounds__(288, 1) k_bulk(const float* x, const float* yb, float* xb, const float* a,
                                                 const float* b, double* part) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);  // [ST][2][RB][1024]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * 2 * RB * 4096);
  uint64_t* empty = full + ST;
  __shared__ double sacc[2 * 4 * 256];
  const int warp = threadIdx.x / 32;
  const long long items_per_cg = R / RB;  // per column group
  const int cg = blockIdx.x & 3;
  const long long slot = blockIdx.x >> 2, nslots = gridDim.x >> 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 8); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 8) {
    if ((threadIdx.x & 31) == 0) {
      int s = 0; unsigned ph = 0;
      for (long long item = slot; item < items_per_cg; item += nslots) {
        mbar_wait(empty + s, ph ^ 1);
        mbar_expect(full + s, 2 * RB * 4096);
        for (int r = 0; r < RB; ++r) {
          long long off = (item * RB + r) * C + cg * 1024;
          bulk_g2s(ring + ((s * 2 + 0) * RB + r) * 1024, x + off, 4096, full + s);
          bulk_g2s(ring + ((s * 2 + 1) * RB + r) * 1024, yb + off, 4096, full + s);
        }
        if (++s == ST) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  const int tx = threadIdx.x;
  const long long c = (long long)cg * 1024 + tx * 4;
  const float4 av = *reinterpret_cast<const float4*>(a + c);
  const float4 bv = *reinterpret_cast<const float4*>(b + c);
  double* sa = sacc + tx;
  if (ACC) for (int q = 0; q < 8; ++q) sa[q * 256] = 0.0;
  int s = 0; unsigned ph = 0;
  for (long long item = slot; item < items_per_cg; item += nslots) {
    mbar_wait(full + s, ph);
    float fa[4] = {0, 0, 0, 0}, fb[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      float4 xv = reinterpret_cast<const float4*>(ring + ((s * 2 + 0) * RB + r) * 1024)[tx];
      float4 yv = reinterpret_cast<const float4*>(ring + ((s * 2 + 1) * RB + r) * 1024)[tx];
      float4 o;
      float da[4], db[4];
      o.x = dsig(av.x, xv.x, bv.x, yv.x, da[0], db[0]);
      o.y = dsig(av.y, xv.y, bv.y, yv.y, da[1], db[1]);
      o.z = dsig(av.z, xv.z, bv.z, yv.z, da[2], db[2]);
      o.w = dsig(av.w, xv.w, bv.w, yv.w, da[3], db[3]);
      __stcs(reinterpret_cast<float4*>(xb + (item * RB + r) * C + c), o);
      for (int j = 0; j < 4; ++j) { fa[j] += da[j]; fb[j] += db[j]; }
    }
    __syncwarp();
    if ((tx & 31) == 0) mbar_arrive(empty + s);
    if (ACC) {
#pragma unroll
      for (int j = 0; j < 4; ++j) { sa[j * 256] += (double)fa[j]; sa[(4 + j) * 256] += (double)fb[j]; }
    }
    if (++s == ST) { s = 0; ph ^= 1; }
  }
  if (ACC) {
    for (int j = 0; j < 4; ++j) {
      part[slot * C + c + j] = sa[j * 256];
      part[(nslots + slot) * C + c + j] = sa[(4 + j) * 256];
    }
  }
}


// ---------------- dyn: per-warp dynamic chunk queue over 32 column strips of 128 columns
template <int U, int CH>
__global__ void __launch_bounds__(256, 4) k_dyn(const float* x, const float* yb, float* xb, const float* a,
                                                const float* b, double* part, unsigned* q) {
  __shared__ double sacc[2 * 4 * 256];
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 8 + threadIdx.x / 32;   // global warp
  const int strip = gw & 31, slot = gw >> 5;           // 32 strips
  const long long c = (long long)strip * 128 + lane * 4;
  const float4 av = *reinterpret_cast<const float4*>(a + c);
  const float4 bv = *reinterpret_cast<const float4*>(b + c);
  double* s = sacc + threadIdx.x;
  for (int qq = 0; qq < 8; ++qq) s[qq * 256] = 0.0;
  const unsigned nch = (unsigned)(R / CH);
  for (;;) {
    unsigned ch = 0;
    if (lane == 0) ch = atomicAdd(q + strip, 1u);
    ch = __shfl_sync(0xffffffffu, ch, 0);
    if (ch >= nch) break;
    const long long r0 = (long long)ch * CH;
    for (int it = 0; it < CH; it += U) {
      float4 xv[U], yv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long off = (r0 + it + u) * C + c;
        xv[u] = *reinterpret_cast<const float4*>(x + off);
        yv[u] = *reinterpret_cast<const float4*>(yb + off);
      }
      float fa[4] = {0, 0, 0, 0}, fb[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long off = (r0 + it + u) * C + c;
        float4 o;
        float da[4], db[4];
        o.x = dsig(av.x, xv[u].x, bv.x, yv[u].x, da[0], db[0]);
        o.y = dsig(av.y, xv[u].y, bv.y, yv[u].y, da[1], db[1]);
        o.z = dsig(av.z, xv[u].z, bv.z, yv[u].z, da[2], db[2]);
        o.w = dsig(av.w, xv[u].w, bv.w, yv[u].w, da[3], db[3]);
        __stcs(reinterpret_cast<float4*>(xb + off), o);
#pragma unroll
        for (int j = 0; j < 4; ++j) { fa[j] += da[j]; fb[j] += db[j]; }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) { s[j * 256] += (double)fa[j]; s[(4 + j) * 256] += (double)fb[j]; }
    }
  }
  for (int j = 0; j < 4; ++j) {
    part[(long long)slot * C + c + j] = s[j * 256];
    part[(long long)(4096 + slot) * C + c + j] = s[(4 + j) * 256];
  }
}


// ---------------- cpa: contiguous row spans, x / ybar rows staged by per-thread
// cp.async (16 B) into a D-deep shared-memory ring: bytes in flight without registers
template <int D, int ACC>
__global__ void __launch_bounds__(256) k_cpa(const float* x, const float* yb, float* xb, const float* a,
                                             const float* b, double* part, long long rpb) {
  extern __shared__ float4 ring[];  // [D][2][256]
  __shared__ double sacc[2 * 4 * 256];
  const int tx = threadIdx.x;
  const long long c = ((long long)blockIdx.x * 256 + tx) * 4;
  const long long r0 = blockIdx.y * rpb;
  const long long r1 = r0 + rpb < R ? r0 + rpb : R;
  const long long n = r1 - r0;
  const float4 av = *reinterpret_cast<const float4*>(a + c);
  const float4 bv = *reinterpret_cast<const float4*>(b + c);
  double* s = sacc + tx;
  if (ACC) for (int q = 0; q < 8; ++q) s[q * 256] = 0.0;
  auto issue = [&](long long i) {
    const int slot = (int)(i % D);
    const long long off = (r0 + i) * C + c;
    const unsigned dx = (unsigned)__cvta_generic_to_shared(&ring[(slot * 2 + 0) * 256 + tx]);
    const unsigned dy = (unsigned)__cvta_generic_to_shared(&ring[(slot * 2 + 1) * 256 + tx]);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dx), "l"(x + off) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dy), "l"(yb + off) : "memory");
  };
  for (int i = 0; i < D; ++i) {
    if (i < n) issue(i);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float fa[4] = {0, 0, 0, 0}, fb[4] = {0, 0, 0, 0};
  for (long long i = 0; i < n; ++i) {
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    const int slot = (int)(i % D);
    const float4 xv = ring[(slot * 2 + 0) * 256 + tx];
    const float4 yv = ring[(slot * 2 + 1) * 256 + tx];
    if (i + D < n) issue(i + D);
    asm volatile("cp.async.commit_group;" ::: "memory");
    float4 o;
    float da[4], db[4];
    o.x = dsig(av.x, xv.x, bv.x, yv.x, da[0], db[0]);
    o.y = dsig(av.y, xv.y, bv.y, yv.y, da[1], db[1]);
    o.z = dsig(av.z, xv.z, bv.z, yv.z, da[2], db[2]);
    o.w = dsig(av.w, xv.w, bv.w, yv.w, da[3], db[3]);
    __stcs(reinterpret_cast<float4*>(xb + (r0 + i) * C + c), o);
    if (ACC) {
#pragma unroll
      for (int j = 0; j < 4; ++j) { fa[j] += da[j]; fb[j] += db[j]; }
      if ((i & 1) == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) { s[j * 256] += (double)fa[j]; s[(4 + j) * 256] += (double)fb[j]; fa[j] = fb[j] = 0; }
      }
    }
  }
  if (ACC) {
#pragma unroll
    for (int j = 0; j < 4; ++j) { s[j * 256] += (double)fa[j]; s[(4 + j) * 256] += (double)fb[j]; }
    long long g = blockIdx.y;
    for (int j = 0; j < 4; ++j) {
      part[g * C + c + j] = s[j * 256];
      part[(gridDim.y + g) * C + c + j] = s[(4 + j) * 256];
    }
  }
}

template <class F>
float timeit(F f, int reps = 20) {
  for (int i = 0; i < 3; ++i) f();
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(e);
  CK(cudaEventSynchronize(e));
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  CK(cudaGetLastError());
  return ms / reps;
}

int main() {
  const long long n = R * C;
  float *x, *yb, *xb, *a, *b;
  double* part;
  CK(cudaMalloc(&x, n * 4));
  CK(cudaMalloc(&yb, n * 4));
  CK(cudaMalloc(&xb, n * 4));
  CK(cudaMalloc(&a, C * 4));
  CK(cudaMalloc(&b, C * 4));
  CK(cudaMalloc(&part, 2ll * 4096 * C * 8));
  CK(cudaMemset(x, 0, n * 4));
  CK(cudaMemset(yb, 0, n * 4));
  CK(cudaMemset(a, 0, C * 4));
  CK(cudaMemset(b, 0, C * 4));
  auto gbs = [&](float ms) { return 12.0 * n / (ms * 1e-3) / 1e9; };
  auto rep = [&](const char* name, float ms) { printf("%-40s %.4f ms %7.1f GB/s\n", name, ms, gbs(ms)); };
  rep("flat U=2", timeit([&] { k_flat<2><<<(unsigned)(n / 4 / 512), 256>>>((const float4*)x, (const float4*)yb, (float4*)xb, n / 4); }));
  rep("flat U=4", timeit([&] { k_flat<4><<<(unsigned)(n / 4 / 1024), 256>>>((const float4*)x, (const float4*)yb, (float4*)xb, n / 4); }));
  unsigned* cnt;
  double* part2;
  CK(cudaMalloc(&cnt, 4 * 4096 * 4));
  CK(cudaMemset(cnt, 0, 4 * 4096 * 4));
  CK(cudaMalloc(&part2, 2ll * 4096 * C * 8));
  for (int gy : {296, 592, 1184}) {
    long long rpb = (R + gy - 1) / gy;
    char nm[96];
#define RUN(ACC, U, M) \
    snprintf(nm, sizeof nm, "span gy=%d acc%d U%d merge%d", gy, ACC, U, M); \
    rep(nm, timeit([&] { k_rows<0, ACC, U, M><<<dim3(4, gy), 256>>>(x, yb, xb, a, b, part, rpb, cnt, part2); }));
    RUN(1, 3, 0) RUN(2, 2, 0)
#define CPA(D) \
    CK(cudaFuncSetAttribute(k_cpa<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, D * 8192)); \
    snprintf(nm, sizeof nm, "cpa gy=%d D%d acc1", gy, D); \
    rep(nm, timeit([&] { k_cpa<D, 1><<<dim3(4, gy), 256, D * 8192>>>(x, yb, xb, a, b, part, rpb); }));
    CPA(2) CPA(3) CPA(4) CPA(6) CPA(8)
  }
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned* q;
  CK(cudaMalloc(&q, 32 * 4));
#define DYN(U, CH) \
  { char nm[96]; snprintf(nm, sizeof nm, "dyn U%d chunk%d", U, CH); \
    rep(nm, timeit([&] { cudaMemsetAsync(q, 0, 128); k_dyn<U, CH><<<nsm * 4, 256>>>(x, yb, xb, a, b, part, q); })); }
  DYN(2, 16) DYN(2, 32) DYN(4, 16) DYN(4, 32) DYN(4, 64) DYN(3, 24) DYN(3, 48)
  return 0;
}
