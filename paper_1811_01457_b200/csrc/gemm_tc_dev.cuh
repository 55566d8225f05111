// Device-side building blocks of the tcgen05 GEMMs (PTX wrappers, tile
// raster, fused epilogue), shared by the single-GEMM kernels (gemm_tc.cu)
// and the persistent GEMM-chain kernel (gemm_chain.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.h"
#include "gemm.h"

namespace sg {
namespace tc {

constexpr int BM = 128;           // UMMA M (cta_group::1)
// A k-block is one 128-byte swizzle row of K: 64 bf16 or 32 fp32 (TF32)
// elements; one UMMA_K step is 32 bytes of K (16 bf16 / 8 TF32).  Stage
// bytes per k-block are therefore the same for both operand types.
template <bool TF32> struct Elem {
  static constexpr int BK = TF32 ? 32 : 64;
  static constexpr int UMMA_K = TF32 ? 8 : 16;
  static constexpr int KSTEPS = BK / UMMA_K;          // 4
  static constexpr uint32_t MN_CHUNK = BK * 128;      // MN-major: EPR x BK box bytes (= LBO)
  static constexpr uint32_t MN_KSTEP = UMMA_K * 128;  // MN-major: next UMMA_K K-rows
  // MN-major 32-bit operands only exist in the 128B swizzle with 32-byte
  // atoms (layout type 1, TMA SWIZZLE_128B_ATOM_32B): 4-row swizzle groups,
  // so the K-direction group stride (SBO) is 512 B instead of 1024 B.
  static constexpr uint32_t MN_SBO = TF32 ? 512 : 1024;
  static constexpr uint32_t MN_LAYOUT = TF32 ? 1 : 2;
};
constexpr int ROW_BYTES = 128;
constexpr int NUM_THREADS = 384;  // 12 warps: TMA, MMA, TMEM, idle, 8 epilogue
constexpr int EPI_WARP0 = 4;
constexpr int EPI_WARPS = 8;      // two per TMEM lane quadrant, each takes half the columns

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Accumulator hand-back: only the TMEM reads must be ordered before it
// (tcgen05.fence::before_thread_sync), not the epilogue's global stores.
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
// non-blocking: has the barrier completed the phase with this parity?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// Operand maps are 3-D {row, rows, batch}: c2 is the batch index (0 for a plain GEMM).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// PDL (griddepcontrol): wait = the prerequisite grid has completed and its
// memory is visible (a no-op without a programmatic dependency);
// launch_dependents = the next kernel in the stream may start its prologue.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
template <bool TF32>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  if (TF32)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread t of warp q gets lane 32q+t
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, 128B swizzle (layout type 2), sm_100 version bit.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// Instruction descriptor: fp32 accumulate (bit 4), A/B format at bits 7/10
// (kind::f16: 1 = bf16; kind::tf32: 2 = tf32), operand majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_tc(int M, int N, bool a_mn, bool b_mn, bool tf32) {
  return (1u << 4) | ((tf32 ? 2u : 1u) << 7) | ((tf32 ? 2u : 1u) << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------------- epilogue
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Epilogue math runs per output element on 8 warps while the tensor cores
// work on the next tile, so it uses the SFU approximations (rel. error
// ~2^-11, below the bf16 rounding of the stored activations).
__device__ __forceinline__ float act_fwd(float z, int act) {
  switch (act) {
    case SG_ACT_SIGMOID: return __fdividef(1.0f, 1.0f + __expf(-z));  // tensor.py:214-215
    case SG_ACT_TANH: return tanh_fast(z);
    case SG_ACT_RELU: return z > 0.0f ? z : 0.0f;
    default: return z;
  }
}
// d act / d z expressed through the saved output h (rules.py:82-94)
__device__ __forceinline__ float act_grad_from_out(float h, int act) {
  switch (act) {
    case SG_ACT_SIGMOID: return h * (1.0f - h);
    case SG_ACT_TANH: return 1.0f - h * h;
    case SG_ACT_RELU: return h > 0.0f ? 1.0f : 0.0f;
    default: return 1.0f;
  }
}

// The activation is uniform per launch: branch once per 32-element chunk,
// not per element (a per-element switch compiles to an indirect branch).
__device__ __forceinline__ void act_fwd_chunk(float (&v)[32], int act) {
  if (act == SG_ACT_SIGMOID) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __fdividef(1.0f, 1.0f + __expf(-v[i]));
  } else if (act == SG_ACT_TANH) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = tanh_fast(v[i]);
  } else if (act == SG_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = v[i] > 0.0f ? v[i] : 0.0f;
  }
}
// Packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2 on sm_100): two lanes of
// work per instruction with the same per-element roundings as the scalar
// forms (an FFMA2 rounds each half like an FFMA).  SG_EPI_SCALAR_MATH=1
// compiles the scalar forms.
#ifndef SG_EPI_SCALAR_MATH
#define SG_EPI_SCALAR_MATH 0
#endif
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ void act_grad_chunk(float (&v)[32], const float (&h)[32], int act) {
#if !SG_EPI_SCALAR_MATH
  if (act == SG_ACT_SIGMOID) {  // v * (h * (1 - h)), the scalar form's three roundings
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 hh = f2(h[i], h[i + 1]);
      const float2 t = __fmul2_rn(hh, __fadd2_rn(f2(1.0f, 1.0f), f2(-h[i], -h[i + 1])));
      const float2 r = __fmul2_rn(f2(v[i], v[i + 1]), t);
      v[i] = r.x, v[i + 1] = r.y;
    }
    return;
  }
  if (act == SG_ACT_TANH) {  // v * fma(-h, h, 1): the contracted scalar form
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float2 t = __ffma2_rn(f2(-h[i], -h[i + 1]), f2(h[i], h[i + 1]), f2(1.0f, 1.0f));
      const float2 r = __fmul2_rn(f2(v[i], v[i + 1]), t);
      v[i] = r.x, v[i + 1] = r.y;
    }
    return;
  }
#endif
  if (act == SG_ACT_SIGMOID) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= h[i] * (1.0f - h[i]);
  } else if (act == SG_ACT_TANH) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= 1.0f - h[i] * h[i];
  } else if (act == SG_ACT_RELU) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = h[i] > 0.0f ? v[i] : 0.0f * v[i];
  }
}

// Tile timeline trace (tools only: built with -DSGB200_GEMM_TRACE into a
// separate library, tools/gemm_trace.py): per CTA and tile iteration, the
// %globaltimer of MMA start, accumulator complete (epilogue wake-up) and
// epilogue end.  Compiled out of the product library.
// Launches are numbered on the device (g_trace_seq: read after the grid
// dependency wait, advanced by the last CTA to finish), so back-to-back and
// graph-replayed launches each get their own region:
//   g_trace[((seq * 148 + cta) * iters + it) * 4 + slot], slot 0..3 as above.
#ifdef SGB200_GEMM_TRACE
__device__ unsigned long long* g_trace = nullptr;
__device__ int g_trace_iters = 0, g_trace_launches = 0;
__device__ unsigned g_trace_seq = 0, g_trace_done = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SG_TRACE(it, slot)                                                                                 \
  do {                                                                                                     \
    if (g_trace && (it) < g_trace_iters && trace_seq < (unsigned)g_trace_launches)                          \
      g_trace[(((long long)trace_seq * 148 + blockIdx.x) * g_trace_iters + (it)) * 4 + (slot)] = gtimer(); \
  } while (0)
#define SG_TRACE_BEGIN() const unsigned trace_seq = *(volatile unsigned*)&g_trace_seq
#define SG_TRACE_END()                                                      \
  do {                                                                      \
    if (threadIdx.x == 0) {                                                 \
      __threadfence();                                                      \
      if (atomicAdd(&g_trace_done, 1u) == gridDim.x - 1) {                  \
        g_trace_done = 0;                                                   \
        atomicAdd(&g_trace_seq, 1u);                                        \
      }                                                                     \
    }                                                                       \
  } while (0)
#else
#define SG_TRACE(it, slot) \
  do {                     \
  } while (0)
#define SG_TRACE_BEGIN() \
  do {                   \
  } while (0)
#define SG_TRACE_END() \
  do {                 \
  } while (0)
#endif

// Epilogue stage profile (trace builds only): cycles spent per stage of a
// 32 x 32 chunk, summed over the lane-0 threads of the first 8 CTAs.
#ifdef SGB200_GEMM_TRACE
__device__ unsigned long long g_cprof[8];
__constant__ int g_cprof_on = 0;  // constant cache: the check adds no global-load latency
#define SG_CPROF_START() long long cprof_t = clock64()
#define SG_CPROF(k)                                                                  \
  do {                                                                               \
    if (g_cprof_on && blockIdx.x < 8 && (threadIdx.x & 31) == 0) {                   \
      const long long now = clock64();                                               \
      atomicAdd(&g_cprof[k], (unsigned long long)(now - cprof_t));                   \
      cprof_t = now;                                                                 \
    }                                                                                \
  } while (0)
#else
#define SG_CPROF_START() \
  do {                   \
  } while (0)
#define SG_CPROF(k) \
  do {              \
  } while (0)
#endif

struct TileCoord {
  int m0, n0;
};
__device__ __forceinline__ TileCoord tile_of(int t, int m_tiles, int n_tiles, int bn) {
  // grouped raster: 8 M-tiles per group so consecutive CTAs share B tiles in L2
  constexpr int G = 8;
  const int per_group = G * n_tiles;
  const int group = t / per_group;
  const int first_m = group * G;
  const int gsize = min(m_tiles - first_m, G);
  const int in_group = t - group * per_group;
  TileCoord c;
  c.m0 = (first_m + in_group % gsize) * BM;
  c.n0 = (in_group / gsize) * bn;
  return c;
}

struct KParams {
  int M, N, K;
  GemmEpilogue epi;
  int splits;         // split-K factor (>= 1); splits > 1 writes raw fp32 partials
  int kb_per_split;   // k-blocks per split
  float* part;        // [splits][M][ld_part] when splits > 1
  long long ld_part;
  int tma_lp, tma_f32;  // outputs written through smem staging + TMA bulk stores
  int aux_stage;        // 1: ACT_GRAD bf16 aux streamed by TMA into the upper half of each staging slot;
                        // 2: BIAS_MSE fp32 targets, 4 KB blocks in the wide slot's upper half
  int raster;           // CTA-pair kernel: M-tiles per raster group
  int tail_split;       // CTA-pair kernel, > 0: tiles are taken row-major; the last tail_split tiles are
  int tail_full;        //   computed as two K-halves each, reduce-added into the zeroed fp32 output
  int batch;            // independent GEMMs (bmm lanes), >= 1
  long long so_f32, so_lp;  // batch strides of out_f32 / out_bf16 (elements)
  int tma_o2 = 0;           // BIAS_ACT_SEED: out2 through TMA (its map in the fp32 output's slot)
  // CTA-pair kernel, splits > 1: per (tile, epilogue-warp region) arrival
  // counters (zeroed) -- the last split to arrive sums the partials in split
  // order and writes the output (no separate reduce launch)
  unsigned* split_cnt = nullptr;
  // optional bias-gradient finalize run by the epilogue warps after their
  // tiles: fin_out[j] = sum_g fin_part[g][j] (the k_colsum_finalize order)
  const float* fin_part = nullptr;
  long long fin_G = 0, fin_ld = 0, fin_N = 0;
  float* fin_out = nullptr;
};

// ----------------------------------------------------- TMA-store epilogue
// Each epilogue warp owns a 1024-byte aligned staging slot.  A 32x32 chunk is
// written row-per-lane in the TMA swizzled layout (conflict-free 16-byte
// stores) and one lane issues a bulk tensor store, so the global writes are
// fully coalesced and asynchronous.
//   narrow slot (4 KB): one staging buffer; the ACT_GRAD aux block in its
//     upper 2 KB, one chunk ahead;
//   wide slot (8 KB, WIDE kernels): two staging buffers used alternately, so
//     a chunk is staged while the previous chunk's store still reads its
//     buffer; for bf16 outputs [stage0 2K | stage1 2K | aux0 2K | aux1 2K]
//     with the aux blocks streamed two chunks ahead, for fp32 outputs
//     [stage0 4K | stage1 4K].
constexpr int STAGE_SLOT = 4096;
constexpr int STAGE_SLOT_WIDE = 8192;
template <bool WIDE> struct Slot {
  static constexpr int BYTES = WIDE ? STAGE_SLOT_WIDE : STAGE_SLOT;
};
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// bulk tensor store with fp32 add into global memory (the split tail tiles)
__device__ __forceinline__ void tma_store_add_3d(const CUtensorMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// bf16 rows are 64 B: SWIZZLE_64B puts 16-byte chunk c of row r at c ^ ((r >> 1) & 3)
__device__ __forceinline__ void stage_bf16(uint8_t* slot, const float (&v)[32], int lane) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * c + 2 * j], v[8 * c + 2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(slot + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
// fp32 rows are 128 B: SWIZZLE_128B puts chunk c of row r at c ^ (r & 7)
__device__ __forceinline__ void stage_f32(uint8_t* slot, const float (&v)[32], int lane) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(slot + lane * 128 + ((c ^ (lane & 7)) << 4)) =
        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}
// warp-collective: stage one chunk and bulk-store it at (n0, row0).
// `alt`: the buffer was last used two stores ago (wide slots), so only the
// older of the (at most two) outstanding stores must have read it out.
template <bool BF16>
__device__ __forceinline__ void warp_tma_store(uint8_t* slot, const CUtensorMap* map, const float (&v)[32], int lane,
                                               int n0, int row0, int bidx, bool add = false, bool alt = false) {
  if (lane == 0) {
    if (alt) bulk_wait_read1();
    else bulk_wait_read0();  // the slot's previous store has been read out
  }
  __syncwarp();
  if (BF16) stage_bf16(slot, v, lane);
  else stage_f32(slot, v, lane);
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    if (add) tma_store_add_3d(map, slot, n0, row0, bidx);
    else tma_store_3d(map, slot, n0, row0, bidx);
    bulk_commit();
  }
}

// ACT_GRAD saved activations through TMA: a 32 x 32 bf16 block (SWIZZLE_64B,
// the layout stage_bf16 writes) lands in the upper 2 KB of the warp's
// staging slot, so the next chunk's block is in flight while this one is
// processed (and the tile's first block while the accumulator is computed).
constexpr int AUX_OFF = 2048;
__device__ __forceinline__ void aux_issue(uint8_t* slot, const CUtensorMap* map, uint64_t* bar, int n0, int row0,
                                          uint32_t bytes = 2048) {
  mbar_expect_tx(bar, bytes);
  tma_load_3d(slot + AUX_OFF, map, bar, n0, row0, 0);
}
__device__ __forceinline__ void aux_read(const uint8_t* slot, float (&h)[32], int lane) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 w = *reinterpret_cast<const uint4*>(slot + AUX_OFF + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4));
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(b[j]);
      h[8 * c + 2 * j] = f.x;
      h[8 * c + 2 * j + 1] = f.y;
    }
  }
}

// Wide slots: aux buffer b of the warp's slot, addressed like the narrow
// layout's (slot + AUX_OFF), so aux_issue / aux_read take the returned base.
__device__ __forceinline__ uint8_t* aux_base_wide(uint8_t* slot, int b) { return slot + 4096 + 2048 * b - AUX_OFF; }
// Wide slots: staging buffer b of the warp's slot.
template <bool BF16>
__device__ __forceinline__ uint8_t* stage_buf(uint8_t* slot, int b) {
  return slot + b * (BF16 ? 2048 : 4096);
}

// One 32x32 accumulator chunk (row m per lane, columns n0..n0+31) through the
// fused epilogue.  `grp` is the 32-row group (bias-gradient partial row),
// `grp_ok` whether that group has any row < M.  Warp-collective (shuffles).
// BIAS_MSE targets staged in shared memory (aux_stage == 2): the block of
// this chunk (shared-window address, 0: not staged) and what to issue into
// the buffer once it has been read.  Passed by value (registers).
struct YStage {
  uint32_t sm;    // smem address of the 4 KB block (aux_base_wide(slot, 0) + AUX_OFF)
  uint8_t* base;  // aux_base_wide(slot, 0), for aux_issue
  const CUtensorMap* map;
  uint64_t* bar;
  int next_n0;  // < 0: no next block
  int row0;
};
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "r"(a));
  return r;
}

template <bool WIDE = false>
__device__ __forceinline__ void epi_chunk(const KParams& p, float (&v)[32], int m, bool row_ok, int grp,
                                          bool grp_ok, int n0, int lane, int split, int bidx, bool hstaged,
                                          const float (&hs)[32], uint8_t* slot, bool radd,
                                          const CUtensorMap* map_lp, const CUtensorMap* map_f32,
                                          int* next_buf = nullptr, YStage ys = YStage{}) {
  SG_CPROF_START();
  const GemmEpilogue& e = p.epi;
  const bool full = n0 + 32 <= p.N;
  const int nn = full ? 32 : p.N - n0;
  if (p.splits > 1) {  // split-K: raw fp32 partial of this K range
    if (row_ok) store_row_f32(p.part + ((long long)split * p.M + m) * p.ld_part + n0, v, nn);
    return;
  }
  if (!grp_ok) return;  // the whole 32-row group is past M (warp-uniform)
  bool ovf = false;      // domain flag of this lane's row (the vote below runs converged)
  if (!row_ok) {
    // rows past M: zeros for the column sums; TMA clips them on store
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.0f;
  } else if (e.mode == SG_EPI_BIAS_ACT || e.mode == SG_EPI_BIAS_ACT_SEED || e.mode == SG_EPI_BIAS_MSE) {
    if (e.bias) {
      float bv[32];
      if (full && (reinterpret_cast<uintptr_t>(e.bias + n0) & 15) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(e.bias + n0 + i));
          bv[i] = b4.x, bv[i + 1] = b4.y, bv[i + 2] = b4.z, bv[i + 3] = b4.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) bv[i] = n0 + i < p.N ? __ldg(e.bias + n0 + i) : 0.0f;
      }
#if !SG_EPI_SCALAR_MATH
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float2 r = __fadd2_rn(f2(v[i], v[i + 1]), f2(bv[i], bv[i + 1]));
        v[i] = r.x, v[i + 1] = r.y;
      }
#else
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += bv[i];
#endif
      SG_CPROF(6);  // bias loaded and added
    }
    if (e.out_pre) store_row_f32(e.out_pre + (long long)m * e.ld_pre + n0, v, nn);
    if (e.act == SG_ACT_SIGMOID) {
      // the reference's scalar_sigmoid computes math.exp(-z): OverflowError for
      // z < -709.78 (tensor.py:214-215); flagged, the value below is still 0
#pragma unroll
      for (int i = 0; i < 32; ++i) ovf |= v[i] <= SIGMOID_OVF_F32;
    }
    act_fwd_chunk(v, e.act);
  } else if (e.mode == SG_EPI_ACT_GRAD) {
    if (hstaged) {
      act_grad_chunk(v, hs, e.act);
    } else {
      float h[32];
      if (e.aux_f32) load_row_f32(e.aux_f32 + (long long)m * e.ld_aux + n0, h, nn);
      else load_row_bf16(e.aux + (long long)m * e.ld_aux + n0, h, nn);
      act_grad_chunk(v, h, e.act);
    }
  }
  if ((e.mode == SG_EPI_BIAS_ACT || e.mode == SG_EPI_BIAS_ACT_SEED) && e.act == SG_ACT_SIGMOID &&
      e.dom) {  // warp-uniform
    if (__any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(e.dom, (unsigned)SG_DOM_EXP_OVERFLOW);
  }
  SG_CPROF(2);  // epilogue math
  const int row0 = m - lane;
  // wide slots alternate the two buffers from store to store (*next_buf: the
  // one not holding the newest outstanding store) -- unless the chunk stores
  // twice (fp32 and bf16 through TMA): those serialise on buffer 0
  const bool alt = WIDE && !(e.out_f32 && p.tma_f32 && e.out_bf16 && p.tma_lp);
  const int nb = WIDE ? *next_buf : 0;
  uint8_t* sbuf32 = alt ? stage_buf<false>(slot, nb) : slot;
  uint8_t* sbuf16 = alt ? stage_buf<true>(slot, nb) : slot;
  if (WIDE && ((e.out_f32 && p.tma_f32) || (e.out_bf16 && p.tma_lp))) *next_buf = alt ? nb ^ 1 : 1;
  if (e.out_f32) {
    if (radd) {  // split tail tile: add this K-half into the zeroed output (two terms: order-free)
      if (p.tma_f32) warp_tma_store<false>(sbuf32, map_f32, v, lane, n0, row0, bidx, true, alt);
      else if (row_ok) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nn) atomicAdd(e.out_f32 + (long long)m * e.ld_f32 + n0 + i, v[i]);
      }
    } else if (p.tma_f32) {
      warp_tma_store<false>(sbuf32, map_f32, v, lane, n0, row0, bidx, false, alt);
    } else if (row_ok) {
      store_row_f32(e.out_f32 + bidx * p.so_f32 + (long long)m * e.ld_f32 + n0, v, nn);
    }
  }
  if (e.out_bf16) {
    if (p.tma_lp) warp_tma_store<true>(sbuf16, map_lp, v, lane, n0, row0, bidx, false, alt);
    else if (row_ok) store_row_bf16(e.out_bf16 + bidx * p.so_lp + (long long)m * e.ld_bf16 + n0, v, nn);
  }
  if (e.mode == SG_EPI_BIAS_MSE) {
    // the MSE loss of the linear top layer (k_mse's arithmetic): d = z - y,
    // loss += d^2, dz = d scale + d scale
    // (rules.py:53-58 on mul(d, d)).  Targets: the TMA-staged block, else
    // this lane's row from global memory -- 4 at a time, so no second
    // 32-float row is live beside the accumulator.
    const float* yrow = e.seed + (long long)m * e.ld_seed + n0;
    const bool yvec = full && (reinterpret_cast<uintptr_t>(yrow) & 15) == 0;
    // loss: fp32 within the 32 x 32 block (a pairwise tree: sums of 8 per
    // lane, then the warp butterfly), fp64 across blocks (sg_sum_f64) --
    // fp64 arithmetic here would sit on the epilogue's critical path
    float l = 0.0f, l8 = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float4 y;
      if (ys.sm) {  // SWIZZLE_128B: chunk c of row `lane` at c ^ (lane & 7)
        y = lds_f4(ys.sm + lane * 128 + ((c ^ (lane & 7)) << 4));
      } else if (row_ok && yvec) {
        y = __ldg(reinterpret_cast<const float4*>(yrow + 4 * c));
      } else {
        y.x = row_ok && 4 * c < nn ? __ldg(yrow + 4 * c) : 0.0f;
        y.y = row_ok && 4 * c + 1 < nn ? __ldg(yrow + 4 * c + 1) : 0.0f;
        y.z = row_ok && 4 * c + 2 < nn ? __ldg(yrow + 4 * c + 2) : 0.0f;
        y.w = row_ok && 4 * c + 3 < nn ? __ldg(yrow + 4 * c + 3) : 0.0f;
      }
      const float yy[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = 4 * c + k;
        const float d = (row_ok && i < nn) ? v[i] - yy[k] : 0.0f;
        l8 += d * d;
        v[i] = d * e.loss_scale + d * e.loss_scale;
      }
      if (c & 1) {
        l += l8;
        l8 = 0.0f;
      }
    }
    SG_CPROF(5);  // targets read, dz formed
    if (ys.sm) {  // the block is read: the buffer takes the next one
#ifndef SG_NO_AUX_FENCE
      fence_proxy_async();
#endif
      __syncwarp();
      if (lane == 0 && ys.next_n0 >= 0) aux_issue(ys.base, ys.map, ys.bar, ys.next_n0, ys.row0, 4096);
    }
    SG_CPROF(6);  // next block issued
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) e.loss_part[(long long)grp * ((p.N + 31) / 32) + n0 / 32] = (double)l * (double)e.loss_scale;
    SG_CPROF(7);  // loss partial reduced and stored
    if (p.tma_o2) {
      warp_tma_store<true>(slot, map_f32, v, lane, n0, row0, bidx);
      if (WIDE) *next_buf = 1;
    } else if (row_ok) {
      store_row_bf16(e.out2_bf16 + (long long)m * e.ld_out2 + n0, v, nn);
    }
  }
  if (e.mode == SG_EPI_BIAS_ACT_SEED) {
    // the activation's cotangent: dz = seed .* act'(h) with h the bf16
    // activation just stored (the value the pullback reads back otherwise)
    float sd[32];
    if (ys.sm) {  // the TMA-staged seed block (SWIZZLE_128B: chunk c of row `lane` at c ^ (lane & 7))
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 y = lds_f4(ys.sm + lane * 128 + ((c ^ (lane & 7)) << 4));
        sd[4 * c] = y.x, sd[4 * c + 1] = y.y, sd[4 * c + 2] = y.z, sd[4 * c + 3] = y.w;
      }
#ifndef SG_NO_AUX_FENCE
      fence_proxy_async();
#endif
      __syncwarp();
      if (lane == 0 && ys.next_n0 >= 0) aux_issue(ys.base, ys.map, ys.bar, ys.next_n0, ys.row0, 4096);
      if (!row_ok)
#pragma unroll
        for (int i = 0; i < 32; ++i) sd[i] = 0.0f;
    } else if (row_ok) {
      load_row_f32(e.seed + (long long)m * e.ld_seed + n0, sd, nn);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) sd[i] = 0.0f;
    }
    if (e.out_bf16)  // the bf16 activation as stored (TF32: the fp32 one as it is)
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __bfloat162float(__float2bfloat16_rn(v[i]));
    act_grad_chunk(sd, v, e.act);  // sd *= act'(h)
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = sd[i];
    // (the fp32 output slot is free in this mode: it carries out2's map)
    if (p.tma_o2) {
      warp_tma_store<true>(slot, map_f32, v, lane, n0, row0, bidx);  // buffer 0, after every read of it
      if (WIDE) *next_buf = 1;
    } else if (row_ok) {
      if (e.out2_f32) store_row_f32(e.out2_f32 + (long long)m * e.ld_out2 + n0, v, nn);
      else store_row_bf16(e.out2_bf16 + (long long)m * e.ld_out2 + n0, v, nn);
    }
  }
  SG_CPROF(3);  // stores issued
  // bias gradient: per-32-row column sums (rules.py:45-46 reduce_like); the
  // transpose-reduce destroys v, so it runs after the stores
  if (e.colsum) warp_colsum_store(v, e.colsum + (long long)grp * e.ld_colsum + n0, lane, nn);
  SG_CPROF(4);  // column sums
}


// ===================================================== 2-SM (CTA pair) variant
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x 256 tile.
// Each CTA stages 128 rows of A and 128 rows (half the N extent) of B per
// k-block (32 KB, 6-deep ring); the leader CTA issues tcgen05.mma with
// M = 256 and the tensor cores read both CTAs' shared memory; each CTA's
// TMEM holds its 128 rows of the fp32 accumulator.  Half the smem operand
// traffic per SM and 2/3 of the L2->SM bytes per FLOP of the 1-SM kernel.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  // relaxed: the accumulator hand-back only needs the preceding tcgen05 fence,
  // not the epilogue's global stores to be acknowledged
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* m, uint32_t leader_bar, int c0,
                                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
template <bool TF32>
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  if (TF32)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // arrive on the barrier in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}


// ------------------------------------------- split-K fix-up and finalize
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// Split-K: this epilogue warp stored its 32 x (chunks*32) fp32 partial of one
// split of a tile; the last of the tile's splits to arrive for this region
// sums all of them in ascending split order (k_splitk_reduce's order) and
// writes the output.  `counter` is the region's arrival counter (reset here
// by the last arriver).  Returns whether this warp finished the region.
__device__ __forceinline__ bool split_region_fixup(const KParams& p, unsigned* counter, int row0, int n_first,
                                                   int chunks, int lane) {
  __syncwarp();
  unsigned last = 0;
  if (lane == 0) {
    const unsigned old = atom_add_acq_rel_gpu(counter, 1u);
    last = old == (unsigned)(p.splits - 1);
    if (last) *counter = 0;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return false;
  __threadfence();
  // rows of the region one at a time, the warp's lanes across its columns
  // (4 per lane, coalesced 16-byte loads); every split's partial of a row is
  // loaded before it is summed in ascending split order
  const GemmEpilogue& e = p.epi;
  const int n = n_first + lane * 4;
  const int nn = min(4, p.N - n);
  const int cols = chunks * 32;
  if (lane * 4 >= cols || nn <= 0) return true;
  const bool vec_out = e.out_f32 && (reinterpret_cast<uintptr_t>(e.out_f32) & 15) == 0 && (e.ld_f32 & 3) == 0;
  constexpr int R = 4;
  for (int r0 = 0; r0 < 32; r0 += R) {
    float4 acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < p.splits; ++s) {
      float4 f[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int m = row0 + r0 + r;
        f[r] = m < p.M ? __ldcg(reinterpret_cast<const float4*>(p.part + ((long long)s * p.M + m) * p.ld_part + n))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (s == 0) {
          acc[r] = f[r];
        } else {
          acc[r].x += f[r].x, acc[r].y += f[r].y, acc[r].z += f[r].z, acc[r].w += f[r].w;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int m = row0 + r0 + r;
      if (m >= p.M) break;
      const float a[4] = {acc[r].x, acc[r].y, acc[r].z, acc[r].w};
      if (e.out_f32) {
        float* dst = e.out_f32 + (long long)m * e.ld_f32 + n;
        if (nn == 4 && vec_out) *reinterpret_cast<float4*>(dst) = acc[r];
        else
          for (int i = 0; i < nn; ++i) dst[i] = a[i];
      }
      if (e.out_bf16)
        for (int i = 0; i < nn; ++i) e.out_bf16[(long long)m * e.ld_bf16 + n + i] = __float2bfloat16_rn(a[i]);
    }
  }
  return true;
}

// Bias-gradient finalize as the epilogue warps' tail job (after their tiles):
// columns j = cta, cta + ctas, ...; for each, 128 threads fold the partial
// rows g = t, t + 128, ... in fp64 and a fixed tree combines them -- the
// arithmetic of k_colsum_finalize, so the result is bit-identical to it.
// `red` is 2 x 128 doubles of shared memory only the epilogue warps use
// (tid = 0..255 over the 8 epilogue warps; named barrier 1).
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void colsum_finalize_tail(const KParams& p, double* red, int tid, int cta, int ctas) {
  const int half = tid >> 7, t = tid & 127;
  for (long long j0 = (long long)cta * 2; j0 < p.fin_N; j0 += 2ll * ctas) {
    const long long j = j0 + half;
    double acc = 0.0;
    if (j < p.fin_N) {
#pragma unroll 4
      for (long long g = t; g < p.fin_G; g += 128) acc += (double)p.fin_part[g * p.fin_ld + j];
    }
    red[half * 128 + t] = acc;
    epi_bar();
    for (int s = 64; s > 0; s >>= 1) {
      if (t < s) red[half * 128 + t] += red[half * 128 + t + s];
      epi_bar();
    }
    if (t == 0 && j < p.fin_N) p.fin_out[j] = (float)red[half * 128];
    epi_bar();
  }
}

// ----------------------------------------------- pair-tile epilogue loop
// The chunks of one 256-wide pair tile for epilogue warp (q, half): TMEM ->
// epi_chunk, with the ACT_GRAD saved-activation blocks streamed by TMA one
// (narrow slots) or two (wide slots) chunks ahead.  epi_aux_prologue issues
// the first block(s) before the accumulator wait; aux_phase holds one
// parity bit per aux buffer.
template <bool WIDE>
__device__ __forceinline__ void epi_aux_prologue(bool staged, int lane, uint8_t* slot, const CUtensorMap* map_aux,
                                                 uint64_t* aux_bars, int n_first, int nch, int N, int row0,
                                                 bool y32 = false) {
  if (!staged || lane != 0) return;
  if (WIDE && y32) {  // one 4 KB fp32 buffer (the slot's upper half), one chunk ahead
    if (n_first < N) aux_issue(aux_base_wide(slot, 0), map_aux, &aux_bars[0], n_first, row0, 4096);
    return;
  }
  if (n_first < N) aux_issue(WIDE ? aux_base_wide(slot, 0) : slot, map_aux, &aux_bars[0], n_first, row0);
  if (WIDE && nch > 1 && n_first + 32 < N) aux_issue(aux_base_wide(slot, 1), map_aux, &aux_bars[1], n_first + 32, row0);
}

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// `after0` runs once the first chunk's stores are issued (the GEMM chain
// publishes the previous unit's rows there, its stores long landed).
template <bool WIDE, class After0 = NoHook>
__device__ __forceinline__ void epi_chunks(const KParams& p, uint32_t tmem_row, int n_first, int c_first, int nch,
                                           int row0, int lane, int split, int bidx, bool radd, uint8_t* slot,
                                           bool staged, const CUtensorMap* map_aux, uint64_t* aux_bars,
                                           uint32_t& aux_phase, const CUtensorMap* map_lp,
                                           const CUtensorMap* map_f32, int& next_buf, After0 after0 = After0{}) {
  const int m = row0 + lane;
  const bool row_ok = m < p.M;
#pragma unroll 1
  for (int j = 0; j < nch; ++j) {
    const int n0 = n_first + j * 32;
    float v[32];
    SG_CPROF_START();
    tmem_ld32(tmem_row + (c_first + j) * 32, v);
    SG_CPROF(0);  // TMEM load
    if (n0 >= p.N) continue;  // warp-uniform; later chunks are past N as well
    float h[32];
    const bool y32 = WIDE && staged && p.aux_stage == 2;  // fp32 targets (warp-uniform)
    YStage ys{};
    if (y32) {  // the epilogue reads the block itself and re-issues the buffer
      mbar_wait(&aux_bars[0], aux_phase & 1);
      aux_phase ^= 1u;
      SG_CPROF(1);
      uint8_t* base = aux_base_wide(slot, 0);
      ys = {smem_u32(base + AUX_OFF), base, map_aux, &aux_bars[0], (j + 1 < nch && n0 + 32 < p.N) ? n0 + 32 : -1,
            row0};
    } else if (staged) {
      const int b = WIDE ? (j & 1) : 0;
      mbar_wait(&aux_bars[b], (aux_phase >> b) & 1);
      aux_phase ^= 1u << b;
      SG_CPROF(1);  // saved activation block arrived
      uint8_t* base = WIDE ? aux_base_wide(slot, b) : slot;
      aux_read(base, h, lane);
#ifndef SG_NO_AUX_FENCE
      fence_proxy_async();  // our reads precede the next async write of the buffer
#endif
      __syncwarp();
      const int ahead = WIDE ? 2 : 1;
      if (lane == 0 && j + ahead < nch && n0 + 32 * ahead < p.N)
        aux_issue(base, map_aux, &aux_bars[b], n0 + 32 * ahead, row0);
    }
    epi_chunk<WIDE>(p, v, m, row_ok, row0 >> 5, row0 < p.M, n0, lane, split, bidx, staged && !y32, h, slot, radd,
                    map_lp, map_f32, &next_buf, ys);
    if (j == 0) after0();
  }
}

}  // namespace tc

// Host-side tensor-map builders (gemm_tc.cu), shared with the chain planner.
namespace tcmap {
int make_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long ld, int box_outer,
             bool tf32, bool mn_major, int batch, long long sbatch);
bool make_out_map(CUtensorMap* map, const void* ptr, bool bf16, long long N, long long M, long long ld, int batch,
                  long long sbatch);
void aux_map(const GemmArgs& g, tc::KParams& p, CUtensorMap& m, bool wide);
void out_maps(const GemmArgs& g, tc::KParams& p, CUtensorMap& mlp, CUtensorMap& mf32);
}  // namespace tcmap

}  // namespace sg
