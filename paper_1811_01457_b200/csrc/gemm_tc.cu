// K3/K4/K5: Dense-layer GEMMs on the 5th-generation tensor cores (sm_100a).
//
//   D[M,N] = sum_k A[m,k] * B[n,k]      (bf16 inputs, fp32 accumulation in TMEM)
//
// Reference: the Dense layer's forward `matmul(h, transpose(W))`
// (nn_train.py:192-193, tensor.py:351-361) and its adjoints
// `matmul(ybar, transpose(v))`, `matmul(transpose(a), ybar)` (rules.py:113-115).
// Each operand is either K-major (row-major [rows][K]) or MN-major
// (row-major [K][rows]), so all three products of a Dense layer run without
// materialised transposes:
//   forward  Z  = X  . W^T : A = X  [B][in]  K-major,  B = W [out][in] K-major
//   backward dX = dZ . W   : A = dZ [B][out] K-major,  B = W [out][in] MN-major
//   backward dW = dZ^T . X : A = dZ [B][out] MN-major, B = X [B][in]   MN-major
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: 128B-swizzled A/B tiles -> smem ring (STAGES deep)
//   warp 1      MMA issuer:   one elected lane issues tcgen05.mma (M=128, N=BN,
//                             K=16) into a double-buffered TMEM accumulator
//   warp 2      TMEM allocator
//   warps 4..7  epilogue:     tcgen05.ld -> registers -> fused bias/activation/
//                             activation-derivative -> global stores, while the
//                             MMA warp already works on the next tile
// Synchronisation is mbarrier-only: full/empty per smem stage (TMA tx-count and
// tcgen05.commit), full/empty per accumulator buffer.
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
__device__ __forceinline__ void act_grad_chunk(float (&v)[32], const float (&h)[32], int act) {
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
  int aux_stage;        // ACT_GRAD bf16 aux streamed by TMA into the upper half of each staging slot
  int raster;           // CTA-pair kernel: M-tiles per raster group
  int tail_split;       // CTA-pair kernel, > 0: tiles are taken row-major; the last tail_split tiles are
  int tail_full;        //   computed as two K-halves each, reduce-added into the zeroed fp32 output
  int batch;            // independent GEMMs (bmm lanes), >= 1
  long long so_f32, so_lp;  // batch strides of out_f32 / out_bf16 (elements)
};

// ----------------------------------------------------- TMA-store epilogue
// Each epilogue warp owns a 4 KB, 1024-byte aligned staging slot.  A 32x32
// chunk is written row-per-lane in the TMA swizzled layout (conflict-free
// 16-byte stores) and one lane issues a bulk tensor store, so the global
// writes are fully coalesced and asynchronous.
constexpr int STAGE_SLOT = 4096;
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
// warp-collective: stage one chunk and bulk-store it at (n0, row0)
template <bool BF16>
__device__ __forceinline__ void warp_tma_store(uint8_t* slot, const CUtensorMap* map, const float (&v)[32], int lane,
                                               int n0, int row0, int bidx, bool add = false) {
  if (lane == 0) bulk_wait_read0();  // the slot's previous store has been read out
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
__device__ __forceinline__ void aux_issue(uint8_t* slot, const CUtensorMap* map, uint64_t* bar, int n0, int row0) {
  mbar_expect_tx(bar, 2048);
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

// One 32x32 accumulator chunk (row m per lane, columns n0..n0+31) through the
// fused epilogue.  `grp` is the 32-row group (bias-gradient partial row),
// `grp_ok` whether that group has any row < M.  Warp-collective (shuffles).
__device__ __forceinline__ void epi_chunk(const KParams& p, float (&v)[32], int m, bool row_ok, int grp,
                                          bool grp_ok, int n0, int lane, int split, int bidx, bool hstaged,
                                          const float (&hs)[32], uint8_t* slot, bool radd,
                                          const CUtensorMap* map_lp, const CUtensorMap* map_f32) {
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
  } else if (e.mode == SG_EPI_BIAS_ACT) {
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
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += bv[i];
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
  if (e.mode == SG_EPI_BIAS_ACT && e.act == SG_ACT_SIGMOID && e.dom) {  // warp-uniform
    if (__any_sync(0xffffffffu, ovf) && lane == 0) atomicOr(e.dom, (unsigned)SG_DOM_EXP_OVERFLOW);
  }
  const int row0 = m - lane;
  if (e.out_f32) {
    if (radd) {  // split tail tile: add this K-half into the zeroed output (two terms: order-free)
      if (p.tma_f32) warp_tma_store<false>(slot, map_f32, v, lane, n0, row0, bidx, true);
      else if (row_ok) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nn) atomicAdd(e.out_f32 + (long long)m * e.ld_f32 + n0 + i, v[i]);
      }
    } else if (p.tma_f32) {
      warp_tma_store<false>(slot, map_f32, v, lane, n0, row0, bidx);
    } else if (row_ok) {
      store_row_f32(e.out_f32 + bidx * p.so_f32 + (long long)m * e.ld_f32 + n0, v, nn);
    }
  }
  if (e.out_bf16) {
    if (p.tma_lp) warp_tma_store<true>(slot, map_lp, v, lane, n0, row0, bidx);
    else if (row_ok) store_row_bf16(e.out_bf16 + bidx * p.so_lp + (long long)m * e.ld_bf16 + n0, v, nn);
  }
  // bias gradient: per-32-row column sums (rules.py:45-46 reduce_like); the
  // transpose-reduce destroys v, so it runs after the stores
  if (e.colsum) warp_colsum_store(v, e.colsum + (long long)grp * e.ld_colsum + n0, lane, nn);
}

template <bool TF32, int BN, int STAGES, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 const __grid_constant__ CUtensorMap tma_olp, const __grid_constant__ CUtensorMap tma_of32,
                 const __grid_constant__ CUtensorMap tma_aux,
                 const KParams p) {
  using E = Elem<TF32>;
  constexpr int BK = E::BK;
  constexpr int A_BYTES = BM * ROW_BYTES;
  constexpr int B_BYTES = BN * ROW_BYTES;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered fp32 accumulator
  static_assert(TMEM_COLS <= 512 && (TMEM_COLS & (TMEM_COLS - 1)) == 0, "TMEM allocation");
  constexpr uint32_t IDESC = idesc_tc(BM, BN, A_MN, B_MN, TF32);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* acc_full = empty_bar + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  uint8_t* stage_slots = smem + STAGES * STAGE_BYTES + 1024;  // 8 x 4 KB epilogue staging
  uint64_t* aux_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 512);  // one per epilogue warp

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int m_tiles = (p.M + BM - 1) / BM;
  const int n_tiles = (p.N + BN - 1) / BN;
  const int tiles_pb = m_tiles * n_tiles;   // output tiles per batch entry
  const int out_tiles = tiles_pb * p.batch;
  const int tiles = out_tiles * p.splits;  // work items: (split, batch, output tile)
  const int num_kb_total = (p.K + BK - 1) / BK;
  // k-block range of work item t
  auto kb_range = [&](int t, int& kb0, int& kb1) {
    const int s = t / out_tiles;
    kb0 = s * p.kb_per_split;
    kb1 = min(num_kb_total, kb0 + p.kb_per_split);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma_a);
    tma_prefetch(&tma_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], EPI_WARPS);  // one arrival per epilogue warp
    }
    for (int w = 0; w < EPI_WARPS; ++w) mbar_init(&aux_bar[w], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the setup above (barriers, TMEM, descriptor
  // prefetch) overlaps the previous kernel's tail; no global memory is touched
  // before the previous grid has completed.
  grid_dep_wait();
  grid_dep_launch();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int u = t % out_tiles, bidx = u / tiles_pb;
        const TileCoord tc = tile_of(u - bidx * tiles_pb, m_tiles, n_tiles, BN);
        int kb0, kb1;
        kb_range(t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / BK; ++j)
              tma_load_3d(sa + j * E::MN_CHUNK, &tma_a, &full_bar[stage], tc.m0 + BK * j, k0, bidx);
          } else {
            tma_load_3d(sa, &tma_a, &full_bar[stage], k0, tc.m0, bidx);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / BK; ++j)
              tma_load_3d(sb + j * E::MN_CHUNK, &tma_b, &full_bar[stage], tc.n0 + BK * j, k0, bidx);
          } else {
            tma_load_3d(sb, &tma_b, &full_bar[stage], k0, tc.n0, bidx);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int kb0, kb1;
        kb_range(t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < E::KSTEPS; ++k) {
            // K-major: the next UMMA_K elements are +32 B inside the swizzle row;
            // MN-major: the next UMMA_K K-rows are +UMMA_K*128 B
            const uint64_t ad = A_MN ? sdesc(sa + k * E::MN_KSTEP, E::MN_CHUNK, E::MN_SBO, E::MN_LAYOUT) : sdesc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? sdesc(sb + k * E::MN_KSTEP, E::MN_CHUNK, E::MN_SBO, E::MN_LAYOUT) : sdesc(sb + k * 32, 16, 1024);
            tc_mma<TF32>(d_tmem, ad, bd, IDESC, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          tc_commit(&empty_bar[stage]);  // smem stage free once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&acc_full[acc]);  // accumulator complete
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ===================== epilogue =====================
    const int ew = warp - EPI_WARP0;
    const int q = ew % 4;   // TMEM lanes 32q..32q+31 (a warp may only touch lanes 32*(warp%4)..)
    const int half = ew / 4;  // which half of the tile's columns
    constexpr int CHUNKS = BN / 32;
    constexpr int CH_PER = CHUNKS / 2;
    int acc = 0;
    uint32_t acc_phase = 0, aux_phase = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int u = t % out_tiles, bidx = u / tiles_pb;
      const TileCoord tc = tile_of(u - bidx * tiles_pb, m_tiles, n_tiles, BN);
      const int row0 = tc.m0 + q * 32;
      const int c0 = half * CH_PER, c1 = (half + 1) * CH_PER;
      uint8_t* slot = stage_slots + ew * STAGE_SLOT;
      const bool staged = p.aux_stage && row0 < p.M;  // warp-uniform
      if (staged && lane == 0 && tc.n0 + c0 * 32 < p.N) aux_issue(slot, &tma_aux, &aux_bar[ew], tc.n0 + c0 * 32, row0);
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      const int m = row0 + lane;
      const bool row_ok = m < p.M;
#pragma unroll 1
      for (int c = c0; c < c1; ++c) {
        const int n0 = tc.n0 + c * 32;
        float v[32];
        tmem_ld32(tmem_base + acc * BN + ((uint32_t)(q * 32) << 16) + c * 32, v);
        if (n0 >= p.N) continue;  // warp-uniform
        float h[32];
        if (staged) {
          mbar_wait(&aux_bar[ew], aux_phase);
          aux_phase ^= 1;
          aux_read(slot, h, lane);
          fence_proxy_async();  // our reads precede the next async write of the buffer
          __syncwarp();
          if (lane == 0 && c + 1 < c1 && n0 + 32 < p.N) aux_issue(slot, &tma_aux, &aux_bar[ew], n0 + 32, row0);
        }
        epi_chunk(p, v, m, row_ok, (tc.m0 >> 5) + q, row0 < p.M, n0, lane, t / out_tiles, bidx, staged, h, slot,
                  false, &tma_olp, &tma_of32);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&acc_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if (warp >= EPI_WARP0 && lane == 0) bulk_wait0();  // staged stores drained before smem goes away
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
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

template <bool TF32, int STAGES, bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
gemm_tc_pair_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                      const __grid_constant__ CUtensorMap tma_olp, const __grid_constant__ CUtensorMap tma_of32,
                      const __grid_constant__ CUtensorMap tma_aux,
                      const KParams p) {
  constexpr int PM = 256, BN = 256, HALF = 128;
  using E = Elem<TF32>;
  constexpr int BK = E::BK;
  constexpr int A_BYTES = HALF * ROW_BYTES;
  constexpr int B_BYTES = HALF * ROW_BYTES;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  constexpr uint32_t IDESC = idesc_tc(PM, BN, A_MN, B_MN, TF32);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* acc_full = empty_bar + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  uint8_t* stage_slots = smem + STAGES * STAGE_BYTES + 1024;  // 8 x 4 KB epilogue staging
  uint64_t* aux_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 512);  // one per epilogue warp

  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int m_tiles = (p.M + PM - 1) / PM;
  const int n_tiles = (p.N + BN - 1) / BN;
  const int tiles_pb = m_tiles * n_tiles;
  const int out_tiles = tiles_pb * p.batch;
  // work units: split-K x batch x tiles, or (tail mode) the full tiles followed
  // by two K-halves of each of the last tail_split tiles (row-major order)
  const int tiles = p.tail_split > 0 ? p.tail_full + 2 * p.tail_split : out_tiles * p.splits;
  const int num_kb_total = (p.K + BK - 1) / BK;
  const int kb_half = (num_kb_total + 1) / 2;
  const int pair = blockIdx.x / 2, pairs = gridDim.x / 2;
  auto kb_range = [&](int t, int& kb0, int& kb1) {
    if (p.tail_split > 0) {
      const bool half = t >= p.tail_full && ((t - p.tail_full) & 1);
      kb0 = t < p.tail_full ? 0 : (half ? kb_half : 0);
      kb1 = t < p.tail_full ? num_kb_total : min(num_kb_total, kb0 + kb_half);
      return;
    }
    const int s = t / out_tiles;
    kb0 = s * p.kb_per_split;
    kb1 = min(num_kb_total, kb0 + p.kb_per_split);
  };
  auto coord = [&](int t) {
    TileCoord c;
    if (p.tail_split > 0) {  // tail mode: row-major tiles
      const int tile = t < p.tail_full ? t : p.tail_full + ((t - p.tail_full) >> 1);
      c.m0 = (tile / n_tiles) * PM;
      c.n0 = (tile % n_tiles) * BN;
      return c;
    }
    const int G = p.raster;  // grouped raster over 256-row pair tiles
    const int u = (t % out_tiles) % tiles_pb;
    const int per_group = G * n_tiles;
    const int group = u / per_group;
    const int first_m = group * G;
    const int gsize = min(m_tiles - first_m, G);
    const int in_group = u - group * per_group;
    c.m0 = (first_m + in_group % gsize) * PM;
    c.n0 = (in_group / gsize) * BN;
    return c;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma_a);
    tma_prefetch(&tma_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2 * EPI_WARPS);  // every epilogue warp of both CTAs
    }
    for (int w = 0; w < EPI_WARPS; ++w) mbar_init(&aux_bar[w], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote traffic
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  grid_dep_wait();  // see gemm_tc_kernel
  grid_dep_launch();
  SG_TRACE_BEGIN();

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < tiles; t += pairs) {
        const TileCoord tc = coord(t);
        const int bidx = (t % out_tiles) / tiles_pb;
        const int am = tc.m0 + (int)rank * HALF, bn = tc.n0 + (int)rank * HALF;
        int kb0, kb1;
        kb_range(t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t fb = mapa_shared(smem_u32(&full_bar[stage]), 0);  // leader's full barrier
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < HALF / BK; ++j)
              tma_load_3d_pair(sa + j * E::MN_CHUNK, &tma_a, fb, am + BK * j, k0, bidx);
          } else {
            tma_load_3d_pair(sa, &tma_a, fb, k0, am, bidx);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < HALF / BK; ++j)
              tma_load_3d_pair(sb + j * E::MN_CHUNK, &tma_b, fb, bn + BK * j, k0, bidx);
          } else {
            tma_load_3d_pair(sb, &tma_b, fb, k0, bn, bidx);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader only) =====================
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int it = 0;
      for (int t = pair; t < tiles; t += pairs, ++it) {
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int kb0, kb1;
        kb_range(t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (kb == kb0) SG_TRACE(it, 0);  // first k-block of the tile ready: MMA starts
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < E::KSTEPS; ++k) {
            const uint64_t ad = A_MN ? sdesc(sa + k * E::MN_KSTEP, E::MN_CHUNK, E::MN_SBO, E::MN_LAYOUT) : sdesc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? sdesc(sb + k * E::MN_KSTEP, E::MN_CHUNK, E::MN_SBO, E::MN_LAYOUT) : sdesc(sb + k * 32, 16, 1024);
            tc_mma_pair<TF32>(d_tmem, ad, bd, IDESC, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          tc_commit_pair(&empty_bar[stage]);  // frees this stage in both CTAs
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair(&acc_full[acc]);  // both CTAs' accumulator halves complete
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ===================== epilogue (both CTAs, own 128 rows) =====================
    const int ew = warp - EPI_WARP0;
    const int q = ew % 4;
    const int half = ew / 4;
    constexpr int CH_PER = (BN / 32) / 2;
    const uint32_t acc_empty_leader0 = mapa_shared(smem_u32(&acc_empty[0]), 0);
    const uint32_t acc_empty_leader1 = mapa_shared(smem_u32(&acc_empty[1]), 0);
    int acc = 0;
    uint32_t acc_phase = 0, aux_phase = 0;
    int it = 0;
    for (int t = pair; t < tiles; t += pairs, ++it) {
      const TileCoord tc = coord(t);
      const int bidx = (t % out_tiles) / tiles_pb;
      const int row0 = tc.m0 + (int)rank * HALF + q * 32;
      const int c0 = half * CH_PER, c1 = (half + 1) * CH_PER;
      uint8_t* slot = stage_slots + ew * STAGE_SLOT;
      const bool staged = p.aux_stage && row0 < p.M;  // warp-uniform
      if (staged && lane == 0 && tc.n0 + c0 * 32 < p.N) aux_issue(slot, &tma_aux, &aux_bar[ew], tc.n0 + c0 * 32, row0);
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      if (ew == 0 && lane == 0) SG_TRACE(it, 1);  // accumulator complete
      const int m = row0 + lane;
      const bool row_ok = m < p.M;
#pragma unroll 1
      for (int c = c0; c < c1; ++c) {
        const int n0 = tc.n0 + c * 32;
        float v[32];
        tmem_ld32(tmem_base + acc * BN + ((uint32_t)(q * 32) << 16) + c * 32, v);
        if (n0 >= p.N) continue;
        float h[32];
        if (staged) {
          mbar_wait(&aux_bar[ew], aux_phase);
          aux_phase ^= 1;
          aux_read(slot, h, lane);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0 && c + 1 < c1 && n0 + 32 < p.N) aux_issue(slot, &tma_aux, &aux_bar[ew], n0 + 32, row0);
        }
        epi_chunk(p, v, m, row_ok, row0 >> 5, row0 < p.M, n0, lane, t / out_tiles, bidx, staged, h, slot,
                  p.tail_split > 0 && t >= p.tail_full, &tma_olp, &tma_of32);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc == 0 ? acc_empty_leader0 : acc_empty_leader1);
      if (lane == 0 && ew == 0) SG_TRACE(it, 2);  // epilogue warp 0 done with the tile
      if (lane == 0 && ew == EPI_WARPS - 1) SG_TRACE(it, 3);  // last epilogue warp done
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if (warp >= EPI_WARP0 && lane == 0) bulk_wait0();  // staged stores drained before smem goes away
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer may still be reading our smem / signalling our barriers
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
  SG_TRACE_END();
}

}  // namespace tc
}  // namespace sg

// ================================================================ host side
namespace sg {

namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

// 2-D operand tensor map over a row-major [outer][ld] buffer (bf16, or fp32
// read as TF32), box {one 128-byte row, box_outer}, 128B swizzle.
// 3-D over `batch` such buffers `sbatch` elements apart (batch 1: a plain matrix).
int make_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long ld, int box_outer,
             bool tf32, bool mn_major, int batch, long long sbatch) {
  EncodeTiled enc = encode_fn();
  if (!enc) return fail(SG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int esz = tf32 ? 4 : 2;
  if (batch <= 1) sbatch = ld * outer;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)(batch < 1 ? 1 : batch)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * esz), (cuuint64_t)(sbatch * esz)};
  cuuint32_t box[3] = {(cuuint32_t)(tc::ROW_BYTES / esz), (cuuint32_t)box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, tf32 ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (tf32 && mn_major) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled");
  return SG_OK;
}

// Output maps for the TMA-store epilogue: box 32 x 32, swizzle matching
// stage_bf16 (64B) / stage_f32 (128B).  Returns false when the buffer does
// not meet TMA's alignment rules (the epilogue then stores directly).
bool make_out_map(CUtensorMap* map, const void* ptr, bool bf16, long long N, long long M, long long ld, int batch,
                  long long sbatch) {
  const long long esz = bf16 ? 2 : 4;
  if (batch <= 1) sbatch = ld * M;
  if (!ptr || (reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esz) % 16 || (sbatch * esz) % 16 || M <= 0 ||
      N <= 0)
    return false;
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)(batch < 1 ? 1 : batch)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * esz), (cuuint64_t)(sbatch * esz)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ACT_GRAD with a bf16 saved activation and a bf16-only output: the aux
// blocks are TMA-streamed through the free half of each staging slot.
void aux_map(const GemmArgs& g, tc::KParams& p, CUtensorMap& m) {
  std::memset(&m, 0, sizeof m);
  p.aux_stage = 0;
  static const bool enabled = [] {
    const char* e = std::getenv("SGB200_GEMM_AUX_TMA");
    return !(e && e[0] == '0');
  }();
  const GemmEpilogue& e = g.epi;
  if (!enabled || e.mode != SG_EPI_ACT_GRAD || !e.aux || e.aux_f32 || e.out_f32 || !p.tma_lp || p.splits > 1 ||
      g.batch > 1 || (reinterpret_cast<uintptr_t>(e.aux) & 15) || (e.ld_aux * 2) % 16)
    return;
  EncodeTiled enc = encode_fn();
  if (!enc) return;
  cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, 1};
  cuuint64_t strides[2] = {(cuuint64_t)(e.ld_aux * 2), (cuuint64_t)(e.ld_aux * 2 * g.M)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(e.aux), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  p.aux_stage = r == CUDA_SUCCESS;
}

void out_maps(const GemmArgs& g, tc::KParams& p, CUtensorMap& mlp, CUtensorMap& mf32) {
  static const bool enabled = [] {
    const char* e = std::getenv("SGB200_GEMM_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  std::memset(&mlp, 0, sizeof mlp);
  std::memset(&mf32, 0, sizeof mf32);
  p.tma_lp = p.tma_f32 = 0;
  if (!enabled || p.splits > 1) return;
  if (g.epi.out_bf16)
    p.tma_lp = make_out_map(&mlp, g.epi.out_bf16, true, g.N, g.M, g.epi.ld_bf16, g.batch, g.so_lp);
  if (g.epi.out_f32)
    p.tma_f32 = make_out_map(&mf32, g.epi.out_f32, false, g.N, g.M, g.epi.ld_f32, g.batch, g.so_f32);
}

// split-K finalize: out = sum_s part[s] in ascending s (deterministic)
// blockIdx.y = row, threads over 4-column groups (no 64-bit divides, float4 loads)
__global__ void k_splitk_reduce(const float* __restrict__ part, int S, int M, int N, long long ldp, float* out,
                                long long ld_out, __nv_bfloat16* out_lp, long long ld_lp) {
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (n >= N) return;
  const bool vec = n + 4 <= N && (ldp % 4) == 0;
  for (long long m = blockIdx.y; m < M; m += gridDim.y) {
  float acc[4];
  if (vec) {
    float4 a = *reinterpret_cast<const float4*>(part + m * ldp + n);
    acc[0] = a.x, acc[1] = a.y, acc[2] = a.z, acc[3] = a.w;
    for (int s = 1; s < S; ++s) {
      const float4 b = *reinterpret_cast<const float4*>(part + ((long long)s * M + m) * ldp + n);
      acc[0] += b.x, acc[1] += b.y, acc[2] += b.z, acc[3] += b.w;
    }
  } else {
    for (int j = 0; j < 4; ++j) {
      acc[j] = n + j < N ? part[m * ldp + n + j] : 0.0f;
      for (int s = 1; s < S; ++s)
        if (n + j < N) acc[j] += part[((long long)s * M + m) * ldp + n + j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (n + j >= N) break;
    if (out) out[m * ld_out + n + j] = acc[j];
    if (out_lp) out_lp[m * ld_lp + n + j] = __float2bfloat16_rn(acc[j]);
  }
  }
}

// Launch with a programmatic dependency on the previous kernel in the stream
// (SGB200_GEMM_PDL=0 disables): the kernel's own griddepcontrol.wait orders
// its memory accesses after the predecessor.
template <class Kern, class... Args>
cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  static const bool pdl = [] {
    const char* e = std::getenv("SGB200_GEMM_PDL");
    return !(e && e[0] == '0');
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
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

static int launch_splitk_reduce(const float* part, int splits, const GemmArgs& g, long long ld_part,
                                cudaStream_t st) {
  const unsigned gx = (unsigned)(((g.N + 3) / 4 + 255) / 256);
  const unsigned gy = (unsigned)(g.M < 65535 ? g.M : 65535);
  k_splitk_reduce<<<dim3(gx, gy), 256, 0, st>>>(part, splits, g.M, g.N, ld_part, g.epi.out_f32, g.epi.ld_f32,
                                                 g.epi.out_bf16, g.epi.ld_bf16);
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

template <bool TF32, int BN, bool A_MN, bool B_MN>
int run(const GemmArgs& g, int num_sms, cudaStream_t st) {
  constexpr int BK = tc::Elem<TF32>::BK;
  constexpr int STAGE = tc::BM * tc::ROW_BYTES + BN * tc::ROW_BYTES;
  constexpr int STAGES = (BN == 256) ? 4 : (BN == 128 ? 6 : 8);
  // operand ring + alignment + barriers (1 KB) + 8 epilogue staging slots
  constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 1024 + tc::EPI_WARPS * tc::STAGE_SLOT;
  static_assert(SMEM <= 232448, "shared memory budget");
  CUtensorMap ma, mb;
  int rc;
  if (A_MN) rc = make_map(&ma, g.A, g.M, g.K, g.lda, BK, TF32, true, g.batch, g.sa);
  else rc = make_map(&ma, g.A, g.K, g.M, g.lda, tc::BM, TF32, false, g.batch, g.sa);
  if (rc) return rc;
  if (B_MN) rc = make_map(&mb, g.B, g.N, g.K, g.ldb, BK, TF32, true, g.batch, g.sb);
  else rc = make_map(&mb, g.B, g.K, g.N, g.ldb, BN, TF32, false, g.batch, g.sb);
  if (rc) return rc;
  auto kern = tc::gemm_tc_kernel<TF32, BN, STAGES, A_MN, B_MN>;
  static std::atomic<uint64_t> attr_set{0};  // per device
  if (first_on_device(attr_set))
    SG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  const int tiles = ((g.M + tc::BM - 1) / tc::BM) * ((g.N + BN - 1) / BN) * g.batch;
  const int num_kb = (g.K + BK - 1) / BK;
  // split-K when the output tiles cannot fill the machine (e.g. dW of a narrow
  // layer: M = N = 1024, K = batch): plain-store epilogues only
  int splits = 1, kb_per = num_kb;
  if (g.epi.mode == SG_EPI_STORE && !g.epi.colsum && g.batch == 1 && tiles * 2 <= num_sms && num_kb >= 8) {
    int s = num_sms / tiles;
    if (s > num_kb / 4) s = num_kb / 4;
    if (s > 16) s = 16;
    if (s >= 2) {
      kb_per = (num_kb + s - 1) / s;
      splits = (num_kb + kb_per - 1) / kb_per;
    }
  }
  tc::KParams p{g.M, g.N, g.K, g.epi, splits, kb_per, nullptr, 0, 0, 0, 0, 8, 0, 0, g.batch, g.so_f32, g.so_lp};
  if (const char* e = std::getenv("SGB200_GEMM_RASTER")) p.raster = std::max(1, std::atoi(e));
  CUtensorMap mlp, mf32, maux;
  out_maps(g, p, mlp, mf32);
  aux_map(g, p, maux);
  float* part = nullptr;
  if (splits > 1) {
    p.ld_part = (g.N + 3) / 4 * 4;
    SG_CUDA_TRY(cudaMallocAsync((void**)&part, (size_t)splits * g.M * p.ld_part * sizeof(float), st));
    p.part = part;
  }
  const int work = tiles * splits;
  const int grid = work < num_sms ? work : num_sms;
  SG_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(tc::NUM_THREADS), SMEM, st, ma, mb, mlp, mf32, maux, p));
  SG_CUDA_TRY(cudaGetLastError());
  if (splits > 1) {
    if (int rc2 = launch_splitk_reduce(part, splits, g, p.ld_part, st)) return rc2;
    SG_CUDA_TRY(cudaFreeAsync(part, st));
  }
  return SG_OK;
}

template <bool TF32, bool A_MN, bool B_MN>
int run_pair(const GemmArgs& g, int num_sms, cudaStream_t st) {
  constexpr int BK = tc::Elem<TF32>::BK;
  constexpr int STAGES = 6;
  constexpr int STAGE = 128 * tc::ROW_BYTES * 2;
  // operand ring + alignment + barriers (1 KB) + 8 epilogue staging slots
  constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 1024 + tc::EPI_WARPS * tc::STAGE_SLOT;
  static_assert(SMEM <= 232448, "shared memory budget");
  CUtensorMap ma, mb;
  int rc;
  if (A_MN) rc = make_map(&ma, g.A, g.M, g.K, g.lda, BK, TF32, true, g.batch, g.sa);
  else rc = make_map(&ma, g.A, g.K, g.M, g.lda, 128, TF32, false, g.batch, g.sa);
  if (rc) return rc;
  if (B_MN) rc = make_map(&mb, g.B, g.N, g.K, g.ldb, BK, TF32, true, g.batch, g.sb);
  else rc = make_map(&mb, g.B, g.K, g.N, g.ldb, 128, TF32, false, g.batch, g.sb);
  if (rc) return rc;
  auto kern = tc::gemm_tc_pair_kernel<TF32, STAGES, A_MN, B_MN>;
  static std::atomic<uint64_t> attr_set{0};  // per device
  if (first_on_device(attr_set))
    SG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  const int pairs_avail = num_sms / 2;
  const int tiles = ((g.M + 255) / 256) * ((g.N + 255) / 256) * g.batch;
  const int num_kb = (g.K + BK - 1) / BK;
  int splits = 1, kb_per = num_kb;
  if (g.epi.mode == SG_EPI_STORE && !g.epi.colsum && g.batch == 1 && tiles * 2 <= pairs_avail && num_kb >= 8) {
    int s = pairs_avail / tiles;
    if (s > num_kb / 4) s = num_kb / 4;
    if (s > 16) s = 16;
    if (s >= 2) {
      kb_per = (num_kb + s - 1) / s;
      splits = (num_kb + kb_per - 1) / kb_per;
    }
  }
  tc::KParams p{g.M, g.N, g.K, g.epi, splits, kb_per, nullptr, 0, 0, 0, 0, 8, 0, 0, g.batch, g.so_f32, g.so_lp};
  if (const char* e = std::getenv("SGB200_GEMM_RASTER")) p.raster = std::max(1, std::atoi(e));
  CUtensorMap mlp, mf32, maux;
  out_maps(g, p, mlp, mf32);
  aux_map(g, p, maux);
  float* part = nullptr;
  if (splits > 1) {
    p.ld_part = (g.N + 3) / 4 * 4;
    SG_CUDA_TRY(cudaMallocAsync((void**)&part, (size_t)splits * g.M * p.ld_part * sizeof(float), st));
    p.part = part;
  }
  int work = tiles * splits;
  // Split tail: when the last wave of pair tiles would run mostly empty (e.g. a
  // 4096^2 dW: 256 tiles = 3 full waves of 74 pairs + 34 tiles), those last
  // tiles are computed as two K-halves each and reduce-added (fp32; two terms,
  // so the sum does not depend on their order) into the zeroed output: every
  // pair then gets at most one half-length unit after its full tiles.
  static const bool tail_ok = [] {
    const char* e = std::getenv("SGB200_GEMM_TAIL");
    return !(e && e[0] == '0');
  }();
  const int n_tiles = (g.N + 255) / 256;
  const int rem = tiles % pairs_avail;
  if (tail_ok && splits == 1 && g.batch == 1 && g.epi.mode == SG_EPI_STORE && g.epi.out_f32 && !g.epi.out_bf16 &&
      !g.epi.colsum && !g.epi.out_pre && num_kb >= 8 && tiles > pairs_avail && rem > 0 && 2 * rem <= pairs_avail) {
    p.tail_full = tiles - rem;
    p.tail_split = rem;
    const long long row0 = (long long)(p.tail_full / n_tiles) * 256;  // first row of the first split tile
    SG_CUDA_TRY(cudaMemset2DAsync(g.epi.out_f32 + row0 * g.epi.ld_f32, (size_t)g.epi.ld_f32 * 4, 0,
                                  (size_t)g.N * 4, (size_t)(g.M - row0), st));
    work = p.tail_full + 2 * rem;
  }
  const int grid = 2 * (work < pairs_avail ? work : pairs_avail);
  SG_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(tc::NUM_THREADS), SMEM, st, ma, mb, mlp, mf32, maux, p));
  SG_CUDA_TRY(cudaGetLastError());
  if (splits > 1) {
    if (int rc2 = launch_splitk_reduce(part, splits, g, p.ld_part, st)) return rc2;
    SG_CUDA_TRY(cudaFreeAsync(part, st));
  }
  return SG_OK;
}

template <bool TF32, int BN>
int run_bn(const GemmArgs& g, int num_sms, cudaStream_t st) {
  if (!g.a_mn && !g.b_mn) return run<TF32, BN, false, false>(g, num_sms, st);
  if (!g.a_mn && g.b_mn) return run<TF32, BN, false, true>(g, num_sms, st);
  if (g.a_mn && g.b_mn) return run<TF32, BN, true, true>(g, num_sms, st);
  return run<TF32, BN, true, false>(g, num_sms, st);
}

template <bool TF32>
int dispatch(const GemmArgs& g, int num_sms, cudaStream_t st) {
  static const int force_bn = [] {
    const char* e = std::getenv("SGB200_GEMM_FORCE_BN");
    return e ? std::atoi(e) : 0;
  }();
  if (force_bn == 64) return run_bn<TF32, 64>(g, num_sms, st);
  if (force_bn == 128) return run_bn<TF32, 128>(g, num_sms, st);
  if (force_bn == 256) return run_bn<TF32, 256>(g, num_sms, st);
  if (g.N <= 64) return run_bn<TF32, 64>(g, num_sms, st);
  if (g.N <= 128) return run_bn<TF32, 128>(g, num_sms, st);
  static const bool pair_ok = [] {
    const char* e = std::getenv("SGB200_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  if (pair_ok && g.M >= 256 && num_sms >= 2) {
    if (!g.a_mn && !g.b_mn) return run_pair<TF32, false, false>(g, num_sms, st);
    if (!g.a_mn && g.b_mn) return run_pair<TF32, false, true>(g, num_sms, st);
    if (g.a_mn && g.b_mn) return run_pair<TF32, true, true>(g, num_sms, st);
    return run_pair<TF32, true, false>(g, num_sms, st);
  }
  return run_bn<TF32, 256>(g, num_sms, st);
}

}  // namespace

#ifdef SGB200_GEMM_TRACE
extern "C" SG_API int sg_gemm_trace_buffer(void* buf, int iters, int launches) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  const unsigned zero = 0;
  SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_trace, &p, sizeof p));
  SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_trace_iters, &iters, sizeof iters));
  SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_trace_launches, &launches, sizeof launches));
  SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_trace_seq, &zero, sizeof zero));
  SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_trace_done, &zero, sizeof zero));
  return SG_OK;
}
#endif

int launch_gemm_tc(const GemmArgs& g, bool tf32, int num_sms, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return fail(SG_EINVAL, "gemm: empty problem");
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!aligned(g.A) || !aligned(g.B)) return fail(SG_EINVAL, "gemm: A and B must be 16-byte aligned");
  const int row_mult = tf32 ? 4 : 8;  // 16-byte TMA strides
  if (g.lda % row_mult || g.ldb % row_mult)
    return fail(SG_EINVAL, tf32 ? "gemm: lda/ldb must be multiples of 4 elements (TF32)"
                                : "gemm: lda/ldb must be multiples of 8 elements");
  if (g.lda < (g.a_mn ? g.M : g.K) || g.ldb < (g.b_mn ? g.N : g.K))
    return fail(SG_EINVAL, "gemm: leading dimension smaller than the row");
  if (g.batch < 1) return fail(SG_EINVAL, "gemm: batch must be >= 1");
  if (g.batch > 1) {
    if (g.epi.colsum || g.epi.out_pre || g.epi.mode == SG_EPI_ACT_GRAD)
      return fail(SG_EINVAL, "gemm: batched GEMMs take the STORE / BIAS_ACT epilogues without colsum / out_pre");
    if ((g.sa * (tf32 ? 4 : 2)) % 16 || (g.sb * (tf32 ? 4 : 2)) % 16)
      return fail(SG_EINVAL, "gemm: batch strides must be multiples of 16 bytes");
  }
  return tf32 ? dispatch<true>(g, num_sms, st) : dispatch<false>(g, num_sms, st);
}

}  // namespace sg
