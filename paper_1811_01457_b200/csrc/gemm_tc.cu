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
#include "gemm_tc_dev.cuh"

namespace sg {
namespace tc {

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

  if (warp < EPI_WARP0) {
  // The TMA / MMA / TMEM warpgroup hands registers to the epilogue warpgroups
  // (warpgroup-collective setmaxnreg; ptxas allocates each branch to its own
  // limit): the 32-column epilogue chunks no longer spill at the 168 cap.
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
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
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");  // (65536 - 128 x 56) / 256, rounded to 8
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

template <bool TF32, int STAGES, bool A_MN, bool B_MN, bool WIDE>
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
    // tail mode: work unit t < tail_full is tile t, the rest are the two
    // K-halves of the remaining tiles; tiles in the same grouped raster as below
    // (row-major order read every B block once per wave: 2.3x the algorithmic
    // DRAM traffic of the TF32 4096^2 dW)
    const int G = p.raster;  // grouped raster over 256-row pair tiles
    const int u = p.tail_split > 0 ? (t < p.tail_full ? t : p.tail_full + ((t - p.tail_full) >> 1))
                                   : (t % out_tiles) % tiles_pb;
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
    for (int w = 0; w < 2 * EPI_WARPS; ++w) mbar_init(&aux_bar[w], 1);
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
    int next_buf = 0;
    int it = 0;
    uint8_t* slot = stage_slots + ew * Slot<WIDE>::BYTES;
    uint64_t* my_aux = &aux_bar[2 * ew];
    for (int t = pair; t < tiles; t += pairs, ++it) {
      const TileCoord tc = coord(t);
      const int bidx = (t % out_tiles) / tiles_pb;
      const int row0 = tc.m0 + (int)rank * HALF + q * 32;
      const int c0 = half * CH_PER;
      const bool staged = p.aux_stage && row0 < p.M;  // warp-uniform
      epi_aux_prologue<WIDE>(staged, lane, slot, &tma_aux, my_aux, tc.n0 + c0 * 32, CH_PER, p.N, row0,
                             p.aux_stage == 2);
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      if (ew == 0 && lane == 0) SG_TRACE(it, 1);  // accumulator complete
      epi_chunks<WIDE>(p, tmem_base + acc * BN + ((uint32_t)(q * 32) << 16), tc.n0 + c0 * 32, c0, CH_PER, row0, lane,
                       t / out_tiles, bidx, p.tail_split > 0 && t >= p.tail_full, slot, staged, &tma_aux, my_aux,
                       aux_phase, &tma_olp, &tma_of32, next_buf);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc == 0 ? acc_empty_leader0 : acc_empty_leader1);
      if (p.splits > 1 && p.split_cnt) {  // in-kernel split-K fix-up of this warp's region of the tile
        const int tile = (tc.m0 / PM) * n_tiles + tc.n0 / BN;
        split_region_fixup(p, p.split_cnt + tile * (2 * EPI_WARPS) + (int)rank * EPI_WARPS + ew, row0,
                           tc.n0 + c0 * 32, CH_PER, lane);
      }
      if (lane == 0 && ew == 0) SG_TRACE(it, 2);  // epilogue warp 0 done with the tile
      if (lane == 0 && ew == EPI_WARPS - 1) SG_TRACE(it, 3);  // last epilogue warp done
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if (warp >= EPI_WARP0 && p.fin_out) {
    // bias-gradient finalize as the epilogue's tail job, in warp 0's staging slot
    if (lane == 0) bulk_wait_read0();
    epi_bar();
    colsum_finalize_tail(p, reinterpret_cast<double*>(stage_slots), threadIdx.x - EPI_WARP0 * 32, blockIdx.x,
                         gridDim.x);
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

namespace tcmap {  // tensor-map builders, shared with gemm_chain.cu

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
  // (N * esz) % 16: TMA stores clip the row end only to 16 bytes -- a ragged
  // row (e.g. 300 bf16) would get the elements up to the next 16-byte
  // boundary written (tools/sanitize_cases.py guard bands); such outputs take
  // the direct-store path
  if (!ptr || (reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esz) % 16 || (sbatch * esz) % 16 || M <= 0 ||
      N <= 0 || (N * esz) % 16)
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
// BIAS_MSE in the wide-slot kernel (wide = true): the fp32 targets, 4 KB
// blocks through the slot's upper half, one chunk ahead (dz is staged in
// the lower half; no fp32 output shares the slot).  Measured on B200: a
// second target buffer with dz stored from registers instead is slower.
void aux_map(const GemmArgs& g, tc::KParams& p, CUtensorMap& m, bool wide) {
  std::memset(&m, 0, sizeof m);
  p.aux_stage = 0;
  static const bool enabled = [] {
    const char* e = std::getenv("SGB200_GEMM_AUX_TMA");
    return !(e && e[0] == '0');
  }();
  const GemmEpilogue& e = g.epi;
  if (e.mode == SG_EPI_BIAS_MSE || e.mode == SG_EPI_BIAS_ACT_SEED) {  // fp32 targets / seed
    if (!enabled || !wide || e.out_f32 || !e.seed || p.splits > 1 || g.batch > 1 ||
        (reinterpret_cast<uintptr_t>(e.seed) & 15) || (e.ld_seed * 4) % 16)
      return;
    EncodeTiled enc = encode_fn();
    if (!enc) return;
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, 1};
    cuuint64_t strides[2] = {(cuuint64_t)(e.ld_seed * 4), (cuuint64_t)(e.ld_seed * 4 * g.M)};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(e.seed), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    p.aux_stage = r == CUDA_SUCCESS ? 2 : 0;
    return;
  }
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
  p.tma_lp = p.tma_f32 = p.tma_o2 = 0;
  if (!enabled || p.splits > 1) return;
  if (g.epi.out_bf16)
    p.tma_lp = make_out_map(&mlp, g.epi.out_bf16, true, g.N, g.M, g.epi.ld_bf16, g.batch, g.so_lp);
  if (g.epi.out_f32)
    p.tma_f32 = make_out_map(&mf32, g.epi.out_f32, false, g.N, g.M, g.epi.ld_f32, g.batch, g.so_f32);
  else if ((g.epi.mode == SG_EPI_BIAS_ACT_SEED || g.epi.mode == SG_EPI_BIAS_MSE) && g.epi.out2_bf16)
    p.tma_o2 = make_out_map(&mf32, g.epi.out2_bf16, true, g.N, g.M, g.epi.ld_out2, 1, 0);  // out2 in the fp32 slot
}

}  // namespace tcmap
using namespace tcmap;

namespace {

// split-K finalize: out = sum_s part[s] in ascending s (deterministic)
// blockIdx.y = row, threads over 4-column groups (no 64-bit divides, float4 loads)
__device__ __forceinline__ void splitk_reduce_cols(const float* __restrict__ part, int S, int M, int N, long long ldp,
                                                   float* out, long long ld_out, __nv_bfloat16* out_lp,
                                                   long long ld_lp, int n) {
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
__global__ void k_splitk_reduce(const float* __restrict__ part, int S, int M, int N, long long ldp, float* out,
                                long long ld_out, __nv_bfloat16* out_lp, long long ld_lp) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the partials come from the GEMM before us (PDL)
  splitk_reduce_cols(part, S, M, N, ldp, out, ld_out, out_lp, ld_lp, (blockIdx.x * blockDim.x + threadIdx.x) * 4);
}
// Deferred split-K: several GEMMs' partials reduced in one launch (blockIdx.z
// = job), with k_splitk_reduce's arithmetic (bit-identical results).
constexpr int MAX_SPLITK_JOBS = 32;
struct SplitkJobs {
  const float* part[MAX_SPLITK_JOBS];
  float* out[MAX_SPLITK_JOBS];
  long long ldp[MAX_SPLITK_JOBS], ld_out[MAX_SPLITK_JOBS];
  int S[MAX_SPLITK_JOBS], M[MAX_SPLITK_JOBS], N[MAX_SPLITK_JOBS];
};
__global__ void k_splitk_reduce_multi(const __grid_constant__ SplitkJobs jobs) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int b = blockIdx.z;
  splitk_reduce_cols(jobs.part[b], jobs.S[b], jobs.M[b], jobs.N[b], jobs.ldp[b], jobs.out[b], jobs.ld_out[b], nullptr,
                     0, (blockIdx.x * blockDim.x + threadIdx.x) * 4);
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

// split-K when the output tiles cannot fill the machine (e.g. dW of a narrow
// layer: M = N = 1024, K = batch): plain-store epilogues only.  `units` =
// SMs (1-SM kernels) or CTA pairs.
void choose_splits(const GemmArgs& g, int tiles, int units, int num_kb, int& splits, int& kb_per) {
  splits = 1;
  kb_per = num_kb;
  if (g.epi.mode == SG_EPI_STORE && !g.epi.colsum && g.batch == 1 && tiles * 2 <= units && num_kb >= 8) {
    int s = units / tiles;
    if (s > num_kb / 4) s = num_kb / 4;
    if (s > 16) s = 16;
    if (s >= 2) {
      kb_per = (num_kb + s - 1) / s;
      splits = (num_kb + kb_per - 1) / kb_per;
    }
  }
}

// The partial buffer of a split-K launch: the caller's (deferred reduce,
// GemmArgs::split_part) or a stream-ordered temporary.
static int split_part_buffer(const GemmArgs& g, int splits, long long ld_part, float** part, cudaStream_t st) {
  const long long need = (long long)splits * g.M * ld_part;
  if (g.split_part) {
    if (g.split_part_elems < need) return fail(SG_EINVAL, "gemm: split_part holds " +
                                               std::to_string(g.split_part_elems) + " floats, " +
                                               std::to_string(need) + " needed");
    *part = g.split_part;
    return SG_OK;
  }
  SG_CUDA_TRY(cudaMallocAsync((void**)part, (size_t)need * sizeof(float), st));
  return SG_OK;
}

static int launch_splitk_reduce(const float* part, int splits, const GemmArgs& g, long long ld_part,
                                cudaStream_t st) {
  const unsigned gx = (unsigned)(((g.N + 3) / 4 + 255) / 256);
  const unsigned gy = (unsigned)(g.M < 65535 ? g.M : 65535);
  SG_CUDA_TRY(launch_pdl(k_splitk_reduce, dim3(gx, gy), dim3(256), 0, st, part, splits, g.M, g.N, ld_part,
                         g.epi.out_f32, g.epi.ld_f32, g.epi.out_bf16, g.epi.ld_bf16));
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
  choose_splits(g, tiles, num_sms, num_kb, splits, kb_per);
  tc::KParams p{g.M, g.N, g.K, g.epi, splits, kb_per, nullptr, 0, 0, 0, 0, 8, 0, 0, g.batch, g.so_f32, g.so_lp};
  if (const char* e = std::getenv("SGB200_GEMM_RASTER")) p.raster = std::max(1, std::atoi(e));
  CUtensorMap mlp, mf32, maux;
  out_maps(g, p, mlp, mf32);
  aux_map(g, p, maux, false);
  float* part = nullptr;
  if (splits > 1) {
    p.ld_part = (g.N + 3) / 4 * 4;
    if ((rc = split_part_buffer(g, splits, p.ld_part, &part, st))) return rc;
    p.part = part;
  }
  const int work = tiles * splits;
  const int grid = work < num_sms ? work : num_sms;
  SG_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(tc::NUM_THREADS), SMEM, st, ma, mb, mlp, mf32, maux, p));
  SG_CUDA_TRY(cudaGetLastError());
  if (splits > 1 && !g.split_part) {  // deferred: the caller reduces (sg_splitk_reduce_multi)
    if (int rc2 = launch_splitk_reduce(part, splits, g, p.ld_part, st)) return rc2;
    SG_CUDA_TRY(cudaFreeAsync(part, st));
  }
  // the 1-SM kernels run a requested bias-gradient finalize as its own launch
  if (g.fin.out) return colsum_finalize_launch(g.fin.part, g.fin.G, g.fin.ld, g.fin.N, g.fin.out, num_sms, st);
  return SG_OK;
}

template <bool TF32, bool A_MN, bool B_MN, bool WIDE>
int run_pair(const GemmArgs& g, int num_sms, cudaStream_t st) {
  constexpr int BK = tc::Elem<TF32>::BK;
  // wide epilogue slots (double-buffered staging, aux two chunks ahead) cost
  // one operand stage of the 227 KB
  constexpr int STAGES = WIDE ? 5 : 6;
  constexpr int STAGE = 128 * tc::ROW_BYTES * 2;
  // operand ring + alignment + barriers (1 KB) + 8 epilogue staging slots
  constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 1024 + tc::EPI_WARPS * tc::Slot<WIDE>::BYTES;
  static_assert(SMEM <= 232448, "shared memory budget");
  CUtensorMap ma, mb;
  int rc;
  if (A_MN) rc = make_map(&ma, g.A, g.M, g.K, g.lda, BK, TF32, true, g.batch, g.sa);
  else rc = make_map(&ma, g.A, g.K, g.M, g.lda, 128, TF32, false, g.batch, g.sa);
  if (rc) return rc;
  if (B_MN) rc = make_map(&mb, g.B, g.N, g.K, g.ldb, BK, TF32, true, g.batch, g.sb);
  else rc = make_map(&mb, g.B, g.K, g.N, g.ldb, 128, TF32, false, g.batch, g.sb);
  if (rc) return rc;
  auto kern = tc::gemm_tc_pair_kernel<TF32, STAGES, A_MN, B_MN, WIDE>;
  static std::atomic<uint64_t> attr_set{0};  // per device
  if (first_on_device(attr_set))
    SG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  const int pairs_avail = num_sms / 2;
  const int tiles = ((g.M + 255) / 256) * ((g.N + 255) / 256) * g.batch;
  const int num_kb = (g.K + BK - 1) / BK;
  int splits = 1, kb_per = num_kb;
  choose_splits(g, tiles, pairs_avail, num_kb, splits, kb_per);
  tc::KParams p{g.M, g.N, g.K, g.epi, splits, kb_per, nullptr, 0, 0, 0, 0, 8, 0, 0, g.batch, g.so_f32, g.so_lp};
  if (const char* e = std::getenv("SGB200_GEMM_RASTER")) p.raster = std::max(1, std::atoi(e));
  CUtensorMap mlp, mf32, maux;
  out_maps(g, p, mlp, mf32);
  aux_map(g, p, maux, WIDE);
  float* part = nullptr;
  unsigned* cnt = nullptr;
  // In-kernel split-K fix-up (SGB200_GEMM_SPLIT_FIXUP=1): measured slower on
  // B200 than the separate ordered reduce (c5 step 3.54 vs 3.16 ms): the last
  // split's reduction lengthens every dW kernel's tail, while k_splitk_reduce
  // runs at full width.  The persistent chain kernel uses it (no launches).
  static const bool fixup = [] {
    const char* e = std::getenv("SGB200_GEMM_SPLIT_FIXUP");
    return e && e[0] == '1';
  }();
  if (splits > 1) {
    p.ld_part = (g.N + 3) / 4 * 4;
    if ((rc = split_part_buffer(g, splits, p.ld_part, &part, st))) return rc;
    p.part = part;
    if (fixup && !g.split_part) {  // the last split of each tile region sums the partials inside the kernel
      const size_t ncnt = (size_t)tiles * 2 * tc::EPI_WARPS;
      SG_CUDA_TRY(cudaMallocAsync((void**)&cnt, ncnt * sizeof(unsigned), st));
      SG_CUDA_TRY(cudaMemsetAsync(cnt, 0, ncnt * sizeof(unsigned), st));
      p.split_cnt = cnt;
    }
  }
  if (g.fin.out) {
    p.fin_part = g.fin.part;
    p.fin_G = g.fin.G;
    p.fin_ld = g.fin.ld;
    p.fin_N = g.fin.N;
    p.fin_out = g.fin.out;
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
    // the split tiles are the last `rem` of the grouped raster (coord() in the
    // kernel): zero every row from the first of them on -- full tiles in those
    // rows store over the zeros afterwards
    const int m_tiles = (g.M + 255) / 256;
    int first_m = m_tiles;
    for (int u = p.tail_full; u < tiles; ++u) {
      const int per_group = p.raster * n_tiles, group = u / per_group, fm = group * p.raster;
      const int gsize = std::min(m_tiles - fm, p.raster);
      first_m = std::min(first_m, fm + (u - group * per_group) % gsize);
    }
    const long long row0 = (long long)first_m * 256;
    SG_CUDA_TRY(cudaMemset2DAsync(g.epi.out_f32 + row0 * g.epi.ld_f32, (size_t)g.epi.ld_f32 * 4, 0,
                                  (size_t)g.N * 4, (size_t)(g.M - row0), st));
    work = p.tail_full + 2 * rem;
  }
  const int grid = 2 * (work < pairs_avail ? work : pairs_avail);
  SG_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(tc::NUM_THREADS), SMEM, st, ma, mb, mlp, mf32, maux, p));
  SG_CUDA_TRY(cudaGetLastError());
  if (splits > 1 && !g.split_part) {  // deferred: the caller reduces (sg_splitk_reduce_multi)
    if (!cnt)
      if (int rc2 = launch_splitk_reduce(part, splits, g, p.ld_part, st)) return rc2;
    SG_CUDA_TRY(cudaFreeAsync(part, st));
    if (cnt) SG_CUDA_TRY(cudaFreeAsync(cnt, st));
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
  // Wide epilogue slots (SGB200_GEMM_WIDE=1): -2..3 % per c5 GEMM alone but
  // neutral to slightly slower over the c5 step (one operand stage fewer).
  static const bool wide = [] {
    const char* e = std::getenv("SGB200_GEMM_WIDE");
    return e && e[0] == '1';
  }();
  // the seeded forward streams its fp32 seed through the wide slots as well
  // (SGB200_SEED_TMA=0: read per row from global memory in the narrow kernel)
  static const bool seed_tma = [] {
    const char* e = std::getenv("SGB200_SEED_TMA");
    return !(e && e[0] == '0');
  }();
  if (pair_ok && g.M >= 256 && num_sms >= 2) {
    // the fused MSE loss streams its fp32 targets through the wide slots
    if (wide || ((g.epi.mode == SG_EPI_BIAS_MSE || (g.epi.mode == SG_EPI_BIAS_ACT_SEED && seed_tma)) &&
                 !g.epi.out_f32)) {
      if (!g.a_mn && !g.b_mn) return run_pair<TF32, false, false, true>(g, num_sms, st);
      if (!g.a_mn && g.b_mn) return run_pair<TF32, false, true, true>(g, num_sms, st);
      if (g.a_mn && g.b_mn) return run_pair<TF32, true, true, true>(g, num_sms, st);
      return run_pair<TF32, true, false, true>(g, num_sms, st);
    }
    if (!g.a_mn && !g.b_mn) return run_pair<TF32, false, false, false>(g, num_sms, st);
    if (!g.a_mn && g.b_mn) return run_pair<TF32, false, true, false>(g, num_sms, st);
    if (g.a_mn && g.b_mn) return run_pair<TF32, true, true, false>(g, num_sms, st);
    return run_pair<TF32, true, false, false>(g, num_sms, st);
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
// epilogue stage profile of the single-GEMM kernels (sg_chain_cprof's twin):
// on != 0 clears and enables, on == 0 disables and reads out 8 counters
extern "C" SG_API int sg_gemm_cprof(int on, unsigned long long* out8) {
  if (on) {
    unsigned long long z[8] = {};
    SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_cprof, z, sizeof z));
  } else if (out8) {
    SG_CUDA_TRY(cudaMemcpyFromSymbol(out8, tc::g_cprof, 8 * sizeof(unsigned long long)));
  }
  SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_cprof_on, &on, sizeof on));
  return SG_OK;
}
#endif

// The split-K factor launch_gemm_tc would pick for g (dispatch's kernel choice
// and choose_splits), and the partials' row pitch.
void plan_gemm_splits(const GemmArgs& g, bool tf32, int num_sms, int* splits, long long* ld_part) {
  const int BK = tf32 ? tc::Elem<true>::BK : tc::Elem<false>::BK;
  const int num_kb = (g.K + BK - 1) / BK;
  const char* fe = std::getenv("SGB200_GEMM_FORCE_BN");
  const int force_bn = fe ? std::atoi(fe) : 0;
  const char* pe = std::getenv("SGB200_GEMM_PAIR");
  const bool pair_ok = !(pe && pe[0] == '0');
  int s = 1, kb_per = num_kb;
  if (!force_bn && g.N > 128 && pair_ok && g.M >= 256 && num_sms >= 2) {
    const int tiles = ((g.M + 255) / 256) * ((g.N + 255) / 256) * g.batch;
    choose_splits(g, tiles, num_sms / 2, num_kb, s, kb_per);
  } else {
    const int bn = force_bn ? force_bn : (g.N <= 64 ? 64 : (g.N <= 128 ? 128 : 256));
    const int tiles = ((g.M + tc::BM - 1) / tc::BM) * ((g.N + bn - 1) / bn) * g.batch;
    choose_splits(g, tiles, num_sms, num_kb, s, kb_per);
  }
  *splits = s;
  *ld_part = (g.N + 3) / 4 * 4;
}

int splitk_reduce_multi(int n, const float* const* parts, const int32_t* S, const int64_t* M, const int64_t* N,
                        const int64_t* ld_part, float* const* outs, const int64_t* ld_out, cudaStream_t st) {
  for (int b0 = 0; b0 < n; b0 += MAX_SPLITK_JOBS) {
    SplitkJobs jobs{};
    const int nb = std::min(n - b0, MAX_SPLITK_JOBS);
    long long nmax = 1, mmax = 1;
    for (int i = 0; i < nb; ++i) {
      const int k = b0 + i;
      if (!parts[k] || !outs[k] || S[k] < 1 || M[k] < 1 || N[k] < 1 || M[k] > INT32_MAX || N[k] > INT32_MAX ||
          ld_part[k] < N[k] || ld_out[k] < N[k])
        return fail(SG_EINVAL, "splitk_reduce_multi: bad job " + std::to_string(k));
      jobs.part[i] = parts[k];
      jobs.out[i] = outs[k];
      jobs.S[i] = S[k];
      jobs.M[i] = (int)M[k];
      jobs.N[i] = (int)N[k];
      jobs.ldp[i] = ld_part[k];
      jobs.ld_out[i] = ld_out[k];
      nmax = std::max(nmax, (long long)N[k]);
      mmax = std::max(mmax, (long long)M[k]);
    }
    const unsigned gx = (unsigned)(((nmax + 3) / 4 + 255) / 256);
    const unsigned gy = (unsigned)(mmax < 65535 ? mmax : 65535);
    SG_CUDA_TRY(launch_pdl(k_splitk_reduce_multi, dim3(gx, gy, nb), dim3(256), 0, st, jobs));
    SG_CUDA_TRY(cudaGetLastError());
  }
  return SG_OK;
}

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
