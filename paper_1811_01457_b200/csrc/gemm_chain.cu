// Persistent GEMM chain: a whole pass of a Dense chain's training step (every
// layer's forward GEMM, or every layer's dX and dW GEMMs) in ONE launch.
//
// Why: the deep narrow MLP (c5: 16 x 1024, batch 32768) runs 47 GEMMs of
// ~55 us per step, and each GEMM launch costs a pipeline fill, a drain of its
// last epilogue and a partial last wave (tools/gemm_trace.py step: 488 us of
// 3.08 ms between GEMMs); at the 8-GPU shard size (batch 4096) every GEMM is a
// single 12 us wave and the gaps are 35 % of the step.  Here the CTA pairs of
// ONE persistent grid walk per-pair lists of work units (256 x 256 output
// tiles, or K-splits of them) across all the chain's GEMMs; a unit waits only
// for the rows of earlier GEMMs it reads (row-block arrival counters in
// global memory, release / acquire at GPU scope, async-proxy fences around
// the TMA traffic), so layer l+1 starts on a row block as soon as layer l
// has written it, and the tensor cores never drain between layers.
//
// Units are the same tiles the single-GEMM CTA-pair kernel (gemm_tc.cu)
// computes, with the same k order, epilogues and split-K summation order
// (fixed, ascending split index), so a chained step is bit-identical to the
// layer-by-layer one.  Split-K tiles are finished inside the kernel: the last
// of a tile's splits to arrive (per 32 x 128 epilogue region) sums the fp32
// partials in split order and writes the output.
//
// The schedule is planned on the host (sg_chain_create): units in the
// chain's order (problem, row block, column block, split), each assigned to
// the CTA pair that a list-scheduling simulation frees first.  Every pair
// processes its list in that global order and dependencies point to earlier
// units only, so the lowest unfinished unit can always progress (no
// deadlock with all CTAs resident: one CTA per SM, grid <= SMs).
//
// Reference: the Dense layer and its adjoints (nn_train.py:189-196,
// rules.py:45-46, 82-94, 113-124, tensor.py:351-361) -- see gemm_tc.cu.
#include <algorithm>
#include <vector>

#include "gemm_tc_dev.cuh"

namespace sg {
int ctx_activate(sg_ctx* ctx);
int ctx_compute_sms(sg_ctx* ctx);

namespace chain {

using namespace tc;

constexpr int PM = 256, PN = 256, HALF = 128, CBK = 64;  // pair tile, k-block (bf16)
// SGB200_CHAIN_WIDE=1: wide epilogue slots + 5 operand stages; default: the
// standalone kernels' narrow slots + 6 stages (2 % faster per chained unit)
template <bool WIDE> struct ChainCfg {
  static constexpr int STAGES = WIDE ? 5 : 6;
};
constexpr int SLOTS = 2 * EPI_WARPS;                     // epilogue warps per pair tile

// A problem's tensor maps live in global memory (TMA reads them there); the
// rest of its description is in the kernel's parameter space, so the
// epilogue reads it through the constant cache with no alias reloads.
struct Maps {
  CUtensorMap a, b, lp, f32, aux;
};
constexpr int MAX_PROBS = 84;  // the problems live in the 32 KB kernel parameter space

struct Problem {
  KParams p;
  int a_mn, b_mn;
  int m_tiles, n_tiles, num_kb;
  int signal;     // dependents exist: arrivals counted in cnt[cnt_off + row block]
  int cnt_off;
  int split_off;  // split-K arrival counters: [tile][SLOTS] from here
  int ndeps;
  int dep_kind[2], dep_cnt_off[2], dep_target[2], dep_m_tiles[2];
};

struct Unit {
  int prob, mb, nb, split;
};

struct Params {
  const Maps* maps;     // [n problems]
  const Unit* units;    // the pairs' lists, concatenated
  const int* list_off;  // [pairs + 1]
  unsigned* cnt;        // row-block arrival counters (zero between launches)
  unsigned* split_cnt;  // split-K arrival counters (reset by their last arriver)
  unsigned* done;       // CTAs finished; the last one clears cnt
  int n_cnt;
  int defer;  // deferred row publishing (SGB200_CHAIN_DEFER, default on)
  Problem probs[MAX_PROBS];
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Producer: block until every row of earlier GEMMs this unit's A operand
// (or, for ALL, anything of them) reads is written.
__device__ __forceinline__ void wait_deps(const Params& P, const Problem& pr, const Unit& un, int kb0, int kb1) {
  for (int d = 0; d < pr.ndeps; ++d) {
    int r0, r1;
    if (pr.dep_kind[d] == SG_DEP_ROWS) {
      r0 = r1 = un.mb;
    } else if (pr.dep_kind[d] == SG_DEP_KROWS) {
      r0 = (kb0 * CBK) / PM;
      r1 = (kb1 * CBK - 1) / PM;
    } else {
      r0 = 0;
      r1 = pr.dep_m_tiles[d] - 1;
    }
    r1 = min(r1, pr.dep_m_tiles[d] - 1);
    const unsigned target = (unsigned)pr.dep_target[d];
    for (int rb = r0; rb <= r1; ++rb) {
      const unsigned* c = P.cnt + pr.dep_cnt_off[d] + rb;
      while (ld_acquire(c) < target) __nanosleep(64);
    }
  }
  fence_proxy_async_global();  // the TMA reads below come after what the acquires made visible
}

// Epilogue warp: publish this warp's part of a finished tile to dependents
// (its TMA stores complete, then a release increment).
__device__ __forceinline__ void signal_rows(const Params& P, const Problem& pr, int mb, int lane) {
  __syncwarp();
  if (lane == 0) {
    bulk_wait0();                // this warp's TMA stores have landed
    fence_proxy_async_global();  // async-proxy writes ordered before the generic release
    if (!pr.p.tma_lp && !pr.p.tma_f32) __threadfence();  // direct stores of the warp (seen through __syncwarp)
    red_release(P.cnt + pr.cnt_off + mb, 1u);
  }
}

// Bulk store groups one chunk of a problem's epilogue commits (a chunk's
// TMA stores: fp32 and / or bf16 output, or the second bf16 output).
__device__ __forceinline__ int chunk_groups(const KParams& p) {
  if (p.splits > 1) return 0;
  const GemmEpilogue& e = p.epi;
  return (e.out_f32 && p.tma_f32) + (e.out_bf16 && p.tma_lp) + (e.out2_bf16 && p.tma_o2);
}
// Deferred publish: called after the NEXT unit's first chunk, whose `newer`
// store groups may still be in flight -- every older group (the published
// unit's stores) has completed once at most `newer` are pending.
__device__ __forceinline__ void signal_rows_deferred(const Params& P, const Problem& pr, int mb, int lane,
                                                     int newer) {
  __syncwarp();
  if (lane == 0) {
    if (newer <= 0) bulk_wait0();
    else if (newer == 1) asm volatile("cp.async.bulk.wait_group 1;" ::: "memory");
    else if (newer == 2) asm volatile("cp.async.bulk.wait_group 2;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group 3;" ::: "memory");
    fence_proxy_async_global();
    if (!pr.p.tma_lp && !pr.p.tma_f32) __threadfence();
    red_release(P.cnt + pr.cnt_off + mb, 1u);
  }
}

// Split-K: the last split to arrive for a region finishes it (split_region_fixup)
// and publishes the finished rows to dependents.
__device__ __forceinline__ void split_fixup(const Params& P, const Problem& pr, const Unit& un, int slot_id,
                                            int row0, int n_first, int chunks, int lane) {
  unsigned* c = P.split_cnt + pr.split_off + (un.mb * pr.n_tiles + un.nb) * SLOTS + slot_id;
  if (!split_region_fixup(pr.p, c, row0, n_first, chunks, lane)) return;
  if (pr.signal) {
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      red_release(P.cnt + pr.cnt_off + un.mb, 1u);
    }
  }
}

template <bool WIDE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
gemm_chain_kernel(const __grid_constant__ Params P) {
  constexpr int CSTAGES = ChainCfg<WIDE>::STAGES;
  constexpr int A_BYTES = HALF * ROW_BYTES;
  constexpr int B_BYTES = HALF * ROW_BYTES;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * PN;
  using E = Elem<false>;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + CSTAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + CSTAGES;
  uint64_t* acc_full = empty_bar + CSTAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  uint32_t* last_flag = tmem_slot + 1;
  uint8_t* stage_slots = smem + CSTAGES * STAGE_BYTES + 1024;
  uint64_t* aux_bar = reinterpret_cast<uint64_t*>(smem + CSTAGES * STAGE_BYTES + 512);

  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int pair = blockIdx.x / 2;
  const int u0 = P.list_off[pair], u1 = P.list_off[pair + 1];

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < CSTAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2 * EPI_WARPS);
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
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  grid_dep_wait();
  grid_dep_launch();
  SG_TRACE_BEGIN();

  if (warp < EPI_WARP0) {
  // registers to the epilogue warpgroups (warpgroup-collective; as gemm_tc_kernel)
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int i = u0; i < u1; ++i) {
        const Unit un = P.units[i];
        const Problem& pr = P.probs[un.prob];
        const int kb0 = un.split * pr.p.kb_per_split;
        const int kb1 = min(pr.num_kb, kb0 + pr.p.kb_per_split);
        wait_deps(P, pr, un, kb0, kb1);
        const int am = un.mb * PM + (int)rank * HALF, bn = un.nb * PN + (int)rank * HALF;
        const bool a_mn = pr.a_mn, b_mn = pr.b_mn;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t fb = mapa_shared(smem_u32(&full_bar[stage]), 0);
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          const int k0 = kb * CBK;
          if (a_mn) {
#pragma unroll
            for (int j = 0; j < HALF / CBK; ++j)
              tma_load_3d_pair(sa + j * E::MN_CHUNK, &P.maps[un.prob].a, fb, am + CBK * j, k0, 0);
          } else {
            tma_load_3d_pair(sa, &P.maps[un.prob].a, fb, k0, am, 0);
          }
          if (b_mn) {
#pragma unroll
            for (int j = 0; j < HALF / CBK; ++j)
              tma_load_3d_pair(sb + j * E::MN_CHUNK, &P.maps[un.prob].b, fb, bn + CBK * j, k0, 0);
          } else {
            tma_load_3d_pair(sb, &P.maps[un.prob].b, fb, k0, bn, 0);
          }
          if (++stage == CSTAGES) {
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
      for (int i = u0; i < u1; ++i) {
        const Unit un = P.units[i];
        const Problem& pr = P.probs[un.prob];
        const int kb0 = un.split * pr.p.kb_per_split;
        const int kb1 = min(pr.num_kb, kb0 + pr.p.kb_per_split);
        const bool a_mn = pr.a_mn, b_mn = pr.b_mn;
        const uint32_t idesc = idesc_tc(PM, PN, a_mn, b_mn, false);
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * PN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (kb == kb0) SG_TRACE(i - u0, 0);  // MMA starts
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < E::KSTEPS; ++k) {
            const uint64_t ad = a_mn ? sdesc(sa + k * E::MN_KSTEP, E::MN_CHUNK, E::MN_SBO, E::MN_LAYOUT)
                                     : sdesc(sa + k * 32, 16, 1024);
            const uint64_t bd = b_mn ? sdesc(sb + k * E::MN_KSTEP, E::MN_CHUNK, E::MN_SBO, E::MN_LAYOUT)
                                     : sdesc(sb + k * 32, 16, 1024);
            tc_mma_pair<false>(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          tc_commit_pair(&empty_bar[stage]);
          if (++stage == CSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair(&acc_full[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
    // ===================== epilogue (both CTAs, own 128 rows) =====================
    const int ew = warp - EPI_WARP0;
    const int q = ew % 4;
    const int half = ew / 4;
    constexpr int CH_PER = (PN / 32) / 2;
    const uint32_t acc_empty_leader0 = mapa_shared(smem_u32(&acc_empty[0]), 0);
    const uint32_t acc_empty_leader1 = mapa_shared(smem_u32(&acc_empty[1]), 0);
    int acc = 0;
    uint32_t acc_phase = 0, aux_phase = 0;
    int next_buf = 0;
    uint8_t* slot = stage_slots + ew * Slot<WIDE>::BYTES;
    uint64_t* my_aux = &aux_bar[2 * ew];
    // A finished unit's rows are published once its TMA stores have landed.
    // Waiting for them right after the unit costs the epilogue 1-1.5 us per
    // unit; when the next unit's accumulator is already complete (its
    // operands did not wait for these rows, so deferring cannot deadlock),
    // the publish moves behind that unit's first chunk instead, by which time
    // the stores have landed.  SGB200_CHAIN_DEFER=0 publishes at once.
    int pend_mb = -1, pend_prob = 0;
    const bool defer = P.defer;
    for (int i = u0; i < u1; ++i) {
      const Unit un = P.units[i];
      const Problem& pr = P.probs[un.prob];
      const KParams& p = pr.p;
      const int m0 = un.mb * PM, n0t = un.nb * PN;
      const int row0 = m0 + (int)rank * HALF + q * 32;
      const int c0 = half * CH_PER;
      const bool staged = p.aux_stage && row0 < p.M;
      const Maps* mp = &P.maps[un.prob];
      epi_aux_prologue<WIDE>(staged, lane, slot, &mp->aux, my_aux, n0t + c0 * 32, CH_PER, p.N, row0);
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      if (ew == 0 && lane == 0) SG_TRACE(i - u0, 1);  // accumulator complete
      auto publish_pending = [&]() {
        if (pend_mb >= 0) {
          // the groups chunk 0 committed: none when this warp's 32-row group
          // lies past M (epi_chunk returns before its stores) -- then every
          // pending group is the published unit's and must complete
          signal_rows_deferred(P, P.probs[pend_prob], pend_mb, lane, row0 < p.M ? chunk_groups(p) : 0);
          pend_mb = -1;
        }
      };
      epi_chunks<WIDE>(p, tmem_base + acc * PN + ((uint32_t)(q * 32) << 16), n0t + c0 * 32, c0, CH_PER, row0, lane,
                       un.split, 0, false, slot, staged, &mp->aux, my_aux, aux_phase, &mp->lp, &mp->f32, next_buf,
                       publish_pending);
      if (pend_mb >= 0) {  // no chunk of this warp's half was inside N: nothing newer in flight
        signal_rows_deferred(P, P.probs[pend_prob], pend_mb, lane, 0);
        pend_mb = -1;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc == 0 ? acc_empty_leader0 : acc_empty_leader1);
      if (lane == 0 && ew == 0) SG_TRACE(i - u0, 2);  // chunks done, accumulator released
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (p.splits > 1) {
        split_fixup(P, pr, un, (int)rank * EPI_WARPS + ew, row0, n0t + c0 * 32, CH_PER, lane);
      } else if (pr.signal) {
        int ready = 0;  // the next unit's accumulator is complete (warp-uniform via lane 0)
        if (defer && i + 1 < u1 && lane == 0) ready = mbar_test(&acc_full[acc], acc_phase);
        ready = __shfl_sync(0xffffffffu, ready, 0);
        if (ready) {
          pend_mb = un.mb;
          pend_prob = un.prob;
        } else {
          signal_rows(P, pr, un.mb, lane);
        }
      }
      if (lane == 0 && ew == 0) SG_TRACE(i - u0, 3);  // warp 0 done (signal / split fix-up included)
    }
  }
  if (warp >= EPI_WARP0 && lane == 0) bulk_wait0();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
  SG_TRACE_END();
  // the last CTA to finish clears the row-block counters for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned old = atomicAdd(P.done, 1u);
    *last_flag = old == gridDim.x - 1;
  }
  __syncthreads();
  if (*last_flag) {
    __threadfence();
    for (int k = threadIdx.x; k < P.n_cnt; k += blockDim.x) P.cnt[k] = 0;
    if (threadIdx.x == 0) *P.done = 0;
    __threadfence();
  }
}

}  // namespace chain
}  // namespace sg

// ================================================================ host side
using namespace sg;

struct sg_chain {
  int device = 0;
  int grid = 0;  // CTAs (2 per pair)
  chain::Params params{};
  void* d_probs = nullptr;
  void* d_units = nullptr;
  void* d_list = nullptr;
  unsigned* d_cnt = nullptr;
  unsigned* d_split = nullptr;
  unsigned* d_done = nullptr;
  float* d_part = nullptr;
  int n_units = 0;
  double est_us = 0.0;
};

namespace {

void chain_free(sg_chain* c) {
  if (!c) return;
  for (void* p : {c->d_probs, c->d_units, c->d_list, (void*)c->d_cnt, (void*)c->d_split, (void*)c->d_done,
                  (void*)c->d_part})
    if (p) cudaFree(p);
  delete c;
}

template <bool WIDE>
constexpr size_t chain_smem() {
  return (size_t)chain::ChainCfg<WIDE>::STAGES * 2 * 128 * tc::ROW_BYTES + 1024 + 1024 +
         tc::EPI_WARPS * tc::Slot<WIDE>::BYTES;
}
static_assert(chain_smem<true>() <= 232448 && chain_smem<false>() <= 232448, "shared memory budget");
bool chain_wide() {
  static const bool w = [] {
    const char* e = std::getenv("SGB200_CHAIN_WIDE");
    return e && e[0] == '1';
  }();
  return w;
}

}  // namespace

#ifdef SGB200_GEMM_TRACE
extern "C" SG_API int sg_chain_trace_buffer(void* buf, int iters, int launches) {
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

#ifdef SGB200_GEMM_TRACE
// epilogue stage profile: on != 0 clears and enables, on == 0 disables and reads out
extern "C" SG_API int sg_chain_cprof(int on, unsigned long long* out8) {
  if (on) {
    unsigned long long z[8] = {0};
    SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_cprof, z, sizeof z));
  } else if (out8) {
    SG_CUDA_TRY(cudaMemcpyFromSymbol(out8, tc::g_cprof, 8 * sizeof(unsigned long long)));
  }
  SG_CUDA_TRY(cudaMemcpyToSymbol(tc::g_cprof_on, &on, sizeof on));
  return SG_OK;
}
#endif

extern "C" {

int sg_chain_create(sg_ctx* ctx, const sg_chain_problem* probs, int32_t n, sg_chain** out) {
  SG_NVTX("sg_chain_create");
  if (!ctx || !probs || !out || n <= 0) return fail(SG_EINVAL, "chain: null argument or empty chain");
  if (int rc = ctx_activate(ctx)) return rc;
  const int pairs = std::max(1, ctx_compute_sms(ctx) / 2);
  if (n > chain::MAX_PROBS) return fail(SG_EINVAL, "chain: at most 84 GEMMs per chain");
  std::vector<chain::Problem> hp(n);
  std::vector<chain::Maps> hm(n);
  long long n_cnt = 0, n_split = 0, n_part = 0;
  std::vector<long long> part_off(n, -1);
  for (int i = 0; i < n; ++i) {
    const sg_chain_problem& cp = probs[i];
    const sg_gemm_desc* d = &cp.gemm;
    chain::Problem& pr = hp[i];
    chain::Maps& mp = hm[i];
    std::memset(&pr, 0, sizeof pr);
    std::memset(&mp, 0, sizeof mp);
    const std::string at = "chain problem " + std::to_string(i) + ": ";
    if (d->precision != SG_PREC_BF16) return fail(SG_EINVAL, at + "chained GEMMs are BF16 tensor-core GEMMs");
    if (d->M <= 0 || d->N <= 0 || d->K <= 0 || d->M > (1ll << 31) - 1 || d->N > (1ll << 31) - 1 ||
        d->K > (1ll << 31) - 1)
      return fail(SG_EINVAL, at + "bad extents");
    if (d->batch > 1) return fail(SG_EINVAL, at + "batched GEMMs do not chain");
    if (d->epilogue < SG_EPI_STORE || d->epilogue > SG_EPI_ACT_GRAD || d->act < SG_ACT_IDENTITY ||
        d->act > SG_ACT_RELU)
      return fail(SG_EINVAL, at + "bad epilogue / activation");
    if (d->epilogue == SG_EPI_ACT_GRAD && !d->aux) return fail(SG_EINVAL, at + "ACT_GRAD needs aux");
    auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    if (!a16(d->A) || !a16(d->B) || d->lda % 8 || d->ldb % 8)
      return fail(SG_EINVAL, at + "A and B must be 16-byte aligned with lda/ldb multiples of 8 elements");
    if (d->lda < (d->a_mn_major ? d->M : d->K) || d->ldb < (d->b_mn_major ? d->N : d->K))
      return fail(SG_EINVAL, at + "leading dimension smaller than the row");
    GemmArgs g{};
    g.M = (int)d->M;
    g.N = (int)d->N;
    g.K = (int)d->K;
    g.A = d->A;
    g.lda = d->lda;
    g.a_mn = d->a_mn_major != 0;
    g.B = d->B;
    g.ldb = d->ldb;
    g.b_mn = d->b_mn_major != 0;
    g.epi.mode = d->epilogue;
    g.epi.act = d->act;
    g.epi.bias = (const float*)d->bias;
    g.epi.aux = (const __nv_bfloat16*)d->aux;
    g.epi.aux_f32 = nullptr;
    g.epi.ld_aux = d->ld_aux;
    g.epi.out_pre = (float*)d->out_pre;
    g.epi.ld_pre = d->ld_pre;
    g.epi.out_f32 = (float*)d->out;
    g.epi.ld_f32 = d->ld_out;
    g.epi.out_bf16 = (__nv_bfloat16*)d->out_lp;
    g.epi.ld_bf16 = d->ld_lp;
    g.epi.colsum = d->colsum;
    g.epi.ld_colsum = d->ld_colsum;
    g.epi.dom = ctx_domain_word(ctx);
    g.batch = 1;
    int rc = g.a_mn ? tcmap::make_map(&mp.a, g.A, g.M, g.K, g.lda, chain::CBK, false, true, 1, 0)
                    : tcmap::make_map(&mp.a, g.A, g.K, g.M, g.lda, 128, false, false, 1, 0);
    if (rc) return rc;
    rc = g.b_mn ? tcmap::make_map(&mp.b, g.B, g.N, g.K, g.ldb, chain::CBK, false, true, 1, 0)
                : tcmap::make_map(&mp.b, g.B, g.K, g.N, g.ldb, 128, false, false, 1, 0);
    if (rc) return rc;
    pr.num_kb = (g.K + chain::CBK - 1) / chain::CBK;
    pr.m_tiles = (g.M + chain::PM - 1) / chain::PM;
    pr.n_tiles = (g.N + chain::PN - 1) / chain::PN;
    int splits = std::max(1, (int)cp.splits);
    if (splits > 1) {
      if (g.epi.mode != SG_EPI_STORE || g.epi.colsum || g.epi.out_pre || !g.epi.out_f32 || g.epi.out_bf16)
        return fail(SG_EINVAL, at + "split-K problems take the STORE epilogue into an fp32 output only");
      splits = std::min(splits, pr.num_kb);
    }
    const int kb_per = (pr.num_kb + splits - 1) / splits;
    splits = (pr.num_kb + kb_per - 1) / kb_per;
    pr.p = tc::KParams{g.M, g.N, g.K, g.epi, splits, kb_per, nullptr, 0, 0, 0, 0, 8, 0, 0, 1, 0, 0};
    tcmap::out_maps(g, pr.p, mp.lp, mp.f32);
    tcmap::aux_map(g, pr.p, mp.aux, false);
    if (splits > 1) {
      pr.p.ld_part = (g.N + 3) / 4 * 4;
      part_off[i] = n_part;
      n_part += (long long)splits * g.M * pr.p.ld_part;
      pr.split_off = (int)n_split;
      n_split += (long long)pr.m_tiles * pr.n_tiles * chain::SLOTS;
    }
    pr.a_mn = g.a_mn;
    pr.b_mn = g.b_mn;
    pr.ndeps = std::max(0, std::min(2, (int)cp.n_deps));
    for (int k = 0; k < pr.ndeps; ++k) {
      const int q = cp.dep_on[k];
      const int kind = cp.dep_kind[k];
      if (q < 0 || q >= i) return fail(SG_EINVAL, at + "dependencies must point to earlier problems");
      const sg_gemm_desc* dq = &probs[q].gemm;
      if (kind == SG_DEP_ROWS && (g.a_mn || dq->M != d->M))
        return fail(SG_EINVAL, at + "ROWS dependency: A must be K-major with the producer's rows");
      if (kind == SG_DEP_KROWS && (!g.a_mn || dq->M != d->K))
        return fail(SG_EINVAL, at + "KROWS dependency: A must be MN-major over the producer's rows");
      if (kind != SG_DEP_ROWS && kind != SG_DEP_KROWS && kind != SG_DEP_ALL)
        return fail(SG_EINVAL, at + "unknown dependency kind");
      hp[q].signal = 1;
      pr.dep_kind[k] = kind;
      pr.dep_m_tiles[k] = (int)((dq->M + chain::PM - 1) / chain::PM);
      pr.dep_target[k] = (int)(((dq->N + chain::PN - 1) / chain::PN) * chain::SLOTS);
      // dep_cnt_off is filled below, once every problem's counter block is known
      pr.dep_cnt_off[k] = q;
    }
  }
  for (int i = 0; i < n; ++i) {
    hp[i].cnt_off = (int)n_cnt;
    n_cnt += hp[i].m_tiles;
  }
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < hp[i].ndeps; ++k) hp[i].dep_cnt_off[k] = hp[hp[i].dep_cnt_off[k]].cnt_off;

  // ---- list schedule: units in chain order, each to the pair freed first
  const double pair_flops = 26.0e12;  // bf16 pair-tile MMA rate, FLOP/s (tools/gemm_trace.py)
  std::vector<double> pair_free(pairs, 0.0);
  std::vector<std::vector<chain::Unit>> lists(pairs);
  std::vector<std::vector<double>> rb_done(n);
  double makespan = 0.0;
  for (int i = 0; i < n; ++i) {
    const chain::Problem& pr = hp[i];
    rb_done[i].assign(pr.m_tiles, 0.0);
    for (int mb = 0; mb < pr.m_tiles; ++mb)
      for (int nb = 0; nb < pr.n_tiles; ++nb)
        for (int s = 0; s < pr.p.splits; ++s) {
          const int kb0 = s * pr.p.kb_per_split, kb1 = std::min(pr.num_kb, kb0 + pr.p.kb_per_split);
          double ready = 0.0;
          for (int k = 0; k < pr.ndeps; ++k) {
            const int q = probs[i].dep_on[k];
            int r0 = 0, r1 = hp[q].m_tiles - 1;
            if (pr.dep_kind[k] == SG_DEP_ROWS) r0 = r1 = mb;
            if (pr.dep_kind[k] == SG_DEP_KROWS) {
              r0 = kb0 * chain::CBK / chain::PM;
              r1 = std::min(hp[q].m_tiles - 1, (kb1 * chain::CBK - 1) / chain::PM);
            }
            for (int r = r0; r <= r1; ++r) ready = std::max(ready, rb_done[q][r]);
          }
          int best = 0;
          for (int pp = 1; pp < pairs; ++pp)
            if (pair_free[pp] < pair_free[best]) best = pp;
          const double cost = 2.0 * chain::PM * chain::PN * (double)(kb1 - kb0) * chain::CBK / pair_flops + 0.3e-6;
          const double start = std::max(pair_free[best], ready);
          pair_free[best] = start + cost;
          rb_done[i][mb] = std::max(rb_done[i][mb], start + cost);
          makespan = std::max(makespan, start + cost);
          lists[best].push_back(chain::Unit{i, mb, nb, s});
        }
  }
  std::vector<chain::Unit> units;
  std::vector<int> list_off(pairs + 1, 0);
  for (int pp = 0; pp < pairs; ++pp) {
    list_off[pp] = (int)units.size();
    units.insert(units.end(), lists[pp].begin(), lists[pp].end());
  }
  list_off[pairs] = (int)units.size();

  sg_chain* c = new sg_chain();
  cudaGetDevice(&c->device);
  c->grid = 2 * pairs;
  c->n_units = (int)units.size();
  c->est_us = makespan * 1e6;
  auto alloc = [&](void** p, size_t bytes) { return cudaMalloc(p, bytes < 64 ? 64 : bytes); };
  cudaError_t e = alloc(&c->d_probs, sizeof(chain::Maps) * n);
  if (e == cudaSuccess) e = alloc(&c->d_units, sizeof(chain::Unit) * units.size());
  if (e == cudaSuccess) e = alloc(&c->d_list, sizeof(int) * list_off.size());
  if (e == cudaSuccess) e = alloc((void**)&c->d_cnt, sizeof(unsigned) * std::max(1ll, n_cnt));
  if (e == cudaSuccess) e = alloc((void**)&c->d_split, sizeof(unsigned) * std::max(1ll, n_split));
  if (e == cudaSuccess) e = alloc((void**)&c->d_done, sizeof(unsigned));
  if (e == cudaSuccess && n_part) e = alloc((void**)&c->d_part, sizeof(float) * n_part);
  if (e != cudaSuccess) {
    chain_free(c);
    return cuda_fail(e, "chain: device allocation");
  }
  for (int i = 0; i < n; ++i)
    if (part_off[i] >= 0) hp[i].p.part = c->d_part + part_off[i];
  e = cudaMemcpy(c->d_probs, hm.data(), sizeof(chain::Maps) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_units, units.data(), sizeof(chain::Unit) * units.size(),
                                       cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(c->d_list, list_off.data(), sizeof(int) * list_off.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(c->d_cnt, 0, sizeof(unsigned) * std::max(1ll, n_cnt));
  if (e == cudaSuccess) e = cudaMemset(c->d_split, 0, sizeof(unsigned) * std::max(1ll, n_split));
  if (e == cudaSuccess) e = cudaMemset(c->d_done, 0, sizeof(unsigned));
  if (e != cudaSuccess) {
    chain_free(c);
    return cuda_fail(e, "chain: upload");
  }
  c->params.maps = static_cast<const chain::Maps*>(c->d_probs);
  for (int i = 0; i < n; ++i) c->params.probs[i] = hp[i];
  c->params.units = static_cast<const chain::Unit*>(c->d_units);
  c->params.list_off = static_cast<const int*>(c->d_list);
  c->params.cnt = c->d_cnt;
  c->params.split_cnt = c->d_split;
  c->params.done = c->d_done;
  c->params.n_cnt = (int)n_cnt;
  {
    const char* e = std::getenv("SGB200_CHAIN_DEFER");
    c->params.defer = !(e && e[0] == '0');
  }
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    e = cudaFuncSetAttribute(chain::gemm_chain_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)chain_smem<true>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(chain::gemm_chain_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)chain_smem<false>());
    if (e != cudaSuccess) {
      chain_free(c);
      return cuda_fail(e, "chain: kernel attributes");
    }
  }
  *out = c;
  return SG_OK;
}

int sg_chain_run(sg_chain* c, void* stream) {
  SG_NVTX("sg_chain_run");
  if (!c) return fail(SG_EINVAL, "null chain");
  SG_CUDA_TRY(cudaSetDevice(c->device));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c->grid);
  cfg.blockDim = dim3(tc::NUM_THREADS);
  const bool wide = chain_wide();
  cfg.dynamicSmemBytes = wide ? chain_smem<true>() : chain_smem<false>();
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (wide) SG_CUDA_TRY(cudaLaunchKernelEx(&cfg, chain::gemm_chain_kernel<true>, c->params));
  else SG_CUDA_TRY(cudaLaunchKernelEx(&cfg, chain::gemm_chain_kernel<false>, c->params));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

int sg_chain_info(const sg_chain* c, int32_t* units, int32_t* ctas, double* est_us) {
  if (!c) return fail(SG_EINVAL, "null chain");
  if (units) *units = c->n_units;
  if (ctas) *ctas = c->grid;
  if (est_us) *est_us = c->est_us;
  return SG_OK;
}

int sg_chain_destroy(sg_chain* c) {
  if (!c) return SG_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  chain_free(c);
  return SG_OK;
}

}  // extern "C"
