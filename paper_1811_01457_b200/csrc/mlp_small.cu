// One-launch training step for small Dense chains (c1: MLP 784-32-10, batch 128).
//
// The reference step (nn_train.py:337-375 / the c1 loss IR of SURVEY §8(d)):
// forward `act(h W^T + b)` per layer (nn_train.py:189-210), loss + seed,
// pullback (rules.py:45-46, 82-94, 113-124), then `p - lr * g` over the flat
// parameter list.  For chains this small the step is latency-bound (13 MFLOP
// for c1): ten separate kernels cost ~4.5 us each even inside a CUDA graph,
// so the whole step runs as ONE cooperative kernel with a single grid-wide
// barrier, fp32 on the CUDA cores:
//
//   phase 1 (rows):    each CTA owns R <= 4 minibatch rows and runs them
//                      through the forward, the loss and the pullback down
//                      to dZ of layer 0 -- all row-local work, activations in
//                      shared memory, weights read from L2 (coalesced rows);
//                      dZ_l and h_l are published to a global scratch area.
//   grid barrier
//   phase 2 (columns): the weight gradients are the reductions over rows,
//                      g[j][k] = sum_r dZ_l[r][j] * h_l[r][k] (k = fan_in is
//                      the bias column, h = 1), ascending r (the reference's
//                      matmul fold order, tensor.py:351-361, in fp32).  Chunks
//                      of 16 columns are spread over the CTAs; each CTA stages
//                      dZ_l and its h columns in shared memory, writes G and
//                      applies SGD to P (and the bf16 shadow) in place.
//
// Deterministic: every sum has a fixed order independent of the launch.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.h"

namespace sg {
int ctx_num_sms(sg_ctx* ctx);
int ctx_activate(sg_ctx* ctx);

namespace ms {

constexpr int MAXL = SG_MLP_SMALL_MAXL;
constexpr int MAXR = 4;      // rows per CTA in phase 1
constexpr int NT = 512;      // threads per CTA
constexpr int KW = 16;       // phase 2: columns per chunk
constexpr int MAXD = 1024;   // widest layer
constexpr int MAX_CTAS = 128;

struct Params {
  int L, B, R, loss;
  int d[MAXL + 1];
  int act[MAXL];
  long long w_off[MAXL], b_off[MAXL], ldw[MAXL];
  float scale, lr;
  float* P;
  float* G;
  __nv_bfloat16* S;
  const float* X;
  long long ldx;
  const float* Y;
  long long ldy;
  float* Z;  // optional top-layer output [B][ldz]
  long long ldz;
  double* loss_out;
  unsigned* dom;       // domain flags (SG_DOM_*, sg_domain_check)
  // scratch
  unsigned* bar;       // {arrivals, generation}
  double* loss_part;   // [B]
  float* hg;           // h_l, l = 1..L-1: hg + h_off[l] + r * d[l]
  float* dzg;          // dZ_l, l = 0..L-1: dzg + dz_off[l] + r * d[l+1]
  long long h_off[MAXL + 1], dz_off[MAXL];
  int chunks;          // phase 2 work items: sum over layers of ceil((d[l] + 1) / KW)
  int wstage;          // 1: every W_l is staged in shared memory by bulk copies (TMA) at launch
  long long ws_base;   // float offset of the staged weights in shared memory (128-byte aligned)
  long long ws_off[MAXL];
  int k4[MAXL];        // staged row stride (fan_in rounded up to 4 floats = 16 bytes)
};

__device__ __forceinline__ float act_f(float z, int a);
// act_f plus the reference's overflow condition: scalar_sigmoid's math.exp(-z)
// raises OverflowError for z < -709.78 (tensor.py:214-215)
__device__ __forceinline__ float act_dom(float z, int a, unsigned* dom) {
  if (a == SG_ACT_SIGMOID && z <= SIGMOID_OVF_F32 && dom) atomicOr(dom, (unsigned)SG_DOM_EXP_OVERFLOW);
  return act_f(z, a);
}
// The c1 loss IR's float64 domain conditions for one softmax row z[0..N)
// (exp overflow, row sum == 0, exp(z_j)/sum == 0; see include/sgb200.h),
// evaluated exactly only when the row holds an extreme logit.  Warp-collective.
__device__ __forceinline__ void softmax_row_domain(const float* z, int N, int lane, float mx, unsigned* dom) {
  float mn = INFINITY;
  for (int c = lane; c < N; c += 32) mn = fminf(mn, z[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (!dom || ((double)mx <= 700.0 && (double)mn >= -700.0)) return;
  if ((double)mx > EXP_MAX_ARG) {
    if (lane == 0) atomicOr(dom, (unsigned)SG_DOM_EXP_OVERFLOW);
    return;
  }
  double se = 0.0;
  for (int c = lane; c < N; c += 32) se += exp((double)z[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  if (se == 0.0) {
    if (lane == 0) atomicOr(dom, (unsigned)SG_DOM_DIV_ZERO);
    return;
  }
  bool zero = false;
  for (int c = lane; c < N; c += 32) zero |= !(exp((double)z[c]) / se > 0.0) && !isnan(z[c]);
  if (__any_sync(0xffffffffu, zero) && lane == 0) atomicOr(dom, (unsigned)SG_DOM_LOG_NONPOS);
}
__device__ __forceinline__ float act_f(float z, int a) {
  switch (a) {
    case SG_ACT_SIGMOID: return 1.0f / (1.0f + expf(-z));  // tensor.py:214-215
    case SG_ACT_TANH: return tanhf(z);
    case SG_ACT_RELU: return z > 0.0f ? z : 0.0f;
    default: return z;
  }
}
// d act / d z through the saved output h (rules.py:82-94)
__device__ __forceinline__ float act_grad_f(float h, int a) {
  switch (a) {
    case SG_ACT_SIGMOID: return h * (1.0f - h);
    case SG_ACT_TANH: return 1.0f - h * h;
    case SG_ACT_RELU: return h > 0.0f ? 1.0f : 0.0f;
    default: return 1.0f;
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* q) { return (uint32_t)__cvta_generic_to_shared(q); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(done)
                 : "r"(smem_u32(bar))
                 : "memory");
  } while (!done);
}

// Sense-reversal grid barrier (the launch is cooperative: all CTAs resident).
// The counter is back at 0 after every use, the generation only grows.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// MR: rows per CTA (compile time, >= p.R) -- no FMAs on duplicated rows
template <int MR>
__global__ void __launch_bounds__(NT, 1) k_mlp_small_step(const __grid_constant__ Params p) {
  extern __shared__ float sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int L = p.L;

  // ------------------------------------------------------------ phase 1
  {
    const int r0 = blockIdx.x * p.R;
    const int nr = max(0, min(p.R, p.B - r0));
    // shared: h_0..h_L (R x d[l] each), then two dZ buffers of R x max width.
    // Offsets, not a pointer array: a local pointer array turns every access
    // into a generic LD/ST instead of LDS/STS.
    auto hs = [&](int l) -> float* {
      int o = 0;
      for (int i = 0; i < l; ++i) o += p.R * p.d[i];
      return sm + o;
    };
    int dmax = 0;
    for (int l = 1; l <= L; ++l) dmax = max(dmax, p.d[l]);
    float* dz_a = hs(L + 1 - 1) + p.R * p.d[L];
    float* dz_b = dz_a + p.R * dmax;

    // weights: one bulk copy per W row into shared memory, all on one
    // mbarrier, in flight while the input rows load (one L2 round trip)
    __shared__ uint64_t wbar;
    float* ws = sm + p.ws_base;
    if (p.wstage) {
      if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
      if (warp == 0) {
        if (lane == 0) {
          uint32_t total = 0;
          for (int l = 0; l < L; ++l) total += (uint32_t)p.d[l + 1] * p.k4[l] * 4u;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&wbar)), "r"(total)
                       : "memory");
        }
        __syncwarp();
        for (int l = 0; l < L; ++l)
          for (int j = lane; j < p.d[l + 1]; j += 32)
            bulk_g2s(ws + p.ws_off[l] + (long long)j * p.k4[l], p.P + p.w_off[l] + (long long)j * p.ldw[l],
                     (uint32_t)p.k4[l] * 4u, &wbar);
      }
    }
    // input rows (fp32)
    for (int i = tid; i < nr * p.d[0]; i += NT) {
      const int r = i / p.d[0], k = i - r * p.d[0];
      hs(0)[i] = p.X[(long long)(r0 + r) * p.ldx + k];
    }
    __syncthreads();
    if (p.wstage) mbar_wait0(&wbar);

    // forward: warp per output column j, lanes split K (coalesced W rows).
    // The step is latency-bound, so every W row is fetched with all of its
    // loads in flight at once (one L2 round trip per column, K <= 1024).
    for (int l = 0; l < L; ++l) {
      const int K = p.d[l], N = p.d[l + 1];
      const float* W = p.P + p.w_off[l];
      const float* bias = p.P + p.b_off[l];
      if (p.wstage) {  // weights in shared memory: warp per column, lanes split K
        const float* wl = ws + p.ws_off[l];
        const float* h0 = hs(l);
        for (int j = warp; j < N; j += NW) {
          const float* w = wl + (long long)j * p.k4[l];
          const float bj = __ldg(bias + j);  // issued before the dot product, not after it
          float acc[MR];
#pragma unroll
          for (int r = 0; r < MR; ++r) acc[r] = 0.0f;
#pragma unroll 8
          for (int k = lane; k < K; k += 32) {
            const float wv = w[k];
#pragma unroll
            for (int r = 0; r < MR; ++r) acc[r] = fmaf(h0[min(r, nr - 1) * K + k], wv, acc[r]);
          }
#pragma unroll
          for (int r = 0; r < MR; ++r) acc[r] = warp_sum(acc[r]);
          if (lane < nr) {
            float z = 0.0f;
#pragma unroll
            for (int r = 0; r < MR; ++r)
              if (r == lane) z = acc[r];
            hs(l + 1)[lane * N + j] = act_dom(z + bj, p.act[l], p.dom);
          }
        }
        __syncthreads();
        continue;
      }
      const int rot = (blockIdx.x * NW) % N;  // CTAs start on different W rows (spreads L2 slices)
      for (int jj = warp; jj < N; jj += NW) {
        const int j = jj + rot < N ? jj + rot : jj + rot - N;
        const float* w = W + (long long)j * p.ldw[l];
        float wv[MAXD / 32];
#pragma unroll
        for (int i = 0; i < MAXD / 32; ++i) {  // clamped address: the load may be issued unpredicated
          const float t = __ldg(w + min(lane + 32 * i, K - 1));
          wv[i] = lane + 32 * i < K ? t : 0.0f;
        }
        const float bj = __ldg(bias + j);
        // branch-free (clamped indices, zero weights past K, rows past nr
        // duplicate the last one): a guarded FMA lets the compiler sink each
        // load into its branch and serialise the L2 round trips
        float acc[MR];
#pragma unroll
        for (int r = 0; r < MR; ++r) acc[r] = 0.0f;
        const float* h0 = hs(l);
#pragma unroll
        for (int i = 0; i < MAXD / 32; ++i) {
          const int k = min(lane + 32 * i, K - 1);
#pragma unroll
          for (int r = 0; r < MR; ++r) acc[r] = fmaf(h0[min(r, nr - 1) * K + k], wv[i], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < MR; ++r) acc[r] = warp_sum(acc[r]);
        if (lane < nr) {
          float z = 0.0f;
#pragma unroll
          for (int r = 0; r < MR; ++r)
            if (r == lane) z = acc[r];
          hs(l + 1)[lane * N + j] = act_dom(z + bj, p.act[l], p.dom);
        }
      }
      __syncthreads();
    }

    // loss + seed: warp per row (top layer output h_L, width N <= MAXD)
    {
      const int N = p.d[L];
      float* dz = dz_a;  // dZ of layer L-1
      for (int r = warp; r < nr; r += NW) {
        const long long row = r0 + r;
        const float* z = hs(L) + r * N;
        const float* y = p.Y + row * p.ldy;
        double lrow = 0.0;
        if (p.loss == SG_LOSS_SOFTMAX_XENT) {
          float mx = -INFINITY;
          for (int c = lane; c < N; c += 32) mx = fmaxf(mx, z[c]);
          mx = warp_max(mx);
          softmax_row_domain(z, N, lane, mx, p.dom);
          float se = 0.0f, sy = 0.0f, syz = 0.0f;
          for (int c = lane; c < N; c += 32) {
            const float d = z[c] - mx, yc = y[c];
            se += expf(d);
            sy += yc;
            syz += yc * d;
          }
          se = warp_sum(se);
          sy = warp_sum(sy);
          syz = warp_sum(syz);
          const float lse = logf(se);
          lrow = (double)(sy * lse - syz);  // -sum y (z - mx - lse)
          for (int c = lane; c < N; c += 32) dz[r * N + c] = (expf(z[c] - mx - lse) * sy - y[c]) * p.scale;
        } else {  // MSE
          double s = 0.0;
          for (int c = lane; c < N; c += 32) {
            const float d = z[c] - y[c];
            s += (double)d * (double)d;
            dz[r * N + c] = d * p.scale + d * p.scale;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          lrow = s;
        }
        // the top layer's own activation: dz = dL/dh .* act'(h)
        if (p.act[L - 1] != SG_ACT_IDENTITY)
          for (int c = lane; c < N; c += 32) dz[r * N + c] *= act_grad_f(z[c], p.act[L - 1]);
        if (p.Z)
          for (int c = lane; c < N; c += 32) p.Z[row * p.ldz + c] = z[c];
        if (lane == 0) p.loss_part[row] = lrow;
      }
      __syncthreads();
    }

    // pullback: dZ_{l-1} = (dZ_l W_l) .* act'_{l-1}(h_l), thread per input column k
    float* cur = dz_a;
    float* nxt = dz_b;
    for (int l = L - 1; l >= 0; --l) {
      const int K = p.d[l], N = p.d[l + 1];
      // publish dZ_l (and h_l for l >= 1) for the column phase
      for (int i = tid; i < nr * N; i += NT) p.dzg[p.dz_off[l] + (long long)r0 * N + i] = cur[i];
      if (l >= 1)
        for (int i = tid; i < nr * K; i += NT) p.hg[p.h_off[l] + (long long)r0 * K + i] = hs(l)[i];
      if (l == 0) break;  // dX of the first layer is not needed
      const float* W = p.P + p.w_off[l];
      if (p.wstage) {
        const float* wl = ws + p.ws_off[l];
        for (int k = tid; k < K; k += NT) {
          float acc[MR];
#pragma unroll
          for (int r = 0; r < MR; ++r) acc[r] = 0.0f;
#pragma unroll 8
          for (int j = 0; j < N; ++j) {
            const float wv = wl[(long long)j * p.k4[l] + k];
#pragma unroll
            for (int r = 0; r < MR; ++r) acc[r] = fmaf(cur[min(r, nr - 1) * N + j], wv, acc[r]);
          }
#pragma unroll
          for (int r = 0; r < MR; ++r)
            if (r < nr) nxt[r * K + k] = acc[r] * act_grad_f(hs(l)[r * K + k], p.act[l - 1]);
        }
        __syncthreads();
        float* t = cur;
        cur = nxt;
        nxt = t;
        continue;
      }
      for (int k = tid; k < K; k += NT) {
        float acc[MR];
#pragma unroll
        for (int r = 0; r < MR; ++r) acc[r] = 0.0f;
        constexpr int JC = 16;  // W column values fetched 16 at a time, all in flight
        for (int j0 = 0; j0 < N; j0 += JC) {
          float wv[JC];
#pragma unroll
          for (int i = 0; i < JC; ++i) {
            const float t = __ldg(W + (long long)min(j0 + i, N - 1) * p.ldw[l] + k);
            wv[i] = j0 + i < N ? t : 0.0f;
          }
#pragma unroll
          for (int i = 0; i < JC; ++i) {
            const int j = min(j0 + i, N - 1);  // wv = 0 past N (branch-free, as above)
#pragma unroll
            for (int r = 0; r < MR; ++r) acc[r] = fmaf(cur[min(r, nr - 1) * N + j], wv[i], acc[r]);
          }
        }
#pragma unroll
        for (int r = 0; r < MR; ++r)
          if (r < nr) nxt[r * K + k] = acc[r] * act_grad_f(hs(l)[r * K + k], p.act[l - 1]);
      }
      __syncthreads();
      float* t = cur;
      cur = nxt;
      nxt = t;
    }
  }


  // chunk -> (layer, first column): ceil((d[l] + 1) / KW) chunks per layer
  auto chunk_of = [&](int c, int& l, int& k0) {
    l = 0;
    k0 = c;
    while ((p.d[l] + KW) / KW <= k0) {
      k0 -= (p.d[l] + KW) / KW;
      ++l;
    }
    k0 *= KW;
  };
  // What this CTA's first chunk needs that no other CTA writes -- the X
  // columns of a layer-0 chunk (cp.async into shared memory) and the P values
  // it will update (registers) -- goes in flight before the grid barrier.
  __syncthreads();  // phase-1 shared-memory traffic is over
  float pv[2] = {0.0f, 0.0f};
  const bool first = blockIdx.x < p.chunks;
  if (first) {
    int l, k0;
    chunk_of(blockIdx.x, l, k0);
    const int K = p.d[l], N = p.d[l + 1], B = p.B;
    const int kw = min(KW, K + 1 - k0);
    if (l == 0) {
      float* hcs = sm + (long long)B * N;
      for (int i = tid; i < B * KW; i += NT) {
        const int r = i / KW, kk = i - r * KW, k = k0 + kk;
        if (kk < kw && k < K)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(hcs + i)),
                       "l"(p.X + (long long)r * p.ldx + k)
                       : "memory");
        else
          hcs[i] = kk < kw ? 1.0f : 0.0f;  // bias column / past the chunk
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int o = tid + q * NT, j = o / KW, kk = o - j * KW, k = k0 + kk;
      if (o < N * KW && kk < kw)
        pv[q] = p.P[k == K ? p.b_off[l] + j : p.w_off[l] + (long long)j * p.ldw[l] + k];
    }
  }
  grid_barrier(p.bar);

  // ------------------------------------------------------------ phase 2
  // chunk = (layer l, columns k0..k0+KW) of [W_l | b_l]^T; column K is the bias.
  for (int c = blockIdx.x; c < p.chunks; c += gridDim.x) {
    int l, k0;
    chunk_of(c, l, k0);
    const bool pre = c == (int)blockIdx.x;  // prefetched above
    const int K = p.d[l], N = p.d[l + 1], B = p.B;
    const int kw = min(KW, K + 1 - k0);
    float* dzs = sm;                  // [B][N]
    float* hcs = sm + (long long)B * N;  // [B][KW]
    const float* dzl = p.dzg + p.dz_off[l];
    for (int i = tid; i < B * N; i += NT) dzs[i] = __ldcg(dzl + i);
    if (pre && l == 0) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else {
      for (int i = tid; i < B * KW; i += NT) {
        const int r = i / KW, kk = i - r * KW, k = k0 + kk;
        float v = 0.0f;
        if (kk < kw) {
          if (k == K) v = 1.0f;
          else if (l == 0) v = p.X[(long long)r * p.ldx + k];
          else v = __ldcg(p.hg + p.h_off[l] + (long long)r * K + k);
        }
        hcs[i] = v;
      }
    }
    __syncthreads();
    int q = 0;
    for (int o = tid; o < N * KW; o += NT, ++q) {
      const int j = o / KW, kk = o - j * KW, k = k0 + kk;
      if (kk >= kw) continue;
      float g = 0.0f;
      for (int r = 0; r < B; ++r) g = fmaf(dzs[r * N + j], hcs[r * KW + kk], g);  // ascending rows
      const long long idx = k == K ? p.b_off[l] + j : p.w_off[l] + (long long)j * p.ldw[l] + k;
      p.G[idx] = g;
      const float old = pre && q < 2 ? (q == 0 ? pv[0] : pv[1]) : p.P[idx];
      const float v = old - p.lr * g;  // nn_train.py:365-372
      p.P[idx] = v;
      if (p.S) p.S[idx] = __float2bfloat16_rn(v);
    }
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1) {  // loss total: row sums in a fixed tree order
    double* red = reinterpret_cast<double*>(sm);
    double v = 0.0;
    for (int r = tid; r < p.B; r += NT) v += __ldcg(p.loss_part + r);
    red[tid] = v;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
      if (tid < s) red[tid] += red[tid + s];
      __syncthreads();
    }
    if (tid == 0) *p.loss_out = red[0] * (double)p.scale;
  }
}

}  // namespace ms
}  // namespace sg

using namespace sg;

namespace {

int plan(const sg_mlp_small_desc* d, ms::Params& p, size_t& smem, size_t& scratch) {
  if (!d) return fail(SG_EINVAL, "null descriptor");
  if (d->L < 1 || d->L > ms::MAXL) return fail(SG_EINVAL, "mlp_small: 1..4 layers");
  if (d->B < 1 || d->B > ms::MAX_CTAS * ms::MAXR) return fail(SG_EINVAL, "mlp_small: batch 1..512");
  if (d->loss != SG_LOSS_SOFTMAX_XENT && d->loss != SG_LOSS_MSE)
    return fail(SG_EINVAL, "mlp_small: softmax_xent or mse loss");
  p = ms::Params{};
  p.L = d->L;
  p.B = d->B;
  p.loss = d->loss;
  p.scale = (float)d->scale;
  p.lr = (float)d->lr;
  int dmax = 0;
  long long hsum = 0;
  for (int l = 0; l <= d->L; ++l) {
    if (d->sizes[l] < 1 || d->sizes[l] > ms::MAXD) return fail(SG_EINVAL, "mlp_small: widths 1..1024");
    p.d[l] = d->sizes[l];
    hsum += d->sizes[l];
    if (l >= 1) dmax = std::max(dmax, (int)d->sizes[l]);
  }
  for (int l = 0; l < d->L; ++l) {
    p.act[l] = d->act[l];
    p.w_off[l] = d->w_off[l];
    p.b_off[l] = d->b_off[l];
    p.ldw[l] = d->ldw[l];
    if (d->ldw[l] < d->sizes[l]) return fail(SG_EINVAL, "mlp_small: ldw < fan_in");
    if ((long long)d->B * d->sizes[l + 1] + (long long)d->B * ms::KW > 56 * 1024)
      return fail(SG_EINVAL, "mlp_small: batch x width too large for the column phase");
  }
  // rows per CTA: every CTA streams all weights from L2 in phase 1; <= 64 CTAs
  // where the batch allows (c1: 2 rows each) -- measured fastest on B200
  p.R = std::max((d->B + ms::MAX_CTAS - 1) / ms::MAX_CTAS, std::min(ms::MAXR, (d->B + 63) / 64));
  if (const char* e = std::getenv("SGB200_MLP_SMALL_R"))  // tuning override
    p.R = std::max((d->B + ms::MAX_CTAS - 1) / ms::MAX_CTAS, std::min(ms::MAXR, std::atoi(e)));
  if (p.R > ms::MAXR) return fail(SG_EINVAL, "mlp_small: batch too large");
  // phase 1: h_0..h_L + two dZ buffers; phase 2: dZ_l [B][N] + h columns [B][KW]
  size_t s1 = ((size_t)p.R * hsum + 2ull * p.R * dmax) * sizeof(float);
  // stage every W_l in shared memory when it fits (rows of fan_in rounded to 16 B)
  {
    long long base = ((long long)p.R * hsum + 2ll * p.R * dmax + 31) / 32 * 32;
    long long off = 0;
    for (int l = 0; l < d->L; ++l) {
      p.k4[l] = (d->sizes[l] + 3) / 4 * 4;
      p.ws_off[l] = off;
      off += (long long)d->sizes[l + 1] * p.k4[l];
    }
    const size_t sw = (size_t)(base + off) * sizeof(float);
    const char* e = std::getenv("SGB200_MLP_SMALL_WSTAGE");
    bool aligned = true;  // bulk copies: 16-byte aligned rows
    for (int l = 0; l < d->L; ++l) aligned = aligned && d->w_off[l] % 4 == 0 && d->ldw[l] % 4 == 0;
    if (aligned && sw <= 160 * 1024 && !(e && e[0] == '0')) {
      p.wstage = 1;
      p.ws_base = base;
      s1 = sw;
    }
  }
  size_t s2 = 0;
  for (int l = 0; l < d->L; ++l)
    s2 = std::max(s2, ((size_t)d->B * d->sizes[l + 1] + (size_t)d->B * ms::KW) * sizeof(float));
  smem = std::max(std::max(s1, s2), (size_t)ms::NT * sizeof(double));  // + the loss tree
  if (smem > 200 * 1024) return fail(SG_EINVAL, "mlp_small: working set exceeds shared memory");
  // phase 2 chunks: ceil((fan_in + 1) / KW) per layer (the +1 is the bias column)
  int n = 0;
  for (int l = 0; l < d->L; ++l) n += (d->sizes[l] + ms::KW) / ms::KW;
  p.chunks = n;
  // scratch: barrier (256 B) | loss_part [B] | h_1..h_{L-1} | dZ_0..dZ_{L-1}
  long long off = 0;
  for (int l = 1; l < d->L; ++l) {
    p.h_off[l] = off;
    off += (long long)d->B * d->sizes[l];
  }
  long long hf = off;
  off = 0;
  for (int l = 0; l < d->L; ++l) {
    p.dz_off[l] = off;
    off += (long long)d->B * d->sizes[l + 1];
  }
  scratch = 256 + (size_t)d->B * 8 + (size_t)hf * 4 + (size_t)off * 4;
  scratch = (scratch + 255) / 256 * 256;
  return SG_OK;
}

}  // namespace

extern "C" {

int sg_mlp_small_scratch_bytes(const sg_mlp_small_desc* d, int64_t* bytes) {
  ms::Params p;
  size_t smem = 0, scratch = 0;
  if (int rc = plan(d, p, smem, scratch)) return rc;
  if (bytes) *bytes = (int64_t)scratch;
  return SG_OK;
}

int sg_mlp_small_step(sg_ctx* ctx, const sg_mlp_small_desc* d, float* P, float* G, void* S_bf16, const float* X,
                      int64_t ldx, const float* Y, int64_t ldy, float* Z, int64_t ldz, double* loss, void* scratch,
                      int64_t scratch_bytes, void* stream) {
  SG_NVTX("sg_mlp_small_step");
  if (!ctx || !P || !G || !X || !Y || !loss || !scratch) return fail(SG_EINVAL, "null argument");
  ms::Params p;
  size_t smem = 0, need = 0;
  if (int rc = plan(d, p, smem, need)) return rc;
  if (scratch_bytes < (int64_t)need) return fail(SG_EINVAL, "mlp_small: scratch too small");
  if (ldx < d->sizes[0] || ldy < d->sizes[d->L] || (Z && ldz < d->sizes[d->L]))
    return fail(SG_EINVAL, "mlp_small: leading dimension smaller than the row");
  if (int rc = ctx_activate(ctx)) return rc;
  if (reinterpret_cast<uintptr_t>(P) % 16) p.wstage = 0;  // (shared memory stays sized for it)
  p.P = P;
  p.G = G;
  p.S = static_cast<__nv_bfloat16*>(S_bf16);
  p.X = X;
  p.ldx = ldx;
  p.Y = Y;
  p.ldy = ldy;
  p.Z = Z;
  p.ldz = ldz;
  p.loss_out = loss;
  p.dom = ctx_domain_word(ctx);
  char* s = static_cast<char*>(scratch);
  p.bar = reinterpret_cast<unsigned*>(s);
  p.loss_part = reinterpret_cast<double*>(s + 256);
  p.hg = reinterpret_cast<float*>(s + 256 + (size_t)d->B * 8);
  long long hf = 0;
  for (int l = 1; l < d->L; ++l) hf += (long long)d->B * d->sizes[l];
  p.dzg = p.hg + hf;
  const int ctas = (d->B + p.R - 1) / p.R;
  auto kern = p.R == 1 ? ms::k_mlp_small_step<1> : (p.R == 2 ? ms::k_mlp_small_step<2> : ms::k_mlp_small_step<4>);
  static std::atomic<uint64_t> attr{0};  // per device (all instantiations)
  if (first_on_device(attr))
    for (auto f : {ms::k_mlp_small_step<1>, ms::k_mlp_small_step<2>, ms::k_mlp_small_step<4>})
      SG_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  // occupancy query cached per (device, rows, shared-memory size): it costs host time every step
  thread_local int occ_dev = -1, occ_r = 0;
  thread_local size_t occ_smem = 0;
  thread_local int occ_per_sm = 0;
  int dev = 0;
  SG_CUDA_TRY(cudaGetDevice(&dev));
  if (occ_dev != dev || occ_smem != smem || occ_r != p.R) {
    SG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_per_sm, kern, ms::NT, smem));
    occ_dev = dev;
    occ_smem = smem;
    occ_r = p.R;
  }
  const int per_sm = occ_per_sm;
  if ((long long)per_sm * ctx_num_sms(ctx) < ctas) return fail(SG_EINVAL, "mlp_small: grid cannot be co-resident");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(ms::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs resident: the grid barrier is safe
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SG_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
  SG_CUDA_TRY(cudaGetLastError());
  return SG_OK;
}

}  // extern "C"
