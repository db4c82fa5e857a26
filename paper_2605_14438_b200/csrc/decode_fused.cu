// The whole BEAM layer forward for decode batches (T <= 64) in ONE persistent
// kernel: one CTA per SM, grid-wide barriers between the phases that need them.
//
// Reference (paths relative to /root/reference/pkg/src/beamoe/):
//   beam_block_forward  beam.py:127-165 (inference branch :159-165)
//   rms_norm            tensor.py:485-508
//   topk_route          moe.py:116-137      stable top-K, softmax over the K kept
//   mask_forward        beam.py:68-72       a = x_n W_m, keep iff a >= 0 (tau = 0.5)
//   mask_route          _kernels.pyx:17-34
//   group_by_expert     _kernels.pyx:37-66  ascending flat order inside an expert
//   grouped_execute     dispatch/__init__.py:129-157 -> expert_forward_np moe.py:96-100
//   combine             dispatch/__init__.py:145-156 (ascending expert id), shared
//                       experts beam.py:163-164, residual beam.py:165
//
// Why one kernel: at decode sizes the layer is a 20-1200 MB weight stream behind a
// 2 MB routing step; separate launches pay a drain/fill bubble at every boundary
// (four of them) and the stream cannot start before the previous kernel ends.
// Here every SM
//   P1  projection: a 16-column x 256-k slice of [W_router ; W_mask]^T (fp32) for
//       all T tokens -> split-K partials;                               [grid barrier]
//   P2  top-K + softmax + mask of token t on CTA t (one warp);          [grid barrier]
//   P3  builds the dispatch plan for all tokens in its own shared memory (a
//       stable counting sort of <= 1024 slots; every CTA gets the identical plan,
//       so no barrier and no global plan);
//   P4  gate/up: streams its contiguous share of (active expert, 4-feature)
//       items through a TMA bulk-copy ring (6 x 32 KB in flight), two groups of
//       8 consumer warps split K, act = silu(g) * u stored bf16;       [grid barrier,
//       consumer warps only: the producer warp already streams P5's weights]
//   P5  down + combine: the CTA owns 16 output rows; for every active expert in
//       ascending id it streams those rows (one bulk copy) and each consumer warp
//       adds ghat * (act . w_row) of the expert's tokens to its row of y in shared
//       memory — ascending expert order per (token, row) by construction, so the
//       combine is fused and deterministic (no per-pair rows, no atomics);
//       finally out = h + y.
// Masked slots never reach P4/P5: no bytes, no FLOPs.
#include "route_device.cuh"

namespace beam {
namespace dec {

constexpr int kCWarps = 16;                   // consumer warps (2 groups of 8 in P4)
constexpr int kThreads = 32 * kCWarps;       // no producer warp: refills are issued by the last reader of a slot
constexpr int kSlotBytes = 32 * 1024;
constexpr int kSlots = 6;
constexpr int kMaxT = 64;
constexpr int kMaxM = 512;                    // T * (K + S)
constexpr int kMaxE = 256;
constexpr int kKC = 256;                      // projection k-chunk (32 lanes x 8)
constexpr int kMaxKC = 16;                    // d_pad <= 4096
constexpr int kRowsDown = 16;                 // output rows per P5 block (one per consumer warp)

struct Args {
  const void* X;  // [T, d_pad] bf16 / f32
  int T;
  int d, d_pad, f_pad, N, E, Keff;
  int act_silu;
  const float* nw;       // RMS-norm weight or null
  const float* gate_wT;  // [2N, d_pad]
  const __nv_bfloat16* w_gu;    // [E, 2 f_pad, d_pad] packed gate/up rows
  const __nv_bfloat16* w_down;  // [E, d_pad, f_pad]
  float* P;              // [nkc][T][2N] projection partials
  __nv_bfloat16* act;    // [M, f_pad]
  unsigned* bar;         // [2] grid barrier: arrival count, generation
  void* out;             // [T, d] dtype of X
  int x_bf16;            // X / out dtype
  int rd;                // rows per P5 block (<= kRowsDown)
  long long prefetch_budget;  // bytes of P5 weights this CTA prefetches into L2 during P4
  int cost_alpha;        // P4 split: cost of an item's weights in token-pass units
  TopkArgs tk;
  unsigned long long* trace;  // diagnostics (beam_trace_decode) or null
};

constexpr int kRB = 4;  // P4 partial-sum buffers in flight

struct Smem {
  // plan
  int cnt[kMaxE];
  int off[kMaxE + 1];
  int act_list[kMaxE];
  int cost[kMaxE + 1];       // P4 cost prefix over the active list
  int tok[kMaxM];
  float w[kMaxM];
  int n_act;
  int i0, i1;                // this CTA's P4 item range
  int n4;                    // number of P4 items of this CTA
  union {
    struct {                 // P2 / P3 scratch
      float lv[2 * 256];     // router logits then mask pre-activations
      int rank[256];
      int sel[32];
      float gsel[32];
      float ssq[kCWarps];
      unsigned bits[kMaxE][2];  // token bitmask per expert (T <= 64)
      int ids[kMaxM];           // P2's masked ids / ghat, staged by the whole CTA
      float gw[kMaxM];
    };
    float red[kRB][kCWarps][64];  // P4 cross-warp partial sums: [buffer][warp][8 tokens x 8 rows]
  };
  // P5 y rows: [token][row]
  float y[kMaxT][kRowsDown];
  // P1 / P5 reduction scratch: [warp][32]
  float pr[kCWarps][32];
  int turn[kRowsDown / 8];      // P5 ordered-accumulation turn per 8-row n-tile
  int done[kSlots];             // readers finished with the slot's current stage
  int tag[kSlots];              // stage currently issued into the slot
  unsigned long long full[kSlots];
  unsigned long long red_full[kRB];   // 16 warps' partials of a P4 pass are in red[b]
  unsigned long long red_empty[kRB];  // the pass's epilogue has read red[b]
  long long clk[16];            // diagnostics: CTA 0 warp 0 accumulated clocks (trace slots 32..47)
};

__device__ __forceinline__ long long* clock_smem() {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  return reinterpret_cast<Smem*>(ring + kSlots * kSlotBytes)->clk;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(unsigned long long* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, unsigned long long* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Diagnostics (beam_trace_decode, Args::trace): %globaltimer of every CTA at the
// phase boundaries, slot 64 + m * grid + cta for mark m < 12; CTA 0 sub-step
// clocks in slots 24..63 (set: clock_mark, accumulated: clock_acc).
__device__ __forceinline__ void trace_mark(unsigned long long* tr, int m) {
  if (tr != nullptr) {  // per-CTA slot, no atomics (the trace must not perturb the phases)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[64 + m * gridDim.x + blockIdx.x] = t;
  }
}
__device__ __forceinline__ void clock_mark(unsigned long long* tr, int slot, long long& last) {
  if (tr != nullptr && blockIdx.x == 0) {
    const long long now = clock64();
    if ((threadIdx.x & 31) == 0) tr[slot] = (unsigned long long)(now - last);
    last = now;
  }
}
__device__ long long* clock_smem();  // Smem::clk (defined after Smem)
__device__ __forceinline__ void clock_acc(unsigned long long* tr, int slot, long long& last) {
  if (tr != nullptr && blockIdx.x == 0 && threadIdx.x < 32) {
    const long long now = clock64();
    if (threadIdx.x == 0) clock_smem()[slot - 32] += now - last;
    last = now;
  }
}

// named barrier over the 16 consumer warps (id 1) / one P4 group (ids 2, 3)
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kCWarps) : "memory"); }
__device__ __forceinline__ void group_sync(int g) { asm volatile("bar.sync %0, 256;" ::"r"(2 + g) : "memory"); }

// Grid-wide barriers (all CTAs co-resident: one per SM, cooperative launch).
// Barrier i has its own counter bar[i] in the zero-initialised workspace: arrive =
// one release-add, wait = acquire-poll until it reaches the grid size.  Counter
// i is reset by CTA 0 once everyone has passed barrier i + 1 (barrier 2's at the
// next launch's barrier 0), so there is no reset on the critical path.  The
// gpu-scope fences also invalidate L1, so plain loads after a barrier see the
// other CTAs' writes.
constexpr int kBarriers = 3;
__device__ __forceinline__ void grid_arrive_wait(unsigned* bar, int i, unsigned nblocks) {
  __threadfence();
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + i) : "memory");
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + i) : "memory");
  } while (v < nblocks);
  __threadfence();
  if (blockIdx.x == 0) bar[(i + kBarriers - 1) % kBarriers] = 0u;
}

__device__ __forceinline__ void grid_barrier_all(unsigned* bar, int i) {
  __syncthreads();
  if (threadIdx.x == 0) grid_arrive_wait(bar, i, gridDim.x);
  __syncthreads();
}

__device__ __forceinline__ void grid_barrier_consumers(unsigned* bar, int i) {
  consumer_sync();
  if (threadIdx.x == 0) grid_arrive_wait(bar, i, gridDim.x);
  consumer_sync();
}

// 8 consecutive activation elements (k % 8 == 0) as floats
template <typename TX>
__device__ __forceinline__ void ldx8(const TX* p, float* o) {
  if constexpr (sizeof(TX) == 2) {
    unpack<__nv_bfloat16>(ld_cached(p), o);
  } else {
    unpack<float>(ld_cached(p), o);
    unpack<float>(ld_cached(p + 4), o + 4);
  }
}

// ---------------------------------------------------------------------------
// P1: projection partials P[kc][t][c] = sum_{k in chunk kc} x[t,k] * w[k] * W[c,k]
// unit = (16-column block, 256-k chunk).  The whole CTA first stages the unit's
// x chunk [T][256] in shared memory (fp32; the ring is free before P4), then
// consumer warp w computes column 16 cb + w for all T tokens from shared memory.
// ---------------------------------------------------------------------------
template <typename TX>
__device__ __forceinline__ void phase_projection(const Args& a, Smem& s, float* xs, int warp, int lane) {
  const int cols = 2 * a.N;
  const int ncb = ceil_div(cols, kCWarps);
  const int nkc = ceil_div(a.d_pad, kKC);
  const TX* X = static_cast<const TX*>(a.X);
  const int T = a.T;
  long long clk = clock64();
  for (int u = blockIdx.x; u < ncb * nkc; u += gridDim.x) {
    const int cb = u / nkc, kc = u % nkc;
    const int k0 = kc * kKC, kn = min(kKC, a.d_pad - k0);  // kn % 8 == 0
    // stage x[:, k0:k0+kn] (8 elements per thread per step, loads of a step unconditional)
    const int n8 = T * (kKC / 8);
    constexpr int kU = 4;
    for (int i0 = threadIdx.x; i0 < n8; i0 += kThreads * kU) {
      constexpr int kL = sizeof(TX) == 2 ? 1 : 2;
      uint4 raw[kU][kL];
#pragma unroll
      for (int uu = 0; uu < kU; ++uu) {
        const int i = min(i0 + uu * kThreads, n8 - 1);
        const int t = i / (kKC / 8), c8 = i % (kKC / 8);
        const int kk = k0 + min(8 * c8, kn - 8);
        const TX* xp = X + (size_t)t * a.d_pad + kk;
#pragma unroll
        for (int l = 0; l < kL; ++l) raw[uu][l] = ld_cached(xp + l * 4);
      }
#pragma unroll
      for (int uu = 0; uu < kU; ++uu) {
        const int i = i0 + uu * kThreads;
        if (i < n8) {
          float xv[8];
          if constexpr (kL == 1) {
            unpack<__nv_bfloat16>(raw[uu][0], xv);
          } else {
            unpack<float>(raw[uu][0], xv);
            unpack<float>(raw[uu][kL - 1], xv + 4);
          }
          float* dst = xs + (size_t)i * 8;
          *reinterpret_cast<float4*>(dst) = make_float4(xv[0], xv[1], xv[2], xv[3]);
          *reinterpret_cast<float4*>(dst + 4) = make_float4(xv[4], xv[5], xv[6], xv[7]);
        }
      }
    }
    __syncthreads();
    if (warp == 0) clock_mark(a.trace, 38, clk);
    if (warp < kCWarps) {
      const int c = cb * kCWarps + warp;
      const int k = k0 + 8 * lane;
      const bool kv = 8 * lane < kn;
      float wv[8];
      if (c < cols && kv) {
        const float* wp = a.gate_wT + (size_t)c * a.d_pad + k;
        unpack<float>(ld_cached(wp), wv);
        unpack<float>(ld_cached(wp + 4), wv + 4);
        if (a.nw) {
          const float4 g0 = ld_norm4(a.nw, k, a.d), g1 = ld_norm4(a.nw, k + 4, a.d);
          wv[0] *= g0.x; wv[1] *= g0.y; wv[2] *= g0.z; wv[3] *= g0.w;
          wv[4] *= g1.x; wv[5] *= g1.y; wv[6] *= g1.z; wv[7] *= g1.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) wv[q] = 0.0f;
      }
      for (int t0 = 0; t0 < T; t0 += 16) {
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float* xp = xs + ((size_t)min(t0 + j, T - 1) * (kKC / 8) + lane) * 8;
          const float4 x0 = *reinterpret_cast<const float4*>(xp);
          const float4 x1 = *reinterpret_cast<const float4*>(xp + 4);
          float sacc = wv[0] * x0.x;
          sacc = fmaf(wv[1], x0.y, sacc);
          sacc = fmaf(wv[2], x0.z, sacc);
          sacc = fmaf(wv[3], x0.w, sacc);
          sacc = fmaf(wv[4], x1.x, sacc);
          sacc = fmaf(wv[5], x1.y, sacc);
          sacc = fmaf(wv[6], x1.z, sacc);
          sacc = fmaf(wv[7], x1.w, sacc);
          acc[j] = sacc;
        }
        warp_reduce_to_smem<16>(acc, s.pr[warp], lane);
        if (c < cols && lane < 16 && t0 + lane < T) a.P[((size_t)kc * T + t0 + lane) * cols + c] = s.pr[warp][lane];
        __syncwarp();
      }
    }
    __syncthreads();  // xs reuse by the next unit
    if (warp == 0) clock_mark(a.trace, 39, clk);
  }
}

// P4 work split by cost, not by item count: an item of expert e costs
// alpha (its 32 KB of weights) + cnt_e (one token's worth of FMAs per unit);
// CTA c takes the items whose cost prefix falls in [c, c + 1) * total / grid.
__device__ __forceinline__ int item_at_cost(const Smem& s, long long target, int groups_e, int alpha) {
  int lo = 0, hi = s.n_act;  // largest a with cost[a] <= target
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s.cost[mid] <= target) lo = mid;
    else hi = mid;
  }
  if (lo >= s.n_act) return s.n_act * groups_e;
  const int ci = alpha + s.cnt[s.act_list[lo]];
  const int k = (int)((target - s.cost[lo] + ci - 1) / ci);  // first item with prefix >= target
  return lo * groups_e + (k < groups_e ? k : groups_e);
}

// The plan, built by the whole CTA without a serial pass: every expert keeps a
// 64-bit mask of its tokens, so a slot's position inside its expert (ascending
// flat index == ascending token, _kernels.pyx:37-66) is a popcount.
__device__ __forceinline__ void build_plan(const Args& a, Smem& s, int warp, int lane, int groups_e, int alpha) {
  const int E = a.E, Keff = a.Keff, M = a.T * Keff;
  long long clk = clock64();
  for (int i = threadIdx.x; i < 2 * E; i += kThreads) (&s.bits[0][0])[i] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < M; i += kThreads) {
    const int e = __ldcg(a.tk.ids32 + i);
    s.ids[i] = e;
    s.gw[i] = __ldcg(a.tk.gw + i);
    if (e >= 0 && e < E) {
      const int t = i / Keff;
      atomicOr(&s.bits[e][t >> 5], 1u << (t & 31));
    }
  }
  __syncthreads();
  if (warp == 0) clock_mark(a.trace, 28, clk);
  if (warp == 0) {
    // counts, offsets, active list and P4 cost prefix: lane l owns experts [l*per, ...)
    const int per = ceil_div(E, 32);
    const int e0 = min(E, lane * per), e1 = min(E, e0 + per);
    int csum = 0, asum = 0, ksum = 0;
    for (int e = e0; e < e1; ++e) {
      const int c = __popc(s.bits[e][0]) + __popc(s.bits[e][1]);
      s.cnt[e] = c;
      csum += c;
      asum += c > 0;
      ksum += c > 0 ? groups_e * (alpha + c) : 0;
    }
    int cx = csum, ax = asum, kx = ksum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int yc = __shfl_up_sync(0xffffffffu, cx, o);
      const int ya = __shfl_up_sync(0xffffffffu, ax, o);
      const int yk = __shfl_up_sync(0xffffffffu, kx, o);
      if (lane >= o) {
        cx += yc;
        ax += ya;
        kx += yk;
      }
    }
    int run = cx - csum, arun = ax - asum, krun = kx - ksum;
    for (int e = e0; e < e1; ++e) {
      const int c = s.cnt[e];
      s.off[e] = run;
      run += c;
      if (c > 0) {
        s.cost[arun] = krun;
        krun += groups_e * (alpha + c);
        s.act_list[arun++] = e;
      }
    }
    if (lane == 31) {
      s.off[E] = cx;
      s.n_act = ax;
      s.cost[ax] = kx;
    }
    __syncwarp();
    if (lane == 0) {
      const long long total = s.cost[s.n_act];
      s.i0 = item_at_cost(s, total * blockIdx.x / gridDim.x, groups_e, alpha);
      s.i1 = item_at_cost(s, total * (blockIdx.x + 1) / gridDim.x, groups_e, alpha);
    }
    clock_mark(a.trace, 29, clk);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < M; i += kThreads) {
    const int e = s.ids[i];
    if (e >= 0 && e < E) {
      const int t = i / Keff;
      const unsigned b0 = s.bits[e][0], b1 = s.bits[e][1];
      const int below = t < 32 ? __popc(b0 & ((1u << t) - 1u)) : __popc(b0) + __popc(b1 & ((1u << (t - 32)) - 1u));
      const int pos = s.off[e] + below;
      s.tok[pos] = t;
      s.w[pos] = s.gw[i];
    }
  }
  __syncthreads();
  if (warp == 0) clock_mark(a.trace, 30, clk);
}

// ---------------------------------------------------------------------------
// P2: gating of token t by the 16 consumer warps of one CTA (reference:
// rms_norm tensor.py:485-487, topk_route moe.py:116-137, mask_forward
// beam.py:68-72, mask_route _kernels.pyx:17-34).  No serial selection loop:
// each expert's rank is the number of experts that beat it (value desc, ties ->
// lower id), counted by four threads over a quarter of the logits each.
// ---------------------------------------------------------------------------
template <typename TX>
__device__ __forceinline__ void topk_cta(const Args& a, Smem& s, int t, int warp, int lane) {
  const TopkArgs& k = a.tk;
  const int tid = threadIdx.x;  // < 512
  const int N = a.N, K = k.K, Keff = a.Keff, cols = 2 * N;
  const int nkc = ceil_div(a.d_pad, kKC);
  long long clk = clock64();
  // sum of squares (tensor.py:485-487) and the split-K partial sums, loads first
  float ss = 0.0f;
  if (k.has_norm) {
    const TX* row = static_cast<const TX*>(a.X) + (size_t)t * a.d_pad;
    float4 xq[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = 4 * tid + 2048 * h;
      xq[h] = kk < a.d_pad ? ld4<TX>(row + kk) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) ss += xq[h].x * xq[h].x + xq[h].y * xq[h].y + xq[h].z * xq[h].z + xq[h].w * xq[h].w;
  }
  float val = 0.0f;
  if (tid < cols) {
    float pv[kMaxKC];
#pragma unroll
    for (int q = 0; q < kMaxKC; ++q) pv[q] = __ldcg(a.P + ((size_t)min(q, nkc - 1) * a.T + t) * cols + tid);
#pragma unroll
    for (int q = 0; q < kMaxKC; ++q)
      if (q < nkc) val += pv[q];
  }
  ss = warp_sum(ss);
  if (lane == 0) s.ssq[warp] = ss;
  consumer_sync();
  float inv = 1.0f;
  if (k.has_norm) {
    float tot = 0.0f;
#pragma unroll
    for (int w = 0; w < kCWarps; ++w) tot += s.ssq[w];
    inv = 1.0f / sqrtf(tot / (float)a.d + 1e-6f);
  }
  if (tid < cols) {
    const float x = val * inv;
    // ranking treats NaN logits as -inf (numpy sorts them last)
    s.lv[tid] = (tid < N && x != x) ? -INFINITY : x;
  }
  if (tid == 0 && k.inv_out) k.inv_out[t] = inv;
  consumer_sync();
  if (warp == 0) clock_mark(a.trace, 24 + 0, clk);
  // rank_j = #{j' : v_j' > v_j or (v_j' == v_j and j' < j)}: 4 threads per expert
  for (int j0 = 0; j0 < N; j0 += kCWarps * 8) {
    const int j = j0 + (tid >> 2), q = tid & 3;
    int r = 0;
    if (j < N) {
      const float vj = s.lv[j];
      const int qa = q * ceil_div(N, 4), qb = min(N, qa + ceil_div(N, 4));
      for (int jj = qa; jj < qb; ++jj) {
        const float v2 = s.lv[jj];
        r += (v2 > vj) || (v2 == vj && jj < j);
      }
    }
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    if (j < N && q == 0) {
      s.rank[j] = r;
      if (r < K) s.sel[r] = j;
    }
  }
  consumer_sync();
  if (warp == 0) clock_mark(a.trace, 24 + 1, clk);
  // softmax over the K kept logits (tensor.py:440-451) and the routed ids
  if (warp == 0) {
    const int j = lane < K ? s.sel[lane] : 0;
    const float top = s.lv[s.sel[0]];
    const float e = lane < K ? expf(s.lv[j] - top) : 0.0f;
    const float g = e / warp_sum(e);
    if (lane < K) {
      const float av = s.lv[N + j];
      const bool keep = av >= k.thr;  // NaN -> masked
      const size_t o = (size_t)t * Keff + lane;
      k.ids32[o] = keep ? j : -1;
      k.gw[o] = keep ? g : 0.0f;
      s.gsel[lane] = g;
      if (k.topk_ids) k.topk_ids[(size_t)t * K + lane] = j;
      if (k.masked_ids) k.masked_ids[(size_t)t * K + lane] = keep ? j : -1;
    } else if (lane < Keff) {  // shared experts: always-on slots, weight 1.0 (beam.py:163-164)
      const size_t o = (size_t)t * Keff + lane;
      k.ids32[o] = N + (lane - K);
      k.gw[o] = 1.0f;
    }
  }
  consumer_sync();
  if (warp == 0) clock_mark(a.trace, 24 + 2, clk);
  // dense outputs (RouterDecision / MaskDecision fields)
  for (int j = tid; j < N; j += kCWarps * 32) {
    const size_t od = (size_t)t * N + j;
    const float x = s.lv[N + j];
    const int r = s.rank[j];
    if (k.logits) k.logits[od] = val * inv;
    if (k.weights) k.weights[od] = r < K ? s.gsel[r] : 0.0f;
    if (k.pre_act) k.pre_act[od] = x;
    if (k.raw_mask) k.raw_mask[od] = sigmoid_ref(x);
    if (k.mask) k.mask[od] = x >= k.thr ? 1.0f : 0.0f;
  }
  if (warp == 0) clock_mark(a.trace, 24 + 3, clk);
}

// ---------------------------------------------------------------------------
// Tensor-core helpers (mma.sync m16n8k16 bf16 -> fp32; operands from the
// swizzled TMA stages through ldmatrix).  The decode stream is HBM-bound; the
// MMA is here to take the multiply-adds off the issue slots (one instruction
// per 2048 MACs instead of 2048 / 32 FFMAs + bf16 unpacking).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0, int c1,
                                            int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

// two consecutive k elements of an activation row, as a bf16 pair (x * nw when normed)
template <typename TX>
__device__ __forceinline__ uint32_t x_pair(const TX* row, const float* nw, int k) {
  if constexpr (sizeof(TX) == 2) {
    const uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(row + k));
    if (nw == nullptr) return v;
    const float2 g = __ldg(reinterpret_cast<const float2*>(nw + k));
    return pack_bf16(__uint_as_float(v << 16) * g.x, __uint_as_float(v & 0xffff0000u) * g.y);
  } else {
    const float2 v = __ldg(reinterpret_cast<const float2*>(row + k));
    if (nw == nullptr) return pack_bf16(v.x, v.y);
    const float2 g = __ldg(reinterpret_cast<const float2*>(nw + k));
    return pack_bf16(v.x * g.x, v.y * g.y);
  }
}

// ---------------------------------------------------------------------------
// The stage stream of one CTA: sequence number n < n4 = its P4 items (4 gate +
// 4 up rows, two TMA boxes), then its P5 stages (row block b, active expert q),
// all through one ring of kSlots slots.  Stage n + kSlots is issued into slot
// n % kSlots by the last reader of stage n (smem counter), so the weight stream
// runs ahead of the consumers, across the P4 -> P5 barrier, without a producer
// warp (which would cap the registers of all 17 warps at 96).
// ---------------------------------------------------------------------------
struct Stream {
  const CUtensorMap* gu;
  const CUtensorMap* dn;
  uint8_t* ring;
  int groups_e, nblk;
};

__device__ __forceinline__ void issue_stage(const Args& a, Smem& s, const Stream& st, int n) {
  const int slot = n % kSlots;
  *reinterpret_cast<volatile int*>(&s.tag[slot]) = n;
  uint8_t* dst = st.ring + slot * kSlotBytes;
  const uint64_t pol_stream = policy_evict_first();
  if (n < s.n4) {
    const int i = s.i0 + n;
    const int e = s.act_list[i / st.groups_e], feat0 = (i % st.groups_e) * 4;
    const int row_g = e * 2 * a.f_pad + (feat0 >> 4) * 32 + (feat0 & 15);
    mbar_expect_tx(&s.full[slot], 2u * 4u * a.d_pad * 2u);
    tma_load_3d(dst, st.gu, &s.full[slot], 0, row_g, 0, pol_stream);
    tma_load_3d(dst + 16384, st.gu, &s.full[slot], 0, row_g + 16, 0, pol_stream);
  } else {
    const int m = n - s.n4;
    if (s.n_act == 0) return;
    const int b = blockIdx.x + (m / s.n_act) * gridDim.x;
    if (b >= st.nblk) return;
    const int q = m % s.n_act;
    mbar_expect_tx(&s.full[slot], (uint32_t)kRowsDown * a.f_pad * 2u);
    tma_load_3d(dst, st.dn, &s.full[slot], 0, s.act_list[q] * a.d_pad + b * a.rd, 0, policy_evict_last());
  }
}

// Wait until stage n has landed in its slot.  A reader may reach stage n before
// stage n - kSlots (same slot) has even been consumed by another warp group, and
// the mbarrier parity alone cannot tell phase p from phase p - 2: wait for the
// slot's tag first (written when the refill is issued), then for the data.
__device__ __forceinline__ void wait_stage(Smem& s, int n, int lane) {
  const int slot = n % kSlots;
  if (lane == 0)
    while (*reinterpret_cast<volatile int*>(&s.tag[slot]) != n) {
    }
  __syncwarp();
  mbar_wait(&s.full[slot], (n / kSlots) & 1);
}

// Called by each of the `readers` warps of stage n once its shared-memory reads
// are done; the last one refills the slot with stage n + kSlots.
__device__ __forceinline__ void release_stage(const Args& a, Smem& s, const Stream& st, int n, int readers, int lane) {
  // The warp's reads of the slot have returned (their registers fed the MMAs),
  // so no memory fence is needed before counting it done; only the refilling
  // thread orders the generic proxy before the async-proxy (TMA) writes.
  __syncwarp();
  if (lane == 0) {
    const int slot = n % kSlots;
    if (atomicAdd(&s.done[slot], 1) == readers - 1) {
      s.done[slot] = 0;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_stage(a, s, st, n + kSlots);
    }
  }
}

// ---------------------------------------------------------------------------
// P4 consumer.  Item = 4 gate rows + the 4 matching up rows of one expert over
// all d_pad columns (two TMA boxes, 16 KB each, [kb][4 rows][64] swizzled).
// A group of 8 warps splits K (warp wi: k-blocks [wi*kbpw, (wi+1)*kbpw)); each
// warp runs m16n8k16 MMAs with M = up to 8 tokens (A = x_n rows from global,
// cached in registers across the items of one expert and token pass), N = the
// 8 weight rows, then the group sums the 8 partial tiles in shared memory and
// one warp applies act = silu(g) * u and stores bf16 act rows.
// ---------------------------------------------------------------------------
constexpr int kKStepsMax = 8;  // k-steps per warp (16 warps split K; d_pad <= 2048)

struct AFrag {
  uint32_t a[kKStepsMax][2];
  int e = -1, t0 = -1;
};

template <typename TX>
__device__ __forceinline__ void load_afrag(const Args& a, const Smem& s, AFrag& f, int e, int t0, int nt, int kb0,
                                           int kbpw, int lane) {
  const TX* X = static_cast<const TX*>(a.X);
  const int j = lane >> 2;
  const int tok = s.tok[s.off[e] + t0 + min(j, nt - 1)];
  const TX* row = X + (size_t)tok * a.d_pad;
  const bool live = j < nt;
  const int nkb = a.d_pad / 64;
#pragma unroll
  for (int ks = 0; ks < kKStepsMax; ++ks) {
    const int kb = kb0 + (ks >> 2);
    const int k = min(kb, nkb - 1) * 64 + (ks & 3) * 16 + (lane & 3) * 2;
    uint32_t lo = x_pair<TX>(row, a.nw, k), hi = x_pair<TX>(row, a.nw, k + 8);
    const bool ok = live && (ks >> 2) < kbpw && kb < nkb;
    f.a[ks][0] = ok ? lo : 0u;
    f.a[ks][1] = ok ? hi : 0u;
  }
  f.e = e;
  f.t0 = t0;
}

__device__ __forceinline__ void mbar_arrive1(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <typename TX>
__device__ __forceinline__ void gateup_item(const Args& a, Smem& s, const uint8_t* stage, int e, int feat0, int warp,
                                            int lane, int& tau, AFrag& f, const Stream& st, int n) {
  const int cnt = s.cnt[e], off = s.off[e];
  const int nkb = a.d_pad / 64;
  const int kbpw = ceil_div(nkb, kCWarps);
  const int kb0 = warp * kbpw;
  // ldmatrix row addresses: lane -> matrix mi = lane / 8 (k-chunk 2 ks + mi of the
  // pair (ks, ks + 1)), weight row r = lane % 8 (gate rows 0-3, up rows 4-7)
  const int mi = lane >> 3, r = lane & 7, gu = r >> 2, r4 = r & 3;
  const uint32_t sbase = smem_u32(stage) + gu * 16384;
  for (int t0 = 0; t0 < cnt; t0 += 8, ++tau) {
    const int nt = min(8, cnt - t0);
    long long clk = clock64();
    if (f.e != e || f.t0 != t0) load_afrag<TX>(a, s, f, e, t0, nt, kb0, kbpw, lane);
    clock_acc(a.trace, 44, clk);
    float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < kKStepsMax; ks += 2) {
      if ((ks >> 2) < kbpw) {
        const int g = 2 * ks + mi;  // 16-byte chunk index within the warp's k range
        const int kb = min(kb0 + (g >> 3), nkb - 1), c = g & 7;
        const int rr = kb * 4 + r4;
        uint32_t b[4];
        ldsm_x4(sbase + rr * 128 + ((c ^ (rr & 7)) << 4), b);
        mma16816(c0, f.a[ks][0], 0u, f.a[ks][1], 0u, b[0], b[1]);
        mma16816(c1, f.a[ks + 1][0], 0u, f.a[ks + 1][1], 0u, b[2], b[3]);
      }
    }
    clock_acc(a.trace, 40, clk);
    if (t0 + 8 >= cnt) release_stage(a, s, st, n, kCWarps, lane);  // last pass: this warp's smem reads are done
    clock_acc(a.trace, 41, clk);
    // partial tile [8 tokens][8 rows] -> red[rb]; no CTA-wide barrier: the pass's
    // epilogue warp (tau mod 16) waits for the 16 arrivals, the others move on
    const int rb = tau % kRB;
    const uint32_t u = (uint32_t)(tau / kRB);
    if (lane == 0) mbar_wait(&s.red_empty[rb], (u & 1) ^ 1);
    __syncwarp();
    float* red = &s.red[rb][0][0];
    *reinterpret_cast<float2*>(red + warp * 64 + (lane >> 2) * 8 + (lane & 3) * 2) = make_float2(c0[0] + c1[0], c0[1] + c1[1]);
    __syncwarp();
    if (lane == 0) mbar_arrive1(&s.red_full[rb]);
    clock_acc(a.trace, 42, clk);
    if (warp == tau % kCWarps) {
      mbar_wait(&s.red_full[rb], u & 1);
      const int j = lane >> 2, q = lane & 3;
      if (j < nt) {
        float gs = 0.0f, us = 0.0f;
#pragma unroll
        for (int w = 0; w < kCWarps; ++w) {
          gs += red[w * 64 + j * 8 + q];
          us += red[w * 64 + j * 8 + q + 4];
        }
        const int tok = s.tok[off + t0 + j];
        const float sc = a.tk.has_norm ? __ldcg(a.tk.inv_out + tok) : 1.0f;  // x_n = x * inv_rms * w
        const float gg = gs * sc, uu = us * sc;
        const float v = a.act_silu ? activation<BEAM_ACT_SILU>(gg) * uu : gg * uu;
        a.act[(size_t)(off + t0 + j) * a.f_pad + feat0 + q] = __float2bfloat16_rn(v);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&s.red_empty[rb]);
    }
    clock_acc(a.trace, 43, clk);
  }
}

// ---------------------------------------------------------------------------
// P5 consumer.  Stage = a 16-row box of expert e's W_down^T (rows of this CTA's
// output block, [kb][16][64] swizzled).  Warp (sg, h) owns n-tile h (rows
// 8h..8h+7) of the stages s = sg mod kStageGroups; per pass of up to 16 tokens
// it runs all f_pad/16 k-steps (A = act rows of the expert, bf16 from global /
// L2), then adds ghat * tile to y[tok][row] once every earlier stage has added
// its own (turn[h]): per (token, row) the experts arrive in ascending id, the
// reference's combine order, without a per-pair buffer.
// ---------------------------------------------------------------------------
constexpr int kNTiles = kRowsDown / 8;
constexpr int kAB = 6;  // P5 k-steps whose A fragments are loaded together
constexpr int kStageGroups = kCWarps / kNTiles;

// The k loop of one P5 pass: A fragments (act rows, global / L2) are loaded in
// batches of 16 k-steps (<= 8 tokens: rows 8-15 of the MMA are zero) or 8
// (9-16 tokens), all loads of a batch in flight together.
template <bool kBig>
__device__ __forceinline__ void down_mma(const Args& a, const __nv_bfloat16* r0, const __nv_bfloat16* r1, bool l0,
                                         bool l1, int nks, uint32_t sbase, int rr, int mi, float (&acc)[2][4]) {
  constexpr int kB = kBig ? 8 : 16;
  constexpr int kR = kBig ? 4 : 2;
  for (int ks0 = 0; ks0 < nks; ks0 += kB) {
    uint32_t af[kB][kR];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const int k = min(ks0 + q, nks - 1) * 16;
      // act was written by other CTAs in this launch: plain (coherent) loads
      af[q][0] = l0 ? *reinterpret_cast<const uint32_t*>(r0 + k) : 0u;
      af[q][1] = l0 ? *reinterpret_cast<const uint32_t*>(r0 + k + 8) : 0u;
      if constexpr (kBig) {
        af[q][2] = l1 ? *reinterpret_cast<const uint32_t*>(r1 + k) : 0u;
        af[q][3] = l1 ? *reinterpret_cast<const uint32_t*>(r1 + k + 8) : 0u;
      }
    }
#pragma unroll
    for (int q = 0; q < kB; q += 2) {
      if (ks0 + q < nks) {
        const int gch = 2 * (ks0 + q) + mi;
        const int kb = gch >> 3, c = gch & 7;
        uint32_t bf[4];
        ldsm_x4(sbase + kb * (kRowsDown * 128) + ((c ^ (rr & 7)) << 4), bf);
        if constexpr (kBig) {
          mma16816(acc[0], af[q][0], af[q][2], af[q][1], af[q][3], bf[0], bf[1]);
          if (ks0 + q + 1 < nks) mma16816(acc[1], af[q + 1][0], af[q + 1][2], af[q + 1][1], af[q + 1][3], bf[2], bf[3]);
        } else {
          mma16816(acc[0], af[q][0], 0u, af[q][1], 0u, bf[0], bf[1]);
          if (ks0 + q + 1 < nks) mma16816(acc[1], af[q + 1][0], 0u, af[q + 1][1], 0u, bf[2], bf[3]);
        }
      }
    }
  }
}

__device__ __forceinline__ void down_stage(const Args& a, Smem& s, const uint8_t* stage, int e, int sidx, int b,
                                           int nrows, bool last_in_block, int h, int lane, const Stream& st,
                                           int n) {
  const int cnt = s.cnt[e], off = s.off[e];
  const int nks = a.f_pad / 16;
  const int mi = lane >> 3, r = lane & 7;
  const int rr = h * 8 + r;
  const uint32_t sbase = smem_u32(stage) + rr * 128;
  const int g = lane >> 2, t4 = lane & 3;
  for (int t0 = 0; t0 < cnt; t0 += 16) {
    const int nt = min(16, cnt - t0);
    const int p0 = off + t0 + min(g, nt - 1), p1 = off + t0 + min(g + 8, nt - 1);
    const bool l0 = g < nt, l1 = g + 8 < nt;
    const __nv_bfloat16* r0 = a.act + (size_t)p0 * a.f_pad + t4 * 2;
    const __nv_bfloat16* r1 = a.act + (size_t)p1 * a.f_pad + t4 * 2;
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    if (nt <= 8) down_mma<false>(a, r0, r1, l0, l1, nks, sbase, rr, mi, acc);
    else down_mma<true>(a, r0, r1, l0, l1, nks, sbase, rr, mi, acc);
    if (t0 + 16 >= cnt) release_stage(a, s, st, n, kNTiles, lane);
    // ordered accumulation into y (turn[h] == sidx)
    if (lane == 0)
      while (*reinterpret_cast<volatile int*>(&s.turn[h]) != sidx) {
      }
    __syncwarp();
    const int row0 = h * 8 + t4 * 2;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int j = g + 8 * half;
      if (j < nt) {
        const int p = off + t0 + j;
        const float wgt = s.w[p];
        float* yr = &s.y[s.tok[p]][0];
        if (row0 < nrows) yr[row0] += (acc[0][2 * half] + acc[1][2 * half]) * wgt;
        if (row0 + 1 < nrows) yr[row0 + 1] += (acc[0][2 * half + 1] + acc[1][2 * half + 1]) * wgt;
      }
    }
    if (t0 + 16 < cnt) {  // more passes of the same stage: keep the turn
      __syncwarp();
      continue;
    }
  }
  __syncwarp();
  if (last_in_block) {  // every expert of the block has been added: out = h + y (beam.py:165)
    const int rb = b * a.rd;
    for (int i = lane; i < a.T * 8; i += 32) {
      const int t = i >> 3, rl = h * 8 + (i & 7), row = rb + rl;
      if (rl < nrows && row < a.d) {
        float* yp = &s.y[t][rl];
        if (sizeof(__nv_bfloat16) == 2 && a.x_bf16) {
          const __nv_bfloat16* X = static_cast<const __nv_bfloat16*>(a.X);
          static_cast<__nv_bfloat16*>(a.out)[(size_t)t * a.d + row] =
              __float2bfloat16_rn(__bfloat162float(X[(size_t)t * a.d_pad + row]) + *yp);
        } else {
          const float* X = static_cast<const float*>(a.X);
          static_cast<float*>(a.out)[(size_t)t * a.d + row] = X[(size_t)t * a.d_pad + row] + *yp;
        }
        *yp = 0.0f;
      }
    }
  }
  __syncwarp();
  __threadfence_block();
  if (lane == 0) *reinterpret_cast<volatile int*>(&s.turn[h]) = sidx + 1;
}

template <typename TX>
__global__ void __launch_bounds__(kThreads, 1)
    decode_layer_kernel(const __grid_constant__ CUtensorMap tm_gu, const __grid_constant__ CUtensorMap tm_dn, Args a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Smem& s = *reinterpret_cast<Smem*>(ring + kSlots * kSlotBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) mbar_init(&s.full[i], 1);
    for (int i = 0; i < kRB; ++i) {
      mbar_init(&s.red_full[i], kCWarps);
      mbar_init(&s.red_empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_gu)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dn)) : "memory");
  }
  if (threadIdx.x < kNTiles) s.turn[threadIdx.x] = 0;
  if (threadIdx.x < 16) s.clk[threadIdx.x] = 0;
  if (threadIdx.x < kSlots) {
    s.done[threadIdx.x] = 0;
    s.tag[threadIdx.x] = -1;
  }
  for (int i = threadIdx.x; i < kMaxT * kRowsDown; i += kThreads) (&s.y[0][0])[i] = 0.0f;

  if (threadIdx.x == 0) trace_mark(a.trace, 0);
  // ---- P1 projection ----
  phase_projection<TX>(a, s, reinterpret_cast<float*>(ring), warp, lane);
  if (threadIdx.x == 0) trace_mark(a.trace, 1);
  grid_barrier_all(a.bar, 0);
  if (threadIdx.x == 0) trace_mark(a.trace, 2);

  // ---- P2 top-K / softmax / mask: token blockIdx.x ----
  if ((int)blockIdx.x < a.T) topk_cta<TX>(a, s, blockIdx.x, warp, lane);
  if (threadIdx.x == 0) trace_mark(a.trace, 3);
  grid_barrier_all(a.bar, 1);
  if (threadIdx.x == 0) trace_mark(a.trace, 4);

  // ---- P3 plan (every CTA, redundantly) ----
  constexpr int FP = 4;  // features per P4 item
  const int groups_e = a.f_pad / FP;
  build_plan(a, s, warp, lane, groups_e, a.cost_alpha);
  const Stream st{&tm_gu, &tm_dn, ring, groups_e, ceil_div(a.d_pad, a.rd)};
  if (threadIdx.x == 0) {
    s.n4 = s.i1 - s.i0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P1 staged x through the ring
    for (int n = 0; n < kSlots; ++n) issue_stage(a, s, st, n);
    // P5's weights for this CTA's first experts go to L2 now (HBM serves them
    // alongside P4's stream; P4's own lines are evict-first)
    long long budget = a.prefetch_budget;
    for (int b = blockIdx.x; b < st.nblk && budget > 0; b += gridDim.x) {
      const int nrows = min(a.rd, a.d_pad - b * a.rd);
      const uint32_t bytes = (uint32_t)nrows * a.f_pad * 2;
      for (int q = 0; q < s.n_act && budget > 0; ++q, budget -= bytes)
        bulk_prefetch_l2(a.w_down + ((size_t)s.act_list[q] * a.d_pad + (size_t)b * a.rd) * a.f_pad, bytes);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) trace_mark(a.trace, 5);

  // ---- P4 gate/up: every item by all 16 warps (K split 16 ways) ----
  const int n4 = s.n4;
  int tau = 0;
  AFrag f;
  for (int n = 0; n < n4; ++n) {
    const int slot = n % kSlots;
    long long clk = clock64();
    wait_stage(s, n, lane);
    clock_acc(a.trace, 32, clk);
    const int i = s.i0 + n;
    const int e = s.act_list[i / groups_e], feat0 = (i % groups_e) * FP;
    gateup_item<TX>(a, s, ring + slot * kSlotBytes, e, feat0, warp, lane, tau, f, st, n);
    clock_acc(a.trace, 33, clk);
  }
  if (threadIdx.x == 0) trace_mark(a.trace, 6);
  grid_barrier_all(a.bar, 2);
  if (threadIdx.x == 0) trace_mark(a.trace, 7);

  // ---- P5 down + combine: stage m of this CTA -> the warps of stage group m mod kStageGroups ----
  const int sg = warp / kNTiles, h = warp % kNTiles;
  const int nact = s.n_act;
  int m = 0;
  for (int b = blockIdx.x; b < st.nblk; b += gridDim.x) {
    const int nrows = min(a.rd, a.d_pad - b * a.rd);
    for (int q = 0; q < nact; ++q, ++m) {
      if (m % kStageGroups != sg) continue;
      const int n = n4 + m;
      const int slot = n % kSlots;
      long long clk = clock64();
      wait_stage(s, n, lane);
      clock_acc(a.trace, 36, clk);
      down_stage(a, s, ring + slot * kSlotBytes, s.act_list[q], m, b, nrows, q == nact - 1, h, lane, st, n);
      clock_acc(a.trace, 37, clk);
    }
  }
  if (threadIdx.x == 0) trace_mark(a.trace, 8);
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x < 16) a.trace[32 + threadIdx.x] = (unsigned long long)s.clk[threadIdx.x];
}

constexpr size_t kSmemBytes = 1024 + (size_t)kSlots * kSlotBytes + sizeof(Smem);
static_assert(kSmemBytes <= 227 * 1024, "decode kernel shared memory exceeds the sm_100 per-CTA limit");

}  // namespace dec

static unsigned long long* g_decode_trace = nullptr;
cudaError_t set_decode_trace(unsigned long long* buf) {
  g_decode_trace = buf;
  return cudaSuccess;
}

bool decode_fused_supported(const beam_layer_t& L, const Dims& g, int T) {
  using namespace dec;
  static const bool on = [] {  // experimental until it beats the kernel chain
    const char* v = getenv("BEAM_FUSED_DECODE");
    return v && v[0] == '1';
  }();
  if (!on) return false;
  // P4 items: 4 gate + 4 up rows over d_pad (two 16 KB boxes, <= 16 k-steps per
  // warp); P5 stages: 16 rows x f_pad in one 32 KB slot
  return L.wdtype == BEAM_BF16 && T >= 1 && T <= kMaxT && T <= num_sms() && g.E <= kMaxE && g.N <= 256 &&
         g.K <= 32 && (long long)T * g.Keff <= kMaxM && g.d_pad % 64 == 0 && g.d_pad <= 2048 &&
         g.f_pad % 64 == 0 && kRowsDown * g.f_pad * 2 <= kSlotBytes;
}

template <typename TX>
static cudaError_t decode_launch(const CUtensorMap& mg, const CUtensorMap& md, const dec::Args& a, cudaStream_t s) {
  using namespace dec;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_layer_kernel<TX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_layer_kernel<TX>, mg, md, a);
}

// Tensor maps are cached per weight buffer (encoding costs host time every call).
struct MapCache {
  const void* base = nullptr;
  uint64_t rows = 0, cols = 0;
  uint32_t box = 0;
  CUtensorMap map;
};

static bool cached_map(MapCache& c, const void* base, uint64_t rows, uint64_t cols, uint32_t box) {
  if (c.base == base && c.rows == rows && c.cols == cols && c.box == box) return true;
  if (!make_tmap_rows_sw128(&c.map, base, rows, cols, box)) return false;
  c.base = base;
  c.rows = rows;
  c.cols = cols;
  c.box = box;
  return true;
}

cudaError_t launch_decode_fused(const beam_layer_t& L, const Dims& g, const void* X, int x_dtype, int T,
                                const TopkArgs& tk, float* P, void* act, unsigned* bar, void* out,
                                cudaStream_t s) {
  using namespace dec;
  static thread_local MapCache cg, cd;
  if (!cached_map(cg, L.w_gu, (uint64_t)g.E * 2 * g.f_pad, g.d_pad, 4) ||
      !cached_map(cd, L.w_down, (uint64_t)g.E * g.d_pad, g.f_pad, kRowsDown))
    return cudaErrorInvalidValue;
  Args a;
  a.X = X;
  a.T = T;
  a.d = g.d;
  a.d_pad = g.d_pad;
  a.f_pad = g.f_pad;
  a.N = g.N;
  a.E = g.E;
  a.Keff = g.Keff;
  a.act_silu = L.activation == BEAM_ACT_SILU;
  a.nw = L.has_norm ? L.norm_w : nullptr;
  a.gate_wT = L.gate_wT;
  a.w_gu = static_cast<const __nv_bfloat16*>(L.w_gu);
  a.w_down = static_cast<const __nv_bfloat16*>(L.w_down);
  a.P = P;
  a.act = static_cast<__nv_bfloat16*>(act);
  a.bar = bar;
  a.out = out;
  a.x_bf16 = x_dtype == BEAM_BF16;
  // P5 row blocks: at most one 16-row box, and enough blocks to give every SM one
  a.rd = std::min(kRowsDown, ceil_div(g.d_pad, num_sms()));
  static const int alpha = [] {
    const char* v = getenv("BEAM_DECODE_COST_ALPHA");  // tuning knob
    return v ? atoi(v) : 4;
  }();
  a.cost_alpha = alpha;
  static const long long budget = [] {
    const char* v = getenv("BEAM_DECODE_PREFETCH_KB");  // tuning knob: per-CTA L2 prefetch of P5 weights
    return v ? atoll(v) * 1024 : 256LL * 1024;
  }();
  a.prefetch_budget = budget;
  a.tk = tk;
  a.trace = g_decode_trace;
  cudaError_t e = x_dtype == BEAM_BF16 ? decode_launch<__nv_bfloat16>(cg.map, cd.map, a, s)
                                       : decode_launch<float>(cg.map, cd.map, a, s);
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace beam
