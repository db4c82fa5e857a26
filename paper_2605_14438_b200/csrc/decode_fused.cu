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
constexpr int kThreads = 32 * (kCWarps + 1);  // + 1 producer warp
constexpr int kSlotBytes = 32 * 1024;
constexpr int kSlots = 6;                     // even: P4 slots alternate between the two groups
constexpr int kMaxT = 64;
constexpr int kMaxM = 1024;                   // T * (K + S)
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
  int rp;                // packed rows per P4 item (8: 4 features, 4: 2 features)
  int rd;                // rows per P5 block (<= kRowsDown)
  long long prefetch_budget;  // bytes of P5 weights this CTA prefetches into L2 during P4
  TopkArgs tk;
};

struct Smem {
  // plan
  int cnt[kMaxE];
  int off[kMaxE + 1];
  int cur[kMaxE];
  int act_list[kMaxE];
  int tok[kMaxM];
  float w[kMaxM];
  int n_act;
  int pad_[3];
  // P4 cross-warp partial sums: [group][buffer][warp][32]
  float red[2][2][8][32];
  // P5 y rows: [token][row]
  float y[kMaxT][kRowsDown];
  // P1 reduction scratch: [warp][32]
  float pr[kCWarps][32];
  unsigned long long full[kSlots];
  unsigned long long empty[kSlots];
};

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
// Diagnostics (beam_trace_decode): %globaltimer min / max over CTAs at the phase
// boundaries, slots [2m] (min) and [2m+1] (max) for mark m.
__device__ unsigned long long* g_dec_trace = nullptr;
__device__ __forceinline__ void trace_mark(int m) {
  unsigned long long* tr = g_dec_trace;
  if (tr != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(tr + 2 * m, t);
    atomicMax(tr + 2 * m + 1, t);
  }
}

// named barrier over the 16 consumer warps (id 1) / one P4 group (ids 2, 3)
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kCWarps) : "memory"); }
__device__ __forceinline__ void group_sync(int g) { asm volatile("bar.sync %0, 256;" ::"r"(2 + g) : "memory"); }

// Grid-wide barrier (all CTAs co-resident: one per SM, cooperative launch).
// count/gen live in the zero-initialised workspace; count returns to 0 at every
// barrier, so the state is valid for the next launch whatever the grid size.
// The gpu-scope fences also invalidate L1, so plain loads after the barrier see
// other CTAs' writes.
__device__ __forceinline__ void grid_barrier_leader(unsigned* bar, unsigned nblocks) {
  volatile unsigned* gen_p = bar + 1;
  const unsigned gen = *gen_p;
  __threadfence();
  const unsigned ticket = atomicAdd(bar, 1u);
  if (ticket == nblocks - 1) {
    atomicExch(bar, 0u);
    __threadfence();
    atomicAdd(bar + 1, 1u);
  } else {
    unsigned g;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    } while (g == gen);
  }
  __threadfence();
}

__device__ __forceinline__ void grid_barrier_all(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) grid_barrier_leader(bar, gridDim.x);
  __syncthreads();
}

__device__ __forceinline__ void grid_barrier_consumers(unsigned* bar) {
  consumer_sync();
  if (threadIdx.x == 0) grid_barrier_leader(bar, gridDim.x);
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
// unit = (16-column block, 256-k chunk); consumer warp w owns column 16 cb + w.
// ---------------------------------------------------------------------------
template <typename TX>
__device__ __forceinline__ void phase_projection(const Args& a, Smem& s, int warp, int lane) {
  const int cols = 2 * a.N;
  const int ncb = ceil_div(cols, kCWarps);
  const int nkc = ceil_div(a.d_pad, kKC);
  const TX* X = static_cast<const TX*>(a.X);
  for (int u = blockIdx.x; u < ncb * nkc; u += gridDim.x) {
    const int cb = u / nkc, kc = u % nkc;
    const int c = cb * kCWarps + warp;
    const int k = kc * kKC + 8 * lane;
    const bool kv = k < a.d_pad;
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
    for (int t0 = 0; t0 < a.T; t0 += 16) {
      float acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        acc[j] = 0.0f;
        if (t0 + j < a.T && kv) {
          float xv[8];
          ldx8<TX>(X + (size_t)(t0 + j) * a.d_pad + k, xv);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[j] = fmaf(wv[q], xv[q], acc[j]);
        }
      }
      warp_reduce_to_smem<16>(acc, s.pr[warp], lane);
      if (c < cols && lane < 16 && t0 + lane < a.T) a.P[((size_t)kc * a.T + t0 + lane) * cols + c] = s.pr[warp][lane];
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// P3: the dispatch plan in shared memory (one warp).  Stable counting sort of
// the surviving slots by expert: inside an expert, ascending flat index t*Keff+k
// (_kernels.pyx:37-66); experts ascending in act_list.  No block padding: the
// layer never reads padding.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void build_plan(const Args& a, Smem& s, int lane) {
  const int E = a.E, M = a.T * a.Keff;
  for (int e = lane; e < E; e += 32) {
    s.cnt[e] = 0;
    s.cur[e] = 0;
  }
  __syncwarp();
  for (int base = 0; base < M; base += 32) {
    const int i = base + lane;
    const int e = i < M ? __ldcg(a.tk.ids32 + i) : -1;
    if (e >= 0 && e < E) atomicAdd(&s.cnt[e], 1);
  }
  __syncwarp();
  // exclusive scans of counts and of the active flags, lane l owns a contiguous run
  const int per = ceil_div(E, 32);
  const int e0 = min(E, lane * per), e1 = min(E, e0 + per);
  int csum = 0, asum = 0;
  for (int e = e0; e < e1; ++e) {
    csum += s.cnt[e];
    asum += s.cnt[e] > 0;
  }
  int cx = csum, ax = asum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yc = __shfl_up_sync(0xffffffffu, cx, o);
    const int ya = __shfl_up_sync(0xffffffffu, ax, o);
    if (lane >= o) {
      cx += yc;
      ax += ya;
    }
  }
  int run = cx - csum, arun = ax - asum;
  for (int e = e0; e < e1; ++e) {
    s.off[e] = run;
    run += s.cnt[e];
    if (s.cnt[e] > 0) s.act_list[arun++] = e;
  }
  if (lane == 31) {
    s.off[E] = cx;
    s.n_act = ax;
  }
  __syncwarp();
  for (int base = 0; base < M; base += 32) {
    const int i = base + lane;
    const int e = i < M ? __ldcg(a.tk.ids32 + i) : -1;
    const bool valid = e >= 0 && e < E;
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? e : E + lane);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid) {
      const int pos = s.off[e] + s.cur[e] + rank;
      s.tok[pos] = i / a.Keff;
      s.w[pos] = __ldcg(a.tk.gw + i);
    }
    __syncwarp();
    if (valid && rank == 0) s.cur[e] += __popc(peers);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// P4 consumer: one item = RP packed rows (RP/2 gate rows, then the matching RP/2
// up rows) of one expert, d_pad columns each.  Warp wi of the group owns 16-byte
// column chunks wi*32 + lane + 256 j; partial sums for RP rows x 4 tokens reduce
// across the warp, then across the group's 8 warps through shared memory.
// ---------------------------------------------------------------------------
template <typename TX, int RP>
__device__ __forceinline__ void gateup_item(const Args& a, Smem& s, const uint8_t* stage, int e, int feat0, int grp,
                                            int wi, int lane, int& rbuf, unsigned long long* empty_bar) {
  constexpr int V = RP * 4;  // RP rows x 4 tokens
  constexpr int FP = RP / 2;
  const int cnt = s.cnt[e], off = s.off[e];
  const int nchunk = a.d_pad / 8;
  const TX* X = static_cast<const TX*>(a.X);
  const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(stage);
  for (int t0 = 0; t0 < cnt; t0 += 4) {
    const int nt = min(4, cnt - t0);
    int tk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) tk[j] = s.tok[off + t0 + (j < nt ? j : 0)];
    float acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0.0f;
    for (int c = wi * 32 + lane; c < nchunk; c += 256) {
      // the (normalised) activations of the pass's tokens first, then one packed
      // weight row at a time: 4 x 8 + 8 live values instead of RP x 8 + 4 x 8
      float xv[4][8];
      float g8[8];
      if (a.nw) {
        const float4 g0 = ld_norm4(a.nw, 8 * c, a.d), g1 = ld_norm4(a.nw, 8 * c + 4, a.d);
        g8[0] = g0.x; g8[1] = g0.y; g8[2] = g0.z; g8[3] = g0.w;
        g8[4] = g1.x; g8[5] = g1.y; g8[6] = g1.z; g8[7] = g1.w;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < nt) {
          ldx8<TX>(X + (size_t)tk[j] * a.d_pad + 8 * c, xv[j]);
          if (a.nw) {
#pragma unroll
            for (int z = 0; z < 8; ++z) xv[j][z] *= g8[z];
          }
        } else {
#pragma unroll
          for (int z = 0; z < 8; ++z) xv[j][z] = 0.0f;
        }
      }
#pragma unroll
      for (int q = 0; q < RP; ++q) {
        float wv[8];
        unpack<__nv_bfloat16>(*reinterpret_cast<const uint4*>(W + (size_t)q * a.d_pad + 8 * c), wv);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int z = 0; z < 8; ++z) acc[q * 4 + j] = fmaf(wv[z], xv[j][z], acc[q * 4 + j]);
      }
    }
    // the last pass over the stage has issued its shared-memory reads: release it
    if (t0 + 4 >= cnt) {
      __syncwarp();
      if (lane == 0) mbar_arrive_cnt(empty_bar, 2);  // 8 warps x 2 = the 16 expected arrivals
    }
    float* red = &s.red[grp][rbuf][0][0];
    warp_reduce_to_smem<V>(acc, red + wi * 32, lane);
    group_sync(grp);
    if (wi == 0) {
      float v = 0.0f;
      if (lane < V) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v += red[q * 32 + lane];
      }
      const float u = __shfl_sync(0xffffffffu, v, (lane + 4 * FP) & 31);
      const int q = lane >> 2, j = lane & 3;
      if (lane < 4 * FP && j < nt) {
        const float sc = a.tk.has_norm ? __ldcg(a.tk.inv_out + tk[j]) : 1.0f;  // x_n = x * inv_rms * w
        const float g = v * sc, uu = u * sc;
        const float r = a.act_silu ? activation<BEAM_ACT_SILU>(g) * uu : g * uu;
        a.act[(size_t)(off + t0 + j) * a.f_pad + feat0 + q] = __float2bfloat16_rn(r);
      }
    }
    rbuf ^= 1;
  }
}

// ---------------------------------------------------------------------------
// P5 consumer: stage = rows [r0, r0 + nrows) of expert e's W_down^T, f_pad
// columns each; warp w owns row w and adds ghat * (act[pos] . row) to y[tok][w]
// for every token of the expert.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void down_item(const Args& a, Smem& s, const uint8_t* stage, int e, int nrows, int warp,
                                          int lane) {
  const int cnt = s.cnt[e], off = s.off[e];
  const int nchunk = a.f_pad / 8;
  if (warp < nrows) {
    const __nv_bfloat16* wr = reinterpret_cast<const __nv_bfloat16*>(stage) + (size_t)warp * a.f_pad;
    for (int t0 = 0; t0 < cnt; t0 += 4) {
      const int nt = min(4, cnt - t0);
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int c = lane; c < nchunk; c += 32) {
        float wv[8];
        unpack<__nv_bfloat16>(*reinterpret_cast<const uint4*>(wr + 8 * c), wv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < nt) {
            float av[8];
            // act was written by other CTAs in this launch: plain (coherent) load
            unpack<__nv_bfloat16>(*reinterpret_cast<const uint4*>(a.act + (size_t)(off + t0 + j) * a.f_pad + 8 * c), av);
#pragma unroll
            for (int z = 0; z < 8; ++z) acc[j] = fmaf(wv[z], av[z], acc[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = warp_sum(acc[j]);
      if (lane < nt) {
        float v = acc[0];
#pragma unroll
        for (int j = 1; j < 4; ++j)
          if (lane == j) v = acc[j];
        const int pos = off + t0 + lane;
        s.y[s.tok[pos]][warp] += v * s.w[pos];  // ascending expert order per (token, row)
      }
    }
  }
}

template <typename TX, typename TO>
__device__ __forceinline__ void write_rows(const Args& a, Smem& s, int r0, int nrows, int warp, int lane) {
  const int row = r0 + warp;
  if (warp < nrows && row < a.d) {
    const TX* X = static_cast<const TX*>(a.X);
    TO* out = static_cast<TO*>(a.out);
    for (int t = lane; t < a.T; t += 32) {
      const float h = to_f32<TX>(X[(size_t)t * a.d_pad + row]);
      out[(size_t)t * a.d + row] = from_f32<TO>(h + s.y[t][warp]);  // beam.py:165
    }
  }
  if (warp < nrows)
    for (int t = lane; t < a.T; t += 32) s.y[t][warp] = 0.0f;
}

template <typename TX, int NPL, int RP>
__global__ void __launch_bounds__(kThreads, 1) decode_layer_kernel(Args a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = smem_raw;
  Smem& s = *reinterpret_cast<Smem*>(smem_raw + kSlots * kSlotBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == kCWarps;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], kCWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < kMaxT * kRowsDown; i += kThreads) (&s.y[0][0])[i] = 0.0f;

  if (threadIdx.x == 0) trace_mark(0);
  // ---- P1 projection ----
  if (!producer) phase_projection<TX>(a, s, warp, lane);
  if (threadIdx.x == 0) trace_mark(1);
  grid_barrier_all(a.bar);
  if (threadIdx.x == 0) trace_mark(2);

  // ---- P2 top-K / softmax / mask: token blockIdx.x ----
  if (warp == 0 && (int)blockIdx.x < a.T)
    topk_token<TX, NPL, kMaxKC, true>(a.P, ceil_div(a.d_pad, kKC), a.T, static_cast<const TX*>(a.X), blockIdx.x,
                                      lane, a.tk);
  if (threadIdx.x == 0) trace_mark(3);
  grid_barrier_all(a.bar);
  if (threadIdx.x == 0) trace_mark(4);

  // ---- P3 plan (every CTA, redundantly) ----
  if (warp == 0) build_plan(a, s, lane);
  __syncthreads();
  if (threadIdx.x == 0) trace_mark(5);

  constexpr int FP = RP / 2;
  const int groups_e = a.f_pad / FP;
  const int n_items = s.n_act * groups_e;
  const int i0 = (int)((long long)n_items * blockIdx.x / gridDim.x);
  const int i1 = (int)((long long)n_items * (blockIdx.x + 1) / gridDim.x);
  const int nblk = ceil_div(a.d_pad, a.rd);

  if (producer) {
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
      // P5's weights for this CTA's first experts go to L2 now (HBM serves them
      // alongside P4's stream; P4's own lines are evict-first)
      long long budget = a.prefetch_budget;
      for (int b = blockIdx.x; b < nblk && budget > 0; b += gridDim.x) {
        const int nrows = min(a.rd, a.d_pad - b * a.rd);
        const uint32_t bytes = (uint32_t)nrows * a.f_pad * 2;
        for (int q = 0; q < s.n_act && budget > 0; ++q, budget -= bytes)
          bulk_prefetch_l2(a.w_down + ((size_t)s.act_list[q] * a.d_pad + (size_t)b * a.rd) * a.f_pad, bytes);
      }
      int n = 0;
      const uint32_t ibytes = (uint32_t)FP * a.d_pad * 2;
      for (int i = i0; i < i1; ++i, ++n) {
        const int slot = n % kSlots;
        mbar_wait(&s.empty[slot], ((n / kSlots) & 1) ^ 1);
        if (i == i0 + kSlots) trace_mark(11);
        const int e = s.act_list[i / groups_e], feat0 = (i % groups_e) * FP;
        const int row_g = (feat0 >> 4) * 32 + (feat0 & 15);
        const __nv_bfloat16* src = a.w_gu + ((size_t)e * 2 * a.f_pad + row_g) * a.d_pad;
        mbar_expect_tx(&s.full[slot], 2 * ibytes);
        bulk_load(ring + slot * kSlotBytes, src, ibytes, &s.full[slot], pol_stream);
        bulk_load(ring + slot * kSlotBytes + ibytes, src + (size_t)16 * a.d_pad, ibytes, &s.full[slot], pol_stream);
      }
      for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        const int nrows = min(a.rd, a.d_pad - b * a.rd);
        const uint32_t bytes = (uint32_t)nrows * a.f_pad * 2;
        for (int q = 0; q < s.n_act; ++q, ++n) {
          const int slot = n % kSlots;
          mbar_wait(&s.empty[slot], ((n / kSlots) & 1) ^ 1);
          mbar_expect_tx(&s.full[slot], bytes);
          bulk_load(ring + slot * kSlotBytes, a.w_down + ((size_t)s.act_list[q] * a.d_pad + (size_t)b * a.rd) * a.f_pad,
                    bytes, &s.full[slot], pol_keep);
        }
      }
      trace_mark(10);
    }
    return;
  }

  // ---- P4 gate/up (consumers) ----
  const int grp = warp >> 3, wi = warp & 7;
  int n = 0, rbuf = 0;
  for (int i = i0; i < i1; ++i, ++n) {
    if ((n & 1) != grp) continue;  // slots alternate between the two groups (kSlots even)
    const int slot = n % kSlots;
    mbar_wait(&s.full[slot], (n / kSlots) & 1);
    const int e = s.act_list[i / groups_e], feat0 = (i % groups_e) * FP;
    gateup_item<TX, RP>(a, s, ring + slot * kSlotBytes, e, feat0, grp, wi, lane, rbuf, &s.empty[slot]);
  }
  if (threadIdx.x == 0) trace_mark(6);
  grid_barrier_consumers(a.bar);
  if (threadIdx.x == 0) trace_mark(7);

  // ---- P5 down + combine (consumers) ----
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int nrows = min(a.rd, a.d_pad - b * a.rd);
    for (int q = 0; q < s.n_act; ++q, ++n) {
      const int slot = n % kSlots;
      mbar_wait(&s.full[slot], (n / kSlots) & 1);
      down_item(a, s, ring + slot * kSlotBytes, s.act_list[q], nrows, warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive_cnt(&s.empty[slot], 1);
    }
    if (sizeof(TX) == 2) write_rows<TX, __nv_bfloat16>(a, s, b * a.rd, nrows, warp, lane);
    else write_rows<TX, float>(a, s, b * a.rd, nrows, warp, lane);
  }
  if (threadIdx.x == 0) trace_mark(8);
}

constexpr size_t kSmemBytes = (size_t)kSlots * kSlotBytes + sizeof(Smem);

}  // namespace dec

cudaError_t set_decode_trace(unsigned long long* buf) {
  return cudaMemcpyToSymbol(dec::g_dec_trace, &buf, sizeof(buf));
}

bool decode_fused_supported(const beam_layer_t& L, const Dims& g, int T) {
  using namespace dec;
  static const bool on = [] {  // experimental until it beats the kernel chain
    const char* v = getenv("BEAM_FUSED_DECODE");
    return v && v[0] == '1';
  }();
  if (!on) return false;
  return L.wdtype == BEAM_BF16 && T >= 1 && T <= kMaxT && T <= num_sms() && g.E <= kMaxE && g.N <= 256 &&
         (long long)T * g.Keff <= kMaxM && g.d_pad <= kMaxKC * kKC && 4 * g.d_pad * 2 <= kSlotBytes &&
         g.f_pad * 2 <= kSlotBytes;
}

template <typename TX, int NPL, int RP>
static cudaError_t decode_launch(const dec::Args& a, cudaStream_t s) {
  using namespace dec;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_layer_kernel<TX, NPL, RP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
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
  return cudaLaunchKernelEx(&cfg, decode_layer_kernel<TX, NPL, RP>, a);
}

cudaError_t launch_decode_fused(const beam_layer_t& L, const Dims& g, const void* X, int x_dtype, int T,
                                const TopkArgs& tk, float* P, void* act, unsigned* bar, void* out,
                                cudaStream_t s) {
  using namespace dec;
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
  a.rp = 8 * g.d_pad * 2 <= kSlotBytes ? 8 : 4;
  a.rd = std::min(kRowsDown, kSlotBytes / (g.f_pad * 2));
  static const long long budget = [] {
    const char* v = getenv("BEAM_DECODE_PREFETCH_KB");  // tuning knob: per-CTA L2 prefetch of P5 weights
    return v ? atoll(v) * 1024 : 256LL * 1024;
  }();
  a.prefetch_budget = budget;
  a.tk = tk;
  const int npl = ceil_div(g.N, 32);
  cudaError_t e;
#define BEAM_DEC(TX_, RP_)                                              \
  if (npl <= 1) e = decode_launch<TX_, 1, RP_>(a, s);                  \
  else if (npl <= 2) e = decode_launch<TX_, 2, RP_>(a, s);             \
  else if (npl <= 4) e = decode_launch<TX_, 4, RP_>(a, s);             \
  else e = decode_launch<TX_, 8, RP_>(a, s);
  if (x_dtype == BEAM_BF16) {
    if (a.rp == 8) { BEAM_DEC(__nv_bfloat16, 8) } else { BEAM_DEC(__nv_bfloat16, 4) }
  } else {
    if (a.rp == 8) { BEAM_DEC(float, 8) } else { BEAM_DEC(float, 4) }
  }
#undef BEAM_DEC
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace beam
