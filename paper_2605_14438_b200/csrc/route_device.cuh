// Device building blocks of the routing half: vector loads, the per-token top-K /
// softmax / mask step, and the block-level stable permute.  Shared by the
// stand-alone kernels (gate.cu, permute.cu) and the fused decode gate kernel.
//
// Reference semantics (/root/reference/pkg/src/beamoe/):
//   topk_select / topk_route   moe.py:116-137     desc value, ties -> lower id; softmax
//                                                 over exactly the K kept logits
//   mask_forward / mask_route  beam.py:68-72, _kernels.pyx:17-34   a >= thr keeps (NaN masked)
//   group_by_expert / align    _kernels.pyx:37-66, dispatch/__init__.py:89-126
#pragma once

#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

// 4 consecutive elements (k % 4 == 0) as float4
template <typename T> __device__ __forceinline__ float4 ld4(const T* p);
template <> __device__ __forceinline__ float4 ld4<float>(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
template <> __device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  return make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                     __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u));
}

// norm weights at k..k+3 (zero beyond d; NULL -> ones)
__device__ __forceinline__ float4 ld_norm4(const float* __restrict__ nw, int k, int d) {
  if (nw == nullptr) return make_float4(1.f, 1.f, 1.f, 1.f);
  if (k + 3 < d && (d & 3) == 0) return __ldg(reinterpret_cast<const float4*>(nw + k));
  return make_float4(k < d ? nw[k] : 0.f, k + 1 < d ? nw[k + 1] : 0.f, k + 2 < d ? nw[k + 2] : 0.f,
                     k + 3 < d ? nw[k + 3] : 0.f);
}

// Loads of data written earlier in the same kernel by other CTAs go through L2.
template <bool CG, typename T>
__device__ __forceinline__ T ld_maybe_cg(const T* p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}


__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The selection half of topk_token, on one token's router logits v / mask
// pre-activations av (lane's columns j = lane + 32 i, NOT yet scaled by the
// token's inv_rms): top-K, softmax over the K kept logits, the routing rule,
// and every output of the token.  Shared by the split-K top-K kernels and the
// cluster gate (which gathers v / av from distributed shared memory).
template <int NPL, int KIND = -1>
__device__ __forceinline__ void topk_finish(float (&v)[NPL], float (&av)[NPL], float inv, int t, int lane,
                                            const TopkArgs& a) {
  const int N = a.N, Nr = KIND == BEAM_ROUTE_BEAM ? a.N : a.Nr, K = a.K, Keff = a.K + a.S;
  const int kind = KIND >= 0 ? KIND : a.kind;
  const bool has_mask = KIND == BEAM_ROUTE_BEAM ? true : a.mask_off >= 0;
  int rank[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) rank[i] = -1;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    v[i] *= inv;
    av[i] *= inv;
  }
  const bool tr = a.trace != nullptr && t == 0 && lane == 0;
  if (tr) a.trace[8] = gtimer();

  // Selection on 64-bit keys (order-preserving float bits << 32 | ~column): one
  // max per butterfly level, and the key order is exactly the reference's
  // (value desc, ties -> lower index, moe.py:116-119); NaN logits rank last.
  unsigned long long key[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    const unsigned fb = __float_as_uint(v[i]);
    const unsigned ord = v[i] != v[i] ? 0u : ((fb & 0x80000000u) ? ~fb : (fb | 0x80000000u));
    key[i] = j < Nr ? (((unsigned long long)ord << 32) | (unsigned)(~j)) : 0ull;
  }
  int top_j = 0;
  for (int r = 0; r < K; ++r) {
    unsigned long long best = key[0];
#pragma unroll
    for (int i = 1; i < NPL; ++i) best = key[i] > best ? key[i] : best;
    // warp max of the 64-bit keys as two 32-bit redux.sync reductions (value
    // order first, then the lowest column among equal values): 2 instructions
    // instead of a 5-level butterfly of 64-bit shuffles
    const unsigned bhi = (unsigned)(best >> 32), blo = (unsigned)best;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, bhi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, bhi == mhi ? blo : 0u);
    best = ((unsigned long long)mhi << 32) | mlo;
    const int bj = (int)(~(unsigned)(best & 0xffffffffull));
    if (r == 0) top_j = bj;
#pragma unroll
    for (int i = 0; i < NPL; ++i)
      if (lane + 32 * i == bj) {
        rank[i] = r;
        key[i] = 0ull;
      }
  }
  if (tr) a.trace[9] = gtimer();
  // the top logit (softmax shift) from the lane that holds column top_j
  float mine = 0.0f;
#pragma unroll
  for (int i = 0; i < NPL; ++i)
    if (lane + 32 * i == top_j) mine = v[i];
  const float top_val = __shfl_sync(0xffffffffu, mine, top_j & 31);

  // softmax over the K kept logits (tensor.py:440-451): exp(l - max) / sum;
  // DYNAMIC: softmax over all N columns (baselines.py:191-192)
  const bool dyn = kind == BEAM_ROUTE_DYNAMIC;
  float part = 0.0f;
#pragma unroll
  for (int i = 0; i < NPL; ++i)
    if (dyn ? (lane + 32 * i < Nr) : (rank[i] >= 0)) part += expf(v[i] - top_val);
  const float denom = warp_sum(part);
  if (tr) a.trace[10] = gtimer();

  // DYNAMIC: the kept prefix — count = #(cumulative mass < phi) + 1 over the
  // descending order (dynamic_select); ranks < K suffice unless the K most
  // probable experts hold less than phi (the reference then plans more slots
  // than candidates and its grouped_execute raises ContractError)
  int count = K;
  float kept_mass = 1.0f;
  if (dyn) {
    // p of rank r -> lane r (the owner of rank r is found with a ballot)
    float p_rank = 0.0f;
    for (int r = 0; r < K; ++r) {
      float cand = 0.0f;
      bool mine_r = false;
#pragma unroll
      for (int i = 0; i < NPL; ++i)
        if (rank[i] == r) {
          cand = expf(v[i] - top_val) / denom;
          mine_r = true;
        }
      const unsigned owner = __ballot_sync(0xffffffffu, mine_r);
      const float pv = __shfl_sync(0xffffffffu, cand, __ffs(owner) - 1);
      if (lane == r) p_rank = pv;
    }
    // inclusive scan of p over ranks 0..K-1 (sequential order: csum is a running sum)
    float csum = p_rank;
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, csum, o);
      if (lane >= o) csum += y;
    }
    const unsigned below = __ballot_sync(0xffffffffu, lane < K && csum < a.phi);
    count = min(__popc(below) + 1, Nr);
    const float mass = __shfl_sync(0xffffffffu, csum, min(count, K) - 1);
    kept_mass = mass;
  }

#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j >= Nr) continue;
    const float x = av[i];
    const float e = expf(v[i] - top_val) / denom;  // softmax value of this column
    const float g = (dyn || rank[i] >= 0) ? e : 0.0f;
    bool keep;
    float w, mval = 1.0f, sval = 0.0f;
    switch (kind) {
      case BEAM_ROUTE_TOPK:
        keep = true;
        w = g;
        break;
      case BEAM_ROUTE_DYNAMIC:
        keep = rank[i] >= 0 && rank[i] < count;
        w = keep ? g / kept_mass : 0.0f;
        break;
      case BEAM_ROUTE_ADA:
        keep = j < N;
        w = keep ? g : 0.0f;
        break;
      case BEAM_ROUTE_SOFT:
        sval = sigmoid_ref(x * a.temp_inv);
        mval = sval >= a.tau ? 1.0f : 0.0f;  // NaN -> 0
        keep = a.binarize ? mval != 0.0f : true;
        w = a.binarize ? g * mval : g * sval;
        break;
      default:  // BEAM
        keep = x >= a.thr;  // NaN -> false
        mval = keep ? 1.0f : 0.0f;
        w = keep ? g : 0.0f;
        sval = sigmoid_ref(x);
        break;
    }
    if (rank[i] >= 0) {
      const int r = rank[i];
      const size_t o = (size_t)t * Keff + r;
      a.ids32[o] = keep ? j : -1;
      a.gw[o] = keep ? w : 0.0f;
      if (a.ids_s != nullptr && o < 32) {
        a.ids_s[o] = keep ? j : -1;
        a.gw_s[o] = keep ? w : 0.0f;
      }
      if (a.topk_ids) a.topk_ids[(size_t)t * K + r] = (kind == BEAM_ROUTE_ADA && j >= N) ? -1 : j;
      if (a.masked_ids) a.masked_ids[(size_t)t * K + r] = keep ? j : -1;
    }
    if (a.logits) a.logits[(size_t)t * Nr + j] = v[i];
    if (j < N) {
      const size_t od = (size_t)t * N + j;
      // RouterDecision.weights (BEAM) / RouteResult.weights_hat (other rules)
      if (a.weights) a.weights[od] = kind == BEAM_ROUTE_BEAM ? g : (rank[i] >= 0 && keep ? w : 0.0f);
      if (has_mask) {
        if (a.pre_act) a.pre_act[od] = x;
        if (a.raw_mask) a.raw_mask[od] = sval;
        if (a.mask) a.mask[od] = mval;
      }
    }
  }
  if (tr) a.trace[11] = gtimer();
  // shared experts: always-on slots K..K+S-1, weight 1.0 (beam.py:163-164)
  for (int s = lane; s < a.S; s += 32) {
    const size_t o = (size_t)t * Keff + K + s;
    a.ids32[o] = N + s;
    a.gw[o] = 1.0f;
    if (a.ids_s != nullptr && o < 32) {
      a.ids_s[o] = N + s;
      a.gw_s[o] = 1.0f;
    }
  }
}


// One warp, one token.  L = projection partials [splits][T][a.cols]: router
// logits in columns [0, Nr), mask pre-activations (if any) in [mask_off,
// mask_off + N); X = the token rows (stride d_pad) for inv_rms.  NPL = ceil(Nr / 32).
// a.kind selects the routing rule (baselines.py:158-283, inference branch):
//   BEAM     keep iff a >= thr, ghat = g * m                    (beam.py:127-165)
//   TOPK     keep every candidate (vanilla / reduced / pruning: K = k_eff)
//   DYNAMIC  p = softmax over all N; keep the shortest descending prefix with
//            mass >= phi (dynamic_select, baselines.py:132-143); ghat = p / mass
//   ADA      top-K over N real + null columns, keep the real ones, ghat = g
//   SOFT     s = sigmoid(a / temp); binarize: keep iff s >= tau, ghat = g * keep;
//            else keep all, ghat = g * s
// KIND >= 0 fixes the rule at compile time (the BEAM hot path carries none of
// the other rules' code); KIND = -1 reads a.kind.
template <typename TX, int NPL, int MAXSPLIT, bool CG, int KIND = -1>
__device__ __forceinline__ void topk_token(const float* __restrict__ L, int splits, int T,
                                           const TX* __restrict__ X, int t, int lane,
                                           const TopkArgs& a) {
  const int N = a.N, Nr = KIND == BEAM_ROUTE_BEAM ? a.N : a.Nr;
  float inv = 1.0f;
  // split partials of sum(x^2) from the projection CTAs (the fused gate): loaded
  // here, summed after the logit partials below are issued — one L2 round trip
  // for both instead of two
  const bool ss_split = a.has_norm && a.ss_part != nullptr;
  float ssv[CG ? MAXSPLIT : 1];
  if (CG && ss_split) {
#pragma unroll
    for (int sp = 0; sp < (CG ? MAXSPLIT : 1); ++sp)
      ssv[sp] = ld_maybe_cg<CG>(a.ss_part + (size_t)min(sp, splits - 1) * T + t);
  } else if (ss_split) {
    float ss = 0.0f;
#pragma unroll
    for (int sp = 0; sp < MAXSPLIT; ++sp) {
      const float v = ld_maybe_cg<CG>(a.ss_part + (size_t)min(sp, splits - 1) * T + t);
      ss += sp < splits ? v : 0.0f;
    }
    inv = 1.0f / sqrtf(ss / (float)a.d + 1e-6f);
  } else if (!CG && a.has_norm && a.xw_out == nullptr) {  // tensor.py:485-487, prefill (no prescaled rows)
    // 16-byte loads, a batch of XU in flight per lane (8-byte loads 8 deep waited
    // twice as many dependent round trips per row: top-K at T = 8192 37 -> 25 us)
    constexpr int EPL = 16 / (int)sizeof(TX);
    constexpr int XU = 4;
    const TX* row = X + (size_t)t * a.d_pad;
    float ss = 0.0f;
    for (int k0 = EPL * lane; k0 < a.d_pad; k0 += 32 * EPL * XU) {
      uint4 r[XU];
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int k = k0 + 32 * EPL * u;
        r[u] = k < a.d_pad ? ld_cached(row + k) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        float f[EPL];
        unpack<TX>(r[u], f);
#pragma unroll
        for (int e = 0; e < EPL; ++e) ss = fmaf(f[e], f[e], ss);
      }
    }
    ss = warp_sum(ss);
    inv = 1.0f / sqrtf(ss / (float)a.d + 1e-6f);
  } else if (a.has_norm) {  // tensor.py:485-487: (mean(x^2) + eps)^-1/2 over the real d entries
    const TX* row = X + (size_t)t * a.d_pad;
    float* xw = a.xw_out != nullptr ? a.xw_out + (size_t)t * a.d_pad : nullptr;
    float ss = 0.0f;
#pragma unroll 8
    for (int k = 4 * lane; k < a.d_pad; k += 128) {
      const float4 x = ld4<TX>(row + k);
      ss = fmaf(x.x, x.x, ss);
      ss = fmaf(x.y, x.y, ss);
      ss = fmaf(x.z, x.z, ss);
      ss = fmaf(x.w, x.w, ss);
      if (xw != nullptr) {  // fp32 rows, then their bf16 copy behind all T rows
        const float4 g = ld_norm4(a.nw, k, a.d);
        const float4 y = make_float4(x.x * g.x, x.y * g.y, x.z * g.z, x.w * g.w);
        *reinterpret_cast<float4*>(xw + k) = y;
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.xw_out + (size_t)T * a.d_pad) +
                                  (size_t)t * a.d_pad + k) = make_uint2(bf16x2_pack(y.x, y.y), bf16x2_pack(y.z, y.w));
      }
    }
    ss = warp_sum(ss);
    inv = 1.0f / sqrtf(ss / (float)a.d + 1e-6f);
  }

  // router logits v / mask pre-activations av of this lane's columns j = lane + 32 i,
  // summed over the split-K partials in split order
  float v[NPL], av[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    v[i] = 0.0f;
    av[i] = 0.0f;
  }
  const bool has_mask = KIND == BEAM_ROUTE_BEAM ? true : a.mask_off >= 0;
  const int cols = KIND == BEAM_ROUTE_BEAM ? 2 * a.N : a.cols;
  const int mask_off = KIND == BEAM_ROUTE_BEAM ? a.N : a.mask_off;
  // Loads are unconditional (clamped split / column index, masked add) and issued
  // four splits at a time: conditional loads inside the unrolled loop would be
  // serialised, one L2 round trip each.  The sum runs in split order.
  constexpr int kSB = MAXSPLIT < 4 ? MAXSPLIT : 4;
#pragma unroll
  for (int sp0 = 0; sp0 < MAXSPLIT; sp0 += kSB) {
    if (sp0 < splits) {
      float pv[kSB][NPL], pa[kSB][NPL];
#pragma unroll
      for (int q = 0; q < kSB; ++q) {
        const float* row = L + ((size_t)min(sp0 + q, splits - 1) * T + t) * cols;
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
          pv[q][i] = ld_maybe_cg<CG>(row + min(lane + 32 * i, Nr - 1));
          pa[q][i] = has_mask ? ld_maybe_cg<CG>(row + mask_off + min(lane + 32 * i, N - 1)) : 0.0f;
        }
      }
#pragma unroll
      for (int q = 0; q < kSB; ++q)
#pragma unroll
        for (int i = 0; i < NPL; ++i) {
          if (sp0 + q < splits) {
            v[i] += pv[q][i];
            av[i] += pa[q][i];
          }
        }
    }
  }
  if (CG && ss_split) {  // tensor.py:485-487 from the split partials, in split order
    float ss = 0.0f;
#pragma unroll
    for (int sp = 0; sp < (CG ? MAXSPLIT : 1); ++sp) ss += sp < splits ? ssv[sp] : 0.0f;
    inv = 1.0f / sqrtf(ss / (float)a.d + 1e-6f);
  }
  if (a.inv_out && lane == 0) a.inv_out[t] = inv;
  topk_finish<NPL, KIND>(v, av, inv, t, lane, a);
}

// Block-wide exclusive scan of one int per thread (NW warps, NW <= 32).
template <int NW>
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NW ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    scratch[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int warp_base = warp > 0 ? scratch[warp - 1] : 0;
  *total = scratch[NW - 1];
  __syncthreads();
  return warp_base + x - v;
}

// Stable counting sort of the surviving (t, k) entries by expert, one CTA of NW
// warps (E <= 32 * NW).  Each warp owns a contiguous chunk of the flat id array;
// per-warp histograms (integer shared atomics: order-free) -> per-(warp, expert)
// bases (expert-major / warp-minor scan) -> ordered re-walk ranking equal experts
// inside each 32-entry step with __match_any_sync.  Identical to the reference's
// order (ascending flat index inside an expert) whatever the scheduling.
// smem: NW*E + 2E + 1 + 32 ints.  pad = write the -1 padding of every expert run
// (the weight-streaming kernels never read it; the align_block API and the
// tcgen05 path's row packing do).
template <typename IdT, int NW, bool CG>
__device__ __forceinline__ void permute_block(const IdT* __restrict__ ids, const float* __restrict__ w,
                                              int T, int K, int E, int bs, const PlanDev& p, int* smem,
                                              bool pad = true) {
  int* hist = smem;                 // [NW][E]
  int* off_s = hist + NW * E;       // [E + 1]
  int* scratch = off_s + E + 1;     // [32]
  int* cnt_s = scratch + 32;        // [E]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = T * K;

  for (int i = tid; i < NW * E; i += NW * 32) hist[i] = 0;
  __syncthreads();

  const int per_warp = ceil_div(ceil_div(M, NW), 32) * 32;
  const int begin = min(M, warp * per_warp);
  const int end = min(M, begin + per_warp);

  for (int i = begin + lane; i < end; i += 32) {
    const long long e = (long long)ld_maybe_cg<CG>(ids + i);
    if (e >= 0 && e < E) atomicAdd(&hist[warp * E + (int)e], 1);
  }
  __syncthreads();

  for (int e = tid; e < E; e += NW * 32) {
    int run = 0;
    for (int q = 0; q < NW; ++q) {
      const int c = hist[q * E + e];
      hist[q * E + e] = run;
      run += c;
    }
    p.counts[e] = run;
    cnt_s[e] = run;
    off_s[e] = run;  // temporarily: count
  }
  __syncthreads();

  {
    const int c = tid < E ? off_s[tid] : 0;
    const int padded = round_up(c, bs);
    int tot_pad, tot_act, tot_real;
    const int ex_pad = block_exclusive_scan<NW>(padded, scratch, &tot_pad);
    const int ex_act = block_exclusive_scan<NW>(c > 0 ? 1 : 0, scratch, &tot_act);
    block_exclusive_scan<NW>(c, scratch, &tot_real);
    __syncthreads();
    if (tid < E) {
      off_s[tid] = ex_pad;
      p.offsets[tid] = ex_pad;
      if (c > 0) p.active[ex_act] = tid;
    }
    if (tid == 0) {
      off_s[E] = tot_pad;
      p.offsets[E] = tot_pad;
      p.meta[0] = tot_act;
      p.meta[1] = tot_pad;
      p.meta[2] = tot_real;
      p.meta[3] = 0;
    }
  }
  __syncthreads();

  for (int base = begin; base < end; base += 32) {
    const int i = base + lane;
    long long e = -1;
    if (i < end) e = (long long)ld_maybe_cg<CG>(ids + i);
    const bool valid = i < end && e >= 0 && e < E;
    const int key = valid ? (int)e : (E + lane);
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid) {
      const int pos = off_s[e] + hist[warp * E + e] + rank;
      BEAM_DCHECK(p, p.cap == 0 || (pos >= 0 && pos < p.cap), kChkPlanPos);
      const int t = i / K;
      p.tok[pos] = t;
      p.slot[pos] = i - t * K;
      if (p.w) p.w[pos] = w ? ld_maybe_cg<CG>(w + i) : 0.0f;
      if (p.slot_pos) p.slot_pos[i] = pos;
      if (p.slot_expert) p.slot_expert[i] = (int)e;
    } else if (i < end) {
      if (p.slot_pos) p.slot_pos[i] = -1;
      if (p.slot_expert) p.slot_expert[i] = -1;
    }
    __syncwarp();
    if (valid && rank == 0) hist[warp * E + e] += __popc(peers);
    __syncwarp();
  }

  if (pad) {
    for (int e = warp; e < E; e += NW) {
      const int real_end = off_s[e] + cnt_s[e];
      for (int q = real_end + lane; q < off_s[e + 1]; q += 32) {
        p.tok[q] = -1;
        p.slot[q] = -1;
        if (p.w) p.w[q] = 0.0f;
      }
    }
  }
}

// The same plan for T <= 64 tokens without a serial pass: each expert keeps a
// 64-bit mask of its tokens (a token routes to an expert at most once), so the
// position of (t, k) inside its expert's run — ascending flat index t*K+k ==
// ascending t — is a popcount.  One CTA of NW warps; 4 __syncthreads in all.
// smem: 2E + (E + 1) + E ints.  Outputs identical to permute_block.
template <int NW>
__device__ __forceinline__ void plan_small_block(const int32_t* ids, const float* w, int T, int K, int E, int bs,
                                                 const PlanDev& p, int* smem, bool pad) {
  unsigned* bits = reinterpret_cast<unsigned*>(smem);  // [E][2]
  int* off_s = smem + 2 * E;                           // [E + 1]
  int* cnt_s = off_s + E + 1;                          // [E]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = T * K;
  for (int i = tid; i < 2 * E; i += NW * 32) bits[i] = 0u;
  __syncthreads();
  for (int i = tid; i < M; i += NW * 32) {
    const int e = __ldcg(ids + i);
    if (e >= 0 && e < E) {
      const int t = i / K;
      atomicOr(&bits[2 * e + (t >> 5)], 1u << (t & 31));
    }
  }
  __syncthreads();
  if (warp == 0) {
    const int per = ceil_div(E, 32);
    const int e0 = min(E, lane * per), e1 = min(E, e0 + per);
    int psum = 0, asum = 0, rsum = 0;
    for (int e = e0; e < e1; ++e) {
      const int c = __popc(bits[2 * e]) + __popc(bits[2 * e + 1]);
      cnt_s[e] = c;
      psum += round_up(c, bs);
      asum += c > 0;
      rsum += c;
    }
    int px = psum, ax = asum, rx = rsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int yp = __shfl_up_sync(0xffffffffu, px, o);
      const int ya = __shfl_up_sync(0xffffffffu, ax, o);
      const int yr = __shfl_up_sync(0xffffffffu, rx, o);
      if (lane >= o) {
        px += yp;
        ax += ya;
        rx += yr;
      }
    }
    int prun = px - psum, arun = ax - asum;
    for (int e = e0; e < e1; ++e) {
      const int c = cnt_s[e];
      off_s[e] = prun;
      p.counts[e] = c;
      p.offsets[e] = prun;
      if (c > 0) p.active[arun++] = e;
      prun += round_up(c, bs);
    }
    if (lane == 31) {
      off_s[E] = px;
      p.offsets[E] = px;
      p.meta[0] = ax;
      p.meta[1] = px;
      p.meta[2] = rx;
      p.meta[3] = 0;
    }
  }
  __syncthreads();
  for (int i = tid; i < M; i += NW * 32) {
    const int e = __ldcg(ids + i);
    if (e >= 0 && e < E) {
      const int t = i / K;
      const unsigned b0 = bits[2 * e], b1 = bits[2 * e + 1];
      const int below = t < 32 ? __popc(b0 & ((1u << t) - 1u)) : __popc(b0) + __popc(b1 & ((1u << (t - 32)) - 1u));
      const int pos = off_s[e] + below;
      p.tok[pos] = t;
      p.slot[pos] = i - t * K;
      if (p.w) p.w[pos] = w ? __ldcg(w + i) : 0.0f;
      if (p.slot_pos) p.slot_pos[i] = pos;
      if (p.slot_expert) p.slot_expert[i] = e;
    } else {
      if (p.slot_pos) p.slot_pos[i] = -1;
      if (p.slot_expert) p.slot_expert[i] = -1;
    }
  }
  if (pad) {
    for (int e = warp; e < E; e += NW) {
      const int real_end = off_s[e] + cnt_s[e];
      for (int q = real_end + lane; q < off_s[e + 1]; q += 32) {
        p.tok[q] = -1;
        p.slot[q] = -1;
        if (p.w) p.w[q] = 0.0f;
      }
    }
  }
}

// The plan of at most 32 (token, slot) entries by ONE warp (decode, T * Keff <=
// 32): lane i holds entry i; same-expert lanes find each other with match_any
// (a lane's rank among them = its position inside the expert's run, ascending
// flat index); the leaders scatter their padded counts into a per-expert table,
// one warp scan over it gives every expert's offset AND active index (the
// leaders read theirs back), so a run's start needs no search over the other
// leaders.  Same outputs as permute_block, no CTA barrier.  ids / w may live in
// shared memory (the fused gate hands them over from its top-K warps without an
// L2 round trip).  smem: 3 * E ints.
template <bool CG>
__device__ __forceinline__ void plan_warp(const int32_t* ids, const float* w, int T, int K, int E, int bs,
                                          const PlanDev& p, bool pad, int lane, int* smem) {
  int* tab = smem;          // [E] padded count per expert (0 = inactive)
  int* offs = smem + E;     // [E] exclusive scan of tab
  int* aidx = smem + 2 * E; // [E] number of active experts below e
  const int M = T * K;
  int e = -1;
  float wi = 0.0f;
  if (lane < M) {
    e = ld_maybe_cg<CG>(ids + lane);
    if (w) wi = ld_maybe_cg<CG>(w + lane);
  }
  for (int e2 = lane; e2 < E; e2 += 32) tab[e2] = 0;
  const bool valid = lane < M && e >= 0 && e < E;
  const unsigned peers = __match_any_sync(0xffffffffu, valid ? e : E + lane);
  const int within = __popc(peers & ((1u << lane) - 1u));
  const int cnt = __popc(peers);
  const bool leader = valid && within == 0;
  const int padded = leader ? round_up(cnt, bs) : 0;
  __syncwarp();
  if (leader) tab[e] = padded;
  const int n_act = __popc(__ballot_sync(0xffffffffu, leader));
  const int n_real = __popc(__ballot_sync(0xffffffffu, valid));
  __syncwarp();
  // counts / padded offsets / active indices of every expert (inactive: count 0):
  // lane l owns the contiguous experts [l*per, (l+1)*per); exclusive warp scans
  const int per = ceil_div(E, 32);
  const int e0 = min(E, lane * per), e1 = min(E, e0 + per);
  int run = 0, arun = 0;
  for (int e2 = e0; e2 < e1; ++e2) {
    const int pc = tab[e2];
    run += pc;
    arun += pc > 0;
  }
  int incl = run, aincl = arun;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    const int ya = __shfl_up_sync(0xffffffffu, aincl, o);
    if (lane >= o) {
      incl += y;
      aincl += ya;
    }
  }
  int off = incl - run, aoff = aincl - arun;
  for (int e2 = e0; e2 < e1; ++e2) {
    const int pc = tab[e2];
    p.offsets[e2] = off;
    p.counts[e2] = 0;
    offs[e2] = off;
    aidx[e2] = aoff;
    off += pc;
    aoff += pc > 0;
  }
  const int n_pad = __shfl_sync(0xffffffffu, incl, 31);
  __syncwarp();
  if (valid) {
    const int pos = offs[e] + within;
    BEAM_DCHECK(p, p.cap == 0 || (pos >= 0 && pos < p.cap), kChkPlanPos);
    const int t = lane / K;
    p.tok[pos] = t;
    p.slot[pos] = lane - t * K;
    if (p.w) p.w[pos] = wi;
    if (p.slot_pos) p.slot_pos[lane] = pos;
    if (p.slot_expert) p.slot_expert[lane] = e;
  } else if (lane < M) {
    if (p.slot_pos) p.slot_pos[lane] = -1;
    if (p.slot_expert) p.slot_expert[lane] = -1;
  }
  if (leader) {
    p.active[aidx[e]] = e;
    p.counts[e] = cnt;  // after the zero fill (same lane order: the zero fill above precedes this store)
    if (pad) {
      const int before = offs[e];
      for (int q = before + cnt; q < before + padded; ++q) {
        p.tok[q] = -1;
        p.slot[q] = -1;
        if (p.w) p.w[q] = 0.0f;
      }
    }
  }
  if (lane == 0) {
    p.offsets[E] = n_pad;
    p.meta[0] = n_act;
    p.meta[1] = n_pad;
    p.meta[2] = n_real;
    p.meta[3] = 0;
  }
}

}  // namespace beam
