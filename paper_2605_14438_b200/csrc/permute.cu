// Masked permute / block alignment: a deterministic, stable counting sort of the
// surviving (token, slot) pairs by expert, with per-expert padding to a multiple
// of block_size.  Masked (-1) and out-of-range ids cost nothing downstream.
//
// Reference semantics (/root/reference/pkg/src/beamoe/):
//   group_by_expert  dispatch/_kernels.pyx:37-66  count pass, exclusive scan,
//                                                 stable scatter in flat t*K+k order
//   align_block      dispatch/__init__.py:89-126  pad each expert run with -1 to
//                                                 ceil(c/bs)*bs
//   (paper listing   PAPER.md:772-782: vLLM's moe_align_block_size skipping -1)
//
// Small inputs: one CTA of 32 warps (permute_block in route_device.cuh).  Large
// inputs (prefill, T*K > 16384): two grid-wide passes — per-CTA histograms with
// the last CTA scanning them into per-(CTA, expert) bases, then an ordered
// scatter that recomputes per-warp bases inside each CTA.  Both give the
// reference's order exactly, independent of scheduling.
#include "route_device.cuh"

namespace beam {

constexpr int kPermuteThreads = 1024;
constexpr int kPermuteWarps = kPermuteThreads / 32;

template <typename IdT>
__global__ void __launch_bounds__(kPermuteThreads, 1)
    permute_kernel(const IdT* __restrict__ ids, const float* __restrict__ w, int T, int K, int E, int bs,
                   PlanDev p) {
  extern __shared__ int smem[];
  permute_block<IdT, kPermuteWarps, false>(ids, w, T, K, E, bs, p, smem);
}

// ---------------------------------------------------------------------------
// multi-CTA permute
// ---------------------------------------------------------------------------
constexpr int kMcThreads = 256;
constexpr int kMcWarps = kMcThreads / 32;
constexpr int kMcChunk = 1024;                  // entries per CTA (T*K / 1024 CTAs in flight)
constexpr int kMcPerWarp = kMcChunk / kMcWarps;  // 128, multiple of 32
constexpr long long kSingleCtaMax = 16384;

// per-warp histograms of this CTA's chunk (shared), sh = [kMcWarps][E]
template <typename IdT>
__device__ __forceinline__ void chunk_hist(const IdT* __restrict__ ids, int M, int E, int* sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kMcWarps * E; i += kMcThreads) sh[i] = 0;
  __syncthreads();
  const int begin = blockIdx.x * kMcChunk + warp * kMcPerWarp;
  const int end = min(M, begin + kMcPerWarp);
  long long ev[kMcPerWarp / 32];  // all of the warp's ids in flight at once
#pragma unroll
  for (int j = 0; j < kMcPerWarp / 32; ++j) {
    const int i = begin + lane + 32 * j;
    ev[j] = i < end ? (long long)ids[i] : -1;
  }
#pragma unroll
  for (int j = 0; j < kMcPerWarp / 32; ++j)
    if (ev[j] >= 0 && ev[j] < E) atomicAdd(&sh[warp * E + (int)ev[j]], 1);
  __syncthreads();
}

// pass 1: hist_g[cta][e] = this CTA's count of expert e; the last CTA converts
// them to exclusive bases over CTAs and writes counts / offsets / active / meta.
template <typename IdT>
__global__ void __launch_bounds__(kMcThreads) permute_hist_kernel(const IdT* __restrict__ ids, int M, int E,
                                                                  int bs, PlanDev p, int* __restrict__ hist_g,
                                                                  int* __restrict__ counter) {
  extern __shared__ int sh[];
  __shared__ int s_last;
  __shared__ int scratch[32];
  __shared__ int carry[3];
  const int tid = threadIdx.x;
  chunk_hist<IdT>(ids, M, E, sh);
  for (int e = tid; e < E; e += kMcThreads) {
    int c = 0;
    for (int q = 0; q < kMcWarps; ++q) c += sh[q * E + e];
    hist_g[(size_t)blockIdx.x * E + e] = c;
  }
  // handoff: CTA barrier, then one acq_rel (gpu scope, cumulative) increment by
  // thread 0; the last CTA's increment acquires every CTA's histogram
  __syncthreads();
  if (tid == 0) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
    s_last = old == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  const int G = gridDim.x;
  if (tid == 0) carry[0] = carry[1] = carry[2] = 0;
  __syncthreads();
  for (int e0 = 0; e0 < E; e0 += kMcThreads) {
    const int e = e0 + tid;
    int run = 0;
    if (e < E) {
      int q = 0;
      for (; q + 32 <= G; q += 32) {  // 32 independent loads per round
        int c[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) c[u] = __ldcg(hist_g + (size_t)(q + u) * E + e);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          hist_g[(size_t)(q + u) * E + e] = run;
          run += c[u];
        }
      }
      for (; q < G; ++q) {
        const int c = __ldcg(hist_g + (size_t)q * E + e);
        hist_g[(size_t)q * E + e] = run;
        run += c;
      }
      p.counts[e] = run;
    }
    int tot_pad, tot_act, tot_real;
    const int ex_pad = block_exclusive_scan<kMcWarps>(e < E ? round_up(run, bs) : 0, scratch, &tot_pad);
    const int ex_act = block_exclusive_scan<kMcWarps>(e < E && run > 0 ? 1 : 0, scratch, &tot_act);
    block_exclusive_scan<kMcWarps>(run, scratch, &tot_real);
    if (e < E) {
      p.offsets[e] = carry[0] + ex_pad;
      if (run > 0) p.active[carry[1] + ex_act] = e;
    }
    __syncthreads();
    if (tid == 0) {
      carry[0] += tot_pad;
      carry[1] += tot_act;
      carry[2] += tot_real;
    }
    __syncthreads();
  }
  if (tid == 0) {
    p.offsets[E] = carry[0];
    p.meta[0] = carry[1];
    p.meta[1] = carry[0];
    p.meta[2] = carry[2];
    p.meta[3] = 0;
    *counter = 0;  // replayable
  }
}

// pass 2: ordered scatter.  Per-warp bases = offsets[e] + CTA base + earlier warps.
template <typename IdT>
__global__ void __launch_bounds__(kMcThreads) permute_scatter_kernel(const IdT* __restrict__ ids,
                                                                     const float* __restrict__ w, int M, int K,
                                                                     int E, PlanDev p,
                                                                     const int* __restrict__ hist_g) {
  extern __shared__ int sh[];  // [kMcWarps][E] counts, then bases
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  chunk_hist<IdT>(ids, M, E, sh);
  for (int e = tid; e < E; e += kMcThreads) {
    int run = p.offsets[e] + hist_g[(size_t)blockIdx.x * E + e];
    for (int q = 0; q < kMcWarps; ++q) {
      const int c = sh[q * E + e];
      sh[q * E + e] = run;
      run += c;
    }
  }
  __syncthreads();
  const int begin = blockIdx.x * kMcChunk + warp * kMcPerWarp;
  const int end = min(M, begin + kMcPerWarp);
  long long ev[kMcPerWarp / 32];  // the warp's ids and weights loaded once, all in flight
  float wv[kMcPerWarp / 32];
#pragma unroll
  for (int j = 0; j < kMcPerWarp / 32; ++j) {
    const int i = begin + lane + 32 * j;
    ev[j] = i < end ? (long long)ids[i] : -1;
    wv[j] = i < end && w != nullptr ? w[i] : 0.0f;
  }
#pragma unroll
  for (int j = 0; j < kMcPerWarp / 32; ++j) {
    const int i = begin + 32 * j + lane;
    if (begin + 32 * j >= end) break;
    const long long e = ev[j];
    const bool valid = i < end && e >= 0 && e < E;
    const int key = valid ? (int)e : (E + lane);
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid) {
      const int pos = sh[warp * E + e] + rank;
      BEAM_DCHECK(p, p.cap == 0 || (pos >= 0 && pos < p.cap), kChkPlanPos);
      const int t = i / K;
      p.tok[pos] = t;
      p.slot[pos] = i - t * K;
      if (p.w) p.w[pos] = wv[j];
      if (p.slot_pos) p.slot_pos[i] = pos;
      if (p.slot_expert) p.slot_expert[i] = (int)e;
    } else if (i < end) {
      if (p.slot_pos) p.slot_pos[i] = -1;
      if (p.slot_expert) p.slot_expert[i] = -1;
    }
    __syncwarp();
    if (valid && rank == 0) sh[warp * E + e] += __popc(peers);
    __syncwarp();
  }
  // padding tails (grid-stride over experts)
  for (int e = blockIdx.x * kMcWarps + warp; e < E; e += gridDim.x * kMcWarps) {
    const int real_end = p.offsets[e] + p.counts[e];
    for (int q = real_end + lane; q < p.offsets[e + 1]; q += 32) {
      p.tok[q] = -1;
      p.slot[q] = -1;
      if (p.w) p.w[q] = 0.0f;
    }
  }
}

size_t permute_scratch_bytes(int T, int K, int E) {
  const long long M = (long long)T * K;
  const long long G = (M + kMcChunk - 1) / kMcChunk;
  return (size_t)(G * E + 64) * sizeof(int);
}

template <typename IdT>
cudaError_t launch_permute(const IdT* ids, const float* w, int T, int K, int E, int bs, const PlanDev& p,
                           int* scratch, cudaStream_t s) {
  if (E > kPermuteThreads || bs < 1) return cudaErrorInvalidValue;
  const long long M = (long long)T * K;
  if (M <= kSingleCtaMax || scratch == nullptr) {
    const size_t smem = (size_t)(kPermuteWarps * E + 2 * E + 1 + 32) * sizeof(int);
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(permute_kernel<IdT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr_set = true;
    }
    permute_kernel<IdT><<<1, kPermuteThreads, smem, s>>>(ids, w, T, K, E, bs, p);
    count_launches(1);
    return cudaGetLastError();
  }
  // scratch: [0, 64) ints = counter (zero-initialised, reset by the last CTA), then hist_g
  int* counter = scratch;
  int* hist_g = scratch + 64;
  const int G = (int)((M + kMcChunk - 1) / kMcChunk);
  const size_t smem = (size_t)kMcWarps * E * sizeof(int);
  static bool attr_mc = false;
  if (!attr_mc) {
    cudaFuncSetAttribute(permute_hist_kernel<IdT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(permute_scatter_kernel<IdT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr_mc = true;
  }
  permute_hist_kernel<IdT><<<G, kMcThreads, smem, s>>>(ids, (int)M, E, bs, p, hist_g, counter);
  permute_scatter_kernel<IdT><<<G, kMcThreads, smem, s>>>(ids, w, (int)M, K, E, p, hist_g);
  count_launches(2);
  return cudaGetLastError();
}

template cudaError_t launch_permute<int32_t>(const int32_t*, const float*, int, int, int, int, const PlanDev&,
                                             int*, cudaStream_t);
template cudaError_t launch_permute<int64_t>(const int64_t*, const float*, int, int, int, int, const PlanDev&,
                                             int*, cudaStream_t);

// ---------------------------------------------------------------------------
// grouped_execute plan preparation: routing weight per planned position, the
// (t, k) -> position map, and the reference's two contract checks
// (dispatch/__init__.py:143-144 nnz(weights_hat) == real slots, :152-153 no
// zero-weight planned slot).  slot_pos / slot_expert must be preset to -1.
// ---------------------------------------------------------------------------
__global__ void plan_prepare_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ offsets,
                                    const int32_t* __restrict__ tokens, const int32_t* __restrict__ slots,
                                    const float* __restrict__ weights_hat, int T, int K, int N, PlanDev p,
                                    int32_t* __restrict__ flags) {
  const int e = blockIdx.x;
  const int c = counts[e], off = offsets[e];
  for (int q = threadIdx.x; q < c; q += blockDim.x) {
    const int t = tokens[off + q], k = slots[off + q];
    const float wv = weights_hat[(size_t)t * N + e];
    p.w[off + q] = wv;
    if (wv == 0.0f && flags) atomicOr(&flags[1], 1);
    p.slot_pos[(size_t)t * K + k] = off + q;
    p.slot_expert[(size_t)t * K + k] = e;
  }
}

__global__ void nnz_count_kernel(const float* __restrict__ x, long long n, const int32_t* __restrict__ meta,
                                 int32_t* __restrict__ flags) {
  int c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    c += x[i] != 0.0f;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&flags[0], c);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicSub(&flags[0], meta[2]);
}

cudaError_t launch_plan_prepare(const int32_t* counts, const int32_t* offsets, const int32_t* tokens,
                                const int32_t* slots, const int32_t* meta, const float* weights_hat, int T, int K,
                                int N, const PlanDev& p, int32_t* flags, cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(p.slot_pos, 0xff, (size_t)T * K * sizeof(int32_t), s))) return e;
  if ((e = cudaMemsetAsync(p.slot_expert, 0xff, (size_t)T * K * sizeof(int32_t), s))) return e;
  if (flags && (e = cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), s))) return e;
  if (N > 0) {
    plan_prepare_kernel<<<N, 256, 0, s>>>(counts, offsets, tokens, slots, weights_hat, T, K, N, p, flags);
    count_launches(1);
  }
  if (flags) {
    const long long n = (long long)T * N;
    const int grid = (int)std::min<long long>(1024, std::max<long long>(1, (n + 255) / 256));
    nnz_count_kernel<<<grid, 256, 0, s>>>(weights_hat, n, meta, flags);
    count_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace beam
