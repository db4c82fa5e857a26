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
// B200 design: one CTA of 32 warps.  Each warp owns a contiguous chunk of the flat
// id array; pass 1 builds per-warp histograms in shared memory (integer atomics:
// order-free), pass 2 turns them into per-(warp, expert) bases with a scan in
// expert-major / warp-minor order, pass 3 re-walks each chunk in order and ranks
// equal experts inside a 32-entry step with __match_any_sync.  The result is the
// reference's order exactly, with no dependence on scheduling.
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

constexpr int kPermuteThreads = 1024;
constexpr int kPermuteWarps = kPermuteThreads / 32;

// Block-wide exclusive scan of one int per thread (1024 threads).
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
    int w = scratch[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    scratch[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const int warp_base = warp > 0 ? scratch[warp - 1] : 0;
  *total = scratch[31];
  __syncthreads();
  return warp_base + x - v;
}

template <typename IdT>
__global__ void __launch_bounds__(kPermuteThreads, 1)
    permute_kernel(const IdT* __restrict__ ids, const float* __restrict__ w, int T, int K, int E,
                   int bs, PlanDev p) {
  extern __shared__ int smem[];
  int* hist = smem;                        // [kPermuteWarps][E]
  int* off_s = hist + kPermuteWarps * E;   // [E + 1]
  int* scratch = off_s + E + 1;            // [32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = T * K;

  for (int i = tid; i < kPermuteWarps * E; i += kPermuteThreads) hist[i] = 0;
  __syncthreads();

  const int per_warp = ceil_div(ceil_div(M, kPermuteWarps), 32) * 32;
  const int begin = min(M, warp * per_warp);
  const int end = min(M, begin + per_warp);

  // pass 1: per-warp histograms
  for (int i = begin + lane; i < end; i += 32) {
    const long long e = (long long)ids[i];
    if (e >= 0 && e < E) atomicAdd(&hist[warp * E + (int)e], 1);
  }
  __syncthreads();

  // pass 2a: per-(warp, expert) exclusive bases, per-expert totals
  for (int e = tid; e < E; e += kPermuteThreads) {
    int run = 0;
    for (int q = 0; q < kPermuteWarps; ++q) {
      const int c = hist[q * E + e];
      hist[q * E + e] = run;
      run += c;
    }
    p.counts[e] = run;
    off_s[e] = run;  // temporarily: count
  }
  __syncthreads();

  // pass 2b: padded offsets + active-expert list (E <= 1024: one expert per thread)
  {
    const int c = tid < E ? off_s[tid] : 0;
    const int padded = round_up(c, bs);
    int tot_pad, tot_act, tot_real;
    const int ex_pad = block_exclusive_scan(padded, scratch, &tot_pad);
    const int ex_act = block_exclusive_scan(c > 0 ? 1 : 0, scratch, &tot_act);
    block_exclusive_scan(c, scratch, &tot_real);
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

  // pass 3: stable scatter
  for (int base = begin; base < end; base += 32) {
    const int i = base + lane;
    long long e = -1;
    if (i < end) e = (long long)ids[i];
    const bool valid = i < end && e >= 0 && e < E;
    const int key = valid ? (int)e : (E + lane);
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid) {
      const int pos = off_s[e] + hist[warp * E + e] + rank;
      const int t = i / K;
      p.tok[pos] = t;
      p.slot[pos] = i - t * K;
      if (p.w) p.w[pos] = w ? w[i] : 0.0f;
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

  // padding tail of every expert run
  for (int e = warp; e < E; e += kPermuteWarps) {
    const int real_end = off_s[e] + p.counts[e];
    for (int q = real_end + lane; q < off_s[e + 1]; q += 32) {
      p.tok[q] = -1;
      p.slot[q] = -1;
      if (p.w) p.w[q] = 0.0f;
    }
  }
}

template <typename IdT>
cudaError_t launch_permute(const IdT* ids, const float* w, int T, int K, int E, int bs,
                           const PlanDev& p, cudaStream_t s) {
  if (E > kPermuteThreads || bs < 1) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(kPermuteWarps * E + E + 1 + 32) * sizeof(int);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(permute_kernel<IdT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  permute_kernel<IdT><<<1, kPermuteThreads, smem, s>>>(ids, w, T, K, E, bs, p);
  count_launches(1);
  return cudaGetLastError();
}

template cudaError_t launch_permute<int32_t>(const int32_t*, const float*, int, int, int, int,
                                             const PlanDev&, cudaStream_t);
template cudaError_t launch_permute<int64_t>(const int64_t*, const float*, int, int, int, int,
                                             const PlanDev&, cudaStream_t);

// ---------------------------------------------------------------------------
// grouped_execute plan preparation: routing weight per planned position, the
// (t, k) -> position map, and the reference's two contract checks
// (dispatch/__init__.py:143-144 nnz(weights_hat) == real slots, :152-153 no
// zero-weight planned slot).  slot_pos / slot_expert must be preset to -1.
// ---------------------------------------------------------------------------
__global__ void plan_prepare_kernel(const int32_t* __restrict__ counts,
                                    const int32_t* __restrict__ offsets,
                                    const int32_t* __restrict__ tokens,
                                    const int32_t* __restrict__ slots,
                                    const float* __restrict__ weights_hat, int T, int K, int N,
                                    PlanDev p, int32_t* __restrict__ flags) {
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

__global__ void nnz_count_kernel(const float* __restrict__ x, long long n,
                                 const int32_t* __restrict__ meta, int32_t* __restrict__ flags) {
  int c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    c += x[i] != 0.0f;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&flags[0], c);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicSub(&flags[0], meta[2]);
}

cudaError_t launch_plan_prepare(const int32_t* counts, const int32_t* offsets,
                                const int32_t* tokens, const int32_t* slots, const int32_t* meta,
                                const float* weights_hat, int T, int K, int N, const PlanDev& p,
                                int32_t* flags, cudaStream_t s) {
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
