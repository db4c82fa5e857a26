// Expert-parallel (EP) data plane: the device halves of the dispatch / combine
// all-to-all around the NCCL collectives (paper_2605_14438_b200/ep.py).
//
// Not in the reference (expert parallelism is its open limitation);
// the per-token semantics are beam_block_forward's (beam.py:127-165): every
// surviving (token, expert) slot runs on the rank owning the expert, partial
// sums come back and are added in ascending rank order (= ascending expert
// ranges, dispatch/__init__.py:145-156), then the residual.
//
// Rank r owns experts [r*n_local, (r+1)*n_local).  Send buffers hold one row per
// (token, destination rank) pair that has at least one surviving slot there —
// deduplicated: a token with several experts on one rank travels once; a token
// whose slots on a rank are all masked does not travel there at all.
//
//   x row    the token's RAW activation row (h dtype, d elements): the owner
//            applies the RMS norm itself, so EP computes what the single-GPU
//            layer computes (norm weight folded into the expert input)
//   meta row int32[2K+1] = K local expert ids (-1: slot not on this rank /
//            masked) | K routing weights ghat (f32 bits) | inv_rms (f32 bits)
//
// Two layouts: FIXED capacity (decode: peer p's rows at [p*cap, p*cap+count_p),
// unused rows carry id -1 — no counts exchange, no host sync, graph-capturable)
// and COMPACT (prefill: peer blocks back to back, offsets from beam_ep_count's
// per-tile counts, so masked slots shrink the all-to-all).
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

constexpr int kEpTile = 256;  // tokens per CTA of the count / pack kernels
constexpr int kEpMaxWorld = 32;

// destination-rank bitmask of token t (bit p: some surviving slot on rank p)
__device__ __forceinline__ unsigned ep_dest_bits(const int64_t* __restrict__ ids, int t, int K, int N,
                                                 int n_local) {
  unsigned bits = 0u;
  for (int k = 0; k < K; ++k) {
    const long long e = ids[(size_t)t * K + k];
    if (e >= 0 && e < N) bits |= 1u << (int)(e / n_local);
  }
  return bits;
}

__global__ void __launch_bounds__(kEpTile) ep_count_kernel(const int64_t* __restrict__ ids, int T, int K, int N,
                                                           int world, int n_local, int32_t* __restrict__ tile_counts) {
  const int t = blockIdx.x * kEpTile + threadIdx.x;
  const unsigned bits = t < T ? ep_dest_bits(ids, t, K, N, n_local) : 0u;
  for (int p = 0; p < world; ++p) {
    const int c = __syncthreads_count((bits >> p) & 1u);
    if (threadIdx.x == 0) tile_counts[(size_t)p * gridDim.x + blockIdx.x] = c;
  }
}

// One CTA per 256-token tile.  cap > 0: FIXED layout (one tile, T <= 256 <= cap
// not required: T <= cap); cap == 0: COMPACT layout from tile_counts [world][ntiles].
template <typename TX>
__global__ void __launch_bounds__(kEpTile) ep_pack_kernel(const TX* __restrict__ h, int T, int d,
                                                          const int64_t* __restrict__ ids,
                                                          const float* __restrict__ weights, int N, int K,
                                                          int world, int n_local, int cap,
                                                          const int32_t* __restrict__ tile_counts, int has_norm,
                                                          TX* __restrict__ x_send, int32_t* __restrict__ meta,
                                                          int32_t* __restrict__ send_pos, int32_t* __restrict__ counts) {
  __shared__ int row_s[kEpMaxWorld][kEpTile];  // destination row of (peer, token), -1 = not sent
  __shared__ int base_s[kEpMaxWorld];
  __shared__ int scan_s[kEpTile / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntiles = gridDim.x, tile = blockIdx.x;
  const int t = tile * kEpTile + tid;
  const int MW = 2 * K + 1;
  griddep_wait();
  const unsigned bits = t < T ? ep_dest_bits(ids, t, K, N, n_local) : 0u;
  if (tid < world) {
    int b;
    if (cap > 0) {
      b = tid * cap;
    } else {  // rows of earlier peers (all tiles), then earlier tiles of this peer
      b = 0;
      for (int q = 0; q < tid; ++q)
        for (int i = 0; i < ntiles; ++i) b += tile_counts[(size_t)q * ntiles + i];
      for (int i = 0; i < tile; ++i) b += tile_counts[(size_t)tid * ntiles + i];
    }
    base_s[tid] = b;
  }
  for (int p = 0; p < world; ++p) {
    // block exclusive scan of the flag: ascending token order inside the peer's rows
    const bool f = (bits >> p) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) scan_s[warp] = __popc(bal);
    __syncthreads();
    int before = __popc(bal & ((1u << lane) - 1u));
    int total = 0;
#pragma unroll
    for (int w = 0; w < kEpTile / 32; ++w) {
      const int c = scan_s[w];
      before += w < warp ? c : 0;
      total += c;
    }
    const int row = f ? base_s[p] + before : -1;
    row_s[p][tid] = row;
    if (t < T) send_pos[(size_t)p * T + t] = row;
    if (cap > 0 && tid == 0) counts[p] = total;
    if (cap > 0) {
      // unused rows of the fixed block: every slot -1 (the owner plans nothing)
      for (int r = total + tid; r < cap; r += kEpTile) {
        int32_t* m = meta + (size_t)(p * cap + r) * MW;
        for (int k = 0; k < K; ++k) m[k] = -1;
        for (int k = K; k < MW; ++k) m[k] = 0;
      }
    }
    __syncthreads();
  }
  // metadata: local ids and weights of the slots the destination owns
  if (t < T) {
    for (int p = 0; p < world; ++p) {
      const int row = row_s[p][tid];
      if (row < 0) continue;
      int32_t* m = meta + (size_t)row * MW;
      for (int k = 0; k < K; ++k) {
        const long long e = ids[(size_t)t * K + k];
        const bool mine = e >= 0 && e < N && (int)(e / n_local) == p;
        m[k] = mine ? (int)(e - (long long)p * n_local) : -1;
        m[K + k] = __float_as_int(mine ? weights[(size_t)t * N + e] : 0.0f);
      }
    }
  }
  // rows: one warp per token — inv_rms from the row (tensor.py:485-487), then
  // the raw row to every destination (16-byte vectors when d allows)
  const int nt = min(kEpTile, T - tile * kEpTile);
  constexpr int V = 16 / sizeof(TX);
  const bool vec = d % V == 0;
  for (int i = warp; i < nt; i += kEpTile / 32) {
    const int tt = tile * kEpTile + i;
    const TX* src = h + (size_t)tt * d;
    float inv = 0.0f;
    if (has_norm) {
      float ss = 0.0f;
      for (int k = lane; k < d; k += 32) {
        const float x = to_f32<TX>(src[k]);
        ss = fmaf(x, x, ss);
      }
      ss = warp_sum(ss);
      inv = 1.0f / sqrtf(ss / (float)d + 1e-6f);
    }
    for (int p = 0; p < world; ++p) {
      const int row = row_s[p][i];
      if (row < 0) continue;
      if (lane == 0) meta[(size_t)row * MW + 2 * K] = __float_as_int(inv);
      TX* dst = x_send + (size_t)row * d;
      if (vec) {
        for (int k = lane * V; k < d; k += 32 * V)
          *reinterpret_cast<uint4*>(dst + k) = __ldg(reinterpret_cast<const uint4*>(src + k));
      } else {
        for (int k = lane; k < d; k += 32) dst[k] = src[k];
      }
    }
  }
}

// Owner side: meta rows -> ids32 / gw (slot-major [n][K]) / inv [n]; with a norm
// weight also xw = x * norm_w (fp32, stride d_pad) — the prescaled rows the
// decode expert kernels read, exactly as the single-GPU gate writes them.
template <typename TX>
__global__ void __launch_bounds__(256) ep_unpack_kernel(const int32_t* __restrict__ meta, int n, int K,
                                                        const TX* __restrict__ x, int d, int d_pad,
                                                        const float* __restrict__ nw, int32_t* __restrict__ ids32,
                                                        float* __restrict__ gw, float* __restrict__ inv,
                                                        float* __restrict__ xw) {
  const int MW = 2 * K + 1;
  griddep_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)n * K;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / K;
    const int k = (int)(i - r * K);
    ids32[i] = meta[r * MW + k];
    gw[i] = __int_as_float(meta[r * MW + K + k]);
    if (k == 0) inv[r] = __int_as_float(meta[r * MW + 2 * K]);
  }
  if (xw != nullptr) {  // fp32 rows, then their bf16 copy behind all n rows (tensor-core items)
    __nv_bfloat16* xw16 = reinterpret_cast<__nv_bfloat16*>(xw + (size_t)n * d_pad);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)n * d_pad;
         i += (long long)gridDim.x * blockDim.x) {
      const long long r = i / d_pad;
      const int k = (int)(i - r * d_pad);
      const float v = k < d ? to_f32<TX>(x[r * d + k]) * nw[k] : 0.0f;
      xw[i] = v;
      xw16[i] = __float2bfloat16_rn(v);
    }
  }
}

// Token side: out[t] = h[t] + sum over ranks p ascending of y_back[send_pos[p, t]]
// (fp32, fixed order).  One warp per (token, 256-column chunk).
template <typename TH>
__global__ void __launch_bounds__(256) ep_combine_kernel(const float* __restrict__ y_back,
                                                         const int32_t* __restrict__ send_pos, int world, int T,
                                                         int d, const TH* __restrict__ h, TH* __restrict__ out) {
  griddep_wait();
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  int pos = -1;
  if (lane < world) pos = send_pos[(size_t)lane * T + t];
  for (int c0 = blockIdx.y * 256; c0 < d; c0 += gridDim.y * 256) {
    float y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = 0.0f;
    for (int p = 0; p < world; ++p) {
      const int r = __shfl_sync(0xffffffffu, pos, p);
      if (r < 0) continue;
      const float* src = y_back + (size_t)r * d;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = c0 + lane + 32 * q;
        if (c < d) y[q] += src[c];
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = c0 + lane + 32 * q;
      if (c < d) out[(size_t)t * d + c] = from_f32<TH>(to_f32<TH>(h[(size_t)t * d + c]) + y[q]);
    }
  }
}

cudaError_t launch_ep_count(const int64_t* ids, int T, int K, int N, int world, int n_local, int32_t* tile_counts,
                            cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  ep_count_kernel<<<ceil_div(T, kEpTile), kEpTile, 0, s>>>(ids, T, K, N, world, n_local, tile_counts);
  count_launches(1);
  return cudaGetLastError();
}

int ep_tiles(int T) { return ceil_div(T, kEpTile); }

cudaError_t launch_ep_pack(const void* h, int h_dtype, int T, int d, const int64_t* ids, const float* weights, int N,
                           int K, int world, int n_local, int cap, const int32_t* tile_counts, int has_norm,
                           void* x_send, int32_t* meta, int32_t* send_pos, int32_t* counts, cudaStream_t s) {
  if (T < 0 || (T == 0 && cap == 0)) return cudaSuccess;
  if (world > kEpMaxWorld || (cap > 0 && (T > cap || T > kEpTile))) return cudaErrorInvalidValue;
  const int grid = std::max(1, ceil_div(T, kEpTile));  // fixed layout, T = 0: one CTA fills the empty blocks
  if (h_dtype == BEAM_BF16)
    launch_pdl(ep_pack_kernel<__nv_bfloat16>, grid, kEpTile, 0, s, (const __nv_bfloat16*)h, T, d, ids, weights, N, K,
               world, n_local, cap, tile_counts, has_norm, (__nv_bfloat16*)x_send, meta, send_pos, counts);
  else
    launch_pdl(ep_pack_kernel<float>, grid, kEpTile, 0, s, (const float*)h, T, d, ids, weights, N, K, world, n_local,
               cap, tile_counts, has_norm, (float*)x_send, meta, send_pos, counts);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_ep_unpack(const int32_t* meta, int n, int K, const void* x, int x_dtype, int d, int d_pad,
                             const float* nw, int32_t* ids32, float* gw, float* inv, float* xw, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long work = (long long)n * (xw ? d_pad : K);
  const int grid = (int)std::min<long long>(num_sms() * 4, std::max<long long>(1, (work + 255) / 256));
  if (x_dtype == BEAM_BF16)
    launch_pdl(ep_unpack_kernel<__nv_bfloat16>, grid, 256, 0, s, meta, n, K, (const __nv_bfloat16*)x, d, d_pad, nw, ids32,
               gw, inv, xw);
  else
    launch_pdl(ep_unpack_kernel<float>, grid, 256, 0, s, meta, n, K, (const float*)x, d, d_pad, nw, ids32, gw, inv, xw);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_ep_combine(const float* y_back, const int32_t* send_pos, int world, int T, int d, const void* h,
                              int h_dtype, void* out, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (world > 32) return cudaErrorInvalidValue;
  const int tiles = ceil_div(T, 8);
  const int gy = std::max(1, std::min(ceil_div(d, 256), ceil_div(num_sms() * 8, tiles)));
  const dim3 grid(tiles, gy);
  if (h_dtype == BEAM_BF16)
    launch_pdl(ep_combine_kernel<__nv_bfloat16>, grid, 256, 0, s, y_back, send_pos, world, T, d,
               (const __nv_bfloat16*)h, (__nv_bfloat16*)out);
  else
    launch_pdl(ep_combine_kernel<float>, grid, 256, 0, s, y_back, send_pos, world, T, d, (const float*)h, (float*)out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
