// Gating: RMS pre-norm, fp32 router + mask-router projection, stable top-K,
// softmax over the K candidates, and the BEAM mask threshold.
//
// Reference semantics (paths relative to /root/reference/pkg/src/beamoe/):
//   rms_norm            tensor.py:485-508   x * (mean(x^2) + 1e-6)^-1/2 * w
//   topk_route          moe.py:122-137      logits = x_n @ router_w; stable top-K
//                                           (desc value, ties -> lower id, moe.py:116-119);
//                                           softmax over exactly the K kept logits
//   mask_forward        beam.py:68-72       a = x_n @ W_m; raw = sigmoid(a); m = raw >= tau
//   mask_route          _kernels.pyx:17-34  id kept iff a[t, id] >= 0
// One fp32 predicate a >= thr (thr = 0 for tau = 0.5) feeds both the mask bit and
// the routed id; NaN -> masked.
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

// ---------------------------------------------------------------------------
// 1. RMS norm + pack: one warp per token.  Writes x_n in fp32 (router input,
//    optional) and in the expert dtype with a zero-padded row stride d_pad.
// ---------------------------------------------------------------------------
template <typename TIn, typename TAct>
__global__ void __launch_bounds__(256) norm_pack_kernel(const TIn* __restrict__ h, int T, int d,
                                                        int d_pad, const float* __restrict__ norm_w,
                                                        float* __restrict__ xn32,
                                                        TAct* __restrict__ xact) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= T) return;
  const TIn* row = h + (size_t)warp * d;
  float inv = 1.0f;
  if (norm_w != nullptr) {
    float ss = 0.0f;
    for (int i = lane; i < d; i += 32) {
      float x = to_f32<TIn>(row[i]);
      ss = fmaf(x, x, ss);
    }
    ss = warp_sum(ss);
    const float ms = ss / (float)d + 1e-6f;
    inv = 1.0f / sqrtf(ms);
  }
  for (int i = lane; i < d_pad; i += 32) {
    float v = 0.0f;
    if (i < d) {
      v = to_f32<TIn>(row[i]);
      if (norm_w != nullptr) v = (v * inv) * norm_w[i];
    }
    if (xn32) xn32[(size_t)warp * d_pad + i] = v;
    if (xact) xact[(size_t)warp * d_pad + i] = from_f32<TAct>(v);
  }
}

cudaError_t launch_norm_pack(const void* h, int h_dtype, int T, int d, int d_pad,
                             const float* norm_w, float* xn32, void* xact, int act_dtype,
                             cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  dim3 grid(ceil_div(T, 8)), block(256);
  if (h_dtype == BEAM_F32 && act_dtype == BEAM_F32)
    norm_pack_kernel<float, float><<<grid, block, 0, s>>>((const float*)h, T, d, d_pad, norm_w, xn32, (float*)xact);
  else if (h_dtype == BEAM_F32 && act_dtype == BEAM_BF16)
    norm_pack_kernel<float, __nv_bfloat16><<<grid, block, 0, s>>>((const float*)h, T, d, d_pad, norm_w, xn32, (__nv_bfloat16*)xact);
  else if (h_dtype == BEAM_BF16 && act_dtype == BEAM_F32)
    norm_pack_kernel<__nv_bfloat16, float><<<grid, block, 0, s>>>((const __nv_bfloat16*)h, T, d, d_pad, norm_w, xn32, (float*)xact);
  else
    norm_pack_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, block, 0, s>>>((const __nv_bfloat16*)h, T, d, d_pad, norm_w, xn32, (__nv_bfloat16*)xact);
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 2. Router + mask-router projection: L[T, cols] = xn32[T, d_pad] . W[cols, d_pad]^T
//    (W = [router^T ; mask^T], fp32).  Register-tiled SIMT SGEMM; each output is
//    a sequential fp32 sum over k, so results do not depend on the grid.
// ---------------------------------------------------------------------------
template <int BM, int BN>
__global__ void __launch_bounds__(256) router_gemm_kernel(const float* __restrict__ X,
                                                          const float* __restrict__ W, int T,
                                                          int cols, int d_pad,
                                                          float* __restrict__ L) {
  constexpr int BK = 32;
  constexpr int TM = BM / 16, TN = BN / 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  for (int k0 = 0; k0 < d_pad; k0 += BK) {
    // A tile: BM rows x BK cols as float4 (BK/4 = 8 float4 per row)
    for (int v = tid; v < BM * (BK / 4); v += 256) {
      const int r = v / (BK / 4), c4 = v % (BK / 4);
      const int m = m0 + r, k = k0 + c4 * 4;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < T && k < d_pad) x = *reinterpret_cast<const float4*>(X + (size_t)m * d_pad + k);
      As[c4 * 4 + 0][r] = x.x;
      As[c4 * 4 + 1][r] = x.y;
      As[c4 * 4 + 2][r] = x.z;
      As[c4 * 4 + 3][r] = x.w;
    }
    for (int v = tid; v < BN * (BK / 4); v += 256) {
      const int r = v / (BK / 4), c4 = v % (BK / 4);
      const int n = n0 + r, k = k0 + c4 * 4;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n < cols && k < d_pad) x = __ldg(reinterpret_cast<const float4*>(W + (size_t)n * d_pad + k));
      Bs[c4 * 4 + 0][r] = x.x;
      Bs[c4 * 4 + 1][r] = x.y;
      Bs[c4 * 4 + 2][r] = x.z;
      Bs[c4 * 4 + 3][r] = x.w;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < BK; ++k) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[k][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[k][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= T) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n < cols) L[(size_t)m * cols + n] = acc[i][j];
    }
  }
}

cudaError_t launch_router_gemm(const float* xn32, const float* gate_wT, int T, int cols,
                               int d_pad, float* L, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (T <= 64) {
    dim3 grid(ceil_div(T, 16), ceil_div(cols, 16));
    router_gemm_kernel<16, 16><<<grid, 256, 0, s>>>(xn32, gate_wT, T, cols, d_pad, L);
  } else {
    dim3 grid(ceil_div(T, 64), ceil_div(cols, 64));
    router_gemm_kernel<64, 64><<<grid, 256, 0, s>>>(xn32, gate_wT, T, cols, d_pad, L);
  }
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 3. Top-K + softmax + mask: one warp per token, N <= 32 * kMaxPerLane.
// ---------------------------------------------------------------------------
constexpr int kMaxPerLane = 16;  // N <= 512

__global__ void __launch_bounds__(256) topk_mask_kernel(
    const float* __restrict__ L, int T, int N, int K, int S, float thr,
    int32_t* __restrict__ ids32, float* __restrict__ gw, int64_t* __restrict__ topk_ids,
    int64_t* __restrict__ masked_ids, float* __restrict__ logits, float* __restrict__ weights,
    float* __restrict__ pre_act, float* __restrict__ raw_mask, float* __restrict__ mask) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const float* lrow = L + (size_t)t * 2 * N;
  const int Keff = K + S;

  float v[kMaxPerLane];
  int rank[kMaxPerLane];
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < N ? lrow[j] : 0.0f;
    rank[i] = -1;
  }

  float top_val = 0.0f;
  for (int r = 0; r < K; ++r) {
    // lane-local best among untaken: value desc, index asc
    bool have = false;
    float bv = 0.0f;
    int bj = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
      const int j = lane + 32 * i;
      if (j < N && rank[i] < 0) {
        if (!have || v[i] > bv) {  // j ascending within a lane: ties keep the lower j
          have = true;
          bv = v[i];
          bj = j;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      const bool ohave = __shfl_xor_sync(0xffffffffu, (int)have, o) != 0;
      const bool better = ohave && (!have || ov > bv || (ov == bv && oj < bj));
      if (better) {
        bv = ov;
        bj = oj;
        have = true;
      }
    }
    if (r == 0) top_val = bv;
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i)
      if (lane + 32 * i == bj) rank[i] = r;
  }

  // softmax over the K kept logits (tensor.py:440-451): exp(l - max) / sum
  float part = 0.0f;
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i)
    if (rank[i] >= 0) part += expf(v[i] - top_val);
  const float denom = warp_sum(part);

#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    const int j = lane + 32 * i;
    if (j >= N) continue;
    const float a = lrow[N + j];
    const bool keep = a >= thr;  // NaN -> false
    const float g = rank[i] >= 0 ? expf(v[i] - top_val) / denom : 0.0f;
    if (rank[i] >= 0) {
      const int r = rank[i];
      const size_t o = (size_t)t * Keff + r;
      ids32[o] = keep ? j : -1;
      gw[o] = keep ? g : 0.0f;
      if (topk_ids) topk_ids[(size_t)t * K + r] = j;
      if (masked_ids) masked_ids[(size_t)t * K + r] = keep ? j : -1;
    }
    const size_t od = (size_t)t * N + j;
    if (logits) logits[od] = v[i];
    if (weights) weights[od] = g;
    if (pre_act) pre_act[od] = a;
    if (raw_mask) raw_mask[od] = sigmoid_ref(a);
    if (mask) mask[od] = keep ? 1.0f : 0.0f;
  }
  // shared experts: always-on slots K..K+S-1, weight 1.0 (beam.py:163-164)
  for (int s = lane; s < S; s += 32) {
    const size_t o = (size_t)t * Keff + K + s;
    ids32[o] = N + s;
    gw[o] = 1.0f;
  }
}

cudaError_t launch_topk_mask(const float* L, int T, int N, int K, int S, float thr,
                             int32_t* ids32, float* gw, int64_t* topk_ids, int64_t* masked_ids,
                             float* logits, float* weights, float* pre_act, float* raw_mask,
                             float* mask, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  topk_mask_kernel<<<ceil_div(T, 8), 256, 0, s>>>(L, T, N, K, S, thr, ids32, gw, topk_ids,
                                                  masked_ids, logits, weights, pre_act, raw_mask,
                                                  mask);
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 4. Stand-alone dispatch.mask_route (_kernels.pyx:17-34), fp32 or fp64 a.
// ---------------------------------------------------------------------------
template <typename AT>
__global__ void mask_route_kernel(const int64_t* __restrict__ ids, const AT* __restrict__ a,
                                  int T, int K, int N, int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)T * K) return;
  const int64_t t = i / K;
  const int64_t e = ids[i];
  int64_t r = -1;
  if (e >= 0 && e < N) {
    const AT x = a[t * N + e];
    if (x >= (AT)0) r = e;  // NaN -> -1
  }
  out[i] = r;
}

cudaError_t launch_mask_route(const int64_t* ids, const void* a, int a_dtype, int T, int K,
                              int N, int64_t* out, cudaStream_t s) {
  const int64_t n = (int64_t)T * K;
  if (n <= 0) return cudaSuccess;
  const int grid = (int)((n + 255) / 256);
  if (a_dtype == BEAM_F64)
    mask_route_kernel<double><<<grid, 256, 0, s>>>(ids, (const double*)a, T, K, N, out);
  else
    mask_route_kernel<float><<<grid, 256, 0, s>>>(ids, (const float*)a, T, K, N, out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
