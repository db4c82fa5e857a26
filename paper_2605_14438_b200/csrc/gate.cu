// Gating: fp32 router + mask-router projection with the RMS pre-norm folded in,
// stable top-K, softmax over the K candidates, and the BEAM mask threshold.
//
// Reference semantics (paths relative to /root/reference/pkg/src/beamoe/):
//   rms_norm            tensor.py:485-508   x_n = x * (mean(x^2) + 1e-6)^-1/2 * w
//   topk_route          moe.py:122-137      logits = x_n @ router_w; stable top-K
//                                           (desc value, ties -> lower id, moe.py:116-119);
//                                           softmax over exactly the K kept logits
//   mask_forward        beam.py:68-72       a = x_n @ W_m; raw = sigmoid(a); m = raw >= tau
//   mask_route          _kernels.pyx:17-34  id kept iff a[t, id] >= 0
// One fp32 predicate a >= thr (thr = 0 for tau = 0.5) feeds both the mask bit and
// the routed id; NaN -> masked.
//
// B200 design: x_n is never materialised.  Because the norm is a per-token scale,
// x_n . W[c] = inv_rms[t] * sum_k h[t,k] * (w[k] * W[c,k]); the projection
// kernels stream h (bf16/f32) against W*w and the top-K kernel (one warp per
// token) computes inv_rms from the same h row, applies it, selects, and writes
// inv_rms for the expert kernels, which normalise x on load.
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

// ---------------------------------------------------------------------------
// 0. pad / convert rows to stride d_pad (only when d_h is not a multiple of 8)
// ---------------------------------------------------------------------------
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(256) pad_rows_kernel(const TIn* __restrict__ h, int T, int d,
                                                       int d_pad, TOut* __restrict__ out) {
  const size_t n = (size_t)T * d_pad;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / d_pad), k = (int)(i % d_pad);
    out[i] = from_f32<TOut>(k < d ? to_f32<TIn>(h[(size_t)t * d + k]) : 0.0f);
  }
}

cudaError_t launch_pad_rows(const void* h, int h_dtype, int T, int d, int d_pad, void* out,
                            int out_dtype, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const int grid = (int)std::min<size_t>(4096, ((size_t)T * d_pad + 255) / 256);
  if (h_dtype == BEAM_F32 && out_dtype == BEAM_F32)
    pad_rows_kernel<float, float><<<grid, 256, 0, s>>>((const float*)h, T, d, d_pad, (float*)out);
  else if (h_dtype == BEAM_F32)
    pad_rows_kernel<float, __nv_bfloat16><<<grid, 256, 0, s>>>((const float*)h, T, d, d_pad, (__nv_bfloat16*)out);
  else if (out_dtype == BEAM_F32)
    pad_rows_kernel<__nv_bfloat16, float><<<grid, 256, 0, s>>>((const __nv_bfloat16*)h, T, d, d_pad, (float*)out);
  else
    pad_rows_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)h, T, d, d_pad, (__nv_bfloat16*)out);
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 1. stand-alone RMS norm (beam_rms_norm): one warp per token, fp32 out
// ---------------------------------------------------------------------------
template <typename TIn>
__global__ void __launch_bounds__(256) rms_norm_kernel(const TIn* __restrict__ h, int T, int d,
                                                       const float* __restrict__ norm_w,
                                                       float* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= T) return;
  const TIn* row = h + (size_t)warp * d;
  float ss = 0.0f;
  for (int i = lane; i < d; i += 32) {
    const float x = to_f32<TIn>(row[i]);
    ss = fmaf(x, x, ss);
  }
  ss = warp_sum(ss);
  const float inv = 1.0f / sqrtf(ss / (float)d + 1e-6f);
  for (int i = lane; i < d; i += 32) out[(size_t)warp * d + i] = (to_f32<TIn>(row[i]) * inv) * norm_w[i];
}

cudaError_t launch_rms_norm(const void* h, int h_dtype, int T, int d, const float* norm_w,
                            float* out, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (h_dtype == BEAM_BF16)
    rms_norm_kernel<__nv_bfloat16><<<ceil_div(T, 8), 256, 0, s>>>((const __nv_bfloat16*)h, T, d, norm_w, out);
  else
    rms_norm_kernel<float><<<ceil_div(T, 8), 256, 0, s>>>((const float*)h, T, d, norm_w, out);
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 2a. Prefill projection (T > 64): register-tiled SIMT SGEMM
//     P[t, c] = sum_k h[t,k] * w[k] * W[c,k]   (h: [T, d_pad] of TX)
// ---------------------------------------------------------------------------
template <typename TX, int BM, int BN>
__global__ void __launch_bounds__(256) router_gemm_kernel(const TX* __restrict__ X,
                                                          const float* __restrict__ nw,
                                                          const float* __restrict__ W, int T,
                                                          int cols, int d, int d_pad,
                                                          float* __restrict__ P) {
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
    for (int v = tid; v < BM * (BK / 4); v += 256) {
      const int r = v / (BK / 4), c4 = v % (BK / 4);
      const int m = m0 + r, k = k0 + c4 * 4;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < T && k < d_pad) x = ld4<TX>(X + (size_t)m * d_pad + k);
      As[c4 * 4 + 0][r] = x.x;
      As[c4 * 4 + 1][r] = x.y;
      As[c4 * 4 + 2][r] = x.z;
      As[c4 * 4 + 3][r] = x.w;
    }
    for (int v = tid; v < BN * (BK / 4); v += 256) {
      const int r = v / (BK / 4), c4 = v % (BK / 4);
      const int n = n0 + r, k = k0 + c4 * 4;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n < cols && k < d_pad) {
        x = __ldg(reinterpret_cast<const float4*>(W + (size_t)n * d_pad + k));
        const float4 g = ld_norm4(nw, k, d);
        x.x *= g.x; x.y *= g.y; x.z *= g.z; x.w *= g.w;
      }
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
      if (n < cols) P[(size_t)m * cols + n] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// 2b. Decode projection (T <= 64): split-K weight-streaming GEMV.  Each warp owns
//     2 columns of W and a k-range, keeps 32 tokens x 2 fp32 accumulators in
//     registers, streams W once per 32-token tile with 16-byte loads and reads h
//     through L1.  Partials go to P[split][T][cols]; the top-K kernel adds the
//     splits in a fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kGemvCols = 2;
constexpr int kGemvTT = 32;
constexpr int kGemvK = 128;  // k elements per lane-row step (32 lanes x 4)

template <typename TX>
__global__ void __launch_bounds__(256) router_gemv_kernel(const TX* __restrict__ X,
                                                          const float* __restrict__ nw,
                                                          const float* __restrict__ W, int T,
                                                          int cols, int d, int d_pad, int kr,
                                                          float* __restrict__ P) {
  extern __shared__ float xs[];  // [kGemvTT][kr] fp32 token tile of this k-range
  __shared__ float red_s[8][kGemvCols * kGemvTT];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int c0 = (blockIdx.x * 8 + wib) * kGemvCols;
  const int split = blockIdx.y;
  const int t0 = blockIdx.z * kGemvTT;
  const int nt = min(kGemvTT, T - t0);
  const int ks = split * kr, ke = min(d_pad, ks + kr);
  const int kn = ke - ks;
  // stage the token tile: every thread issues its loads before any use
  for (int v = threadIdx.x; v < nt * (kn >> 2); v += 256) {
    const int t = v / (kn >> 2), k4 = v % (kn >> 2);
    const float4 x = ld4<TX>(X + (size_t)(t0 + t) * d_pad + ks + 4 * k4);
    *reinterpret_cast<float4*>(xs + t * kr + 4 * k4) = x;
  }
  // this warp's weight chunks (all in flight at once)
  constexpr int kMaxSteps = 8;  // kr <= 8 * 128
  float4 wa[kMaxSteps], wb[kMaxSteps];
  const float* w0 = W + (size_t)min(c0, cols - 1) * d_pad;
  const float* w1 = W + (size_t)min(c0 + 1, cols - 1) * d_pad;
#pragma unroll
  for (int i = 0; i < kMaxSteps; ++i) {
    const int k = ks + 4 * lane + kGemvK * i;
    if (k < ke) {
      wa[i] = __ldg(reinterpret_cast<const float4*>(w0 + k));
      wb[i] = __ldg(reinterpret_cast<const float4*>(w1 + k));
      const float4 g = ld_norm4(nw, k, d);
      wa[i].x *= g.x; wa[i].y *= g.y; wa[i].z *= g.z; wa[i].w *= g.w;
      wb[i].x *= g.x; wb[i].y *= g.y; wb[i].z *= g.z; wb[i].w *= g.w;
    }
  }
  __syncthreads();
  float acc[kGemvCols * kGemvTT];
#pragma unroll
  for (int i = 0; i < kGemvCols * kGemvTT; ++i) acc[i] = 0.0f;
#pragma unroll
  for (int i = 0; i < kMaxSteps; ++i) {
    const int kk = 4 * lane + kGemvK * i;  // offset inside the k-range
    if (ks + kk < ke) {
      const float4 a = wa[i], b = wb[i];
#pragma unroll
      for (int t = 0; t < kGemvTT; ++t) {
        if (t < nt) {
          const float4 x = *reinterpret_cast<const float4*>(xs + t * kr + kk);
          float s0 = acc[t], s1 = acc[kGemvTT + t];
          s0 = fmaf(a.x, x.x, s0); s0 = fmaf(a.y, x.y, s0); s0 = fmaf(a.z, x.z, s0); s0 = fmaf(a.w, x.w, s0);
          s1 = fmaf(b.x, x.x, s1); s1 = fmaf(b.y, x.y, s1); s1 = fmaf(b.z, x.z, s1); s1 = fmaf(b.w, x.w, s1);
          acc[t] = s0;
          acc[kGemvTT + t] = s1;
        }
      }
    }
  }
  warp_reduce_to_smem<kGemvCols * kGemvTT>(acc, red_s[wib], lane);
  if (c0 < cols) {
    for (int i = lane; i < kGemvCols * kGemvTT; i += 32) {
      const int j = i / kGemvTT, t = i % kGemvTT;
      if (t < nt && c0 + j < cols) P[((size_t)split * T + t0 + t) * cols + c0 + j] = red_s[wib][i];
    }
  }
}

static int gemv_kr(int T, int cols, int d_pad) {
  const int col_ctas = ceil_div(cols, 8 * kGemvCols);
  const int tok_ctas = ceil_div(T, kGemvTT);
  int s = ceil_div(num_sms(), col_ctas * tok_ctas);
  const int smax = ceil_div(d_pad, kGemvK);
  const int smin = ceil_div(d_pad, 8 * kGemvK);  // kr <= 1024 (registers / smem)
  if (s < smin) s = smin;
  s = s < 1 ? 1 : (s > smax ? smax : s);
  return ceil_div(ceil_div(d_pad, s), kGemvK) * kGemvK;
}

int router_splits(int T, int cols, int d_pad) {
  if (T > 64) return 1;
  return ceil_div(d_pad, gemv_kr(T, cols, d_pad));
}

cudaError_t launch_router(const void* X, int x_dtype, const float* norm_w, const float* gate_wT,
                          int T, int cols, int d, int d_pad, float* P, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (T <= 64) {
    const int kr = gemv_kr(T, cols, d_pad);
    dim3 grid(ceil_div(cols, 8 * kGemvCols), ceil_div(d_pad, kr), ceil_div(T, kGemvTT));
    const size_t smem = (size_t)kGemvTT * kr * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(router_gemv_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      cudaFuncSetAttribute(router_gemv_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      attr = true;
    }
    if (x_dtype == BEAM_BF16)
      router_gemv_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>((const __nv_bfloat16*)X, norm_w, gate_wT, T, cols, d, d_pad, kr, P);
    else
      router_gemv_kernel<float><<<grid, 256, smem, s>>>((const float*)X, norm_w, gate_wT, T, cols, d, d_pad, kr, P);
  } else {
    dim3 grid(ceil_div(T, 64), ceil_div(cols, 64));
    if (x_dtype == BEAM_BF16)
      router_gemm_kernel<__nv_bfloat16, 64, 64><<<grid, 256, 0, s>>>((const __nv_bfloat16*)X, norm_w, gate_wT, T, cols, d, d_pad, P);
    else
      router_gemm_kernel<float, 64, 64><<<grid, 256, 0, s>>>((const float*)X, norm_w, gate_wT, T, cols, d, d_pad, P);
  }
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 3. Top-K + softmax + mask: one warp per token, N <= 32 * kMaxPerLane.
//    Computes inv_rms from the token's h row, sums the projection partials,
//    selects the K largest (desc value, asc index), writes everything.
// ---------------------------------------------------------------------------
constexpr int kMaxPerLane = 16;  // N <= 512

template <typename TX>
__global__ void __launch_bounds__(128) topk_mask_kernel(
    const float* __restrict__ L, int splits, const TX* __restrict__ X, int d, int d_pad,
    int has_norm, int T, int N, int K, int S, float thr, float* __restrict__ inv_out,
    int32_t* __restrict__ ids32, float* __restrict__ gw, int64_t* __restrict__ topk_ids,
    int64_t* __restrict__ masked_ids, float* __restrict__ logits, float* __restrict__ weights,
    float* __restrict__ pre_act, float* __restrict__ raw_mask, float* __restrict__ mask) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int Keff = K + S;

  float inv = 1.0f;
  if (has_norm) {  // tensor.py:485-487: (mean(x^2) + eps)^-1/2 over the real d entries
    const TX* row = X + (size_t)t * d_pad;
    float ss = 0.0f;
#pragma unroll 8
    for (int k = 4 * lane; k < d_pad; k += 128) {
      const float4 x = ld4<TX>(row + k);
      ss = fmaf(x.x, x.x, ss);
      ss = fmaf(x.y, x.y, ss);
      ss = fmaf(x.z, x.z, ss);
      ss = fmaf(x.w, x.w, ss);
    }
    ss = warp_sum(ss);
    inv = 1.0f / sqrtf(ss / (float)d + 1e-6f);
  }
  if (inv_out && lane == 0) inv_out[t] = inv;

  // router logits v and mask pre-activations av of this lane's experts, summed
  // over the split-K partials in split order (all loads of a split in flight)
  float v[kMaxPerLane], av[kMaxPerLane];
  int rank[kMaxPerLane];
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    v[i] = 0.0f;
    av[i] = 0.0f;
    rank[i] = -1;
  }
  for (int sp = 0; sp < splits; ++sp) {
    const float* row = L + ((size_t)sp * T + t) * 2 * N;
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
      const int j = lane + 32 * i;
      if (j < N) {
        v[i] += row[j];
        av[i] += row[N + j];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxPerLane; ++i) {
    v[i] *= inv;
    av[i] *= inv;
  }

  float top_val = 0.0f;
  for (int r = 0; r < K; ++r) {
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
    const float a = av[i];
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

cudaError_t launch_topk_mask(const float* L, int splits, const void* X, int x_dtype, int d,
                             int d_pad, int has_norm, int T, int N, int K, int S, float thr,
                             float* inv_out, int32_t* ids32, float* gw, int64_t* topk_ids,
                             int64_t* masked_ids, float* logits, float* weights, float* pre_act,
                             float* raw_mask, float* mask, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const int grid = ceil_div(T, 4);
  if (x_dtype == BEAM_BF16)
    topk_mask_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(L, splits, (const __nv_bfloat16*)X, d, d_pad, has_norm, T, N, K, S, thr, inv_out, ids32, gw, topk_ids, masked_ids, logits, weights, pre_act, raw_mask, mask);
  else
    topk_mask_kernel<float><<<grid, 128, 0, s>>>(L, splits, (const float*)X, d, d_pad, has_norm, T, N, K, S, thr, inv_out, ids32, gw, topk_ids, masked_ids, logits, weights, pre_act, raw_mask, mask);
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
