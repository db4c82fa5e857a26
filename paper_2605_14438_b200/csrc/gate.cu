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
#include "route_device.cuh"

namespace beam {

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
//     2 columns of W and a k-range; the CTA stages its 32-token tile of h for that
//     k-range in shared memory with all loads in flight, every warp issues all of
//     its weight loads up front, then accumulates 32 tokens x 2 columns in
//     registers.  Partials go to P[split][T][cols]; consumers add the splits in a
//     fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kGemvCols = 2;
constexpr int kGemvTT = 32;
constexpr int kGemvK = 128;      // k elements per lane-row step (32 lanes x 4)
constexpr int kGemvSteps = 8;    // kr <= 1024
constexpr int kFusedMaxSplit = 4;

template <typename TX, int TT>
__device__ __forceinline__ void router_gemv_body(const TX* __restrict__ X, const float* __restrict__ nw,
                                                 const float* __restrict__ W, int T, int cols, int d,
                                                 int d_pad, int kr, float* __restrict__ P, float* xs,
                                                 float* red_s, float* __restrict__ ssp = nullptr,
                                                 float* __restrict__ xw = nullptr) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int c0 = (blockIdx.x * 8 + wib) * kGemvCols;
  const int split = blockIdx.y;
  const int t0 = blockIdx.z * TT;
  const int nt = min(TT, T - t0);
  const int ks = split * kr, ke = min(d_pad, ks + kr);
  const int kn = ke - ks;
  {
    // token tile -> shared memory, loads batched U deep (each iteration's load
    // would otherwise wait a full memory round trip before the next is issued)
    constexpr int U = 4;
    const int n4 = nt * (kn >> 2);
    for (int v0 = threadIdx.x; v0 < n4; v0 += 256 * U) {
      float4 xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + 256 * u;
        const int t = v / (kn >> 2), k4 = v % (kn >> 2);
        xv[u] = v < n4 ? ld4<TX>(X + (size_t)(t0 + t) * d_pad + ks + 4 * k4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + 256 * u;
        const int t = v / (kn >> 2), k4 = v % (kn >> 2);
        if (v < n4) *reinterpret_cast<float4*>(xs + t * kr + 4 * k4) = xv[u];
      }
    }
  }
  float4 wa[kGemvSteps], wb[kGemvSteps];
  const float* w0 = W + (size_t)min(c0, cols - 1) * d_pad;
  const float* w1 = W + (size_t)min(c0 + 1, cols - 1) * d_pad;
#pragma unroll
  for (int i = 0; i < kGemvSteps; ++i) {
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
  if (ssp != nullptr && blockIdx.x == 0) {
    // per-split partial sums of x^2 for inv_rms (the top-K step adds the splits
    // in order instead of re-reading the token rows); overlaps the weight loads
    for (int t = wib; t < nt; t += 8) {
      float q = 0.0f;
      for (int k4 = lane; k4 < (kn >> 2); k4 += 32) {
        const float4 x = *reinterpret_cast<const float4*>(xs + t * kr + 4 * k4);
        q = fmaf(x.x, x.x, q);
        q = fmaf(x.y, x.y, q);
        q = fmaf(x.z, x.z, q);
        q = fmaf(x.w, x.w, q);
      }
      q = warp_sum(q);
      if (lane == 0) ssp[(size_t)split * T + t0 + t] = q;
    }
  }
  if (ssp != nullptr && xw != nullptr) {
    // the norm-weighted token rows x * w (fp32, exactly the product the decode
    // gate/up kernels formed per chunk) for the expert stage: its inner loop
    // then loads one row per token and does no per-chunk norm multiply; a bf16
    // copy right behind them ([T, d_pad] after the fp32 rows) feeds the
    // tensor-core items as one MMA operand.  Spread over the tile's column CTAs
    // (they all hold the token tile), so no CTA's projection waits on all of it.
    {
      __nv_bfloat16* xw16 = reinterpret_cast<__nv_bfloat16*>(xw + (size_t)T * d_pad);
      for (int v = threadIdx.x + 256 * blockIdx.x; v < nt * (kn >> 2); v += 256 * gridDim.x) {
        const int t = v / (kn >> 2), k4 = v % (kn >> 2);
        const float4 x = *reinterpret_cast<const float4*>(xs + t * kr + 4 * k4);
        const float4 g = ld_norm4(nw, ks + 4 * k4, d);
        const float4 y = make_float4(x.x * g.x, x.y * g.y, x.z * g.z, x.w * g.w);
        const size_t o = (size_t)(t0 + t) * d_pad + ks + 4 * k4;
        *reinterpret_cast<float4*>(xw + o) = y;
        *reinterpret_cast<uint2*>(xw16 + o) = make_uint2(bf16x2_pack(y.x, y.y), bf16x2_pack(y.z, y.w));
      }
    }
  }
  float acc[kGemvCols * TT];
#pragma unroll
  for (int i = 0; i < kGemvCols * TT; ++i) acc[i] = 0.0f;
#pragma unroll
  for (int i = 0; i < kGemvSteps; ++i) {
    const int kk = 4 * lane + kGemvK * i;
    if (ks + kk < ke) {
      const float4 a = wa[i], b = wb[i];
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        if (t < nt) {
          const float4 x = *reinterpret_cast<const float4*>(xs + t * kr + kk);
          float s0 = acc[t], s1 = acc[TT + t];
          s0 = fmaf(a.x, x.x, s0); s0 = fmaf(a.y, x.y, s0); s0 = fmaf(a.z, x.z, s0); s0 = fmaf(a.w, x.w, s0);
          s1 = fmaf(b.x, x.x, s1); s1 = fmaf(b.y, x.y, s1); s1 = fmaf(b.z, x.z, s1); s1 = fmaf(b.w, x.w, s1);
          acc[t] = s0;
          acc[TT + t] = s1;
        }
      }
    }
  }
  warp_reduce_to_smem<kGemvCols * TT>(acc, red_s + wib * kGemvCols * TT, lane);
  if (c0 < cols) {
    for (int i = lane; i < kGemvCols * TT; i += 32) {
      const int j = i / TT, t = i % TT;
      if (t < nt && c0 + j < cols) P[((size_t)split * T + t0 + t) * cols + c0 + j] = red_s[wib * kGemvCols * TT + i];
    }
  }
}

template <typename TX>
__global__ void __launch_bounds__(256) router_gemv_kernel(const TX* __restrict__ X,
                                                          const float* __restrict__ nw,
                                                          const float* __restrict__ W, int T,
                                                          int cols, int d, int d_pad, int kr,
                                                          float* __restrict__ P) {
  extern __shared__ float xs[];
  __shared__ float red_s[8 * kGemvCols * kGemvTT];
  router_gemv_body<TX, kGemvTT>(X, nw, W, T, cols, d, d_pad, kr, P, xs, red_s);
}

// k-range per split: enough CTAs to cover the SMs, kr <= kGemvSteps * 128
static int gemv_kr(int T, int cols, int d_pad, int max_split, int tt = kGemvTT) {
  const int col_ctas = ceil_div(cols, 8 * kGemvCols);
  const int tok_ctas = ceil_div(T, tt);
  int s = ceil_div(num_sms(), col_ctas * tok_ctas);
  const int smin = ceil_div(d_pad, kGemvSteps * kGemvK);
  s = std::min(s, max_split);
  s = std::min(s, ceil_div(d_pad, kGemvK));
  s = std::max(s, smin);
  return ceil_div(ceil_div(d_pad, s), kGemvK) * kGemvK;
}

// The decode projection writes at most kRouterMaxSplit split-K partials: the
// workspace holds that many [T][cols] slabs (abi.cu carve) and the top-K kernel
// sums at most that many.  kr <= kGemvSteps * kGemvK = 1024 covers d_pad <= 16384.
constexpr int kRouterMaxSplit = 16;

int router_splits(int T, int cols, int d_pad) {
  if (T > 64) return 1;
  return ceil_div(d_pad, gemv_kr(T, cols, d_pad, kRouterMaxSplit));
}

template <typename K>
static void set_smem(K kernel, int bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

cudaError_t launch_router(const void* X, int x_dtype, const float* norm_w, const float* gate_wT,
                          int T, int cols, int d, int d_pad, float* P, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (T <= 64) {
    const int kr = gemv_kr(T, cols, d_pad, kRouterMaxSplit);
    dim3 grid(ceil_div(cols, 8 * kGemvCols), ceil_div(d_pad, kr), ceil_div(T, kGemvTT));
    if ((int)grid.y > kRouterMaxSplit) return cudaErrorInvalidValue;  // d_pad > 16384: before any launch
    const size_t smem = (size_t)kGemvTT * kr * sizeof(float);
    static bool attr = false;
    if (!attr) {
      set_smem(router_gemv_kernel<__nv_bfloat16>, kGemvTT * kGemvSteps * kGemvK * 4);
      set_smem(router_gemv_kernel<float>, kGemvTT * kGemvSteps * kGemvK * 4);
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
// 3. Stand-alone top-K + softmax + mask (prefill / wide N): one warp per token.
// ---------------------------------------------------------------------------
template <typename TX, int NPL, int KIND>
__global__ void __launch_bounds__(128, NPL <= 4 ? 8 : 1) topk_mask_kernel(const float* __restrict__ L, int splits,
                                                        const TX* __restrict__ X, int T, TopkArgs a) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  topk_token<TX, NPL, 16, false, KIND>(L, splits, T, X, t, threadIdx.x & 31, a);
}

template <typename TX, int KIND>
static void topk_dispatch_k(const float* L, int splits, const void* X, int T, const TopkArgs& a, cudaStream_t s) {
  const int grid = ceil_div(T, 4);
  const int npl = ceil_div(a.Nr, 32);
  if (npl <= 1) topk_mask_kernel<TX, 1, KIND><<<grid, 128, 0, s>>>(L, splits, (const TX*)X, T, a);
  else if (npl <= 2) topk_mask_kernel<TX, 2, KIND><<<grid, 128, 0, s>>>(L, splits, (const TX*)X, T, a);
  else if (npl <= 4) topk_mask_kernel<TX, 4, KIND><<<grid, 128, 0, s>>>(L, splits, (const TX*)X, T, a);
  else if (npl <= 8) topk_mask_kernel<TX, 8, KIND><<<grid, 128, 0, s>>>(L, splits, (const TX*)X, T, a);
  else topk_mask_kernel<TX, 16, KIND><<<grid, 128, 0, s>>>(L, splits, (const TX*)X, T, a);
}

template <typename TX>
static void topk_dispatch(const float* L, int splits, const void* X, int T, const TopkArgs& a, cudaStream_t s) {
  if (a.kind == BEAM_ROUTE_BEAM && a.Nr == a.N && a.cols == 2 * a.N && a.mask_off == a.N)
    topk_dispatch_k<TX, BEAM_ROUTE_BEAM>(L, splits, X, T, a, s);
  else
    topk_dispatch_k<TX, -1>(L, splits, X, T, a, s);
}

cudaError_t launch_topk_mask(const float* L, int splits, const void* X, int x_dtype, int T,
                             const TopkArgs& a, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (splits > kRouterMaxSplit) return cudaErrorInvalidValue;
  if (x_dtype == BEAM_BF16) topk_dispatch<__nv_bfloat16>(L, splits, X, T, a, s);
  else topk_dispatch<float>(L, splits, X, T, a, s);
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 3b. Fused decode gate (T <= 64, E <= 256): projection + top-K + permute in ONE
//     launch.  Every CTA computes its projection partials; the last CTA of each
//     32-token tile (global counter, threadfence pattern) runs top-K / mask for
//     the tile; the last tile to finish runs the stable permute for all tokens.
//     Counters live at the start of the zero-initialised workspace and are reset
//     by their last user, so the kernel is replayable (CUDA graphs).
// ---------------------------------------------------------------------------
constexpr int kFusedTT = 8;        // tokens per fused-gate tile (one warp per token in phase 2)

// Diagnostics (beam_trace_gate): when set, the fused gate records %globaltimer
// at its phase boundaries: [0] first CTA start (min), [1] last CTA start (max),
// [2] first / [3] last projection done, [6] last top-K tile start, [4] last top-K
// tile done, [7] permute start, [5] permute done.
__device__ unsigned long long* g_gate_trace = nullptr;


__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void trace_minmax(int lo, int hi) {
  unsigned long long* tr = g_gate_trace;
  if (tr != nullptr && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    if (lo >= 0) atomicMin(tr + lo, t);
    if (hi >= 0) atomicMax(tr + hi, t);
  }
}
constexpr int kCounterSlots = 16;  // [0, 8) token tiles, [15] tiles-done

template <typename TX, int NPL, int KIND>
__global__ void __launch_bounds__(256) gate_fused_kernel(const TX* __restrict__ X, const float* __restrict__ nw,
                                                         const float* __restrict__ W, int T, int d, int d_pad,
                                                         int kr, float* __restrict__ P, TopkArgs a, int E,
                                                         int bs, bool pad, PlanDev p, int* __restrict__ counters,
                                                         float* __restrict__ xw) {
  extern __shared__ float xs[];  // phase 1: token tile; phase 3: permute scratch
  __shared__ float red_s[8 * kGemvCols * kFusedTT];
  __shared__ int s_last;
  const int cols = a.cols;
  float* ssp = nw != nullptr ? P + (size_t)kFusedMaxSplit * T * cols : nullptr;
  trace_minmax(0, 1);
  router_gemv_body<TX, kFusedTT>(X, nw, W, T, cols, d, d_pad, kr, P, xs, red_s, ssp, xw);
  trace_minmax(2, 3);

  // ---- last CTA of this token tile: top-K + mask ----
  // handoff: the CTA barrier orders every thread's partial stores before thread
  // 0's acq_rel (gpu scope, cumulative) counter increment; the last CTA's
  // increment acquires all of them (no per-thread __threadfence)
  __syncthreads();
  const int tile = blockIdx.z;
  if (threadIdx.x == 0) s_last = atom_add_acq_rel(&counters[tile], 1) == (int)(gridDim.x * gridDim.y) - 1;
  __syncthreads();
  if (!s_last) return;
  trace_minmax(-1, 6);
  const int t0 = tile * kFusedTT, nt = min(kFusedTT, T - t0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool one_warp_plan = gridDim.z == 1 && T * (a.K + a.S) <= 32;
  TopkArgs b = a;
  b.ss_part = ssp;
  b.trace = g_gate_trace;
  int* scratch = reinterpret_cast<int*>(xs);  // plan_warp: [0, 3 E) (reads ids_s / gw_s before writing there)
  if (one_warp_plan) {
    b.ids_s = scratch + 320;
    b.gw_s = reinterpret_cast<float*>(scratch + 352);
  }
  for (int t = t0 + warp; t < t0 + nt; t += 8)
    topk_token<TX, NPL, kFusedMaxSplit, true, KIND>(P, gridDim.y, T, X, t, lane, b);
  if (threadIdx.x == 0) counters[tile] = 0;
  __syncthreads();
  trace_minmax(-1, 4);
  if (one_warp_plan) {
    // one token tile and <= 32 slots: this CTA holds every routed id (its own
    // warps just wrote them, mirrored in shared memory) — one warp builds the
    // plan, no second handoff
    trace_minmax(-1, 7);
    if (warp == 0) plan_warp<false>(b.ids_s, b.gw_s, T, a.K + a.S, E, bs, p, pad, lane, scratch);
    trace_minmax(-1, 5);
    return;
  }

  // ---- last token tile overall: permute all T tokens ----
  __syncthreads();
  if (threadIdx.x == 0) s_last = atom_add_acq_rel(&counters[kCounterSlots - 1], 1) == (int)gridDim.z - 1;
  __syncthreads();
  if (!s_last) return;
  trace_minmax(-1, 7);
  // (plan_small_block<8> — the bitmask plan — measured slower here than the
  // counting sort: 5.0 vs 4.0 us at T = 1, 7.3 vs 5.6 us at T = 64)
  permute_block<int32_t, 8, true>(a.ids32, a.gw, T, a.K + a.S, E, bs, p, reinterpret_cast<int*>(xs), pad);
  if (threadIdx.x == 0) counters[kCounterSlots - 1] = 0;
  __syncthreads();
  trace_minmax(-1, 5);
}

cudaError_t set_gate_trace(unsigned long long* buf) {
  return cudaMemcpyToSymbol(g_gate_trace, &buf, sizeof(buf));
}

bool gate_fused_supported(int T, int N, int E, int d_pad) {
  return T >= 1 && T <= 64 && N <= 512 && E <= 256 && d_pad % 4 == 0;
}

template <typename TX, int NPL, int KIND>
static cudaError_t fused_launch(dim3 grid, size_t smem, const void* X, const float* nw, const float* W, int T,
                                int d, int d_pad, int kr, float* P, const TopkArgs& a, int E, int bs,
                                bool pad, const PlanDev& p, int* counters, float* xw, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    set_smem(gate_fused_kernel<TX, NPL, KIND>, 160 * 1024);
    attr = true;
  }
  gate_fused_kernel<TX, NPL, KIND><<<grid, 256, smem, s>>>((const TX*)X, nw, W, T, d, d_pad, kr, P, a, E, bs, pad, p, counters,
                                                            nw != nullptr ? xw : nullptr);
  return cudaGetLastError();
}

cudaError_t launch_gate_fused(const void* X, int x_dtype, const float* norm_w, const float* gate_wT, int T,
                              int d, int d_pad, float* P, const TopkArgs& a, int E, int bs,
                              bool pad, const PlanDev& p, int* counters, cudaStream_t s, float* xw) {
  const int cols = a.cols;
  const int kr = gemv_kr(T, cols, d_pad, kFusedMaxSplit, kFusedTT);
  dim3 grid(ceil_div(cols, 8 * kGemvCols), ceil_div(d_pad, kr), ceil_div(T, kFusedTT));
  if ((int)grid.y > kFusedMaxSplit || (int)grid.z > kCounterSlots - 1) return cudaErrorInvalidValue;
  const size_t smem = std::max((size_t)kFusedTT * kr * sizeof(float), (size_t)(8 * E + 2 * E + 1 + 32) * sizeof(int));
  const int npl = ceil_div(a.Nr, 32);
  cudaError_t e;
#define BEAM_FUSED(TX_, K_)                                                                                    \
  if (npl <= 1) e = fused_launch<TX_, 1, K_>(grid, smem, X, norm_w, gate_wT, T, d, d_pad, kr, P, a, E, bs, pad, p, counters, xw, s); \
  else if (npl <= 2) e = fused_launch<TX_, 2, K_>(grid, smem, X, norm_w, gate_wT, T, d, d_pad, kr, P, a, E, bs, pad, p, counters, xw, s); \
  else if (npl <= 4) e = fused_launch<TX_, 4, K_>(grid, smem, X, norm_w, gate_wT, T, d, d_pad, kr, P, a, E, bs, pad, p, counters, xw, s); \
  else if (npl <= 8) e = fused_launch<TX_, 8, K_>(grid, smem, X, norm_w, gate_wT, T, d, d_pad, kr, P, a, E, bs, pad, p, counters, xw, s); \
  else e = fused_launch<TX_, 16, K_>(grid, smem, X, norm_w, gate_wT, T, d, d_pad, kr, P, a, E, bs, pad, p, counters, xw, s);
  const bool beam = a.kind == BEAM_ROUTE_BEAM && a.Nr == a.N && a.cols == 2 * a.N && a.mask_off == a.N;
  if (x_dtype == BEAM_BF16) {
    if (beam) { BEAM_FUSED(__nv_bfloat16, BEAM_ROUTE_BEAM) } else { BEAM_FUSED(__nv_bfloat16, -1) }
  } else {
    if (beam) { BEAM_FUSED(float, BEAM_ROUTE_BEAM) } else { BEAM_FUSED(float, -1) }
  }
#undef BEAM_FUSED
  count_launches(1);
  return e;
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

// ---------------------------------------------------------------------------
// 5. Stand-alone topk_select (moe.py:116-119): argsort(-logits, stable)[:k] on
//    arbitrary fp32 / fp64 logits.  One warp per row; round r picks the best
//    entry strictly below round r-1's pick in the total order (value desc, ties
//    -> lower index), so no per-entry state is kept for any N.  numpy's order:
//    -0.0 == +0.0 (stable), +inf first, -inf after every finite value, NaN last.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long order_key(double x) {
  if (x != x) return 0ull;  // NaN: last
  if (x == 0.0) x = 0.0;    // -0.0 ties with +0.0 (stable sort keeps index order)
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // >= 1 for every non-NaN value
}

template <typename TL>
__global__ void __launch_bounds__(256) topk_select_kernel(const TL* __restrict__ L, int T, int N, int K,
                                                          int64_t* __restrict__ out) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const TL* r = L + (size_t)row * N;
  unsigned long long lk = ~0ull;  // previous pick (key, index); the first round has no bound
  int lj = -1;
  for (int k = 0; k < K; ++k) {
    unsigned long long bk = 0ull;
    int bj = 0x7fffffff;
    for (int j = lane; j < N; j += 32) {
      const unsigned long long key = order_key((double)r[j]);
      const bool below = k == 0 || key < lk || (key == lk && j > lj);
      const bool better = key > bk || (key == bk && j < bj);
      if (below && better) {
        bk = key;
        bj = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ok > bk || (ok == bk && oj < bj)) {
        bk = ok;
        bj = oj;
      }
    }
    if (lane == 0) out[(size_t)row * K + k] = bj;
    lk = bk;
    lj = bj;
  }
}

cudaError_t launch_topk_select(const void* logits, int dtype, int T, int N, int K, int64_t* out, cudaStream_t s) {
  if (T <= 0 || K <= 0) return cudaSuccess;
  const int grid = ceil_div(T, 8);
  if (dtype == BEAM_F64)
    topk_select_kernel<double><<<grid, 256, 0, s>>>((const double*)logits, T, N, K, out);
  else
    topk_select_kernel<float><<<grid, 256, 0, s>>>((const float*)logits, T, N, K, out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
