// Weight-streaming grouped SwiGLU experts (decode / fp32 path).
//
// Reference: dispatch.grouped_execute (/root/reference/pkg/src/beamoe/dispatch/
// __init__.py:129-157) running expert_forward_np (moe.py:96-100)
//     O_e = (act(X_e W_gate) * (X_e W_up)) W_down,   y[rows] += O_e * ghat
// over the surviving slots of every expert, ascending expert id.
//
// B200 design (HBM-bound regime: few tokens per expert).  Only experts the mask
// left active are touched: work items (active expert, row group) are enumerated
// on the device from the permute kernel's active list — no host sync, no bytes
// for masked experts.  One CTA (256 threads) owns an item and splits its K range
// across all threads, so every weight byte of the item is requested at once
// (8 x 16-byte L1-bypassing loads per thread) and small batches are latency-, not
// issue-bound.  Partial dot products are reduced with a warp transpose-reduce
// butterfly, then across warps through shared memory in a fixed order
// (deterministic, independent of the grid).  Two launches:
//   gateup: 4 gate + 4 up rows per item -> act[pos, f] = act(g) * u   (fp32)
//   down:   2 x 8 output rows per item  -> opair[pos, d] = ghat * (act . W_down)
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
// CTA-item kernels (T <= 2): resident CTAs per SM = weight bytes in flight per SM
// (32 KB each); the warp-item kernels keep 2.
constexpr int kCtaPerSm = 2;

// EPC consecutive input elements (at a multiple of EPC) as floats.
template <typename TX, int EPC>
__device__ __forceinline__ void load_x(const TX* __restrict__ p, float* out) {
  if constexpr (sizeof(TX) * EPC == 16) {
    unpack<TX>(ld_cached(p), out);
  } else if constexpr (sizeof(TX) == 4) {  // f32 input, 8-wide chunk: two 16 B loads
    unpack<float>(ld_cached(p), out);
    unpack<float>(ld_cached(p + 4), out + 4);
  } else {  // bf16 input, 4-wide chunk: one 8 B load
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    out[0] = __uint_as_float(v.x << 16);
    out[1] = __uint_as_float(v.x & 0xffff0000u);
    out[2] = __uint_as_float(v.y << 16);
    out[3] = __uint_as_float(v.y & 0xffff0000u);
  }
}

// ---------------------------------------------------------------------------
// gate / up
// ---------------------------------------------------------------------------
template <typename TW, typename TX, int ACT, int TB>
__device__ __forceinline__ void gateup_cta_tile(const TW* __restrict__ W, int row_g,
                                            const TX* __restrict__ X, const float* __restrict__ inv,
                                            const float* __restrict__ nw, int d, int d_pad, int f_pad,
                                            int feat0, const int32_t* __restrict__ tokp, int pos0,
                                            int ntok, float* __restrict__ act, float* part,
                                            float* red) {
  constexpr int EPC = Chunk<TW>::kElems;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nch = d_pad / EPC;
  int tk[TB];
#pragma unroll
  for (int j = 0; j < TB; ++j) tk[j] = tokp[j < ntok ? j : 0];
  float acc[8 * TB];
#pragma unroll
  for (int i = 0; i < 8 * TB; ++i) acc[i] = 0.0f;
  const TW* wbase = W + (size_t)row_g * d_pad;

  for (int c = tid; c < nch; c += kThreads) {
    uint4 wv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) wv[q] = ld_stream(wbase + ((q & 3) + (q >> 2) * 16) * d_pad + c * EPC);
    float xf[TB][EPC];
#pragma unroll
    for (int j = 0; j < TB; ++j) load_x<TX, EPC>(X + (size_t)tk[j] * d_pad + c * EPC, xf[j]);
    if (nw) {  // x * w here; the per-token inv_rms is applied after the reduction
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        const int k = c * EPC + e;
        const float ge = k < d ? __ldg(nw + k) : 0.0f;
#pragma unroll
        for (int j = 0; j < TB; ++j) xf[j][e] *= ge;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float wf[EPC];
      unpack<TW>(wv[q], wf);
#pragma unroll
      for (int j = 0; j < TB; ++j)
#pragma unroll
        for (int e = 0; e < EPC; ++e) acc[q * TB + j] = fmaf(wf[e], xf[j][e], acc[q * TB + j]);
    }
  }
  // warp butterfly, then a fixed-order cross-warp sum
  warp_reduce_to_smem<8 * TB>(acc, part + warp * 8 * TB, lane);
  __syncthreads();
  if (tid < 8 * TB) {
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) s += part[q * 8 * TB + tid];
    red[tid] = s;
  }
  __syncthreads();
  if (tid < 4 * TB) {
    const int p = tid / TB, j = tid % TB;
    if (j < ntok) {
      // x_n = x * inv_rms * w: the per-token inv_rms factors out of the dot product
      const float s = inv ? inv[tk[j]] : 1.0f;
      const float gs = red[p * TB + j] * s, u = red[(4 + p) * TB + j] * s;
      act[(size_t)(pos0 + j) * f_pad + feat0 + p] = activation<ACT>(gs) * u;
    }
  }
}

template <typename TW, typename TX, int ACT>
__global__ void __launch_bounds__(kThreads, kCtaPerSm) gateup_cta_kernel(const TW* __restrict__ Wgu,
                                                             const TX* __restrict__ X,
                                                             const float* __restrict__ inv,
                                                             const float* __restrict__ nw, int d,
                                                             int d_pad, int f_pad, PlanDev p,
                                                             float* __restrict__ act) {
  __shared__ float part[kWarps * 32];
  __shared__ float red[32];
  griddep_wait();
  const int groups = f_pad / 4;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = blockIdx.x; item < total; item += gridDim.x) {
    const int a = (int)(item / groups), g = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    const TW* W = Wgu + (size_t)e * 2 * f_pad * d_pad;
    const int feat0 = g * 4;
    const int row_g = (feat0 >> 4) * 32 + (feat0 & 15);
    for (int t0 = 0; t0 < cnt;) {  // T <= 2 (small_batch): at most 2 tokens per expert
      const int r = cnt - t0;
      if (r >= 2) {
        gateup_cta_tile<TW, TX, ACT, 2>(W, row_g, X, inv, nw, d, d_pad, f_pad, feat0, p.tok + off + t0,
                                    off + t0, 2, act, part, red);
        t0 += 2;
      } else {
        gateup_cta_tile<TW, TX, ACT, 1>(W, row_g, X, inv, nw, d, d_pad, f_pad, feat0, p.tok + off + t0,
                                    off + t0, 1, act, part, red);
        t0 += 1;
      }
      __syncthreads();  // part/red reuse
    }
  }
}

// ---------------------------------------------------------------------------
// down: two halves of the CTA each own 8 output rows
// ---------------------------------------------------------------------------
template <typename TW, int TB>
__device__ __forceinline__ void down_cta_tile(const TW* __restrict__ W, int row0, int rows_valid,
                                          const float* __restrict__ act, int f_pad, int d_pad,
                                          int pos0, int ntok, const float* __restrict__ wpos,
                                          float* __restrict__ opair, float* part, float* red) {
  constexpr int EPC = Chunk<TW>::kElems;
  constexpr int kHalf = kThreads / 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = tid / kHalf, ht = tid % kHalf;
  const int nch = f_pad / EPC;
  const int rbase = row0 + 8 * half;
  float acc[8 * TB];
#pragma unroll
  for (int i = 0; i < 8 * TB; ++i) acc[i] = 0.0f;
  const float* ar[TB];
#pragma unroll
  for (int j = 0; j < TB; ++j) ar[j] = act + (size_t)(pos0 + (j < ntok ? j : 0)) * f_pad;

  if (8 * half < rows_valid) {
    const TW* wbase = W + (size_t)rbase * f_pad;
    for (int c = ht; c < nch; c += kHalf) {
      uint4 wv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) wv[q] = ld_stream(wbase + q * f_pad + c * EPC);
      float af[TB][EPC];
#pragma unroll
      for (int j = 0; j < TB; ++j)
#pragma unroll
        for (int v = 0; v < EPC / 4; ++v) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(ar[j] + c * EPC) + v);
          af[j][4 * v + 0] = x.x;
          af[j][4 * v + 1] = x.y;
          af[j][4 * v + 2] = x.z;
          af[j][4 * v + 3] = x.w;
        }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float wf[EPC];
        unpack<TW>(wv[q], wf);
#pragma unroll
        for (int j = 0; j < TB; ++j)
#pragma unroll
          for (int e = 0; e < EPC; ++e) acc[q * TB + j] = fmaf(wf[e], af[j][e], acc[q * TB + j]);
      }
    }
  }
  // per-half reduction (warps 0-3 -> rows 0-7, warps 4-7 -> rows 8-15)
  warp_reduce_to_smem<8 * TB>(acc, part + warp * 8 * TB, lane);
  __syncthreads();
  if (ht < 8 * TB) {
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < kWarps / 2; ++q) s += part[(half * (kWarps / 2) + q) * 8 * TB + ht];
    red[half * 8 * TB + ht] = s;
  }
  __syncthreads();
  if (ht < 8 * TB) {
    const int q = ht / TB, j = ht % TB;
    if (j < ntok && 8 * half + q < rows_valid)
      opair[(size_t)(pos0 + j) * d_pad + rbase + q] = red[half * 8 * TB + q * TB + j] * wpos[j];
  }
}

template <typename TW>
__global__ void __launch_bounds__(kThreads, kCtaPerSm) down_cta_kernel(const TW* __restrict__ Wd,
                                                           const float* __restrict__ act, int d_pad,
                                                           int f_pad, PlanDev p,
                                                           float* __restrict__ opair) {
  __shared__ float part[kWarps * 32];
  __shared__ float red[64];
  griddep_wait();
  const int groups = ceil_div(d_pad, 16);
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = blockIdx.x; item < total; item += gridDim.x) {
    const int a = (int)(item / groups), g = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    const TW* W = Wd + (size_t)e * d_pad * f_pad;
    const int row0 = g * 16, rows_valid = min(16, d_pad - row0);
    for (int t0 = 0; t0 < cnt;) {  // T <= 2 (small_batch): at most 2 tokens per expert
      const int r = cnt - t0;
      if (r >= 2) {
        down_cta_tile<TW, 2>(W, row0, rows_valid, act, f_pad, d_pad, off + t0, 2, p.w + off + t0, opair,
                         part, red);
        t0 += 2;
      } else {
        down_cta_tile<TW, 1>(W, row0, rows_valid, act, f_pad, d_pad, off + t0, 1, p.w + off + t0, opair,
                         part, red);
        t0 += 1;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// warp-item kernels (T > 8): one warp streams a row group of an expert over the
// whole K range; many warps per SM keep the HBM pipe full without CTA barriers.
// ---------------------------------------------------------------------------
template <typename TW, typename TX, int ACT, int TB>
__device__ __forceinline__ void gateup_warp_tile(const TW* __restrict__ W, int row_g,
                                                 const TX* __restrict__ X, const float* __restrict__ inv,
                                                 const float* __restrict__ nw, int d, int d_pad, int f_pad,
                                                 int feat0, const int32_t* __restrict__ tokp, int pos0,
                                                 int ntok, float* __restrict__ act, float* red, int lane) {
  constexpr int EPC = Chunk<TW>::kElems;
  const int nch = d_pad / EPC;
  int tk[TB];
#pragma unroll
  for (int j = 0; j < TB; ++j) tk[j] = tokp[j < ntok ? j : 0];
  float acc[8 * TB];
#pragma unroll
  for (int i = 0; i < 8 * TB; ++i) acc[i] = 0.0f;
  const TW* wbase = W + (size_t)row_g * d_pad;
  for (int c = lane; c < nch; c += 32) {
    uint4 wv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) wv[q] = ld_stream(wbase + ((q & 3) + (q >> 2) * 16) * d_pad + c * EPC);
    float xf[TB][EPC];
#pragma unroll
    for (int j = 0; j < TB; ++j) load_x<TX, EPC>(X + (size_t)tk[j] * d_pad + c * EPC, xf[j]);
    if (nw) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
        const int k = c * EPC + e;
        const float ge = k < d ? __ldg(nw + k) : 0.0f;
#pragma unroll
        for (int j = 0; j < TB; ++j) xf[j][e] *= ge;
      }
    }
    // rows in pairs (2p, 2p+1) through FFMA2: half the FMA instructions
#pragma unroll
    for (int p2 = 0; p2 < 4; ++p2) {
      float wa[EPC], wb[EPC];
      unpack<TW>(wv[2 * p2], wa);
      unpack<TW>(wv[2 * p2 + 1], wb);
#pragma unroll
      for (int j = 0; j < TB; ++j)
#pragma unroll
        for (int e = 0; e < EPC; ++e)
          ffma2(acc[(2 * p2) * TB + j], acc[(2 * p2 + 1) * TB + j], wa[e], wb[e], xf[j][e]);
    }
  }
  warp_reduce_to_smem<8 * TB>(acc, red, lane);
  if (lane < 4 * TB) {
    const int p = lane / TB, j = lane % TB;
    if (j < ntok) {
      const float s = inv ? inv[tk[j]] : 1.0f;
      const float gs = red[p * TB + j] * s, u = red[(4 + p) * TB + j] * s;
      act[(size_t)(pos0 + j) * f_pad + feat0 + p] = activation<ACT>(gs) * u;
    }
  }
  __syncwarp();
}

template <typename TW, typename TX, int ACT>
__global__ void __launch_bounds__(kThreads, 2) gateup_warp_kernel(const TW* __restrict__ Wgu,
                                                                  const TX* __restrict__ X,
                                                                  const float* __restrict__ inv,
                                                                  const float* __restrict__ nw, int d,
                                                                  int d_pad, int f_pad, PlanDev p,
                                                                  float* __restrict__ act) {
  __shared__ float red_s[kWarps][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * kWarps + wib, nwarps = gridDim.x * kWarps;
  griddep_wait();
  const int groups = f_pad / 4;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = gwarp; item < total; item += nwarps) {
    const int a = (int)(item / groups), g = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    const TW* W = Wgu + (size_t)e * 2 * f_pad * d_pad;
    const int feat0 = g * 4;
    const int row_g = (feat0 >> 4) * 32 + (feat0 & 15);
    for (int t0 = 0; t0 < cnt;) {
      const int r = cnt - t0;
      if (r >= 3) {
        gateup_warp_tile<TW, TX, ACT, 4>(W, row_g, X, inv, nw, d, d_pad, f_pad, feat0, p.tok + off + t0,
                                         off + t0, min(r, 4), act, red_s[wib], lane);
        t0 += 4;
      } else if (r == 2) {
        gateup_warp_tile<TW, TX, ACT, 2>(W, row_g, X, inv, nw, d, d_pad, f_pad, feat0, p.tok + off + t0,
                                         off + t0, 2, act, red_s[wib], lane);
        t0 += 2;
      } else {
        gateup_warp_tile<TW, TX, ACT, 1>(W, row_g, X, inv, nw, d, d_pad, f_pad, feat0, p.tok + off + t0,
                                         off + t0, 1, act, red_s[wib], lane);
        t0 += 1;
      }
    }
  }
}

template <typename TW, int TB>
__device__ __forceinline__ void down_warp_tile(const TW* __restrict__ W, int row0,
                                               const float* __restrict__ act, int f_pad, int d_pad,
                                               int pos0, int ntok, const float* __restrict__ wpos,
                                               float* __restrict__ opair, float* red, int lane) {
  constexpr int EPC = Chunk<TW>::kElems;
  const int nch = f_pad / EPC;
  float acc[8 * TB];
#pragma unroll
  for (int i = 0; i < 8 * TB; ++i) acc[i] = 0.0f;
  const float* ar[TB];
#pragma unroll
  for (int j = 0; j < TB; ++j) ar[j] = act + (size_t)(pos0 + (j < ntok ? j : 0)) * f_pad;
  const TW* wbase = W + (size_t)row0 * f_pad;
  for (int c = lane; c < nch; c += 32) {
    uint4 wv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) wv[q] = ld_stream(wbase + q * f_pad + c * EPC);
    float af[TB][EPC];
#pragma unroll
    for (int j = 0; j < TB; ++j)
#pragma unroll
      for (int v = 0; v < EPC / 4; ++v) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(ar[j] + c * EPC) + v);
        af[j][4 * v + 0] = x.x;
        af[j][4 * v + 1] = x.y;
        af[j][4 * v + 2] = x.z;
        af[j][4 * v + 3] = x.w;
      }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float wf[EPC];
      unpack<TW>(wv[q], wf);
#pragma unroll
      for (int j = 0; j < TB; ++j)
#pragma unroll
        for (int e = 0; e < EPC; ++e) acc[q * TB + j] = fmaf(wf[e], af[j][e], acc[q * TB + j]);
    }
  }
  warp_reduce_to_smem<8 * TB>(acc, red, lane);
  if (lane < 8 * TB) {
    const int q = lane / TB, j = lane % TB;
    if (j < ntok) opair[(size_t)(pos0 + j) * d_pad + row0 + q] = red[q * TB + j] * wpos[j];
  }
  __syncwarp();
}

template <typename TW>
__global__ void __launch_bounds__(kThreads, 2) down_warp_kernel(const TW* __restrict__ Wd,
                                                                const float* __restrict__ act, int d_pad,
                                                                int f_pad, PlanDev p,
                                                                float* __restrict__ opair) {
  __shared__ float red_s[kWarps][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * kWarps + wib, nwarps = gridDim.x * kWarps;
  griddep_wait();
  const int groups = d_pad / 8;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = gwarp; item < total; item += nwarps) {
    const int a = (int)(item / groups), g = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    const TW* W = Wd + (size_t)e * d_pad * f_pad;
    for (int t0 = 0; t0 < cnt;) {
      const int r = cnt - t0;
      if (r >= 3) {
        down_warp_tile<TW, 4>(W, g * 8, act, f_pad, d_pad, off + t0, min(r, 4), p.w + off + t0, opair,
                              red_s[wib], lane);
        t0 += 4;
      } else if (r == 2) {
        down_warp_tile<TW, 2>(W, g * 8, act, f_pad, d_pad, off + t0, 2, p.w + off + t0, opair, red_s[wib],
                              lane);
        t0 += 2;
      } else {
        down_warp_tile<TW, 1>(W, g * 8, act, f_pad, d_pad, off + t0, 1, p.w + off + t0, opair, red_s[wib],
                              lane);
        t0 += 1;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <typename TW, typename TX>
static void gateup_dispatch(const beam_layer_t& L, const Dims& g, const void* X, const float* inv,
                            const float* nw, const PlanDev& p, float* act, int grid, bool cta,
                            cudaStream_t s) {
  if (cta) {
    if (L.activation == BEAM_ACT_SILU)
      launch_pdl(gateup_cta_kernel<TW, TX, BEAM_ACT_SILU>, grid, kThreads, 0, s, (const TW*)L.w_gu, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
    else
      launch_pdl(gateup_cta_kernel<TW, TX, BEAM_ACT_IDENTITY>, grid, kThreads, 0, s, (const TW*)L.w_gu, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
  } else {
    if (L.activation == BEAM_ACT_SILU)
      launch_pdl(gateup_warp_kernel<TW, TX, BEAM_ACT_SILU>, grid, kThreads, 0, s, (const TW*)L.w_gu, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
    else
      launch_pdl(gateup_warp_kernel<TW, TX, BEAM_ACT_IDENTITY>, grid, kThreads, 0, s, (const TW*)L.w_gu, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
  }
}

// Small batches (few tokens, few active experts) are latency-bound: one CTA per
// item puts every weight byte of the item in flight at once.  Larger batches
// stream with warp items (no CTA barriers).
static bool small_batch(int T) { return T <= 2; }

cudaError_t launch_gateup_simt(const beam_layer_t& L, const Dims& g, const void* X, int x_dtype, int T,
                               const float* inv, const float* nw, const PlanDev& p, float* act,
                               cudaStream_t s) {
  const bool xb = x_dtype == BEAM_BF16;
  const bool cta = small_batch(T);
  const int grid = num_sms() * (cta ? kCtaPerSm : 2);
  if (L.wdtype == BEAM_BF16) {
    if (xb) gateup_dispatch<__nv_bfloat16, __nv_bfloat16>(L, g, X, inv, nw, p, act, grid, cta, s);
    else gateup_dispatch<__nv_bfloat16, float>(L, g, X, inv, nw, p, act, grid, cta, s);
  } else {
    if (xb) gateup_dispatch<float, __nv_bfloat16>(L, g, X, inv, nw, p, act, grid, cta, s);
    else gateup_dispatch<float, float>(L, g, X, inv, nw, p, act, grid, cta, s);
  }
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_down_simt(const beam_layer_t& L, const Dims& g, int T, const PlanDev& p,
                             const float* act, float* opair, cudaStream_t s) {
  const bool cta = small_batch(T);
  const int grid = num_sms() * (cta ? kCtaPerSm : 2);
  if (L.wdtype == BEAM_BF16) {
    if (cta) launch_pdl(down_cta_kernel<__nv_bfloat16>, grid, kThreads, 0, s, (const __nv_bfloat16*)L.w_down, act, g.d_pad, g.f_pad, p, opair);
    else launch_pdl(down_warp_kernel<__nv_bfloat16>, grid, kThreads, 0, s, (const __nv_bfloat16*)L.w_down, act, g.d_pad, g.f_pad, p, opair);
  } else {
    if (cta) launch_pdl(down_cta_kernel<float>, grid, kThreads, 0, s, (const float*)L.w_down, act, g.d_pad, g.f_pad, p, opair);
    else launch_pdl(down_warp_kernel<float>, grid, kThreads, 0, s, (const float*)L.w_down, act, g.d_pad, g.f_pad, p, opair);
  }
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
