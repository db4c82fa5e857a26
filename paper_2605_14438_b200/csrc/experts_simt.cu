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
// (deterministic, independent of the grid).  Two stages:
//   gateup: 4 gate + 4 up rows per item -> act[pos, f] = act(g) * u   (fp32)
//   down:   2 x 8 output rows per item  -> opair[pos, d] = ghat * (act . W_down)
#include <cstdlib>
#include <type_traits>

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

// Checked build: an item's plan run [off, off + cnt) lies inside the plan and
// its token indices inside [0, T) (lane 0 of the first item of each expert).
__device__ __forceinline__ void check_item(const PlanDev& p, int off, int cnt, bool first) {
#ifdef BEAM_DEVICE_CHECKS
  if (p.check == nullptr || !first) return;
  BEAM_DCHECK(p, p.cap == 0 || (off >= 0 && off + cnt <= p.cap), kChkPlanPos);
  if (p.T > 0)
    for (int q = 0; q < cnt; ++q) {
      const int t = p.tok[off + q];
      BEAM_DCHECK(p, t >= 0 && t < p.T, kChkToken);
    }
#endif
}

// ---------------------------------------------------------------------------
// gate / up
// ---------------------------------------------------------------------------
template <typename TW, typename TX, int ACT, int TB>
__device__ __forceinline__ void gateup_cta_tile(const TW* __restrict__ W, int row_g,
                                            const TX* __restrict__ X, const float* __restrict__ inv,
                                            const float* __restrict__ nw, int d, int d_pad, int f_pad,
                                            int feat0, const int32_t* __restrict__ tokp, int pos0,
                                            int ntok, TW* __restrict__ act, float* part,
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
      act[(size_t)(pos0 + j) * f_pad + feat0 + p] = from_f32<TW>(activation<ACT>(gs) * u);
    }
  }
}

template <typename TW, typename TX, int ACT>
__global__ void __launch_bounds__(kThreads, kCtaPerSm) gateup_cta_kernel(const TW* __restrict__ Wgu,
                                                             const TX* __restrict__ X,
                                                             const float* __restrict__ inv,
                                                             const float* __restrict__ nw, int d,
                                                             int d_pad, int f_pad, PlanDev p,
                                                             TW* __restrict__ act) {
  __shared__ float part[kWarps * 32];
  __shared__ float red[32];
  griddep_wait();
  const int groups = f_pad / 4;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = blockIdx.x; item < total; item += gridDim.x) {
    const int a = (int)(item / groups), g = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    if (threadIdx.x == 0) check_item(p, off, cnt, g == 0);
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
                                          const TW* __restrict__ act, int f_pad, int d_pad,
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
  const TW* ar[TB];
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
      for (int j = 0; j < TB; ++j) load_x<TW, EPC>(ar[j] + c * EPC, af[j]);  // act rows in the weights' dtype
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
                                                           const TW* __restrict__ act, int d_pad,
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
    if (threadIdx.x == 0) check_item(p, off, cnt, g == 0);
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
                                                 int ntok, TW* __restrict__ act, float* red, int lane) {
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
      act[(size_t)(pos0 + j) * f_pad + feat0 + p] = from_f32<TW>(activation<ACT>(gs) * u);
    }
  }
  __syncwarp();
}

template <typename TW, typename TX, int ACT>
__device__ __forceinline__ void gateup_warp_items(const TW* __restrict__ Wgu, const TX* __restrict__ X,
                                                  const float* __restrict__ inv, const float* __restrict__ nw,
                                                  int d, int d_pad, int f_pad, PlanDev p,
                                                  TW* __restrict__ act, float (*red_s)[32]) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * kWarps + wib, nwarps = gridDim.x * kWarps;
  const int groups = f_pad / 4;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = gwarp; item < total; item += nwarps) {
    const int a = (int)(item / groups), g = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    if (lane == 0) check_item(p, off, cnt, g == 0);
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

template <typename TW, typename TX, int ACT>
__global__ void __launch_bounds__(kThreads, 2) gateup_warp_kernel(const TW* __restrict__ Wgu,
                                                                  const TX* __restrict__ X,
                                                                  const float* __restrict__ inv,
                                                                  const float* __restrict__ nw, int d,
                                                                  int d_pad, int f_pad, PlanDev p,
                                                                  TW* __restrict__ act) {
  __shared__ float red_s[kWarps][32];
  griddep_wait();
  gateup_warp_items<TW, TX, ACT>(Wgu, X, inv, nw, d, d_pad, f_pad, p, act, red_s);
}

template <typename TW, int TB>
__device__ __forceinline__ void down_warp_tile(const TW* __restrict__ W, int row0,
                                               const TW* __restrict__ act, int f_pad, int d_pad,
                                               int pos0, int ntok, const float* __restrict__ wpos,
                                               float* __restrict__ opair, float* red, int lane) {
  constexpr int EPC = Chunk<TW>::kElems;
  const int nch = f_pad / EPC;
  float acc[8 * TB];
#pragma unroll
  for (int i = 0; i < 8 * TB; ++i) acc[i] = 0.0f;
  const TW* ar[TB];
#pragma unroll
  for (int j = 0; j < TB; ++j) ar[j] = act + (size_t)(pos0 + (j < ntok ? j : 0)) * f_pad;
  const TW* wbase = W + (size_t)row0 * f_pad;
  for (int c = lane; c < nch; c += 32) {
    uint4 wv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) wv[q] = ld_stream(wbase + q * f_pad + c * EPC);
    float af[TB][EPC];
#pragma unroll
    for (int j = 0; j < TB; ++j) load_x<TW, EPC>(ar[j] + c * EPC, af[j]);
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
__device__ __forceinline__ void down_warp_items(const TW* __restrict__ Wd, const TW* __restrict__ act, int d_pad,
                                                int f_pad, PlanDev p, float* __restrict__ opair,
                                                float (*red_s)[32]) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * kWarps + wib, nwarps = gridDim.x * kWarps;
  const int groups = d_pad / 8;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = gwarp; item < total; item += nwarps) {
    const int a = (int)(item / groups), g = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    if (lane == 0) check_item(p, off, cnt, g == 0);
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

template <typename TW>
__global__ void __launch_bounds__(kThreads, 2) down_warp_kernel(const TW* __restrict__ Wd,
                                                                const TW* __restrict__ act, int d_pad,
                                                                int f_pad, PlanDev p,
                                                                float* __restrict__ opair) {
  __shared__ float red_s[kWarps][32];
  griddep_wait();
  down_warp_items<TW>(Wd, act, d_pad, f_pad, p, opair, red_s);
}

// ---------------------------------------------------------------------------
// tensor-core warp-item kernels (bf16 weights, no in-kernel norm multiply; T > 2):
// the same weight stream, but the multiply-adds run on mma.sync m16n8k16 (one
// instruction per 16 x 8 x 16 MACs instead of FFMA2s + bf16 unpacking), so a
// warp spends its issue slots on loads.  A warp item is 16 weight rows (8 gate +
// 8 up rows of 8 features, or 16 down rows) x up to 8 tokens per pass.  Each
// lane streams 16 contiguous bytes of two rows per 32-k step straight into its
// A fragment: the k order inside a step is permuted identically for A and B,
// which a dot product does not see.  fp32 token operands are split x = hi + lo
// into two bf16 terms (two MMAs, ~16 significant bits), so the result keeps the
// FFMA kernels' accuracy; bf16 tokens are exact in one term.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// (x0, x1) -> bf16 pairs hi and lo with x ~= hi + lo
__device__ __forceinline__ void split_pair(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  hi = bf16x2(x0, x1);
  lo = bf16x2(x0 - __uint_as_float(hi << 16), x1 - __uint_as_float(hi & 0xffff0000u));
}

// B operand of one 32-k step: this lane's 8 k values of its token row, as 4
// bf16 pairs (hi) and, for fp32 rows, 4 residual pairs (lo)
template <typename TX>
struct BStep {
  uint32_t hi[4], lo[4];
};
template <typename TX>
__device__ __forceinline__ void load_bstep(const TX* p, bool ok, BStep<TX>& b) {
  if constexpr (sizeof(TX) == 2) {
    const uint4 v = ok ? ld_cached(p) : make_uint4(0u, 0u, 0u, 0u);
    b.hi[0] = v.x; b.hi[1] = v.y; b.hi[2] = v.z; b.hi[3] = v.w;
  } else {
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f), v = u;
    if (ok) {
      u = __ldg(reinterpret_cast<const float4*>(p));
      v = __ldg(reinterpret_cast<const float4*>(p) + 1);
    }
    split_pair(u.x, u.y, b.hi[0], b.lo[0]);
    split_pair(u.z, u.w, b.hi[1], b.lo[1]);
    split_pair(v.x, v.y, b.hi[2], b.lo[2]);
    split_pair(v.z, v.w, b.hi[3], b.lo[3]);
  }
}
// c += A(rows r0 | r1, this step) * B: two k16 MMAs per step (x2 for hi + lo)
template <typename TX>
__device__ __forceinline__ void mma_step(float (&c)[4], const uint4& w0, const uint4& w1, const BStep<TX>& b) {
  mma_bf16_16816(c, w0.x, w1.x, w0.y, w1.y, b.hi[0], b.hi[1]);
  mma_bf16_16816(c, w0.z, w1.z, w0.w, w1.w, b.hi[2], b.hi[3]);
  if constexpr (sizeof(TX) == 4) {
    mma_bf16_16816(c, w0.x, w1.x, w0.y, w1.y, b.lo[0], b.lo[1]);
    mma_bf16_16816(c, w0.z, w1.z, w0.w, w1.w, b.lo[2], b.lo[3]);
  }
}

constexpr int kMmaUnroll = 4;  // 32-k steps in flight per lane (4 x 32 B of weights); mma_rows sums 4 accumulators

// rows r0 (lanes' group g) and r1 = r0 + gap of W [*, K] against the token rows
// xrow (this lane's B token), over K in 32-element steps
template <typename TX>
__device__ __forceinline__ void mma_rows(const __nv_bfloat16* __restrict__ w0p, const __nv_bfloat16* __restrict__ w1p,
                                         const TX* __restrict__ xrow, int K, int q, float (&c)[4]) {
  const int steps = (K + 31) / 32;
  // one accumulator per unrolled step: the MMAs of a step do not wait on the
  // previous step's (fixed final summation order: deterministic)
  float cu[kMmaUnroll][4];
#pragma unroll
  for (int u = 0; u < kMmaUnroll; ++u) cu[u][0] = cu[u][1] = cu[u][2] = cu[u][3] = 0.0f;
  for (int s0 = 0; s0 < steps; s0 += kMmaUnroll) {
    uint4 a0[kMmaUnroll], a1[kMmaUnroll];
    BStep<TX> b[kMmaUnroll];
#pragma unroll
    for (int u = 0; u < kMmaUnroll; ++u) {
      const int k = (s0 + u) * 32 + q * 8;
      const bool ok = s0 + u < steps && k < K;
      a0[u] = ok ? ld_stream(w0p + k) : make_uint4(0u, 0u, 0u, 0u);
      a1[u] = ok ? ld_stream(w1p + k) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kMmaUnroll; ++u) {
      const int k = (s0 + u) * 32 + q * 8;
      load_bstep<TX>(xrow + k, s0 + u < steps && k < K, b[u]);
    }
#pragma unroll
    for (int u = 0; u < kMmaUnroll; ++u) mma_step<TX>(cu[u], a0[u], a1[u], b[u]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (cu[0][i] + cu[1][i]) + (cu[2][i] + cu[3][i]);
}

template <typename TX, int ACT>
__device__ __forceinline__ void gateup_mma_items(const __nv_bfloat16* __restrict__ Wgu, const TX* __restrict__ X,
                                                 const float* __restrict__ inv, int d_pad, int f_pad,
                                                 PlanDev p, __nv_bfloat16* __restrict__ act) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5), nwarps = gridDim.x * kWarps;
  const int groups = f_pad / 8;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = gwarp; item < total; item += nwarps) {
    const int a = (int)(item / groups), gi = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    if (lane == 0) check_item(p, off, cnt, gi == 0);
    const int feat0 = gi * 8;
    // packed W_gu: per 16 features, 16 gate rows then 16 up rows
    const int rg = (feat0 >> 4) * 32 + (feat0 & 15) + g;
    const __nv_bfloat16* W = Wgu + (size_t)e * 2 * f_pad * d_pad;
    for (int t0 = 0; t0 < cnt; t0 += 8) {
      const int nt = min(8, cnt - t0);
      const int* tokp = p.tok + off + t0;
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      mma_rows<TX>(W + (size_t)rg * d_pad, W + (size_t)(rg + 16) * d_pad, X + (size_t)tokp[g < nt ? g : 0] * d_pad,
                   d_pad, q, c);
      // c[0], c[1]: gate of feature feat0 + g for tokens 2q, 2q + 1; c[2], c[3]: up
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = 2 * q + j;
        if (n < nt) {
          const float s = inv ? inv[tokp[n]] : 1.0f;
          act[(size_t)(off + t0 + n) * f_pad + feat0 + g] = __float2bfloat16_rn(activation<ACT>(c[j] * s) * (c[2 + j] * s));
        }
      }
    }
  }
}

__device__ __forceinline__ void down_mma_items(const __nv_bfloat16* __restrict__ Wd, const __nv_bfloat16* __restrict__ act,
                                               int d_pad, int f_pad, PlanDev p, float* __restrict__ opair) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5), nwarps = gridDim.x * kWarps;
  const int groups = (d_pad + 15) / 16;
  const long long total = (long long)p.meta[0] * groups;
  for (long long item = gwarp; item < total; item += nwarps) {
    const int a = (int)(item / groups), gi = (int)(item % groups);
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    if (lane == 0) check_item(p, off, cnt, gi == 0);
    const int r0 = gi * 16 + g, r1 = r0 + 8;
    const __nv_bfloat16* W = Wd + (size_t)e * d_pad * f_pad;
    // rows past d_pad (d_pad % 16 == 8) read row d_pad - 1 and are not stored
    const __nv_bfloat16* w0p = W + (size_t)min(r0, d_pad - 1) * f_pad;
    const __nv_bfloat16* w1p = W + (size_t)min(r1, d_pad - 1) * f_pad;
    for (int t0 = 0; t0 < cnt; t0 += 8) {
      const int nt = min(8, cnt - t0);
      const int pos0 = off + t0;
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      // bf16 act rows: one k16 MMA pair per step (no hi / lo split)
      mma_rows<__nv_bfloat16>(w0p, w1p, act + (size_t)(pos0 + (g < nt ? g : 0)) * f_pad, f_pad, q, c);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = 2 * q + j;
        if (n < nt) {
          const float wn = p.w[pos0 + n];
          if (r0 < d_pad) opair[(size_t)(pos0 + n) * d_pad + r0] = c[j] * wn;
          if (r1 < d_pad) opair[(size_t)(pos0 + n) * d_pad + r1] = c[2 + j] * wn;
        }
      }
    }
  }
}

// Which item kernel runs is decided on the device from the plan: the MMA items
// (16 rows x 8 tokens) pay off once experts carry enough surviving tokens on
// average (R >= tok * E_act) and there are enough of them to give every warp >= 3
// (they are 2x larger than the FFMA items, which otherwise keep more warps and
// weight bytes in flight).  Q30 sweep on B200: T=64 s=0 347 -> 275 us, T=64
// s=0.25 281 -> 251 us; T=16 s=0.25 (58 experts) 132 us FFMA vs 137 us MMA.
__device__ __forceinline__ bool use_mma_items(const PlanDev& p, int items_per_expert, int tok_per_expert) {
  const int e_act = p.meta[0];
  return p.meta[2] >= tok_per_expert * e_act && (long long)e_act * items_per_expert >= 3LL * gridDim.x * kWarps;
}
// tokens per active expert from which the MMA items win.  With bf16 operands on
// both sides (one MMA pair per 32-k step) gate/up items win from 2 tokens per
// expert (profiles/r02/mma_tok_ab.txt, Q30: T=32 s=0 241.2 -> 221.4 us, T=64
// s=0.5 221.6 -> 215.2 us; 1 loses at T=16); down items from 2.
constexpr int kMmaTokGateUp = 2, kMmaTokDown = 2;
// (BEAM_MMA_TOK_GU / BEAM_MMA_TOK_DN override the two thresholds: tuning runs)
static int mma_tok(int which) {
  static const int v[2] = {[] { const char* e = getenv("BEAM_MMA_TOK_GU"); return e ? atoi(e) : kMmaTokGateUp; }(),
                           [] { const char* e = getenv("BEAM_MMA_TOK_DN"); return e ? atoi(e) : kMmaTokDown; }()};
  return v[which];
}

// FFMA-only launch: the host picks it when T * Keff rules the tensor-core items
// out (mma_possible); otherwise the one-launch mix kernels below run, and the
// device picks the item kind from the plan.
template <typename TX, int ACT>
__global__ void __launch_bounds__(kThreads, 2) gateup_ffma_kernel(const __nv_bfloat16* __restrict__ Wgu,
                                                                  const TX* __restrict__ X,
                                                                  const float* __restrict__ inv,
                                                                  const float* __restrict__ nw, int d,
                                                                  int d_pad, int f_pad, PlanDev p,
                                                                  __nv_bfloat16* __restrict__ act, int tok) {
  // nw is always null here; a runtime argument keeps the register allocation of
  // gateup_warp_kernel (a literal null makes ptxas spill)
  __shared__ float red_s[kWarps][32];
  griddep_wait();
  if (!use_mma_items(p, f_pad / 8, tok))
    gateup_warp_items<__nv_bfloat16, TX, ACT>(Wgu, X, inv, nw, d, d_pad, f_pad, p, act, red_s);
}

// One launch for both item kinds (the device picks from the plan): the FFMA body
// is a separate, non-inlined function so the kernel's register allocation is the
// larger body's, not their sum (inlined together they spill); the tensor-core
// body stays inline (as a call it lost 4-8 %).
template <typename TX, int ACT>
__device__ __forceinline__ void gateup_mma_body(const __nv_bfloat16* __restrict__ Wgu, const TX* __restrict__ X,
                                             const float* __restrict__ inv, int d_pad, int f_pad, PlanDev p,
                                             __nv_bfloat16* __restrict__ act) {
  gateup_mma_items<TX, ACT>(Wgu, X, inv, d_pad, f_pad, p, act);
}
template <typename TX, int ACT>
__device__ __noinline__ void gateup_ffma_body(const __nv_bfloat16* __restrict__ Wgu, const TX* __restrict__ X,
                                              const float* __restrict__ inv, const float* __restrict__ nw, int d,
                                              int d_pad, int f_pad, PlanDev p, __nv_bfloat16* __restrict__ act) {
  __shared__ float red_s[kWarps][32];
  gateup_warp_items<__nv_bfloat16, TX, ACT>(Wgu, X, inv, nw, d, d_pad, f_pad, p, act, red_s);
}
template <typename TXM, typename TXF, int ACT>
__global__ void __launch_bounds__(kThreads, 2) gateup_mix_kernel(const __nv_bfloat16* __restrict__ Wgu,
                                                                 const TXM* __restrict__ Xm,
                                                                 const TXF* __restrict__ Xf,
                                                                 const float* __restrict__ inv,
                                                                 const float* __restrict__ nw, int d, int d_pad,
                                                                 int f_pad, PlanDev p,
                                                                 __nv_bfloat16* __restrict__ act, int tok) {
  griddep_wait();
  if (use_mma_items(p, f_pad / 8, tok)) gateup_mma_body<TXM, ACT>(Wgu, Xm, inv, d_pad, f_pad, p, act);
  else gateup_ffma_body<TXF, ACT>(Wgu, Xf, inv, nw, d, d_pad, f_pad, p, act);
}

__device__ __forceinline__ void down_mma_body(const __nv_bfloat16* __restrict__ Wd, const __nv_bfloat16* __restrict__ act,
                                           int d_pad, int f_pad, PlanDev p, float* __restrict__ opair) {
  down_mma_items(Wd, act, d_pad, f_pad, p, opair);
}
__device__ __noinline__ void down_ffma_body(const __nv_bfloat16* __restrict__ Wd, const __nv_bfloat16* __restrict__ act,
                                            int d_pad, int f_pad, PlanDev p, float* __restrict__ opair) {
  __shared__ float red_s[kWarps][32];
  down_warp_items<__nv_bfloat16>(Wd, act, d_pad, f_pad, p, opair, red_s);
}
__global__ void __launch_bounds__(kThreads, 2) down_mix_kernel(const __nv_bfloat16* __restrict__ Wd,
                                                               const __nv_bfloat16* __restrict__ act, int d_pad,
                                                               int f_pad, PlanDev p, float* __restrict__ opair, int tok) {
  griddep_wait();
  if (use_mma_items(p, (d_pad + 15) / 16, tok)) down_mma_body(Wd, act, d_pad, f_pad, p, opair);
  else down_ffma_body(Wd, act, d_pad, f_pad, p, opair);
}

__global__ void __launch_bounds__(kThreads, 2) down_ffma_kernel(const __nv_bfloat16* __restrict__ Wd,
                                                                const __nv_bfloat16* __restrict__ act, int d_pad,
                                                                int f_pad, PlanDev p, float* __restrict__ opair, int tok) {
  __shared__ float red_s[kWarps][32];
  griddep_wait();
  if (!use_mma_items(p, (d_pad + 15) / 16, tok)) down_warp_items<__nv_bfloat16>(Wd, act, d_pad, f_pad, p, opair, red_s);
}

// Host side of use_mma_items: E_act * items >= 3 * warps needs E_act >= e_min,
// and R >= tok * E_act needs T * Keff >= R >= tok * e_min.
static bool mma_possible(long long slots, int items_per_expert, int tok_per_expert, int grid) {
  if (slots < 0) return true;  // unknown slot count: let the device decide
  const long long e_min = (3LL * grid * kWarps + items_per_expert - 1) / items_per_expert;
  return slots >= tok_per_expert * e_min;
}

// mma kernels: bf16 weights, token rows without a pending norm multiply
// (BEAM_DECODE_MMA=0 keeps the FFMA kernels)
static bool mma_enabled() {
  static const int v = [] {
    const char* e = getenv("BEAM_DECODE_MMA");
    return e == nullptr ? 1 : atoi(e);
  }();
  return v != 0;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <typename TW, typename TX>
static void gateup_dispatch(const beam_layer_t& L, const Dims& g, const void* X, const float* inv,
                            const float* nw, const PlanDev& p, void* act_v, int grid, bool cta,
                            long long slots, cudaStream_t s, const void* X16) {
  TW* act = static_cast<TW*>(act_v);  // act rows in the weights' dtype
  if (cta) {
    if (L.activation == BEAM_ACT_SILU)
      launch_pdl(gateup_cta_kernel<TW, TX, BEAM_ACT_SILU>, grid, kThreads, 0, s, (const TW*)L.w_gu, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
    else
      launch_pdl(gateup_cta_kernel<TW, TX, BEAM_ACT_IDENTITY>, grid, kThreads, 0, s, (const TW*)L.w_gu, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
  } else if (std::is_same<TW, __nv_bfloat16>::value && nw == nullptr && mma_enabled()) {
    if constexpr (std::is_same<TW, __nv_bfloat16>::value) {  // bf16 act rows
      const __nv_bfloat16* W = (const __nv_bfloat16*)L.w_gu;
      const int tok = mma_tok(0);
      const bool mma = mma_possible(slots, g.f_pad / 8, tok, grid);
      // tensor-core items read the bf16 copy of the rows when there is one
      // (one MMA pair per step instead of the fp32 hi + lo pairs)
      const bool b16 = X16 != nullptr;
      if (!mma) {  // the tensor-core items are ruled out from the slot count
        if (L.activation == BEAM_ACT_SILU)
          launch_pdl(gateup_ffma_kernel<TX, BEAM_ACT_SILU>, grid, kThreads, 0, s, W, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act, tok);
        else
          launch_pdl(gateup_ffma_kernel<TX, BEAM_ACT_IDENTITY>, grid, kThreads, 0, s, W, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act, tok);
      } else if (b16) {  // one launch, item kind picked on the device
        if (L.activation == BEAM_ACT_SILU)
          launch_pdl(gateup_mix_kernel<__nv_bfloat16, TX, BEAM_ACT_SILU>, grid, kThreads, 0, s, W, (const __nv_bfloat16*)X16, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act, tok);
        else
          launch_pdl(gateup_mix_kernel<__nv_bfloat16, TX, BEAM_ACT_IDENTITY>, grid, kThreads, 0, s, W, (const __nv_bfloat16*)X16, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act, tok);
      } else {
        if (L.activation == BEAM_ACT_SILU)
          launch_pdl(gateup_mix_kernel<TX, TX, BEAM_ACT_SILU>, grid, kThreads, 0, s, W, (const TX*)X, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act, tok);
        else
          launch_pdl(gateup_mix_kernel<TX, TX, BEAM_ACT_IDENTITY>, grid, kThreads, 0, s, W, (const TX*)X, (const TX*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act, tok);
      }
    }
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
                               const float* inv, const float* nw, const PlanDev& p, void* act,
                               cudaStream_t s, long long slots, const void* X16) {
  const bool xb = x_dtype == BEAM_BF16;
  const bool cta = small_batch(T);
  const int grid = num_sms() * (cta ? kCtaPerSm : 2);
  if (L.wdtype == BEAM_BF16) {
    if (xb) gateup_dispatch<__nv_bfloat16, __nv_bfloat16>(L, g, X, inv, nw, p, act, grid, cta, slots, s, X16);
    else gateup_dispatch<__nv_bfloat16, float>(L, g, X, inv, nw, p, act, grid, cta, slots, s, X16);
  } else {
    if (xb) gateup_dispatch<float, __nv_bfloat16>(L, g, X, inv, nw, p, act, grid, cta, slots, s, nullptr);
    else gateup_dispatch<float, float>(L, g, X, inv, nw, p, act, grid, cta, slots, s, nullptr);
  }
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_down_simt(const beam_layer_t& L, const Dims& g, int T, const PlanDev& p,
                             const void* act, float* opair, cudaStream_t s, long long slots) {
  const bool cta = small_batch(T);
  const int grid = num_sms() * (cta ? kCtaPerSm : 2);
  if (L.wdtype == BEAM_BF16) {
    if (cta) launch_pdl(down_cta_kernel<__nv_bfloat16>, grid, kThreads, 0, s, (const __nv_bfloat16*)L.w_down, (const __nv_bfloat16*)act, g.d_pad, g.f_pad, p, opair);
    else if (mma_enabled()) {
      const int tok = mma_tok(1);
      const bool mma = mma_possible(slots, (g.d_pad + 15) / 16, tok, grid);
      if (mma) launch_pdl(down_mix_kernel, grid, kThreads, 0, s, (const __nv_bfloat16*)L.w_down, (const __nv_bfloat16*)act, g.d_pad, g.f_pad, p, opair, tok);
      else launch_pdl(down_ffma_kernel, grid, kThreads, 0, s, (const __nv_bfloat16*)L.w_down, (const __nv_bfloat16*)act, g.d_pad, g.f_pad, p, opair, tok);
    }
    else launch_pdl(down_warp_kernel<__nv_bfloat16>, grid, kThreads, 0, s, (const __nv_bfloat16*)L.w_down, (const __nv_bfloat16*)act, g.d_pad, g.f_pad, p, opair);
  } else {
    if (cta) launch_pdl(down_cta_kernel<float>, grid, kThreads, 0, s, (const float*)L.w_down, (const float*)act, g.d_pad, g.f_pad, p, opair);
    else launch_pdl(down_warp_kernel<float>, grid, kThreads, 0, s, (const float*)L.w_down, (const float*)act, g.d_pad, g.f_pad, p, opair);
  }
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
