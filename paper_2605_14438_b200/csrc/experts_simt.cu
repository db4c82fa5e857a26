// Weight-streaming grouped SwiGLU experts (decode / fp32 path).
//
// Reference: dispatch.grouped_execute (/root/reference/pkg/src/beamoe/dispatch/
// __init__.py:129-157) running expert_forward_np (moe.py:96-100)
//     O_e = (act(X_e W_gate) * (X_e W_up)) W_down,   y[rows] += O_e * ghat
// over the surviving slots of every expert, ascending expert id.
//
// B200 design (HBM-bound regime: few tokens per expert).  Only experts that the
// mask left active are touched: work items are (active expert, row group) pairs
// enumerated on the device from the permute kernel's active list, so no host
// sync and no bytes for masked experts.  Each warp streams a group of weight
// rows with 16-byte L1-bypassing loads and applies them to all of the expert's
// tokens (up to 4 per pass) held in registers; partial dot products are
// combined with a transpose-reduce butterfly.  Two launches:
//   gateup: 4 gate + 4 up rows per item -> act[pos, f] = act(g) * u   (fp32)
//   down:   8 output rows per item      -> opair[pos, d] = ghat * (act . W_down)
// Accumulation order is fixed by the code (lane-strided k, then butterfly),
// never by scheduling, so results are deterministic.
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

template <typename TW, int ACT, int TB>
__device__ __forceinline__ void gateup_tile(const TW* __restrict__ W, int row_g,
                                            const TW* __restrict__ X, int d_pad, int f_pad,
                                            int feat0, const int32_t* __restrict__ tokp, int pos0,
                                            int ntok, float* __restrict__ act, float* red,
                                            int lane) {
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
    for (int j = 0; j < TB; ++j) unpack<TW>(ld_cached(X + (size_t)tk[j] * d_pad + c * EPC), xf[j]);
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
  warp_reduce_to_smem<8 * TB>(acc, red, lane);
  if (lane < 4 * TB) {
    const int p = lane / TB, j = lane % TB;
    if (j < ntok) {
      const float g = red[p * TB + j], u = red[(4 + p) * TB + j];
      act[(size_t)(pos0 + j) * f_pad + feat0 + p] = activation<ACT>(g) * u;
    }
  }
  __syncwarp();
}

template <typename TW, int ACT>
__global__ void __launch_bounds__(256, 2) gateup_kernel(const TW* __restrict__ Wgu,
                                                        const TW* __restrict__ X, int d_pad,
                                                        int f_pad, PlanDev p,
                                                        float* __restrict__ act) {
  __shared__ float red_s[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * 8 + wib, nwarps = gridDim.x * 8;
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
        gateup_tile<TW, ACT, 4>(W, row_g, X, d_pad, f_pad, feat0, p.tok + off + t0, off + t0,
                                min(r, 4), act, red_s[wib], lane);
        t0 += 4;
      } else if (r == 2) {
        gateup_tile<TW, ACT, 2>(W, row_g, X, d_pad, f_pad, feat0, p.tok + off + t0, off + t0, 2,
                                act, red_s[wib], lane);
        t0 += 2;
      } else {
        gateup_tile<TW, ACT, 1>(W, row_g, X, d_pad, f_pad, feat0, p.tok + off + t0, off + t0, 1,
                                act, red_s[wib], lane);
        t0 += 1;
      }
    }
  }
}

template <typename TW, int TB>
__device__ __forceinline__ void down_tile(const TW* __restrict__ W, int row0,
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
__global__ void __launch_bounds__(256, 2) down_kernel(const TW* __restrict__ Wd,
                                                      const float* __restrict__ act, int d_pad,
                                                      int f_pad, PlanDev p,
                                                      float* __restrict__ opair) {
  __shared__ float red_s[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * 8 + wib, nwarps = gridDim.x * 8;
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
        down_tile<TW, 4>(W, g * 8, act, f_pad, d_pad, off + t0, min(r, 4), p.w + off + t0, opair,
                         red_s[wib], lane);
        t0 += 4;
      } else if (r == 2) {
        down_tile<TW, 2>(W, g * 8, act, f_pad, d_pad, off + t0, 2, p.w + off + t0, opair,
                         red_s[wib], lane);
        t0 += 2;
      } else {
        down_tile<TW, 1>(W, g * 8, act, f_pad, d_pad, off + t0, 1, p.w + off + t0, opair,
                         red_s[wib], lane);
        t0 += 1;
      }
    }
  }
}

cudaError_t launch_gateup_simt(const beam_layer_t& L, const Dims& g, const void* xact,
                               const PlanDev& p, float* act, cudaStream_t s) {
  const int grid = num_sms() * 2;
  if (L.wdtype == BEAM_BF16) {
    using TW = __nv_bfloat16;
    if (L.activation == BEAM_ACT_SILU)
      gateup_kernel<TW, BEAM_ACT_SILU><<<grid, 256, 0, s>>>((const TW*)L.w_gu, (const TW*)xact, g.d_pad, g.f_pad, p, act);
    else
      gateup_kernel<TW, BEAM_ACT_IDENTITY><<<grid, 256, 0, s>>>((const TW*)L.w_gu, (const TW*)xact, g.d_pad, g.f_pad, p, act);
  } else {
    using TW = float;
    if (L.activation == BEAM_ACT_SILU)
      gateup_kernel<TW, BEAM_ACT_SILU><<<grid, 256, 0, s>>>((const TW*)L.w_gu, (const TW*)xact, g.d_pad, g.f_pad, p, act);
    else
      gateup_kernel<TW, BEAM_ACT_IDENTITY><<<grid, 256, 0, s>>>((const TW*)L.w_gu, (const TW*)xact, g.d_pad, g.f_pad, p, act);
  }
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_down_simt(const beam_layer_t& L, const Dims& g, const PlanDev& p,
                             const float* act, float* opair, cudaStream_t s) {
  const int grid = num_sms() * 2;
  if (L.wdtype == BEAM_BF16)
    down_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)L.w_down, act, g.d_pad, g.f_pad, p, opair);
  else
    down_kernel<float><<<grid, 256, 0, s>>>((const float*)L.w_down, act, g.d_pad, g.f_pad, p, opair);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
