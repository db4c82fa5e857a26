// Weighted combine (unpermute): y[t] = sum over t's surviving slots, in ascending
// expert id, of the already ghat-weighted expert rows; then (optionally) the
// residual out = h + y.
//
// Reference order (/root/reference/pkg/src/beamoe/): y starts at zero and
// accumulates experts in ascending id (dispatch/__init__.py:145-156), then the
// shared experts in index order (beam.py:163-164), then out = h + y (beam.py:165).
// Shared experts are planned as ids N..N+S-1, so one ascending pass reproduces it.
// Deterministic: a fixed sequential fp32 sum per element, no atomics.
//
// One warp per (token, 256-column chunk), 8 tokens per CTA, grid.y = column
// chunks (so a 64-token decode step still spreads over 64 CTAs; at prefill sizes
// grid.y shrinks and a warp takes several chunks): the warp ranks
// the token's <= 32 slots by expert id with shuffles (no shared memory, no CTA
// barrier), then each lane sums 8 columns with 16-byte loads of the per-pair
// rows (fp32 on the decode path, bf16 on the prefill path: the sum stays fp32),
// all rows' loads in flight before the ordered adds.
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

constexpr int kCombineWarps = 8;
constexpr int kCombineTargetCtas = 148 * 3 * 4;  // ~4 waves of 3 CTAs per SM (scaled to the SM count)

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  return a | (b << 16);
}

template <typename TP>
__device__ __forceinline__ void ld_pair8(const TP* p, float* v) {
  if constexpr (sizeof(TP) == 2) {
    unpack<__nv_bfloat16>(__ldg(reinterpret_cast<const uint4*>(p)), v);
  } else {
    unpack<float>(__ldg(reinterpret_cast<const uint4*>(p)), v);
    unpack<float>(__ldg(reinterpret_cast<const uint4*>(p) + 1), v + 4);
  }
}

template <typename TH, typename TO, typename TP>
__global__ void __launch_bounds__(32 * kCombineWarps, 3) combine_kernel(const int32_t* __restrict__ slot_expert,
                                                                     const int32_t* __restrict__ slot_pos,
                                                                     const TP* __restrict__ opair, int T, int Keff,
                                                                     int d, int d_pad, const TH* __restrict__ h,
                                                                     TO* __restrict__ out, bool vec, PlanDev chk) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * kCombineWarps + (threadIdx.x >> 5);
  if (t >= T) return;
  // lane k < Keff holds slot k.  Plan positions are laid out by ascending expert
  // (then ascending flat index), and a token meets each expert once, so ascending
  // position == the reference's ascending-expert order: rank = number of surviving
  // slots with a smaller position (no second, dependent load of the slot's expert)
  int pos = -1;
  if (lane < Keff) pos = slot_pos[(size_t)t * Keff + lane];
  BEAM_DCHECK(chk, chk.cap == 0 || pos < chk.cap, kChkSlotPos);
  int rank = 0, nv = 0;
#pragma unroll 4
  for (int j = 0; j < min(Keff, 32); ++j) {
    const int pj = __shfl_sync(0xffffffffu, pos, j);
    nv += pj >= 0;
    rank += pj >= 0 && pos >= 0 && pj < pos;
  }
  // sorted[r] = pos of the slot with rank r (r < nv)
  int sorted_pos = -1;
  for (int j = 0; j < min(Keff, 32); ++j) {
    const int rj = __shfl_sync(0xffffffffu, rank, j);
    const int pj = __shfl_sync(0xffffffffu, pos, j);
    if (pj >= 0 && rj == lane) sorted_pos = pj;
  }
  // a warp walks column chunks blockIdx.y, +gridDim.y, ... with the same slot
  // ranking (one slot_pos round trip for all of them)
  for (int cy = blockIdx.y; cy * 256 < d; cy += gridDim.y) {
    const int c0 = cy * 256 + 8 * lane;
    float y[8], hv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = 0.0f;
    const bool vrow = vec && c0 + 8 <= d;
    if (vrow && h != nullptr) {  // residual row issued before the pair rows (latency overlap)
      const uint4* hp = reinterpret_cast<const uint4*>(h + (size_t)t * d + c0);
      if constexpr (sizeof(TH) == 2) {
        unpack<__nv_bfloat16>(__ldg(hp), hv);
      } else {
        unpack<float>(__ldg(hp), hv);
        unpack<float>(__ldg(hp + 1), hv + 4);
      }
    }
    // rows stay packed in registers until their (ordered) add: 4 regs per bf16
    // row, so 8 rows in flight cost 32 registers, not 64 (occupancy = bytes in
    // flight for this HBM-bound gather)
    constexpr int kRows = sizeof(TP) == 2 ? 8 : 4;
    constexpr int kL = sizeof(TP) == 2 ? 1 : 2;
    for (int r0 = 0; r0 < nv; r0 += kRows) {
      uint4 raw[kRows][kL];
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        const int pr = __shfl_sync(0xffffffffu, sorted_pos, r0 + q < nv ? r0 + q : 0);
        if (r0 + q < nv && c0 < d) {
          const uint4* src = reinterpret_cast<const uint4*>(opair + (size_t)pr * d_pad + c0);
#pragma unroll
          for (int l = 0; l < kL; ++l) raw[q][l] = __ldg(src + l);
        }
      }
#pragma unroll
      for (int q = 0; q < kRows; ++q)
        if (r0 + q < nv) {
          float v[8];
          if constexpr (kL == 1) {
            unpack<__nv_bfloat16>(raw[q][0], v);
          } else {
            unpack<float>(raw[q][0], v);
            unpack<float>(raw[q][1], v + 4);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) y[i] += v[i];
        }
    }
    if (vrow) {
      // 16-byte row loads / stores (d % 8 == 0 and 16-byte aligned rows)
      if (h != nullptr) {
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = hv[i] + y[i];
      }
      uint4* op = reinterpret_cast<uint4*>(out + (size_t)t * d + c0);
      if constexpr (sizeof(TO) == 2) {
        uint4 o;
        o.x = pack_bf16x2(y[0], y[1]);
        o.y = pack_bf16x2(y[2], y[3]);
        o.z = pack_bf16x2(y[4], y[5]);
        o.w = pack_bf16x2(y[6], y[7]);
        *op = o;
      } else {
        op[0] = make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]), __float_as_uint(y[3]));
        op[1] = make_uint4(__float_as_uint(y[4]), __float_as_uint(y[5]), __float_as_uint(y[6]), __float_as_uint(y[7]));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = c0 + i;
        if (c < d) {
          float o = y[i];
          if (h != nullptr) o = to_f32<TH>(h[(size_t)t * d + c]) + o;
          out[(size_t)t * d + c] = from_f32<TO>(o);
        }
      }
    }
  }
}

template <typename TP>
static cudaError_t combine_dispatch(const PlanDev& p, const TP* opair, int T, int Keff, int d, int d_pad,
                                    const void* h, int h_dtype, void* out, int out_dtype, cudaStream_t s) {
  const bool vec = d % 8 == 0 && (reinterpret_cast<uintptr_t>(h) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const int chunks = ceil_div(d, 256);
  // enough chunk columns for ~4 waves of 3 CTAs per SM, no more: every extra
  // column repeats the slot ranking and its dependent slot_pos load
  // (T = 8192, d = 2048: 2 columns of 4 chunks, combine 77 -> 59 us)
  const int tiles = ceil_div(T, kCombineWarps);
  const int gy = std::max(1, std::min(chunks, ceil_div(kCombineTargetCtas * num_sms() / 148, tiles)));
  const dim3 grid(tiles, gy);
  const int thr = 32 * kCombineWarps;
  if (out_dtype == BEAM_F32 && h_dtype == BEAM_F32)
    return launch_pdl(combine_kernel<float, float, TP>, grid, thr, 0, s, p.slot_expert, p.slot_pos, opair, T, Keff, d, d_pad, (const float*)h, (float*)out, vec, p);
  if (out_dtype == BEAM_BF16 && h_dtype == BEAM_BF16)
    return launch_pdl(combine_kernel<__nv_bfloat16, __nv_bfloat16, TP>, grid, thr, 0, s, p.slot_expert, p.slot_pos, opair, T, Keff, d, d_pad, (const __nv_bfloat16*)h, (__nv_bfloat16*)out, vec, p);
  if (out_dtype == BEAM_F32)
    return launch_pdl(combine_kernel<__nv_bfloat16, float, TP>, grid, thr, 0, s, p.slot_expert, p.slot_pos, opair, T, Keff, d, d_pad, (const __nv_bfloat16*)h, (float*)out, vec, p);
  return launch_pdl(combine_kernel<float, __nv_bfloat16, TP>, grid, thr, 0, s, p.slot_expert, p.slot_pos, opair, T, Keff, d, d_pad, (const float*)h, (__nv_bfloat16*)out, vec, p);
}

cudaError_t launch_combine(const PlanDev& p, const void* opair, int opair_dtype, int T, int Keff, int d, int d_pad,
                           const void* h, int h_dtype, void* out, int out_dtype, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (Keff > 32) return cudaErrorInvalidValue;  // one lane per slot
  cudaError_t e = opair_dtype == BEAM_BF16
                      ? combine_dispatch(p, (const __nv_bfloat16*)opair, T, Keff, d, d_pad, h, h_dtype, out, out_dtype, s)
                      : combine_dispatch(p, (const float*)opair, T, Keff, d, d_pad, h, h_dtype, out, out_dtype, s);
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace beam
