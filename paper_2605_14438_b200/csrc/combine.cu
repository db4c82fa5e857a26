// Weighted combine (unpermute): y[t] = sum over t's surviving slots, in ascending
// expert id, of the already ghat-weighted expert rows; then (optionally) the
// residual out = h + y.
//
// Reference order (/root/reference/pkg/src/beamoe/): y starts at zero and
// accumulates experts in ascending id (dispatch/__init__.py:145-156), then the
// shared experts in index order (beam.py:163-164), then out = h + y (beam.py:165).
// Shared experts are planned as ids N..N+S-1, so one ascending pass reproduces it.
// Deterministic: a fixed sequential fp32 sum per element, no atomics.  The
// per-pair rows are fp32 (decode) or bf16 (prefill: halves the HBM traffic of
// the down-projection epilogue and this kernel; the sum stays fp32).
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

// 4 consecutive per-pair values as floats
__device__ __forceinline__ float4 ld_pair4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld_pair4(const __nv_bfloat16* p) {
  const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  return make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                     __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u));
}

template <typename TH, typename TO, typename TP>
__global__ void __launch_bounds__(256) combine_kernel(const int32_t* __restrict__ slot_expert,
                                                      const int32_t* __restrict__ slot_pos,
                                                      const TP* __restrict__ opair, int Keff, int d, int d_pad,
                                                      const TH* __restrict__ h, TO* __restrict__ out) {
  extern __shared__ int sm[];
  int* ex = sm;                 // [Keff]
  int* ps = sm + Keff;          // [Keff]
  int* sorted = sm + 2 * Keff;  // [Keff]
  __shared__ int nvalid_s;
  griddep_wait();
  const int t = blockIdx.x;
  for (int k = threadIdx.x; k < Keff; k += blockDim.x) {
    const int pos = slot_pos[(size_t)t * Keff + k];
    ex[k] = pos >= 0 ? slot_expert[(size_t)t * Keff + k] : -1;
    ps[k] = pos;
  }
  if (threadIdx.x == 0) nvalid_s = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < Keff; k += blockDim.x) {
    const int e = ex[k];
    if (e < 0) continue;
    int r = 0;
    for (int j = 0; j < Keff; ++j) {
      const int ej = ex[j];
      r += ej >= 0 && (ej < e || (ej == e && j < k));
    }
    sorted[r] = ps[k];
    atomicAdd(&nvalid_s, 1);
  }
  __syncthreads();
  const int nv = nvalid_s;
  // one 8-column group per thread (16-byte loads of bf16 rows); the (up to 8 per
  // batch) expert rows of a group are loaded back to back, then added in
  // ascending expert order
  const int d8 = d_pad >> 3;
  for (int c8 = threadIdx.x; c8 < d8; c8 += blockDim.x) {
    if (8 * c8 >= d) break;
    float y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) y[q] = 0.0f;
    for (int r0 = 0; r0 < nv; r0 += 8) {
      float4 v[8][2];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (r0 + q < nv) {
          const TP* row = opair + (size_t)sorted[r0 + q] * d_pad + 8 * c8;
          if constexpr (sizeof(TP) == 2) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(row));
            v[q][0] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                                  __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
            v[q][1] = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xffff0000u),
                                  __uint_as_float(u.w << 16), __uint_as_float(u.w & 0xffff0000u));
          } else {
            v[q][0] = ld_pair4(row);
            v[q][1] = ld_pair4(row + 4);
          }
        }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (r0 + q < nv) {
          y[0] += v[q][0].x;
          y[1] += v[q][0].y;
          y[2] += v[q][0].z;
          y[3] += v[q][0].w;
          y[4] += v[q][1].x;
          y[5] += v[q][1].y;
          y[6] += v[q][1].z;
          y[7] += v[q][1].w;
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = 8 * c8 + q;
      if (c < d) {
        float o = y[q];
        if (h != nullptr) o = to_f32<TH>(h[(size_t)t * d + c]) + o;
        out[(size_t)t * d + c] = from_f32<TO>(o);
      }
    }
  }
}

template <typename TP>
static cudaError_t combine_dispatch(const PlanDev& p, const TP* opair, int T, int Keff, int d, int d_pad,
                                    const void* h, int h_dtype, void* out, int out_dtype, cudaStream_t s) {
  const size_t smem = (size_t)3 * Keff * sizeof(int);
  if (out_dtype == BEAM_F32 && h_dtype == BEAM_F32)
    return launch_pdl(combine_kernel<float, float, TP>, T, 256, smem, s, p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const float*)h, (float*)out);
  if (out_dtype == BEAM_BF16 && h_dtype == BEAM_BF16)
    return launch_pdl(combine_kernel<__nv_bfloat16, __nv_bfloat16, TP>, T, 256, smem, s, p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const __nv_bfloat16*)h, (__nv_bfloat16*)out);
  if (out_dtype == BEAM_F32)
    return launch_pdl(combine_kernel<__nv_bfloat16, float, TP>, T, 256, smem, s, p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const __nv_bfloat16*)h, (float*)out);
  return launch_pdl(combine_kernel<float, __nv_bfloat16, TP>, T, 256, smem, s, p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const float*)h, (__nv_bfloat16*)out);
}

cudaError_t launch_combine(const PlanDev& p, const void* opair, int opair_dtype, int T, int Keff, int d, int d_pad,
                           const void* h, int h_dtype, void* out, int out_dtype, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  cudaError_t e = opair_dtype == BEAM_BF16
                      ? combine_dispatch(p, (const __nv_bfloat16*)opair, T, Keff, d, d_pad, h, h_dtype, out, out_dtype, s)
                      : combine_dispatch(p, (const float*)opair, T, Keff, d, d_pad, h, h_dtype, out, out_dtype, s);
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace beam
