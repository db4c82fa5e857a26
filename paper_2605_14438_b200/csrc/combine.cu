// Weighted combine (unpermute): y[t] = sum over t's surviving slots, in ascending
// expert id, of the already ghat-weighted expert rows; then (optionally) the
// residual out = h + y.
//
// Reference order (/root/reference/pkg/src/beamoe/): y starts at zero and
// accumulates experts in ascending id (dispatch/__init__.py:145-156), then the
// shared experts in index order (beam.py:163-164), then out = h + y (beam.py:165).
// Shared experts are planned as ids N..N+S-1, so one ascending pass reproduces it.
// Deterministic: a fixed sequential fp32 sum per element, no atomics.
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

template <typename TH, typename TO>
__global__ void __launch_bounds__(256) combine_kernel(const int32_t* __restrict__ slot_expert,
                                                      const int32_t* __restrict__ slot_pos,
                                                      const float* __restrict__ opair, int Keff,
                                                      int d, int d_pad, const TH* __restrict__ h,
                                                      TO* __restrict__ out) {
  extern __shared__ int sm[];
  int* ex = sm;              // [Keff]
  int* ps = sm + Keff;       // [Keff]
  int* sorted = sm + 2 * Keff;  // [Keff]
  __shared__ int nvalid_s;
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
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float y = 0.0f;
    for (int r = 0; r < nv; ++r) y += opair[(size_t)sorted[r] * d_pad + c];
    if (h != nullptr) y = to_f32<TH>(h[(size_t)t * d + c]) + y;
    out[(size_t)t * d + c] = from_f32<TO>(y);
  }
}

cudaError_t launch_combine(const PlanDev& p, const float* opair, int T, int Keff, int d, int d_pad,
                           const void* h, int h_dtype, void* out, int out_dtype, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  const size_t smem = (size_t)3 * Keff * sizeof(int);
  if (out_dtype == BEAM_F32 && h_dtype == BEAM_F32)
    combine_kernel<float, float><<<T, 256, smem, s>>>(p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const float*)h, (float*)out);
  else if (out_dtype == BEAM_BF16 && h_dtype == BEAM_BF16)
    combine_kernel<__nv_bfloat16, __nv_bfloat16><<<T, 256, smem, s>>>(p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const __nv_bfloat16*)h, (__nv_bfloat16*)out);
  else if (out_dtype == BEAM_F32 && h_dtype == BEAM_BF16)
    combine_kernel<__nv_bfloat16, float><<<T, 256, smem, s>>>(p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const __nv_bfloat16*)h, (float*)out);
  else
    combine_kernel<float, __nv_bfloat16><<<T, 256, smem, s>>>(p.slot_expert, p.slot_pos, opair, Keff, d, d_pad, (const float*)h, (__nv_bfloat16*)out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
