// Mask-router training kernels: the closed-form straight-through
// backward of BEAM and its sparsity regulariser.
//
// Reference (/root/reference/pkg/src/beamoe/beam.py):
//   sparsity_loss   :87-97    sum over each token's top-K candidates of sigmoid(a),
//                             / (K*T)  (raw mask values lie in (0, 1): |.| is identity)
//   ste_backward    :100-124  dL/da_i = (dL_task/dghat_i * g_i + beta/(K*T) * [g_i > 0])
//                                       * sigma'(a_i)   (binariser = identity)
//   training forward :146-157 every top-K candidate is evaluated (moe.py:223-279
//                             compute_ids), so dL_task/dghat_i = <dy, E_i(x_n)> exists
//                             for masked candidates too.
//
// B200 design: the candidate pass reuses the inference plan / expert kernels with
// unit slot weights (the expert rows land un-scaled in `opair`), then ONE kernel per
// token computes the K slot dots with dy and writes the dense STE gradient row —
// the [T, N] upstream of the reference is never materialised.  All reductions run
// in a fixed order (warp butterflies, a single-CTA tree): results are independent
// of the grid and bit-reproducible.
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

// ids32 / unit weights of the candidate plan from the gate's top-K ids.
__global__ void candidates_kernel(const int64_t* __restrict__ topk, int M, int32_t* __restrict__ ids32,
                                  float* __restrict__ gw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  griddep_wait();
  ids32[i] = (int32_t)topk[i];
  gw[i] = 1.0f;
}

cudaError_t launch_candidates(const int64_t* topk, int M, int32_t* ids32, float* gw, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  candidates_kernel<<<ceil_div(M, 256), 256, 0, s>>>(topk, M, ids32, gw);
  count_launches(1);
  return cudaGetLastError();
}

template <typename TO> __device__ __forceinline__ float ld_row(const TO* p);
template <> __device__ __forceinline__ float ld_row<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ld_row<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// sigma'(a) = s (1 - s) with the reference's two-tail sigmoid (tensor.py:406-411)
__device__ __forceinline__ float ste_term(float up_g, float g, float a, float bt) {
  const float s = sigmoid_ref(a);
  return (up_g + (g > 0.0f ? bt : 0.0f)) * (s * (1.0f - s));
}

// One warp per token: dghat[t,k] = <dy[t], O[slot_pos[t,k]]> for the K candidate
// slots (O = un-weighted expert rows of the candidate pass), then the dense
// gradient row: exact 0 off the candidate set, the closed form on it.
template <typename TO>
__global__ void __launch_bounds__(256) mask_grad_kernel(const float* __restrict__ dy, int d,
                                                        const TO* __restrict__ O, int d_pad,
                                                        const int32_t* __restrict__ slot_pos,
                                                        const int64_t* __restrict__ topk,
                                                        const float* __restrict__ weights,
                                                        const float* __restrict__ pre_act, int T, int N,
                                                        int K, float bt, float* __restrict__ grad,
                                                        float* __restrict__ dghat) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  griddep_wait();
  const float* dyr = dy + (size_t)t * d;
  float mine = 0.0f;
  for (int k = 0; k < K; ++k) {
    const int pos = slot_pos[(size_t)t * K + k];
    float part = 0.0f;
    if (pos >= 0) {
      const TO* orow = O + (size_t)pos * d_pad;
#pragma unroll 4
      for (int c = lane; c < d; c += 32) part = fmaf(dyr[c], ld_row<TO>(orow + c), part);
    }
    const float dot = warp_sum(part);
    if (lane == k) mine = dot;
  }
  float* gr = grad + (size_t)t * N;
  for (int j = lane; j < N; j += 32) gr[j] = 0.0f;
  __syncwarp();  // orders the zero fill before the candidate entries (same warp)
  if (lane < K) {
    const int64_t id = topk[(size_t)t * K + lane];
    if (dghat) dghat[(size_t)t * K + lane] = mine;
    if (id >= 0 && id < N) {
      const size_t o = (size_t)t * N + id;
      const float g = weights[o];
      gr[id] = ste_term(mine * g, g, pre_act[o], bt);
    }
  }
}

cudaError_t launch_mask_grad(const float* dy, int d, const void* O, int o_dtype, int d_pad,
                             const int32_t* slot_pos, const int64_t* topk, const float* weights,
                             const float* pre_act, int T, int N, int K, float bt, float* grad,
                             float* dghat, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (K > 32) return cudaErrorInvalidValue;
  const dim3 grid(ceil_div(T, 8));
  cudaError_t e;
  if (o_dtype == BEAM_BF16)
    e = launch_pdl(mask_grad_kernel<__nv_bfloat16>, grid, 256, 0, s, dy, d, (const __nv_bfloat16*)O, d_pad,
                   slot_pos, topk, weights, pre_act, T, N, K, bt, grad, dghat);
  else
    e = launch_pdl(mask_grad_kernel<float>, grid, 256, 0, s, dy, d, (const float*)O, d_pad, slot_pos, topk,
                   weights, pre_act, T, N, K, bt, grad, dghat);
  count_launches(1);
  return e;
}

// Dense closed form (beam.py:121-124): grad = (up * w + bt * [w > 0]) * s (1 - s).
__global__ void ste_dense_kernel(const float* __restrict__ up, const float* __restrict__ w,
                                 const float* __restrict__ a, long long n, float bt,
                                 float* __restrict__ grad) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float g = w[i];
    grad[i] = ste_term(up[i] * g, g, a[i], bt);
  }
}

cudaError_t launch_ste_dense(const float* up, const float* w, const float* a, long long n, float bt,
                             float* grad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = (n + 255) / 256;
  const int grid = (int)(blocks < 8LL * num_sms() ? blocks : 8LL * num_sms());
  ste_dense_kernel<<<grid, 256, 0, s>>>(up, w, a, n, bt, grad);
  count_launches(1);
  return cudaGetLastError();
}

// sparsity_loss: one CTA, thread i sums entries i, i + 256, ... in order (fp64, as
// the reference), then a fixed shared-memory tree.
__global__ void __launch_bounds__(256) sparsity_loss_kernel(const float* __restrict__ raw,
                                                            const int64_t* __restrict__ topk, int T,
                                                            int N, int K, float* __restrict__ loss) {
  __shared__ double part[256];
  griddep_wait();
  const long long M = (long long)T * K;
  double s = 0.0;
  for (long long i = threadIdx.x; i < M; i += 256) {
    const int64_t id = topk[i];
    if (id >= 0 && id < N) s += (double)raw[(i / K) * N + id];
  }
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[0] = (float)(part[0] / ((double)T * (double)K));
}

cudaError_t launch_sparsity_loss(const float* raw, const int64_t* topk, int T, int N, int K, float* loss,
                                 cudaStream_t s) {
  if (T <= 0 || K <= 0) return cudaMemsetAsync(loss, 0, sizeof(float), s);
  cudaError_t e = launch_pdl(sparsity_loss_kernel, dim3(1), dim3(256), 0, s, raw, topk, T, N, K, loss);
  count_launches(1);
  return e;
}

}  // namespace beam
