// Decode experts, bulk-copy weight streaming (bf16 weights, T up to ~64).
//
// Reference: dispatch.grouped_execute (/root/reference/pkg/src/beamoe/dispatch/
// __init__.py:129-157) -> expert_forward_np (moe.py:96-100).
//
// B200 design: the decode path is a pure weight stream (each activated expert's
// rows are read exactly once per layer call, masked experts never), so the
// kernel is built around the copy engine, not around load instructions:
//   * one persistent CTA per SM; warp 0 is a producer that walks this CTA's work
//     items (active expert, row block) and issues 1-D bulk copies
//     (cp.async.bulk global -> shared, mbarrier complete_tx) into a 6-8 deep ring
//     of 24-32 KB stages, so ~190 KB per SM are always in flight regardless of
//     what the consumers are doing;
//   * consumer warps each own whole rows of the stage (gate+up pair, or 4 down
//     rows), read them from shared memory, apply them to ALL of the expert's
//     tokens (4 per pass, weights re-read from smem, never from HBM), reduce in
//     registers (no CTA barriers) and release the stage with an mbarrier arrive.
// Active-expert lists, counts and token lists come from the permute kernel on
// the device (no host sync).  Accumulation order is fixed (deterministic).
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {
namespace stream {

constexpr int kConsumers = 4;                  // consumer warps
constexpr int kThreads = 32 * (kConsumers + 1);
constexpr int kSmem = 192 * 1024;              // stage ring
constexpr int kTB = 4;                         // tokens per pass

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completion on an mbarrier; weights are
// streamed once, so mark them evict-first in L2
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 8 bf16 weights from shared memory
__device__ __forceinline__ void lds_bf16x8(const __nv_bfloat16* p, float* out) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  unpack<__nv_bfloat16>(v, out);
}

// x chunk of 8 elements (k % 8 == 0) as floats
template <typename TX>
__device__ __forceinline__ void ldx8(const TX* p, float* out) {
  if constexpr (sizeof(TX) == 2) {
    unpack<__nv_bfloat16>(ld_cached(p), out);
  } else {
    unpack<float>(ld_cached(p), out);
    unpack<float>(ld_cached(p + 4), out + 4);
  }
}

// Reduce V lane-partials to lane-uniform sums (V <= 8): plain butterflies.
template <int V>
__device__ __forceinline__ void warp_allreduce(float (&v)[V]) {
#pragma unroll
  for (int i = 0; i < V; ++i) v[i] = warp_sum(v[i]);
}

// ---------------------------------------------------------------------------
// gate / up: item = (active expert, group of 4 features) -> stage = 4 gate rows
// + 4 up rows (two contiguous 4-row blocks of the packed layout).  Consumer warp
// w owns feature w of the group (its gate row and its up row).
// ---------------------------------------------------------------------------
template <typename TX, int ACT>
__global__ void __launch_bounds__(kThreads, 1)
    gateup_stream_kernel(const __nv_bfloat16* __restrict__ Wgu, const TX* __restrict__ X,
                         const float* __restrict__ inv, const float* __restrict__ nw, int d, int d_pad, int f_pad,
                         PlanDev p, float* __restrict__ act) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = 8 * d_pad * 2;
  const int nstages = min(8, kSmem / stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nstages * stage_bytes);
  uint64_t* empty = full + nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  griddep_wait();
  const int groups = f_pad / 4;
  const int total = p.meta[0] * groups;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x) {
        const int a = item / groups, g = item % groups;
        const int e = p.active[a];
        const int feat0 = g * 4;
        const int row_g = (feat0 >> 4) * 32 + (feat0 & 15);
        const __nv_bfloat16* base = Wgu + ((size_t)e * 2 * f_pad + row_g) * d_pad;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], stage_bytes);
        uint8_t* dst = smem + stage * stage_bytes;
        bulk_load(dst, base, stage_bytes / 2, &full[stage], pol);                            // gate rows
        bulk_load(dst + stage_bytes / 2, base + 16 * d_pad, stage_bytes / 2, &full[stage], pol);  // up rows
        if (++stage == nstages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  // consumers
  const int w = warp - 1;  // feature within the group
  int stage = 0;
  uint32_t phase = 0;
  const int nchunk = d_pad / 8;  // 16-byte chunks per row
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int a = item / groups, g = item % groups;
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    mbar_wait(&full[stage], phase);
    const __nv_bfloat16* wg = reinterpret_cast<const __nv_bfloat16*>(smem + stage * stage_bytes) + w * d_pad;
    const __nv_bfloat16* wu = wg + 4 * d_pad;
    for (int t0 = 0; t0 < cnt; t0 += kTB) {
      const int nt = min(kTB, cnt - t0);
      int tk[kTB];
#pragma unroll
      for (int j = 0; j < kTB; ++j) tk[j] = p.tok[off + t0 + (j < nt ? j : 0)];
      float ag[kTB], au[kTB];
#pragma unroll
      for (int j = 0; j < kTB; ++j) ag[j] = au[j] = 0.0f;
      for (int c = lane; c < nchunk; c += 32) {
        float gw[8], uw[8];
        lds_bf16x8(wg + 8 * c, gw);
        lds_bf16x8(wu + 8 * c, uw);
        if (nw) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int k = 8 * c + q;
            const float s = k < d ? __ldg(nw + k) : 0.0f;
            gw[q] *= s;
            uw[q] *= s;
          }
        }
#pragma unroll
        for (int j = 0; j < kTB; ++j) {
          if (j < nt) {
            float x[8];
            ldx8<TX>(X + (size_t)tk[j] * d_pad + 8 * c, x);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              ag[j] = fmaf(gw[q], x[q], ag[j]);
              au[j] = fmaf(uw[q], x[q], au[j]);
            }
          }
        }
      }
      warp_allreduce<kTB>(ag);
      warp_allreduce<kTB>(au);
      if (lane < kTB && lane < nt) {
        float gs = 0.f, us = 0.f;
#pragma unroll
        for (int j = 0; j < kTB; ++j)
          if (j == lane) {
            gs = ag[j];
            us = au[j];
          }
        const float s = inv ? inv[tk[lane]] : 1.0f;  // x_n = x * inv_rms * w
        act[(size_t)(off + t0 + lane) * f_pad + g * 4 + w] = activation<ACT>(gs * s) * (us * s);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == nstages) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// ---------------------------------------------------------------------------
// down: item = (active expert, block of 16 output rows) -> stage = 16 contiguous
// rows of W_d^T; consumer warp w owns rows 4w..4w+3.
// ---------------------------------------------------------------------------
constexpr int kDownRows = 16;

__global__ void __launch_bounds__(kThreads, 1)
    down_stream_kernel(const __nv_bfloat16* __restrict__ Wd, const float* __restrict__ act, int d_pad, int f_pad,
                       PlanDev p, float* __restrict__ opair) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = kDownRows * f_pad * 2;
  const int nstages = min(8, kSmem / stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nstages * stage_bytes);
  uint64_t* empty = full + nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  griddep_wait();
  const int groups = d_pad / kDownRows;
  const int total = p.meta[0] * groups;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x) {
        const int a = item / groups, g = item % groups;
        const int e = p.active[a];
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], stage_bytes);
        bulk_load(smem + stage * stage_bytes, Wd + ((size_t)e * d_pad + g * kDownRows) * f_pad, stage_bytes,
                  &full[stage], pol);
        if (++stage == nstages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  const int w = warp - 1;
  int stage = 0;
  uint32_t phase = 0;
  const int nchunk = f_pad / 8;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int a = item / groups, g = item % groups;
    const int e = p.active[a];
    const int cnt = p.counts[e], off = p.offsets[e];
    mbar_wait(&full[stage], phase);
    const __nv_bfloat16* wr = reinterpret_cast<const __nv_bfloat16*>(smem + stage * stage_bytes) + 4 * w * f_pad;
    for (int t0 = 0; t0 < cnt; t0 += kTB) {
      const int nt = min(kTB, cnt - t0);
      float acc[4][kTB];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < kTB; ++j) acc[r][j] = 0.0f;
      for (int c = lane; c < nchunk; c += 32) {
        float xs[kTB][8];
#pragma unroll
        for (int j = 0; j < kTB; ++j) {
          if (j < nt) {
            const float* ap = act + (size_t)(off + t0 + j) * f_pad + 8 * c;
            const float4 u = __ldg(reinterpret_cast<const float4*>(ap));
            const float4 v = __ldg(reinterpret_cast<const float4*>(ap) + 1);
            xs[j][0] = u.x; xs[j][1] = u.y; xs[j][2] = u.z; xs[j][3] = u.w;
            xs[j][4] = v.x; xs[j][5] = v.y; xs[j][6] = v.z; xs[j][7] = v.w;
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          float wv[8];
          lds_bf16x8(wr + r * f_pad + 8 * c, wv);
#pragma unroll
          for (int j = 0; j < kTB; ++j)
            if (j < nt) {
#pragma unroll
              for (int q = 0; q < 8; ++q) acc[r][j] = fmaf(wv[q], xs[j][q], acc[r][j]);
            }
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) warp_allreduce<kTB>(acc[r]);
      if (lane < 4 * kTB) {
        const int r = lane / kTB, j = lane % kTB;
        if (j < nt) {
          float v = 0.f;
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int jj = 0; jj < kTB; ++jj)
              if (rr == r && jj == j) v = acc[rr][jj];
          const int pos = off + t0 + j;
          opair[(size_t)pos * d_pad + g * kDownRows + 4 * w + r] = v * p.w[pos];
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == nstages) {
      stage = 0;
      phase ^= 1;
    }
  }
}

}  // namespace stream

bool stream_supported(const beam_layer_t& L, const Dims& g) {
  return L.wdtype == BEAM_BF16 && g.d_pad % 16 == 0 && g.f_pad % 16 == 0 && 8 * g.d_pad * 2 <= stream::kSmem &&
         stream::kDownRows * g.f_pad * 2 <= stream::kSmem && g.d_pad % stream::kDownRows == 0;
}

static size_t stream_smem(int stage_bytes) {
  const int nst = std::min(8, stream::kSmem / stage_bytes);
  return (size_t)nst * stage_bytes + 2 * nst * sizeof(uint64_t);
}

cudaError_t launch_gateup_stream(const beam_layer_t& L, const Dims& g, const void* X, int x_dtype,
                                 const float* inv, const float* nw, const PlanDev& p, float* act, cudaStream_t s) {
  using namespace stream;
  const size_t smem = stream_smem(8 * g.d_pad * 2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gateup_stream_kernel<__nv_bfloat16, BEAM_ACT_SILU>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem + 1024);
    cudaFuncSetAttribute(gateup_stream_kernel<__nv_bfloat16, BEAM_ACT_IDENTITY>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem + 1024);
    cudaFuncSetAttribute(gateup_stream_kernel<float, BEAM_ACT_SILU>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem + 1024);
    cudaFuncSetAttribute(gateup_stream_kernel<float, BEAM_ACT_IDENTITY>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem + 1024);
    attr = true;
  }
  const __nv_bfloat16* W = (const __nv_bfloat16*)L.w_gu;
  cudaError_t e;
  const int grid = num_sms();
  if (x_dtype == BEAM_BF16) {
    if (L.activation == BEAM_ACT_SILU)
      e = launch_pdl(gateup_stream_kernel<__nv_bfloat16, BEAM_ACT_SILU>, grid, kThreads, smem, s, W, (const __nv_bfloat16*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
    else
      e = launch_pdl(gateup_stream_kernel<__nv_bfloat16, BEAM_ACT_IDENTITY>, grid, kThreads, smem, s, W, (const __nv_bfloat16*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
  } else {
    if (L.activation == BEAM_ACT_SILU)
      e = launch_pdl(gateup_stream_kernel<float, BEAM_ACT_SILU>, grid, kThreads, smem, s, W, (const float*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
    else
      e = launch_pdl(gateup_stream_kernel<float, BEAM_ACT_IDENTITY>, grid, kThreads, smem, s, W, (const float*)X, inv, nw, g.d, g.d_pad, g.f_pad, p, act);
  }
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_down_stream(const beam_layer_t& L, const Dims& g, const PlanDev& p, const float* act,
                               float* opair, cudaStream_t s) {
  using namespace stream;
  const size_t smem = stream_smem(kDownRows * g.f_pad * 2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(down_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem + 1024);
    attr = true;
  }
  cudaError_t e = launch_pdl(down_stream_kernel, num_sms(), kThreads, smem, s, (const __nv_bfloat16*)L.w_down, act,
                             g.d_pad, g.f_pad, p, opair);
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace beam
