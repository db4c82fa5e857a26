// Decode gate on thread-block clusters: projection + top-K + mask + plan with
// no global-memory handoff inside a token tile.
//
// Reference semantics: rms_norm tensor.py:485-508, topk_route moe.py:116-137,
// mask_forward beam.py:68-72, mask_route _kernels.pyx:17-34, align_block
// dispatch/__init__.py:89-126 (the same device building blocks as gate.cu:
// topk_finish, plan_warp, permute_block in route_device.cuh).
//
// One cluster of CS CTAs per tile of TT tokens.  CTA rank c owns the projection
// columns [c*cpc, (c+1)*cpc) (router logits, then mask pre-activations) over the
// FULL hidden dimension, so every column is final in the CTA that computes it:
//   1. each warp stages one token of the tile as x * norm_w (fp32) in shared
//      memory and its sum of squares (inv_rms); warps stream their column
//      pairs of the fp32 router weights against the tile (FFMA), reduce with a
//      transpose butterfly and leave the logits in shared memory;
//   2. cluster barrier; token i of the tile: warp 0 of CTA i gathers its 2N
//      values from the CS CTAs' shared memory (DSMEM loads), selects (top-K,
//      softmax, mask: topk_finish) and writes every output;
//   3. one tile holding all T*(K+S) <= 32 slots: the routed ids land in CTA 0's
//      shared memory (DSMEM stores) and after a second cluster barrier one warp
//      builds the plan (plan_warp); several tiles: the last cluster to finish
//      (one gpu-scope fence + atomic per cluster) runs the counting-sort permute.
// The 2 MB of Qwen3-30B router weights are read by CS SMs per tile (16 x 128 KB)
// instead of through split-K partials in global memory and two last-CTA
// handoffs (gate.cu: gate_fused_kernel).
#include <cooperative_groups.h>

#include "route_device.cuh"

namespace cg = cooperative_groups;

namespace beam {

constexpr int kCgTT = 8;         // tokens per cluster tile (one staging warp each)
constexpr int kCgWarps = 8;
constexpr int kCgThreads = 32 * kCgWarps;
constexpr int kCgMaxCpc = 64;    // columns per CTA (cols <= 64 * cluster size)
constexpr int kCgBatch = 8;      // 128-element k steps of weight loads in flight per lane

template <typename TX, int NPL, int KIND>
__global__ void __launch_bounds__(kCgThreads, 1)
    gate_cluster_kernel(const TX* __restrict__ X, const float* __restrict__ nw, const float* __restrict__ W, int T,
                        int d, int d_pad, int cpc, TopkArgs a, int E, int bs, bool pad, PlanDev p,
                        int* __restrict__ counter, float* __restrict__ xw) {
  extern __shared__ __align__(16) float smem[];
  float* xs = smem;                                   // [kCgTT][d_pad] x * norm_w
  __shared__ float logit_s[kCgTT][kCgMaxCpc];         // this CTA's columns, final (unscaled by inv_rms)
  __shared__ float inv_s[kCgTT];
  __shared__ float red_s[kCgWarps][2 * kCgTT];
  __shared__ int32_t ids_s[32];
  __shared__ float gw_s[32];
  __shared__ int s_last;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tile = blockIdx.x / cs;
  const int tiles = gridDim.x / cs;
  const int t0 = tile * kCgTT, nt = min(kCgTT, T - t0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cols = a.cols;
  griddep_wait();

  // ---- 1a. stage the tile: warp w <-> token w ----
  if (warp < nt) {
    const TX* row = X + (size_t)(t0 + warp) * d_pad;
    float* dst = xs + (size_t)warp * d_pad;
    float ss = 0.0f;
    for (int k = 4 * lane; k < d_pad; k += 128) {
      const float4 x = ld4<TX>(row + k);
      ss = fmaf(x.x, x.x, ss);
      ss = fmaf(x.y, x.y, ss);
      ss = fmaf(x.z, x.z, ss);
      ss = fmaf(x.w, x.w, ss);
      const float4 g = ld_norm4(nw, k, d);
      *reinterpret_cast<float4*>(dst + k) = make_float4(x.x * g.x, x.y * g.y, x.z * g.z, x.w * g.w);
    }
    ss = warp_sum(ss);
    if (lane == 0) inv_s[warp] = a.has_norm ? 1.0f / sqrtf(ss / (float)a.d + 1e-6f) : 1.0f;
  }
  __syncthreads();
  if (xw != nullptr) {  // the prescaled rows for the decode expert kernels: a slice per CTA
    const int per = ceil_div(d_pad / 4, cs) * 4;
    const int k0 = rank * per, k1 = min(d_pad, k0 + per);
    for (int i = threadIdx.x; i < nt * (per / 4); i += kCgThreads) {
      const int tt = i / (per / 4), k = k0 + 4 * (i % (per / 4));
      if (k < k1)
        *reinterpret_cast<float4*>(xw + (size_t)(t0 + tt) * d_pad + k) =
            *reinterpret_cast<const float4*>(xs + (size_t)tt * d_pad + k);
    }
  }

  // ---- 1b. projection: warp w streams column pairs c0, c0 + 1 over the whole K ----
  const int cbase = rank * cpc;
  for (int cp = 2 * warp; cp < cpc; cp += 2 * kCgWarps) {
    const int c0 = cbase + cp;
    const float* w0 = W + (size_t)min(c0, cols - 1) * d_pad;
    const float* w1 = W + (size_t)min(c0 + 1, cols - 1) * d_pad;
    float acc[2 * kCgTT];
#pragma unroll
    for (int i = 0; i < 2 * kCgTT; ++i) acc[i] = 0.0f;
    for (int kb = 0; kb < d_pad; kb += 128 * kCgBatch) {
      float4 wa[kCgBatch], wb[kCgBatch];
#pragma unroll
      for (int i = 0; i < kCgBatch; ++i) {
        const int k = kb + 128 * i + 4 * lane;
        wa[i] = k < d_pad ? __ldg(reinterpret_cast<const float4*>(w0 + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
        wb[i] = k < d_pad ? __ldg(reinterpret_cast<const float4*>(w1 + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < kCgBatch; ++i) {
        const int k = kb + 128 * i + 4 * lane;
        if (k < d_pad) {
#pragma unroll
          for (int tt = 0; tt < kCgTT; ++tt) {
            if (tt < nt) {
              const float4 x = *reinterpret_cast<const float4*>(xs + (size_t)tt * d_pad + k);
              float s0 = acc[tt], s1 = acc[kCgTT + tt];
              s0 = fmaf(wa[i].x, x.x, s0); s0 = fmaf(wa[i].y, x.y, s0); s0 = fmaf(wa[i].z, x.z, s0); s0 = fmaf(wa[i].w, x.w, s0);
              s1 = fmaf(wb[i].x, x.x, s1); s1 = fmaf(wb[i].y, x.y, s1); s1 = fmaf(wb[i].z, x.z, s1); s1 = fmaf(wb[i].w, x.w, s1);
              acc[tt] = s0;
              acc[kCgTT + tt] = s1;
            }
          }
        }
      }
    }
    warp_reduce_to_smem<2 * kCgTT>(acc, red_s[warp], lane);
    if (lane < 2 * kCgTT) {
      const int j = lane / kCgTT, tt = lane % kCgTT;
      if (cp + j < cpc) logit_s[tt][cp + j] = red_s[warp][lane];
    }
    __syncwarp();
  }
  cluster.sync();  // every column of the tile final and visible cluster-wide

  // ---- 2. top-K / softmax / mask: token i by warp 0 of CTA i ----
  const bool one_warp_plan = tiles == 1 && T * (a.K + a.S) <= 32;
  if (rank < nt && warp == 0) {
    const int i = rank;
    const int Nr = KIND == BEAM_ROUTE_BEAM ? a.N : a.Nr;
    const int mask_off = KIND == BEAM_ROUTE_BEAM ? a.N : a.mask_off;
    float v[NPL], av[NPL];
#pragma unroll
    for (int q = 0; q < NPL; ++q) {  // all DSMEM loads issued before any is used
      const int j = min(lane + 32 * q, Nr - 1);
      const float* src = cluster.map_shared_rank(&logit_s[i][j % cpc], j / cpc);
      v[q] = *src;
      if (mask_off >= 0) {
        const int jm = mask_off + min(lane + 32 * q, a.N - 1);
        av[q] = *cluster.map_shared_rank(&logit_s[i][jm % cpc], jm / cpc);
      } else {
        av[q] = 0.0f;
      }
    }
    TopkArgs b = a;
    if (one_warp_plan) {  // the plan warp (CTA 0) reads the routed ids from its shared memory
      b.ids_s = cluster.map_shared_rank(ids_s, 0);
      b.gw_s = cluster.map_shared_rank(gw_s, 0);
    }
    topk_finish<NPL, KIND>(v, av, inv_s[i], t0 + i, lane, b);
    if (!one_warp_plan) __threadfence();  // ids32 / gw visible before this cluster reports done
  }
  if (one_warp_plan) {
    cluster.sync();
    if (rank == 0 && warp == 0) plan_warp<false>(ids_s, gw_s, T, a.K + a.S, E, bs, p, pad, lane, reinterpret_cast<int*>(xs));
    return;
  }
  // ---- 3. several tiles: the last cluster to finish runs the permute ----
  cluster.sync();
  if (rank != 0) return;
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1) == tiles - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  permute_block<int32_t, kCgWarps, true>(a.ids32, a.gw, T, a.K + a.S, E, bs, p, reinterpret_cast<int*>(xs), pad);
  if (threadIdx.x == 0) *counter = 0;  // replayable (CUDA graphs)
}

static int g_cluster_size = -1;  // 16 where the part allows it, else 8 (0 = clusters unusable)

template <typename TX, int NPL, int KIND>
static cudaError_t cluster_launch(int cs, int tiles, size_t smem, const void* X, const float* nw, const float* W, int T,
                                  int d, int d_pad, int cpc, const TopkArgs& a, int E, int bs, bool pad,
                                  const PlanDev& p, int* counter, float* xw, cudaStream_t s) {
  auto kern = gate_cluster_kernel<TX, NPL, KIND>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * tiles);
  cfg.blockDim = dim3(kCgThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, (const TX*)X, nw, W, T, d, d_pad, cpc, a, E, bs, pad, p, counter, xw);
}

// Cluster size this part runs the gate kernel with (probed once: 16 needs the
// non-portable opt-in and a GPC with 16 free SMs).
static int probe_cluster_size(size_t smem) {
  if (g_cluster_size >= 0) return g_cluster_size;
  auto kern = gate_cluster_kernel<__nv_bfloat16, 4, BEAM_ROUTE_BEAM>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  g_cluster_size = 0;
  for (int cs : {16, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kCgThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n >= 1) {
      g_cluster_size = cs;
      break;
    }
    cudaGetLastError();
  }
  return g_cluster_size;
}

static bool cluster_gate_enabled() {
  static const bool on = [] {
    const char* v = getenv("BEAM_GATE_CLUSTER");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool gate_cluster_supported(int T, int cols, int Nr, int E, int d_pad) {
  return cluster_gate_enabled() && T >= 1 && T <= 64 && Nr <= 512 && cols <= kCgMaxCpc * 8 && E <= 256 &&
         d_pad % 4 == 0 && (size_t)kCgTT * d_pad * sizeof(float) <= 192 * 1024;
}

cudaError_t launch_gate_cluster(const void* X, int x_dtype, const float* norm_w, const float* gate_wT, int T, int d,
                                int d_pad, const TopkArgs& a, int E, int bs, bool pad, const PlanDev& p, int* counter,
                                float* xw, cudaStream_t s) {
  const size_t smem = std::max<size_t>((size_t)kCgTT * d_pad * sizeof(float),
                                       (size_t)(kCgWarps * E + 2 * E + 1 + 32 + 64) * sizeof(int));
  const int cs = probe_cluster_size(smem);
  if (cs == 0) return cudaErrorNotSupported;
  const int cpc = ceil_div(a.cols, cs);
  if (cpc > kCgMaxCpc) return cudaErrorInvalidValue;
  const int tiles = ceil_div(T, kCgTT);
  const int npl = ceil_div(a.Nr, 32);
  const bool beam = a.kind == BEAM_ROUTE_BEAM && a.Nr == a.N && a.cols == 2 * a.N && a.mask_off == a.N;
  cudaError_t e;
#define BEAM_CG(TX_, K_)                                                                                          \
  if (npl <= 1) e = cluster_launch<TX_, 1, K_>(cs, tiles, smem, X, norm_w, gate_wT, T, d, d_pad, cpc, a, E, bs, pad, p, counter, xw, s); \
  else if (npl <= 2) e = cluster_launch<TX_, 2, K_>(cs, tiles, smem, X, norm_w, gate_wT, T, d, d_pad, cpc, a, E, bs, pad, p, counter, xw, s); \
  else if (npl <= 4) e = cluster_launch<TX_, 4, K_>(cs, tiles, smem, X, norm_w, gate_wT, T, d, d_pad, cpc, a, E, bs, pad, p, counter, xw, s); \
  else if (npl <= 8) e = cluster_launch<TX_, 8, K_>(cs, tiles, smem, X, norm_w, gate_wT, T, d, d_pad, cpc, a, E, bs, pad, p, counter, xw, s); \
  else e = cluster_launch<TX_, 16, K_>(cs, tiles, smem, X, norm_w, gate_wT, T, d, d_pad, cpc, a, E, bs, pad, p, counter, xw, s);
  if (x_dtype == BEAM_BF16) {
    if (beam) { BEAM_CG(__nv_bfloat16, BEAM_ROUTE_BEAM) } else { BEAM_CG(__nv_bfloat16, -1) }
  } else {
    if (beam) { BEAM_CG(float, BEAM_ROUTE_BEAM) } else { BEAM_CG(float, -1) }
  }
#undef BEAM_CG
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace beam
