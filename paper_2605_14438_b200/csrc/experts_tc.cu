// Grouped SwiGLU experts on the 5th-generation tensor cores (prefill path).
//
// Reference: dispatch.grouped_execute (/root/reference/pkg/src/beamoe/dispatch/
// __init__.py:129-157) -> expert_forward_np (moe.py:96-100):
//     O_e = (silu(X_e W_gate) * (X_e W_up)) W_down,  y[rows] += O_e * ghat
//
// B200 design ("swap AB" grouped GEMM, one persistent kernel per GEMM):
//   * A = expert weights (UMMA M = 128 weight rows per tile, K-major, bf16),
//     B = the expert's surviving tokens in plan order (UMMA N = tokens, K-major),
//     D = fp32 accumulator in TMEM (two 256-column buffers: the epilogue of tile
//     i overlaps the MMAs of tile i+1).
//   * Tiles (expert, m-tile, n-tile) are enumerated on the device from the plan
//     counts — masked slots never become tiles; the MMA N of each tile is the
//     expert's remaining token count rounded up to 16, so partial tiles cost no
//     tensor-core work and no B bytes beyond the next 64-row TMA box.
//   * Warp roles: warp 0 = TMA producer (SWIZZLE_128B boxes into a 4-stage
//     mbarrier ring), warp 1 = tcgen05.mma issuer (one elected thread,
//     tcgen05.commit frees smem stages / publishes accumulators), warps 2-5 =
//     epilogue (tcgen05.ld -> registers -> global).
//   * GEMM1 (gate/up, K = d): packed rows interleave 16 gate + 16 up rows per
//     32, so one warp's TMEM lanes hold matching gate/up rows; the epilogue
//     computes act = silu(g) * u (fp32) and stores bf16 act[pos, f].
//   * GEMM2 (down, K = f): epilogue scales by the routing weight ghat and stores
//     fp32 opair[pos, d] for the deterministic ascending-expert combine.
#include <cuda.h>

#include <cstdlib>

#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {
namespace tc {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int kStages = 4;
constexpr int kBBox = 64;  // B rows per TMA box
constexpr int kABytes = BM * BK * 2;
constexpr int kBBytes = BN * BK * 2;
constexpr int kBBoxBytes = kBBox * BK * 2;
constexpr int kTmemCols = 512;
constexpr int kThreads = 192;
constexpr int kMaxE = 1024;

struct Args {
  int mode;  // 0 gate/up, 1 down, 2 router projection (fp32 out, no weight)
  int E;
  int m_rows;  // A rows per expert
  int K;
  int b_kblocks;  // B k-blocks before the coordinate wraps (router: 3 bf16 splits of W share one h)
  const int32_t* counts;
  const int32_t* offsets;
  const float* w;
  __nv_bfloat16* act;
  int f_pad;
  void* opair;  // mode 1: [cap, d_pad] bf16 per-pair rows; mode 2: fp32 logits
  int d_pad;
  int bn;  // token-tile width (<= BN, multiple of 16): narrower tiles spread few-expert GEMMs over more SMs
  int p_cols, p_T;  // mode 2: logits P[split][p_T][p_cols], split = A row / p_cols
  int apol;         // weight-tile L2 policy (a_policy)
  int epi_skip;     // diagnostics (BEAM_EPI_SKIP=1): TMEM drained but no math / stores
  int epi_direct;   // mode 1: store rows straight from registers (BEAM_EPI_DIRECT=1; default off)
  int b_rows = 0;   // checked build: rows of the B operand (packed tokens / act)
  unsigned* check = nullptr;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// L2 policies: weights stream through once (evict first); token tiles are re-read
// by every m-tile of their expert (evict last)
__device__ __forceinline__ uint64_t l2_policy(bool evict_first) {
  uint64_t p;
  if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Weight (A) tile policy: evict-first when every weight tile is read by one unit
// only (one token tile per expert), evict-normal when several token tiles of an
// expert re-read it (prefill at low sparsity).  apol: 0 auto, 1 first, 2 normal, 3 last.
__device__ __forceinline__ uint64_t a_policy(int apol, bool multi_ntile) {
  uint64_t p;
  if (apol == 3) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (apol == 2 || (apol == 0 && multi_ntile)) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;              // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

struct Tile {
  int e, m_tile, a_row0, b_row0, ntok, nmma;
};

// Work unit u = (expert, m-group of CM m-tiles, n-tile); CTA `rank` of the cluster
// takes m-tile mg*CM + rank, all CTAs of a cluster share the token (B) tile.
__device__ __forceinline__ Tile decode(int u, const int* tile_off, int E, int MG, int CM, int rank,
                                       const Args& a) {
  // largest e with tile_off[e] * MG <= u
  int lo = 0, hi = E;  // invariant: tile_off[lo]*MG <= u < tile_off[hi]*MG
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tile_off[mid] * MG <= u) lo = mid;
    else hi = mid;
  }
  Tile r;
  r.e = lo;
  const int nt = tile_off[lo + 1] - tile_off[lo];
  const int local = u - tile_off[lo] * MG;
  r.m_tile = (local / nt) * CM + rank;
  const int n_tile = local % nt;
  r.a_row0 = lo * a.m_rows + r.m_tile * BM;
  const int tok0 = n_tile * a.bn;
  r.ntok = min(a.bn, (a.mode == 2 ? a.p_T : a.counts[lo]) - tok0);
  r.b_row0 = (a.mode == 2 ? 0 : a.offsets[lo]) + tok0;
  r.nmma = (r.ntok + 15) & ~15;
  return r;
}

constexpr int kStgBytes = 32 * BM * 4;  // epilogue staging: 32 tokens x 128 rows (fp32 worst case)

// named barrier over the 4 epilogue warps of one group (ids 1, 2)
__device__ __forceinline__ void epi_bar(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

// One accumulator tile -> global, 32 token columns at a time.  The 4 epilogue
// warps (TMEM lanes 32*w4..) transpose through shared memory so every global
// store is a contiguous token row (128-512 B per warp instruction) instead of
// a scattered column.
//   mode 0: act[pos, f]   = bf16(silu(gate) * up)  (64 features per tile)
//   mode 1: opair[pos, d] = bf16(ghat[pos] * acc)  (128 output channels)
//   mode 2: P[t, c]       = acc (fp32, router / mask logits)
// A group of 4 epilogue warps (one per TMEM lane quadrant, barrier `bar`) takes
// the 32-token chunks c_begin, c_begin + c_step, ...
__device__ __forceinline__ void epilogue_tile(const Args& args, const Tile& tl, uint32_t tbase, int w4, int lane,
                                              uint8_t* stg, int c_begin = 0, int c_step = 32, int bar = 1) {
  for (int c0 = c_begin; c0 < tl.ntok; c0 += c_step) {
    const int rows = min(32, tl.ntok - c0);
    float v[32];
    tmem_ld32(tbase + c0, v);
    if (args.epi_skip) continue;
    if (args.mode == 0) {
      // lanes 0-15 hold gate rows, 16-31 the matching up rows, of features 16*w4 + (lane & 15).
      // Staging rows are 128 B (one bank sweep), so token rows j and 16 + j written
      // by the two half-warps would hit the same banks: rows 16..31 store their
      // features XOR 32 (the other half of the banks) — conflict-free, undone on read.
      __nv_bfloat16* s = reinterpret_cast<__nv_bfloat16*>(stg);  // [32 tokens][64 features]
      const int fl = 16 * w4 + (lane & 15);
      const bool lo = lane < 16;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float send = lo ? v[16 + j] : v[j];
        const float r = __shfl_xor_sync(0xffffffffu, send, 16);
        const float g = lo ? v[j] : r;
        const float u = lo ? r : v[16 + j];
        s[(lo ? j : 16 + j) * 64 + (lo ? fl : fl ^ 32)] = __float2bfloat16_rn(activation<BEAM_ACT_SILU>(g) * u);
      }
      epi_bar(bar);
      for (int row = w4; row < rows; row += 4) {
        const uint32_t val = reinterpret_cast<const uint32_t*>(s + row * 64)[row < 16 ? lane : lane ^ 16];
        reinterpret_cast<uint32_t*>(args.act + (size_t)(tl.b_row0 + c0 + row) * args.f_pad + tl.m_tile * 64)[lane] = val;
      }
    } else if (args.mode == 1 && args.epi_direct) {
      // direct: for token j the warp's 32 lanes hold 32 consecutive channels, so
      // each store is a contiguous 64-byte row segment — no staging, no barrier
      const float wl = lane < rows ? __ldg(args.w + tl.b_row0 + c0 + lane) : 0.0f;
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.opair) + (size_t)(tl.b_row0 + c0) * args.d_pad +
                           tl.m_tile * BM + 32 * w4 + lane;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float wj = __shfl_sync(0xffffffffu, wl, j);
        if (j < rows) dst[(size_t)j * args.d_pad] = __float2bfloat16_rn(v[j] * wj);
      }
      continue;
    } else if (args.mode == 1) {
      __nv_bfloat16* s = reinterpret_cast<__nv_bfloat16*>(stg);  // [32 tokens][128 channels]
      const float wl = lane < rows ? __ldg(args.w + tl.b_row0 + c0 + lane) : 0.0f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float wj = __shfl_sync(0xffffffffu, wl, j);
        s[j * BM + 32 * w4 + lane] = __float2bfloat16_rn(v[j] * wj);
      }
      epi_bar(bar);
      for (int row = w4; row < rows; row += 4) {
        const uint2 val = reinterpret_cast<const uint2*>(s + row * BM)[lane];
        reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(args.opair) + (size_t)(tl.b_row0 + c0 + row) * args.d_pad +
                                 tl.m_tile * BM)[lane] = val;
      }
    } else {
      float* s = reinterpret_cast<float*>(stg);  // [32 tokens][128 columns]
#pragma unroll
      for (int j = 0; j < 32; ++j) s[j * BM + 32 * w4 + lane] = v[j];
      epi_bar(bar);
      // A rows are [split][p_cols] (split-K over the bf16 terms of W): row block
      // m_tile*BM lies inside one split
      const int r0 = tl.m_tile * BM, sp = r0 / args.p_cols, col0 = r0 % args.p_cols;
      float* P = reinterpret_cast<float*>(args.opair) + ((size_t)sp * args.p_T) * args.p_cols + col0;
      for (int row = w4; row < rows; row += 4) {
        const float4 val = reinterpret_cast<const float4*>(s + row * BM)[lane];
        reinterpret_cast<float4*>(P + (size_t)(tl.b_row0 + c0 + row) * args.p_cols)[lane] = val;
      }
    }
    epi_bar(bar);  // staging reused by the next chunk
  }
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// B box multicast to every CTA of the cluster (same smem offset, each CTA's barrier)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// MMA completion arrives on the barrier at the same offset in every CTA of the cluster
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}

// CM = cluster size along M: the CTAs of a cluster compute CM consecutive m-tiles of
// the same (expert, token tile) and share every B (token) stage through TMA
// multicast, dividing the L2 -> SM operand traffic of B by CM.
template <int CM>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        Args args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                                  // kStages x 16 KB
  uint8_t* sb = smem + kStages * kABytes;              // kStages x 32 KB
  uint8_t* stg = sb + kStages * kBBytes;               // epilogue staging
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + kStgBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* tile_off = reinterpret_cast<int*>(tmem_slot + 4);  // [E + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_wait();  // PDL: the plan / operands come from the previous kernel
  const int E = args.E;
  const int MT = args.m_rows / BM;
  const int KB = args.K / BK;

  // per-expert n-tile prefix (masked experts: zero tiles)
  if (warp == 0) {
    int carry = 0;
    if (lane == 0) tile_off[0] = 0;
    for (int base = 0; base < E; base += 32) {
      const int e = base + lane;
      int v = e < E ? ((args.mode == 2 ? args.p_T : args.counts[e]) + args.bn - 1) / args.bn : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (e < E) tile_off[e + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CM);  // released by the MMAs of every CTA in the cluster
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  fence_before();
  if constexpr (CM > 1) cluster_sync_all();  // barrier inits visible cluster-wide
  else __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int rank = CM > 1 ? (int)cluster_rank() : 0;
  const uint16_t cmask = (uint16_t)((1u << CM) - 1u);
  const int MG = MT / CM;
  const int total = tile_off[E] * MG;
  const int u0 = blockIdx.x / CM, ustep = gridDim.x / CM;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t polB = l2_policy(false);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = u0; t < total; t += ustep) {
        const Tile tl = decode(t, tile_off, E, MG, CM, rank, args);
        const uint64_t polA = args.mode == 2 ? polB : a_policy(args.apol, tile_off[tl.e + 1] - tile_off[tl.e] > 1);
        const int nbox = (tl.nmma + kBBox - 1) / kBBox;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kABytes + nbox * kBBoxBytes);
          tma_load_2d(sa + stage * kABytes, &tmA, &full[stage], kb * BK, tl.a_row0, polA);
          for (int c = 0; c < nbox; ++c) {
            if constexpr (CM > 1) {
              if (c % CM == rank)
                tma_load_2d_mc(sb + stage * kBBytes + c * kBBoxBytes, &tmB, &full[stage],
                               (kb % args.b_kblocks) * BK, tl.b_row0 + c * kBBox, cmask);
            } else {
              tma_load_2d(sb + stage * kBBytes + c * kBBoxBytes, &tmB, &full[stage], (kb % args.b_kblocks) * BK,
                          tl.b_row0 + c * kBBox, polB);
            }
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc_base = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = u0; t < total; t += ustep) {
        const Tile tl = decode(t, tile_off, E, MG, CM, rank, args);
        const uint32_t idesc = idesc_base | ((uint32_t)(tl.nmma >> 3) << 17);
        const uint32_t tmem_d = tmem_base + acc * BN;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sa + stage * kABytes));
          const uint64_t bd = sdesc_sw128(smem_u32(sb + stage * kBBytes));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16(tmem_d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          if constexpr (CM > 1) mma_commit_mc(&empty[stage], cmask);
          else mma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5 -> TMEM lanes 32*(warp%4)) ----------------
    const int lane_base = 32 * (warp & 3);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = u0; t < total; t += ustep) {
      const Tile tl = decode(t, tile_off, E, MG, CM, rank, args);
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      epilogue_tile(args, tl, tmem_base + ((uint32_t)lane_base << 16) + acc * BN, warp & 3, lane, stg);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  fence_before();
  if constexpr (CM > 1) cluster_sync_all();  // no CTA leaves while peers may still multicast into it
  else __syncthreads();
  fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
}

// ---------------------------------------------------------------------------
// 2-SM variant (cta_group::2): a CTA pair computes a 256-row x N tile with one
// tcgen05.mma issued by the leader.  Each CTA stages its own 128 weight rows and
// HALF of the token rows, so per-SM operand traffic per FLOP drops by 1.5x vs
// the 1-SM kernel and the ring holds 6 stages.  The TMA loads of both CTAs
// signal the leader's full barrier; the leader's commits release both CTAs'
// stages (multicast); both epilogues release the leader's accumulator barrier.
// ---------------------------------------------------------------------------
constexpr int kStages2 = 6;
constexpr int kMaxE2 = 256;  // experts the 2-SM kernel's shared tile prefix holds (6 stages fill the rest)
constexpr int kBHalfBytes = (BN / 2) * BK * 2;  // 16 KB: 128 token rows

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}


__device__ __forceinline__ void mma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

constexpr int kThreads2 = 320;  // producer, MMA, 2 x 4 epilogue warps

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    grouped_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            Args args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                                  // kStages2 x 16 KB (this CTA's 128 weight rows)
  uint8_t* sb = smem + kStages2 * kABytes;             // kStages2 x 16 KB (this CTA's half of the tokens)
  uint8_t* stg = sb + kStages2 * kBHalfBytes;          // epilogue staging, one per epilogue group
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + 2 * kStgBytes);
  uint64_t* empty = full + kStages2;
  uint64_t* tfull = empty + kStages2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* tile_off = reinterpret_cast<int*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_rank();
  griddep_wait();
  const int E = args.E;
  const int MT = args.m_rows / BM;
  const int KB = args.K / BK;

  if (warp == 0) {
    int carry = 0;
    if (lane == 0) tile_off[0] = 0;
    for (int base = 0; base < E; base += 32) {
      const int e = base + lane;
      int v = e < E ? ((args.mode == 2 ? args.p_T : args.counts[e]) + args.bn - 1) / args.bn : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (e < E) tile_off[e + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 1);   // leader's: one expect_tx arrival + both CTAs' bytes
      mbar_init(&empty[s], 1);  // released by the leader's multicast commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16);  // 8 epilogue warps x 2 CTAs (used on the leader)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  fence_before();
  cluster_sync_all();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int MG = MT / 2;
  const int total = tile_off[E] * MG;
  const int u0 = blockIdx.x / 2, ustep = gridDim.x / 2;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (lane == 0) {
      const uint64_t polB = l2_policy(false);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = u0; t < total; t += ustep) {
        const Tile tl = decode(t, tile_off, E, MG, 2, rank, args);
#ifdef BEAM_DEVICE_CHECKS
        if (args.check != nullptr && args.b_rows > 0 && tl.b_row0 + tl.ntok > args.b_rows) atomicOr(args.check, kChkTile);
#endif
        const uint64_t polA = args.mode == 2 ? polB : a_policy(args.apol, tile_off[tl.e + 1] - tile_off[tl.e] > 1);
        const int half = tl.nmma >> 1;  // token rows staged by each CTA
        const int nbox = (half + kBBox - 1) / kBBox;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t lbar = mapa_u32(smem_u32(&full[stage]), 0);
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * (kABytes + nbox * kBBoxBytes));
          tma_load_2d_2sm(sa + stage * kABytes, &tmA, lbar, kb * BK, tl.a_row0, polA);
          for (int c = 0; c < nbox; ++c)
            tma_load_2d_2sm(sb + stage * kBHalfBytes + c * kBBoxBytes, &tmB, lbar, (kb % args.b_kblocks) * BK,
                            tl.b_row0 + rank * half + c * kBBox, polB);
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    if (lane == 0 && rank == 0) {
      const uint32_t idesc_base = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = u0; t < total; t += ustep) {
        const Tile tl = decode(t, tile_off, E, MG, 2, 0, args);
        const uint32_t idesc = idesc_base | ((uint32_t)(tl.nmma >> 3) << 17);
        const uint32_t tmem_d = tmem_base + acc * BN;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint64_t ad = sdesc_sw128(smem_u32(sa + stage * kABytes));
          const uint64_t bd = sdesc_sw128(smem_u32(sb + stage * kBHalfBytes));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_2sm(tmem_d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit_2sm(&empty[stage]);
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_2sm(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue (both CTAs: own TMEM = own 128 rows) ----------------
    // warps 2-5 and 6-9: two groups covering the 4 TMEM lane quadrants each,
    // alternating 32-token chunks
    const int lane_base = 32 * (warp & 3);
    const int grp = (warp - 2) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = u0; t < total; t += ustep) {
      const Tile tl = decode(t, tile_off, E, MG, 2, rank, args);
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      epilogue_tile(args, tl, tmem_base + ((uint32_t)lane_base << 16) + acc * BN, warp & 3, lane,
                    stg + grp * kStgBytes, 32 * grp, 64, 1 + grp);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(mapa_u32(smem_u32(&tempty[acc]), 0));
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  fence_before();
  cluster_sync_all();
  fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
}

// x_n rows in plan order, bf16 (B operand of GEMM1): X[p] = bf16(h[tok_p] * inv * w).
// One warp per row, every 16-byte chunk of the row loaded before any is written
// (raw registers: 4 per bf16 chunk); without a norm a bf16 row is a plain copy.
template <typename TX>
__global__ void __launch_bounds__(256) pack_x_kernel(const TX* __restrict__ h, const float* __restrict__ inv,
                                                     const float* __restrict__ nw, int d, int d_pad,
                                                     PlanDev p, int cap, __nv_bfloat16* __restrict__ X) {
  extern __shared__ float nws[];  // norm weights (zero-padded to d_pad), shared by all rows
  if (nw)
    for (int k = threadIdx.x; k < d_pad; k += blockDim.x) nws[k] = k < d ? nw[k] : 0.0f;
  __syncthreads();
  griddep_wait();
  const int total = min(p.meta[1], cap);
  BEAM_DCHECK(p, p.meta[1] <= cap, kChkPlanPos);
  const int lane = threadIdx.x & 31;
  constexpr int kL = sizeof(TX) == 2 ? 1 : 2;  // 16-byte loads per 8 elements
  constexpr int kU = sizeof(TX) == 2 ? 8 : 4;  // 8-element chunks per lane in flight
  const bool scale = inv != nullptr || nw != nullptr;
  const int stride = gridDim.x * 8;
  int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  int tok_next = row < total ? p.tok[row] : -1;
  for (; row < total; row += stride) {
    // the next row's token index is in flight while this row is copied (one
    // dependent L2 round trip per row instead of two)
    const int tok = tok_next;
    tok_next = row + stride < total ? p.tok[row + stride] : -1;
    BEAM_DCHECK(p, p.T == 0 || tok < p.T, kChkToken);
    __nv_bfloat16* dst = X + (size_t)row * d_pad;
    if (tok < 0) {
      for (int k = lane * 8; k < d_pad; k += 256) *reinterpret_cast<uint4*>(dst + k) = make_uint4(0, 0, 0, 0);
      continue;
    }
    const float s = inv ? inv[tok] : 1.0f;
    const TX* src = h + (size_t)tok * d_pad;
    for (int k0 = lane * 8; k0 < d_pad; k0 += 256 * kU) {
      uint4 raw[kU][kL];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // all loads first
        const int k = min(k0 + 256 * u, d_pad - 8);
#pragma unroll
        for (int l = 0; l < kL; ++l) raw[u][l] = ld_cached(src + k + 4 * l);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int k = k0 + 256 * u;
        if (k >= d_pad) continue;
        if (sizeof(TX) == 2 && !scale) {
          *reinterpret_cast<uint4*>(dst + k) = raw[u][0];
          continue;
        }
        float x[8];
        if constexpr (kL == 1) {
          unpack<__nv_bfloat16>(raw[u][0], x);
        } else {
          unpack<float>(raw[u][0], x);
          unpack<float>(raw[u][1], x + 4);
        }
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // x_n = (x * inv_rms) * w (tensor.py:487)
          const float g0 = nw ? nws[k + 2 * q] : 1.0f, g1 = nw ? nws[k + 2 * q + 1] : 1.0f;
          const __nv_bfloat162 v2 = __floats2bfloat162_rn((x[2 * q] * s) * g0, (x[2 * q + 1] * s) * g1);
          o[q] = *reinterpret_cast<const uint32_t*>(&v2);
        }
        *reinterpret_cast<uint4*>(dst + k) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tc

// 3-D view (64 columns, rows, cols / 64) of a row-major bf16 [rows, cols] matrix
// with 128-byte swizzling: one box = box_rows rows x all columns, laid out in
// shared memory as [cols / 64][box_rows][64] with the 16-byte chunks of every
// 128-byte row XOR-permuted by (row index mod 8) — ldmatrix-conflict-free.
bool make_tmap_rows_sw128(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  tc::EncodeTiledFn fn = tc::encode_fn();
  if (!fn || cols % 64 != 0 || cols / 64 > 256 || box_rows > 256) return false;
  const cuuint64_t dims[3] = {64, rows, cols / 64};
  const cuuint64_t strides[2] = {cols * 2, 128};
  const cuuint32_t box[3] = {64, box_rows, (cuuint32_t)(cols / 64)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace tc {

static size_t smem_bytes(int E) {
  return 1024 + (size_t)kStages * (kABytes + kBBytes) + kStgBytes + (2 * kStages + 4) * 8 + 16 + (size_t)(E + 1) * 4;
}

}  // namespace tc

bool tc_supported(const beam_layer_t& L, const Dims& g) {
  return L.wdtype == BEAM_BF16 && L.activation == BEAM_ACT_SILU && g.d_pad % 128 == 0 &&
         g.f_pad % 64 == 0 && (2 * g.f_pad) % tc::BM == 0 && g.E <= tc::kMaxE;
}

cudaError_t launch_pack_x(const void* h, int h_dtype, const float* inv, const float* nw, const Dims& g,
                          const PlanDev& p, int cap, void* xperm, cudaStream_t s) {
  // one resident wave (grid-stride rows): a grid sized for 8 CTAs / SM ran in
  // ~2.7 waves at the kernel's 3 resident CTAs / SM
  static int resident[2] = {0, 0};
  int& nb = resident[h_dtype == BEAM_BF16 ? 0 : 1];
  if (nb == 0) {
    if (h_dtype == BEAM_BF16)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tc::pack_x_kernel<__nv_bfloat16>, 256, g.d_pad * sizeof(float));
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tc::pack_x_kernel<float>, 256, g.d_pad * sizeof(float));
    nb = std::max(nb, 1);
  }
  const int grid = std::max(1, std::min(num_sms() * nb, (cap + 7) / 8));
  if (h_dtype == BEAM_BF16)
    launch_pdl(tc::pack_x_kernel<__nv_bfloat16>, grid, 256, g.d_pad * sizeof(float), s, (const __nv_bfloat16*)h, inv, nw, g.d, g.d_pad, p, cap, (__nv_bfloat16*)xperm);
  else
    launch_pdl(tc::pack_x_kernel<float>, grid, 256, g.d_pad * sizeof(float), s, (const float*)h, inv, nw, g.d, g.d_pad, p, cap, (__nv_bfloat16*)xperm);
  count_launches(1);
  return cudaGetLastError();
}

// Persistent launch: one CTA per SM in clusters of CM along M (CM = largest of
// 4, 2, 1 dividing the number of 128-row m-tiles), programmatic serialization
// with the previous kernel when `pdl`.
template <int CM>
static cudaError_t launch_gemm_cm(const CUtensorMap& mA, const CUtensorMap& mB, const tc::Args& a, size_t smem,
                                  bool pdl, cudaStream_t s) {
  using namespace tc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(grouped_gemm_kernel<CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes(kMaxE));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((num_sms() / CM) * CM);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  at[n].id = cudaLaunchAttributeClusterDimension;
  at[n].val.clusterDim.x = CM;
  at[n].val.clusterDim.y = 1;
  at[n].val.clusterDim.z = 1;
  ++n;
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  cudaError_t e = cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<CM>, mA, mB, a);
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

static size_t smem_bytes_2sm(int E) {
  using namespace tc;
  static_assert(1024 + kStages2 * (kABytes + kBHalfBytes) + 2 * kStgBytes + (2 * kStages2 + 4) * 8 + 16 + (kMaxE2 + 1) * 4 <= 227 * 1024,
                "2-SM GEMM shared memory");
  return 1024 + (size_t)kStages2 * (kABytes + kBHalfBytes) + 2 * kStgBytes + (2 * kStages2 + 4) * 8 + 16 +
         (size_t)(E + 1) * 4;
}

static cudaError_t launch_gemm_2sm(const CUtensorMap& mA, const CUtensorMap& mB, const tc::Args& a, bool pdl,
                                   cudaStream_t s) {
  using namespace tc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(grouped_gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes_2sm(kMaxE2));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((num_sms() / 2) * 2);
  cfg.blockDim = dim3(kThreads2);
  cfg.dynamicSmemBytes = smem_bytes_2sm(a.E);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, grouped_gemm_2sm_kernel, mA, mB, a);
  count_launches(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// GEMM kernel choice: 0 = auto (2-SM pairs when the m-tiles pair up), 1 = 1-SM.
static int g_gemm_variant = 0;

static cudaError_t launch_gemm(const CUtensorMap& mA, const CUtensorMap& mB, const tc::Args& a, size_t smem,
                               bool pdl, cudaStream_t s) {
  const int mt = a.m_rows / tc::BM;
  pdl = pdl && pdl_enabled();
  if (g_gemm_variant == 0 && mt % 2 == 0 && a.E <= tc::kMaxE2) return launch_gemm_2sm(mA, mB, a, pdl, s);
  return launch_gemm_cm<1>(mA, mB, a, smem, pdl, s);
}

void set_gemm_variant(int v) { g_gemm_variant = v; }

cudaError_t launch_experts_tc(const beam_layer_t& L, const Dims& g, const void* xperm, const PlanDev& p,
                              int cap, void* act16, void* opair, cudaStream_t s) {
  using namespace tc;
  CUtensorMap mA1, mB1, mA2, mB2;
  if (!make_map(&mA1, L.w_gu, (uint64_t)g.E * 2 * g.f_pad, g.d_pad, BM) ||
      !make_map(&mB1, xperm, (uint64_t)cap, g.d_pad, kBBox) ||
      !make_map(&mA2, L.w_down, (uint64_t)g.E * g.d_pad, g.f_pad, BM) ||
      !make_map(&mB2, act16, (uint64_t)cap, g.f_pad, kBBox))
    return cudaErrorInvalidValue;
  const size_t smem = smem_bytes(g.E);
  static const int apol = [] {
    const char* v = getenv("BEAM_GEMM_APOL");  // tuning knob (a_policy)
    return v ? atoi(v) : 0;
  }();
  static const int epi_direct = [] {  // measured slower than the staged transpose (GEMM2 278 vs 260 us)
    const char* v = getenv("BEAM_EPI_DIRECT");
    return v && v[0] == '1' ? 1 : 0;
  }();
  static const int epi_skip = [] {
    const char* v = getenv("BEAM_EPI_SKIP");  // diagnostics only: invalid results
    return v && v[0] == '1' ? 1 : 0;
  }();
  Args a1{0, g.E, 2 * g.f_pad, g.d_pad, g.d_pad / BK, p.counts, p.offsets, p.w, (__nv_bfloat16*)act16, g.f_pad, opair, g.d_pad, BN, 0, 0, apol, epi_skip, epi_direct, cap, p.check};
  cudaError_t e = launch_gemm(mA1, mB1, a1, smem, true, s);
  if (e != cudaSuccess) return e;
  Args a2{1, g.E, g.d_pad, g.f_pad, g.f_pad / BK, p.counts, p.offsets, p.w, (__nv_bfloat16*)act16, g.f_pad, opair, g.d_pad, BN, 0, 0, apol, epi_skip, epi_direct, cap, p.check};
  return launch_gemm(mA2, mB2, a2, smem, true, s);
}

// ---------------------------------------------------------------------------
// Prefill router / mask-router projection on the tensor cores.
// logits = h . (w_norm o W)^T with h bf16 (exact) and W split into three bf16
// terms W ~= hi + mid + lo (24 significant bits): the three products are exact
// in fp32 and accumulate in fp32, i.e. fp32-accurate routing at bf16
// tensor-core speed.  The three terms are stacked as 3 row blocks of A (M =
// 3 * cols): three split-K partial products [3][T][cols] that the top-K kernel
// sums in order, and three times more work units than one K = 3 d_pad GEMM
// (the tile count, not the FLOPs, bounds this small GEMM).
// ---------------------------------------------------------------------------
__global__ void split_router_kernel(const float* __restrict__ W, const float* __restrict__ nw, int cols, int d,
                                    int d_pad, __nv_bfloat16* __restrict__ A3) {
  const size_t n = (size_t)cols * d_pad;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / d_pad), k = (int)(i % d_pad);
    const float w = W[i] * (nw ? (k < d ? nw[k] : 0.0f) : 1.0f);
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    const float r1 = w - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
    // [3][cols][d_pad]: the three terms are three row blocks (split-K units)
    A3[(size_t)c * d_pad + k] = hi;
    A3[((size_t)cols + c) * d_pad + k] = mid;
    A3[((size_t)2 * cols + c) * d_pad + k] = lo;
  }
}

cudaError_t launch_router_split(const float* gate_wT, const float* norm_w, int cols, int d, int d_pad, void* A3,
                                cudaStream_t s) {
  split_router_kernel<<<std::min(4096, (int)(((size_t)cols * d_pad + 255) / 256)), 256, 0, s>>>(
      gate_wT, norm_w, cols, d, d_pad, reinterpret_cast<__nv_bfloat16*>(A3));
  count_launches(1);
  return cudaGetLastError();
}

bool router_tc_supported(int T, int cols, int d_pad, int x_dtype) {
  return T > 64 && x_dtype == BEAM_BF16 && cols % tc::BM == 0 && d_pad % tc::BK == 0;
}

size_t router_tc_scratch_bytes(int cols, int d_pad) { return (size_t)cols * 3 * d_pad * 2 + 256; }

int router_tc_splits() { return 3; }

// w3: the cached split (beam_layer_t.gate_w3) or NULL (split into `scratch` here)
cudaError_t launch_router_tc(const void* X, const float* norm_w, const float* gate_wT, const void* w3, int T, int cols,
                             int d, int d_pad, float* P, void* scratch, cudaStream_t s) {
  using namespace tc;
  const void* A3 = w3;
  if (A3 == nullptr) {
    cudaError_t e = launch_router_split(gate_wT, norm_w, cols, d, d_pad, scratch, s);
    if (e != cudaSuccess) return e;
    A3 = scratch;
  }
  CUtensorMap mA, mB;
  if (!make_map(&mA, A3, 3ull * cols, d_pad, BM) || !make_map(&mB, X, (uint64_t)T, d_pad, kBBox))
    return cudaErrorInvalidValue;
  // one "expert" of T tokens (count taken from p_T: no device-side plan)
  static const int env_bn = [] {
    const char* v = getenv("BEAM_ROUTER_BN");  // tuning knob
    return v ? atoi(v) : 0;
  }();
  int bn = env_bn >= 16 && env_bn <= BN && env_bn % 16 == 0 ? env_bn : BN;
  Args a{2, 1, 3 * cols, d_pad, d_pad / BK, nullptr, nullptr, nullptr, nullptr, 0, P, 0, bn, cols, T};
  return launch_gemm(mA, mB, a, smem_bytes(1), true, s);
}

}  // namespace beam
