// Shared device helpers for the BEAM B200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/beam_b200.h"

namespace beam {

constexpr int kWarp = 32;

__host__ __device__ inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ inline int ceil_div(int x, int m) { return (x + m - 1) / m; }

// ---------------------------------------------------------------------------
// numerics — fp32 restatements of the reference's definitions
// ---------------------------------------------------------------------------

// tensor.py:406-411: two-tail, overflow-free sigmoid.
__device__ __forceinline__ float sigmoid_ref(float x) {
  float z = expf(-fabsf(x));
  float t = 1.0f / (1.0f + z);
  return x >= 0.0f ? t : 1.0f - t;
}

// moe.py:38-39 (silu) / moe.py:42 (identity).
template <int ACT>
__device__ __forceinline__ float activation(float x) {
  if constexpr (ACT == BEAM_ACT_SILU) return x * sigmoid_ref(x);
  else return x;
}

// ---------------------------------------------------------------------------
// 16-byte vector chunks: 8 x bf16 or 4 x f32
// ---------------------------------------------------------------------------

template <typename T> struct Chunk;
template <> struct Chunk<__nv_bfloat16> { static constexpr int kElems = 8; };
template <> struct Chunk<float> { static constexpr int kElems = 4; };

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  // weights are read once per call: don't pollute L1
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_cached(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

template <typename T>
__device__ __forceinline__ void unpack(const uint4& v, float* out);

template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& v, float* out) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

template <>
__device__ __forceinline__ void unpack<float>(const uint4& v, float* out) {
  out[0] = __uint_as_float(v.x);
  out[1] = __uint_as_float(v.y);
  out[2] = __uint_as_float(v.z);
  out[3] = __uint_as_float(v.w);
}

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// (lo, hi) -> one 32-bit word of two bf16 (round to nearest even), lo in the low half
__device__ __forceinline__ uint32_t bf16x2_pack(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ---------------------------------------------------------------------------
// device-checked build (-DBEAM_DEVICE_CHECKS, libbeam_b200_checked.so): index
// bounds the kernels rely on are asserted; a violation ORs `code` into the
// plan's check word (read back by beam_debug_checks) instead of trapping.  The
// substitute for compute-sanitizer memcheck, which this GPU pool does not run.
// ---------------------------------------------------------------------------
enum : unsigned {
  kChkPlanPos = 1u,      // a plan position outside [0, cap)
  kChkExpert = 2u,       // an expert id outside [0, E)
  kChkToken = 4u,        // a token index outside [0, T)
  kChkSlotPos = 8u,      // a combine slot position outside [0, cap)
  kChkTile = 16u,        // a tensor-core tile reaching past the packed rows
  kChkEpRow = 32u,       // an expert-parallel send row outside its buffer
};
#ifdef BEAM_DEVICE_CHECKS
#define BEAM_DCHECK(plan, cond, code)                                    \
  do {                                                                   \
    if ((plan).check != nullptr && !(cond)) atomicOr((plan).check, (code)); \
  } while (0)
#else
#define BEAM_DCHECK(plan, cond, code) \
  do {                                \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// programmatic dependent launch (PDL): kernels of the layer chain are launched
// with programmatic stream serialization, so a kernel's launch and prologue
// overlap its predecessor's tail; griddep_wait() blocks until the predecessor
// grid has completed and its memory is visible (no-op without PDL).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------------------
// warp reductions
// ---------------------------------------------------------------------------

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Two fp32 FMAs in one Blackwell FFMA2 (fma.rn.f32x2): (a0, a1) += (w0, w1) * (x, x).
// Same per-lane rounding as two fmaf calls; the operand pairs are register pairs
// ptxas allocates adjacently (no extra moves in the loops that use it).
__device__ __forceinline__ void ffma2(float& a0, float& a1, float w0, float w1, float x) {
  asm("{\n\t.reg .b64 ra, rw, rx;\n\t"
      "mov.b64 ra, {%0, %1};\n\t"
      "mov.b64 rw, {%2, %3};\n\t"
      "mov.b64 rx, {%4, %4};\n\t"
      "fma.rn.f32x2 ra, rw, rx, ra;\n\t"
      "mov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(w0), "f"(w1), "f"(x));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reduce V per-lane partial sums across the warp with a transpose-reduce
// butterfly (V/2 + V/4 + ... shuffles instead of 5 per value).  On return the
// full sums are in smem_out[0..V) (V must be a power of two).
template <int V>
__device__ __forceinline__ void warp_reduce_to_smem(float (&v)[V], float* smem_out, int lane) {
  int base = 0;
  int cnt = V;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    if (cnt > 1) {
      const int half = cnt >> 1;
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < V / 2; ++i) {
        if (i < half) {
          float send = upper ? v[i] : v[i + half];
          float keep = upper ? v[i + half] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (upper) base += half;
      cnt = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
  // every lane holds cnt (== max(V/32, 1)) finished sums starting at `base`
  if (V >= 32 || (lane & (32 / V - 1)) == 0) {
#pragma unroll
    for (int i = 0; i < (V >= 32 ? V / 32 : 1); ++i) smem_out[base + i] = v[i];
  }
  __syncwarp();
}

}  // namespace beam
