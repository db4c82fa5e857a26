// Internal launcher declarations shared by the .cu translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <utility>

#include "../../include/beam_b200.h"

namespace beam {

// Geometry derived from a beam_layer_t.
struct Dims {
  int d, f, N, K, S, E, Keff, d_pad, f_pad;
};

inline Dims dims_of(const beam_layer_t& L) {
  Dims g;
  g.d = L.d_h;
  g.f = L.d_ff;
  g.N = L.num_experts;
  g.K = L.top_k;
  g.S = L.num_shared;
  g.E = L.num_experts + L.num_shared;
  g.Keff = L.top_k + L.num_shared;
  g.d_pad = (L.d_h + 7) / 8 * 8;
  g.f_pad = (L.d_ff + 15) / 16 * 16;
  return g;
}

// Device-side dispatch plan (all int32 unless noted), carved from workspace.
struct PlanDev {
  int32_t* counts;       // [E]
  int32_t* offsets;      // [E+1] padded exclusive scan
  int32_t* active;       // [E]
  int32_t* meta;         // [4] num_active, padded_total, real_total, flag
  int32_t* tok;          // [cap]
  int32_t* slot;         // [cap]
  float* w;              // [cap] routing weight of each planned position
  int32_t* slot_pos;     // [T*Keff] position of (t,k) in the plan, -1 if dropped
  int32_t* slot_expert;  // [T*Keff] expert of (t,k), -1 if dropped
  // device-checked build (BEAM_DEVICE_CHECKS): allocation bounds of the plan and
  // the flag word violations are ORed into (beam_debug_checks); 0 / null = off
  int cap = 0, T = 0;
  unsigned* check = nullptr;
};

// Arguments of the per-token top-K / softmax / mask step (route_device.cuh).
struct TopkArgs {
  int N, K, S;  // routed experts, top-k, shared experts (always-on slots K..K+S-1)
  float thr;    // keep iff a >= thr
  // routing rule (BEAM_ROUTE_*) and its projection layout: router logits in
  // columns [0, Nr) of a row of `cols` partials, mask pre-activations at mask_off
  // (-1: none)
  int kind = BEAM_ROUTE_BEAM, Nr = 0, cols = 0, mask_off = 0;
  float phi = 0.5f, temp_inv = 1.0f, tau = 0.5f;
  int binarize = 1;
  int has_norm, d, d_pad;
  float* inv_out;  // [T] inverse RMS (for the expert kernels)
  int32_t* ids32;  // [T, K+S] masked ids (int32), -1 = dropped
  float* gw;       // [T, K+S] ghat per slot
  int64_t* topk_ids;
  int64_t* masked_ids;
  float *logits, *weights, *pre_act, *raw_mask, *mask;  // dense [T, N] (optional)
  // fused decode gate only: per-split partial sums of x^2 ([splits][T], from the
  // projection CTAs, replaces the re-read of the token row for inv_rms), and a
  // shared-memory mirror of ids32 / gw (entries t*(K+S)+k < 32) for the plan warp
  const float* ss_part = nullptr;
  int32_t* ids_s = nullptr;
  float* gw_s = nullptr;
  unsigned long long* trace = nullptr;  // diagnostics: %globaltimer at top-K sub-steps of token 0
  // split decode gate: the top-K step also writes the prescaled rows x * norm_w
  // (fp32, stride d_pad) for the weight-streaming expert kernels
  const float* nw = nullptr;
  float* xw_out = nullptr;
};

int num_sms();
cudaError_t record(cudaError_t e);

// Launch with programmatic stream serialization (PDL) so the kernel's launch and
// prologue overlap the previous kernel on the stream.  Kernels launched this way
// call griddep_wait() before reading their predecessor's outputs.
// Programmatic dependent launch on (default) / off (BEAM_NO_PDL=1, diagnostics).
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
void count_launches(int n);  // bookkeeping for beam_kernel_launches()

// gate.cu
cudaError_t launch_pad_rows(const void* h, int h_dtype, int T, int d, int d_pad, void* out,
                            int out_dtype, cudaStream_t s);
cudaError_t launch_rms_norm(const void* h, int h_dtype, int T, int d, const float* norm_w,
                            float* out, cudaStream_t s);
int router_splits(int T, int cols, int d_pad);  // split-K factor of launch_router
cudaError_t launch_router(const void* X, int x_dtype, const float* norm_w, const float* gate_wT,
                          int T, int cols, int d, int d_pad, float* P, cudaStream_t s);
cudaError_t launch_topk_mask(const float* L, int splits, const void* X, int x_dtype, int T,
                             const TopkArgs& a, cudaStream_t s);
bool gate_fused_supported(int T, int N, int E, int d_pad);
cudaError_t launch_gate_fused(const void* X, int x_dtype, const float* norm_w, const float* gate_wT, int T,
                              int d, int d_pad, float* P, const TopkArgs& a, int E, int bs,
                              bool pad, const PlanDev& p, int* counters, cudaStream_t s,
                              float* xw = nullptr);  // xw: [T, d_pad] x * norm_w (fp32) when norm_w is set
cudaError_t launch_mask_route(const int64_t* ids, const void* a, int a_dtype, int T, int K,
                              int N, int64_t* out, cudaStream_t s);
cudaError_t launch_topk_select(const void* logits, int dtype, int T, int N, int K, int64_t* out, cudaStream_t s);

// permute.cu
// scratch: permute_scratch_bytes() bytes, zero-initialised once (multi-CTA path
// for large T*K; the kernels leave it reusable).  nullptr -> single-CTA path.
size_t permute_scratch_bytes(int T, int K, int E);
template <typename IdT>
cudaError_t launch_permute(const IdT* ids, const float* w, int T, int K, int E, int bs,
                           const PlanDev& p, int* scratch, cudaStream_t s);
cudaError_t launch_plan_prepare(const int32_t* counts, const int32_t* offsets,
                                const int32_t* tokens, const int32_t* slots, const int32_t* meta,
                                const float* weights_hat, int T, int K, int N,
                                const PlanDev& p, int32_t* flags, cudaStream_t s);

// experts_simt.cu
// slots: planned (token, slot) entries when the caller knows them (T * Keff),
// -1 = unknown; only prunes the MMA launch, never changes results
// act: [cap, f_pad] rows in the weight dtype (bf16 or fp32) between the two stages
// X16 (optional): the same rows as X in bf16 — the tensor-core items' operand
cudaError_t launch_gateup_simt(const beam_layer_t& L, const Dims& g, const void* X, int x_dtype, int T,
                               const float* inv, const float* nw, const PlanDev& p, void* act,
                               cudaStream_t s, long long slots = -1, const void* X16 = nullptr);
cudaError_t launch_down_simt(const beam_layer_t& L, const Dims& g, int T, const PlanDev& p,
                             const void* act, float* opair, cudaStream_t s, long long slots = -1);
// Decode expert stage on externally routed rows (no norm): gate/up then down.
inline cudaError_t launch_experts_simt(const beam_layer_t& L, const Dims& g, const void* X,
                                       int x_dtype, int T, const PlanDev& p, void* act, float* opair,
                                       cudaStream_t s) {
  cudaError_t e = launch_gateup_simt(L, g, X, x_dtype, T, nullptr, nullptr, p, act, s);
  if (e != cudaSuccess) return e;
  return launch_down_simt(L, g, T, p, act, opair, s);
}

// experts_tc.cu (tcgen05 grouped GEMM, prefill)
bool make_tmap_rows_sw128(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
bool tc_supported(const beam_layer_t& L, const Dims& g);
cudaError_t launch_pack_x(const void* h, int h_dtype, const float* inv, const float* nw, const Dims& g,
                          const PlanDev& p, int cap, void* xperm, cudaStream_t s);
void set_gemm_variant(int v);  // 0 = 2-SM pairs when possible, 1 = 1-SM kernel
bool router_tc_supported(int T, int cols, int d_pad, int x_dtype);
size_t router_tc_scratch_bytes(int cols, int d_pad);
int router_tc_splits();  // split-K partials the tensor-core router writes
cudaError_t launch_router_split(const float* gate_wT, const float* norm_w, int cols, int d, int d_pad, void* A3,
                                cudaStream_t s);
cudaError_t launch_router_tc(const void* X, const float* norm_w, const float* gate_wT, const void* w3, int T, int cols, int d,
                             int d_pad, float* P, void* scratch, cudaStream_t s);
// opair written as bf16 [cap, d_pad] (combine reads it with BEAM_BF16)
cudaError_t launch_experts_tc(const beam_layer_t& L, const Dims& g, const void* xperm, const PlanDev& p,
                              int cap, void* act16, void* opair, cudaStream_t s);

// ep.cu (expert-parallel dispatch / combine halves around the collectives)
int ep_tiles(int T);
cudaError_t launch_ep_count(const int64_t* ids, int T, int K, int N, int world, int n_local, int32_t* tile_counts,
                            cudaStream_t s);
cudaError_t launch_ep_pack(const void* h, int h_dtype, int T, int d, const int64_t* ids, const float* weights, int N,
                           int K, int world, int n_local, int cap, const int32_t* tile_counts, int has_norm,
                           void* x_send, int32_t* meta, int32_t* send_pos, int32_t* counts, cudaStream_t s);
cudaError_t launch_ep_unpack(const int32_t* meta, int n, int K, const void* x, int x_dtype, int d, int d_pad,
                             const float* nw, int32_t* ids32, float* gw, float* inv, float* xw, cudaStream_t s);
cudaError_t launch_ep_combine(const float* y_back, const int32_t* send_pos, int world, int T, int d, const void* h,
                              int h_dtype, void* out, cudaStream_t s);

// combine.cu
cudaError_t launch_combine(const PlanDev& p, const void* opair, int opair_dtype, int T, int Keff, int d, int d_pad,
                           const void* h, int h_dtype, void* out, int out_dtype,
                           cudaStream_t s);

// train.cu (mask-router backward)
cudaError_t launch_candidates(const int64_t* topk, int M, int32_t* ids32, float* gw, cudaStream_t s);
cudaError_t launch_mask_grad(const float* dy, int d, const void* O, int o_dtype, int d_pad,
                             const int32_t* slot_pos, const int64_t* topk, const float* weights,
                             const float* pre_act, int T, int N, int K, float bt, float* grad,
                             float* dghat, cudaStream_t s);
cudaError_t launch_ste_dense(const float* up, const float* w, const float* a, long long n, float bt,
                             float* grad, cudaStream_t s);
cudaError_t launch_sparsity_loss(const float* raw, const int64_t* topk, int T, int N, int K, float* loss,
                                 cudaStream_t s);

// trace.cu (SparsityTrace rows from the gate outputs)
cudaError_t launch_trace_rows(const int64_t* topk, const int64_t* masked, const int64_t* seq,
                              const int64_t* pos, const int64_t* tok, int T, int K, int layer, int phase,
                              int64_t* rows, unsigned long long* active, cudaStream_t s);

cudaError_t set_gate_trace(unsigned long long* buf);

}  // namespace beam
