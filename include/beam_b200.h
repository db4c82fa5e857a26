/*
 * beam_b200.h — C ABI of the B200-native BEAM MoE-layer hot path.
 *
 * The reference (arxiv 2605.14438, package `beamoe`, /root/reference/pkg) has
 * exactly one native plugin boundary on this path: the dispatch backend module
 * (`beamoe.dispatch._kernels`, Cython) registered in `_BACKENDS`
 * (src/beamoe/dispatch/__init__.py:21-44) and exposing
 *     mask_route(topk_ids int64[T,K], mask_logits f64[T,N]) -> int64[T,K]
 *     group_by_expert(ids int64[T,K], num_experts) -> (counts, token_order, slot_order)
 * (src/beamoe/dispatch/_kernels.pyx:17-34, :37-66).  Everything else on the
 * path is Python (beam.py / moe.py / dispatch/__init__.py).  This library
 * replaces that backend AND the Python stages around it:
 *
 *   beam_mask_route        <- _kernels.pyx:17-34       (dispatch.mask_route, __init__.py:55-62)
 *   beam_group_by_expert   <- _kernels.pyx:37-66 + the padding loop of
 *                             dispatch.align_block (__init__.py:89-126)
 *   beam_grouped_execute   <- dispatch.grouped_execute (__init__.py:129-157)
 *                             incl. its contract checks (:143-144, :152-153)
 *   beam_layer_forward     <- beam.beam_block_forward(training=False)
 *                             (beam.py:127-165: rms_norm -> topk_route ->
 *                              mask_forward -> mask_route -> align_block ->
 *                              grouped_execute -> shared experts -> residual)
 *   beam_gate              <- the routing half of the above (moe.topk_route
 *                             moe.py:122-137 + beam.mask_forward beam.py:68-72
 *                             + mask_route) = RouterDecision / MaskDecision
 *   beam_moe_execute       <- the dispatch half of the above for externally
 *                             supplied (masked ids, weights): used by the
 *                             expert-parallel path on each rank.
 *
 * Conventions: all pointers are DEVICE pointers unless stated; every entry
 * launches on `stream` only, never allocates, never synchronises the host, and
 * returns BEAM_OK or a negative status.  Scratch comes from the caller's
 * workspace (size from beam_workspace_bytes); the workspace must be zero-filled
 * once before its first use (it holds grid-completion counters that every call
 * leaves at zero — re-zero it after a failed call).  Results are deterministic
 * and independent of grid size (no floating-point atomics).
 */
#ifndef BEAM_B200_H
#define BEAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* beam_stream_t; /* == cudaStream_t */

enum {
  BEAM_OK = 0,
  BEAM_ERR_ARG = -1,          /* bad pointer / size / dtype                     */
  BEAM_ERR_UNSUPPORTED = -2,  /* shape outside what the kernels were built for  */
  BEAM_ERR_CUDA = -3,         /* a CUDA launch failed (see beam_last_cuda_error) */
  BEAM_ERR_WORKSPACE = -4     /* workspace smaller than beam_workspace_bytes()  */
};

enum { BEAM_F32 = 0, BEAM_BF16 = 1, BEAM_F64 = 2 };
enum { BEAM_ACT_SILU = 0, BEAM_ACT_IDENTITY = 1 };

/* Routing rules of baselines.route (baselines.py:158-283, inference branch). */
enum {
  BEAM_ROUTE_BEAM = 0,    /* binary expert-activation mask (beam)                       */
  BEAM_ROUTE_TOPK = 1,    /* vanilla_topk / topk_reduced (k_small) / topk_pruning (k_infer) */
  BEAM_ROUTE_DYNAMIC = 2, /* moe_dynamic: top-p prefix of the full softmax, mass >= phi     */
  BEAM_ROUTE_ADA = 3,     /* ada_moe: top-K over N + null_count columns, nulls skipped      */
  BEAM_ROUTE_SOFT = 4     /* soft_mask / soft_mask_tempered: sigmoid(a / temp) weights      */
};

/* One routing rule.  gate_wT of the layer holds, per kind: BEAM / SOFT
 * [router N ; mask N] rows, TOPK / DYNAMIC [router N] (mask rows ignored),
 * ADA [router N + null_count] (no mask). */
typedef struct {
  int kind;        /* BEAM_ROUTE_*                                                   */
  int k;           /* candidates per token (k_eff for TOPK; top_k otherwise)         */
  int null_count;  /* ADA: extra router columns                                      */
  float phi;       /* DYNAMIC: probability mass                                     */
  float temp;      /* SOFT: temperature (temp_floor for soft_mask_tempered, else 1) */
  float tau;       /* SOFT: mask threshold probability                              */
  int binarize;    /* SOFT: 1 -> weights * (sigmoid(a/temp) >= tau), masked slots skipped;
                      0 -> weights * sigmoid(a/temp), every candidate executes      */
} beam_route_t;

/* Packed parameters of one BEAM MoE block (moe.py:169-192, beam.py:33-48).
 * Shapes use E = num_experts + num_shared, d_pad = round_up(d_h, 8),
 * f_pad = round_up(d_ff, 16).  Padding entries are zero.
 *   norm_w  f32 [d_h]                 (NULL when has_norm == 0)
 *   gate_wT f32 [2N, d_pad]           rows 0..N-1 = router_w^T, rows N..2N-1 = mask_w^T
 *   w_gu    wdtype [E, 2*f_pad, d_pad] gate/up rows interleaved in 32-row groups:
 *           packed row 32*b + i (i<16) = gate feature 16*b+i, 32*b+16+i = up feature 16*b+i
 *   w_down  wdtype [E, d_pad, f_pad]  (= w_down^T per expert: row = output channel)
 * Experts 0..N-1 are routed, N..E-1 are the shared experts (weight 1.0, added
 * after the routed ones, beam.py:163-164).
 *   gate_w3 (optional, NULL = built per call) bf16 [3, gate_w3_cols, d_pad]: the
 *           prefill tensor-core router's operand, (norm_w o gate_wT rows) split
 *           into hi / mid / lo bf16 terms (beam_router_split), cached at pack time */
typedef struct {
  int d_h, d_ff, num_experts, top_k, num_shared;
  int has_norm;
  int activation;       /* BEAM_ACT_* */
  int wdtype;           /* BEAM_BF16 or BEAM_F32 (expert weights and expert inputs) */
  float mask_threshold; /* keep slot iff pre-activation a >= threshold (0.0f <=> tau = 0.5) */
  const float* norm_w;
  const float* gate_wT;
  const void* w_gu;
  const void* w_down;
  const void* gate_w3;
  int gate_w3_cols;
} beam_layer_t;

/* The three-term bf16 split of the (norm-weighted) projection rows for the
 * prefill tensor-core router: out [3, cols, d_pad] bf16 (hi + mid + lo carry the
 * 24 significant bits of norm_w[k] * gate_wT[c, k]); norm_w may be NULL. */
int beam_router_split(const float* gate_wT, const float* norm_w, int cols, int d, int d_pad, void* out,
                      beam_stream_t stream);

/* Optional outputs of beam_layer_forward (any may be NULL except `out`). */
typedef struct {
  void* out;               /* [T, d_h], dtype of h: h + y                        */
  int64_t* topk_ids;       /* [T, K] rank order (RouterDecision.topk_indices)    */
  float* logits;           /* [T, N] router logits (RouterDecision.logits)       */
  float* weights;          /* [T, N] dense top-K softmax (RouterDecision.weights)*/
  float* pre_activation;   /* [T, N] mask router a (MaskDecision.pre_activation) */
  float* raw_mask;         /* [T, N] sigmoid(a)    (MaskDecision.raw_mask)       */
  float* mask;             /* [T, N] 1.0 iff a >= threshold (MaskDecision.mask)  */
  int64_t* masked_ids;     /* [T, K] dispatch.mask_route output                  */
  void* decision_event;    /* cudaEvent_t (may be NULL): beam_layer_forward[_routed]
                              records it on the stream as soon as every decision
                              output above is complete (after the gate), so a host
                              caller can copy them out while the experts run      */
} beam_outputs_t;

/* Bytes of scratch the entries below need for T tokens, routed-id rows of width
 * K (0 = the layer's top_k + num_shared) and the given block size. */
size_t beam_workspace_bytes(const beam_layer_t* layer, int T, int K, int block_size);

/* beam.beam_block_forward(h, block, training=False, block_size) (beam.py:127-165).
 * h: [T, d_h] of h_dtype (BEAM_F32 or BEAM_BF16). */
int beam_layer_forward(const beam_layer_t* layer, const void* h, int h_dtype, int T,
                       int block_size, const beam_outputs_t* outputs, void* workspace,
                       size_t workspace_bytes, beam_stream_t stream);

/* baselines.block_forward(h, block, strategy, training=False, block_size)
 * (baselines.py:286-323): the routing rule `route` (NULL = BEAM with the layer's
 * mask_threshold), then the same masked permute / grouped experts / combine.
 * Outputs: out; topk_ids [T, k] = RouteResult.candidate_ids; masked_ids [T, k] =
 * kept_ids; logits [T, N (+ null_count)]; weights [T, N] = weights_hat; for BEAM /
 * SOFT pre_activation, raw_mask (sigmoid(a / temp)) and mask (the hard bits). */
int beam_layer_forward_routed(const beam_layer_t* layer, const beam_route_t* route, const void* h,
                              int h_dtype, int T, int block_size, const beam_outputs_t* outputs,
                              void* workspace, size_t workspace_bytes, beam_stream_t stream);
size_t beam_workspace_bytes_routed(const beam_layer_t* layer, const beam_route_t* route, int T,
                                   int block_size);

/* The gating half alone (rms_norm -> topk_route -> mask_forward -> mask_route):
 * fills the decision outputs of `outputs` (outputs->out is ignored). */
int beam_gate(const beam_layer_t* layer, const void* h, int h_dtype, int T,
              const beam_outputs_t* outputs, void* workspace, size_t workspace_bytes,
              beam_stream_t stream);

/* Dispatch half for externally routed tokens (expert-parallel ranks):
 * y[t] = sum over k (ascending expert id) of w[t,k] * E_{ids[t,k]}(x[t])  (ids < 0 skipped).
 * x: [T, d_h] of x_dtype; ids int32 [T, K]; w f32 [T, K]; y f32 [T, d_h]. */
int beam_moe_execute(const beam_layer_t* layer, const void* x, int x_dtype, int T, int K,
                     const int32_t* ids, const float* w, float* y, void* workspace,
                     size_t workspace_bytes, beam_stream_t stream);

/* dispatch.mask_route (_kernels.pyx:17-34): out[t,k] = ids[t,k] if
 * 0 <= ids[t,k] < N and a[t, ids[t,k]] >= 0 else -1.  a: [T, N] of a_dtype
 * (BEAM_F32 or BEAM_F64), NaN -> -1. */
int beam_mask_route(const int64_t* topk_ids, const void* a, int a_dtype, int T, int K, int N,
                    int64_t* out, beam_stream_t stream);

/* moe.topk_select (moe.py:116-119): out[t, :] = argsort(-logits[t], stable)[:K]
 * for logits [T, N] of dtype (BEAM_F32 or BEAM_F64) — value descending, ties to
 * the lower index, -0.0 == +0.0, -inf after every finite value, NaN last
 * (numpy's sort order). */
int beam_topk_select(const void* logits, int dtype, int T, int N, int K, int64_t* out,
                     beam_stream_t stream);

/* dispatch.align_block (group_by_expert _kernels.pyx:37-66 + padding, __init__.py:106-119).
 * ids int64 [T, K] (entries outside [0, N) are ignored).  Outputs (int32):
 *   counts [N]; offsets [N+1] padded exclusive scan (offsets[N] = padded total);
 *   tokens/slots [cap] with cap = T*K + N*(block_size-1): per expert, the real
 *   (token, slot) pairs in ascending flat order then -1 padding;
 *   active [N] ascending ids of experts with counts > 0; meta [4] =
 *   {num_active, padded_total, real_total, 0}. */
int beam_group_by_expert(const int64_t* ids, int T, int K, int N, int block_size,
                         int32_t* counts, int32_t* offsets, int32_t* tokens, int32_t* slots,
                         int32_t* active, int32_t* meta, void* workspace, size_t workspace_bytes,
                         beam_stream_t stream);
/* Scratch for beam_group_by_expert: with at least this many ZERO-INITIALISED
 * bytes (reusable across calls; the kernels leave it zeroed), T*K > 16384 runs
 * the multi-CTA permute that beam_layer_forward uses at prefill sizes; with
 * NULL / fewer bytes the single-CTA permute (same results, bit for bit). */
size_t beam_group_by_expert_workspace_bytes(int T, int K, int N);

/* dispatch.grouped_execute (__init__.py:129-157) on a plan from beam_group_by_expert.
 * x: [T, d_h] of x_dtype, weights_hat f32 [T, N] dense, y f32 [T, d_h].
 * flags int32[2] (may be NULL): flags[0] = nnz(weights_hat) - real_total,
 * flags[1] = 1 if a planned slot has zero weight (the reference's ContractErrors). */
int beam_grouped_execute(const beam_layer_t* layer, const void* x, int x_dtype, int T, int K,
                         int block_size, const int32_t* counts, const int32_t* offsets,
                         const int32_t* tokens, const int32_t* slots, const int32_t* active,
                         const int32_t* meta, const float* weights_hat, float* y, int32_t* flags,
                         void* workspace, size_t workspace_bytes, beam_stream_t stream);

/* tensor.rms_norm / MoEBlock.normalize (tensor.py:485-508, moe.py:214-215):
 * out[t] = h[t] * (mean(h[t]^2) + 1e-6)^-1/2 * norm_w, fp32 out [T, d]. */
int beam_rms_norm(const void* h, int h_dtype, int T, int d, const float* norm_w, float* out,
                  beam_stream_t stream);

/* ---- mask-router training ------------------------------------
 * beam.ste_backward (beam.py:100-124), dense [T, N] f32:
 *   grad = (upstream * weights + beta / (K*T) * [weights > 0]) * s * (1 - s),
 *   s = sigmoid(pre_act) (tensor.py:406-411).  beta < 0 -> BEAM_ERR_ARG
 *   (the reference's ContractError). */
int beam_ste_backward(const float* upstream, const float* weights, const float* pre_act, int T,
                      int N, int K, float beta, float* grad, beam_stream_t stream);
/* beam.sparsity_loss (beam.py:87-97): sum over each token's top-K candidates
 * of raw_mask, / (T*K).  raw_mask f32 [T, N], topk_ids int64 [T, K]; loss f32[1].
 * Deterministic (one CTA, fixed summation order). */
int beam_sparsity_loss(const float* raw_mask, const int64_t* topk_ids, int T, int N, int K,
                       float* loss, beam_stream_t stream);
/* Mask-router backward of beam_block_forward(training=True) (beam.py:146-157):
 * the training forward evaluates EVERY top-K candidate (masked ones included,
 * moe.py:223-279 compute_ids), so for L = sum(out * dy) + beta * sparsity_loss
 *   dghat[t,k] = <dy[t], E_{topk[t,k]}(x_n[t])>            (dL_task/dghat)
 *   grad_pre_act[t,i] = ste_backward(dghat scattered to [T,N], weights, a)
 * One call: gate (fills outputs->topk_ids / weights / pre_activation [/ raw_mask],
 * which must be non-NULL) -> plan over all candidates with unit weights ->
 * experts -> fused slot-dot + closed-form STE kernel.  dy f32 [T, d_h];
 * grad_pre_act f32 [T, N] (exact 0 off the candidate set); dghat f32 [T, K]
 * and loss_reg f32[1] (= sparsity_loss, needs outputs->raw_mask) optional.
 * Workspace: beam_workspace_bytes(layer, T, 0, block_size). */
int beam_mask_backward(const beam_layer_t* layer, const void* h, int h_dtype, int T, const float* dy,
                       float beta, int block_size, const beam_outputs_t* outputs, float* grad_pre_act,
                       float* dghat, float* loss_reg, void* workspace, size_t workspace_bytes,
                       beam_stream_t stream);

/* Sparsity-trace rows of one layer call (analysis.SparsityTrace, analysis.py:15-86;
 * trainer._record_routes, trainer.py:554-574), built on the device from the gate
 * outputs: rows int64 [T*K][8] = {sequence_id, position, layer, rank (1-based),
 * expert_id (= topk_ids), mask_bit (= masked_ids >= 0), phase (0 prefill, 1 decode),
 * token_id}.  sequence_id / position / token_id int64 [T] may be NULL (0, t, 0).
 * active_count (u64, may be NULL) is incremented by the executed slots (Avg-K). */
int beam_trace_rows(const int64_t* topk_ids, const int64_t* masked_ids, const int64_t* sequence_id,
                    const int64_t* position, const int64_t* token_id, int T, int K, int layer, int phase,
                    int64_t* rows, unsigned long long* active_count, beam_stream_t stream);

/* Diagnostics.
 * beam_kernel_launches: kernels this library launched since load.
 * beam_profile_begin/end: record CUDA events on the launch stream at the stage
 * boundaries of the next `max_calls` beam_layer_forward calls; _end syncs on the
 * last one and returns per-stage sums in ms: stage_ms[5] = {gate, permute,
 * experts_gateup, experts_down, combine}. */
unsigned long long beam_kernel_launches(void);
/* Expert-stage kernel choice for beam_layer_forward: 0 = auto (tcgen05 grouped
 * GEMM when bf16 weights and >= 32 tokens per expert on average, else the
 * weight-streaming kernels), 1 = force weight streaming, 2 = force tcgen05. */
int beam_set_expert_path(int mode);
int beam_profile_begin(int max_calls);
int beam_profile_end(float* stage_ms, int* calls);
/* ---- expert parallelism (paper_2605_14438_b200/ep.py; not in the reference,
 * whose PAPER.md:712 lists EP as open).  Rank r of `world` owns experts
 * [r*N/world, (r+1)*N/world).  A send row per (token, destination rank) with at
 * least one surviving slot there (deduplicated); x row = the token's raw h row,
 * meta row = int32[2K+1]: K local ids (-1 = not this rank's / masked) | K ghat
 * (f32 bits) | inv_rms (f32 bits).  FIXED layout (cap > 0, T <= cap <= 256):
 * peer p's rows at [p*cap, p*cap + counts[p]), the rest with ids -1 (no counts
 * exchange, no host sync).  COMPACT layout (cap == 0): peer blocks back to back
 * at offsets from beam_ep_count's per-tile counts [world][beam_ep_tiles(T)].
 * send_pos [world, T] = row of (peer, token) or -1. */
int beam_ep_tiles(int T);
int beam_ep_count(const int64_t* masked_ids, int T, int K, int N, int world, int32_t* tile_counts,
                  beam_stream_t stream);
int beam_ep_pack(const void* h, int h_dtype, int T, int d, const int64_t* masked_ids, const float* weights,
                 int N, int K, int world, int cap, const int32_t* tile_counts, int has_norm, void* x_send,
                 int32_t* meta, int32_t* send_pos, int32_t* counts, beam_stream_t stream);
/* Owner side: the local experts (local->num_experts = N/world, norm_w = the
 * block's RMS weight or has_norm 0) on n received rows -> y f32 [n, d_h]
 * (ghat-weighted, ascending local expert id; no residual).  mode: 0 auto,
 * 1 weight streaming (decode), 2 tcgen05 grouped GEMM. */
size_t beam_ep_workspace_bytes(const beam_layer_t* local, int n, int K, int mode);
int beam_ep_execute(const beam_layer_t* local, const void* x, int x_dtype, int n, int K, const int32_t* meta,
                    int mode, float* y, void* workspace, size_t workspace_bytes, beam_stream_t stream);
/* Token side: out[t] = h[t] + sum over ranks p ascending of y_back[send_pos[p, t]]. */
int beam_ep_combine(const float* y_back, const int32_t* send_pos, int world, int T, int d, const void* h,
                    int h_dtype, void* out, beam_stream_t stream);

/* Fused decode gate phase timestamps (%globaltimer ns) into a device buffer of 16
 * u64 (caller initialises [0],[2] to ~0 and the rest to 0); NULL disables:
 * {first CTA start, last CTA start, first / last projection done,
 *  last top-K tile done, permute done, last top-K tile start, permute start,
 *  token 0: partials summed, top-K selected, softmax done, outputs stored}. */
int beam_trace_gate(unsigned long long* dev_buf);
const char* beam_last_cuda_error(void);
/* Device-checked build (libbeam_b200_checked.so, -DBEAM_DEVICE_CHECKS): index
 * bounds the kernels rely on (plan positions < capacity, token indices < T,
 * expert ids < E, combine slot positions, tensor-core tiles inside the packed
 * rows) are asserted on the device; violations OR a bit into *dev_flag (a
 * zeroed device word; NULL = off).  The regular library returns
 * BEAM_ERR_UNSUPPORTED. */
int beam_debug_checks(unsigned* dev_flag);
/* sizeof the ABI structs (0 beam_layer_t, 1 beam_outputs_t, 2 beam_route_t): lets
 * FFI bindings check their struct mirrors against the compiled library. */
size_t beam_abi_sizeof(int which);
const char* beam_build_info(void);
/* 1 if `p` is page-locked host memory the GPU can address at the same pointer
 * (UVA-mapped), so kernels may write results straight into it (the host-output
 * path of beam_block_forward passes such a buffer as outputs->out). */
int beam_host_mapped(const void* p);

#ifdef __cplusplus
}
#endif
#endif /* BEAM_B200_H */
