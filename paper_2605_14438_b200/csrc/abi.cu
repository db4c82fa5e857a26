// C ABI entry points (include/beam_b200.h): argument validation, workspace
// carving and the launch sequence of each reference-facing operation.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <vector>

#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

static thread_local char g_last_error[256] = "";

cudaError_t record(cudaError_t e) {
  if (e != cudaSuccess) snprintf(g_last_error, sizeof(g_last_error), "%s", cudaGetErrorString(e));
  return e;
}

static std::atomic<unsigned long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

// Stage timing for beam_layer_forward (diagnostics; see beam_profile_begin).
constexpr int kStageMarks = 6;  // start, gate, permute, gateup, down, combine
struct Profiler {
  bool on = false;
  int max_calls = 0, calls = 0;
  std::vector<cudaEvent_t> ev;
};
static Profiler g_prof;

static void prof_mark(int mark, cudaStream_t s) {
  if (!g_prof.on || g_prof.calls >= g_prof.max_calls) return;
  cudaEventRecord(g_prof.ev[(size_t)g_prof.calls * kStageMarks + mark], s);
  if (mark == kStageMarks - 1) ++g_prof.calls;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// Bump allocator over the caller's workspace (256-byte aligned pieces).
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

// Checked build: the device word violations are ORed into (beam_debug_checks).
static unsigned* g_check_flag = nullptr;

// Expert path choice: 0 = auto, 1 = weight-streaming SIMT, 2 = tcgen05 grouped GEMM.
static std::atomic<int> g_expert_path{0};

static bool use_tc(const beam_layer_t& L, const Dims& g, int T, int Krow) {
  const int mode = g_expert_path.load();
  if (mode == 1 || !tc_supported(L, g)) return false;
  if (mode == 2) return true;
  return (long long)T * Krow >= 32LL * g.E;  // >= 32 tokens per expert on average
}

struct LayerWs {
  bool tc;
  int cap;
  int* counters;   // [64] grid-completion counters (zero-initialised workspace; reset after use)
  int* pscratch;   // multi-CTA permute scratch (its first 64 ints are a counter)
  void* rscratch;  // prefill tensor-core router: bf16 3-way split of the gate weights
  void* xperm;     // [cap, d_pad] bf16 x_n in plan order (tc path)
  void* act16;     // [cap, f_pad] bf16 (tc path)
  void* xpad;      // [T, d_pad] input rows re-strided (only when d_h % 8 != 0)
  float* inv;      // [T] inverse RMS per token
  float* logits2;  // [splits][T][2N] projection partials
  int32_t* ids32;
  float* gw;
  PlanDev plan;
  float* act;
  float* opair;
  float* xw;       // [T, d_pad] x * norm_w, fp32, then the same rows in bf16 (decode: written by the gate)
};

// One layout serves every entry (sized for the largest user, beam_layer_forward).
// x_bytes: element size of the activation rows (4 covers both dtypes).
// force_tc: -1 = the use_tc rule, 0 = weight streaming, 1 = tensor cores (when supported)
static size_t carve(const beam_layer_t& L, int T, int Kids, int bs, void* ws, LayerWs* o, int cols = 0,
                    int force_tc = -1) {
  const Dims g = dims_of(L);
  if (cols < 2 * g.N) cols = 2 * g.N;  // projection columns (router [+ null] [+ mask])
  const int Krow = Kids > g.Keff ? Kids : g.Keff;
  const size_t M = (size_t)T * Krow;
  const size_t cap = M + (size_t)g.E * (size_t)(bs > 0 ? bs - 1 : 0);
  Carver c(ws);
  LayerWs w;
  w.counters = c.take<int>(64);
  w.pscratch = c.take<int>(permute_scratch_bytes(T, Krow, g.E) / sizeof(int));
  w.rscratch = T > 64 ? c.take<char>(router_tc_scratch_bytes(cols, g.d_pad)) : nullptr;
  w.tc = force_tc < 0 ? use_tc(L, g, T, Krow) : (force_tc == 1 && tc_supported(L, g));
  w.cap = (int)cap;
  w.xperm = w.tc ? c.take<__nv_bfloat16>(cap * g.d_pad) : nullptr;
  w.act16 = w.tc ? c.take<__nv_bfloat16>(cap * g.f_pad) : nullptr;
  w.xpad = g.d != g.d_pad ? c.take<float>((size_t)T * g.d_pad) : nullptr;
  w.inv = c.take<float>((size_t)T);
  w.logits2 = c.take<float>((size_t)(T <= 64 ? 16 : 3) * T * cols);  // split-K partials (<= 16 / 3 splits)
  w.ids32 = c.take<int32_t>(M);
  w.gw = c.take<float>(M);
  w.plan.counts = c.take<int32_t>(g.E);
  w.plan.offsets = c.take<int32_t>(g.E + 1);
  w.plan.active = c.take<int32_t>(g.E);
  w.plan.meta = c.take<int32_t>(4);
  w.plan.tok = c.take<int32_t>(cap);
  w.plan.slot = c.take<int32_t>(cap);
  w.plan.w = c.take<float>(cap);
  w.plan.slot_pos = c.take<int32_t>(M);
  w.plan.slot_expert = c.take<int32_t>(M);
  w.plan.cap = (int)cap;
  w.plan.T = T;
  w.plan.check = g_check_flag;
  w.act = w.tc ? nullptr : c.take<float>(cap * g.f_pad);
  w.opair = c.take<float>(cap * g.d_pad);
  w.xw = (T <= 64 && L.has_norm) ? c.take<float>((size_t)T * g.d_pad * 3 / 2 + 4) : nullptr;
  if (o) *o = w;
  return c.off + 256;
}

// Input rows with stride d_pad (a padded copy in the workspace when needed).
static cudaError_t strided_input(const Dims& g, const void* h, int h_dtype, int T, LayerWs& w,
                                 const void** X, cudaStream_t s) {
  if (g.d == g.d_pad) {
    *X = h;
    return cudaSuccess;
  }
  *X = w.xpad;
  return launch_pad_rows(h, h_dtype, T, g.d, g.d_pad, w.xpad, h_dtype, s);
}

// Expert stage on plan `p` for rows X (no norm): the tcgen05 grouped GEMM when
// the workspace was carved for it (w.tc), else weight streaming.  Returns the
// dtype of the per-pair rows in w.opair (the combine's input).
static cudaError_t run_experts(const beam_layer_t& L, const Dims& g, const void* X, int x_dtype, int T,
                               const PlanDev& p, LayerWs& w, int* opair_dtype, cudaStream_t s) {
  cudaError_t e;
  if (w.tc) {
    *opair_dtype = BEAM_BF16;
    if ((e = launch_pack_x(X, x_dtype, nullptr, nullptr, g, p, w.cap, w.xperm, s)) != cudaSuccess) return e;
    return launch_experts_tc(L, g, w.xperm, p, w.cap, w.act16, w.opair, s);
  }
  *opair_dtype = BEAM_F32;
  return launch_experts_simt(L, g, X, x_dtype, T, p, w.act, w.opair, s);
}

static int validate(const beam_layer_t* L) {
  if (!L) return BEAM_ERR_ARG;
  if (L->d_h < 1 || L->d_ff < 1 || L->num_experts < 1 || L->top_k < 1 ||
      L->top_k > L->num_experts || L->num_shared < 0)
    return BEAM_ERR_ARG;
  if (L->wdtype != BEAM_BF16 && L->wdtype != BEAM_F32) return BEAM_ERR_ARG;
  if (L->activation != BEAM_ACT_SILU && L->activation != BEAM_ACT_IDENTITY) return BEAM_ERR_ARG;
  if (L->num_experts > 512 || L->num_experts + L->num_shared > 1024) return BEAM_ERR_UNSUPPORTED;
  if (L->top_k + L->num_shared > 32) return BEAM_ERR_UNSUPPORTED;  // combine: one lane per slot
  if (!L->gate_wT || !L->w_gu || !L->w_down) return BEAM_ERR_ARG;
  if (L->has_norm && !L->norm_w) return BEAM_ERR_ARG;
  return BEAM_OK;
}

static int status(cudaError_t e) { return record(e) == cudaSuccess ? BEAM_OK : BEAM_ERR_CUDA; }

// Decode gate: the fused single-launch gate (gate.cu: projection + top-K +
// permute with last-CTA handoffs) at every decode size it supports; the three
// separate launches (split-K projection, top-K, permute) measured equal or
// slower (B200, L2 flushed, Q30 layer, s = 0 / 0.5: T=8 117.6/85.7 vs
// 117.2/86.1 us, T=16 161.1/116.0 vs 163.2/116.8, T=64 283.3/225.2 vs
// 286.7/229.2; profiles/r02/gate_modes.jsonl).  BEAM_GATE_MODE=fused|split
// forces one (diagnostics).
constexpr int kFusedGateMaxT = 64;
static bool use_fused_gate(int T) {
  static const int m = [] {
    const char* v = getenv("BEAM_GATE_MODE");
    if (v == nullptr) return 0;
    return v[0] == 'f' ? 1 : v[0] == 's' ? 2 : 0;
  }();
  return m == 1 || (m == 0 && T <= kFusedGateMaxT);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("BEAM_NO_PDL");
    return !(v && v[0] == '1');
  }();
  return on;
}

// BEAM_DEBUG_SYNC=1: synchronise after every stage and name the failing one in
// beam_last_cuda_error (diagnostics for asynchronous kernel faults).
static bool debug_sync() {
  static const bool on = [] {
    const char* v = getenv("BEAM_DEBUG_SYNC");
    return v && v[0] == '1';
  }();
  return on;
}

static int status_at(cudaError_t e, const char* what) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(e));
  return BEAM_ERR_CUDA;
}

#define BEAM_TRY(expr)                                           \
  do {                                                           \
    cudaError_t _e = (expr);                                     \
    if (_e != cudaSuccess) return status(_e);                    \
    if (debug_sync()) {                                          \
      _e = cudaDeviceSynchronize();                              \
      if (_e != cudaSuccess) return status_at(_e, #expr);        \
    }                                                            \
  } while (0)

}  // namespace beam

using namespace beam;

extern "C" {

size_t beam_workspace_bytes(const beam_layer_t* layer, int T, int K, int block_size) {
  if (validate(layer) != BEAM_OK || T < 0 || K < 0) return 0;
  return carve(*layer, T, K, block_size < 1 ? 1 : block_size, nullptr, nullptr);
}

// A routing rule resolved against the layer (beam_route_t, NULL = BEAM).
struct Spec {
  int kind = BEAM_ROUTE_BEAM;
  int K = 0, Keff = 0;        // candidates per token, + shared experts
  int Nr = 0, cols = 0, mask_off = 0;
  float phi = 0.5f, temp_inv = 1.0f, tau = 0.5f, thr = 0.0f;
  int binarize = 1;
};

static int spec_of(const beam_layer_t& L, const beam_route_t* r, Spec* sp) {
  const Dims g = dims_of(L);
  Spec s;
  s.thr = L.mask_threshold;
  s.K = g.K;
  s.Nr = g.N;
  s.cols = 2 * g.N;
  s.mask_off = g.N;
  if (r != nullptr) {
    s.kind = r->kind;
    switch (r->kind) {
      case BEAM_ROUTE_BEAM:
        break;
      case BEAM_ROUTE_TOPK:
      case BEAM_ROUTE_DYNAMIC:
        s.K = r->k;
        s.cols = g.N;
        s.mask_off = -1;
        if (r->kind == BEAM_ROUTE_DYNAMIC && !(r->phi > 0.0f && r->phi <= 1.0f)) return BEAM_ERR_ARG;
        s.phi = r->phi;
        break;
      case BEAM_ROUTE_ADA:
        if (r->null_count < 0) return BEAM_ERR_ARG;
        s.K = r->k;
        s.Nr = g.N + r->null_count;
        s.cols = s.Nr;
        s.mask_off = -1;
        break;
      case BEAM_ROUTE_SOFT:
        if (!(r->temp > 0.0f) || !(r->tau > 0.0f && r->tau < 1.0f)) return BEAM_ERR_ARG;
        s.K = r->k;
        s.temp_inv = 1.0f / r->temp;
        s.tau = r->tau;
        s.binarize = r->binarize != 0;
        break;
      default:
        return BEAM_ERR_ARG;
    }
  }
  if (s.K < 1 || s.K > s.Nr || s.Nr > 512) return BEAM_ERR_ARG;
  if (s.K + g.S > 32) return BEAM_ERR_UNSUPPORTED;
  s.Keff = s.K + g.S;
  *sp = s;
  return BEAM_OK;
}

static TopkArgs topk_args(const beam_layer_t& L, const Dims& g, const beam_outputs_t* o, LayerWs& w,
                          const Spec& sp) {
  TopkArgs a;
  a.N = g.N;
  a.K = sp.K;
  a.S = g.S;
  a.thr = sp.thr;
  a.kind = sp.kind;
  a.Nr = sp.Nr;
  a.cols = sp.cols;
  a.mask_off = sp.mask_off;
  a.phi = sp.phi;
  a.temp_inv = sp.temp_inv;
  a.tau = sp.tau;
  a.binarize = sp.binarize;
  a.has_norm = L.has_norm;
  a.d = g.d;
  a.d_pad = g.d_pad;
  a.inv_out = w.inv;
  a.ids32 = w.ids32;
  a.gw = w.gw;
  a.topk_ids = o->topk_ids;
  a.masked_ids = o->masked_ids;
  a.logits = o->logits;
  a.weights = o->weights;
  a.pre_act = o->pre_activation;
  a.raw_mask = o->raw_mask;
  a.mask = o->mask;
  return a;
}

// The gating half shared by beam_layer_forward and beam_gate.
// xw (optional): [T, d_pad] fp32 x * norm_w, written by the top-K step (layer_forward's
// prescaled decode rows)
static cudaError_t run_gate(const beam_layer_t& L, const Dims& g, const void* X, int h_dtype, int T,
                            const beam_outputs_t* o, LayerWs& w, cudaStream_t s, const Spec& sp,
                            float* xw = nullptr) {
  const float* nw = L.has_norm ? L.norm_w : nullptr;
  cudaError_t e;
  int splits;
  if (w.rscratch && router_tc_supported(T, sp.cols, g.d_pad, h_dtype)) {
    const void* w3 = (L.gate_w3 != nullptr && L.gate_w3_cols == sp.cols) ? L.gate_w3 : nullptr;
    e = launch_router_tc(X, nw, L.gate_wT, w3, T, sp.cols, g.d, g.d_pad, w.logits2, w.rscratch, s);
    splits = router_tc_splits();
  } else {
    e = launch_router(X, h_dtype, nw, L.gate_wT, T, sp.cols, g.d, g.d_pad, w.logits2, s);
    splits = router_splits(T, sp.cols, g.d_pad);
  }
  if (e != cudaSuccess) return e;
  TopkArgs ta = topk_args(L, g, o, w, sp);
  if (xw != nullptr && L.has_norm) {
    ta.nw = L.norm_w;
    ta.xw_out = xw;
  }
  return launch_topk_mask(w.logits2, splits, X, h_dtype, T, ta, s);
}

static int layer_forward(const beam_layer_t* layer, const beam_route_t* route, const void* h, int h_dtype, int T,
                         int block_size, const beam_outputs_t* o, void* workspace, size_t workspace_bytes,
                         beam_stream_t stream) {
  int rc = validate(layer);
  if (rc) return rc;
  Spec sp;
  if ((rc = spec_of(*layer, route, &sp)) != BEAM_OK) return rc;
  if (T < 0 || block_size < 1 || !o || !o->out || (T > 0 && !h)) return BEAM_ERR_ARG;
  if (h_dtype != BEAM_F32 && h_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  const beam_layer_t& L = *layer;
  const Dims g = dims_of(L);
  LayerWs w;
  if (carve(L, T, sp.Keff, block_size, workspace, &w, sp.cols) > workspace_bytes || !workspace)
    return BEAM_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const void* X = nullptr;

  prof_mark(0, s);
  BEAM_TRY(strided_input(g, h, h_dtype, T, w, &X, s));
  // decode with an RMS norm: the fused gate also writes x * norm_w (fp32) for the
  // weight-streaming expert kernels
  // decode with an RMS norm: the gate also writes x * norm_w (fp32) for the
  // weight-streaming expert kernels (their tensor-core items need no per-chunk
  // norm multiply)
  const bool fused = use_fused_gate(T) && gate_fused_supported(T, g.N, g.E, g.d_pad);
  const bool prescaled = L.has_norm && w.xw != nullptr && !w.tc;
  if (fused) {
    // small decode batches: projection + top-K + permute in one launch
    BEAM_TRY(launch_gate_fused(X, h_dtype, L.has_norm ? L.norm_w : nullptr, L.gate_wT, T, g.d, g.d_pad,
                               w.logits2, topk_args(L, g, o, w, sp), g.E, block_size, w.tc, w.plan, w.counters, s,
                               prescaled ? w.xw : nullptr));
    prof_mark(1, s);
  } else {
    BEAM_TRY(run_gate(L, g, X, h_dtype, T, o, w, s, sp, prescaled ? w.xw : nullptr));
    prof_mark(1, s);
    BEAM_TRY(launch_permute<int32_t>(w.ids32, w.gw, T, sp.Keff, g.E, block_size, w.plan, w.pscratch, s));
  }
  if (o->decision_event) BEAM_TRY(cudaEventRecord(static_cast<cudaEvent_t>(o->decision_event), s));
  prof_mark(2, s);
  if (w.tc) {
    BEAM_TRY(launch_pack_x(X, h_dtype, L.has_norm ? w.inv : nullptr, L.has_norm ? L.norm_w : nullptr, g,
                           w.plan, w.cap, w.xperm, s));
    BEAM_TRY(launch_experts_tc(L, g, w.xperm, w.plan, w.cap, w.act16, w.opair, s));
    prof_mark(3, s);
    prof_mark(4, s);
  } else {
    if (prescaled)
      BEAM_TRY(launch_gateup_simt(L, g, w.xw, BEAM_F32, T, w.inv, nullptr, w.plan, w.act, s, (long long)T * sp.Keff,
                                  w.xw + (size_t)T * g.d_pad));
    else
      BEAM_TRY(launch_gateup_simt(L, g, X, h_dtype, T, L.has_norm ? w.inv : nullptr,
                                  L.has_norm ? L.norm_w : nullptr, w.plan, w.act, s));
    prof_mark(3, s);
    BEAM_TRY(launch_down_simt(L, g, T, w.plan, w.act, w.opair, s));
    prof_mark(4, s);
  }
  BEAM_TRY(launch_combine(w.plan, w.opair, w.tc ? BEAM_BF16 : BEAM_F32, T, sp.Keff, g.d, g.d_pad, h, h_dtype, o->out, h_dtype, s));
  prof_mark(5, s);
  return BEAM_OK;
}

int beam_layer_forward(const beam_layer_t* layer, const void* h, int h_dtype, int T,
                       int block_size, const beam_outputs_t* o, void* workspace,
                       size_t workspace_bytes, beam_stream_t stream) {
  return layer_forward(layer, nullptr, h, h_dtype, T, block_size, o, workspace, workspace_bytes, stream);
}

int beam_layer_forward_routed(const beam_layer_t* layer, const beam_route_t* route, const void* h,
                              int h_dtype, int T, int block_size, const beam_outputs_t* o,
                              void* workspace, size_t workspace_bytes, beam_stream_t stream) {
  return layer_forward(layer, route, h, h_dtype, T, block_size, o, workspace, workspace_bytes, stream);
}

size_t beam_workspace_bytes_routed(const beam_layer_t* layer, const beam_route_t* route, int T, int block_size) {
  Spec sp;
  if (validate(layer) != BEAM_OK || T < 0 || spec_of(*layer, route, &sp) != BEAM_OK) return 0;
  return carve(*layer, T, sp.Keff, block_size < 1 ? 1 : block_size, nullptr, nullptr, sp.cols);
}

int beam_gate(const beam_layer_t* layer, const void* h, int h_dtype, int T,
              const beam_outputs_t* o, void* workspace, size_t workspace_bytes,
              beam_stream_t stream) {
  int rc = validate(layer);
  if (rc) return rc;
  if (T < 0 || !o || (T > 0 && !h)) return BEAM_ERR_ARG;
  if (h_dtype != BEAM_F32 && h_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  const beam_layer_t& L = *layer;
  const Dims g = dims_of(L);
  LayerWs w;
  if (carve(L, T, 0, 1, workspace, &w) > workspace_bytes || !workspace) return BEAM_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const void* X = nullptr;
  BEAM_TRY(strided_input(g, h, h_dtype, T, w, &X, s));
  Spec sp;
  spec_of(L, nullptr, &sp);
  BEAM_TRY(run_gate(L, g, X, h_dtype, T, o, w, s, sp));
  return BEAM_OK;
}

int beam_moe_execute(const beam_layer_t* layer, const void* x, int x_dtype, int T, int K,
                     const int32_t* ids, const float* wts, float* y, void* workspace,
                     size_t workspace_bytes, beam_stream_t stream) {
  int rc = validate(layer);
  if (rc) return rc;
  if (T < 0 || K < 1 || (T > 0 && (!x || !ids || !wts || !y))) return BEAM_ERR_ARG;
  if (K > 32) return BEAM_ERR_UNSUPPORTED;
  if (x_dtype != BEAM_F32 && x_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  const beam_layer_t& L = *layer;
  const Dims g = dims_of(L);
  LayerWs w;
  if (carve(L, T, K, 1, workspace, &w) > workspace_bytes || !workspace) return BEAM_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const void* X = nullptr;
  BEAM_TRY(strided_input(g, x, x_dtype, T, w, &X, s));
  BEAM_TRY(launch_permute<int32_t>(ids, wts, T, K, g.E, 1, w.plan, w.pscratch, s));
  int od = BEAM_F32;
  BEAM_TRY(run_experts(L, g, X, x_dtype, T, w.plan, w, &od, s));
  BEAM_TRY(launch_combine(w.plan, w.opair, od, T, K, g.d, g.d_pad, nullptr, BEAM_F32, y, BEAM_F32, s));
  return BEAM_OK;
}

// ---------------------------------------------------------------------------
// expert parallelism (ep.cu; paper_2605_14438_b200/ep.py)
// ---------------------------------------------------------------------------
int beam_ep_tiles(int T) { return T > 0 ? ep_tiles(T) : 0; }

int beam_ep_count(const int64_t* masked_ids, int T, int K, int N, int world, int32_t* tile_counts,
                  beam_stream_t stream) {
  if (T < 0 || K < 1 || N < 1 || world < 1 || world > 32 || N % world) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  if (!masked_ids || !tile_counts) return BEAM_ERR_ARG;
  return status(launch_ep_count(masked_ids, T, K, N, world, N / world, tile_counts,
                                reinterpret_cast<cudaStream_t>(stream)));
}

int beam_ep_pack(const void* h, int h_dtype, int T, int d, const int64_t* masked_ids, const float* weights, int N,
                 int K, int world, int cap, const int32_t* tile_counts, int has_norm, void* x_send, int32_t* meta,
                 int32_t* send_pos, int32_t* counts, beam_stream_t stream) {
  if (T < 0 || d < 1 || K < 1 || N < 1 || world < 1 || world > 32 || N % world || cap < 0) return BEAM_ERR_ARG;
  if (h_dtype != BEAM_F32 && h_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (cap > 0 && T > cap) return BEAM_ERR_ARG;
  if (cap > 0 && T > 256) return BEAM_ERR_UNSUPPORTED;  // fixed capacity: decode-sized batches
  if (cap == 0 && T > 0 && !tile_counts) return BEAM_ERR_ARG;
  if (T == 0 && cap == 0) return BEAM_OK;  // (fixed layout with T == 0 still fills its empty blocks)
  if ((T > 0 && (!h || !masked_ids || !weights || !send_pos)) || !x_send || !meta || (cap > 0 && !counts))
    return BEAM_ERR_ARG;
  return status(launch_ep_pack(h, h_dtype, T, d, masked_ids, weights, N, K, world, N / world, cap, tile_counts,
                               has_norm, x_send, meta, send_pos, counts, reinterpret_cast<cudaStream_t>(stream)));
}

static size_t ep_carve(const beam_layer_t& L, int n, int K, int mode, void* ws, LayerWs* o, float** xw) {
  const Dims g = dims_of(L);
  size_t off = carve(L, n, K, 1, ws, o, 0, mode == 1 ? 0 : mode == 2 ? 1 : -1);
  off = (off + 255) & ~size_t(255);
  if (xw) *xw = ws ? reinterpret_cast<float*>(static_cast<char*>(ws) + off) : nullptr;
  return off + (L.has_norm ? (size_t)n * g.d_pad * (sizeof(float) + sizeof(__nv_bfloat16)) : 0) + 256;
}

size_t beam_ep_workspace_bytes(const beam_layer_t* local, int n, int K, int mode) {
  if (validate(local) != BEAM_OK || n < 0 || K < 1 || mode < 0 || mode > 2) return 0;
  LayerWs w;
  return ep_carve(*local, n, K, mode, nullptr, &w, nullptr);
}

int beam_ep_execute(const beam_layer_t* local, const void* x, int x_dtype, int n, int K, const int32_t* meta,
                    int mode, float* y, void* workspace, size_t workspace_bytes, beam_stream_t stream) {
  int rc = validate(local);
  if (rc) return rc;
  if (n < 0 || K < 1 || K > 32 || mode < 0 || mode > 2) return K > 32 ? BEAM_ERR_UNSUPPORTED : BEAM_ERR_ARG;
  if (x_dtype != BEAM_F32 && x_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (local->num_shared != 0) return BEAM_ERR_ARG;
  if (n == 0) return BEAM_OK;
  if (!x || !meta || !y) return BEAM_ERR_ARG;
  const beam_layer_t& L = *local;
  const Dims g = dims_of(L);
  LayerWs w;
  float* xw = nullptr;
  if (!workspace || ep_carve(L, n, K, mode, workspace, &w, &xw) > workspace_bytes) return BEAM_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool prescale = L.has_norm && !w.tc;
  BEAM_TRY(launch_ep_unpack(meta, n, K, x, x_dtype, g.d, g.d_pad, L.norm_w, w.ids32, w.gw, w.inv,
                            prescale ? xw : nullptr, s));
  BEAM_TRY(launch_permute<int32_t>(w.ids32, w.gw, n, K, g.E, 1, w.plan, w.pscratch, s));
  const float* inv = L.has_norm ? w.inv : nullptr;
  if (w.tc) {
    const void* X = nullptr;
    BEAM_TRY(strided_input(g, x, x_dtype, n, w, &X, s));
    BEAM_TRY(launch_pack_x(X, x_dtype, inv, L.has_norm ? L.norm_w : nullptr, g, w.plan, w.cap, w.xperm, s));
    BEAM_TRY(launch_experts_tc(L, g, w.xperm, w.plan, w.cap, w.act16, w.opair, s));
  } else if (prescale) {
    BEAM_TRY(launch_gateup_simt(L, g, xw, BEAM_F32, n, inv, nullptr, w.plan, w.act, s, (long long)n * K,
                                xw + (size_t)n * g.d_pad));
    BEAM_TRY(launch_down_simt(L, g, n, w.plan, w.act, w.opair, s));
  } else {
    const void* X = nullptr;
    BEAM_TRY(strided_input(g, x, x_dtype, n, w, &X, s));
    BEAM_TRY(launch_gateup_simt(L, g, X, x_dtype, n, nullptr, nullptr, w.plan, w.act, s));
    BEAM_TRY(launch_down_simt(L, g, n, w.plan, w.act, w.opair, s));
  }
  BEAM_TRY(launch_combine(w.plan, w.opair, w.tc ? BEAM_BF16 : BEAM_F32, n, K, g.d, g.d_pad, nullptr, BEAM_F32, y,
                          BEAM_F32, s));
  return BEAM_OK;
}

int beam_ep_combine(const float* y_back, const int32_t* send_pos, int world, int T, int d, const void* h,
                    int h_dtype, void* out, beam_stream_t stream) {
  if (world < 1 || world > 32 || T < 0 || d < 1) return BEAM_ERR_ARG;
  if (h_dtype != BEAM_F32 && h_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  if (!send_pos || !h || !out) return BEAM_ERR_ARG;
  return status(launch_ep_combine(y_back, send_pos, world, T, d, h, h_dtype, out,
                                  reinterpret_cast<cudaStream_t>(stream)));
}

int beam_mask_route(const int64_t* topk_ids, const void* a, int a_dtype, int T, int K, int N,
                    int64_t* out, beam_stream_t stream) {
  if (T < 0 || K < 0 || N < 1) return BEAM_ERR_ARG;
  if ((size_t)T * K == 0) return BEAM_OK;
  if (!topk_ids || !a || !out) return BEAM_ERR_ARG;
  if (a_dtype != BEAM_F32 && a_dtype != BEAM_F64) return BEAM_ERR_ARG;
  return status(launch_mask_route(topk_ids, a, a_dtype, T, K, N, out,
                                  reinterpret_cast<cudaStream_t>(stream)));
}

int beam_topk_select(const void* logits, int dtype, int T, int N, int K, int64_t* out, beam_stream_t stream) {
  if (T < 0 || N < 1 || K < 1 || K > N) return BEAM_ERR_ARG;
  if (dtype != BEAM_F32 && dtype != BEAM_F64) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  if (!logits || !out) return BEAM_ERR_ARG;
  return status(launch_topk_select(logits, dtype, T, N, K, out, reinterpret_cast<cudaStream_t>(stream)));
}

int beam_group_by_expert(const int64_t* ids, int T, int K, int N, int block_size,
                         int32_t* counts, int32_t* offsets, int32_t* tokens, int32_t* slots,
                         int32_t* active, int32_t* meta, void* workspace, size_t workspace_bytes,
                         beam_stream_t stream) {
  if (T < 0 || K < 0 || N < 0 || block_size < 1) return BEAM_ERR_ARG;
  if (N > 1024) return BEAM_ERR_UNSUPPORTED;
  if (!offsets || !meta || (N > 0 && (!counts || !active))) return BEAM_ERR_ARG;
  if ((size_t)T * K > 0 && (!ids || !tokens || !slots)) return BEAM_ERR_ARG;
  PlanDev p{};
  p.counts = counts;
  p.offsets = offsets;
  p.active = active;
  p.meta = meta;
  p.tok = tokens;
  p.slot = slots;
  int* scratch = (workspace && workspace_bytes >= permute_scratch_bytes(T, K, N)) ? static_cast<int*>(workspace) : nullptr;
  return status(launch_permute<int64_t>(ids, nullptr, T, K, N, block_size, p, scratch,
                                        reinterpret_cast<cudaStream_t>(stream)));
}

size_t beam_group_by_expert_workspace_bytes(int T, int K, int N) {
  if (T < 0 || K < 0 || N < 0) return 0;
  return permute_scratch_bytes(T, K, N);
}

int beam_grouped_execute(const beam_layer_t* layer, const void* x, int x_dtype, int T, int K,
                         int block_size, const int32_t* counts, const int32_t* offsets,
                         const int32_t* tokens, const int32_t* slots, const int32_t* active,
                         const int32_t* meta, const float* weights_hat, float* y, int32_t* flags,
                         void* workspace, size_t workspace_bytes, beam_stream_t stream) {
  int rc = validate(layer);
  if (rc) return rc;
  if (T < 0 || K < 1 || block_size < 1) return BEAM_ERR_ARG;
  if (K > 32) return BEAM_ERR_UNSUPPORTED;
  if (x_dtype != BEAM_F32 && x_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  if (!x || !counts || !offsets || !tokens || !slots || !active || !meta || !weights_hat || !y)
    return BEAM_ERR_ARG;
  const beam_layer_t& L = *layer;
  const Dims g = dims_of(L);
  LayerWs w;
  if (carve(L, T, K, block_size, workspace, &w) > workspace_bytes || !workspace)
    return BEAM_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PlanDev p = w.plan;
  p.counts = const_cast<int32_t*>(counts);
  p.offsets = const_cast<int32_t*>(offsets);
  p.active = const_cast<int32_t*>(active);
  p.meta = const_cast<int32_t*>(meta);
  p.tok = const_cast<int32_t*>(tokens);
  p.slot = const_cast<int32_t*>(slots);
  const void* X = nullptr;
  BEAM_TRY(strided_input(g, x, x_dtype, T, w, &X, s));
  BEAM_TRY(launch_plan_prepare(counts, offsets, tokens, slots, meta, weights_hat, T, K, g.N, p,
                               flags, s));
  int od = BEAM_F32;
  BEAM_TRY(run_experts(L, g, X, x_dtype, T, p, w, &od, s));
  BEAM_TRY(launch_combine(p, w.opair, od, T, K, g.d, g.d_pad, nullptr, BEAM_F32, y, BEAM_F32, s));
  return BEAM_OK;
}

int beam_ste_backward(const float* upstream, const float* weights, const float* pre_act, int T, int N,
                      int K, float beta, float* grad, beam_stream_t stream) {
  if (!(beta >= 0.0f)) return BEAM_ERR_ARG;  // beam.py:117-118
  if (T < 0 || N < 1 || K < 1) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  if (!upstream || !weights || !pre_act || !grad) return BEAM_ERR_ARG;
  const float bt = (float)((double)beta / ((double)K * (double)T));
  return status(launch_ste_dense(upstream, weights, pre_act, (long long)T * N, bt, grad,
                                 reinterpret_cast<cudaStream_t>(stream)));
}

int beam_sparsity_loss(const float* raw_mask, const int64_t* topk_ids, int T, int N, int K, float* loss,
                       beam_stream_t stream) {
  if (T < 0 || N < 1 || K < 0 || !loss) return BEAM_ERR_ARG;
  if ((size_t)T * K > 0 && (!raw_mask || !topk_ids)) return BEAM_ERR_ARG;
  return status(launch_sparsity_loss(raw_mask, topk_ids, T, N, K, loss, reinterpret_cast<cudaStream_t>(stream)));
}

int beam_mask_backward(const beam_layer_t* layer, const void* h, int h_dtype, int T, const float* dy,
                       float beta, int block_size, const beam_outputs_t* o, float* grad, float* dghat,
                       float* loss_reg, void* workspace, size_t workspace_bytes, beam_stream_t stream) {
  int rc = validate(layer);
  if (rc) return rc;
  if (!(beta >= 0.0f) || T < 0 || block_size < 1 || !o) return BEAM_ERR_ARG;
  if (h_dtype != BEAM_F32 && h_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  if (T > 0 && (!h || !dy || !grad || !o->topk_ids || !o->weights || !o->pre_activation)) return BEAM_ERR_ARG;
  if (loss_reg && !o->raw_mask) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  const beam_layer_t& L = *layer;
  const Dims g = dims_of(L);
  Spec sp;
  spec_of(L, nullptr, &sp);
  LayerWs w;
  if (carve(L, T, sp.Keff, block_size, workspace, &w, sp.cols) > workspace_bytes || !workspace)
    return BEAM_ERR_WORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const void* X = nullptr;
  BEAM_TRY(strided_input(g, h, h_dtype, T, w, &X, s));
  // training forward, routing half (beam.py:141-142): decision + mask outputs
  BEAM_TRY(run_gate(L, g, X, h_dtype, T, o, w, s, sp));
  // every candidate, masked ones included (beam.py:146-157), with unit slot weights
  BEAM_TRY(launch_candidates(o->topk_ids, T * g.K, w.ids32, w.gw, s));
  BEAM_TRY(launch_permute<int32_t>(w.ids32, w.gw, T, g.K, g.E, block_size, w.plan, w.pscratch, s));
  const float* inv = L.has_norm ? w.inv : nullptr;
  const float* nw = L.has_norm ? L.norm_w : nullptr;
  if (w.tc) {
    BEAM_TRY(launch_pack_x(X, h_dtype, inv, nw, g, w.plan, w.cap, w.xperm, s));
    BEAM_TRY(launch_experts_tc(L, g, w.xperm, w.plan, w.cap, w.act16, w.opair, s));
  } else {
    BEAM_TRY(launch_gateup_simt(L, g, X, h_dtype, T, inv, nw, w.plan, w.act, s));
    BEAM_TRY(launch_down_simt(L, g, T, w.plan, w.act, w.opair, s));
  }
  const float bt = (float)((double)beta / ((double)g.K * (double)T));
  BEAM_TRY(launch_mask_grad(dy, g.d, w.opair, w.tc ? BEAM_BF16 : BEAM_F32, g.d_pad, w.plan.slot_pos,
                            o->topk_ids, o->weights, o->pre_activation, T, g.N, g.K, bt, grad, dghat, s));
  if (loss_reg) BEAM_TRY(launch_sparsity_loss(o->raw_mask, o->topk_ids, T, g.N, g.K, loss_reg, s));
  return BEAM_OK;
}

int beam_trace_rows(const int64_t* topk_ids, const int64_t* masked_ids, const int64_t* sequence_id,
                    const int64_t* position, const int64_t* token_id, int T, int K, int layer, int phase,
                    int64_t* rows, unsigned long long* active_count, beam_stream_t stream) {
  if (T < 0 || K < 1 || (phase != 0 && phase != 1)) return BEAM_ERR_ARG;
  if (T > 0 && (!topk_ids || !masked_ids || !rows)) return BEAM_ERR_ARG;
  return status(launch_trace_rows(topk_ids, masked_ids, sequence_id, position, token_id, T, K, layer, phase, rows,
                                  active_count, reinterpret_cast<cudaStream_t>(stream)));
}

int beam_router_split(const float* gate_wT, const float* norm_w, int cols, int d, int d_pad, void* out,
                      beam_stream_t stream) {
  if (!gate_wT || !out || cols < 1 || d < 1 || d_pad < d) return BEAM_ERR_ARG;
  return status(launch_router_split(gate_wT, norm_w, cols, d, d_pad, out, reinterpret_cast<cudaStream_t>(stream)));
}

int beam_rms_norm(const void* h, int h_dtype, int T, int d, const float* norm_w, float* out,
                  beam_stream_t stream) {
  if (T < 0 || d < 1) return BEAM_ERR_ARG;
  if (T == 0) return BEAM_OK;
  if (!h || !norm_w || !out) return BEAM_ERR_ARG;
  if (h_dtype != BEAM_F32 && h_dtype != BEAM_BF16) return BEAM_ERR_ARG;
  return status(launch_rms_norm(h, h_dtype, T, d, norm_w, out, reinterpret_cast<cudaStream_t>(stream)));
}

unsigned long long beam_kernel_launches(void) { return g_launches.load(); }

int beam_set_expert_path(int mode) {
  if (mode < 0 || mode > 3) return BEAM_ERR_ARG;
  g_expert_path.store(mode == 3 ? 2 : mode);
  set_gemm_variant(mode == 3 ? 1 : 0);
  return BEAM_OK;
}

int beam_profile_begin(int max_calls) {
  if (max_calls < 1) return BEAM_ERR_ARG;
  for (cudaEvent_t e : g_prof.ev) cudaEventDestroy(e);
  g_prof.ev.assign((size_t)max_calls * kStageMarks, nullptr);
  for (auto& e : g_prof.ev)
    if (cudaEventCreate(&e) != cudaSuccess) return status(cudaGetLastError());
  g_prof.max_calls = max_calls;
  g_prof.calls = 0;
  g_prof.on = true;
  return BEAM_OK;
}

int beam_profile_end(float* stage_ms, int* calls) {
  if (!g_prof.on) return BEAM_ERR_ARG;
  g_prof.on = false;
  for (int k = 0; k < kStageMarks - 1; ++k) stage_ms[k] = 0.0f;
  if (g_prof.calls > 0) {
    cudaError_t e = cudaEventSynchronize(g_prof.ev[(size_t)g_prof.calls * kStageMarks - 1]);
    if (e != cudaSuccess) return status(e);
  }
  for (int c = 0; c < g_prof.calls; ++c)
    for (int k = 0; k < kStageMarks - 1; ++k) {
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, g_prof.ev[(size_t)c * kStageMarks + k], g_prof.ev[(size_t)c * kStageMarks + k + 1]);
      stage_ms[k] += ms;
    }
  *calls = g_prof.calls;
  for (cudaEvent_t e : g_prof.ev) cudaEventDestroy(e);
  g_prof.ev.clear();
  return BEAM_OK;
}

int beam_trace_gate(unsigned long long* dev_buf) { return status(beam::set_gate_trace(dev_buf)); }

const char* beam_last_cuda_error(void) { return g_last_error; }

int beam_debug_checks(unsigned* dev_flag) {
#ifdef BEAM_DEVICE_CHECKS
  g_check_flag = dev_flag;
  return BEAM_OK;
#else
  (void)dev_flag;
  return BEAM_ERR_UNSUPPORTED;  // only libbeam_b200_checked.so carries the checks
#endif
}

size_t beam_abi_sizeof(int which) {
  switch (which) {
    case 0: return sizeof(beam_layer_t);
    case 1: return sizeof(beam_outputs_t);
    case 2: return sizeof(beam_route_t);
    default: return 0;
  }
}

int beam_host_mapped(const void* p) {
  cudaPointerAttributes a;
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p ? 1 : 0;
}

#define BEAM_STR2(x) #x
#define BEAM_STR(x) BEAM_STR2(x)
const char* beam_build_info(void) {
#ifdef BEAM_DEVICE_CHECKS
  return "beam_b200 sm_100a nvcc " BEAM_STR(__CUDACC_VER_MAJOR__) "." BEAM_STR(__CUDACC_VER_MINOR__) " device-checked";
#else
  return "beam_b200 sm_100a nvcc " BEAM_STR(__CUDACC_VER_MAJOR__) "." BEAM_STR(__CUDACC_VER_MINOR__);
#endif
}

}  // extern "C"
