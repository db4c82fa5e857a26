// Sparsity trace rows as a by-product of the gate.
//
// Reference: analysis.SparsityTrace (/root/reference/pkg/src/beamoe/analysis.py:15-86)
// records, per (sequence, position, layer) cell, K rows
//   sequence_id, position, layer, rank (1 = highest weight), expert_id, mask_bit,
//   phase, token_id
// (trainer._record_routes, trainer.py:554-574).  Here the rows are built on the
// device straight from the gate's outputs (topk_ids in rank order, masked_ids =
// -1 where the slot did not execute), one thread per row, plus the executed-slot
// count of the call (integer atomics: order-free, exact) for Avg-K.
#include "beam_common.cuh"
#include "beam_internal.h"

namespace beam {

__global__ void trace_rows_kernel(const int64_t* __restrict__ topk, const int64_t* __restrict__ masked,
                                  const int64_t* __restrict__ seq, const int64_t* __restrict__ pos,
                                  const int64_t* __restrict__ tok, int T, int K, int layer, int phase,
                                  int64_t* __restrict__ rows, unsigned long long* __restrict__ active) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long M = (long long)T * K;
  int bit = 0;
  if (i < M) {
    const long long t = i / K;
    const int r = (int)(i - t * K);
    bit = masked[i] >= 0 ? 1 : 0;
    int64_t* row = rows + i * 8;
    row[0] = seq ? seq[t] : 0;
    row[1] = pos ? pos[t] : t;
    row[2] = layer;
    row[3] = r + 1;
    row[4] = topk[i];
    row[5] = bit;
    row[6] = phase;
    row[7] = tok ? tok[t] : 0;
  }
  if (active) {
    const unsigned n = __popc(__ballot_sync(0xffffffffu, bit));
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(active, (unsigned long long)n);
  }
}

cudaError_t launch_trace_rows(const int64_t* topk, const int64_t* masked, const int64_t* seq,
                              const int64_t* pos, const int64_t* tok, int T, int K, int layer, int phase,
                              int64_t* rows, unsigned long long* active, cudaStream_t s) {
  const long long M = (long long)T * K;
  if (M <= 0) return cudaSuccess;
  trace_rows_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(topk, masked, seq, pos, tok, T, K, layer, phase,
                                                                rows, active);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace beam
