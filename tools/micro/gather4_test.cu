// Probe: TMA tile::gather4 (2-D tensor map, 128-byte swizzle) — which box shape
// it accepts and the shared-memory layout it produces (diagnostics only).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, int r0, int r1, int r2, int r3, int col, uint16_t* out, int nbytes) {
  __shared__ __align__(1024) uint8_t buf[8192];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(nbytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
            su32(buf)),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(su32(&bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 10000000;\n\t@!p bra W;\n\t}" ::"r"(
            su32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  const int R = 64, C = 256;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 1000 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, R * C * 2);
  cudaMalloc(&o, 8192);
  cudaMemcpy(d, h.data(), R * C * 2, cudaMemcpyHostToDevice);
  for (int boxh : {1, 4}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxh};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box h=%d encode=%d\n", boxh, (int)r);
    if (r) continue;
    cudaMemset(o, 0, 8192);
    const int nbytes = 4 * 64 * 2;
    k<<<1, 128>>>(m, 5, 17, 2, 40, 64, o, nbytes);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  launch: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    std::vector<uint16_t> g(nbytes / 2);
    cudaMemcpy(g.data(), o, nbytes, cudaMemcpyDeviceToHost);
    for (int row = 0; row < 4; ++row) {
      printf("  smem row %d:", row);
      for (int ch = 0; ch < 8; ++ch) printf(" %d", g[row * 64 + ch * 8]);
      printf("\n");
    }
  }
  return 0;
}
