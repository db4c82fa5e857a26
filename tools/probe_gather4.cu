// Probe: does a TMA tile::gather4 load into a SWIZZLE_128B tensor map place 4
// gathered rows in shared memory exactly like a tile load of 4 consecutive rows
// (so a UMMA K-major SW128 operand can be assembled from gathered token rows)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_gather4 tools/probe_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tile_map, const __grid_constant__ CUtensorMap g_map,
                      int r0, const int* rows, uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(2 * 1024) : "memory");
    // (a) tile load: 8 consecutive rows r0..r0+7, 64 columns -> sm[0, 1024)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(sm)),
        "l"(reinterpret_cast<uint64_t>(&tile_map)), "r"(0), "r"(r0), "r"(su32(&bar))
        : "memory");
    // (b) two gather4 loads of rows[0..3] / rows[4..7] -> sm[1024, 1536) / sm[1536, 2048)
    for (int h = 0; h < 2; ++h)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
          "%3, %4, %5, %6}], [%7];" ::"r"(su32(sm + 1024 + 512 * h)),
          "l"(reinterpret_cast<uint64_t>(&g_map)), "r"(0), "r"(rows[4 * h]), "r"(rows[4 * h + 1]), "r"(rows[4 * h + 2]),
          "r"(rows[4 * h + 3]), "r"(su32(&bar))
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
          su32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}

int main() {
  const int R = 64, C = 128;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)((r << 8) | c);
  void* dx;
  cudaMalloc(&dx, h.size() * 2);
  cudaMemcpy(dx, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeTiledFn enc = (EncodeTiledFn)fp;
  const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  const cuuint64_t strides[1] = {(cuuint64_t)C * 2};
  const cuuint32_t estr[2] = {1, 1};
  CUtensorMap tile_map, g1, g4;
  const cuuint32_t box8[2] = {64, 8}, box1[2] = {64, 1}, box4[2] = {64, 4};
  CUresult e1 = enc(&tile_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, strides, box8, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult e2 = enc(&g1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, strides, box1, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult e3 = enc(&g4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, strides, box4, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: tile %d, gather box1 %d, gather box4 %d\n", (int)e1, (int)e2, (int)e3);
  int* drows;
  uint16_t* dout;
  cudaMalloc(&drows, 8 * 4);
  cudaMalloc(&dout, 1024 * 2);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  const int r0 = 16;
  for (int variant = 0; variant < 3; variant += 2) {  // box {64,4} (variant 1) is an illegal instruction: gather4 needs box rows = 1
    // variant 0/1: gather the same consecutive rows (must equal the tile load);
    // variant 2: scattered rows (must equal the tile layout with those rows)
    int rows[8];
    for (int i = 0; i < 8; ++i) rows[i] = variant < 2 ? r0 + i : (i * 7 + 3) % R;
    cudaMemcpy(drows, rows, sizeof(rows), cudaMemcpyHostToDevice);
    const CUtensorMap& gm = variant == 1 ? g4 : g1;
    if ((variant == 1 ? e3 : e2) != CUDA_SUCCESS) {
      printf("variant %d: map not encodable\n", variant);
      continue;
    }
    cudaMemset(dout, 0xff, 2048);
    probe<<<1, 128, 8192>>>(tile_map, gm, r0, drows, dout);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("variant %d: %s\n", variant, cudaGetErrorString(err));
      return 1;
    }
    // out holds sm[0, 2048): [0,512) u16 = tile rows, [512, 1024) = gathered rows
    std::vector<uint16_t> o(1024);
    cudaMemcpy(o.data(), dout, 2048, cudaMemcpyDeviceToHost);
    // expected gathered layout: the tile layout with row i replaced by rows[i]
    int bad = 0;
    for (int i = 0; i < 512; ++i) {
      const uint16_t t = o[i];  // tile: (row r0 + j) << 8 | col
      const int tr = (t >> 8) - r0, tc = t & 0xff;
      const uint16_t want = (uint16_t)((rows[tr] << 8) | tc);
      if (o[512 + i] != want) ++bad;
    }
    printf("variant %d (%s): %d of 512 halfwords differ from the tile layout; first row chunks:", variant,
           variant == 0 ? "box {64,1}, consecutive rows" : variant == 1 ? "box {64,4}, consecutive rows" : "box {64,1}, scattered rows",
           bad);
    for (int k = 0; k < 8; ++k) printf(" %04x/%04x", o[k * 8], o[512 + k * 8]);
    printf("\n");
  }
  return 0;
}
