// Microbenchmark: legacy mma.sync m16n8k16 bf16 latency / throughput, ldmatrix,
// L2 / HBM load latency, shuffle latency on this GPU (diagnostics only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int CHAINS>
__global__ void hmma_kernel(long long* out, int iters, uint32_t seed) {
  float c[CHAINS][4];
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  uint32_t a = seed ^ threadIdx.x, b = seed * 3 + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) mma16816(c[i], a, b, a, b, b, a);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (threadIdx.x % 32 == 0) out[blockIdx.x * 64 + threadIdx.x / 32] = (t1 - t0);
  if (s == 12345.f) out[0] = 1;
}

__global__ void shfl_kernel(long long* out, int iters) {
  float v = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) v += __shfl_xor_sync(0xffffffffu, v, 1);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (v == 1.2345f) out[1] = 1;
}

__global__ void chase_kernel(const int* p, int n, long long* out) {
  int i = 0;
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) i = __ldcg(p + i);
  long long t1 = clock64();
  out[0] = t1 - t0;
  out[1] = i;
}

__global__ void bar_kernel(long long* out, int iters) {
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 1 << 20);
  long long h[64 * 148];
  const int iters = 4096;
  // latency: 1 warp, 1 chain
  hmma_kernel<1><<<1, 32>>>(d, iters, 7);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("HMMA dependent latency: %.1f cyc\n", (double)h[0] / iters);
  hmma_kernel<8><<<1, 32>>>(d, iters, 7);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("HMMA 1 warp 8 chains: %.1f cyc / mma\n", (double)h[0] / iters / 8);
  for (int w : {4, 8, 16, 32}) {
    hmma_kernel<8><<<1, 32 * w>>>(d, iters, 7);
    cudaMemcpy(h, d, 8 * 64, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < w; ++i) mx = h[i] > mx ? h[i] : mx;
    double per_sm = (double)iters * 8 * w / mx;
    printf("HMMA %d warps/SM 8 chains: %.2f mma/cyc/SM = %.0f MAC/cyc/SM\n", w, per_sm, per_sm * 2048);
  }
  shfl_kernel<<<1, 32>>>(d, iters);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("SHFL dependent latency: %.1f cyc\n", (double)h[0] / iters);
  bar_kernel<<<1, 512>>>(d, iters);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads 512 thr: %.1f cyc\n", (double)h[0] / iters);
  // pointer chase: L2 (small ring) and HBM (large stride ring)
  int* p;
  const int n = 1 << 26;  // 256 MB
  cudaMalloc(&p, (size_t)n * 4);
  int* hp = new int[n];
  for (int stride : {64, 1 << 20}) {
    const int m = stride == 64 ? (1 << 14) : 200;  // 4 MB ring (L2) / 200 hops across 256 MB
    for (int i = 0; i < n; ++i) hp[i] = 0;
    for (int k = 0; k < m; ++k) hp[(size_t)k * stride % n] = (int)(((size_t)(k + 1) * stride) % n % ((size_t)m * stride));
    cudaMemcpy(p, hp, (size_t)n * 4, cudaMemcpyHostToDevice);
    chase_kernel<<<1, 1>>>(p, m, d);  // cold
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("load latency cold (%s): %.1f cyc\n", stride == 64 ? "4 MB ring, 256 B stride" : "4 MB stride", (double)h[0] / m);
    chase_kernel<<<1, 1>>>(p, m, d);  // warm
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("load latency warm (%s): %.1f cyc\n", stride == 64 ? "4 MB ring, 256 B stride" : "4 MB stride", (double)h[0] / m);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
