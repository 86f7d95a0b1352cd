// MUFU.EX2 throughput probe: W warps per CTA, 1 CTA per SM, 32 independent chains per thread
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_bw tools/mufu_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int iters, float* sink, unsigned long long* out) {
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = -0.001f * (threadIdx.x + j);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[j]));
      x[j] = y - 1.0001f;
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += x[j];
  if (s == 1234.5f) sink[0] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  float* s; unsigned long long* d; cudaMalloc(&s, 4); cudaMalloc(&d, 148 * 8);
  const int iters = 1000;
  for (int W : {4, 8, 16}) {
    probe<<<148, W * 32>>>(iters, s, d);
    probe<<<148, W * 32>>>(iters, s, d);
    cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d: %.2f ex2 lanes/clk/SM (%.1f cycles per 32-exp round per warp)\n", W,
           (double)W * 32 * 32 * iters / h, (double)h / iters);
  }
  return 0;
}
