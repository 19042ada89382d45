// TMEM load bandwidth probe: W warps of one CTA repeatedly tcgen05.ld
// 32x32b.x32 (4 KB per warp per load) from their lane quadrant; cycles per
// byte per SM. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -I../../paper_2111_04007_b200/csrc tmem_bw.cu -o tmem_bw
#include <cstdio>
#include "sm100.cuh"
using namespace vp;

__global__ void probe(int iters, int cols_span, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t trow = ((warp & 3) * 32) << 16;
  const uint32_t cbase = (warp >> 2) * 32;
  float acc = 0.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32], w[32];
    const uint32_t c = (cbase + (i * 64) % cols_span) % 512;
    tmem_ld32(tmem + trow + c, v);
    tmem_ld32(tmem + trow + ((c + 256) % 512), w);
    tmem_ld_wait();
#pragma unroll
    for (int k = 0; k < 32; ++k) acc += __uint_as_float(v[k]) + __uint_as_float(w[k]);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4096 * 4);
  const int iters = 4096;
  for (int w : {4, 8, 12, 16}) {
    probe<<<1, 32 * w>>>(iters, 256, d, sink);
    probe<<<1, 32 * w>>>(iters, 256, d, sink);
    unsigned long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = static_cast<double>(iters) * w * 2 * 4096;
    printf("{\"warps\": %d, \"cycles\": %llu, \"bytes_per_clk\": %.1f}\n", w, cyc, bytes / cyc);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
