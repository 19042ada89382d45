// MUFU throughput probe: tanh.approx.f32 vs ex2.approx.f32 vs rcp.approx,
// 8 warps x 8 independent chains, ops per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/mufu_rate.cu -o tools/micro/mufu_rate
#include <cstdio>
template <int OP>
__global__ void probe(int iters, float* out, unsigned long long* cyc) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0.001f * (threadIdx.x + i);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(v[i]));
      if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; unsigned long long* c; cudaMalloc(&o, 4096 * 4); cudaMalloc(&c, 8);
  const char* names[3] = {"tanh", "ex2", "rcp"};
  for (int threads : {256, 512, 1024}) {
    for (int op = 0; op < 3; ++op) {
      const int iters = 2048;
      for (int rep = 0; rep < 2; ++rep) {
        if (op == 0) probe<0><<<1, threads>>>(iters, o, c);
        if (op == 1) probe<1><<<1, threads>>>(iters, o, c);
        if (op == 2) probe<2><<<1, threads>>>(iters, o, c);
      }
      unsigned long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
      printf("{\"op\": \"%s\", \"threads\": %d, \"ops_per_clk_per_sm\": %.2f}\n", names[op], threads,
             (double)iters * 8 * threads / cyc);
    }
  }
  return 0;
}
