// tcgen05.mma issue cost when descriptors change every instruction group:
// (a) one lane issues (if (lane == 0), descriptors in per-thread registers,
//     moved to uniform registers per MMA), (b) the whole warp computes the
// (warp-uniform) descriptors and elect.sync picks the issuing lane inside
// the asm. M=128 N=64 K=16 SS, 8 MMAs per group, base alternating between
// two buffers every group.
#include <cstdio>
#include "sm100.cuh"
using namespace vp;

__device__ __forceinline__ void umma_f16_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}

template <int MODE>
__global__ void probe(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 2 * (16384 + 16384) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t id = idesc_bf16(128, 64, false, true);
  if (threadIdx.x < 32) {
    const bool issuer = MODE == 1 || threadIdx.x == 0;
    if (issuer) {
      const unsigned long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        const uint32_t sA = smem_u32(sm + (r & 1) * 32768), sB = sA + 16384;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = sdesc_sw128(sA + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sB + k * 2048, 8192, 1024);
          if (MODE == 0) umma_f16(tmem + (r & 1) * 64, ad, bd, id, k > 0);
          else umma_f16_elect(tmem + (r & 1) * 64, ad, bd, id, k > 0);
        }
      }
      if (MODE == 0) umma_commit(&bar);
      else umma_commit_elect(&bar);
      mbar_wait(&bar, 0);
      const unsigned long long t1 = clock64();
      if (threadIdx.x == 0) out[0] = t1 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 2 * 32768 + 1024;
  const int reps = 256;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) probe<0><<<1, 128, smem>>>(reps, d);
      else probe<1><<<1, 128, smem>>>(reps, d);
    }
    unsigned long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"mode\": \"%s\", \"clk_per_mma\": %.1f}\n", mode ? "warp+elect" : "single lane",
           cyc / (8.0 * reps));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
