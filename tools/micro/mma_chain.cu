// tcgen05.mma kind::f16 M=128 K=16 issue probe: cycles per instruction for
// N in {32, 64, 128, 256} when consecutive instructions accumulate into 1, 2
// or 4 independent TMEM accumulators (SS mode, K-major SW128 operands).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_2111_04007_b200/csrc -I include tools/micro/mma_chain.cu
#include <cstdio>
#include "sm100.cuh"
using namespace vp;

template <int n, int chains, int mn_major_b, int mn_major_a = 0, int ts = 0>
__global__ void probe(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sA = smem_u32(sm), sB = smem_u32(sm + 16384);
    const uint32_t id = idesc_bf16(128, n, mn_major_a != 0, mn_major_b != 0);
    // warm-up
    for (int k = 0; k < 4; ++k)
      umma_f16(tmem, sdesc_sw128(sA + k * 32, 16, 1024), sdesc_sw128(sB + k * 32, 16, 1024), id, k > 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int c = 0; c < chains; ++c) {
          const uint64_t bd = mn_major_b ? sdesc_sw128(sB + k * 2048, 16384, 1024)
                                         : sdesc_sw128(sB + k * 32, 16, 1024);
          const uint64_t ad = mn_major_a ? sdesc_sw128(sA + k * 2048, 8192, 1024)
                                         : sdesc_sw128(sA + k * 32, 16, 1024);
          if (ts) umma_f16_ts(tmem + c * n, tmem + 448 + k * 8, bd, id, 1u);
          else umma_f16(tmem + c * n, ad, bd, id, 1u);
        }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 1);
    const unsigned long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int n, int chains, int mn, int mna = 0, int ts = 0>
void run1(unsigned long long* d, int reps) {
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(probe<n, chains, mn, mna, ts>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<n, chains, mn, mna, ts><<<1, 128, smem>>>(reps, d);
  probe<n, chains, mn, mna, ts><<<1, 128, smem>>>(reps, d);
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double inst = 4.0 * reps * chains;
  printf("{\"N\": %d, \"chains\": %d, \"b_mn_major\": %d, \"a_mn_major\": %d, \"ts\": %d, \"clk_per_mma\": %.1f, \"floor\": %d, "
         "\"flop_per_clk\": %.0f}\n", n, chains, mn, mna, ts, cyc / inst, n / 2, 2.0 * 128 * n * 16 * inst / cyc);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int reps = 256;
  run1<32, 1, 0>(d, reps); run1<32, 2, 0>(d, reps); run1<32, 4, 0>(d, reps);
  run1<64, 1, 0>(d, reps); run1<64, 2, 0>(d, reps); run1<64, 4, 0>(d, reps);
  run1<128, 1, 0>(d, reps); run1<128, 2, 0>(d, reps); run1<128, 4, 0>(d, reps);
  run1<256, 1, 0>(d, reps); run1<256, 2, 0>(d, reps);
  run1<32, 1, 1>(d, reps); run1<32, 4, 1>(d, reps);
  run1<64, 1, 1>(d, reps); run1<64, 2, 1>(d, reps); run1<64, 4, 1>(d, reps);
  // the attention backward's operand forms: dQ (A MN-major, B MN-major),
  // dV (A from TMEM, B MN-major), dK (A K-major, B MN-major), S/dP (both K-major)
  run1<64, 1, 1, 1, 0>(d, reps); run1<128, 1, 1, 1, 0>(d, reps);
  run1<64, 1, 1, 0, 1>(d, reps); run1<128, 1, 0, 0, 1>(d, reps); run1<32, 1, 1, 1, 0>(d, reps);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
