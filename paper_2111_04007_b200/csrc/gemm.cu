// Persistent warp-specialised bf16 GEMM for sm_100a: TMA -> SMEM (128B
// swizzle) -> tcgen05.mma (cta_group::1, UMMA 128xBNx16) -> TMEM (double-
// buffered fp32 accumulator) -> fused epilogue.
//
//   warp 0     : TMA producer (one elected lane)
//   warp 1     : MMA issuer   (one elected lane)
//   warp 2     : TMEM allocator
//   warps 4..7 : epilogue (TMEM lane quadrant = warp % 4)
//
// This is the K1 kernel of DESIGN.md: every dense contraction of a stage's
// forward, recompute and backward (QKV, attention-out, FC1, FC2, LM head;
// dgrad and wgrad). The reference only prices it (sp/calibration.py:219-221).
#include "sm100.cuh"
#include "vpipe.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace vp {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;

// Dropout of the branch output before the residual add (BIAS_RESID only):
// out = resid + dropout(acc + bias), mask of element (row, col) keyed by the
// device-resident seed and the call site's salt (common.cuh, K7).
struct EpiDrop {
  const uint64_t* seed;   // nullptr: no dropout
  uint32_t salt;
  uint32_t thr;
  float scale;
};

template <int NV>
__device__ __forceinline__ void apply_drop(const EpiDrop& d, int64_t row, int64_t col0, int64_t N,
                                           float (&v)[NV]) {
  const uint32_t key = drop_key(d.seed, d.salt);
  const uint64_t p0 = static_cast<uint64_t>(row * N + col0) >> 1;   // N, col0 even
#pragma unroll
  for (int q = 0; q < NV / 2; ++q) {
    const uint32_t k = drop_keep2(key, p0 + q, d.thr);
    v[2 * q] = (k & 1u) ? v[2 * q] * d.scale : 0.f;
    v[2 * q + 1] = (k & 2u) ? v[2 * q + 1] * d.scale : 0.f;
  }
}

struct EpiArgs {
  void* D;
  int64_t ldd;
  const __nv_bfloat16* bias;
  __nv_bfloat16* aux;
  int64_t ldaux;
  EpiDrop drop;
};

template <int BN, int STAGES>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFFSET + 256 + 1024;  // + barriers + align slack
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const EpiArgs& e, int64_t row, int64_t col0,
                                               int64_t M, int64_t N, const uint32_t (&raw)[32]) {
  if (row >= M) return;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]);
  const bool full = (col0 + 32 <= N);
  if constexpr (EPI == VP_EPI_ACC_F32 || EPI == VP_EPI_STORE_F32) {
    float* d = reinterpret_cast<float*>(e.D) + row * e.ldd + col0;
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        if constexpr (EPI == VP_EPI_ACC_F32) {
          float4 p = *reinterpret_cast<const float4*>(d + i);
          o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
        }
        *reinterpret_cast<float4*>(d + i) = o;
      }
    } else {
      for (int i = 0; i < 32 && col0 + i < N; ++i) {
        if constexpr (EPI == VP_EPI_ACC_F32) d[i] += v[i];
        else d[i] = v[i];
      }
    }
    return;
  } else {
    __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(e.D) + row * e.ldd + col0;
    if constexpr (EPI == VP_EPI_BIAS || EPI == VP_EPI_BIAS_GELU || EPI == VP_EPI_BIAS_RESID) {
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 bb = *reinterpret_cast<const uint4*>(e.bias + col0 + i);
          const __nv_bfloat16* bh = reinterpret_cast<const __nv_bfloat16*>(&bb);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[i + j] += __bfloat162float(bh[j]);
        }
      } else {
        for (int i = 0; i < 32 && col0 + i < N; ++i) v[i] += __bfloat162float(e.bias[col0 + i]);
      }
    }
    if constexpr (EPI == VP_EPI_BIAS_GELU) {
      // GELU of the bf16-rounded pre-activation; a saving forward stores
      // gelu'(pre) in aux for the backward's DGELU multiply
      float dg[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        v[i] = gelu_tanh_and_grad(__bfloat162float(__float2bfloat16(v[i])), dg[i]);
      if (e.aux) {
        __nv_bfloat16* a = e.aux + row * e.ldaux + col0;
        if (full) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 o;
            o.x = pack_bf16(dg[i], dg[i + 1]);
            o.y = pack_bf16(dg[i + 2], dg[i + 3]);
            o.z = pack_bf16(dg[i + 4], dg[i + 5]);
            o.w = pack_bf16(dg[i + 6], dg[i + 7]);
            *reinterpret_cast<uint4*>(a + i) = o;
          }
        } else {
          for (int i = 0; i < 32 && col0 + i < N; ++i) a[i] = __float2bfloat16(dg[i]);
        }
      }
    }
    if constexpr (EPI == VP_EPI_BIAS_RESID) {
      if (e.drop.seed != nullptr) apply_drop(e.drop, row, col0, N, v);
    }
    if constexpr (EPI == VP_EPI_BIAS_RESID || EPI == VP_EPI_DGELU || EPI == VP_EPI_RESID) {
      const __nv_bfloat16* a = e.aux + row * e.ldaux + col0;
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 bb = *reinterpret_cast<const uint4*>(a + i);
          const __nv_bfloat16* ah = reinterpret_cast<const __nv_bfloat16*>(&bb);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float x = __bfloat162float(ah[j]);
            if constexpr (EPI == VP_EPI_BIAS_RESID || EPI == VP_EPI_RESID) v[i + j] += x;
            else v[i + j] *= x;  // aux = gelu'(pre), stored by the forward
          }
        }
      } else {
        for (int i = 0; i < 32 && col0 + i < N; ++i) {
          float x = __bfloat162float(a[i]);
          if constexpr (EPI == VP_EPI_BIAS_RESID || EPI == VP_EPI_RESID) v[i] += x;
          else v[i] *= x;
        }
      }
    }
    if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 o;
        o.x = pack_bf16(v[i], v[i + 1]);
        o.y = pack_bf16(v[i + 2], v[i + 3]);
        o.z = pack_bf16(v[i + 4], v[i + 5]);
        o.w = pack_bf16(v[i + 6], v[i + 7]);
        *reinterpret_cast<uint4*>(d + i) = o;
      }
    } else {
      for (int i = 0; i < 32 && col0 + i < N; ++i) d[i] = __float2bfloat16(v[i]);
    }
  }
}

__device__ __forceinline__ void tile_coords(int64_t t, int64_t tiles_m, int64_t tiles_n,
                                            int64_t& mb, int64_t& nb, int64_t G = 8) {
  // Grouped rasterisation: G M-tiles share each sweep over N for L2 reuse of B.
  const int64_t per_group = G * tiles_n;
  const int64_t group = t / per_group;
  const int64_t first_m = group * G;
  const int64_t gsize = min(tiles_m - first_m, G);
  const int64_t r = t % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

template <int BN, int STAGES, int EPI, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                int64_t M, int64_t N, int64_t K, EpiArgs epi) {
  using S = Smem<BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id();
  const int64_t tiles_m = (M + BM - 1) / BM;
  const int64_t tiles_n = (N + BN - 1) / BN;
  const int64_t n_tiles = tiles_m * tiles_n;
  const int64_t n_kb = (K + BK - 1) / BK;
  constexpr uint32_t kTmemCols = 2 * BN;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane_id() == 0) {
      // ===== TMA producer =====
      uint32_t stage = 0, phase = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int64_t mb, nb;
        tile_coords(t, tiles_m, tiles_n, mb, nb);
        const int32_t m0 = static_cast<int32_t>(mb * BM);
        const int32_t n0 = static_cast<int32_t>(nb * BN);
        for (int64_t kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::STAGE_BYTES;
          uint8_t* sb = sa + S::A_BYTES;
          mbar_expect_tx(&full_bar[stage], S::STAGE_BYTES);
          const int32_t k0 = static_cast<int32_t>(kb * BK);
          if constexpr (!A_MN) {
            tma_load_2d(sa, &tmA, &full_bar[stage], k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_2d(sa + c * (64 * BK * 2), &tmA, &full_bar[stage], m0 + 64 * c, k0);
          }
          if constexpr (!B_MN) {
            tma_load_2d(sb, &tmB, &full_bar[stage], k0, n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d(sb + c * (64 * BK * 2), &tmB, &full_bar[stage], n0 + 64 * c, k0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ===== MMA issuer (whole warp; elect.sync issues) =====
      constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
      uint32_t stage = 0, phase = 0;
      uint32_t local = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++local) {
        const uint32_t acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int64_t kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * S::STAGE_BYTES);
          const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: +32 B per 16-element K step inside the 128 B swizzle row.
            // MN-major: +16 rows * 128 B per K step; 64-wide M/N chunks are
            // 64*BK*2 bytes apart (LBO).
            const uint64_t ad = A_MN ? sdesc_sw128(sa + k * 2048, 64 * BK * 2, 1024)
                                     : sdesc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? sdesc_sw128(sb + k * 2048, 64 * BK * 2, 1024)
                                     : sdesc_sw128(sb + k * 32, 16, 1024);
            umma_f16_w(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit_w(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_w(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // ===== Epilogue =====
    const uint32_t q = warp & 3;  // TMEM lane quadrant
    uint32_t local = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++local) {
      int64_t mb, nb;
      tile_coords(t, tiles_m, tiles_n, mb, nb);
      const uint32_t acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int64_t row = mb * BM + q * 32 + lane_id();
      const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        const int64_t col0 = nb * BN + c;
        if (col0 >= N) break;
        uint32_t raw[32];
        tmem_ld32(taddr + c, raw);
        tmem_ld_wait();
        epilogue_chunk<EPI>(epi, row, col0, M, N, raw);
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ===========================================================================
// 2-CTA variant (the default path): a cluster of two SMs computes a 256x256
// tile with tcgen05.mma.cta_group::2 (UMMA 256x256x16). Each CTA loads its
// 128 rows of A and its 128-column half of B (halving per-SM operand
// traffic), the leader CTA issues the MMAs, and each CTA drains its 128-row
// half of the accumulator from its own TMEM. The epilogue stages each
// warp's 32-row sub-tile in 128B-swizzled smem and writes it with TMA
// (bulk store, or bulk reduce-add for fp32 gradient accumulation), so global
// writes are full-line and asynchronous. Split-K (weight gradients with a
// small output and long K) is only used with the reduce-add epilogue.
// ===========================================================================
constexpr int kStages2 = 5;
constexpr int kStageBytes2 = 2 * 128 * BK * 2;        // A half + B half per CTA = 32 KB
constexpr int kEpiWarps2 = 8;                          // 2 per TMEM lane quadrant (column halves)
constexpr int kThreads2 = 128 + 32 * kEpiWarps2;
constexpr int kStagingPerWarp = 8192;                  // 2 x 4 KB epilogue buffers
constexpr int kSmem2 = kStages2 * kStageBytes2 + kEpiWarps2 * kStagingPerWarp + 512 + 1024;
// Per-epilogue pipeline shape: single-output epilogues stage through one
// 4 KB buffer per warp and spend the freed shared memory on a 6th operand
// stage (more TMA bytes in flight: the mainloop of K=1024 tiles otherwise
// waits on L2 latency ~20% of the time); two-buffer epilogues (an aux tile
// prefetched or two outputs) keep 8 KB per warp and 5 stages.
template <int EPI>
struct G2Cfg {
  static constexpr bool kTwoBuf = EPI == VP_EPI_BIAS_GELU || EPI == VP_EPI_BIAS_RESID ||
                                  EPI == VP_EPI_DGELU || EPI == VP_EPI_RESID;
  static constexpr int kStages = kTwoBuf ? 5 : 6;
  static constexpr int kStaging = kTwoBuf ? 8192 : 4096;
  static constexpr int kSmem = kStages * kStageBytes2 + kEpiWarps2 * kStaging + 512 + 1024;
};

struct Epi2 {
  const __nv_bfloat16* bias;
  const __nv_bfloat16* aux_in;  // RESID / DGELU operand
  int64_t ldaux;
  int64_t group;                // rasterisation group (M tiles per N sweep)
  float* colsum_ws;             // optional: per-32-row partial column sums of D (fp32)
  EpiDrop drop;                 // BIAS_RESID: dropout of the branch before the residual add
  int dbg;                      // experiment switches (traced builds only)
};

// Sum of v[0..63] over the 32 lanes (rows) of a warp, scattered so that lane
// l ends with the totals of columns 2l and 2l+1 (5 halving exchange steps:
// 62 shuffles instead of 64 full butterflies).
__device__ __forceinline__ float2 warp_colsum64(const float (&v)[64], uint32_t lane) {
  float t[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const bool hi = lane & 16;
    const float send = hi ? v[i] : v[i + 32];
    const float keep = hi ? v[i + 32] : v[i];
    t[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int w = 16, bit = 8; w >= 2; w >>= 1, bit >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const bool hi = lane & bit;
      const float send = hi ? t[i] : t[i + w];
      const float keep = hi ? t[i + w] : t[i];
      t[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
  return make_float2(t[0], t[1]);
}

__device__ __forceinline__ void store_row_swizzled(uint8_t* buf, uint32_t row,
                                                   const uint4 (&chunks)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
    *reinterpret_cast<uint4*>(buf + row * 128 + ((k ^ (row & 7)) << 4)) = chunks[k];
}

template <int EPI>
__device__ __forceinline__ void epi2_apply(const Epi2& e, int64_t row, int64_t col0, int64_t M,
                                           int64_t N, float (&v)[64], float (&pre)[64],
                                           const float (&xin)[64]) {
  // bias (columns col0..col0+63), guarded for the ragged right edge
  if constexpr (EPI == VP_EPI_BIAS || EPI == VP_EPI_BIAS_GELU || EPI == VP_EPI_BIAS_RESID) {
    if (col0 + 64 <= N) {
#pragma unroll
      for (int i = 0; i < 64; i += 8) {
        float b[8];
        unpack8(*reinterpret_cast<const uint4*>(e.bias + col0 + i), b);
#pragma unroll
        for (int j = 0; j < 8; j += 2)
          f2unpack(fadd2(f2pack(v[i + j], v[i + j + 1]), f2pack(b[j], b[j + 1])), v[i + j],
                   v[i + j + 1]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (col0 + i < N) v[i] += __bfloat162float(e.bias[col0 + i]);
    }
  }
  if constexpr (EPI == VP_EPI_BIAS_GELU) {
    // GELU of the bf16-rounded pre-activation; the saving forward also keeps
    // gelu'(pre) (-> aux) so the backward's DGELU epilogue is one multiply
    // (two columns per FFMA2 / FMUL2; the pre-activation rounded to bf16 by
    // one cvt per pair)
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      const __nv_bfloat162 r = __floats2bfloat162_rn(v[i], v[i + 1]);
      const uint32_t rb = *reinterpret_cast<const uint32_t*>(&r);
      const uint64_t x = f2pack(__uint_as_float(rb << 16), __uint_as_float(rb & 0xFFFF0000u));
      if (e.aux_in != nullptr) {
        uint64_t dg;
        f2unpack(gelu_tanh_and_grad2(x, dg), v[i], v[i + 1]);
        f2unpack(dg, pre[i], pre[i + 1]);
      } else {
        f2unpack(gelu_tanh2(x), v[i], v[i + 1]);
      }
    }
  }
  if constexpr (EPI == VP_EPI_BIAS_RESID) {
    if (e.drop.seed != nullptr) apply_drop(e.drop, row, col0, N, v);
  }
  if constexpr (EPI == VP_EPI_BIAS_RESID || EPI == VP_EPI_DGELU || EPI == VP_EPI_RESID) {
    // aux row values were staged in smem by TMA (see gemm2_kernel)
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if constexpr (EPI == VP_EPI_DGELU) v[i] *= xin[i];  // aux = gelu'(pre)
      else v[i] += xin[i];
    }
  }
}

__device__ __forceinline__ void load_row_swizzled(const uint8_t* buf, uint32_t row, float (&x)[64]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(buf + row * 128 + ((k ^ (row & 7)) << 4)), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[8 * k + j] = f[j];
  }
}

#ifdef VP_GEMM_TRACE
__device__ unsigned long long g_vp_gemm_trace[296][4];
// epilogue warp 4 of each CTA: [0] tfull wait, [1] TMEM loads, [2] math,
// [3] staging-buffer waits, [4] smem stores + TMA issue, [5] total
__device__ unsigned long long g_vp_gemm_etrace[296][6];
#define ETR(slot, t) do { if (warp == 4 && lane == 0) et[slot] += clock64() - (t); } while (0)
#else
#define ETR(slot, t) do {} while (0)
#endif
template <int EPI, bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX,
                 int64_t M, int64_t N, int64_t K, int split_k, Epi2 epi) {
  using C = G2Cfg<EPI>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* staging = smem + C::kStages * kStageBytes2;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + kEpiWarps2 * C::kStaging);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tfull_bar = empty_bar + C::kStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;        // [2] (leader's are used)
  uint64_t* aux_bar = tempty_bar + 2;          // [kEpiWarps2][2] aux-tile TMA prefetch
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + 2 * kEpiWarps2);

  constexpr bool kF32Out = (EPI == VP_EPI_ACC_F32 || EPI == VP_EPI_STORE_F32);
  constexpr bool kAuxIn = (EPI == VP_EPI_BIAS_RESID || EPI == VP_EPI_DGELU || EPI == VP_EPI_RESID);
  const uint32_t warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t tiles_m = (M + 255) / 256;
  const int64_t tiles_n = (N + 255) / 256;
  const int64_t n_tiles = tiles_m * tiles_n;
  const int64_t n_kb = (K + BK - 1) / BK;
  const int64_t kb_per = (n_kb + split_k - 1) / split_k;
  const int64_t n_units = n_tiles * split_k;
  const int64_t cid = blockIdx.x >> 1;
  const int64_t n_clusters = gridDim.x >> 1;

  if (warp == 0 && lane_id() == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmD);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * kEpiWarps2);
    }
    for (int a = 0; a < 2 * kEpiWarps2; ++a) mbar_init(&aux_bar[a], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto unit_coords = [&](int64_t u, int64_t& mb, int64_t& nb, int64_t& kb0, int64_t& kb1) {
    const int64_t t = u / split_k, ks = u % split_k;
    tile_coords(t, tiles_m, tiles_n, mb, nb, epi.group);
    kb0 = ks * kb_per;
    kb1 = min(n_kb, kb0 + kb_per);
  };

  if (warp == 0) {
    {
      // ===== TMA producer (both CTAs; whole warp, elect.sync issues) =====
      uint32_t stage = 0, phase = 0;
      for (int64_t u = cid; u < n_units; u += n_clusters) {
        int64_t mb, nb, kb0, kb1;
        unit_coords(u, mb, nb, kb0, kb1);
        const int32_t m0 = static_cast<int32_t>(mb * 256 + rank * 128);
        const int32_t n0 = static_cast<int32_t>(nb * 256 + rank * 128);
        for (int64_t kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * kStageBytes2;
          uint8_t* sb = sa + 128 * BK * 2;
          if (leader) mbar_expect_tx_w(&full_bar[stage], 2 * kStageBytes2);
          const int32_t k0 = static_cast<int32_t>(kb * BK);
          if constexpr (!A_MN) {
            tma_load_2d_2sm_w(sa, &tmA, &full_bar[stage], k0, m0);
          } else {
            tma_load_2d_2sm_w(sa, &tmA, &full_bar[stage], m0, k0);
            tma_load_2d_2sm_w(sa + 64 * BK * 2, &tmA, &full_bar[stage], m0 + 64, k0);
          }
          if constexpr (!B_MN) {
            tma_load_2d_2sm_w(sb, &tmB, &full_bar[stage], k0, n0);
          } else {
            tma_load_2d_2sm_w(sb, &tmB, &full_bar[stage], n0, k0);
            tma_load_2d_2sm_w(sb + 64 * BK * 2, &tmB, &full_bar[stage], n0 + 64, k0);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer (leader CTA only; whole warp, elect.sync issues) =====
      constexpr uint32_t idesc = idesc_bf16(256, 256, A_MN, B_MN);
      uint32_t stage = 0, phase = 0, local = 0;
#ifdef VP_GEMM_TRACE
      unsigned long long w_full = 0, w_tempty = 0, t_begin = clock64();
#endif
      for (int64_t u = cid; u < n_units; u += n_clusters, ++local) {
        int64_t mb, nb, kb0, kb1;
        unit_coords(u, mb, nb, kb0, kb1);
        const uint32_t acc = local & 1;
#ifdef VP_GEMM_TRACE
        unsigned long long t0 = clock64();
#endif
        mbar_wait(&tempty_bar[acc], ((local >> 1) & 1) ^ 1);
#ifdef VP_GEMM_TRACE
        w_tempty += clock64() - t0;
#endif
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * 256;
        for (int64_t kb = kb0; kb < kb1; ++kb) {
#ifdef VP_GEMM_TRACE
          unsigned long long t1 = clock64();
#endif
          mbar_wait(&full_bar[stage], phase);
#ifdef VP_GEMM_TRACE
          w_full += clock64() - t1;
#endif
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes2);
          const uint32_t sb = sa + 128 * BK * 2;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? sdesc_sw128(sa + k * 2048, 64 * BK * 2, 1024)
                                     : sdesc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? sdesc_sw128(sb + k * 2048, 64 * BK * 2, 1024)
                                     : sdesc_sw128(sb + k * 32, 16, 1024);
            umma_f16_2sm_w(tmem_d, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit_2sm_w(&empty_bar[stage], 0x3);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_w(&tfull_bar[acc], 0x3);
      }
#ifdef VP_GEMM_TRACE
      g_vp_gemm_trace[blockIdx.x][0] = w_full;
      g_vp_gemm_trace[blockIdx.x][1] = w_tempty;
      g_vp_gemm_trace[blockIdx.x][2] = clock64() - t_begin;
      g_vp_gemm_trace[blockIdx.x][3] = local;
#endif
    }
  } else if (warp >= 4) {
    // ===== Epilogue (both CTAs): rows [rank*128 + q*32, +32) of the tile,
    // columns [half*128, +128) =====
    const uint32_t q = warp & 3;
    const uint32_t half = (warp - 4) >> 2;
    uint8_t* wbuf = staging + (warp - 4) * C::kStaging;
    uint32_t local = 0, nbuf = 0;
    uint32_t aux_phase = 0;  // parity of the two aux-prefetch barriers of this warp
    const uint32_t lane = lane_id();
    unsigned long long et[6] = {0, 0, 0, 0, 0, 0};
    const unsigned long long e_begin = clock64();
    (void)et; (void)e_begin;
    for (int64_t u = cid; u < n_units; u += n_clusters, ++local) {
      int64_t mb, nb, kb0, kb1;
      unit_coords(u, mb, nb, kb0, kb1);
      const uint32_t acc = local & 1;
      unsigned long long tq = clock64();
      mbar_wait(&tfull_bar[acc], (local >> 1) & 1);
      ETR(0, tq);
      tc_fence_after();
      const int32_t row0 = static_cast<int32_t>(mb * 256 + rank * 128 + q * 32);
      const int64_t row = row0 + lane;
      const uint32_t taddr = tmem_base + ((q * 32) << 16) + acc * 256;
      if constexpr (kF32Out) {
#pragma unroll 1
        for (int c = half * 128; c < half * 128 + 128; c += 32) {
          const int32_t col0 = static_cast<int32_t>(nb * 256 + c);
          if (col0 >= N) break;
          uint32_t raw[32];
          tmem_ld32(taddr + c, raw);
          tmem_ld_wait();
          uint8_t* buf = wbuf + (C::kTwoBuf ? (nbuf & 1) * 4096 : 0);
          if (lane == 0) {
            if constexpr (C::kTwoBuf) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          uint4 ch[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ch[k] = make_uint4(raw[4 * k], raw[4 * k + 1], raw[4 * k + 2], raw[4 * k + 3]);
          store_row_swizzled(buf, lane, ch);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            if constexpr (EPI == VP_EPI_ACC_F32) tma_reduce_add_2d(&tmD, buf, col0, row0);
            else tma_store_2d(&tmD, buf, col0, row0);
            bulk_commit();
          }
          ++nbuf;
        }
      } else {
        uint64_t* abar = aux_bar + 2 * (warp - 4);
        if constexpr (kAuxIn) {
          // Prefetch this warp's two 32x64 aux sub-tiles into its staging
          // buffers (they are overwritten in place by the outputs below).
          if (lane == 0) {
            bulk_wait_read<0>();
#pragma unroll
            for (int ci = 0; ci < 2; ++ci) {
              const int32_t col0 = static_cast<int32_t>(nb * 256 + half * 128 + ci * 64);
              if (col0 < N) {
                mbar_expect_tx(&abar[ci], 4096);
                tma_load_2d(wbuf + ci * 4096, &tmX, &abar[ci], col0, row0);
              }
            }
          }
          __syncwarp();
        }
#pragma unroll 1
        for (int ci = 0; ci < 2; ++ci) {
          const int c = half * 128 + ci * 64;
          const int32_t col0 = static_cast<int32_t>(nb * 256 + c);
          if (col0 >= N) break;
          unsigned long long tq = clock64();
          float v[64], pre[64], xin[64];
          {
            uint32_t raw[32];
            tmem_ld32(taddr + c, raw);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]);
            tmem_ld32(taddr + c + 32, raw);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[32 + i] = __uint_as_float(raw[i]);
          }
          ETR(1, tq);
          tq = clock64();
          if constexpr (kAuxIn) {
            // per-chunk phase: a ragged last N tile skips chunks (and their
            // prefetch), so the barrier phase is not the tile count
            mbar_wait(&abar[ci], (aux_phase >> ci) & 1u);
            aux_phase ^= 1u << ci;
            load_row_swizzled(wbuf + ci * 4096, lane, xin);
            __syncwarp();  // every lane has read its aux row before outputs overwrite it
          }
#ifdef VP_GEMM_TRACE
          if (epi.dbg & 1) {
#pragma unroll
            for (int i = 0; i < 64; ++i) pre[i] = v[i];
          } else
#endif
          epi2_apply<EPI>(epi, row, col0, M, N, v, pre, xin);
#ifdef VP_GEMM_TRACE
          if (warp == 4) {  // make the math complete before the stamp
            float z = 0.f;
#pragma unroll
            for (int i = 0; i < 64; ++i) z += v[i] + pre[i];
            if (z == 12345.678f) v[0] = z;
          }
#endif
          ETR(2, tq);
          if (epi.colsum_ws != nullptr) {
            // fused bias gradient: this warp's 32-row partial sums of the
            // 64 output columns -> colsum_ws[row0 / 32][col]
            if (row >= M) {
#pragma unroll
              for (int i = 0; i < 64; ++i) v[i] = 0.f;
            }
            const float2 cs = warp_colsum64(v, lane);
            const int64_t c = col0 + 2 * lane;
            if (c < N && row0 < M)
              *reinterpret_cast<float2*>(epi.colsum_ws + (row0 >> 5) * N + c) = cs;
          }
          if (EPI == VP_EPI_BIAS_GELU && epi.aux_in != nullptr) {
            // pre-activation (aux) then activation (D): both buffers in turn
            tq = clock64();
            if (lane == 0) bulk_wait_read<0>();
            __syncwarp();
            ETR(3, tq);
            tq = clock64();
            uint4 ch[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              float f[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) f[j] = pre[8 * k + j];
              ch[k] = pack8(f);
            }
            store_row_swizzled(wbuf, lane, ch);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              float f[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) f[j] = v[8 * k + j];
              ch[k] = pack8(f);
            }
            store_row_swizzled(wbuf + 4096, lane, ch);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
#ifdef VP_GEMM_TRACE
              if (!(epi.dbg & 2)) {
#endif
              tma_store_2d(&tmX, wbuf, col0, row0);
              tma_store_2d(&tmD, wbuf + 4096, col0, row0);
#ifdef VP_GEMM_TRACE
              }
#endif
              bulk_commit();
            }
            ETR(4, tq);
          } else {
            uint8_t* buf = wbuf + (kAuxIn ? ci : (C::kTwoBuf ? (nbuf & 1) : 0)) * 4096;
            tq = clock64();
            if (!kAuxIn) {
              if (lane == 0) {
                if constexpr (C::kTwoBuf) bulk_wait_read<1>();
                else bulk_wait_read<0>();
              }
              __syncwarp();
            }
            ETR(3, tq);
            tq = clock64();
            uint4 ch[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              float f[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) f[j] = v[8 * k + j];
              ch[k] = pack8(f);
            }
            store_row_swizzled(buf, lane, ch);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmD, buf, col0, row0);
              bulk_commit();
            }
            ETR(4, tq);
            ++nbuf;
          }
        }
      }
      // accumulator drained: release it to the leader's MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty_bar[acc], 0);
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
#ifdef VP_GEMM_TRACE
    if (warp == 4 && lane == 0) {
      et[5] = clock64() - e_begin;
      for (int i = 0; i < 6; ++i) g_vp_gemm_etrace[blockIdx.x][i] = et[i];
    }
#endif
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
}

#ifdef VP_GEMM_TRACE
}  // namespace
extern "C" int vp_debug_gemm_trace(unsigned long long* mma, unsigned long long* epi) {
  cudaError_t e = cudaMemcpyFromSymbol(mma, g_vp_gemm_trace, sizeof(g_vp_gemm_trace));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(epi, g_vp_gemm_etrace, sizeof(g_vp_gemm_etrace));
  return e;
}
namespace {
#endif
// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D tensor map (bf16 or fp32): inner dim contiguous, rows `ld` elements apart.
bool make_tmap(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
               uint32_t box_inner, uint32_t box_outer, bool f32 = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint64_t esz = f32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                  2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int sm_count() { return device_sms(); }

template <int BN, int STAGES, int EPI, bool A_MN, bool B_MN>
int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, int64_t M, int64_t N, int64_t K,
             const EpiArgs& e, cudaStream_t st) {
  using S = Smem<BN, STAGES>;
  auto kern = gemm_kernel<BN, STAGES, EPI, A_MN, B_MN>;
  if (cudaError_t err = vp::smem_optin(kern, S::TOTAL); err != cudaSuccess) return err;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = static_cast<int>(std::min<int64_t>(tiles, sm_count()));
  kern<<<grid, kThreads, S::TOTAL, st>>>(ta, tb, M, N, K, e);
  return cudaGetLastError();
}

template <int BN, int EPI>
int dispatch_layout(bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
                    int64_t M, int64_t N, int64_t K, const EpiArgs& e, cudaStream_t st) {
  constexpr int STAGES = BN == 256 ? 4 : 6;
  if (!a_mn && !b_mn) return launch_t<BN, STAGES, EPI, false, false>(ta, tb, M, N, K, e, st);
  if (!a_mn && b_mn) return launch_t<BN, STAGES, EPI, false, true>(ta, tb, M, N, K, e, st);
  if (a_mn && !b_mn) return launch_t<BN, STAGES, EPI, true, false>(ta, tb, M, N, K, e, st);
  return launch_t<BN, STAGES, EPI, true, true>(ta, tb, M, N, K, e, st);
}

template <int BN>
int dispatch_epi(int epi, bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
                 int64_t M, int64_t N, int64_t K, const EpiArgs& e, cudaStream_t st) {
  switch (epi) {
    case VP_EPI_STORE: return dispatch_layout<BN, VP_EPI_STORE>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    case VP_EPI_BIAS: return dispatch_layout<BN, VP_EPI_BIAS>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    case VP_EPI_BIAS_GELU:
      return dispatch_layout<BN, VP_EPI_BIAS_GELU>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    case VP_EPI_BIAS_RESID:
      return dispatch_layout<BN, VP_EPI_BIAS_RESID>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    case VP_EPI_DGELU: return dispatch_layout<BN, VP_EPI_DGELU>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    case VP_EPI_RESID: return dispatch_layout<BN, VP_EPI_RESID>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    case VP_EPI_ACC_F32:
      return dispatch_layout<BN, VP_EPI_ACC_F32>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    case VP_EPI_STORE_F32:
      return dispatch_layout<BN, VP_EPI_STORE_F32>(a_mn, b_mn, ta, tb, M, N, K, e, st);
    default: return VP_ERR_ARGS;
  }
}


template <int EPI, bool A_MN, bool B_MN>
int launch2_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td,
              const CUtensorMap& tx, int64_t M, int64_t N, int64_t K, int split_k,
              const Epi2& e, cudaStream_t st) {
  auto kern = gemm2_kernel<EPI, A_MN, B_MN>;
  if (cudaError_t err = vp::smem_optin(kern, G2Cfg<EPI>::kSmem); err != cudaSuccess) return err;
  const int64_t units = ((M + 255) / 256) * ((N + 255) / 256) * split_k;
  int64_t clusters = std::min<int64_t>(units, sm_count() / 2);
#ifdef VP_GEMM_TRACE
  if (const char* c = getenv("VP_GEMM_MAXCL")) clusters = std::min<int64_t>(clusters, atoi(c));
#endif
  kern<<<static_cast<unsigned>(2 * clusters), kThreads2, G2Cfg<EPI>::kSmem, st>>>(ta, tb, td, tx, M, N, K,
                                                                        split_k, e);
  return cudaGetLastError();
}

template <int EPI>
int dispatch2_layout(bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
                     const CUtensorMap& td, const CUtensorMap& tx, int64_t M, int64_t N, int64_t K,
                     int split_k, const Epi2& e, cudaStream_t st) {
  if (!a_mn && !b_mn) return launch2_t<EPI, false, false>(ta, tb, td, tx, M, N, K, split_k, e, st);
  if (!a_mn && b_mn) return launch2_t<EPI, false, true>(ta, tb, td, tx, M, N, K, split_k, e, st);
  if (a_mn && !b_mn) return launch2_t<EPI, true, false>(ta, tb, td, tx, M, N, K, split_k, e, st);
  return launch2_t<EPI, true, true>(ta, tb, td, tx, M, N, K, split_k, e, st);
}

int gemm2_dispatch(int epi, bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
                   const CUtensorMap& td, const CUtensorMap& tx, int64_t M, int64_t N, int64_t K,
                   int split_k, const Epi2& e, cudaStream_t st) {
#define D2(E) return dispatch2_layout<E>(a_mn, b_mn, ta, tb, td, tx, M, N, K, split_k, e, st)
  switch (epi) {
    case VP_EPI_STORE: D2(VP_EPI_STORE);
    case VP_EPI_BIAS: D2(VP_EPI_BIAS);
    case VP_EPI_BIAS_GELU: D2(VP_EPI_BIAS_GELU);
    case VP_EPI_BIAS_RESID: D2(VP_EPI_BIAS_RESID);
    case VP_EPI_DGELU: D2(VP_EPI_DGELU);
    case VP_EPI_RESID: D2(VP_EPI_RESID);
    case VP_EPI_ACC_F32: D2(VP_EPI_ACC_F32);
    case VP_EPI_STORE_F32: D2(VP_EPI_STORE_F32);
    default: return VP_ERR_ARGS;
  }
#undef D2
}

}  // namespace
}  // namespace vp

extern "C" int vp_device_sm_count(int* out) {
  if (!out) return VP_ERR_ARGS;
  *out = vp::sm_count();
  return VP_OK;
}

static int gemm_entry(int a_kmajor, int b_kmajor, int epilogue, const void* A, int64_t lda,
                      const void* B, int64_t ldb, void* D, int64_t ldd, const void* bias,
                      void* aux, int64_t ldaux, int64_t M, int64_t N, int64_t K, int flags,
                      void* stream, float* colsum_ws = nullptr,
                      vp::EpiDrop drop = vp::EpiDrop{nullptr, 0, 0, 1.f}) {
  using namespace vp;
  if (M <= 0 || N <= 0 || K <= 0 || !A || !B || !D) return VP_ERR_ARGS;
  if ((lda % 8) || (ldb % 8) || (ldd % 8)) return VP_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
       reinterpret_cast<uintptr_t>(D)) & 15)
    return VP_ERR_UNSUPPORTED;
  const bool needs_bias = epilogue == VP_EPI_BIAS || epilogue == VP_EPI_BIAS_GELU ||
                          epilogue == VP_EPI_BIAS_RESID;
  if (needs_bias && !bias) return VP_ERR_ARGS;
  if ((epilogue == VP_EPI_BIAS_RESID || epilogue == VP_EPI_DGELU || epilogue == VP_EPI_RESID) &&
      !aux)
    return VP_ERR_ARGS;
  if (aux && (ldaux % 8)) return VP_ERR_UNSUPPORTED;
  const bool a_mn = !a_kmajor, b_mn = !b_kmajor;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool f32_out = epilogue == VP_EPI_ACC_F32 || epilogue == VP_EPI_STORE_F32;
  const bool use2 = !(flags & VP_GEMM_DIRECT_STORE) && !getenv("VP_GEMM_1SM") &&
                    (ldd % (f32_out ? 4 : 8)) == 0;
  if (colsum_ws && (!use2 || f32_out || (N % 2))) return VP_ERR_UNSUPPORTED;
  if (drop.seed && (epilogue != VP_EPI_BIAS_RESID || (N % 2))) return VP_ERR_UNSUPPORTED;
  if (use2) {
    CUtensorMap ta, tb, td, tx;
    bool ok = a_mn ? make_tmap(&ta, A, M, K, lda, 64, BK) : make_tmap(&ta, A, K, M, lda, BK, 128);
    ok = ok && (b_mn ? make_tmap(&tb, B, N, K, ldb, 64, BK) : make_tmap(&tb, B, K, N, ldb, BK, 128));
    ok = ok && (f32_out ? make_tmap(&td, D, N, M, ldd, 32, 32, true)
                        : make_tmap(&td, D, N, M, ldd, 64, 32));
    if ((epilogue == VP_EPI_BIAS_GELU && aux) || epilogue == VP_EPI_BIAS_RESID ||
        epilogue == VP_EPI_DGELU || epilogue == VP_EPI_RESID)
      ok = ok && make_tmap(&tx, aux, N, M, ldaux, 64, 32);
    else tx = td;
    if (!ok) return VP_ERR_UNSUPPORTED;
    // Split K only when the reduce-add epilogue makes it exact-by-construction
    // per split and the output tiles cannot fill the clusters.
    int split = 1;
    const int64_t tiles = ((M + 255) / 256) * ((N + 255) / 256);
    const int64_t clusters = sm_count() / 2;
    if (epilogue == VP_EPI_ACC_F32 && tiles < clusters) {
      // Smallest split reaching (near-)best wave efficiency; every split adds
      // one fp32 reduce-add pass over the output, and each split keeps >= 16
      // k-blocks (1024 of K) so the mainloop amortises the tile prologue.
      const int64_t n_kb = (K + BK - 1) / BK;
      double best = double(tiles) / double(clusters);
      const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(8, n_kb / 16));
      for (int64_t sp = 2; sp <= smax; ++sp) {
        const int64_t units = tiles * sp;
        const int64_t rounds = (units + clusters - 1) / clusters;
        const double eff = double(units) / double(rounds * clusters);
        if (eff > best + 0.05) {
          best = eff;
          split = static_cast<int>(sp);
        }
      }
      if (const char* f = getenv("VP_GEMM_SPLITK")) split = std::max(1, atoi(f));
    }
    if (colsum_ws) split = 1;
    int64_t group = 8;
    if (const char* g = getenv("VP_GEMM_GROUP")) group = std::max(1, atoi(g));
    Epi2 e{reinterpret_cast<const __nv_bfloat16*>(bias), reinterpret_cast<const __nv_bfloat16*>(aux),
           ldaux, group, colsum_ws, drop, 0};
#ifdef VP_GEMM_TRACE
    if (const char* g = getenv("VP_GEMM_DBG")) e.dbg = atoi(g);
#endif
    return gemm2_dispatch(epilogue, a_mn, b_mn, ta, tb, td, tx, M, N, K, split, e, st);
  }
  const int BNsel = N <= 128 ? 128 : 256;
  CUtensorMap ta, tb;
  bool ok = a_mn ? make_tmap(&ta, A, M, K, lda, 64, BK) : make_tmap(&ta, A, K, M, lda, BK, BM);
  ok = ok && (b_mn ? make_tmap(&tb, B, N, K, ldb, 64, BK)
                   : make_tmap(&tb, B, K, N, ldb, BK, BNsel));
  if (!ok) return VP_ERR_UNSUPPORTED;
  EpiArgs e{D, ldd, reinterpret_cast<const __nv_bfloat16*>(bias),
            reinterpret_cast<__nv_bfloat16*>(aux), ldaux, drop};
  if (BNsel == 256) return dispatch_epi<256>(epilogue, a_mn, b_mn, ta, tb, M, N, K, e, st);
  return dispatch_epi<128>(epilogue, a_mn, b_mn, ta, tb, M, N, K, e, st);
}

extern "C" int vp_gemm_bf16(int a_kmajor, int b_kmajor, int epilogue, const void* A, int64_t lda,
                            const void* B, int64_t ldb, void* D, int64_t ldd, const void* bias,
                            void* aux, int64_t ldaux, int64_t M, int64_t N, int64_t K,
                            void* stream) {
  return gemm_entry(a_kmajor, b_kmajor, epilogue, A, lda, B, ldb, D, ldd, bias, aux, ldaux, M, N,
                    K, 0, stream);
}

extern "C" int vp_gemm_bf16_ex(int a_kmajor, int b_kmajor, int epilogue, const void* A,
                               int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                               const void* bias, void* aux, int64_t ldaux, int64_t M, int64_t N,
                               int64_t K, int flags, void* stream) {
  return gemm_entry(a_kmajor, b_kmajor, epilogue, A, lda, B, ldb, D, ldd, bias, aux, ldaux, M, N,
                    K, flags, stream);
}

extern "C" int vp_gemm_bf16_dropout(int a_kmajor, int b_kmajor, const void* A, int64_t lda,
                                    const void* B, int64_t ldb, void* D, int64_t ldd,
                                    const void* bias, const void* resid, int64_t ldres, int64_t M,
                                    int64_t N, int64_t K, float p, const uint64_t* seed,
                                    uint32_t salt, int flags, void* stream) {
  if (p < 0.f || p >= 1.f) return VP_ERR_ARGS;
  if (p > 0.f && !seed) return VP_ERR_ARGS;
  vp::EpiDrop drop{nullptr, 0, 0, 1.f};
  if (p > 0.f) {
    const uint32_t thr = vp::drop_threshold(p);
    drop = vp::EpiDrop{seed, salt, thr, vp::drop_scale(thr)};
  }
  return gemm_entry(a_kmajor, b_kmajor, VP_EPI_BIAS_RESID, A, lda, B, ldb, D, ldd, bias,
                    const_cast<void*>(resid), ldres, M, N, K, flags, stream, nullptr, drop);
}


namespace vp {
namespace {
// dbias[c] += sum over parts of ws[part][c] in a fixed order (32 columns x 32
// part-lanes per block, 8 independent loads per thread).
__global__ void __launch_bounds__(1024) colsum_f32_reduce(const float* __restrict__ ws,
                                                          float* __restrict__ out, int parts,
                                                          int64_t cols) {
  __shared__ float sh[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < cols) {
    int p = ty;
    for (; p + 7 * 32 < parts; p += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += ws[static_cast<int64_t>(p + u * 32) * cols + c];
    }
    for (; p < parts; p += 32) acc[0] += ws[static_cast<int64_t>(p) * cols + c];
  }
  sh[ty][tx] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  __syncthreads();
  if (ty == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += sh[i][tx];
    out[c] += t;
  }
}
}  // namespace
}  // namespace vp

extern "C" int64_t vp_gemm_dbias_ws_elems(int64_t M, int64_t N) { return ((M + 31) / 32) * N; }

extern "C" int vp_gemm_bf16_dbias(int a_kmajor, int b_kmajor, int epilogue, const void* A,
                                  int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                                  const void* bias, void* aux, int64_t ldaux, int64_t M, int64_t N,
                                  int64_t K, float* dbias, float* workspace, void* stream) {
  if (!dbias || !workspace) return VP_ERR_ARGS;
  int rc = gemm_entry(a_kmajor, b_kmajor, epilogue, A, lda, B, ldb, D, ldd, bias, aux, ldaux, M,
                      N, K, 0, stream, workspace);
  if (rc) return rc;
  const int parts = static_cast<int>((M + 31) / 32);
  vp::colsum_f32_reduce<<<static_cast<unsigned>((N + 31) / 32), 1024, 0,
                          reinterpret_cast<cudaStream_t>(stream)>>>(workspace, dbias, parts, N);
  return cudaGetLastError();
}
