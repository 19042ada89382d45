// Fused attention backward on tcgen05 (K3 of DESIGN.md), head_dim 64 and 96.
//
// One CTA per (128-key block, batch*head); it loops over the 128-query blocks
// the keys are visible to (causal: i >= kb) and produces dK, dV for its keys
// plus its share of every dQ_i, accumulated across CTAs in an fp32 buffer by
// TMA reduce-add (the only cross-CTA traffic). S and dP are computed once per
// (key block, query block) pair — five MMAs per pair instead of the seven of
// the two-kernel form (attention_tc.cu, kept as the deterministic path).
//
//   warp 0      TMA producer: K, V once; Q_i, dO_i and lse_i, delta_i (bulk
//               copy) into a 2-stage ring
//   warp 1      MMA issuer (one thread), per query block i:
//                 S^T  = K Q_i^T              TMEM [0,128)
//                 dP^T = V dO_i^T             TMEM [128,256)
//                 dV  += P^T dO_i             TMEM [256,320)
//                 dK  += dS^T Q_i             TMEM [320,384)
//                 dQ_i = dS K                 TMEM [384,448) / [448,512) (ping-pong)
//               S/dP of block i+1 are issued before the gradient MMAs of i,
//               so the tensor core runs while block i's softmax is computed.
//   warp 2      TMEM allocator (all 512 columns; 1 CTA per SM)
//   warps 4-11  thread = key row (TMEM lane); the two warps of a lane
//               quadrant split the 128 query columns. P^T = exp2(S^T c - lse),
//               dS^T = P^T (dP^T - delta) -> smem (bf16, SW128, K-major for
//               dV/dK and MN-major for dQ through a second descriptor);
//               then dQ_{i-1}: TMEM -> smem (fp32, SW128) -> TMA reduce-add.
//               At the end dK (x scale) and dV -> dqkv.
// dQacc is zeroed by the delta pre-pass and scaled to bf16 by a post-pass.
//
// head_dim 96 (GPT-2 2.5B / 8.3B): S^T, dP^T, dV, dK and P^T take
// 128+128+96+96+64 TMEM columns, so dQ_i has no columns of its own: it is
// computed into S^T's columns once the softmax warps have loaded the next
// block's S^T (S^T_{i+1} was issued before dQ_i, so the tensor core never
// idles for it), and S^T_{i+2} is issued after the drain warps have read
// dQ_i out — a full softmax block of slack on both sides. Tiles are a
// 64-wide SWIZZLE_128B chunk plus a 32-wide SWIZZLE_64B chunk (no padding to
// 128), the Q/dO ring has 2 stages and the dQ staging tiles are 16 rows,
// which fits the 227 KB of shared memory.
#include "sm100.cuh"
#include "tmap.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace vp {
#ifdef VP_BWD_TRACE
__device__ unsigned long long g_vp_trace[4][16][16];
#define TR(slot) \
  do { if (blockIdx.x < 4 && it < 16) g_vp_trace[blockIdx.x][it][slot] = clock64(); } while (0)
#define TRJ(jj, slot) \
  do { if (blockIdx.x < 4 && (jj) < 16) g_vp_trace[blockIdx.x][jj][slot] = clock64(); } while (0)
#else
#define TR(slot) do {} while (0)
#define TRJ(jj, slot) do {} while (0)
#endif
namespace {

constexpr int FB_M = 128;  // keys per CTA
constexpr int FB_N = 128;  // queries per inner block
constexpr int FB_CW = 8;   // softmax-gradient warps (4..11)
constexpr int FB_DW = 4;   // dQ drain warps (12..15), one per TMEM lane quadrant
constexpr int FB_THREADS = 128 + 32 * (FB_CW + FB_DW);
constexpr int64_t kConvParts = 64;  // row parts of the dQ convert / Q-bias column sums

template <int D>
struct FbSmem {
  static constexpr bool WIDE = D == 96;
  static constexpr int NS = WIDE ? 2 : 3;                    // Q/dO ring stages
  static constexpr int C0 = 128 * 128;                       // 128 rows x 64 bf16 (SW128)
  static constexpr int C1 = WIDE ? 128 * 64 : 0;             // 128 rows x 32 bf16 (SW64)
  static constexpr int TILE = C0 + C1;                       // one 128-row operand
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + TILE;
  static constexpr int Q_OFF = V_OFF + TILE;                 // [NS] {Q, dO}, stride 2*TILE
  static constexpr int DST_OFF = Q_OFF + NS * 2 * TILE;      // dS^T [2 buffers][2 chunks C0]
  static constexpr int STG_ROWS = WIDE ? 16 : 32;            // dQ staging rows per TMA reduce
  static constexpr int STG = STG_ROWS * 128;                 // per drain warp
  static constexpr int STG_OFF = DST_OFF + 2 * 2 * C0;
  static constexpr int LV_OFF = STG_OFF + FB_DW * STG;       // lse/delta [NS][2][128] f32
  static constexpr int BAR_OFF = LV_OFF + NS * 2 * FB_N * 4;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
  // TMEM: S^T 0, dP^T 128, dV 256, dK 256+D, P^T (bf16x2) 448; dQ at 384
  // (head_dim 64) or in S^T's columns (96)
  static constexpr int T_DV = 256, T_DK = 256 + D, T_P = 448, T_DQ = WIDE ? 0 : 384;
  static_assert(T_DK + D <= T_P, "attention bwd TMEM budget");
};
static_assert(FbSmem<64>::TOTAL <= 232448 && FbSmem<96>::TOTAL <= 232448, "attention bwd smem");

// Sum of v[0..31] over the 32 lanes, lane l ending with the total of
// element l (halving exchanges: 31 shuffles).
__device__ __forceinline__ float warp_colsum32(const float (&v)[32], uint32_t lane) {
  float t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const bool hi = lane & 16;
    t[i] = (hi ? v[i + 16] : v[i]) + __shfl_xor_sync(0xffffffffu, hi ? v[i] : v[i + 16], 16);
  }
#pragma unroll
  for (int w = 8, bit = 8; w >= 1; w >>= 1, bit >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const bool hi = lane & bit;
      t[i] = (hi ? t[i + w] : t[i]) + __shfl_xor_sync(0xffffffffu, hi ? t[i] : t[i + w], bit);
    }
  }
  return t[0];
}


// TMEM columns (512, one CTA per SM), head_dim 64:
//   [0,128) S^T   [128,256) dP^T   [256,320) dV   [320,384) dK   [384,448) dQ
//   [448,512) P^T as packed bf16x2 (A operand of the dV MMA)
// head_dim 96: dV [256,352), dK [352,448), P^T [448,512), dQ_i in [0,96)
// between the loads of S^T_{i+1} and the MMA of S^T_{i+2}.
// DROP (K7 attention dropout, mask as the forward's): the dV MMA consumes the
// dropped P^T (the 1/(1-p) scale applied to dV at the end), dS^T = P^T *
// (mask * dP^T / (1-p) - delta).
template <int D, bool CAUSAL, bool DROP>
__global__ void __launch_bounds__(FB_THREADS, 1)
    attn_bwd_fused(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                   const __grid_constant__ CUtensorMap tmQKV1,
                   const __grid_constant__ CUtensorMap tmDO1,
                   const __grid_constant__ CUtensorMap tmDQ, const float* __restrict__ lse,
                   const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, int S, int H,
                   int BH, int bh_chunk, float scale_log2, float scale,
                   float* __restrict__ dq_acc, float* __restrict__ kv_part, AttnDrop drop) {
  using L = FbSmem<D>;
  constexpr bool WIDE = L::WIDE;
  constexpr int FB_NS = L::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;     // [NS]
  uint64_t* q_empty = bars + 4;    // [NS]
  uint64_t* st_full = bars + 7;    // [2] per 64-query half of S^T/dP^T
  uint64_t* st_empty = bars + 9;   // [2]
  uint64_t* p_full = bars + 11;    // P^T (TMEM) + dS^T (smem) of a block written
  uint64_t* pt_empty = bars + 12;  // dV MMA consumed P^T
  uint64_t* ds_empty = bars + 13;  // [2] dK/dQ MMAs consumed dS^T buffer
  uint64_t* dq_full = bars + 15;
  uint64_t* dq_empty = bars + 16;
  uint64_t* acc_full = bars + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);

  // CTA order: (batch, head) pairs in chunks of bh_chunk; inside a chunk
  // longest-first (all key blocks 0 — most query blocks — then 1, ...). The
  // chunk bounds the set of (b, h) whose Q / dO / dQ-accumulator are live at
  // once so their re-reads (one per key block) hit L2: with one global
  // longest-first order every (b, h) is revisited a full wave later and at
  // B*H = 512 the kernel read 3.8x its algorithmic bytes from DRAM (chunks
  // of 128: -5% time at B*H = 512, unchanged at 128).
  const int n_kbt = (S + FB_M - 1) / FB_M;
  auto decode = [&](int cta, int& kb_, int& bh_) {
    const int chunk = cta / (bh_chunk * n_kbt);
    const int within = cta % (bh_chunk * n_kbt);
    const int csz = min(bh_chunk, BH - chunk * bh_chunk);
    kb_ = within / csz;
    bh_ = chunk * bh_chunk + within % csz;
  };
  int kb, bh;
  decode(static_cast<int>(blockIdx.x), kb, bh);
  const int b = bh / H, h = bh % H;
  const int k0 = kb * FB_M;
  const int n_qb = (S + FB_N - 1) / FB_N;
  const int i0 = CAUSAL ? kb : 0;  // FB_M == FB_N
  const int n_it = n_qb - i0;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int Hd = H * D;
  const float* lse_bh = lse + static_cast<int64_t>(bh) * S;
  const float* del_bh = delta + static_cast<int64_t>(bh) * S;
  float* sv = reinterpret_cast<float*>(smem + L::LV_OFF);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    tma_prefetch(&tmDO);
    if constexpr (WIDE) {
      tma_prefetch(&tmQKV1);
      tma_prefetch(&tmDO1);
    }
    tma_prefetch(&tmDQ);
    mbar_init(kv_full, 1);
    for (int i = 0; i < FB_NS; ++i) {
      mbar_init(&q_full[i], 2);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], FB_CW);
      mbar_init(&ds_empty[i], 1);
    }
    mbar_init(p_full, FB_CW);
    mbar_init(pt_empty, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, FB_DW);
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tdP = tmem + 128, tDV = tmem + L::T_DV, tDK = tmem + L::T_DK,
                 tDQ = tmem + L::T_DQ, tP = tmem + L::T_P;
  // one 128-row operand tile: d 0..63 (SW128) and, head_dim 96, d 64..95
  // (SW64) C0 bytes further
  auto load_tile = [&](uint8_t* dst, const CUtensorMap* m0, const CUtensorMap* m1,
                       uint64_t* bar, int col, int row) {
    tma_load_3d(dst, m0, bar, col, row, b);
    if constexpr (WIDE) tma_load_3d(dst + L::C0, m1, bar, col + 64, row, b);
  };

  if (warp == 0) {
    // ===== producer =====
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * L::TILE);
      load_tile(smem + L::K_OFF, &tmQKV, &tmQKV1, kv_full, Hd + h * D, k0);
      load_tile(smem + L::V_OFF, &tmQKV, &tmQKV1, kv_full, 2 * Hd + h * D, k0);
    }
    for (int it = 0; it < n_it; ++it) {
      const int st = it % FB_NS;
      const uint32_t ph = (it / FB_NS) & 1;
      const int qi = (i0 + it) * FB_N;
      const bool full_blk = qi + FB_N <= S && ((reinterpret_cast<uintptr_t>(lse_bh + qi) |
                                                reinterpret_cast<uintptr_t>(del_bh + qi)) & 15) == 0;
      float* dst = sv + st * 2 * FB_N;
      uint8_t* sq = smem + L::Q_OFF + st * 2 * L::TILE;
      if (lane == 0) {
        mbar_wait(&q_empty[st], ph ^ 1);
        mbar_expect_tx(&q_full[st], 2 * L::TILE + (full_blk ? 2 * FB_N * 4 : 0));
        load_tile(sq, &tmQKV, &tmQKV1, &q_full[st], h * D, qi);
        load_tile(sq + L::TILE, &tmDO, &tmDO1, &q_full[st], h * D, qi);
        if (full_blk) {
          bulk_g2s(dst, lse_bh + qi, FB_N * 4, &q_full[st]);
          bulk_g2s(dst + FB_N, del_bh + qi, FB_N * 4, &q_full[st]);
          mbar_arrive(&q_full[st]);
        }
      }
      if (!full_blk) {
        __syncwarp();
        mbar_wait(&q_empty[st], ph ^ 1);
        for (int t = lane; t < FB_N; t += 32) {
          const int q = qi + t;
          dst[t] = q < S ? lse_bh[q] : 0.f;
          dst[FB_N + t] = q < S ? del_bh[q] : 0.f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idST = idesc_bf16(128, FB_N, false, false);
      constexpr uint32_t idG = idesc_bf16(128, 64, false, true);
      constexpr uint32_t idG1 = idesc_bf16(128, 32, false, true);
      constexpr uint32_t idQ = idesc_bf16(128, 64, true, true);
      constexpr uint32_t idQ1 = idesc_bf16(128, 32, true, true);
      const uint32_t sK = smem_u32(smem + L::K_OFF), sV = smem_u32(smem + L::V_OFF);
      // K-major operand (rows = keys or queries, K = d): k-th 16-wide d step
      auto kdesc = [](uint32_t base, int k) {
        return k < 4 ? sdesc_sw128(base + k * 32, 16, 1024)
                     : sdesc_sw64(base + L::C0 + (k - 4) * 32, 16, 512);
      };
      // MN-major operand with N = d (Q, dO, K as B of dK, dV, dQ): rows
      // 16k..16k+15 of the d 0..63 chunk, or of the d 64..95 chunk
      auto ndesc0 = [](uint32_t base, int k) { return sdesc_sw128(base + k * 2048, L::C0, 1024); };
      auto ndesc1 = [](uint32_t base, int k) {
        return sdesc_sw64(base + L::C0 + k * 1024, L::C1, 512);
      };
      mbar_wait(kv_full, 0);
      auto issue_grad = [&](int j) {
        const int qs = j % FB_NS;
        const uint32_t sQ = smem_u32(smem + L::Q_OFF + qs * 2 * L::TILE);
        const uint32_t sdO = sQ + L::TILE;
        const uint32_t sdSt = smem_u32(smem + L::DST_OFF + (j & 1) * 2 * L::C0);
        mbar_wait(p_full, j & 1);
        TRJ(j, 10);
        tc_fence_after();
        // dV += P^T dO (A = P^T from TMEM)
#pragma unroll
        for (int k = 0; k < FB_N / 16; ++k)
          umma_f16_ts(tDV, tP + k * 8, ndesc0(sdO, k), idG, (j > 0 || k > 0) ? 1u : 0u);
        if constexpr (WIDE) {
#pragma unroll
          for (int k = 0; k < FB_N / 16; ++k)
            umma_f16_ts(tDV + 64, tP + k * 8, ndesc1(sdO, k), idG1, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(pt_empty);
        // dK += dS^T Q
#pragma unroll
        for (int k = 0; k < FB_N / 16; ++k) {
          const uint32_t koff = (k >> 2) * L::C0 + (k & 3) * 32;
          umma_f16(tDK, sdesc_sw128(sdSt + koff, 16, 1024), ndesc0(sQ, k), idG,
                   (j > 0 || k > 0) ? 1u : 0u);
          if constexpr (WIDE)
            umma_f16(tDK + 64, sdesc_sw128(sdSt + koff, 16, 1024), ndesc1(sQ, k), idG1,
                     (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&q_empty[qs]);  // Q_j, dO_j no longer needed
        if constexpr (!WIDE) {
          // dQ_j = dS K once the drain warps emptied dQ_{j-1}
          mbar_wait(dq_empty, (j & 1) ^ 1);
        } else if (j + 1 < n_it) {
          // dQ_j into S^T's columns once S^T_{j+1} / dP^T_{j+1} are loaded
          mbar_wait(&st_empty[0], (j + 1) & 1);
          mbar_wait(&st_empty[1], (j + 1) & 1);
        }
        TRJ(j, 11);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < FB_M / 16; ++k) {
          umma_f16(tDQ, sdesc_sw128(sdSt + k * 2048, L::C0, 1024), ndesc0(sK, k), idQ,
                   k > 0 ? 1u : 0u);
          if constexpr (WIDE)
            umma_f16(tDQ + 64, sdesc_sw128(sdSt + k * 2048, L::C0, 1024), ndesc1(sK, k), idQ1,
                     k > 0 ? 1u : 0u);
        }
        umma_commit(dq_full);
        umma_commit(&ds_empty[j & 1]);
        TRJ(j, 12);
      };
      for (int it = 0; it < n_it; ++it) {
        const int qs = it % FB_NS;
        const uint32_t sQ = smem_u32(smem + L::Q_OFF + qs * 2 * L::TILE);
        const uint32_t sdO = sQ + L::TILE;
        mbar_wait(&q_full[qs], (it / FB_NS) & 1);
        TR(8);
        // two 64-query halves: half 0 may overwrite TMEM as soon as every
        // warp has loaded its half-0 columns of the previous block
        mbar_wait(&st_empty[0], (it & 1) ^ 1);
        mbar_wait(&st_empty[1], (it & 1) ^ 1);
        // head_dim 96: dQ_{it-2} (in S^T's columns) drained
        if (WIDE && it >= 2) mbar_wait(dq_empty, it & 1);
        TR(9);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          umma_f16(tS, kdesc(sK, k), kdesc(sQ, k), idST, k > 0);
          umma_f16(tdP, kdesc(sV, k), kdesc(sdO, k), idST, k > 0);
        }
        umma_commit(&st_full[0]);
        umma_commit(&st_full[1]);
        if (it >= 1) issue_grad(it - 1);
      }
      issue_grad(n_it - 1);
      umma_commit(acc_full);
    }
  } else if (warp >= 4 && warp < 4 + FB_CW) {
    // ===== softmax-gradient warps: thread = key row =====
    const uint32_t qd = warp & 3;
    const int chalf = static_cast<int>(warp - 4) >> 2;
    const int r = qd * 32 + lane;
    const int key = k0 + r;
    const uint32_t trow = (qd * 32) << 16;
    const uint32_t rowG = smem_u32(smem + L::DST_OFF + r * 128);
    const uint32_t lv_base = smem_u32(sv);
    uint32_t dkey = 0;
    if constexpr (DROP) dkey = drop_key(drop.seed, drop.salt);

    // P^T, dS^T for 32 query columns starting at q0c into packed bf16x2 words
    // (lse, delta of the first 4 queries are loaded by the caller, l0/d0,
    // before it waits for the TMEM loads; each group prefetches the next
    // group's pair so the shared-memory latency overlaps the math)
    auto softmax_grad = [&](auto masked, const uint32_t (&rs)[32], const uint32_t (&rd)[32],
                            uint32_t lv, int q0c, int qlo, uint32_t (&pp)[16],
                            uint32_t (&pg)[16], uint32_t mword, float4 l4, float4 d4) {
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        float4 nl4 = l4, nd4 = d4;
        if (g < 7) {
          nl4 = lds128f(lv + 16 * (g + 1));
          nd4 = lds128f(lv + FB_N * 4 + 16 * (g + 1));
        }
        const float lq[4] = {l4.x, l4.y, l4.z, l4.w};
        const float dq[4] = {d4.x, d4.y, d4.z, d4.w};
        float p[4], gr[4];
        if (!DROP || drop.mask_k != nullptr) {
          // two query columns per FFMA2 / FSUB2 / FMUL2; dropout keep bits
          // as all-ones / zero AND masks on P and on the dP scale
#pragma unroll
          for (int t = 0; t < 4; t += 2) {
            const int i = 4 * g + t;
            const uint64_t x2 = ffma2(f2pack(__uint_as_float(rs[i]), __uint_as_float(rs[i + 1])),
                                      f2pack(scale_log2, scale_log2), f2pack(-lq[t], -lq[t + 1]));
            float a, b;
            f2unpack(x2, a, b);
            float pa = fast_exp2(a), pb = fast_exp2(b);
            if constexpr (decltype(masked)::value) {
              const int q = q0c + i;
              pa = (q >= qlo && q < S) ? pa : 0.f;
              pb = (q + 1 >= qlo && q + 1 < S) ? pb : 0.f;
            }
            uint64_t g2;
            if constexpr (DROP) {
              const uint32_t ka = 0u - ((mword >> i) & 1u), kb = 0u - ((mword >> (i + 1)) & 1u);
              p[t] = __uint_as_float(__float_as_uint(pa) & ka);
              p[t + 1] = __uint_as_float(__float_as_uint(pb) & kb);
              const uint32_t sb = __float_as_uint(drop.scale);
              g2 = fmul2(f2pack(pa, pb),
                         ffma2(f2pack(__uint_as_float(rd[i]), __uint_as_float(rd[i + 1])),
                               f2pack(__uint_as_float(sb & ka), __uint_as_float(sb & kb)),
                               f2pack(-dq[t], -dq[t + 1])));
            } else {
              p[t] = pa;
              p[t + 1] = pb;
              g2 = fmul2(f2pack(pa, pb),
                         fsub2(f2pack(__uint_as_float(rd[i]), __uint_as_float(rd[i + 1])),
                               f2pack(dq[t], dq[t + 1])));
            }
            f2unpack(g2, gr[t], gr[t + 1]);
          }
        } else {
          // no pre-drawn bits (S % 32 != 0): one hash per element; the same
          // arithmetic as above, so both forms give identical gradients
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int i = 4 * g + t;
            float pv = fast_exp2(fmaf(__uint_as_float(rs[i]), scale_log2, -lq[t]));
            if constexpr (decltype(masked)::value) {
              const int q = q0c + i;
              pv = (q >= qlo && q < S) ? pv : 0.f;
            }
            const uint64_t e = (static_cast<uint64_t>(bh) * S + (q0c + i)) * S + key;
            const uint32_t bits = drop_bits(dkey, e >> 1);
            const bool keep = ((key & 1) ? (bits >> 16) : (bits & 0xFFFFu)) >= drop.thr;
            p[t] = keep ? pv : 0.f;
            gr[t] = pv * fmaf(__uint_as_float(rd[i]), keep ? drop.scale : 0.f, -dq[t]);
          }
        }
        const __nv_bfloat162 p01 = __floats2bfloat162_rn(p[0], p[1]);
        const __nv_bfloat162 p23 = __floats2bfloat162_rn(p[2], p[3]);
        const __nv_bfloat162 g01 = __floats2bfloat162_rn(gr[0], gr[1]);
        const __nv_bfloat162 g23 = __floats2bfloat162_rn(gr[2], gr[3]);
        pp[2 * g] = *reinterpret_cast<const uint32_t*>(&p01);
        pp[2 * g + 1] = *reinterpret_cast<const uint32_t*>(&p23);
        pg[2 * g] = *reinterpret_cast<const uint32_t*>(&g01);
        pg[2 * g + 1] = *reinterpret_cast<const uint32_t*>(&g23);
        l4 = nl4;
        d4 = nd4;
      }
    };

    auto load_mwords = [&](int itn, uint32_t (&mw)[2]) {
      mw[0] = mw[1] = 0u;
      if (drop.mask_k != nullptr && key < S && itn < n_it) {
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int qw = ((i0 + itn) * FB_N + cc * 64 + chalf * 32) >> 5;
          if (qw * 32 < S)
            mw[cc] = __ldg(drop.mask_k + (static_cast<uint64_t>(bh) * (S >> 5) + qw) * S + key);
        }
      }
    };
    uint32_t mnext[2] = {0u, 0u};
    if constexpr (DROP) load_mwords(0, mnext);
    for (int it = 0; it < n_it; ++it) {
      const int qs = it % FB_NS;
      const int qi = (i0 + it) * FB_N;
      const bool need_mask = (qi + FB_N > S) || (CAUSAL && qi < k0 + FB_M - 1);
      const int qlo = CAUSAL ? key : 0;
      const uint32_t dsb = rowG + (it & 1) * 2 * L::C0;
      // dropout keep bits of this block's two 32-query column groups (one
      // global word each), loaded one block ahead so their latency hides
      // behind a whole block of work
      uint32_t mwords[2] = {mnext[0], mnext[1]};
      if constexpr (DROP) load_mwords(it + 1, mnext);
      if (warp == 4 && lane == 0) TR(0);
      mbar_wait(&q_full[qs], (it / FB_NS) & 1);
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = cc * 64 + chalf * 32;
        uint32_t rs[32], rd[32], pp[16], pg[16];
        mbar_wait(&st_full[cc], it & 1);
        if (warp == 4 && lane == 0) { if (cc == 0) TR(1); else TR(3); }
        tc_fence_after();
        tmem_ld32(tS + trow + c, rs);
        tmem_ld32(tdP + trow + c, rd);
        const uint32_t lv = lv_base + (qs * 2 * FB_N + c) * 4;
        const float4 l4 = lds128f(lv), d4 = lds128f(lv + FB_N * 4);
        tmem_ld_wait();
        // this half of S/dP consumed: the next block's half may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&st_empty[cc]);
        const uint32_t mword = mwords[cc];
        if (need_mask)
          softmax_grad(std::true_type{}, rs, rd, lv, qi + c, qlo, pp, pg, mword, l4, d4);
        else
          softmax_grad(std::false_type{}, rs, rd, lv, qi + c, qlo, pp, pg, mword, l4, d4);
        if (warp == 4 && lane == 0) { if (cc == 0) TR(2); else TR(4); }
        if (cc == 0) {
          mbar_wait(pt_empty, (it & 1) ^ 1);                  // dV of the previous block done
          mbar_wait(&ds_empty[it & 1], ((it >> 1) & 1) ^ 1);  // dS^T buffer free
          tc_fence_after();
          if (warp == 4 && lane == 0) TR(5);
        }
        tmem_st16(tP + trow + (c >> 1), pp);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sts128(dsb + cc * L::C0 + (((chalf * 4 + k) ^ (r & 7)) << 4),
                 make_uint4(pg[4 * k], pg[4 * k + 1], pg[4 * k + 2], pg[4 * k + 3]));
      }
      tmem_st_wait();
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (warp == 4 && lane == 0) TR(6);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    {
      // the two warps of a lane quadrant take D/2 columns each (32 | 48)
      constexpr int DC = D / 2;
      const int c = chalf * DC;
      uint32_t rk[32], rv[32];
      float fk[48], fv[48];
      tmem_ld32(tDK + trow + c, rk);
      tmem_ld32(tDV + trow + c, rv);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        fk[i] = key < S ? __uint_as_float(rk[i]) * scale : 0.f;
        fv[i] = key < S ? __uint_as_float(rv[i]) * (DROP ? drop.scale : 1.f) : 0.f;
      }
      if constexpr (DC > 32) {
        uint32_t rk2[16], rv2[16];
        tmem_ld16(tDK + trow + c + 32, rk2);
        tmem_ld16(tDV + trow + c + 32, rv2);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          fk[32 + i] = key < S ? __uint_as_float(rk2[i]) * scale : 0.f;
          fv[32 + i] = key < S ? __uint_as_float(rv2[i]) * (DROP ? drop.scale : 1.f) : 0.f;
        }
      }
      if (key < S) {
        __nv_bfloat16* row = dqkv + (static_cast<int64_t>(b) * S + key) * (3 * Hd) + h * D + c;
#pragma unroll
        for (int i = 0; i < DC; i += 8) {
          *reinterpret_cast<uint4*>(row + Hd + i) = pack8(*reinterpret_cast<float(*)[8]>(fk + i));
          *reinterpret_cast<uint4*>(row + 2 * Hd + i) = pack8(*reinterpret_cast<float(*)[8]>(fv + i));
        }
      }
      if (kv_part != nullptr) {
        // K/V bias gradient: this warp's 32 keys summed per column (lane l
        // ends with column c + l) -> kv_part[(b, kb, quadrant)][K | V column]
        float* dst = kv_part + ((static_cast<int64_t>(b) * gridDim.x / BH + kb) * 4 + qd) * (2 * Hd);
        const float sk = warp_colsum32(*reinterpret_cast<float(*)[32]>(fk), lane);
        const float sv = warp_colsum32(*reinterpret_cast<float(*)[32]>(fv), lane);
        dst[h * D + c + lane] = sk;
        dst[Hd + h * D + c + lane] = sv;
        if constexpr (DC > 32) {
          float tk[32], tv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            tk[i] = i < 16 ? fk[32 + i] : 0.f;
            tv[i] = i < 16 ? fv[32 + i] : 0.f;
          }
          const float sk2 = warp_colsum32(tk, lane), sv2 = warp_colsum32(tv, lane);
          if (lane < 16) {
            dst[h * D + c + 32 + lane] = sk2;
            dst[Hd + h * D + c + 32 + lane] = sv2;
          }
        }
      }
    }
  } else if (warp >= 4 + FB_CW) {
    // ===== dQ drain: TMEM -> smem (fp32, SW128) -> TMA reduce-add =====
    const uint32_t qd = warp & 3;
    const uint32_t trow = (qd * 32) << 16;
    uint8_t* stg = smem + L::STG_OFF + qd * L::STG;
    // 32 fp32 columns of this warp's 32 query rows into dQacc (column col),
    // L::STG_ROWS rows per TMA reduce through the staging tile
    auto reduce32 = [&](const uint32_t (&v)[32], int col, int q) {
#pragma unroll
      for (int part = 0; part < 32 / L::STG_ROWS; ++part) {
        if (lane == 0) bulk_wait_read<0>();  // previous reduce has read the staging tile
        __syncwarp();
        if (static_cast<int>(lane) / L::STG_ROWS == part) {
          const int rr = static_cast<int>(lane) % L::STG_ROWS;
          const uint32_t s0 = smem_u32(stg + rr * 128);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            sts128(s0 + ((k ^ (rr & 7)) << 4),
                   make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_3d(&tmDQ, stg, col, q + part * L::STG_ROWS, b);
          bulk_commit();
        }
      }
    };
    for (int j = 0; j < n_it; ++j) {
      const int q = (i0 + j) * FB_N + qd * 32;
      uint32_t v0[32], v1[32];
      mbar_wait(dq_full, j & 1);
      if (warp == 4 + FB_CW && lane == 0) TRJ(j, 13);
      tc_fence_after();
      uint32_t v2[WIDE ? 32 : 1];
      tmem_ld32(tDQ + trow, v0);
      tmem_ld32(tDQ + trow + 32, v1);
      if constexpr (WIDE) tmem_ld32(tDQ + trow + 64, v2);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
      reduce32(v0, h * D, q);
      reduce32(v1, h * D + 32, q);
      if constexpr (WIDE) reduce32(v2, h * D + 64, q);
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// delta[b,h,s] = sum_d O * dO (fp32) and dQacc[t, :] = 0, one (token, head)
// row per G-lane group (8 lanes x 8 elements at head_dim 64, 4 x 24 at 96).
template <int D>
__global__ void __launch_bounds__(256) attn_delta_zero_kernel(
    const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
    float* __restrict__ delta, float* __restrict__ dq_acc, int64_t tokens, int S, int H,
    unsigned* __restrict__ counters) {
  constexpr int G = D == 96 ? 4 : D / 8;
  constexpr int E = D / G;
  if (blockIdx.x == 0 && threadIdx.x < 64) counters[threadIdx.x] = 0u;
  const int lane = threadIdx.x & 31;
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  const int li = lane % G;
  float acc = 0.f;
  const bool ok = row < tokens * H;
  if (ok) {
    const int64_t off = row * D + li * E;
#pragma unroll
    for (int e = 0; e < E; e += 8) {
      float a[8], g[8];
      unpack8(*reinterpret_cast<const uint4*>(o + off + e), a);
      unpack8(*reinterpret_cast<const uint4*>(dout + off + e), g);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += a[j] * g[j];
      float4* z = reinterpret_cast<float4*>(dq_acc + off + e);
      z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
#pragma unroll
  for (int m = G / 2; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (ok && li == 0) {
    const int64_t t = row / H;
    const int h = static_cast<int>(row % H);
    const int64_t b = t / S, s = t % S;
    delta[(b * H + h) * S + s] = acc;
  }
}

// dqkv[t, 0:Hd] = bf16(dQacc[t, :] * scale)
__global__ void __launch_bounds__(256) dq_convert_kernel(const float* __restrict__ dq_acc,
                                                         __nv_bfloat16* __restrict__ dqkv,
                                                         int64_t tokens, int Hd, float scale) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i >= tokens * Hd) return;
  const int64_t t = i / Hd;
  const int c = static_cast<int>(i % Hd);
  const float4 a = reinterpret_cast<const float4*>(dq_acc + i)[0];
  const float4 b = reinterpret_cast<const float4*>(dq_acc + i)[1];
  float f[8] = {a.x * scale, a.y * scale, a.z * scale, a.w * scale,
                b.x * scale, b.y * scale, b.z * scale, b.w * scale};
  *reinterpret_cast<uint4*>(dqkv + t * (3 * static_cast<int64_t>(Hd)) + c) = pack8(f);
}

// The same conversion fused with the Q bias gradient: CTA (256 columns, row
// part) with 8 row-lanes x 4 rows in flight, column partials ->
// part_ws[part][Hd]; the last CTA of a column block (arrival counter) sums the
// parts in a fixed order (deterministic) into dbias.
__global__ void __launch_bounds__(256) dq_convert_bias_kernel(
    const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int64_t tokens, int Hd,
    float scale, int64_t rpp, int parts, float* __restrict__ part_ws,
    unsigned* __restrict__ counters, float* __restrict__ dbias) {
  __shared__ float sh[8][256 + 4];
  __shared__ bool is_last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int cb = blockIdx.x * 256;
  const int c0 = cb + tx * 8;
  const int64_t r0 = blockIdx.y * rpp, r1 = min(tokens, r0 + rpp);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < Hd) {
#pragma unroll 4
    for (int64_t t = r0 + ty; t < r1; t += 8) {
      const float4* src = reinterpret_cast<const float4*>(dq_acc + t * Hd + c0);
      const float4 a = src[0], b = src[1];
      float f[8] = {a.x * scale, a.y * scale, a.z * scale, a.w * scale,
                    b.x * scale, b.y * scale, b.z * scale, b.w * scale};
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += f[j];
      *reinterpret_cast<uint4*>(dqkv + t * (3 * static_cast<int64_t>(Hd)) + c0) = pack8(f);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) sh[ty][tx * 8 + j] = acc[j];
  __syncthreads();
  {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x];
    if (cb + static_cast<int>(threadIdx.x) < Hd)
      part_ws[static_cast<int64_t>(blockIdx.y) * Hd + cb + threadIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    is_last = atomicAdd(&counters[blockIdx.x], 1u) == static_cast<unsigned>(parts - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < Hd) {
    // 4 parts in flight per step (the tail of the last CTA is latency-bound);
    // the grouping is fixed, so the sum order does not depend on timing
    float g4[4][8] = {};
    int p = ty;
    for (; p + 24 < parts; p += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int pp = p + 8 * u;
        const float4* src = reinterpret_cast<const float4*>(part_ws + static_cast<int64_t>(pp) * Hd + c0);
        const float4 a = __ldcg(src), b = __ldcg(src + 1);
        g4[u][0] += a.x; g4[u][1] += a.y; g4[u][2] += a.z; g4[u][3] += a.w;
        g4[u][4] += b.x; g4[u][5] += b.y; g4[u][6] += b.z; g4[u][7] += b.w;
      }
    }
    for (; p < parts; p += 8) {
      const int pp = p;
      const float4* src = reinterpret_cast<const float4*>(part_ws + static_cast<int64_t>(pp) * Hd + c0);
      const float4 a = __ldcg(src), b = __ldcg(src + 1);
      g4[0][0] += a.x; g4[0][1] += a.y; g4[0][2] += a.z; g4[0][3] += a.w;
      g4[0][4] += b.x; g4[0][5] += b.y; g4[0][6] += b.z; g4[0][7] += b.w;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = (g4[0][j] + g4[1][j]) + (g4[2][j] + g4[3][j]);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 8; ++j) sh[ty][tx * 8 + j] = f[j];
  __syncthreads();
  {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x];
    if (cb + static_cast<int>(threadIdx.x) < Hd) dbias[cb + threadIdx.x] += t;
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0u;
}

// dbias[c] += sum over partial rows of kv_part[row][c] (fixed order): 32
// columns x 32 row-lanes per block, 8 independent loads per thread.
__global__ void __launch_bounds__(1024) kv_bias_reduce(const float* __restrict__ kv_part,
                                                       float* __restrict__ dbias, int prow, int n) {
  __shared__ float sh[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < n) {
    int r = ty;
    for (; r + 7 * 32 < prow; r += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += kv_part[static_cast<int64_t>(r + u * 32) * n + c];
    }
    for (; r < prow; r += 32) acc[0] += kv_part[static_cast<int64_t>(r) * n + c];
  }
  sh[ty][tx] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  __syncthreads();
  if (ty == 0 && c < n) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += sh[i][tx];
    dbias[c] += t;
  }
}

template <int D, bool CAUSAL, bool DROP>
int fused_t(const void* qkv, const void* o, const void* dout, const float* lse, float* delta,
            float* dq_acc, void* dqkv, int64_t B, int64_t S, int64_t H, float* dbias,
            float* part_ws, unsigned* counters, float* kv_part, const AttnDrop& drop,
            cudaStream_t st) {
  using L = FbSmem<D>;
  const int64_t tokens = B * S;
  const int Hd = static_cast<int>(H * D);
  CUtensorMap tq, tdo, tq1, tdo1, tdq;
  if (!make_tmap_bsc(&tq, qkv, 3 * H * D, S, B, 128) ||
      !make_tmap_bsc(&tdo, dout, H * D, S, B, 128) ||
      !make_tmap_bsc(&tq1, qkv, 3 * H * D, S, B, 128, true) ||
      !make_tmap_bsc(&tdo1, dout, H * D, S, B, 128, true) ||
      !make_tmap_bsc_f32(&tdq, dq_acc, H * D, S, B, L::STG_ROWS))
    return VP_ERR_UNSUPPORTED;
  auto k = attn_bwd_fused<D, CAUSAL, DROP>;
  if (cudaError_t e = smem_optin(k, L::TOTAL); e != cudaSuccess) return e;
  const int64_t rows = tokens * H;
  constexpr int G = D == 96 ? 4 : D / 8;
  attn_delta_zero_kernel<D><<<static_cast<unsigned>((rows * G + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(o), reinterpret_cast<const __nv_bfloat16*>(dout),
      delta, dq_acc, tokens, static_cast<int>(S), static_cast<int>(H), counters);
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = 1.4426950408889634f * scale;
  const int n_kb = static_cast<int>((S + FB_M - 1) / FB_M);
  const int BH = static_cast<int>(B * H);
  static const int env_chunk = getenv("VP_ATTN_BH_CHUNK") ? atoi(getenv("VP_ATTN_BH_CHUNK")) : 0;
  const int bh_chunk = std::max(1, std::min(BH, env_chunk > 0 ? env_chunk : 128));
  k<<<static_cast<unsigned>(n_kb * BH), FB_THREADS, L::TOTAL, st>>>(
      tq, tdo, tq1, tdo1, tdq, lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), static_cast<int>(S),
      static_cast<int>(H), BH, bh_chunk, scale_log2, scale, dq_acc,
      dbias ? kv_part : nullptr,
      drop);
  if (!dbias) {
    dq_convert_kernel<<<static_cast<unsigned>((tokens * Hd / 8 + 255) / 256), 256, 0, st>>>(
        dq_acc, reinterpret_cast<__nv_bfloat16*>(dqkv), tokens, Hd, scale);
  } else {
    const int col_blocks = (Hd + 255) / 256;
    int parts = static_cast<int>(std::min<int64_t>(kConvParts, std::max<int64_t>(
        1, (8 * static_cast<int64_t>(device_sms()) + col_blocks - 1) / col_blocks)));
    const int64_t rpp = (tokens + parts - 1) / parts;
    parts = static_cast<int>((tokens + rpp - 1) / rpp);
    dq_convert_bias_kernel<<<dim3(col_blocks, parts), 256, 0, st>>>(
        dq_acc, reinterpret_cast<__nv_bfloat16*>(dqkv), tokens, Hd, scale, rpp, parts, part_ws,
        counters, dbias);
    const int prow = static_cast<int>(B * n_kb * 4);
    kv_bias_reduce<<<(2 * Hd + 31) / 32, 1024, 0, st>>>(kv_part, dbias + Hd, prow, 2 * Hd);
  }
  return launch_status();
}

}  // namespace

// Workspace of the fused backward (fp32 elements, 16-byte aligned pieces):
// delta [B*H*S] | dQacc [B*S*H*D] | Q-bias partials [kConvParts][H*D] |
// arrival counters [64] | K/V-bias partials [B*n_kb*4][2*H*D]
static int64_t al4(int64_t n) { return (n + 3) / 4 * 4; }
int64_t attention_bwd_fused_ws(int64_t B, int64_t S, int64_t H, int64_t D) {
  const int64_t n_kb = (S + FB_M - 1) / FB_M;
  return al4(B * H * S) + al4(B * S * H * D) + al4(kConvParts * H * D) + 64 +
         B * n_kb * 4 * 2 * H * D;
}

bool attention_bwd_fused_ok(int64_t D) { return D == 64 || D == 96; }

int attention_bwd_fused(const void* qkv, const void* o, const void* dout, const float* lse,
                        void* dqkv, float* ws, int64_t B, int64_t S, int64_t H, int64_t D,
                        int causal, float* dbias, const AttnDrop& drop, cudaStream_t st) {
  float* delta = ws;
  float* dq_acc = delta + al4(B * H * S);
  float* part_ws = dq_acc + al4(B * S * H * D);
  unsigned* counters = reinterpret_cast<unsigned*>(part_ws + al4(kConvParts * H * D));
  float* kv_part = reinterpret_cast<float*>(counters) + 64;
#define FT(DD, C, DR) fused_t<DD, C, DR>(qkv, o, dout, lse, delta, dq_acc, dqkv, B, S, H, dbias, \
                                         part_ws, counters, kv_part, drop, st)
  if (D == 96) {
    if (drop.seed) return causal ? FT(96, true, true) : FT(96, false, true);
    return causal ? FT(96, true, false) : FT(96, false, false);
  }
  if (D != 64) return VP_ERR_UNSUPPORTED;
  if (drop.seed) return causal ? FT(64, true, true) : FT(64, false, true);
  return causal ? FT(64, true, false) : FT(64, false, false);
#undef FT
}

}  // namespace vp

#ifdef VP_BWD_TRACE
extern "C" int vp_debug_bwd_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vp::g_vp_trace, sizeof(vp::g_vp_trace));
}
#endif
