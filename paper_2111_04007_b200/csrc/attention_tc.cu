// Fused attention forward on tcgen05 (K2 of DESIGN.md).
//
// CTA = 128 queries of one (batch, head); keys in blocks of 128.
//   warp 0      TMA producer: Q once, then (K_j, V_j) into a 2-stage ring
//   warp 1      MMA issuer:   S_j = Q K_j^T -> TMEM (ping-pong S0/S1),
//                             O += P_j V_j  -> TMEM (one accumulator)
//   warp 2      TMEM allocator (512 columns: S0 S1 O)
//   warps 4..7  softmax: thread = query row (TMEM lane), whole row per
//               thread (no shuffles); online max/sum; P_j -> smem (bf16,
//               128B-swizzled K-major) for the PV MMA. O stays in TMEM: it is
//               rescaled in place (tcgen05.ld/st) only when some row's running
//               max grows by more than 2^8 (lazy correction; P <= 2^8 keeps
//               bf16/fp32 exact enough). O/LSE are written at the end.
// The MMA for S_{j+1} is issued before O_j so the tensor core works while
// the softmax warps process block j.
#include "sm100.cuh"
#include "tmap.cuh"

#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdlib>

namespace vp {
namespace {

constexpr int TA_BM = 128;
constexpr int TA_BN = 64;   // keys per block: TMEM S0|S1|O = 64+64+<=128 <= 256 cols -> 2 CTAs/SM
constexpr int TA_THREADS = 256;
// K/V ring depth: deep enough to cover the L2->SMEM TMA latency of a block
// while the previous ones are consumed. With P in TMEM (D <= 96) the smem P
// buffers are not needed and D = 64 affords 5 stages at 2 CTAs/SM: the MMA
// warp issues S_{j+2} right after the softmax warps load S_j, so block
// j+2's K/V must already be resident then.
__host__ __device__ constexpr int ta_stages(int D) { return D == 64 ? 5 : 3; }
// head_dim 96 tiles are stored compact — a 64-wide SWIZZLE_128B chunk and a
// 32-wide SWIZZLE_64B chunk — so Q + 3 K/V stages take 99 KB and two CTAs
// fit on an SM (padded to 128 columns it was one CTA per SM).

template <int D>
struct TaSmem {
  // TMEM (256 columns, 2 CTAs/SM): S double-buffered [0,128), O [128,128+D),
  // then, when they fit, Q (A operand of S = Q K^T, TS mode) and P (A operand
  // of O += P V, TS mode) as packed bf16 pairs. Operands kept in TMEM are
  // not re-read from shared memory by every MMA (the forward is bound by
  // shared-memory bandwidth otherwise).
  static constexpr bool QT = D == 64;                // Q in TMEM (32 cols)
  static constexpr bool PT = D <= 96;                // P in TMEM (32 cols)
  static constexpr int TQ = 128 + D;                 // TMEM column of Q
  static constexpr int TP = 128 + D + (QT ? D / 2 : 0);  // TMEM column of P
  static_assert(TP + (PT ? 32 : 0) <= 256, "attention fwd TMEM budget");
  static constexpr int CH = (D + 63) / 64;           // 64-wide d-chunks (128 B rows)
  static constexpr bool NARROW = D == 96;            // d 64..95 as a 32-wide SW64 chunk
  static constexpr int QCH = 128 * 128;              // one Q d-chunk: 128 rows x 128 B
  static constexpr int KCH = TA_BN * 128;            // one K/V d-chunk: 64 rows x 128 B
  static constexpr int QTILE = NARROW ? QCH + 128 * 64 : QCH * CH;
  static constexpr int KTILE = NARROW ? KCH + TA_BN * 64 : KCH * CH;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = QTILE;                // [stage]
  static constexpr int STAGES = ta_stages(D);
  static constexpr int V_OFF = K_OFF + STAGES * KTILE;
  static constexpr int P_OFF = V_OFF + STAGES * KTILE;  // [2][128 x 64] bf16 (smem P only)
  static constexpr int BAR_OFF = P_OFF + (PT ? 0 : 2 * 128 * TA_BN * 2);
  static constexpr int RED_OFF = BAR_OFF + 256;      // [2 bufs][2 halves][128 rows] f32 (SW = 8)
  static constexpr int TOTAL = RED_OFF + 2 * 2 * 128 * 4 + 1024;
};

#ifdef VP_BWD_TRACE
__device__ unsigned long long g_vp_ftrace[4][32][8];
#define TRF(j, slot) \
  do { if (blockIdx.x < 1 && blockIdx.y < 4 && (j) < 32) g_vp_ftrace[blockIdx.y][j][slot] = clock64(); } while (0)
#else
#define TRF(j, slot) do {} while (0)
#endif
// Attention-probability dropout (K7, DROP; AttnDrop in common.cuh): P_ij is
// kept iff the mask bit of element ((b*H + h)*S + i)*S + j is set; the row
// sum l (and the LSE) use the undropped P, the 1/(1-p) scale is folded into
// the final O = acc * scale / l.
// SW softmax warps per CTA: 4 (thread = query row, all 64 keys of a block)
// or 8 (head_dim 64: the two warps of a TMEM lane quadrant split a block's
// keys 32/32 — half the per-thread work per block and twice the warps to hide
// the MUFU / TMEM / barrier latencies; the row max is exchanged through shared
// memory under a 64-thread named barrier, the row sums only at the end).
template <int D, bool CAUSAL, bool DROP, int SW = 4>
__global__ void __launch_bounds__(128 + 32 * SW, 2)
    attn_fwd_tc(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmKV,
                const __grid_constant__ CUtensorMap tmQKV1,
                const __grid_constant__ CUtensorMap tmKV1, __nv_bfloat16* __restrict__ out,
                float* __restrict__ lse, int S, int H, int n_qb, float scale_log2, AttnDrop drop) {
  static_assert(SW == 4 || (SW == 8 && D == 64), "split softmax: head_dim 64 only");
  constexpr int NK = TA_BN * 4 / SW;      // keys per softmax thread per block
  using L = TaSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  static_assert(L::STAGES <= 8, "attention fwd barrier layout");
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;              // [STAGES <= 8]
  uint64_t* kv_empty = bars + 9;             // [STAGES]
  uint64_t* s_full = bars + 17;              // [2]
  uint64_t* s_empty = bars + 19;             // [2]
  uint64_t* o_full = bars + 21;              // [2]: PV_j commits o_full[j & 1]
  uint64_t* p_full = bars + 23;              // [2]
  uint64_t* q_tmem = bars + 25;              // Q copied into TMEM (the softmax warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 26);

  const int qb = n_qb - 1 - static_cast<int>(blockIdx.x);  // heavy (late) causal blocks first
  const int bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int q0 = qb * TA_BM;
  int n_kb = (S + TA_BN - 1) / TA_BN;
  if (CAUSAL) n_kb = min(n_kb, (q0 + TA_BM + TA_BN - 1) / TA_BN);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int Hd = H * D;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    tma_prefetch(&tmKV);
    if constexpr (L::NARROW) {
      tma_prefetch(&tmQKV1);
      tma_prefetch(&tmKV1);
    }
    mbar_init(q_full, 1);
    for (int i = 0; i < L::STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], SW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&o_full[i], 1);
      mbar_init(&p_full[i], SW);
    }
    mbar_init(q_tmem, SW);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== producer =====
      mbar_expect_tx(q_full, L::QTILE);
#pragma unroll
      for (int c = 0; c < L::CH; ++c) {
        if (L::NARROW && c == 1)
          tma_load_3d(smem + L::Q_OFF + L::QCH, &tmQKV1, q_full, h * D + 64, q0, b);
        else
          tma_load_3d(smem + L::Q_OFF + c * L::QCH, &tmQKV, q_full, h * D + c * 64, q0, b);
      }
      for (int j = 0; j < n_kb; ++j) {
        const int st = j % L::STAGES;
        mbar_wait(&kv_empty[st], ((j / L::STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * L::KTILE);
#pragma unroll
        for (int c = 0; c < L::CH; ++c) {
          const CUtensorMap* m = (L::NARROW && c == 1) ? &tmKV1 : &tmKV;
          tma_load_3d(smem + L::K_OFF + st * L::KTILE + c * L::KCH, m, &kv_full[st],
                      Hd + h * D + c * 64, j * TA_BN, b);
          tma_load_3d(smem + L::V_OFF + st * L::KTILE + c * L::KCH, m, &kv_full[st],
                      2 * Hd + h * D + c * 64, j * TA_BN, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idS = idesc_bf16(128, TA_BN, false, false);
      constexpr uint32_t idO = idesc_bf16(128, L::NARROW ? 64 : D, false, true);
      constexpr uint32_t idO1 = idesc_bf16(128, 32, false, true);
      const uint32_t sQ = smem_u32(smem + L::Q_OFF);
      const uint32_t sP = smem_u32(smem + L::P_OFF);
      mbar_wait(q_full, 0);
      if constexpr (L::QT) mbar_wait(q_tmem, 0);  // softmax warps copied Q into TMEM
      auto issue_pv = [&](int j) {
        const int st = j % L::STAGES;
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);  // P_j written (and O rescaled if needed)
        TRF(j, 5);
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + L::V_OFF + st * L::KTILE);
        const uint32_t sPj = sP + (j & 1) * 128 * TA_BN * 2;
#pragma unroll
        for (int k = 0; k < TA_BN / 16; ++k) {
          // B = V [key][d] MN-major: +16 rows * 128 B per 16 keys; d-chunks KCH apart
          const uint64_t bd = sdesc_sw128(sV + k * 2048, L::KCH, 1024);
          if constexpr (L::NARROW) {
            // d 0..63 and d 64..95 (SW64 rows of 64 B: +1 KB per 16 keys)
            umma_f16_ts(tmem + 128, tmem + L::TP + k * 8, bd, idO, (j > 0 || k > 0) ? 1u : 0u);
            umma_f16_ts(tmem + 192, tmem + L::TP + k * 8,
                        sdesc_sw64(sV + L::KCH + k * 1024, L::KCH, 512), idO1,
                        (j > 0 || k > 0) ? 1u : 0u);
          } else if constexpr (L::PT) {
            umma_f16_ts(tmem + 128, tmem + L::TP + k * 8, bd, idO, (j > 0 || k > 0) ? 1u : 0u);
          } else {
            // A = P [q][key] K-major (one 128 B row chunk): +32 B per 16 keys
            const uint64_t ad = sdesc_sw128(sPj + k * 32, 16, 1024);
            umma_f16(tmem + 128, ad, bd, idO, (j > 0 || k > 0) ? 1u : 0u);
          }
        }
        umma_commit(&o_full[j & 1]);
        umma_commit(&kv_empty[st]);
      };
      auto issue_s = [&](int j) {
        const int st = j % L::STAGES;
        mbar_wait(&kv_full[st], (j / L::STAGES) & 1);
        mbar_wait(&s_empty[j & 1], ((j >> 1) & 1) ^ 1);
        TRF(j, 4);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + L::K_OFF + st * L::KTILE);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          if (L::NARROW && k >= 4) {
            umma_f16(tmem + (j & 1) * TA_BN, sdesc_sw64(sQ + L::QCH + (k - 4) * 32, 16, 512),
                     sdesc_sw64(sK + L::KCH + (k - 4) * 32, 16, 512), idS, 1u);
            continue;
          }
          const uint64_t bd = sdesc_sw128(sK + (k >> 2) * L::KCH + (k & 3) * 32, 16, 1024);
          if constexpr (L::QT) {
            umma_f16_ts(tmem + (j & 1) * TA_BN, tmem + L::TQ + k * 8, bd, idS, k > 0);
          } else {
            umma_f16(tmem + (j & 1) * TA_BN,
                     sdesc_sw128(sQ + (k >> 2) * L::QCH + (k & 3) * 32, 16, 1024), bd, idS, k > 0);
          }
        }
        umma_commit(&s_full[j & 1]);
      };
      // S_{j+2} is issued as soon as the softmax warps have LOADED S_j (its
      // TMEM buffer is free then), ahead of PV_j, which waits for them to
      // FINISH block j: the next score block is computed while a block's
      // softmax runs, instead of after it (the MMA issue order used to gate
      // S_{j+2} on P_j; clock64 timelines, profiles/r02/r02w_*)
      if (n_kb > 0) issue_s(0);
      if (n_kb > 1) issue_s(1);
      for (int j = 0; j < n_kb; ++j) {
        if (j + 2 < n_kb) issue_s(j + 2);
        issue_pv(j);
      }
    }
  } else if (warp >= 4) {
    // ===== softmax / correction / epilogue: thread = query row =====
    const uint32_t qd = warp & 3;
    const int half = static_cast<int>(warp - 4) >> 2;   // 0 when SW == 4
    const int koff = half * NK;                          // this thread's keys in a block
    const int r = qd * 32 + lane;
    const int q = q0 + r;
    const uint32_t trow = (qd * 32) << 16;
    const uint32_t tO = tmem + trow + 128;
    uint8_t* sP = smem + L::P_OFF;
    float* red = reinterpret_cast<float*>(smem + L::RED_OFF);
    float m = -FLT_MAX, l = 0.f;
    uint32_t dkey = 0;
    if constexpr (DROP) dkey = drop_key(drop.seed, drop.salt);
    if constexpr (L::QT) {
      // Q row r (128 B, swizzled in smem) -> TMEM as the A operand of S = Q K^T
      mbar_wait(q_full, 0);
      const uint32_t qrow = smem_u32(smem + L::Q_OFF + r * 128);
      uint32_t qw[32];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint4 u;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                     : "r"(qrow + ((k ^ (r & 7)) << 4)));
        qw[4 * k] = u.x; qw[4 * k + 1] = u.y; qw[4 * k + 2] = u.z; qw[4 * k + 3] = u.w;
      }
      if (SW == 4 || half == 0) tmem_st16(tmem + trow + L::TQ, qw);
      if (SW == 4 || half == 1) tmem_st16(tmem + trow + L::TQ + 16, qw + 16);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_tmem);
    }
    for (int j = 0; j < n_kb; ++j) {
      // keep bits of keys j*64 .. +63 for this row: the pre-drawn mask's two
      // coalesced words, requested before the wait so the load latency hides
      uint32_t mk0 = 0, mk1 = 0;
      if constexpr (DROP) {
        const int kk0 = j * TA_BN;
        if (drop.mask_q != nullptr && q < S) {
          const uint32_t* mq = drop.mask_q + (static_cast<uint64_t>(bh) * (S >> 5) + (kk0 >> 5)) * S + q;
          mk0 = __ldg(mq);
          if (kk0 + 32 < S) mk1 = __ldg(mq + S);
        }
      }
      if (warp == 4 && lane == 0) TRF(j, 0);
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      if (warp == 4 && lane == 0) TRF(j, 1);
      tc_fence_after();
      const uint32_t ts = tmem + trow + (j & 1) * TA_BN + koff;
      const int k0 = j * TA_BN + koff;   // this thread's first key
      const bool need_mask = (k0 + NK > S) || (CAUSAL && k0 + NK - 1 > q0);
      // One TMEM read of the block's scores (64 fp32 per row, in registers);
      // row max with 8 independent partial maxima (short dependency chains).
      // Masking is one compare per element against the row's key limit
      // (keys >= lim are dead: past the sequence or above the diagonal).
      const int lim = CAUSAL ? min(S, q + 1) : S;
      uint32_t sc[NK];
      tmem_ld32(ts, *reinterpret_cast<uint32_t(*)[32]>(sc));
      if constexpr (NK == 64) tmem_ld32(ts + 32, *reinterpret_cast<uint32_t(*)[32]>(sc + 32));
      tmem_ld_wait();
      // S_j consumed: the MMA warp may reuse this TMEM buffer
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[j & 1]);
      // masked scores -> -inf: exp2 gives exactly 0, no select per element
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < NK; ++i)
          if (k0 + i >= lim) sc[i] = __float_as_uint(-INFINITY);
      }
      // row max: 3-input FMNMX3, 8 independent chains
      float pm[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) pm[t] = __uint_as_float(sc[t]);
#pragma unroll
      for (int i = 8; i < NK; i += 16) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
          pm[t] = fmax3(pm[t], __uint_as_float(sc[i + t]), __uint_as_float(sc[i + 8 + t]));
      }
      float mx = fmax3(fmax3(pm[0], pm[1], pm[2]), fmax3(pm[3], pm[4], pm[5]),
                       fmaxf(pm[6], pm[7]));
      if constexpr (SW == 8) {
        // the row's other 32 keys are in the partner warp: exchange maxima
        // (double-buffered slot, 64-thread named barrier per lane quadrant)
        float* rb = red + (j & 1) * 256;
        rb[half * 128 + r] = mx;
        asm volatile("bar.sync %0, 64;" ::"r"(1 + static_cast<int>(qd)) : "memory");
        mx = fmaxf(mx, rb[(half ^ 1) * 128 + r]);
      }
      const float m_cand = fmaxf(m, mx * scale_log2);
      const bool grow = m_cand > m + 8.f;   // lazy: keep a stale max unless it grew > 2^8
      const float m_new = grow ? m_cand : m;
      const float corr = fast_exp2(m - m_new);  // 1 when !grow; 0 for the first block
      // P = exp2(s*scale - m) (scale-and-shift and the row sums two lanes per
      // FFMA2 / FADD2), row sum
      const uint64_t sc2 = f2pack(scale_log2, scale_log2), nm2 = f2pack(-m_new, -m_new);
      uint64_t ps2[4] = {0ull, 0ull, 0ull, 0ull};
      uint4 pk[NK / 8];
      const uint64_t dpair = (((static_cast<uint64_t>(bh) * S + q) * S) + k0) >> 1;

#pragma unroll
      for (int g = 0; g < NK / 8; ++g) {
        float f[8];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint64_t x2 = ffma2(f2pack(__uint_as_float(sc[g * 8 + 2 * t]),
                                           __uint_as_float(sc[g * 8 + 2 * t + 1])), sc2, nm2);
          float a, b;
          f2unpack(x2, a, b);
          // (exp2 moved to the FMA pipes by a polynomial for 1/4 or 1/2 of
          // the pairs, and the 8-warp split softmax, both measured no faster:
          // the phase is latency-bound on the MUFU results, r02z)
          f[2 * t] = fast_exp2(a);
          f[2 * t + 1] = fast_exp2(b);
          ps2[t] = fadd2(ps2[t], f2pack(f[2 * t], f[2 * t + 1]));
        }
        if constexpr (DROP) {
          if (drop.mask_q != nullptr) {
            const uint32_t mw = ((g + half * 4) < 4 ? mk0 : mk1) >> ((g & 3) * 8);
#pragma unroll
            for (int t = 0; t < 8; ++t) f[t] = ((mw >> t) & 1u) ? f[t] : 0.f;
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const uint32_t kk = drop_keep2(dkey, dpair + g * 4 + t, drop.thr);
              f[2 * t] = (kk & 1u) ? f[2 * t] : 0.f;
              f[2 * t + 1] = (kk & 2u) ? f[2 * t + 1] : 0.f;
            }
          }
        }
        pk[g] = pack8(f);
      }
      if (warp == 4 && lane == 0) TRF(j, 2);
      // P buffer: TMEM (single, last read by PV_{j-1}) or smem (j & 1, by PV_{j-2})
      if constexpr (L::PT) {
        if (j >= 1) mbar_wait(&o_full[(j - 1) & 1], ((j - 1) >> 1) & 1);
      } else {
        if (j >= 2) mbar_wait(&o_full[j & 1], ((j - 2) >> 1) & 1);
      }
      if (j >= 1 && __any_sync(0xffffffffu, grow)) {
        // rescale O in place: needs PV_{j-1} complete
        mbar_wait(&o_full[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
        {
#pragma unroll 1
          for (int c = (SW == 8 ? half * (D / 2) : 0); c < (SW == 8 ? (half + 1) * (D / 2) : D);
               c += 32) {
            uint32_t raw[32];
            tmem_ld32(tO + c, raw);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) raw[i] = __float_as_uint(__uint_as_float(raw[i]) * corr);
            tmem_st32(tO + c, raw);
          }
          tmem_st_wait();
        }
      }
      if constexpr (L::PT) {
        tmem_st16(tmem + trow + L::TP + (koff >> 1), reinterpret_cast<const uint32_t*>(pk));
        if constexpr (NK == 64)
          tmem_st16(tmem + trow + L::TP + 16, reinterpret_cast<const uint32_t*>(pk + 4));
        tmem_st_wait();
      } else {
        const uint32_t rowp = smem_u32(sP + (j & 1) * 128 * TA_BN * 2 + r * 128);
#pragma unroll
        for (int g = 0; g < NK / 8; ++g)
          sts128(rowp + (((g + (koff >> 3)) ^ (r & 7)) << 4), pk[g]);
      }
      if (warp == 4 && lane == 0) TRF(j, 3);
      float ps[8];
#pragma unroll
      for (int t = 0; t < 4; ++t) f2unpack(ps2[t], ps[2 * t], ps[2 * t + 1]);
      const float sum = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
      l = l * corr + sum;
      m = m_new;
    }
    if constexpr (SW == 8) {   // the row sum's other half is the partner warp's
      red[half * 128 + r] = l;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + static_cast<int>(qd)) : "memory");
      l += red[(half ^ 1) * 128 + r];
    }
    mbar_wait(&o_full[(n_kb - 1) & 1], ((n_kb - 1) >> 1) & 1);
    tc_fence_after();
    const float inv = (DROP ? drop.scale : 1.f) / l;
    __nv_bfloat16* orow = out + (static_cast<int64_t>(b) * S + q) * Hd + h * D;
#pragma unroll 1
    for (int c = (SW == 8 ? half * (D / 2) : 0); c < (SW == 8 ? (half + 1) * (D / 2) : D);
         c += 32) {
      uint32_t raw[32];
      tmem_ld32(tO + c, raw);
      tmem_ld_wait();
      if (q < S) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          float f[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) f[t] = __uint_as_float(raw[i + t]) * inv;
          *reinterpret_cast<uint4*>(orow + c + i) = pack8(f);
        }
      }
    }
    if (q < S && half == 0) lse[static_cast<int64_t>(bh) * S + q] = m + __log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}



// ===========================================================================
// Backward on tcgen05 (K3 of DESIGN.md). Deterministic: no atomics.
//   dkdv kernel: CTA = 128 keys of one (b, h); loops over 64-query blocks.
//     S^T = K Q^T, dP^T = V dO^T            (TMEM, double-buffered)
//     P^T = exp2(S^T*scale - lse[q]), dS^T = P^T (dP^T - delta[q])  (thread = key)
//     dV += P^T dO, dK += dS^T Q            (TMEM accumulators, A from smem)
//   dq kernel:   CTA = 128 queries; loops over 64-key blocks.
//     S = Q K^T, dP = dO V^T; dS = P (dP - delta)  (thread = query)
//     dQ += dS K
// The same smem tile serves as a K-major operand (QK^T) and as an MN-major
// operand (dS^T Q) through two descriptors — no transposes in memory.
// ===========================================================================
constexpr int TB_M = 128;  // rows owned by the CTA (keys for dkdv, queries for dq)
constexpr int TB_N = 64;   // inner block (queries for dkdv, keys for dq)
// 8 compute warps: two per TMEM lane quadrant, each owning half of the 64
// columns (the backward has no row reductions, so columns split freely).
constexpr int TB_CW = 8;
constexpr int TB_THREADS = 128 + 32 * TB_CW;

template <int D>
struct TbSmem {
  // D <= 64: 2 CTAs/SM (one S/dP/P buffer, 2 stages, 256 TMEM cols, < 113 KB
  // smem) so one CTA's prologue / final drain overlaps the other's loop.
  // D > 64: 1 CTA/SM with double buffers and 3 stages.
  static constexpr int NB = D <= 64 ? 1 : 2;   // S/dP (TMEM) and P/dS (smem) buffers
  static constexpr int NS = D <= 64 ? 2 : 3;   // stages of the streamed 64-row operands
  static constexpr int MINB = D <= 64 ? 2 : 1; // CTAs per SM
  static constexpr int CH = (D + 63) / 64;
  static constexpr int BIG = 128 * 128;   // one d-chunk of a 128-row tile
  static constexpr int SMALL = TB_N * 128;  // one d-chunk of a 64-row tile
  static constexpr int A_OFF = 0;                         // K (dkdv) / Q (dq)   [128 x D]
  static constexpr int B_OFF = A_OFF + BIG * CH;          // V (dkdv) / dO (dq)  [128 x D]
  static constexpr int X_OFF = B_OFF + BIG * CH;          // Q_i / K_j  [NS][64 x D]
  static constexpr int Y_OFF = X_OFF + NS * SMALL * CH;   // dO_i / V_j [NS][64 x D]
  static constexpr int P_OFF = Y_OFF + NS * SMALL * CH;   // P^T [NB][128 x 64] (dkdv only)
  static constexpr int G_OFF = P_OFF + NB * 128 * TB_N * 2;  // dS / dS^T [NB][128 x 64]
  static constexpr int V_OFF = G_OFF + NB * 128 * TB_N * 2;  // lse/delta [NS][2][64] f32
  static constexpr int BAR_OFF = V_OFF + NS * 2 * TB_N * 4;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
  static constexpr int TMEM_KV = NB * 128 + 2 * D <= 256 ? 256 : 512;  // dkdv allocation
  static constexpr int TMEM_Q = NB * 128 + D <= 256 ? 256 : 512;       // dq allocation
};

template <int D, bool CAUSAL, bool DROP>
__global__ void __launch_bounds__(TB_THREADS, TbSmem<D>::MINB)
    attn_bwd_dkdv_tc(const __grid_constant__ CUtensorMap tmQKV128,
                     const __grid_constant__ CUtensorMap tmQKV64,
                     const __grid_constant__ CUtensorMap tmDO64, const float* __restrict__ lse,
                     const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, int S,
                     int H, float scale_log2, float scale, AttnDrop drop) {
  using L = TbSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;     // [NS] (TMA tx + producer-warp arrive for lse/delta)
  uint64_t* q_empty = bars + 5;    // [NS]
  uint64_t* st_full = bars + 9;    // [2]
  uint64_t* st_empty = bars + 11;  // [2]
  uint64_t* p_full = bars + 13;    // [2]
  uint64_t* p_empty = bars + 15;   // [2]
  uint64_t* acc_full = bars + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);

  const int kb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int k0 = kb * TB_M;
  const int n_qb = (S + TB_N - 1) / TB_N;
  const int i0 = CAUSAL ? k0 / TB_N : 0;
  const int n_it = n_qb - i0;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int Hd = H * D;
  const float* lse_bh = lse + static_cast<int64_t>(bh) * S;
  const float* del_bh = delta + static_cast<int64_t>(bh) * S;
  float* sv = reinterpret_cast<float*>(smem + L::V_OFF);  // [stage][lse|delta][64]

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV128);
    tma_prefetch(&tmQKV64);
    tma_prefetch(&tmDO64);
    mbar_init(kv_full, 1);
    for (int i = 0; i < L::NS; ++i) {
      mbar_init(&q_full[i], 2);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], TB_CW);
      mbar_init(&p_full[i], TB_CW);
      mbar_init(&p_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, L::TMEM_KV);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int NB = L::NB;
  const uint32_t tS = tmem, tP = tmem + NB * 64, tDV = tmem + NB * 128, tDK = tmem + NB * 128 + D;

  if (warp == 0) {
    // ===== producer: K/V once; per query block Q_i, dO_i (TMA) + lse/delta (warp) =====
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * L::BIG * L::CH);
#pragma unroll
      for (int c = 0; c < L::CH; ++c) {
        tma_load_3d(smem + L::A_OFF + c * L::BIG, &tmQKV128, kv_full, Hd + h * D + c * 64, k0, b);
        tma_load_3d(smem + L::B_OFF + c * L::BIG, &tmQKV128, kv_full, 2 * Hd + h * D + c * 64,
                    k0, b);
      }
    }
    for (int it = 0; it < n_it; ++it) {
      const int st = it % L::NS;
      const uint32_t ph = (it / L::NS) & 1;
      const int qi = (i0 + it) * TB_N;
      // lse/delta rows of a full 64-query block arrive by bulk copy on the
      // same barrier (no thread waits on global latency); a ragged last
      // block is loaded by the warp.
      const bool full_blk = qi + TB_N <= S && ((reinterpret_cast<uintptr_t>(lse_bh + qi) |
                                                reinterpret_cast<uintptr_t>(del_bh + qi)) & 15) == 0;
      float* dst = sv + st * 2 * TB_N;
      if (lane == 0) {
        mbar_wait(&q_empty[st], ph ^ 1);
        mbar_expect_tx(&q_full[st], 2 * L::SMALL * L::CH + (full_blk ? 2 * TB_N * 4 : 0));
#pragma unroll
        for (int c = 0; c < L::CH; ++c) {
          tma_load_3d(smem + L::X_OFF + st * L::SMALL * L::CH + c * L::SMALL, &tmQKV64,
                      &q_full[st], h * D + c * 64, qi, b);
          tma_load_3d(smem + L::Y_OFF + st * L::SMALL * L::CH + c * L::SMALL, &tmDO64,
                      &q_full[st], h * D + c * 64, qi, b);
        }
        if (full_blk) {
          bulk_g2s(dst, lse_bh + qi, TB_N * 4, &q_full[st]);
          bulk_g2s(dst + TB_N, del_bh + qi, TB_N * 4, &q_full[st]);
          mbar_arrive(&q_full[st]);
        }
      }
      if (!full_blk) {
        __syncwarp();
        mbar_wait(&q_empty[st], ph ^ 1);  // all lanes: stage free
        for (int t = lane; t < TB_N; t += 32) {
          const int q = qi + t;
          dst[t] = q < S ? lse_bh[q] : 0.f;
          dst[TB_N + t] = q < S ? del_bh[q] : 0.f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idST = idesc_bf16(128, TB_N, false, false);
      constexpr uint32_t idG = idesc_bf16(128, D, false, true);
      const uint32_t sK = smem_u32(smem + L::A_OFF), sV = smem_u32(smem + L::B_OFF);
      mbar_wait(kv_full, 0);
      auto issue_grad = [&](int it) {
        const int st = it % NB;
        const int qs = it % L::NS;
        mbar_wait(&p_full[st], (it / NB) & 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + L::X_OFF + qs * L::SMALL * L::CH);
        const uint32_t sdO = smem_u32(smem + L::Y_OFF + qs * L::SMALL * L::CH);
        const uint32_t sPt = smem_u32(smem + L::P_OFF + st * 128 * TB_N * 2);
        const uint32_t sdSt = smem_u32(smem + L::G_OFF + st * 128 * TB_N * 2);
#pragma unroll
        for (int k = 0; k < TB_N / 16; ++k) {
          const uint32_t acc = (it > 0 || k > 0) ? 1u : 0u;
          umma_f16(tDV, sdesc_sw128(sPt + k * 32, 16, 1024),
                   sdesc_sw128(sdO + k * 2048, L::SMALL, 1024), idG, acc);
          umma_f16(tDK, sdesc_sw128(sdSt + k * 32, 16, 1024),
                   sdesc_sw128(sQ + k * 2048, L::SMALL, 1024), idG, acc);
        }
        umma_commit(&p_empty[st]);
        umma_commit(&q_empty[qs]);
      };
      for (int it = 0; it < n_it; ++it) {
        const int st = it % NB;
        const int qs = it % L::NS;
        mbar_wait(&q_full[qs], (it / L::NS) & 1);
        mbar_wait(&st_empty[st], ((it / NB) & 1) ^ 1);
        tc_fence_after();
        const uint32_t sQ = smem_u32(smem + L::X_OFF + qs * L::SMALL * L::CH);
        const uint32_t sdO = smem_u32(smem + L::Y_OFF + qs * L::SMALL * L::CH);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t ob = (k >> 2) * L::BIG + (k & 3) * 32;
          const uint32_t os = (k >> 2) * L::SMALL + (k & 3) * 32;
          umma_f16(tS + st * TB_N, sdesc_sw128(sK + ob, 16, 1024), sdesc_sw128(sQ + os, 16, 1024),
                   idST, k > 0);
          umma_f16(tP + st * TB_N, sdesc_sw128(sV + ob, 16, 1024),
                   sdesc_sw128(sdO + os, 16, 1024), idST, k > 0);
        }
        umma_commit(&st_full[st]);
        if (it >= 1) issue_grad(it - 1);
      }
      if (n_it > 0) issue_grad(n_it - 1);
      umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    // ===== P^T / dS^T: thread = key row; this warp owns 32 of the 64 columns =====
    const uint32_t qd = warp & 3;
    const int chalf = static_cast<int>(warp - 4) >> 2;
    const int r = qd * 32 + lane;
    const int key = k0 + r;
    const int qlo = CAUSAL ? key : 0;
    const uint32_t trow = (qd * 32) << 16;
    uint32_t dkey = 0;
    if constexpr (DROP) dkey = drop_key(drop.seed, drop.salt);
    for (int it = 0; it < n_it; ++it) {
      const int st = it % NB;
      const int qi = (i0 + it) * TB_N;
      mbar_wait(&st_full[st], (it / NB) & 1);
      mbar_wait(&p_empty[st], ((it / NB) & 1) ^ 1);
      mbar_wait(&q_full[it % L::NS], (it / L::NS) & 1);  // lse/delta of this stage
      tc_fence_after();
      const float* slse = sv + (it % L::NS) * 2 * TB_N;
      const float* sdel = slse + TB_N;
      const bool need_mask = (qi + TB_N > S) || (CAUSAL && qi < k0 + TB_M - 1);
      const uint32_t rowP = smem_u32(smem + L::P_OFF + st * 128 * TB_N * 2 + r * 128);
      const uint32_t rowG = smem_u32(smem + L::G_OFF + st * 128 * TB_N * 2 + r * 128);
      uint32_t mword = 0;   // keep bits of queries qi+chalf*32 .. +31 for this key
      if constexpr (DROP) {
        const int qw = (qi >> 5) + chalf;
        if (drop.mask_k != nullptr && key < S && qw * 32 < S)
          mword = drop.mask_k[(static_cast<uint64_t>(bh) * (S >> 5) + qw) * S + key];
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        // 16 queries at a time (keeps the register footprint small enough
        // for 2 CTAs/SM)
        const int c = chalf * 32 + hh * 16;
        uint32_t rs[16], rd[16];
        tmem_ld16(tS + trow + st * TB_N + c, rs);
        tmem_ld16(tP + trow + st * TB_N + c, rd);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float lq[8], dq[8], fp[8], fg[8];
          const float4 a0 = *reinterpret_cast<const float4*>(slse + c + g * 8);
          const float4 a1 = *reinterpret_cast<const float4*>(slse + c + g * 8 + 4);
          const float4 d0 = *reinterpret_cast<const float4*>(sdel + c + g * 8);
          const float4 d1 = *reinterpret_cast<const float4*>(sdel + c + g * 8 + 4);
          lq[0] = a0.x; lq[1] = a0.y; lq[2] = a0.z; lq[3] = a0.w;
          lq[4] = a1.x; lq[5] = a1.y; lq[6] = a1.z; lq[7] = a1.w;
          dq[0] = d0.x; dq[1] = d0.y; dq[2] = d0.z; dq[3] = d0.w;
          dq[4] = d1.x; dq[5] = d1.y; dq[6] = d1.z; dq[7] = d1.w;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int i = g * 8 + t;
            float pv = fast_exp2(fmaf(__uint_as_float(rs[i]), scale_log2, -lq[t]));
            if (need_mask) {
              const int qq = qi + c + i;
              pv = (qq >= qlo && qq < S) ? pv : 0.f;
            }
            if constexpr (DROP) {
              // element (query qi+c+i, this key): the forward's key-major bit
              // mask when it wrote one, else one hash per element
              bool keep;
              if (drop.mask_k != nullptr) {
                keep = (mword >> (hh * 16 + i)) & 1u;
              } else {
                const uint64_t e = (static_cast<uint64_t>(bh) * S + (qi + c + i)) * S + key;
                const uint32_t bits = drop_bits(dkey, e >> 1);
                keep = ((key & 1) ? (bits >> 16) : (bits & 0xFFFFu)) >= drop.thr;
              }
              fp[t] = keep ? pv : 0.f;
              fg[t] = pv * ((keep ? __uint_as_float(rd[i]) * drop.scale : 0.f) - dq[t]);
            } else {
              fp[t] = pv;
              fg[t] = pv * (__uint_as_float(rd[i]) - dq[t]);
            }
          }
          const int chunk = (c >> 3) + g;
          const int sw = (chunk ^ (r & 7)) << 4;
          sts128(rowP + sw, pack8(fp));
          sts128(rowG + sw, pack8(fg));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&st_empty[st]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[st]);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    __nv_bfloat16* row = dqkv + (static_cast<int64_t>(b) * S + key) * (3 * Hd);
#pragma unroll 1
    for (int c = chalf * 32; c < D; c += 64) {
      uint32_t rk[32], rv[32];
      tmem_ld32(tDK + trow + c, rk);
      tmem_ld32(tDV + trow + c, rv);
      tmem_ld_wait();
      if (key < S) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          float fk[8], fv[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            fk[t] = n_it > 0 ? __uint_as_float(rk[i + t]) * scale : 0.f;
            fv[t] = n_it > 0 ? __uint_as_float(rv[i + t]) * (DROP ? drop.scale : 1.f) : 0.f;
          }
          *reinterpret_cast<uint4*>(row + Hd + h * D + c + i) = pack8(fk);
          *reinterpret_cast<uint4*>(row + 2 * Hd + h * D + c + i) = pack8(fv);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, L::TMEM_KV);
  }
}

template <int D, bool CAUSAL, bool DROP>
__global__ void __launch_bounds__(TB_THREADS, TbSmem<D>::MINB)
    attn_bwd_dq_tc(const __grid_constant__ CUtensorMap tmQKV128,
                   const __grid_constant__ CUtensorMap tmQKV64,
                   const __grid_constant__ CUtensorMap tmDO128, const float* __restrict__ lse,
                   const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, int S, int H,
                   int n_qb, float scale_log2, float scale, AttnDrop drop) {
  using L = TbSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* a_full = bars + 0;
  uint64_t* k_full = bars + 1;     // [NS]
  uint64_t* k_empty = bars + 5;    // [NS]
  uint64_t* s_full = bars + 9;     // [2]
  uint64_t* s_empty = bars + 11;   // [2]
  uint64_t* g_full = bars + 13;    // [2]
  uint64_t* g_empty = bars + 15;   // [2]
  uint64_t* acc_full = bars + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);

  const int qb = n_qb - 1 - static_cast<int>(blockIdx.x);
  const int bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int q0 = qb * TB_M;
  int n_kb = (S + TB_N - 1) / TB_N;
  if (CAUSAL) n_kb = min(n_kb, (q0 + TB_M + TB_N - 1) / TB_N);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int Hd = H * D;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV128);
    tma_prefetch(&tmQKV64);
    tma_prefetch(&tmDO128);
    mbar_init(a_full, 1);
    for (int i = 0; i < L::NS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], TB_CW);
      mbar_init(&g_full[i], TB_CW);
      mbar_init(&g_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, L::TMEM_Q);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int NB = L::NB;
  const uint32_t tS = tmem, tP = tmem + NB * 64, tDQ = tmem + NB * 128;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(a_full, 2 * L::BIG * L::CH);
#pragma unroll
      for (int c = 0; c < L::CH; ++c) {
        tma_load_3d(smem + L::A_OFF + c * L::BIG, &tmQKV128, a_full, h * D + c * 64, q0, b);
        tma_load_3d(smem + L::B_OFF + c * L::BIG, &tmDO128, a_full, h * D + c * 64, q0, b);
      }
      for (int j = 0; j < n_kb; ++j) {
        const int st = j % L::NS;
        mbar_wait(&k_empty[st], ((j / L::NS) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], 2 * L::SMALL * L::CH);
#pragma unroll
        for (int c = 0; c < L::CH; ++c) {
          tma_load_3d(smem + L::X_OFF + st * L::SMALL * L::CH + c * L::SMALL, &tmQKV64,
                      &k_full[st], Hd + h * D + c * 64, j * TB_N, b);
          tma_load_3d(smem + L::Y_OFF + st * L::SMALL * L::CH + c * L::SMALL, &tmQKV64,
                      &k_full[st], 2 * Hd + h * D + c * 64, j * TB_N, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16(128, TB_N, false, false);
      constexpr uint32_t idG = idesc_bf16(128, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::A_OFF), sdO = smem_u32(smem + L::B_OFF);
      mbar_wait(a_full, 0);
      auto issue_dq = [&](int j) {
        const int st = j % NB;
        const int ks = j % L::NS;
        mbar_wait(&g_full[st], (j / NB) & 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + L::X_OFF + ks * L::SMALL * L::CH);
        const uint32_t sdS = smem_u32(smem + L::G_OFF + st * 128 * TB_N * 2);
#pragma unroll
        for (int k = 0; k < TB_N / 16; ++k)
          umma_f16(tDQ, sdesc_sw128(sdS + k * 32, 16, 1024),
                   sdesc_sw128(sK + k * 2048, L::SMALL, 1024), idG, (j > 0 || k > 0) ? 1u : 0u);
        umma_commit(&g_empty[st]);
        umma_commit(&k_empty[ks]);
      };
      for (int j = 0; j < n_kb; ++j) {
        const int st = j % NB;
        const int ks = j % L::NS;
        mbar_wait(&k_full[ks], (j / L::NS) & 1);
        mbar_wait(&s_empty[st], ((j / NB) & 1) ^ 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + L::X_OFF + ks * L::SMALL * L::CH);
        const uint32_t sV = smem_u32(smem + L::Y_OFF + ks * L::SMALL * L::CH);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t ob = (k >> 2) * L::BIG + (k & 3) * 32;
          const uint32_t os = (k >> 2) * L::SMALL + (k & 3) * 32;
          umma_f16(tS + st * TB_N, sdesc_sw128(sQ + ob, 16, 1024), sdesc_sw128(sK + os, 16, 1024),
                   idS, k > 0);
          umma_f16(tP + st * TB_N, sdesc_sw128(sdO + ob, 16, 1024),
                   sdesc_sw128(sV + os, 16, 1024), idS, k > 0);
        }
        umma_commit(&s_full[st]);
        if (j >= 1) issue_dq(j - 1);
      }
      issue_dq(n_kb - 1);
      umma_commit(acc_full);
    }
  } else if (warp >= 4) {
    const uint32_t qd = warp & 3;
    const int chalf = static_cast<int>(warp - 4) >> 2;
    const int r = qd * 32 + lane;
    const int q = q0 + r;
    const uint32_t trow = (qd * 32) << 16;
    const int lim = CAUSAL ? min(S, q + 1) : S;
    const float lrow = q < S ? lse[static_cast<int64_t>(bh) * S + q] : 0.f;
    const float drow = q < S ? delta[static_cast<int64_t>(bh) * S + q] : 0.f;
    uint32_t dkey = 0;
    if constexpr (DROP) dkey = drop_key(drop.seed, drop.salt);
    for (int j = 0; j < n_kb; ++j) {
      const int st = j % NB;
      const int kj = j * TB_N;
      mbar_wait(&s_full[st], (j / NB) & 1);
      mbar_wait(&g_empty[st], ((j / NB) & 1) ^ 1);
      tc_fence_after();
      const bool need_mask = (kj + TB_N > S) || (CAUSAL && kj + TB_N - 1 > q0);
      const uint32_t rowG = smem_u32(smem + L::G_OFF + st * 128 * TB_N * 2 + r * 128);
      {
        const int c = chalf * 32;
        uint32_t rs[32], rd[32];
        tmem_ld32(tS + trow + st * TB_N + c, rs);
        tmem_ld32(tP + trow + st * TB_N + c, rd);
        tmem_ld_wait();
        float pv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          pv[i] = fast_exp2(fmaf(__uint_as_float(rs[i]), scale_log2, -lrow));
        if (need_mask) {
#pragma unroll
          for (int i = 0; i < 32; ++i) pv[i] = (kj + c + i < lim) ? pv[i] : 0.f;
        }
        if constexpr (DROP) {
          // dP = mask * dP_dropped / (1 - p); thread = query: the pre-drawn
          // word of keys kj+c .. +31, or pairs of keys hashed
          if (drop.mask_q != nullptr) {
            const int kw = (kj + c) >> 5;
            const uint32_t mw = (q < S && kw * 32 < S)
                ? drop.mask_q[(static_cast<uint64_t>(bh) * (S >> 5) + kw) * S + q] : 0u;
#pragma unroll
            for (int t = 0; t < 32; ++t)
              rd[t] = __float_as_uint(((mw >> t) & 1u) ? __uint_as_float(rd[t]) * drop.scale : 0.f);
          } else {
            const uint64_t p0 = ((static_cast<uint64_t>(bh) * S + q) * S + kj + c) >> 1;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              const uint32_t kk = drop_keep2(dkey, p0 + t, drop.thr);
              rd[2 * t] = __float_as_uint((kk & 1u) ? __uint_as_float(rd[2 * t]) * drop.scale : 0.f);
              rd[2 * t + 1] =
                  __float_as_uint((kk & 2u) ? __uint_as_float(rd[2 * t + 1]) * drop.scale : 0.f);
            }
          }
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float fg[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int i = g * 8 + t;
            fg[t] = pv[i] * (__uint_as_float(rd[i]) - drow);
          }
          const int chunk = (c >> 3) + g;
          sts128(rowG + ((chunk ^ (r & 7)) << 4), pack8(fg));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&g_full[st]);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    __nv_bfloat16* row = dqkv + (static_cast<int64_t>(b) * S + q) * (3 * Hd) + h * D;
#pragma unroll 1
    for (int c = chalf * 32; c < D; c += 64) {
      uint32_t rq[32];
      tmem_ld32(tDQ + trow + c, rq);
      tmem_ld_wait();
      if (q < S) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          float f[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) f[t] = __uint_as_float(rq[i + t]) * scale;
          *reinterpret_cast<uint4*>(row + c + i) = pack8(f);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, L::TMEM_Q);
  }
}

template <int D, bool CAUSAL, bool DROP>
int bwd_tc_t(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv,
             int64_t B, int64_t S, int64_t H, const AttnDrop& drop, cudaStream_t st) {
  using L = TbSmem<D>;
  CUtensorMap q128, q64, do64, do128;
  const uint64_t cols = 3 * H * D;
  if (!make_tmap_bsc(&q128, qkv, cols, S, B, 128) || !make_tmap_bsc(&q64, qkv, cols, S, B, 64) ||
      !make_tmap_bsc(&do64, dout, H * D, S, B, 64) || !make_tmap_bsc(&do128, dout, H * D, S, B, 128))
    return VP_ERR_UNSUPPORTED;
  auto k1 = attn_bwd_dkdv_tc<D, CAUSAL, DROP>;
  auto k2 = attn_bwd_dq_tc<D, CAUSAL, DROP>;
  if (cudaError_t e = smem_optin(k1, L::TOTAL); e != cudaSuccess) return e;
  if (cudaError_t e = smem_optin(k2, L::TOTAL); e != cudaSuccess) return e;
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = 1.4426950408889634f * scale;
  const int n_kb = static_cast<int>((S + TB_M - 1) / TB_M);
  k1<<<dim3(n_kb, static_cast<unsigned>(B * H)), TB_THREADS, L::TOTAL, st>>>(
      q128, q64, do64, lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), static_cast<int>(S),
      static_cast<int>(H), scale_log2, scale, drop);
  const int n_qb = static_cast<int>((S + TB_M - 1) / TB_M);
  k2<<<dim3(n_qb, static_cast<unsigned>(B * H)), TB_THREADS, L::TOTAL, st>>>(
      q128, q64, do128, lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), static_cast<int>(S),
      static_cast<int>(H), n_qb, scale_log2, scale, drop);
  return launch_status();
}

template <int D>
int bwd_tc_d(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv,
             int64_t B, int64_t S, int64_t H, int causal, const AttnDrop& dr, cudaStream_t st) {
  if (dr.seed)
    return causal ? bwd_tc_t<D, true, true>(qkv, dout, lse, delta, dqkv, B, S, H, dr, st)
                  : bwd_tc_t<D, false, true>(qkv, dout, lse, delta, dqkv, B, S, H, dr, st);
  return causal ? bwd_tc_t<D, true, false>(qkv, dout, lse, delta, dqkv, B, S, H, dr, st)
                : bwd_tc_t<D, false, false>(qkv, dout, lse, delta, dqkv, B, S, H, dr, st);
}
}  // namespace

int attention_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* delta,
                     void* dqkv, int64_t B, int64_t S, int64_t H, int64_t D, int causal,
                     float p, const uint64_t* seed, uint32_t salt, const uint32_t* mask_q,
                     const uint32_t* mask_k, cudaStream_t st) {
  if ((3 * H * D) % 8) return VP_ERR_UNSUPPORTED;
  const AttnDrop dr = (S % 32) ? make_attn_drop(p, seed, salt)
                               : make_attn_drop(p, seed, salt, mask_q, mask_k);
  if (dr.seed && (S & 1)) return VP_ERR_UNSUPPORTED;
  switch (D) {
    case 64: return bwd_tc_d<64>(qkv, dout, lse, delta, dqkv, B, S, H, causal, dr, st);
    case 96: return bwd_tc_d<96>(qkv, dout, lse, delta, dqkv, B, S, H, causal, dr, st);
    case 128: return bwd_tc_d<128>(qkv, dout, lse, delta, dqkv, B, S, H, causal, dr, st);
    default: return VP_ERR_UNSUPPORTED;
  }
}

namespace {
template <int D, bool CAUSAL, bool DROP>
int fwd_tc_t(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H,
             const AttnDrop& drop, cudaStream_t st) {
  using L = TaSmem<D>;
  CUtensorMap tm, tkv, tm1, tkv1;
  if (!make_tmap_bsc(&tm, qkv, 3 * H * D, S, B, 128)) return VP_ERR_UNSUPPORTED;
  if (!make_tmap_bsc(&tkv, qkv, 3 * H * D, S, B, TA_BN)) return VP_ERR_UNSUPPORTED;
  if (!make_tmap_bsc(&tm1, qkv, 3 * H * D, S, B, 128, true)) return VP_ERR_UNSUPPORTED;
  if (!make_tmap_bsc(&tkv1, qkv, 3 * H * D, S, B, TA_BN, true)) return VP_ERR_UNSUPPORTED;
  const int n_qb = static_cast<int>((S + TA_BM - 1) / TA_BM);
  dim3 grid(n_qb, static_cast<unsigned>(B * H));
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  // 4 softmax warps (a thread owns a whole row); VP_ATTN_FWD_SW=8 selects
  // the split-row variant for head_dim 64 — measured slower (179 vs 164 us
  // at 32x1024x16x64 causal, r02q): the extra warps do not hide more than
  // the max exchange and its named barrier add
  static const bool sw8 = getenv("VP_ATTN_FWD_SW") && atoi(getenv("VP_ATTN_FWD_SW")) == 8;
  if constexpr (D == 64) {
    if (sw8) {
      auto k = attn_fwd_tc<D, CAUSAL, DROP, 8>;
      if (cudaError_t e = smem_optin(k, L::TOTAL); e != cudaSuccess) return e;
      k<<<grid, 128 + 32 * 8, L::TOTAL, st>>>(tm, tkv, tm1, tkv1, reinterpret_cast<__nv_bfloat16*>(o), lse,
                                              static_cast<int>(S), static_cast<int>(H), n_qb,
                                              scale_log2, drop);
      return launch_status();
    }
  }
  auto k = attn_fwd_tc<D, CAUSAL, DROP, 4>;
  if (cudaError_t e = smem_optin(k, L::TOTAL); e != cudaSuccess) return e;
  k<<<grid, TA_THREADS, L::TOTAL, st>>>(tm, tkv, tm1, tkv1, reinterpret_cast<__nv_bfloat16*>(o), lse,
                                        static_cast<int>(S), static_cast<int>(H), n_qb,
                                        scale_log2, drop);
  return launch_status();
}

}  // namespace

#ifdef VP_BWD_TRACE
extern "C" int vp_debug_fwd_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_vp_ftrace, sizeof(g_vp_ftrace));
}
#endif
namespace {
template <int D>
int fwd_tc_d(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H, int causal,
             const AttnDrop& dr, cudaStream_t st) {
  if (dr.seed)
    return causal ? fwd_tc_t<D, true, true>(qkv, o, lse, B, S, H, dr, st)
                  : fwd_tc_t<D, false, true>(qkv, o, lse, B, S, H, dr, st);
  return causal ? fwd_tc_t<D, true, false>(qkv, o, lse, B, S, H, dr, st)
                : fwd_tc_t<D, false, false>(qkv, o, lse, B, S, H, dr, st);
}
}  // namespace

int attention_fwd_tc(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H,
                     int64_t D, int causal, float p, const uint64_t* seed, uint32_t salt,
                     const uint32_t* mask_q, cudaStream_t st) {
  if ((3 * H * D) % 8) return VP_ERR_UNSUPPORTED;
  const AttnDrop dr = make_attn_drop(p, seed, salt, (S % 32) ? nullptr : mask_q);
  if (dr.seed && (S & 1)) return VP_ERR_UNSUPPORTED;
  switch (D) {
    case 64: return fwd_tc_d<64>(qkv, o, lse, B, S, H, causal, dr, st);
    case 96: return fwd_tc_d<96>(qkv, o, lse, B, S, H, causal, dr, st);
    case 128: return fwd_tc_d<128>(qkv, o, lse, B, S, H, causal, dr, st);
    default: return VP_ERR_UNSUPPORTED;
  }
}

}  // namespace vp
