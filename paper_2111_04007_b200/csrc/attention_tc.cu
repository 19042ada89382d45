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

#include <cudaTypedefs.h>

#include <cfloat>

namespace vp {
namespace {

constexpr int TA_BM = 128;
constexpr int TA_BN = 64;   // keys per block: TMEM S0|S1|O = 64+64+<=128 <= 256 cols -> 2 CTAs/SM
constexpr int TA_THREADS = 256;
constexpr int TA_STAGES = 2;

template <int D>
struct TaSmem {
  static constexpr int CH = (D + 63) / 64;           // 64-wide d-chunks (128 B rows)
  static constexpr int QCH = 128 * 128;              // one Q d-chunk: 128 rows x 128 B
  static constexpr int KCH = TA_BN * 128;            // one K/V d-chunk: 64 rows x 128 B
  static constexpr int QTILE = QCH * CH;
  static constexpr int KTILE = KCH * CH;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = QTILE;                // [stage]
  static constexpr int V_OFF = K_OFF + TA_STAGES * KTILE;
  static constexpr int P_OFF = V_OFF + TA_STAGES * KTILE;  // [128 x 64] bf16 = 16 KB
  static constexpr int BAR_OFF = P_OFF + 128 * TA_BN * 2;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D, bool CAUSAL>
__global__ void __launch_bounds__(TA_THREADS, 2)
    attn_fwd_tc(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmKV,
                __nv_bfloat16* __restrict__ out,
                float* __restrict__ lse, int S, int H, int n_qb, float scale_log2) {
  using L = TaSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;              // [2]
  uint64_t* kv_empty = bars + 3;             // [2]
  uint64_t* s_full = bars + 5;               // [2]
  uint64_t* s_empty = bars + 7;              // [2]
  uint64_t* o_full = bars + 9;
  uint64_t* p_full = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

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
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    mbar_init(o_full, 1);
    mbar_init(p_full, 4);
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
      for (int c = 0; c < L::CH; ++c)
        tma_load_3d(smem + L::Q_OFF + c * L::QCH, &tmQKV, q_full, h * D + c * 64, q0, b);
      for (int j = 0; j < n_kb; ++j) {
        const int st = j % TA_STAGES;
        mbar_wait(&kv_empty[st], ((j / TA_STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * L::KTILE);
#pragma unroll
        for (int c = 0; c < L::CH; ++c) {
          tma_load_3d(smem + L::K_OFF + st * L::KTILE + c * L::KCH, &tmKV, &kv_full[st],
                      Hd + h * D + c * 64, j * TA_BN, b);
          tma_load_3d(smem + L::V_OFF + st * L::KTILE + c * L::KCH, &tmKV, &kv_full[st],
                      2 * Hd + h * D + c * 64, j * TA_BN, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idS = idesc_bf16(128, TA_BN, false, false);
      constexpr uint32_t idO = idesc_bf16(128, D, false, true);
      const uint32_t sQ = smem_u32(smem + L::Q_OFF);
      const uint32_t sP = smem_u32(smem + L::P_OFF);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int j) {
        const int st = j % TA_STAGES;
        mbar_wait(p_full, j & 1);  // P_j written and O rescaled by the softmax warps
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + L::V_OFF + st * L::KTILE);
#pragma unroll
        for (int k = 0; k < TA_BN / 16; ++k) {
          // A = P [q][key] K-major (one 128 B row chunk): +32 B per 16 keys
          const uint64_t ad = sdesc_sw128(sP + k * 32, 16, 1024);
          // B = V [key][d] MN-major: +16 rows * 128 B per 16 keys; d-chunks KCH apart
          const uint64_t bd = sdesc_sw128(sV + k * 2048, L::KCH, 1024);
          umma_f16(tmem + 2 * TA_BN, ad, bd, idO, (j > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(o_full);
        umma_commit(&kv_empty[st]);
      };
      for (int j = 0; j < n_kb; ++j) {
        const int st = j % TA_STAGES;
        mbar_wait(&kv_full[st], (j / TA_STAGES) & 1);
        mbar_wait(&s_empty[j & 1], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + L::K_OFF + st * L::KTILE);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          umma_f16(tmem + (j & 1) * TA_BN,
                   sdesc_sw128(sQ + (k >> 2) * L::QCH + (k & 3) * 32, 16, 1024),
                   sdesc_sw128(sK + (k >> 2) * L::KCH + (k & 3) * 32, 16, 1024), idS, k > 0);
        }
        umma_commit(&s_full[j & 1]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(n_kb - 1);
    }
  } else if (warp >= 4) {
    // ===== softmax / correction / epilogue: thread = query row =====
    const uint32_t qd = warp & 3;
    const int r = qd * 32 + lane;
    const int q = q0 + r;
    const uint32_t trow = (qd * 32) << 16;
    const uint32_t tO = tmem + trow + 2 * TA_BN;
    uint8_t* sP = smem + L::P_OFF;
    float m = -FLT_MAX, l = 0.f;
    for (int j = 0; j < n_kb; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t ts = tmem + trow + (j & 1) * TA_BN;
      const int k0 = j * TA_BN;
      const bool need_mask = (k0 + TA_BN > S) || (CAUSAL && k0 + TA_BN - 1 > q0);
      // pass 1: row max
      float mx = -FLT_MAX;
#pragma unroll
      for (int c = 0; c < TA_BN; c += 32) {
        uint32_t raw[32];
        tmem_ld32(ts + c, raw);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x = __uint_as_float(raw[i]);
          if (need_mask) {
            const int key = k0 + c + i;
            if (key >= S || (CAUSAL && key > q)) x = -FLT_MAX;
          }
          mx = fmaxf(mx, x);
        }
      }
      const float m_cand = fmaxf(m, mx * scale_log2);
      const bool grow = m_cand > m + 8.f;   // lazy: keep a stale max unless it grew > 2^8
      const float m_new = grow ? m_cand : m;
      const float corr = fast_exp2(m - m_new);  // 1 when !grow; 0 for the first block
      if (j >= 1) {
        // PV_{j-1} done: O is final for m and the P buffer is free
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, grow)) {
#pragma unroll 1
          for (int c = 0; c < D; c += 32) {
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
      // pass 2: P = exp2(s*scale - m), row sum, P -> smem (bf16, swizzled)
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < TA_BN; c += 32) {
        uint32_t raw[32];
        tmem_ld32(ts + c, raw);
        tmem_ld_wait();
        // 32 keys = 4 x 16-byte chunks of the row's 128 B (64 keys)
        uint8_t* rowp = sP + r * 128;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float f[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int i = g * 8 + t;
            const float x = __uint_as_float(raw[i]);
            bool dead = false;
            if (need_mask) {
              const int key = k0 + c + i;
              dead = key >= S || (CAUSAL && key > q);
            }
            f[t] = dead ? 0.f : fast_exp2(fmaf(x, scale_log2, -m_new));
            sum += f[t];
          }
          const int chunk = ((c & 63) >> 3) + g;
          *reinterpret_cast<uint4*>(rowp + ((chunk ^ (r & 7)) << 4)) = pack8(f);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[j & 1]);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      l = l * corr + sum;
      m = m_new;
    }
    mbar_wait(o_full, (n_kb - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + (static_cast<int64_t>(b) * S + q) * Hd + h * D;
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
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
    if (q < S) lse[static_cast<int64_t>(bh) * S + q] = m + __log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode3() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3D map over a [B, S, cols] bf16 activation: box {64 cols, rows, 1}.
bool make_tmap_bsc(CUtensorMap* map, const void* base, uint64_t cols, uint64_t S, uint64_t B,
                   uint32_t rows) {
  auto fn = encode3();
  if (!fn) return false;
  cuuint64_t dims[3] = {cols, S, B};
  cuuint64_t strides[2] = {cols * 2, S * cols * 2};
  cuuint32_t box[3] = {64, rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, bool CAUSAL>
int fwd_tc_t(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H,
             cudaStream_t st) {
  using L = TaSmem<D>;
  CUtensorMap tm, tkv;
  if (!make_tmap_bsc(&tm, qkv, 3 * H * D, S, B, 128)) return VP_ERR_UNSUPPORTED;
  if (!make_tmap_bsc(&tkv, qkv, 3 * H * D, S, B, TA_BN)) return VP_ERR_UNSUPPORTED;
  auto k = attn_fwd_tc<D, CAUSAL>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const int n_qb = static_cast<int>((S + TA_BM - 1) / TA_BM);
  dim3 grid(n_qb, static_cast<unsigned>(B * H));
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  k<<<grid, TA_THREADS, L::TOTAL, st>>>(tm, tkv, reinterpret_cast<__nv_bfloat16*>(o), lse,
                                        static_cast<int>(S), static_cast<int>(H), n_qb,
                                        scale_log2);
  return launch_status();
}

}  // namespace

int attention_fwd_tc(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H,
                     int64_t D, int causal, cudaStream_t st) {
  if ((3 * H * D) % 8) return VP_ERR_UNSUPPORTED;
  switch (D) {
    case 64: return causal ? fwd_tc_t<64, true>(qkv, o, lse, B, S, H, st)
                           : fwd_tc_t<64, false>(qkv, o, lse, B, S, H, st);
    case 96: return causal ? fwd_tc_t<96, true>(qkv, o, lse, B, S, H, st)
                           : fwd_tc_t<96, false>(qkv, o, lse, B, S, H, st);
    case 128: return causal ? fwd_tc_t<128, true>(qkv, o, lse, B, S, H, st)
                            : fwd_tc_t<128, false>(qkv, o, lse, B, S, H, st);
    default: return VP_ERR_UNSUPPORTED;
  }
}

}  // namespace vp
