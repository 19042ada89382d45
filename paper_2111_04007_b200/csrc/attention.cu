// Fused multi-head attention forward / backward over packed qkv (K2/K3 of
// DESIGN.md). Flash-style: the S = QK^T tile, online softmax and PV stay
// on-chip; only O and the per-row log-sum-exp are written. Backward is
// deterministic (no atomics): one kernel produces dK/dV per key block,
// another dQ per query block, both recomputing P from the saved LSE.
//
// Round-1 implementation uses warp-level mma.sync (m16n8k16 bf16) with
// ldmatrix operand loads and cp.async double buffering; the tcgen05/TMEM
// version is the next step listed in DESIGN.md.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"

namespace vp {

int attention_fwd_tc(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H,
                     int64_t D, int causal, cudaStream_t st);
int attention_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* delta,
                     void* dqkv, int64_t B, int64_t S, int64_t H, int64_t D, int causal,
                     cudaStream_t st);
int64_t attention_bwd_fused_ws(int64_t B, int64_t S, int64_t H, int64_t D);
bool attention_bwd_fused_ok(int64_t D);
int attention_bwd_fused(const void* qkv, const void* o, const void* dout, const float* lse,
                        void* dqkv, float* ws, int64_t B, int64_t S, int64_t H, int causal,
                        float* dbias, cudaStream_t st);

namespace {

constexpr int ATT_BM = 64;  // query rows per CTA (16 per warp)
constexpr int ATT_BN = 64;  // keys per iteration
constexpr int ATT_THREADS = 128;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

template <int D>
struct Tile {
  static constexpr int LD = D + 8;  // padded row (bank-conflict-free ldmatrix)
  static constexpr int ELEMS = 64 * LD;
};

// Async load of 64 rows x D (bf16) starting at token row r0 into a padded
// smem tile; rows >= rows_valid are zero-filled.
template <int D>
__device__ __forceinline__ void load_tile(__nv_bfloat16* s, const __nv_bfloat16* g, int64_t ld,
                                          int r0, int rows_valid) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < 64 * CH; i += ATT_THREADS) {
    const int r = i / CH, c = i % CH;
    const bool ok = (r0 + r) < rows_valid;
    const __nv_bfloat16* src = g + static_cast<int64_t>(ok ? r0 + r : 0) * ld + c * 8;
    cp_async16(smem_u32(s + r * Tile<D>::LD + c * 8), src, ok);
  }
}

// Row-major 16x16 A-operand fragment (rows m0.., cols k0..) via ldmatrix.x4.
template <int D>
__device__ __forceinline__ void frag_a(const __nv_bfloat16* s, int m0, int k0, uint32_t (&a)[4]) {
  const int lane = threadIdx.x & 31;
  const int row = m0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int col = k0 + (lane >> 4) * 8;
  ldsm_x4(smem_u32(s + row * Tile<D>::LD + col), a);
}
// B operand for two n8 tiles (n0, n0+8) x k16 where B[k][n] = T[n][k]
// (T stored row-major, rows = n): non-transposed ldmatrix.
template <int D>
__device__ __forceinline__ void frag_b_nt(const __nv_bfloat16* s, int n0, int k0,
                                          uint32_t (&b)[4]) {
  const int lane = threadIdx.x & 31;
  const int row = n0 + (lane & 7) + (lane >> 4) * 8;
  const int col = k0 + ((lane >> 3) & 1) * 8;
  ldsm_x4(smem_u32(s + row * Tile<D>::LD + col), b);
  // b[0],b[1] -> n-tile n0 ; b[2],b[3] -> n-tile n0+8
}
// B operand for two n8 tiles where B[k][n] = T[k][n] (T row-major, rows = k):
// transposed ldmatrix.
template <int D>
__device__ __forceinline__ void frag_b_tn(const __nv_bfloat16* s, int k0, int n0,
                                          uint32_t (&b)[4]) {
  const int lane = threadIdx.x & 31;
  const int row = k0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int col = n0 + (lane >> 4) * 8;
  ldsm_x4_t(smem_u32(s + row * Tile<D>::LD + col), b);
}

// ============================================================== forward
template <int D, bool CAUSAL>
__global__ void __launch_bounds__(ATT_THREADS)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                    float* __restrict__ lse, int S, int H, float scale_log2) {
  extern __shared__ __align__(16) __nv_bfloat16 sm[];
  __nv_bfloat16* sQ = sm;
  __nv_bfloat16* sK = sQ + Tile<D>::ELEMS;           // [2]
  __nv_bfloat16* sV = sK + 2 * Tile<D>::ELEMS;       // [2]
  const int qb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int64_t ld = 3LL * H * D;
  const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * S * ld;
  const __nv_bfloat16* gq = base + h * D;
  const __nv_bfloat16* gk = base + (H + h) * D;
  const __nv_bfloat16* gv = base + (2 * H + h) * D;
  const int q0 = qb * ATT_BM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int n_blocks = (S + ATT_BN - 1) / ATT_BN;
  if (CAUSAL) n_blocks = min(n_blocks, (q0 + ATT_BM + ATT_BN - 1) / ATT_BN);

  load_tile<D>(sQ, gq, ld, q0, S);
  load_tile<D>(sK, gk, ld, 0, S);
  load_tile<D>(sV, gv, ld, 0, S);
  cp_commit();

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.f, 0.f};
  const int row_a = q0 + warp * 16 + (lane >> 2);  // rows row_a and row_a + 8

  for (int j = 0; j < n_blocks; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_blocks) {
      load_tile<D>(sK + (buf ^ 1) * Tile<D>::ELEMS, gk, ld, (j + 1) * ATT_BN, S);
      load_tile<D>(sV + (buf ^ 1) * Tile<D>::ELEMS, gv, ld, (j + 1) * ATT_BN, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const __nv_bfloat16* cK = sK + buf * Tile<D>::ELEMS;
    const __nv_bfloat16* cV = sV + buf * Tile<D>::ELEMS;
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a[4];
      frag_a<D>(sQ, warp * 16, kk * 16, a);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bb[4];
        frag_b_nt<D>(cK, nt * 16, kk * 16, bb);
        mma16816(s[2 * nt], a, bb[0], bb[1]);
        mma16816(s[2 * nt + 1], a, bb[2], bb[3]);
      }
    }
    // mask + online softmax (scores scaled into the log2 domain)
    const int k0 = j * ATT_BN;
    float mx[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + nt * 8 + (lane & 3) * 2 + (e & 1);
        const int row = row_a + (e >> 1) * 8;
        float v = s[nt][e] * scale_log2;
        if (key >= S || (CAUSAL && key > row)) v = -FLT_MAX;
        s[nt][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r]);
      corr[r] = exp2f(m_r[r] - mn);
      m_r[r] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = s[nt][e] == -FLT_MAX ? 0.f : exp2f(s[nt][e] - m_r[e >> 1]);
        s[nt][e] = p;
        rs[e >> 1] += p;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_r[r] = l_r[r] * corr[r] + rs[r];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      uint32_t a[4];
      a[0] = pack2(s[2 * t][0], s[2 * t][1]);
      a[1] = pack2(s[2 * t][2], s[2 * t][3]);
      a[2] = pack2(s[2 * t + 1][0], s[2 * t + 1][1]);
      a[3] = pack2(s[2 * t + 1][2], s[2 * t + 1][3]);
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t bb[4];
        frag_b_tn<D>(cV, t * 16, dn * 16, bb);
        mma16816(o[2 * dn], a, bb[0], bb[1]);
        mma16816(o[2 * dn + 1], a, bb[2], bb[3]);
      }
    }
    __syncthreads();
  }
  cp_wait<0>();
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  const int64_t ldo = static_cast<int64_t>(H) * D;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = row_a + r * 8;
    if (row >= S) continue;
    const float inv = 1.f / l_r[r];
    __nv_bfloat16* orow = out + (static_cast<int64_t>(b) * S + row) * ldo + h * D;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int col = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(orow + col) = pack2(o[i][2 * r] * inv, o[i][2 * r + 1] * inv);
    }
    if ((lane & 3) == 0) lse[static_cast<int64_t>(bh) * S + row] = m_r[r] + log2f(l_r[r]);
  }
}

// ============================================================== backward
// delta[b,h,s] = sum_d dO * O. One row (token, head) per group of D/8 lanes,
// each lane one 16-byte vector of O and of dO: a warp reads contiguous
// 512-byte spans; shuffle reduction inside the group.
template <int D>
__global__ void __launch_bounds__(256) attn_delta_kernel(const __nv_bfloat16* __restrict__ o,
                                                         const __nv_bfloat16* __restrict__ dout,
                                                         float* __restrict__ delta, int64_t tokens,
                                                         int S, int H) {
  constexpr int G = D / 8;  // lanes per row: 8 (D=64), 12 (D=96: 32 lanes hold 2 rows + 8 idle)
  constexpr int RPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int sub = lane / G, li = lane % G;
  const int64_t row = warp * RPW + sub;  // row = token * H + head
  float acc = 0.f;
  const bool ok = sub < RPW && row < tokens * H;
  if (ok) {
    const int64_t off = row * D + li * 8;  // rows are contiguous: [T, H*D]
    float a[8], g[8];
    unpack8(*reinterpret_cast<const uint4*>(o + off), a);
    unpack8(*reinterpret_cast<const uint4*>(dout + off), g);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += a[j] * g[j];
  }
  // group sum in fixed lane order (G need not be a power of two)
  float tot = 0.f;
#pragma unroll
  for (int k = 0; k < G; ++k) tot += __shfl_sync(0xffffffffu, acc, (sub * G + k) & 31);
  acc = tot;
  if (ok && li == 0) {
    const int64_t t = row / H;
    const int h = static_cast<int>(row % H);
    const int64_t b = t / S, s = t % S;
    delta[(b * H + h) * S + s] = acc;
  }
}

// dK, dV for one block of 64 keys; loops over query blocks.
template <int D, bool CAUSAL>
__global__ void __launch_bounds__(ATT_THREADS)
    attn_bwd_dkdv_kernel(const __nv_bfloat16* __restrict__ qkv,
                         const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                         const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, int S,
                         int H, float scale_log2, float scale) {
  extern __shared__ __align__(16) __nv_bfloat16 sm[];
  __nv_bfloat16* sK = sm;
  __nv_bfloat16* sV = sK + Tile<D>::ELEMS;
  __nv_bfloat16* sQ = sV + Tile<D>::ELEMS;        // [2]
  __nv_bfloat16* sdO = sQ + 2 * Tile<D>::ELEMS;   // [2]
  float* sL = reinterpret_cast<float*>(sdO + 2 * Tile<D>::ELEMS);  // [2][64]
  float* sDl = sL + 2 * 64;                                        // [2][64]
  const int kb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int64_t ld = 3LL * H * D, ldo = static_cast<int64_t>(H) * D;
  const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * S * ld;
  const __nv_bfloat16* gq = base + h * D;
  const __nv_bfloat16* gk = base + (H + h) * D;
  const __nv_bfloat16* gv = base + (2 * H + h) * D;
  const __nv_bfloat16* gdo = dout + static_cast<int64_t>(b) * S * ldo + h * D;
  const float* gl = lse + static_cast<int64_t>(bh) * S;
  const float* gd = delta + static_cast<int64_t>(bh) * S;
  const int k0 = kb * ATT_BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_q = (S + ATT_BM - 1) / ATT_BM;
  const int qb0 = CAUSAL ? k0 / ATT_BM : 0;

  auto load_q = [&](int qb, int buf) {
    load_tile<D>(sQ + buf * Tile<D>::ELEMS, gq, ld, qb * ATT_BM, S);
    load_tile<D>(sdO + buf * Tile<D>::ELEMS, gdo, ldo, qb * ATT_BM, S);
    if (threadIdx.x < 64) {
      const int q = qb * ATT_BM + threadIdx.x;
      sL[buf * 64 + threadIdx.x] = q < S ? gl[q] : 0.f;
      sDl[buf * 64 + threadIdx.x] = q < S ? gd[q] : 0.f;
    }
  };
  load_tile<D>(sK, gk, ld, k0, S);
  load_tile<D>(sV, gv, ld, k0, S);
  load_q(qb0, 0);
  cp_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int key_a = k0 + warp * 16 + (lane >> 2);  // keys key_a, key_a + 8

  for (int qb = qb0; qb < n_q; ++qb) {
    const int buf = (qb - qb0) & 1;
    __syncthreads();  // previous iteration done with buf^1 (incl. sL/sDl)
    if (qb + 1 < n_q) load_q(qb + 1, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const __nv_bfloat16* cQ = sQ + buf * Tile<D>::ELEMS;
    const __nv_bfloat16* cdO = sdO + buf * Tile<D>::ELEMS;
    const float* cL = sL + buf * 64;
    const float* cD = sDl + buf * 64;
    const int q0 = qb * ATT_BM;
    // S^T = K Q^T  and  dP^T = V dO^T   (rows = keys, cols = queries)
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ak[4], av[4];
      frag_a<D>(sK, warp * 16, kk * 16, ak);
      frag_a<D>(sV, warp * 16, kk * 16, av);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bq[4], bo[4];
        frag_b_nt<D>(cQ, nt * 16, kk * 16, bq);
        frag_b_nt<D>(cdO, nt * 16, kk * 16, bo);
        mma16816(st[2 * nt], ak, bq[0], bq[1]);
        mma16816(st[2 * nt + 1], ak, bq[2], bq[3]);
        mma16816(dpt[2 * nt], av, bo[0], bo[1]);
        mma16816(dpt[2 * nt + 1], av, bo[2], bo[3]);
      }
    }
    // P^T and dS^T
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = q0 + ql;
        const int key = key_a + (e >> 1) * 8;
        float p = exp2f(st[nt][e] * scale_log2 - cL[ql]);
        if (q >= S || key >= S || (CAUSAL && key > q)) p = 0.f;
        st[nt][e] = p;
        dpt[nt][e] = p * (dpt[nt][e] - cD[ql]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      uint32_t ap[4], ads[4];
      ap[0] = pack2(st[2 * t][0], st[2 * t][1]);
      ap[1] = pack2(st[2 * t][2], st[2 * t][3]);
      ap[2] = pack2(st[2 * t + 1][0], st[2 * t + 1][1]);
      ap[3] = pack2(st[2 * t + 1][2], st[2 * t + 1][3]);
      ads[0] = pack2(dpt[2 * t][0], dpt[2 * t][1]);
      ads[1] = pack2(dpt[2 * t][2], dpt[2 * t][3]);
      ads[2] = pack2(dpt[2 * t + 1][0], dpt[2 * t + 1][1]);
      ads[3] = pack2(dpt[2 * t + 1][2], dpt[2 * t + 1][3]);
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t bo[4], bq[4];
        frag_b_tn<D>(cdO, t * 16, dn * 16, bo);
        frag_b_tn<D>(cQ, t * 16, dn * 16, bq);
        mma16816(dv[2 * dn], ap, bo[0], bo[1]);
        mma16816(dv[2 * dn + 1], ap, bo[2], bo[3]);
        mma16816(dk[2 * dn], ads, bq[0], bq[1]);
        mma16816(dk[2 * dn + 1], ads, bq[2], bq[3]);
      }
    }
  }
  cp_wait<0>();
  const int64_t ldq = 3LL * H * D;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = key_a + r * 8;
    if (key >= S) continue;
    __nv_bfloat16* row = dqkv + (static_cast<int64_t>(b) * S + key) * ldq;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int col = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(row + (H + h) * D + col) =
          pack2(dk[i][2 * r] * scale, dk[i][2 * r + 1] * scale);
      *reinterpret_cast<uint32_t*>(row + (2 * H + h) * D + col) =
          pack2(dv[i][2 * r], dv[i][2 * r + 1]);
    }
  }
}

// dQ for one block of 64 queries; loops over key blocks.
template <int D, bool CAUSAL>
__global__ void __launch_bounds__(ATT_THREADS)
    attn_bwd_dq_kernel(const __nv_bfloat16* __restrict__ qkv,
                       const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                       const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, int S,
                       int H, float scale_log2, float scale) {
  extern __shared__ __align__(16) __nv_bfloat16 sm[];
  __nv_bfloat16* sQ = sm;
  __nv_bfloat16* sdO = sQ + Tile<D>::ELEMS;
  __nv_bfloat16* sK = sdO + Tile<D>::ELEMS;      // [2]
  __nv_bfloat16* sV = sK + 2 * Tile<D>::ELEMS;   // [2]
  const int qb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int64_t ld = 3LL * H * D, ldo = static_cast<int64_t>(H) * D;
  const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * S * ld;
  const __nv_bfloat16* gq = base + h * D;
  const __nv_bfloat16* gk = base + (H + h) * D;
  const __nv_bfloat16* gv = base + (2 * H + h) * D;
  const __nv_bfloat16* gdo = dout + static_cast<int64_t>(b) * S * ldo + h * D;
  const int q0 = qb * ATT_BM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int n_blocks = (S + ATT_BN - 1) / ATT_BN;
  if (CAUSAL) n_blocks = min(n_blocks, (q0 + ATT_BM + ATT_BN - 1) / ATT_BN);
  const int row_a = q0 + warp * 16 + (lane >> 2);
  float lrow[2], drow[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = row_a + r * 8;
    lrow[r] = row < S ? lse[static_cast<int64_t>(bh) * S + row] : 0.f;
    drow[r] = row < S ? delta[static_cast<int64_t>(bh) * S + row] : 0.f;
  }
  load_tile<D>(sQ, gq, ld, q0, S);
  load_tile<D>(sdO, gdo, ldo, q0, S);
  load_tile<D>(sK, gk, ld, 0, S);
  load_tile<D>(sV, gv, ld, 0, S);
  cp_commit();
  float dq[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int j = 0; j < n_blocks; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_blocks) {
      load_tile<D>(sK + (buf ^ 1) * Tile<D>::ELEMS, gk, ld, (j + 1) * ATT_BN, S);
      load_tile<D>(sV + (buf ^ 1) * Tile<D>::ELEMS, gv, ld, (j + 1) * ATT_BN, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const __nv_bfloat16* cK = sK + buf * Tile<D>::ELEMS;
    const __nv_bfloat16* cV = sV + buf * Tile<D>::ELEMS;
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t aq[4], ao[4];
      frag_a<D>(sQ, warp * 16, kk * 16, aq);
      frag_a<D>(sdO, warp * 16, kk * 16, ao);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bk[4], bv[4];
        frag_b_nt<D>(cK, nt * 16, kk * 16, bk);
        frag_b_nt<D>(cV, nt * 16, kk * 16, bv);
        mma16816(s[2 * nt], aq, bk[0], bk[1]);
        mma16816(s[2 * nt + 1], aq, bk[2], bk[3]);
        mma16816(dp[2 * nt], ao, bv[0], bv[1]);
        mma16816(dp[2 * nt + 1], ao, bv[2], bv[3]);
      }
    }
    const int k0 = j * ATT_BN;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + nt * 8 + (lane & 3) * 2 + (e & 1);
        const int row = row_a + (e >> 1) * 8;
        float p = exp2f(s[nt][e] * scale_log2 - lrow[e >> 1]);
        if (key >= S || row >= S || (CAUSAL && key > row)) p = 0.f;
        s[nt][e] = p * (dp[nt][e] - drow[e >> 1]);  // dS
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      uint32_t a[4];
      a[0] = pack2(s[2 * t][0], s[2 * t][1]);
      a[1] = pack2(s[2 * t][2], s[2 * t][3]);
      a[2] = pack2(s[2 * t + 1][0], s[2 * t + 1][1]);
      a[3] = pack2(s[2 * t + 1][2], s[2 * t + 1][3]);
#pragma unroll
      for (int dn = 0; dn < D / 16; ++dn) {
        uint32_t bk[4];
        frag_b_tn<D>(cK, t * 16, dn * 16, bk);
        mma16816(dq[2 * dn], a, bk[0], bk[1]);
        mma16816(dq[2 * dn + 1], a, bk[2], bk[3]);
      }
    }
    __syncthreads();
  }
  cp_wait<0>();
  const int64_t ldq = 3LL * H * D;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = row_a + r * 8;
    if (row >= S) continue;
    __nv_bfloat16* dst = dqkv + (static_cast<int64_t>(b) * S + row) * ldq + h * D;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const int col = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(dst + col) = pack2(dq[i][2 * r] * scale, dq[i][2 * r + 1] * scale);
    }
  }
}

template <typename K>
void set_smem(K k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

template <int D, bool CAUSAL>
int fwd_t(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H, cudaStream_t st) {
  const size_t smem = 5 * Tile<D>::ELEMS * sizeof(__nv_bfloat16);
  auto k = attn_fwd_kernel<D, CAUSAL>;
  set_smem(k, smem);
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  dim3 grid(static_cast<unsigned>((S + ATT_BM - 1) / ATT_BM), static_cast<unsigned>(B * H));
  k<<<grid, ATT_THREADS, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(qkv),
                                     reinterpret_cast<__nv_bfloat16*>(o), lse,
                                     static_cast<int>(S), static_cast<int>(H), scale_log2);
  return launch_status();
}

template <int D, bool CAUSAL>
int bwd_t(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
          float* delta, int64_t B, int64_t S, int64_t H, cudaStream_t st) {
  const int64_t tokens = B * S;
  constexpr int RPW = 32 / (D / 8);
  const int64_t warps = (tokens * H + RPW - 1) / RPW;
  attn_delta_kernel<D><<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(o), reinterpret_cast<const __nv_bfloat16*>(dout),
      delta, tokens, static_cast<int>(S), static_cast<int>(H));
  if (!getenv("VP_ATTN_LEGACY"))
    return attention_bwd_tc(qkv, dout, lse, delta, dqkv, B, S, H, D, CAUSAL, st);
  const float scale = 1.f / sqrtf(static_cast<float>(D));
  const float scale_log2 = 1.4426950408889634f * scale;
  dim3 grid(static_cast<unsigned>((S + 63) / 64), static_cast<unsigned>(B * H));
  const size_t smem_kv = 6 * Tile<D>::ELEMS * sizeof(__nv_bfloat16) + 4 * 64 * sizeof(float);
  auto k1 = attn_bwd_dkdv_kernel<D, CAUSAL>;
  set_smem(k1, smem_kv);
  k1<<<grid, ATT_THREADS, smem_kv, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<const __nv_bfloat16*>(dout),
      lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), static_cast<int>(S),
      static_cast<int>(H), scale_log2, scale);
  const size_t smem_q = 6 * Tile<D>::ELEMS * sizeof(__nv_bfloat16);
  auto k2 = attn_bwd_dq_kernel<D, CAUSAL>;
  set_smem(k2, smem_q);
  k2<<<grid, ATT_THREADS, smem_q, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<const __nv_bfloat16*>(dout),
      lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), static_cast<int>(S),
      static_cast<int>(H), scale_log2, scale);
  return launch_status();
}

}  // namespace

}  // namespace vp

using namespace vp;

extern "C" int vp_attention_fwd(const void* qkv, void* o, float* lse, int64_t batch, int64_t seq,
                                int64_t heads, int64_t head_dim, int causal, void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0) return VP_ERR_ARGS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // tcgen05/TMEM kernel (attention_tc.cu); the mma.sync kernel below is kept
  // only as an A/B reference (VP_ATTN_LEGACY=1).
  if (!getenv("VP_ATTN_LEGACY"))
    return attention_fwd_tc(qkv, o, lse, batch, seq, heads, head_dim, causal, st);
  switch (head_dim) {
    case 64: return causal ? fwd_t<64, true>(qkv, o, lse, batch, seq, heads, st)
                           : fwd_t<64, false>(qkv, o, lse, batch, seq, heads, st);
    case 96: return causal ? fwd_t<96, true>(qkv, o, lse, batch, seq, heads, st)
                           : fwd_t<96, false>(qkv, o, lse, batch, seq, heads, st);
    case 128: return causal ? fwd_t<128, true>(qkv, o, lse, batch, seq, heads, st)
                            : fwd_t<128, false>(qkv, o, lse, batch, seq, heads, st);
    default: return VP_ERR_UNSUPPORTED;
  }
}

// delta_ws: batch*heads*seq floats.
extern "C" int vp_attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse,
                                void* dqkv, float* delta_ws, int64_t batch, int64_t seq,
                                int64_t heads, int64_t head_dim, int causal, void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || !delta_ws) return VP_ERR_ARGS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
#define BWD(DD)                                                                          \
  return causal ? bwd_t<DD, true>(qkv, o, dout, lse, dqkv, delta_ws, batch, seq, heads, st) \
                : bwd_t<DD, false>(qkv, o, dout, lse, dqkv, delta_ws, batch, seq, heads, st)
  switch (head_dim) {
    case 64: BWD(64);
    case 96: BWD(96);
    case 128: BWD(128);
    default: return VP_ERR_UNSUPPORTED;
  }
#undef BWD
}

extern "C" int64_t vp_attention_bwd_ws_elems(int64_t batch, int64_t seq, int64_t heads,
                                             int64_t head_dim) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || head_dim <= 0) return 0;
  return attention_bwd_fused_ws(batch, seq, heads, head_dim);
}

extern "C" int vp_attention_bwd_ex(const void* qkv, const void* o, const void* dout,
                                   const float* lse, void* dqkv, float* workspace,
                                   int64_t ws_elems, int64_t batch, int64_t seq, int64_t heads,
                                   int64_t head_dim, int causal, int flags, float* dbias,
                                   void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || !workspace) return VP_ERR_ARGS;
  if (ws_elems < attention_bwd_fused_ws(batch, seq, heads, head_dim)) return VP_ERR_ARGS;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return VP_ERR_ARGS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool det = (flags & VP_ATTN_DETERMINISTIC) || getenv("VP_ATTN_DETERMINISTIC") ||
                   getenv("VP_ATTN_LEGACY");
  if (!det && attention_bwd_fused_ok(head_dim))
    return attention_bwd_fused(qkv, o, dout, lse, dqkv, workspace, batch, seq, heads, causal,
                               dbias, st);
  if (dbias) return VP_ERR_UNSUPPORTED;  // bias sums are fused only into the one-pass kernel
  return vp_attention_bwd(qkv, o, dout, lse, dqkv, workspace, batch, seq, heads, head_dim, causal,
                          stream);
}
