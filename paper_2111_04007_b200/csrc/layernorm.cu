// LayerNorm forward / backward (K4 of DESIGN.md). HBM-bound.
//
// Rows are short (h <= 4096 bf16 = 8 KB), so one warp owns a row: the row
// sits in registers as 16-byte vectors and the row statistics are warp
// shuffles. The grid is persistent (a few CTAs per SM) and every warp walks
// its rows with the NEXT row's loads issued before the current row is
// reduced and stored, so loads and stores of consecutive rows overlap
// instead of running as one load wave followed by one store wave.
//
// Backward, h <= 1024: one fused pass — dx (optionally accumulated into
// the residual gradient already in dx) plus per-lane register partials of
// dgamma = sum dy*xhat, dbeta = sum dy and, optionally, dsum = sum dx (the
// bias gradient of the residual branch that produced dy's consumer), reduced
// across the CTA in shared memory and across CTAs by a fixed-order kernel
// (deterministic). Wider rows use dx + column-partial kernels.
#include "common.cuh"
#include "sm100.cuh"

#include <algorithm>
#include <cstdlib>

namespace vp {
namespace {

constexpr int kWarps = 8;

template <int NV>
__device__ __forceinline__ void load_row(const __nv_bfloat16* p, int nvec, int lane, uint4 (&v)[NV]) {
  const uint4* r = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    v[i] = c < nvec ? r[c] : make_uint4(0u, 0u, 0u, 0u);
  }
}

// ----------------------------------------------------------------- forward
template <int NV>
__global__ void __launch_bounds__(kWarps * 32)
    ln_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                  const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y,
                  float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows,
                  int cols, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int nvec = cols >> 3;
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
  uint4 cur[NV];
  if (row < rows) load_row<NV>(x + row * cols, nvec, lane, cur);
  for (; row < rows; row += nwarps) {
    uint4 nxt[NV];
    const int64_t nrow = row + nwarps;
    if (nrow < rows) load_row<NV>(x + nrow * cols, nvec, lane, nxt);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float v[8];
      unpack8(cur[i], v);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
    const float mu = warp_sum(s) / cols;
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (lane + i * 32 < nvec) {
        float v[8];
        unpack8(cur[i], v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = v[j] - mu;
          ss += d * d;
        }
      }
    }
    const float rs = rsqrtf(warp_sum(ss) / cols + eps);
    if (lane == 0) {
      mean_out[row] = mu;
      rstd_out[row] = rs;
    }
    uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < nvec) {
        float v[8], gg[8], bb[8], o[8];
        unpack8(cur[i], v);
        unpack8(gv[c], gg);
        unpack8(bv[c], bb);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (v[j] - mu) * rs * gg[j] + bb[j];
        yr[c] = pack8(o);
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) cur[i] = nxt[i];
  }
}

// Shared-memory row slot of the TMA-staged backward ring (128 B aligned).
__host__ __device__ constexpr int ring_row_bytes(int cols) { return ((cols * 2 + 127) / 128) * 128; }

// Forward for wide rows: a group of W warps per row (1/W of the vectors
// each), row sums exchanged through shared memory with a named barrier per
// group; the next row's slice is loaded before the current one is reduced.
template <int W, int G, int NV>
__global__ void __launch_bounds__(W * G * 32)
    ln_fwd_group_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                        const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y,
                        float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows,
                        int cols, float eps) {
  __shared__ float xch[G][2][2][W];  // [group][row parity][sum | sumsq-dev][member]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp / W, mem = warp % W;
  const int nvec = cols >> 3, hvec = nvec / W, v0 = mem * hvec;
  const int64_t ngroups = static_cast<int64_t>(gridDim.x) * G;
  const uint4* gv = reinterpret_cast<const uint4*>(g) + v0;
  const uint4* bv = reinterpret_cast<const uint4*>(b) + v0;
  auto load = [&](int64_t row, uint4 (&v)[NV]) {
    const uint4* r = reinterpret_cast<const uint4*>(x + row * cols) + v0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      v[i] = c < hvec ? r[c] : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  int64_t row = static_cast<int64_t>(blockIdx.x) * G + grp;
  uint4 cur[NV];
  if (row < rows) load(row, cur);
  int parity = 0;
  for (; row < rows; row += ngroups, parity ^= 1) {
    uint4 nxt[NV];
    if (row + ngroups < rows) load(row + ngroups, nxt);
    float v[NV][8];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      unpack8(cur[i], v[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[i][j];
    }
    s = warp_sum(s);
    if (lane == 0) xch[grp][parity][0][mem] = s;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(W * 32) : "memory");
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) tot += xch[grp][parity][0][w];
    const float mu = tot / cols;
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      if (lane + i * 32 < hvec) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = v[i][j] - mu;
          ss += d * d;
        }
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) xch[grp][parity][1][mem] = ss;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(W * 32) : "memory");
    float tss = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) tss += xch[grp][parity][1][w];
    const float rs = rsqrtf(tss / cols + eps);
    if (mem == 0 && lane == 0) {
      mean_out[row] = mu;
      rstd_out[row] = rs;
    }
    uint4* yr = reinterpret_cast<uint4*>(y + row * cols) + v0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < hvec) {
        float gg[8], bb[8], o[8];
        unpack8(gv[c], gg);
        unpack8(bv[c], bb);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mu) * rs * gg[j] + bb[j];
        yr[c] = pack8(o);
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) cur[i] = nxt[i];
  }
}

// ------------------------------------------------------- fused backward
// ws[cta][3][cols]: dgamma, dbeta, dsum partials of this CTA's rows.
template <int NV, bool SUM>
__global__ void __launch_bounds__(kWarps * 32, 1)
    ln_bwd_fused_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                        const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                        const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx,
                        float* __restrict__ ws, int64_t rows, int cols, int accumulate) {
  extern __shared__ float red[];  // [kWarps][cols]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = cols >> 3;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  float ag[NV][8], ab[NV][8], as[SUM ? NV : 1][8];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ag[i][j] = 0.f;
      ab[i][j] = 0.f;
      if constexpr (SUM) as[i][j] = 0.f;
    }
  int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  uint4 xc[NV], dc[NV];
  if (row < rows) {
    load_row<NV>(x + row * cols, nvec, lane, xc);
    load_row<NV>(dy + row * cols, nvec, lane, dc);
  }
  for (; row < rows; row += nwarps) {
    uint4 pu[NV];
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
    if (accumulate) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = lane + i * 32;
        pu[i] = c < nvec ? dxr[c] : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    uint4 xn[NV], dn[NV];
    const int64_t nrow = row + nwarps;
    if (nrow < rows) {
      load_row<NV>(x + nrow * cols, nvec, lane, xn);
      load_row<NV>(dy + nrow * cols, nvec, lane, dn);
    }
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < nvec) {
        float xv[8], dv[8], gg[8];
        unpack8(xc[i], xv);
        unpack8(dc[i], dv);
        unpack8(gv[c], gg);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xv[j] - mu) * rs;
          const float gy = dv[j] * gg[j];
          s1 += gy;
          s2 += gy * xh;
          ag[i][j] += dv[j] * xh;
          ab[i][j] += dv[j];
        }
      }
    }
    const float m1 = warp_sum(s1) / cols, m2 = warp_sum(s2) / cols;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < nvec) {
        float xv[8], dv[8], gg[8], o[8];
        unpack8(xc[i], xv);
        unpack8(dc[i], dv);
        unpack8(gv[c], gg);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs * (dv[j] * gg[j] - m1 - (xv[j] - mu) * rs * m2);
        if (accumulate) {
          float p[8];
          unpack8(pu[i], p);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += p[j];
        }
        if constexpr (SUM) {
#pragma unroll
          for (int j = 0; j < 8; ++j) as[i][j] += o[j];
        }
        dxr[c] = pack8(o);
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      xc[i] = xn[i];
      dc[i] = dn[i];
    }
  }
  // CTA reduction, one quantity at a time through [kWarps][cols] smem
  constexpr int NQ = SUM ? 3 : 2;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    float* mine = red + warp * cols;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < nvec) {
        float* dst = mine + c * 8;
        const float* src = q == 0 ? ag[i] : (q == 1 ? ab[i] : as[SUM ? i : 0]);
        reinterpret_cast<float4*>(dst)[0] = make_float4(src[0], src[1], src[2], src[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(src[4], src[5], src[6], src[7]);
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) t += red[w * cols + c];
      ws[(static_cast<int64_t>(blockIdx.x) * 3 + q) * cols + c] = t;
    }
    __syncthreads();
  }
}

// ------------------------------------- fused backward, warp groups per row
// A row is split between the W warps of a group (1/W of the 16-byte vectors
// each; G groups per CTA): x and dy are unpacked once into fp32 registers,
// gamma stays in registers for the whole kernel, and the two row sums
// (dy*g, dy*g*xhat) are exchanged through shared memory with a named
// barrier over the group's W*32 threads. 1/W of the columns per thread keeps
// the register-resident partials (dgamma, dbeta, dsum) small: W=2 for
// h <= 1024 (12 warps per SM), W=4/8 for the 1920/3072/4096-wide rows of the
// larger models (8 warps per SM).
constexpr int kPairs = 6;
template <int W, int G, int NV, bool SUM>
__global__ void __launch_bounds__(W * G * 32, 1)
    ln_bwd_group_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                       const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                       const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx,
                       float* __restrict__ ws, int64_t rows, int cols, int accumulate) {
  extern __shared__ float red[];  // [G][cols] reduction buffer
  __shared__ float xch[G][2][W][2];  // [group][row parity][member][s1, s2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp / W, half = warp % W;  // group, member
  const int nvec = cols >> 3, hvec = nvec / W;   // vectors per member
  const int v0 = half * hvec;
  const int64_t npairs = static_cast<int64_t>(gridDim.x) * G;
  float gam[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < hvec) unpack8(reinterpret_cast<const uint4*>(g)[v0 + c], gam[i]);
    else
#pragma unroll
      for (int j = 0; j < 8; ++j) gam[i][j] = 0.f;
  }
  float ag[NV][8], ab[NV][8], as[SUM ? NV : 1][8];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ag[i][j] = 0.f;
      ab[i][j] = 0.f;
      if constexpr (SUM) as[i][j] = 0.f;
    }
  auto load_half = [&](const __nv_bfloat16* base, int64_t row, uint4 (&v)[NV]) {
    const uint4* r = reinterpret_cast<const uint4*>(base + row * cols) + v0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      v[i] = c < hvec ? r[c] : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  int64_t row = static_cast<int64_t>(blockIdx.x) * G + pair;
  uint4 xc[NV], dc[NV];
  if (row < rows) {
    load_half(x, row, xc);
    load_half(dy, row, dc);
  }
  int parity = 0;
  for (; row < rows; row += npairs, parity ^= 1) {
    uint4 pu[NV];
    if (accumulate) load_half(dx, row, pu);
    uint4 xn[NV], dn[NV];
    const int64_t nrow = row + npairs;
    if (nrow < rows) {
      load_half(x, nrow, xn);
      load_half(dy, nrow, dn);
    }
    const float mu = mean[row], rs = rstd[row];
    float xf[NV][8], df[NV][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      unpack8(xc[i], xf[i]);
      unpack8(dc[i], df[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xh = (xf[i][j] - mu) * rs;
        const float gy = df[i][j] * gam[i][j];
        s1 += gy;
        s2 = fmaf(gy, xh, s2);
        ag[i][j] = fmaf(df[i][j], xh, ag[i][j]);
        ab[i][j] += df[i][j];
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      xch[pair][parity][half][0] = s1;
      xch[pair][parity][half][1] = s2;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(W * 32) : "memory");
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {  // fixed order: every member gets the same sums
      t1 += xch[pair][parity][w][0];
      t2 += xch[pair][parity][w][1];
    }
    const float m1 = t1 / cols, m2 = t2 / cols;
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols) + v0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < hvec) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xf[i][j] - mu) * rs;
          o[j] = rs * fmaf(-xh, m2, fmaf(df[i][j], gam[i][j], -m1));
        }
        if (accumulate) {
          float pv[8];
          unpack8(pu[i], pv);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += pv[j];
        }
        if constexpr (SUM) {
#pragma unroll
          for (int j = 0; j < 8; ++j) as[i][j] += o[j];
        }
        dxr[c] = pack8(o);
      }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      xc[i] = xn[i];
      dc[i] = dn[i];
    }
  }
  // CTA reduction over the pairs, one quantity at a time
  constexpr int NQ = SUM ? 3 : 2;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    float* mine = red + pair * cols + v0 * 8;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < hvec) {
        const float* src = q == 0 ? ag[i] : (q == 1 ? ab[i] : as[SUM ? i : 0]);
        float4* dst = reinterpret_cast<float4*>(mine + c * 8);
        dst[0] = make_float4(src[0], src[1], src[2], src[3]);
        dst[1] = make_float4(src[4], src[5], src[6], src[7]);
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < G; ++w) t += red[w * cols + c];
      ws[(static_cast<int64_t>(blockIdx.x) * 3 + q) * cols + c] = t;
    }
    __syncthreads();
  }
}

// Dropout of the residual branch whose output gradient the LN backward
// finishes (K7): gy = mask(dx) / (1-p) is written beside dx and the column
// sums (the branch's bias gradient) are taken over gy as the GEMMs read it.
struct LnDrop {
  __nv_bfloat16* gy;
  const uint64_t* seed;
  uint32_t salt, thr;
  float scale;
};

// Fused backward, TMA-staged (rows <= 1024 wide): the group kernel's math
// with every group's x / dy / residual-gradient rows streamed through a ring
// of R slots in shared memory by 1-D bulk copies issued by the group's first
// lane, mean/rstd of the next row loaded one row ahead. The register version
// holds ~1 row per group in flight at 1 CTA/SM (its partials pin ~165
// registers) and reaches 3.75 TB/s; the ring keeps R rows per group in
// flight without registers. A slot is refilled right after the group's
// named barrier, by which point every member has its slice in registers.
template <int W, int G, int NV, bool SUM, int R, bool DROP = false>
__global__ void __launch_bounds__(W * G * 32)
    ln_bwd_ring_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                       const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                       const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx,
                       float* __restrict__ ws, int64_t rows, int cols, int accumulate,
                       LnDrop drop) {
  static_assert(!DROP || SUM, "the dropout variant also sums the branch bias gradient");
  extern __shared__ __align__(128) uint8_t ring_smem[];
  __shared__ float xch[G][2][W][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp / W, half = warp % W;
  const int nvec = cols >> 3, hvec = nvec / W;
  const int v0 = half * hvec;
  const int rb = ring_row_bytes(cols);
  const int nt = accumulate ? 3 : 2;  // x, dy (, dx) per slot
  const uint32_t bytes = static_cast<uint32_t>(cols) * 2u;
  float* red = reinterpret_cast<float*>(ring_smem);  // [G][cols], after the loop only
  uint8_t* ring = ring_smem + static_cast<size_t>(G) * cols * sizeof(float) +
                  static_cast<size_t>(pair) * R * 3 * rb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring_smem + static_cast<size_t>(G) * cols * 4 +
                                               static_cast<size_t>(G) * R * 3 * rb) +
                   pair * R;
  const int64_t npairs = static_cast<int64_t>(gridDim.x) * G;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * G + pair;
  const bool issuer = half == 0 && lane == 0;
  auto issue = [&](int slot, int64_t row) {
    uint8_t* d = ring + slot * 3 * rb;
    mbar_expect_tx(&bars[slot], bytes * nt);
    bulk_g2s(d, x + row * cols, bytes, &bars[slot]);
    bulk_g2s(d + rb, dy + row * cols, bytes, &bars[slot]);
    if (accumulate) bulk_g2s(d + 2 * rb, dx + row * cols, bytes, &bars[slot]);
  };
  if (issuer) {
#pragma unroll
    for (int r = 0; r < R; ++r) mbar_init(&bars[r], 1);
    fence_mbar_init();
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (row0 + r * npairs < rows) issue(r, row0 + r * npairs);
  }
  // members wait on barriers the issuer initialised
  asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(W * 32) : "memory");
  float gam[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < hvec) unpack8(reinterpret_cast<const uint4*>(g)[v0 + c], gam[i]);
    else
#pragma unroll
      for (int j = 0; j < 8; ++j) gam[i][j] = 0.f;
  }
  float ag[NV][8], ab[NV][8], as[SUM ? NV : 1][8];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ag[i][j] = 0.f;
      ab[i][j] = 0.f;
      if constexpr (SUM) as[i][j] = 0.f;
    }
  float mu = 0.f, rs = 0.f;
  if (row0 < rows) {
    mu = mean[row0];
    rs = rstd[row0];
  }
  uint32_t dkey = 0;
  if constexpr (DROP) dkey = drop_key(drop.seed, drop.salt);
  int it = 0, parity = 0;
  for (int64_t row = row0; row < rows; row += npairs, ++it, parity ^= 1) {
    const int slot = it % R;
    const int64_t nrow = row + npairs;
    float mu_n = 0.f, rs_n = 0.f;
    if (nrow < rows) {
      mu_n = mean[nrow];
      rs_n = rstd[nrow];
    }
    mbar_wait(&bars[slot], (it / R) & 1);
    const uint4* sx = reinterpret_cast<const uint4*>(ring + slot * 3 * rb) + v0;
    const uint4* sd = reinterpret_cast<const uint4*>(ring + slot * 3 * rb + rb) + v0;
    const uint4* sp = reinterpret_cast<const uint4*>(ring + slot * 3 * rb + 2 * rb) + v0;
    uint4 pu[NV];
    float xf[NV][8], df[NV][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      const bool ok = c < hvec;
      unpack8(ok ? sx[c] : make_uint4(0u, 0u, 0u, 0u), xf[i]);
      unpack8(ok ? sd[c] : make_uint4(0u, 0u, 0u, 0u), df[i]);
      pu[i] = (ok && accumulate) ? sp[c] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float xh = (xf[i][j] - mu) * rs;
        const float gy = df[i][j] * gam[i][j];
        s1 += gy;
        s2 = fmaf(gy, xh, s2);
        ag[i][j] = fmaf(df[i][j], xh, ag[i][j]);
        ab[i][j] += df[i][j];
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      xch[pair][parity][half][0] = s1;
      xch[pair][parity][half][1] = s2;
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(W * 32) : "memory");
    if (issuer) {
      const int64_t rrow = row + R * npairs;
      if (rrow < rows) {
        fence_async_smem();  // members' generic reads of the slot precede the refill
        issue(slot, rrow);
      }
    }
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      t1 += xch[pair][parity][w][0];
      t2 += xch[pair][parity][w][1];
    }
    const float m1 = t1 / cols, m2 = t2 / cols;
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols) + v0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < hvec) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xf[i][j] - mu) * rs;
          o[j] = rs * fmaf(-xh, m2, fmaf(df[i][j], gam[i][j], -m1));
        }
        if (accumulate) {
          float pv[8];
          unpack8(pu[i], pv);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += pv[j];
        }
        const uint4 ob = pack8(o);
        if constexpr (DROP) {
          // the branch sees mask(dx) of the bf16 dx; its bias gradient is
          // the column sum of what the GEMMs read (bf16 gy)
          float f[8];
          unpack8(ob, f);
          drop8(f, dkey, row * cols + static_cast<int64_t>(v0 + c) * 8, drop.thr, drop.scale);
          const uint4 gb = pack8(f);
          reinterpret_cast<uint4*>(drop.gy + row * cols)[v0 + c] = gb;
          unpack8(gb, f);
#pragma unroll
          for (int j = 0; j < 8; ++j) as[i][j] += f[j];
        } else if constexpr (SUM) {
#pragma unroll
          for (int j = 0; j < 8; ++j) as[i][j] += o[j];
        }
        dxr[c] = ob;
      }
    }
    mu = mu_n;
    rs = rs_n;
  }
  __syncthreads();  // CTA reduction of the partials (red[] sits in front of the ring)
  constexpr int NQ = SUM ? 3 : 2;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    float* mine = red + pair * cols + v0 * 8;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < hvec) {
        const float* src = q == 0 ? ag[i] : (q == 1 ? ab[i] : as[SUM ? i : 0]);
        float4* dst = reinterpret_cast<float4*>(mine + c * 8);
        dst[0] = make_float4(src[0], src[1], src[2], src[3]);
        dst[1] = make_float4(src[4], src[5], src[6], src[7]);
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < G; ++w) t += red[w * cols + c];
      ws[(static_cast<int64_t>(blockIdx.x) * 3 + q) * cols + c] = t;
    }
    __syncthreads();
  }
}

// -------------------------------------------------- split backward (wide)
// dx only: one warp per row (rows >> SMs here), row in registers.
template <int NV>
__global__ void __launch_bounds__(kWarps * 32)
    ln_bwd_dx_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                     const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                     const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx, int64_t rows,
                     int cols, int accumulate) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nvec = cols >> 3;
  uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const float mu = mean[row], rs = rstd[row];
  uint4 xu[NV], du[NV], pu[NV];
  load_row<NV>(x + row * cols, nvec, lane, xu);
  load_row<NV>(dy + row * cols, nvec, lane, du);
  if (accumulate) load_row<NV>(dx + row * cols, nvec, lane, pu);
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < nvec) {
      float xv[8], dv[8], gg[8];
      unpack8(xu[i], xv);
      unpack8(du[i], dv);
      unpack8(gv[c], gg);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float gy = dv[j] * gg[j];
        s1 += gy;
        s2 += gy * (xv[j] - mu) * rs;
      }
    }
  }
  const float m1 = warp_sum(s1) / cols, m2 = warp_sum(s2) / cols;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < nvec) {
      float xv[8], dv[8], gg[8], o[8];
      unpack8(xu[i], xv);
      unpack8(du[i], dv);
      unpack8(gv[c], gg);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = rs * (dv[j] * gg[j] - m1 - (xv[j] - mu) * rs * m2);
      if (accumulate) {
        float p[8];
        unpack8(pu[i], p);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += p[j];
      }
      dxr[c] = pack8(o);
    }
  }
}

// Column partials over a row range: dgamma, dbeta (from dy, x) and, when
// dsum is wanted, the sum of the finished dx. ws[part][3][cols].
__global__ void __launch_bounds__(256) ln_param_partial(const __nv_bfloat16* __restrict__ dy,
                                                        const __nv_bfloat16* __restrict__ x,
                                                        const __nv_bfloat16* __restrict__ dx,
                                                        const float* __restrict__ mean,
                                                        const float* __restrict__ rstd,
                                                        float* __restrict__ ws, int64_t rows,
                                                        int cols, int64_t rows_per_part) {
  __shared__ float sh[8][3][256 + 4];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * 32 + tx) * 8;
  const int64_t r0 = blockIdx.y * rows_per_part;
  const int64_t r1 = min(rows, r0 + rows_per_part);
  float ag[8], ab[8], as[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) ag[j] = ab[j] = as[j] = 0.f;
  if (c0 < cols) {
#pragma unroll 2
    for (int64_t r = r0 + ty; r < r1; r += 8) {
      float xv[8], dv[8];
      unpack8(*reinterpret_cast<const uint4*>(x + r * cols + c0), xv);
      unpack8(*reinterpret_cast<const uint4*>(dy + r * cols + c0), dv);
      const float mu = mean[r], rs = rstd[r];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ag[j] += dv[j] * (xv[j] - mu) * rs;
        ab[j] += dv[j];
      }
      if (dx) {
        float o[8];
        unpack8(*reinterpret_cast<const uint4*>(dx + r * cols + c0), o);
#pragma unroll
        for (int j = 0; j < 8; ++j) as[j] += o[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sh[ty][0][tx * 8 + j] = ag[j];
    sh[ty][1][tx * 8 + j] = ab[j];
    sh[ty][2][tx * 8 + j] = as[j];
  }
  __syncthreads();
  const int64_t cb = static_cast<int64_t>(blockIdx.x) * 256;
  for (int i = threadIdx.x; i < 3 * 256; i += 256) {
    const int q = i >> 8, cc = i & 255;
    if (cb + cc >= cols) continue;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][q][cc];
    ws[(static_cast<int64_t>(blockIdx.y) * 3 + q) * cols + cb + cc] = t;
  }
}

// Fixed-order reduction of ws[parts][3][cols] into dgamma, dbeta (and dsum):
// 32 columns x 32 part-lanes per block, 8 independent loads per thread.
__global__ void __launch_bounds__(1024) ln_param_reduce(const float* __restrict__ ws,
                                                        float* __restrict__ dgamma,
                                                        float* __restrict__ dbeta,
                                                        float* __restrict__ dsum, int parts,
                                                        int cols, int nq) {
  __shared__ float sh[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;  // over nq*cols
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int q = c / cols, col = c % cols;
  if (c < nq * cols) {
    const float* base = ws + static_cast<int64_t>(q) * cols + col;
    const int64_t stride = 3 * static_cast<int64_t>(cols);
    int p = ty;
    for (; p + 7 * 32 < parts; p += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += base[(p + u * 32) * stride];
    }
    for (; p < parts; p += 32) acc[0] += base[p * stride];
  }
  sh[ty][tx] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  __syncthreads();
  if (ty == 0 && c < nq * cols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += sh[i][tx];
    float* out = q == 0 ? dgamma : (q == 1 ? dbeta : dsum);
    out[col] += t;
  }
}

}  // namespace

// CTAs of the persistent row kernels: enough warps per SM to keep ~2 rows
// per warp in flight.
static int row_ctas(int64_t rows, int per_sm) {
  int64_t want = static_cast<int64_t>(device_sms()) * per_sm;
  const int64_t need = (rows + kWarps - 1) / kWarps;
  return static_cast<int>(want < need ? want : need);
}

}  // namespace vp

using namespace vp;

#define LN_DISPATCH(NVV, ...)                   \
  switch (NVV) {                                \
    case 1: { constexpr int NV = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int NV = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int NV = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int NV = 4; __VA_ARGS__; } break; \
    case 6: { constexpr int NV = 6; __VA_ARGS__; } break; \
    case 8: { constexpr int NV = 8; __VA_ARGS__; } break; \
    case 12: { constexpr int NV = 12; __VA_ARGS__; } break; \
    case 16: { constexpr int NV = 16; __VA_ARGS__; } break; \
    default: return VP_ERR_UNSUPPORTED;         \
  }

static int pick_nv(int64_t cols) {
  const int64_t need = (cols / 8 + 31) / 32;
  for (int nv : {1, 2, 3, 4, 6, 8, 12, 16})
    if (nv >= need) return nv;
  return -1;
}

extern "C" int vp_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y,
                                float* mean, float* rstd, int64_t rows, int64_t cols, float eps,
                                void* stream) {
  if (rows <= 0 || cols <= 0 || (cols % 8)) return VP_ERR_ARGS;
  const int nv = pick_nv(cols);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nvec = cols / 8;
  if (nv > 4 && nvec % 4 == 0 && (nvec / 4 + 31) / 32 <= 4 && !getenv("VP_LN_WARP_ROW")) {
    // wide rows: 4 warps per row, 2 rows per CTA, 4 CTAs per SM
    const int need = static_cast<int>((nvec / 4 + 31) / 32);
    const unsigned grid = static_cast<unsigned>(
        std::min<int64_t>(4 * static_cast<int64_t>(device_sms()), (rows + 1) / 2));
#define LNF(NN)                                                                              \
  ln_fwd_group_kernel<4, 2, NN><<<grid, 256, 0, st>>>(                                       \
      reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(gamma), \
      reinterpret_cast<const __nv_bfloat16*>(beta), reinterpret_cast<__nv_bfloat16*>(y), mean, \
      rstd, rows, static_cast<int>(cols), eps)
    if (need == 1) LNF(1);
    else if (need == 2) LNF(2);
    else if (need == 3) LNF(3);
    else LNF(4);
#undef LNF
    return launch_status();
  }
  const int grid = row_ctas(rows, 4);
  LN_DISPATCH(nv, ln_fwd_kernel<NV><<<grid, kWarps * 32, 0, st>>>(
                      reinterpret_cast<const __nv_bfloat16*>(x),
                      reinterpret_cast<const __nv_bfloat16*>(gamma),
                      reinterpret_cast<const __nv_bfloat16*>(beta),
                      reinterpret_cast<__nv_bfloat16*>(y), mean, rstd, rows,
                      static_cast<int>(cols), eps));
  return launch_status();
}

// Parts of the split path's column reduction: ~32 rows each, <= 296.
static int split_parts(int64_t rows) {
  int64_t parts = (rows + 31) / 32;
  if (parts > 296) parts = 296;
  return static_cast<int>(parts < 1 ? 1 : parts);
}

extern "C" int64_t vp_layernorm_ws_elems(int64_t cols) { return 3 * 296 * cols; }

namespace vp {
namespace {
// The LN backward of vp_layernorm_bwd_ex / _dropout (drop.gy != nullptr:
// the fused dropout variant, ring path only — VP_ERR_UNSUPPORTED otherwise).
int ln_bwd(const void* dy, const void* x, const void* gamma, const float* mean,
           const float* rstd, void* dx, float* dgamma, float* dbeta, float* dsum, int64_t rows,
           int64_t cols, int accumulate, float* workspace, const LnDrop& drop, void* stream) {
  if (rows <= 0 || cols <= 0 || (cols % 8) || !workspace) return VP_ERR_ARGS;
  const bool dropping = drop.gy != nullptr;
  if (dropping && !dsum) return VP_ERR_ARGS;
  const int nv = pick_nv(cols);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nq = dsum ? 3 : 2;
  const int c3 = static_cast<int>(nq * cols);
  int parts;
  const int64_t nvec = cols / 8;
  // warps per row W: 2 up to h=1024, else the smallest W in {4, 8} giving
  // <= 3 vectors per lane (W must divide the row's vectors)
  int W = 0, need = 0;
  if (nvec % 2 == 0 && (nvec / 2 + 31) / 32 <= 2) {
    W = 2;
    need = static_cast<int>((nvec / 2 + 31) / 32);
  } else if (nvec % 4 == 0 && (nvec / 4 + 31) / 32 <= 3) {
    W = 4;
    need = static_cast<int>((nvec / 4 + 31) / 32);
  } else if (nvec % 8 == 0 && (nvec / 8 + 31) / 32 <= 3) {
    W = 8;
    need = static_cast<int>((nvec / 8 + 31) / 32);
  }
  if (getenv("VP_LN_WARP_ROW")) W = 0;
  if (dropping && (W == 0 || getenv("VP_LN_NO_RING"))) return VP_ERR_UNSUPPORTED;
  if (W) {
    auto launch = [&](auto kern, int G) {
      parts = static_cast<int>(std::min<int64_t>(device_sms(), (rows + G - 1) / G));
      const size_t smem = static_cast<size_t>(G) * cols * sizeof(float);
      smem_optin(reinterpret_cast<const void*>(kern), 96 * 1024);
      kern<<<parts, W * G * 32, smem, st>>>(
          reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(x),
          reinterpret_cast<const __nv_bfloat16*>(gamma), mean, rstd,
          reinterpret_cast<__nv_bfloat16*>(dx), workspace, rows, static_cast<int>(cols),
          accumulate);
    };
#define LN_G(WW, GG, NN)                                                              \
  (dsum ? launch(ln_bwd_group_kernel<WW, GG, NN, true>, GG)                            \
        : launch(ln_bwd_group_kernel<WW, GG, NN, false>, GG))
    static const bool no_ring = getenv("VP_LN_NO_RING") != nullptr;
    int attr_err = 0;
    auto launch_ring = [&](auto kern, int WW, int GG, int R) {
      parts = static_cast<int>(std::min<int64_t>(device_sms(), (rows + GG - 1) / GG));
      const size_t smem = static_cast<size_t>(GG) * cols * sizeof(float) +
                          static_cast<size_t>(GG) * R * 3 * ring_row_bytes(cols) +
                          GG * R * sizeof(uint64_t);
      attr_err = smem_optin(reinterpret_cast<const void*>(kern), 200 * 1024);
      if (attr_err) return;
      kern<<<parts, WW * GG * 32, smem, st>>>(
          reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(x),
          reinterpret_cast<const __nv_bfloat16*>(gamma), mean, rstd,
          reinterpret_cast<__nv_bfloat16*>(dx), workspace, rows, static_cast<int>(cols),
          accumulate, drop);
    };
    // TMA-staged ring (R rows per group in flight); smem = G*cols*4 + G*R*3*row bytes
#define LN_R(WW, GG, NN, RR)                                                                 \
  (dropping ? launch_ring(ln_bwd_ring_kernel<WW, GG, NN, true, RR, true>, WW, GG, RR)        \
   : dsum   ? launch_ring(ln_bwd_ring_kernel<WW, GG, NN, true, RR>, WW, GG, RR)              \
            : launch_ring(ln_bwd_ring_kernel<WW, GG, NN, false, RR>, WW, GG, RR))
    if (!no_ring && W == 2) {
      if (need == 1) LN_R(2, kPairs, 1, 3);
      else LN_R(2, kPairs, 2, 3);
      if (attr_err) return attr_err;
    } else if (!no_ring && W == 4) {
      if (need == 1) LN_R(4, 3, 1, 3);
      else if (need == 2) LN_R(4, 3, 2, 3);
      else LN_R(4, 2, 3, 3);
      if (attr_err) return attr_err;
    } else if (!no_ring && W == 8) {
      if (need == 1) LN_R(8, 1, 1, 4);
      else if (need == 2) LN_R(8, 1, 2, 4);
      else LN_R(8, 1, 3, 4);
      if (attr_err) return attr_err;
    } else if (W == 2) {
      if (need == 1) LN_G(2, kPairs, 1);
      else LN_G(2, kPairs, 2);
    } else if (W == 4) {
      if (need == 1) LN_G(4, 2, 1);
      else if (need == 2) LN_G(4, 2, 2);
      else LN_G(4, 2, 3);
    } else {
      if (need == 1) LN_G(8, 1, 1);
      else if (need == 2) LN_G(8, 1, 2);
      else LN_G(8, 1, 3);
    }
#undef LN_G
#undef LN_R
  } else if (nv <= 4) {
    // one CTA per SM (register-resident partials); 8 rows per warp pass
    parts = row_ctas(rows, 1);
    const size_t smem = static_cast<size_t>(kWarps) * cols * sizeof(float);  // <= 32 KB
    auto launch = [&](auto kern) {
      kern<<<parts, kWarps * 32, smem, st>>>(
          reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(x),
          reinterpret_cast<const __nv_bfloat16*>(gamma), mean, rstd,
          reinterpret_cast<__nv_bfloat16*>(dx), workspace, rows, static_cast<int>(cols),
          accumulate);
    };
    switch (nv) {
      case 1: dsum ? launch(ln_bwd_fused_kernel<1, true>) : launch(ln_bwd_fused_kernel<1, false>); break;
      case 2: dsum ? launch(ln_bwd_fused_kernel<2, true>) : launch(ln_bwd_fused_kernel<2, false>); break;
      case 3: dsum ? launch(ln_bwd_fused_kernel<3, true>) : launch(ln_bwd_fused_kernel<3, false>); break;
      default: dsum ? launch(ln_bwd_fused_kernel<4, true>) : launch(ln_bwd_fused_kernel<4, false>); break;
    }
  } else {
    LN_DISPATCH(nv, ln_bwd_dx_kernel<NV><<<static_cast<unsigned>((rows + kWarps - 1) / kWarps),
                                           kWarps * 32, 0, st>>>(
                        reinterpret_cast<const __nv_bfloat16*>(dy),
                        reinterpret_cast<const __nv_bfloat16*>(x),
                        reinterpret_cast<const __nv_bfloat16*>(gamma), mean, rstd,
                        reinterpret_cast<__nv_bfloat16*>(dx), rows, static_cast<int>(cols),
                        accumulate));
    parts = split_parts(rows);
    const int64_t rpp = (rows + parts - 1) / parts;
    ln_param_partial<<<dim3(static_cast<unsigned>((cols + 255) / 256), parts), 256, 0, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(x),
        dsum ? reinterpret_cast<const __nv_bfloat16*>(dx) : nullptr, mean, rstd, workspace, rows,
        static_cast<int>(cols), rpp);
  }
  ln_param_reduce<<<(c3 + 31) / 32, 1024, 0, st>>>(workspace, dgamma, dbeta, dsum, parts,
                                                   static_cast<int>(cols), nq);
  return launch_status();
}
}  // namespace
}  // namespace vp

extern "C" int vp_layernorm_bwd_ex(const void* dy, const void* x, const void* gamma,
                                   const float* mean, const float* rstd, void* dx, float* dgamma,
                                   float* dbeta, float* dsum, int64_t rows, int64_t cols,
                                   int accumulate, float* workspace, void* stream) {
  return ln_bwd(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, dsum, rows, cols, accumulate,
                workspace, LnDrop{nullptr, nullptr, 0u, 0u, 1.f}, stream);
}

extern "C" int vp_layernorm_bwd_dropout(const void* dy, const void* x, const void* gamma,
                                        const float* mean, const float* rstd, void* dx,
                                        float* dgamma, float* dbeta, float* dsum, void* gy,
                                        float p, const uint64_t* seed, uint32_t salt,
                                        int64_t rows, int64_t cols, int accumulate,
                                        float* workspace, void* stream) {
  if (!gy || !seed || !dsum || p <= 0.f || p >= 1.f) return VP_ERR_ARGS;
  const uint32_t thr = drop_threshold(p);
  return ln_bwd(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, dsum, rows, cols, accumulate,
                workspace,
                LnDrop{reinterpret_cast<__nv_bfloat16*>(gy), seed, salt, thr, drop_scale(thr)},
                stream);
}

extern "C" int vp_layernorm_bwd(const void* dy, const void* x, const void* gamma,
                                const float* mean, const float* rstd, void* dx, float* dgamma,
                                float* dbeta, int64_t rows, int64_t cols, int accumulate,
                                float* workspace, void* stream) {
  return vp_layernorm_bwd_ex(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, nullptr, rows, cols,
                             accumulate, workspace, stream);
}
