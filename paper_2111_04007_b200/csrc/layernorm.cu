// LayerNorm forward / backward (K4 of DESIGN.md). HBM-bound: one warp per
// row, the row held in registers as 16-byte vectors, warp-shuffle
// reductions, fp32 statistics. Backward reduces dgamma/dbeta
// deterministically: per-CTA partial sums -> a column-reduction kernel.
#include "common.cuh"

namespace vp {
namespace {

constexpr int kWarps = 8;

template <int NV>
__global__ void __launch_bounds__(kWarps * 32)
    ln_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                  const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y,
                  float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows,
                  int cols, float eps) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nvec = cols >> 3;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  float v[NV][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < nvec) {
      unpack8(xr[c], v[i]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[i][j];
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[i][j] = 0.f;
    }
  }
  const float mu = warp_sum(s) / cols;
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (lane + i * 32 < nvec) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = v[i][j] - mu;
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
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < nvec) {
      float gg[8], bb[8], o[8];
      unpack8(gv[c], gg);
      unpack8(bv[c], bb);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (v[i][j] - mu) * rs * gg[j] + bb[j];
      yr[c] = pack8(o);
    }
  }
}

// dx = rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat)); partial dgamma /
// dbeta per CTA into ws[gridDim.x][2][cols]. Each warp accumulates its rows'
// dgamma/dbeta into its own shared-memory slice (lane-private columns, no
// atomics); the row is streamed twice (the second pass hits L1/L2).
template <int NV>
__global__ void __launch_bounds__(kWarps * 32)
    ln_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                  const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                  const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx,
                  float* __restrict__ ws, int64_t rows, int cols, int accumulate,
                  int rows_per_cta) {
  // [kWarps][2][8][nvec]: element j of vector c at [j * nvec + c] so the 32
  // lanes of a warp (consecutive c) hit consecutive banks.
  extern __shared__ float red[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = cols >> 3;
  float* mine = red + warp * 2 * cols;
  for (int c = lane; c < 2 * cols; c += 32) mine[c] = 0.f;
  __syncwarp();
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  for (int64_t row = r0 + warp; row < r1; row += kWarps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * cols);
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < nvec) {
        float xv[8], dv[8], gg[8];
        unpack8(xr[c], xv);
        unpack8(dyr[c], dv);
        unpack8(gv[c], gg);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xv[j] - mu) * rs;
          const float gy = dv[j] * gg[j];
          s1 += gy;
          s2 += gy * xh;
          mine[j * nvec + c] += dv[j] * xh;
          mine[cols + j * nvec + c] += dv[j];
        }
      }
    }
    const float m1 = warp_sum(s1) / cols, m2 = warp_sum(s2) / cols;
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < nvec) {
        float xv[8], dv[8], gg[8], o[8];
        unpack8(xr[c], xv);
        unpack8(dyr[c], dv);
        unpack8(gv[c], gg);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs * (dv[j] * gg[j] - m1 - (xv[j] - mu) * rs * m2);
        if (accumulate) {
          float p[8];
          unpack8(dxr[c], p);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += p[j];
        }
        dxr[c] = pack8(o);
      }
    }
  }
  __syncthreads();
  // ws[part][2*cols] in natural column order
  for (int i = threadIdx.x; i < 2 * cols; i += blockDim.x) {
    const int half = i / cols, col = i % cols;
    const int src = half * cols + (col & 7) * nvec + (col >> 3);
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) acc += red[w * 2 * cols + src];
    ws[static_cast<int64_t>(blockIdx.x) * 2 * cols + i] = acc;
  }
}

// Small-row variant (cols <= 1024): each warp keeps its row (x, dy) in
// registers and its lanes' dgamma/dbeta partials in registers across all
// rows it handles; gamma is read from L1; one shared-memory reduction per
// CTA at the end.
template <int NV>
__global__ void __launch_bounds__(kWarps * 32)
    ln_bwd_reg_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                      const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                      const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx,
                      float* __restrict__ ws, int64_t rows, int cols, int accumulate,
                      int rows_per_cta) {
  extern __shared__ float red[];  // [kWarps][2][cols]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = cols >> 3;
  float dg[NV][8], db[NV][8];
  const uint4* gv = reinterpret_cast<const uint4*>(g);
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) dg[i][j] = db[i][j] = 0.f;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  for (int64_t row = r0 + warp; row < r1; row += kWarps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * cols);
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
    const float mu = mean[row], rs = rstd[row];
    uint4 xu[NV], du[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < nvec) {
        xu[i] = xr[c];
        du[i] = dyr[c];
      }
    }
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
          const float xh = (xv[j] - mu) * rs;
          const float gy = dv[j] * gg[j];
          s1 += gy;
          s2 += gy * xh;
          dg[i][j] += dv[j] * xh;
          db[i][j] += dv[j];
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
          unpack8(dxr[c], p);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += p[j];
        }
        dxr[c] = pack8(o);
      }
    }
  }
  float* mine = red + warp * 2 * cols;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < nvec) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        mine[c * 8 + j] = dg[i][j];
        mine[cols + c * 8 + j] = db[i][j];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * cols; i += blockDim.x) {
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) acc += red[w * 2 * cols + i];
    ws[static_cast<int64_t>(blockIdx.x) * 2 * cols + i] = acc;
  }
}


// dx only (no parameter gradients): one warp per row, row in registers,
// low register count -> full occupancy. Used with ln_param_partial below.
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
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * cols);
  uint4* dxr = reinterpret_cast<uint4*>(dx + row * cols);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const float mu = mean[row], rs = rstd[row];
  uint4 xu[NV], du[NV], pu[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < nvec) {
      xu[i] = xr[c];
      du[i] = dyr[c];
      if (accumulate) pu[i] = dxr[c];
    }
  }
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

// dgamma/dbeta partial column sums: block = 32 column-groups (8 columns,
// 16-byte loads) x 8 row-lanes over a row range; ws[part][2*cols].
__global__ void __launch_bounds__(256) ln_param_partial(const __nv_bfloat16* __restrict__ dy,
                                                        const __nv_bfloat16* __restrict__ x,
                                                        const float* __restrict__ mean,
                                                        const float* __restrict__ rstd,
                                                        float* __restrict__ ws, int64_t rows,
                                                        int cols, int64_t rows_per_part) {
  __shared__ float sh[8][2][256 + 4];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * 32 + tx) * 8;
  const int64_t r0 = blockIdx.y * rows_per_part;
  const int64_t r1 = min(rows, r0 + rows_per_part);
  float ag[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float ab[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
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
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sh[ty][0][tx * 8 + j] = ag[j];
    sh[ty][1][tx * 8 + j] = ab[j];
  }
  __syncthreads();
  const int64_t cb = static_cast<int64_t>(blockIdx.x) * 256;
  for (int i = threadIdx.x; i < 512; i += 256) {
    const int half = i >> 8, cc = i & 255;
    if (cb + cc >= cols) continue;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][half][cc];
    ws[static_cast<int64_t>(blockIdx.y) * 2 * cols + half * cols + cb + cc] = t;
  }
}

// 32 columns x 32 part-lanes per block, 8 independent loads in flight per
// thread; fixed-order tree => deterministic.
__global__ void __launch_bounds__(1024) ln_param_reduce(const float* __restrict__ ws,
                                                        float* __restrict__ dgamma,
                                                        float* __restrict__ dbeta, int parts,
                                                        int cols) {
  __shared__ float sh[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < 2 * cols) {
    int p = ty;
    for (; p + 7 * 32 < parts; p += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += ws[static_cast<int64_t>(p + u * 32) * 2 * cols + c];
    }
    for (; p < parts; p += 32) acc[0] += ws[static_cast<int64_t>(p) * 2 * cols + c];
  }
  sh[ty][tx] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  __syncthreads();
  if (ty == 0 && c < 2 * cols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += sh[i][tx];
    if (c < cols) dgamma[c] += t;
    else dbeta[c - cols] += t;
  }
}

}  // namespace

int ln_partials(int64_t rows) {
  // row partitions of the dgamma/dbeta column reduction: ~32 rows each
  // (4 per row-lane), at most 1024 partials.
  int64_t parts = (rows + 31) / 32;
  if (parts > 1024) parts = 1024;
  return static_cast<int>(parts < 1 ? 1 : parts);
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
  const dim3 grid(static_cast<unsigned>((rows + kWarps - 1) / kWarps));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LN_DISPATCH(nv, ln_fwd_kernel<NV><<<grid, kWarps * 32, 0, st>>>(
                      reinterpret_cast<const __nv_bfloat16*>(x),
                      reinterpret_cast<const __nv_bfloat16*>(gamma),
                      reinterpret_cast<const __nv_bfloat16*>(beta),
                      reinterpret_cast<__nv_bfloat16*>(y), mean, rstd, rows,
                      static_cast<int>(cols), eps));
  return launch_status();
}

// workspace: >= 2 * ln_partials(rows) * cols floats (callers pass 2*296*cols).
extern "C" int vp_layernorm_bwd(const void* dy, const void* x, const void* gamma,
                                const float* mean, const float* rstd, void* dx, float* dgamma,
                                float* dbeta, int64_t rows, int64_t cols, int accumulate,
                                float* workspace, void* stream) {
  if (rows <= 0 || cols <= 0 || (cols % 8) || !workspace) return VP_ERR_ARGS;
  const int nv = pick_nv(cols);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LN_DISPATCH(nv, ln_bwd_dx_kernel<NV><<<static_cast<unsigned>((rows + kWarps - 1) / kWarps),
                                         kWarps * 32, 0, st>>>(
                      reinterpret_cast<const __nv_bfloat16*>(dy),
                      reinterpret_cast<const __nv_bfloat16*>(x),
                      reinterpret_cast<const __nv_bfloat16*>(gamma), mean, rstd,
                      reinterpret_cast<__nv_bfloat16*>(dx), rows, static_cast<int>(cols),
                      accumulate));
  const int parts = ln_partials(rows);
  const int64_t rpp = (rows + parts - 1) / parts;
  ln_param_partial<<<dim3(static_cast<unsigned>((cols + 255) / 256), parts), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(x), mean,
      rstd, workspace, rows, static_cast<int>(cols), rpp);
  const int c2 = static_cast<int>(2 * cols);
  ln_param_reduce<<<(c2 + 31) / 32, 1024, 0, st>>>(workspace, dgamma, dbeta, parts,
                                                   static_cast<int>(cols));
  return launch_status();
}
