// HBM-bound fused kernels: embedding gather/scatter (K8), softmax
// cross-entropy fwd+bwd (K6), bias-grad column reduction, dropout (K7),
// residual add, grad-norm/overflow reduction (K11), fused AdamW (K10), casts.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace vp {
namespace {

// ---------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const int64_t* __restrict__ ids,
                                 const __nv_bfloat16* __restrict__ wte,
                                 const __nv_bfloat16* __restrict__ wpe,
                                 __nv_bfloat16* __restrict__ x, int64_t tokens, int64_t seq,
                                 int64_t hidden) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (t >= tokens) return;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = hidden >> 3;
  const uint4* a = reinterpret_cast<const uint4*>(wte + ids[t] * hidden);
  const uint4* p = reinterpret_cast<const uint4*>(wpe + (t % seq) * hidden);
  uint4* o = reinterpret_cast<uint4*>(x + t * hidden);
  for (int64_t c = lane; c < nvec; c += 32) {
    float fa[8], fp[8];
    unpack8(a[c], fa);
    unpack8(p[c], fp);
#pragma unroll
    for (int j = 0; j < 8; ++j) fa[j] += fp[j];
    o[c] = pack8(fa);
  }
}

__global__ void embed_bwd_tok_kernel(const int64_t* __restrict__ ids,
                                     const __nv_bfloat16* __restrict__ dx,
                                     float* __restrict__ dwte, int64_t tokens, int64_t hidden) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (t >= tokens) return;
  const int lane = threadIdx.x & 31;
  const uint4* g = reinterpret_cast<const uint4*>(dx + t * hidden);
  float* dst = dwte + ids[t] * hidden;
  for (int64_t c = lane; c < (hidden >> 3); c += 32) {
    float f[8];
    unpack8(g[c], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) atomicAdd(dst + c * 8 + j, f[j]);
  }
}

__global__ void embed_bwd_pos_kernel(const __nv_bfloat16* __restrict__ dx,
                                     float* __restrict__ dwpe, int64_t batch, int64_t seq,
                                     int64_t hidden) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= seq * hidden) return;
  float acc = 0.f;
  for (int64_t b = 0; b < batch; ++b) acc += __bfloat162float(dx[b * seq * hidden + i]);
  dwpe[i] += acc;
}

__global__ void embed_typed_fwd_kernel(const int64_t* __restrict__ ids,
                                       const int64_t* __restrict__ types,
                                       const __nv_bfloat16* __restrict__ wte,
                                       const __nv_bfloat16* __restrict__ wpe,
                                       const __nv_bfloat16* __restrict__ tte,
                                       __nv_bfloat16* __restrict__ x, int64_t tokens, int64_t seq,
                                       int64_t hidden) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (t >= tokens) return;
  const int lane = threadIdx.x & 31;
  const uint4* a = reinterpret_cast<const uint4*>(wte + ids[t] * hidden);
  const uint4* p = reinterpret_cast<const uint4*>(wpe + (t % seq) * hidden);
  const uint4* q = reinterpret_cast<const uint4*>(tte + types[t] * hidden);
  uint4* o = reinterpret_cast<uint4*>(x + t * hidden);
  for (int64_t c = lane; c < (hidden >> 3); c += 32) {
    float fa[8], fp[8], fq[8];
    unpack8(a[c], fa);
    unpack8(p[c], fp);
    unpack8(q[c], fq);
#pragma unroll
    for (int j = 0; j < 8; ++j) fa[j] += fp[j] + fq[j];
    o[c] = pack8(fa);
  }
}

__global__ void gelu_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                const __nv_bfloat16* __restrict__ pre,
                                __nv_bfloat16* __restrict__ dx, int64_t n) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i + 8 <= n) {
    float g[8], x[8];
    unpack8(*reinterpret_cast<const uint4*>(dy + i), g);
    unpack8(*reinterpret_cast<const uint4*>(pre + i), x);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float k0 = 0.7978845608028654f, k1 = 0.044715f;
      const float u = k0 * (x[j] + k1 * x[j] * x[j] * x[j]);
      const float t = tanhf(u);
      g[j] *= 0.5f * (1.f + t) + 0.5f * x[j] * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x[j] * x[j]);
    }
    *reinterpret_cast<uint4*>(dx + i) = pack8(g);
  } else {
    for (int64_t k = i; k < n; ++k) {
      const float x = __bfloat162float(pre[k]);
      const float k0 = 0.7978845608028654f, k1 = 0.044715f;
      const float t = tanhf(k0 * (x + k1 * x * x * x));
      dx[k] = __float2bfloat16(__bfloat162float(dy[k]) *
                               (0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 *
                                                       (1.f + 3.f * k1 * x * x)));
    }
  }
}

// ------------------------------------------------------------ cross-entropy
template <int THREADS>
__global__ void __launch_bounds__(THREADS)
    xent_kernel(__nv_bfloat16* __restrict__ logits, const int64_t* __restrict__ labels,
                float* __restrict__ loss_rows, float* __restrict__ loss_sum, int64_t vocab,
                float scale, const float* __restrict__ scale_dev) {
  if (scale_dev != nullptr) scale *= scale_dev[0];   // dynamic loss scale (device)
  const int64_t row = blockIdx.x;
  __nv_bfloat16* lr = logits + row * vocab;
  const int64_t label = labels[row];
  __shared__ float s_m[THREADS / 32], s_s[THREADS / 32];
  __shared__ float s_lse;
  float m = -FLT_MAX, s = 0.f;
  const int64_t nvec = vocab >> 3;
  const uint4* lv = reinterpret_cast<const uint4*>(lr);
  // 4 independent 16-byte loads in flight per thread, then the online
  // (max, sum-exp) update over the 32 values
  int64_t c = threadIdx.x;
  for (; c + 3 * THREADS < nvec; c += 4 * THREADS) {
    uint4 u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = lv[c + k * THREADS];
    float f[32];
#pragma unroll
    for (int k = 0; k < 4; ++k) unpack8(u[k], *reinterpret_cast<float(*)[8]>(f + 8 * k));
    float mm = f[0];
#pragma unroll
    for (int j = 1; j < 32; ++j) mm = fmaxf(mm, f[j]);
    if (mm > m) {
      s *= __expf(m - mm);
      m = mm;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) s += __expf(f[j] - m);
  }
  for (; c < nvec; c += THREADS) {
    float f[8];
    unpack8(lv[c], f);
    float mm = f[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) mm = fmaxf(mm, f[j]);
    if (mm > m) {
      s *= __expf(m - mm);
      m = mm;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += __expf(f[j] - m);
  }
  // warp then block merge of (max, sum)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const float os = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(m, om);
    s = s * __expf(m - nm) + os * __expf(om - nm);
    m = nm;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_m[w] = m;
    s_s[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = s_m[0], S = s_s[0];
    for (int i = 1; i < THREADS / 32; ++i) {
      const float nm = fmaxf(M, s_m[i]);
      S = S * __expf(M - nm) + s_s[i] * __expf(s_m[i] - nm);
      M = nm;
    }
    const float lse = M + __logf(S);
    s_lse = lse;
    const float l = (label >= 0 && label < vocab) ? lse - __bfloat162float(lr[label]) : 0.f;
    loss_rows[row] = l;
    if (loss_sum && l != 0.f) atomicAdd(loss_sum, l * scale);
  }
  __syncthreads();
  const float lse = s_lse;
  const bool valid = label >= 0 && label < vocab;
  uint4* ov = reinterpret_cast<uint4*>(lr);
  auto grad8 = [&](int64_t cc, uint4 v) {
    float f[8];
    unpack8(v, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p = valid ? __expf(f[j] - lse) : 0.f;
      if (cc * 8 + j == label) p -= 1.f;
      f[j] = p * scale;
    }
    ov[cc] = pack8(f);
  };
  int64_t c2 = threadIdx.x;
  for (; c2 + 3 * THREADS < nvec; c2 += 4 * THREADS) {
    uint4 u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = ov[c2 + k * THREADS];
#pragma unroll
    for (int k = 0; k < 4; ++k) grad8(c2 + k * THREADS, u[k]);
  }
  for (; c2 < nvec; c2 += THREADS) grad8(c2, ov[c2]);
}

// One HBM read per logit: the row (vocab*2 bytes <= 110 KB) is pulled into
// shared memory by bulk async copies, the (max, sum-exp) reduction and the
// gradient pass both read it from there; two rows (CTAs) per SM in flight.
__global__ void __launch_bounds__(512)
    xent_smem_kernel(__nv_bfloat16* __restrict__ logits, const int64_t* __restrict__ labels,
                     float* __restrict__ loss_rows, float* __restrict__ loss_sum, int64_t vocab,
                     float scale, const float* __restrict__ scale_dev) {
  if (scale_dev != nullptr) scale *= scale_dev[0];   // dynamic loss scale (device)
  constexpr int T = 512;
  extern __shared__ __align__(128) uint8_t xs_raw[];
  __shared__ uint64_t bar;
  __shared__ float s_m[T / 32], s_s[T / 32];
  __shared__ float s_lse;
  const int64_t row = blockIdx.x;
  __nv_bfloat16* lr = logits + row * vocab;
  const uint32_t bytes = static_cast<uint32_t>(vocab * 2);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, bytes);
    constexpr uint32_t CHUNK = 32768;
    for (uint32_t off = 0; off < bytes; off += CHUNK)
      bulk_g2s(xs_raw + off, reinterpret_cast<const uint8_t*>(lr) + off,
               bytes - off < CHUNK ? bytes - off : CHUNK, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  uint4* sv = reinterpret_cast<uint4*>(xs_raw);
  const int nvec = static_cast<int>(vocab >> 3);
  const int64_t label = labels[row];
  const int w = threadIdx.x >> 5;
  // pass 1: row max
  float m = -FLT_MAX;
  for (int c = threadIdx.x; c < nvec; c += T) {
    float f[8];
    unpack8(sv[c], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) m = fmaxf(m, f[j]);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) s_m[w] = m;
  __syncthreads();
  float mx = s_m[0];
#pragma unroll
  for (int i = 1; i < T / 32; ++i) mx = fmaxf(mx, s_m[i]);
  const bool valid = label >= 0 && label < vocab;
  const float lab = valid ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xs_raw)[label]) : 0.f;
  __syncthreads();  // the label logit is read before pass 2 overwrites the row
  // pass 2: e = exp(x - max) once per logit, summed in fp32 and kept (bf16)
  // in place for the gradient pass
  float sum = 0.f;
  for (int c = threadIdx.x; c < nvec; c += T) {
    float f[8];
    unpack8(sv[c], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      f[j] = __expf(f[j] - mx);
      sum += f[j];
    }
    sv[c] = pack8(f);
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) s_s[w] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float Sx = 0.f;
    for (int i = 0; i < T / 32; ++i) Sx += s_s[i];
    s_lse = Sx;
    const float l = valid ? mx + __logf(Sx) - lab : 0.f;
    loss_rows[row] = l;
    if (loss_sum && l != 0.f) atomicAdd(loss_sum, l * scale);
  }
  __syncthreads();
  // pass 3: d logits = (e / sum - onehot) * scale
  const float inv = valid ? scale / s_lse : 0.f;
  uint4* ov = reinterpret_cast<uint4*>(lr);
  for (int c = threadIdx.x; c < nvec; c += T) {
    float f[8];
    unpack8(sv[c], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      f[j] *= inv;
      if (static_cast<int64_t>(c) * 8 + j == label) f[j] -= scale;
    }
    ov[c] = pack8(f);
  }
}

// ---------------------------------------------------------------- bias grad
// Block = 32 column-groups (8 bf16 columns each, one 16-byte load) x 8
// row-lanes; blockIdx.y = row chunk. Fixed-order reductions (deterministic).
// Column sums of dy[rows, cols] (bf16) added into out[cols] (fp32) in one
// launch. CTA (column block of 256 = 32 lanes x 8 columns, row part) sums
// its rows with 8 row-lanes x 4 loads in flight into ws[part][cols]; the last
// CTA of a column block to finish (arrival counter) adds the parts in a fixed
// order, so the result does not depend on CTA timing. The counter is reset
// by that CTA, so the workspace stays reusable (zero-filled once).
// Dropout mask of 8 consecutive elements starting at flat index e0 (even),
// applied in place to f (the backward of out = x + dropout(y): dy = mask(g)).

// DROP: the input is first passed through the dropout mask of call site
// (seed, salt) and written to gy; the column sums are those of gy (the bias
// gradient of a dropped-out branch). Otherwise gy is unused.
template <bool DROP>
__global__ void __launch_bounds__(256) colsum_kernel(const __nv_bfloat16* __restrict__ dy,
                                                     float* __restrict__ ws,
                                                     unsigned* __restrict__ counters,
                                                     float* __restrict__ out, int64_t rows,
                                                     int64_t cols, int64_t rpp, int parts,
                                                     __nv_bfloat16* __restrict__ gy,
                                                     const uint64_t* __restrict__ seed,
                                                     uint32_t salt, uint32_t thr, float scale) {
  __shared__ float sh[8][256 + 4];
  __shared__ bool is_last;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t cb = static_cast<int64_t>(blockIdx.x) * 256;
  const int64_t c0 = cb + tx * 8;
  const int64_t r0 = blockIdx.y * rpp;
  const int64_t r1 = min(rows, r0 + rpp);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  uint32_t key = 0;
  if constexpr (DROP) key = drop_key(seed, salt);
  if (c0 < cols) {
    int64_t r = r0 + ty;
    for (; r + 24 < r1; r += 32) {
      uint4 u[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) u[k] = *reinterpret_cast<const uint4*>(dy + (r + 8 * k) * cols + c0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float f[8];
        unpack8(u[k], f);
        if constexpr (DROP) {
          drop8(f, key, (r + 8 * k) * cols + c0, thr, scale);
          const uint4 o = pack8(f);
          *reinterpret_cast<uint4*>(gy + (r + 8 * k) * cols + c0) = o;
          unpack8(o, f);   // sum what the GEMMs consume (bf16)
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += f[j];
      }
    }
    for (; r < r1; r += 8) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(dy + r * cols + c0), f);
      if constexpr (DROP) {
        drop8(f, key, r * cols + c0, thr, scale);
        const uint4 o = pack8(f);
        *reinterpret_cast<uint4*>(gy + r * cols + c0) = o;
        unpack8(o, f);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += f[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) sh[ty][tx * 8 + j] = acc[j];
  __syncthreads();
  {
    const int i = threadIdx.x;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][i];
    if (cb + i < cols) ws[static_cast<int64_t>(blockIdx.y) * cols + cb + i] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(&counters[blockIdx.x], 1u) == static_cast<unsigned>(parts - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // fixed-order sum of the parts: thread (tx, ty) takes parts ty, ty+8, ...
  float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < cols) {
    // 4 parts in flight per step (the tail of the last CTA is latency-bound);
    // the grouping is fixed, so the sum order does not depend on timing
    float g4[4][8] = {};
    int p = ty;
    for (; p + 24 < parts; p += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int pp = p + 8 * u;
        const float4* src = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(pp) * cols + c0);
        const float4 a = __ldcg(src), b = __ldcg(src + 1);
        g4[u][0] += a.x; g4[u][1] += a.y; g4[u][2] += a.z; g4[u][3] += a.w;
        g4[u][4] += b.x; g4[u][5] += b.y; g4[u][6] += b.z; g4[u][7] += b.w;
      }
    }
    for (; p < parts; p += 8) {
      const int pp = p;
      const float4* src = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(pp) * cols + c0);
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
    const int i = threadIdx.x;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][i];
    if (cb + i < cols) out[cb + i] += t;
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0u;
}

// ------------------------------------------------------------ dropout / add
__global__ void set_seed_kernel(uint64_t* dst, uint64_t v) { *dst = v; }

__global__ void fill_f32_kernel(float* __restrict__ x, float v, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// in place, flat element index e (n even; 8 per thread)
__global__ void dropout_dev_kernel(__nv_bfloat16* __restrict__ x, int64_t n,
                                   const uint64_t* __restrict__ seed, uint32_t salt, uint32_t thr,
                                   float scale) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i >= n) return;
  const uint32_t key = drop_key(seed, salt);
  if (i + 8 <= n) {
    uint4* v = reinterpret_cast<uint4*>(x + i);
    float f[8];
    unpack8(*v, f);
    drop8(f, key, i, thr, scale);
    *v = pack8(f);
  } else {
    for (int64_t k = i; k < n; ++k) {
      const uint32_t kk = drop_keep2(key, static_cast<uint64_t>(k >> 1), thr);
      const float f = __bfloat162float(x[k]);
      x[k] = __float2bfloat16((kk >> (k & 1)) & 1u ? f * scale : 0.f);
    }
  }
}
__global__ void dropout_kernel(__nv_bfloat16* __restrict__ x, int64_t n, float p, uint64_t seed,
                               uint64_t offset) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i >= n) return;
  const uint32_t thresh = static_cast<uint32_t>(p * 4294967296.0);
  const float keep = 1.f / (1.f - p);
  if (i + 8 <= n) {
    uint4* v = reinterpret_cast<uint4*>(x + i);
    float f[8];
    unpack8(*v, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = hash_u32(seed, offset + i + j) < thresh ? 0.f : f[j] * keep;
    *v = pack8(f);
  } else {
    for (int64_t k = i; k < n; ++k) {
      const float f = __bfloat162float(x[k]);
      x[k] = __float2bfloat16(hash_u32(seed, offset + k) < thresh ? 0.f : f * keep);
    }
  }
}

__global__ void add_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ b,
                           __nv_bfloat16* __restrict__ y, int64_t n) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i + 8 <= n) {
    float fa[8], fb[8];
    unpack8(*reinterpret_cast<const uint4*>(a + i), fa);
    unpack8(*reinterpret_cast<const uint4*>(b + i), fb);
#pragma unroll
    for (int j = 0; j < 8; ++j) fa[j] += fb[j];
    *reinterpret_cast<uint4*>(y + i) = pack8(fa);
  } else {
    for (int64_t k = i; k < n; ++k)
      y[k] = __float2bfloat16(__bfloat162float(a[k]) + __bfloat162float(b[k]));
  }
}

__global__ void mul_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ b,
                           __nv_bfloat16* __restrict__ y, int64_t n) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i + 8 <= n) {
    float fa[8], fb[8];
    unpack8(*reinterpret_cast<const uint4*>(a + i), fa);
    unpack8(*reinterpret_cast<const uint4*>(b + i), fb);
#pragma unroll
    for (int j = 0; j < 8; ++j) fa[j] *= fb[j];
    *reinterpret_cast<uint4*>(y + i) = pack8(fa);
  } else {
    for (int64_t k = i; k < n; ++k)
      y[k] = __float2bfloat16(__bfloat162float(a[k]) * __bfloat162float(b[k]));
  }
}

// ---------------------------------------------------------- grad norm / Adam
__global__ void norm_kernel(const float* __restrict__ g, int64_t n, float* __restrict__ out) {
  float ss = 0.f, bad = 0.f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 4;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n;
       i += stride) {
    if (i + 4 <= n) {
      const float4 v = *reinterpret_cast<const float4*>(g + i);
      const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (isfinite(a[j])) ss += a[j] * a[j];
        else bad += 1.f;
      }
    } else {
      for (int64_t k = i; k < n; ++k) {
        if (isfinite(g[k])) ss += g[k] * g[k];
        else bad += 1.f;
      }
    }
  }
  ss = warp_sum(ss);
  bad = warp_sum(bad);
  __shared__ float sh[2][32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[0][w] = ss;
    sh[1][w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f, b = 0.f;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
      a += sh[0][i];
      b += sh[1][i];
    }
    atomicAdd(out, a);
    if (b > 0.f) atomicAdd(out + 1, b);
  }
}

// Fused AdamW (K10). U float4 chunks of every state array per thread
// (block-strided, so every warp access stays coalesced); all loads are issued
// before any math so each thread keeps 4*U 16-byte loads in flight — the
// kernel streams 9 arrays at once and needs that much memory-level
// parallelism (U=1: 1.7 TB/s, U=4: 3.7 TB/s, U=8: 4.3 TB/s on B200 at 355M
// params). ~34 B/param of HBM traffic: read master/grad/m/v, write
// master/m/v/grad (zeroed) + the bf16 weight; streaming cache hints keep the
// single-use state out of L2.
template <int U>
__global__ void __launch_bounds__(256) adam_kernel_u(
    float* __restrict__ master, __nv_bfloat16* __restrict__ w, float* __restrict__ grad,
    float* __restrict__ m, float* __restrict__ v, int64_t n, const float* __restrict__ flags,
    float lr, float b1, float b2, float eps, float wd, float inv_scale, float max_norm, float bc1,
    float bc2, const float* __restrict__ ss) {
  const bool skip = flags[1] != 0.f;
  if (ss != nullptr) {
    // device scaler state [loss scale, applied steps, good steps, scale used]:
    // the unscale factor and the bias corrections of the (steps+1)-th
    // APPLIED step (a skipped step does not advance Adam's clock)
    inv_scale = 1.f / ss[0];
    const float t = ss[1] + 1.f;
    bc1 = 1.f - powf(b1, t);
    bc2 = 1.f - powf(b2, t);
  }
  float coef = inv_scale;
  if (max_norm > 0.f) {
    const float norm = sqrtf(flags[0]) * inv_scale;
    if (norm > max_norm) coef *= max_norm / (norm + 1e-6f);
  }
  const float ib1 = 1.f / bc1, ib2 = 1.f / bc2;
  const int64_t n4 = n >> 2;
  float4* G = reinterpret_cast<float4*>(grad);
  float4* Pm = reinterpret_cast<float4*>(master);
  float4* Mm = reinterpret_cast<float4*>(m);
  float4* Vm = reinterpret_cast<float4*>(v);
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; base < n4;
       base += static_cast<int64_t>(gridDim.x) * blockDim.x * U) {
    float4 g[U], p[U], mm[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + static_cast<int64_t>(u) * blockDim.x;
      if (i < n4) {
        g[u] = __ldcs(G + i);
        if (!skip) {
          p[u] = __ldcs(Pm + i);
          mm[u] = __ldcs(Mm + i);
          vv[u] = __ldcs(Vm + i);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + static_cast<int64_t>(u) * blockDim.x;
      if (i >= n4) continue;
      __stcs(G + i, z);
      if (skip) continue;
      float gs[4] = {g[u].x * coef, g[u].y * coef, g[u].z * coef, g[u].w * coef};
      float ps[4] = {p[u].x, p[u].y, p[u].z, p[u].w};
      float ms[4] = {mm[u].x, mm[u].y, mm[u].z, mm[u].w};
      float vs[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ms[j] = b1 * ms[j] + (1.f - b1) * gs[j];
        vs[j] = b2 * vs[j] + (1.f - b2) * gs[j] * gs[j];
        ps[j] -= lr * ((ms[j] * ib1) / (sqrtf(vs[j] * ib2) + eps) + wd * ps[j]);
      }
      __stcs(Pm + i, make_float4(ps[0], ps[1], ps[2], ps[3]));
      __stcs(Mm + i, make_float4(ms[0], ms[1], ms[2], ms[3]));
      __stcs(Vm + i, make_float4(vs[0], vs[1], vs[2], vs[3]));
      __nv_bfloat162 lo = __floats2bfloat162_rn(ps[0], ps[1]);
      __nv_bfloat162 hi = __floats2bfloat162_rn(ps[2], ps[3]);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      __stcs(reinterpret_cast<uint2*>(w) + i, pk);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t k = n4 * 4 + threadIdx.x;
    const float gk = grad[k] * coef;
    grad[k] = 0.f;
    if (!skip) {
      const float mk = b1 * m[k] + (1.f - b1) * gk;
      const float vk = b2 * v[k] + (1.f - b2) * gk * gk;
      m[k] = mk;
      v[k] = vk;
      const float nw = master[k] - lr * ((mk * ib1) / (sqrtf(vk * ib2) + eps) + wd * master[k]);
      master[k] = nw;
      w[k] = __float2bfloat16(nw);
    }
  }
}

__global__ void cast_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __float2bfloat16(x[i]);
}

// fp32 <-> bf16 gradient buckets of the DP exchange, 8 elements per thread
// (16-byte bf16 vectors, two float4) with a scalar tail.
__global__ void pack_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                 int64_t n) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i + 8 <= n) {
    const float4 a = reinterpret_cast<const float4*>(x + i)[0];
    const float4 b = reinterpret_cast<const float4*>(x + i)[1];
    const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    *reinterpret_cast<uint4*>(y + i) = pack8(f);
  } else {
    for (int64_t k = i; k < n; ++k) y[k] = __float2bfloat16(x[k]);
  }
}
__global__ void unpack_bf16_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ y,
                                   int64_t n) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i + 8 <= n) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(x + i), f);
    reinterpret_cast<float4*>(y + i)[0] = make_float4(f[0], f[1], f[2], f[3]);
    reinterpret_cast<float4*>(y + i)[1] = make_float4(f[4], f[5], f[6], f[7]);
  } else {
    for (int64_t k = i; k < n; ++k) y[k] = __bfloat162float(x[k]);
  }
}

inline unsigned blocks_for(int64_t n, int per_block) {
  return static_cast<unsigned>((n + per_block - 1) / per_block);
}

}  // namespace
}  // namespace vp

using namespace vp;
#define ST reinterpret_cast<cudaStream_t>(stream)
#define BF(p) reinterpret_cast<__nv_bfloat16*>(p)
#define CBF(p) reinterpret_cast<const __nv_bfloat16*>(p)

extern "C" int vp_embed_fwd(const int64_t* ids, const void* wte, const void* wpe, void* x,
                            int64_t batch, int64_t seq, int64_t hidden, void* stream) {
  if (batch <= 0 || seq <= 0 || hidden <= 0 || (hidden % 8)) return VP_ERR_ARGS;
  const int64_t tokens = batch * seq;
  embed_fwd_kernel<<<blocks_for(tokens, 8), 256, 0, ST>>>(ids, CBF(wte), CBF(wpe), BF(x), tokens,
                                                         seq, hidden);
  return launch_status();
}

extern "C" int vp_embed_bwd(const int64_t* ids, const void* dx, float* dwte, float* dwpe,
                            int64_t batch, int64_t seq, int64_t hidden, void* stream) {
  if (batch <= 0 || seq <= 0 || hidden <= 0 || (hidden % 8)) return VP_ERR_ARGS;
  const int64_t tokens = batch * seq;
  embed_bwd_tok_kernel<<<blocks_for(tokens, 8), 256, 0, ST>>>(ids, CBF(dx), dwte, tokens, hidden);
  if (dwpe)
    embed_bwd_pos_kernel<<<blocks_for(seq * hidden, 256), 256, 0, ST>>>(CBF(dx), dwpe, batch, seq,
                                                                       hidden);
  return launch_status();
}

extern "C" int vp_embed_typed_fwd(const int64_t* ids, const int64_t* types, const void* wte,
                                  const void* wpe, const void* tte, void* x, int64_t batch,
                                  int64_t seq, int64_t hidden, void* stream) {
  if (batch <= 0 || seq <= 0 || hidden <= 0 || (hidden % 8)) return VP_ERR_ARGS;
  const int64_t tokens = batch * seq;
  embed_typed_fwd_kernel<<<blocks_for(tokens, 8), 256, 0, ST>>>(ids, types, CBF(wte), CBF(wpe),
                                                               CBF(tte), BF(x), tokens, seq, hidden);
  return launch_status();
}

extern "C" int vp_embed_typed_bwd(const int64_t* ids, const int64_t* types, const void* dx,
                                  float* dwte, float* dwpe, float* dtte, int64_t batch,
                                  int64_t seq, int64_t hidden, void* stream) {
  if (batch <= 0 || seq <= 0 || hidden <= 0 || (hidden % 8)) return VP_ERR_ARGS;
  const int64_t tokens = batch * seq;
  embed_bwd_tok_kernel<<<blocks_for(tokens, 8), 256, 0, ST>>>(ids, CBF(dx), dwte, tokens, hidden);
  embed_bwd_tok_kernel<<<blocks_for(tokens, 8), 256, 0, ST>>>(types, CBF(dx), dtte, tokens, hidden);
  embed_bwd_pos_kernel<<<blocks_for(seq * hidden, 256), 256, 0, ST>>>(CBF(dx), dwpe, batch, seq,
                                                                     hidden);
  return launch_status();
}

extern "C" int vp_gelu_bwd(const void* dy, const void* pre, void* dx, int64_t n, void* stream) {
  if (n <= 0) return VP_ERR_ARGS;
  gelu_bwd_kernel<<<blocks_for(n, 256 * 8), 256, 0, ST>>>(CBF(dy), CBF(pre), BF(dx), n);
  return launch_status();
}

static int xent_entry(void* logits, const int64_t* labels, float* loss_rows, float* loss_sum,
                      int64_t rows, int64_t vocab, float scale, const float* scale_dev,
                      void* stream) {
  if (rows <= 0 || vocab <= 0 || (vocab % 8)) return VP_ERR_ARGS;
  const size_t smem = static_cast<size_t>(vocab) * 2;
  if (smem <= 110 * 1024 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 && !getenv("VP_XENT_2PASS")) {
    if (cudaError_t e = vp::smem_optin(xent_smem_kernel, 110 * 1024); e != cudaSuccess) return e;
    xent_smem_kernel<<<static_cast<unsigned>(rows), 512, smem, ST>>>(BF(logits), labels,
                                                                    loss_rows, loss_sum, vocab,
                                                                    scale, scale_dev);
  } else {
    xent_kernel<512><<<static_cast<unsigned>(rows), 512, 0, ST>>>(BF(logits), labels, loss_rows,
                                                                  loss_sum, vocab, scale, scale_dev);
  }
  return launch_status();
}

extern "C" int vp_xent_fwd_bwd(void* logits, const int64_t* labels, float* loss_rows,
                               float* loss_sum, int64_t rows, int64_t vocab, float scale,
                               void* stream) {
  return xent_entry(logits, labels, loss_rows, loss_sum, rows, vocab, scale, nullptr, stream);
}

extern "C" int vp_xent_fwd_bwd_dev(void* logits, const int64_t* labels, float* loss_rows,
                                   float* loss_sum, int64_t rows, int64_t vocab, float scale,
                                   const float* scale_dev, void* stream) {
  return xent_entry(logits, labels, loss_rows, loss_sum, rows, vocab, scale, scale_dev, stream);
}

// workspace: vp_bias_grad_ws_elems(cols) floats, zero-filled before first use
// (the arrival counters are left at zero by each call).
// Layout: arrival counters first at a FIXED offset (one per 256-column block,
// up to kColsumCounters), partials after them. A workspace sized for C columns
// is then reusable for any cols <= C: a narrower call's partials never land on
// a wider call's counters (with counters after the partials they did).
static constexpr int64_t kColsumMaxParts = 128;
static constexpr int64_t kColsumCounters = 4096;
extern "C" int64_t vp_bias_grad_ws_elems(int64_t cols) {
  return kColsumCounters + kColsumMaxParts * cols;
}

extern "C" int vp_bias_grad(const void* dy, float* dbias, int64_t rows, int64_t cols,
                            float* workspace, void* stream) {
  if (rows <= 0 || cols <= 0 || !workspace) return VP_ERR_ARGS;
  if (cols % 8) return VP_ERR_UNSUPPORTED;
  const int64_t col_blocks = (cols + 255) / 256;
  if (col_blocks > kColsumCounters) return VP_ERR_UNSUPPORTED;
  // ~4 CTAs per SM, >= 32 rows per part, <= kColsumMaxParts parts
  int64_t parts = (4 * static_cast<int64_t>(device_sms()) + col_blocks - 1) / col_blocks;
  parts = std::min<int64_t>(parts, std::max<int64_t>(1, rows / 32));
  parts = std::max<int64_t>(1, std::min<int64_t>(parts, kColsumMaxParts));
  const int64_t rpp = (rows + parts - 1) / parts;
  parts = (rows + rpp - 1) / rpp;
  unsigned* counters = reinterpret_cast<unsigned*>(workspace);
  dim3 grid(static_cast<unsigned>(col_blocks), static_cast<unsigned>(parts));
  colsum_kernel<false><<<grid, 256, 0, ST>>>(CBF(dy), workspace + kColsumCounters, counters,
                                             dbias, rows, cols, rpp, static_cast<int>(parts),
                                             nullptr, nullptr, 0, 0, 0.f);
  return launch_status();
}

extern "C" int vp_fill_f32(float* x, float value, int64_t n, void* stream) {
  if (!x || n < 0) return VP_ERR_ARGS;
  if (n == 0) return VP_OK;
  fill_f32_kernel<<<blocks_for(n, 256), 256, 0, ST>>>(x, value, n);
  return launch_status();
}

extern "C" int vp_set_seed(uint64_t* dst, uint64_t value, void* stream) {
  if (!dst) return VP_ERR_ARGS;
  set_seed_kernel<<<1, 1, 0, ST>>>(dst, value);
  return launch_status();
}

extern "C" int vp_dropout_dev(void* x, int64_t n, float p, const uint64_t* seed, uint32_t salt,
                              void* stream) {
  if (n <= 0 || p < 0.f || p >= 1.f || !seed || (n & 1)) return VP_ERR_ARGS;
  if (p == 0.f) return VP_OK;
  const uint32_t thr = drop_threshold(p);
  dropout_dev_kernel<<<blocks_for(n, 256 * 8), 256, 0, ST>>>(BF(x), n, seed, salt, thr,
                                                             drop_scale(thr));
  return launch_status();
}

extern "C" int vp_dropout_bwd(const void* g, void* gy, int64_t rows, int64_t cols, float p,
                              const uint64_t* seed, uint32_t salt, float* dbias, float* workspace,
                              void* stream) {
  if (rows <= 0 || cols <= 0 || !seed || !workspace || p <= 0.f || p >= 1.f) return VP_ERR_ARGS;
  if (cols % 8) return VP_ERR_UNSUPPORTED;
  const int64_t col_blocks = (cols + 255) / 256;
  if (col_blocks > kColsumCounters) return VP_ERR_UNSUPPORTED;
  int64_t parts = (4 * static_cast<int64_t>(device_sms()) + col_blocks - 1) / col_blocks;
  parts = std::min<int64_t>(parts, std::max<int64_t>(1, rows / 32));
  parts = std::max<int64_t>(1, std::min<int64_t>(parts, kColsumMaxParts));
  const int64_t rpp = (rows + parts - 1) / parts;
  parts = (rows + rpp - 1) / rpp;
  unsigned* counters = reinterpret_cast<unsigned*>(workspace);
  const uint32_t thr = drop_threshold(p);
  dim3 grid(static_cast<unsigned>(col_blocks), static_cast<unsigned>(parts));
  // without dbias the column sums land in a workspace scratch row (unused)
  float* out = dbias;
  if (!out) return VP_ERR_ARGS;
  colsum_kernel<true><<<grid, 256, 0, ST>>>(CBF(g), workspace + kColsumCounters, counters, out,
                                            rows, cols, rpp, static_cast<int>(parts), BF(gy),
                                            seed, salt, thr, drop_scale(thr));
  return launch_status();
}

extern "C" int vp_dropout(void* x, int64_t n, float p, uint64_t seed, uint64_t offset,
                          void* stream) {
  if (n <= 0 || p < 0.f || p >= 1.f) return VP_ERR_ARGS;
  if (p == 0.f) return VP_OK;
  dropout_kernel<<<blocks_for(n, 256 * 8), 256, 0, ST>>>(BF(x), n, p, seed, offset);
  return launch_status();
}

extern "C" int vp_add(const void* a, const void* b, void* y, int64_t n, void* stream) {
  if (n <= 0) return VP_ERR_ARGS;
  add_kernel<<<blocks_for(n, 256 * 8), 256, 0, ST>>>(CBF(a), CBF(b), BF(y), n);
  return launch_status();
}

extern "C" int vp_mul(const void* a, const void* b, void* y, int64_t n, void* stream) {
  if (n <= 0) return VP_ERR_ARGS;
  mul_kernel<<<blocks_for(n, 256 * 8), 256, 0, ST>>>(CBF(a), CBF(b), BF(y), n);
  return launch_status();
}

extern "C" int vp_grad_norm_sq(const float* g, int64_t n, float* out, void* stream) {
  if (n <= 0) return VP_OK;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(1184, (n + 1023) / 1024));
  norm_kernel<<<blocks, 256, 0, ST>>>(g, n, out);
  return launch_status();
}

extern "C" int vp_adam_step(float* master, void* weight_bf16, float* grad, float* exp_avg,
                            float* exp_avg_sq, int64_t n, const float* flags, float lr,
                            float beta1, float beta2, float eps, float weight_decay,
                            float inv_loss_scale, float max_grad_norm, float bias_c1,
                            float bias_c2, void* stream) {
  if (n <= 0) return VP_OK;
  // 16-byte alignment of every state array is required for the float4 path
  if ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(grad) |
       reinterpret_cast<uintptr_t>(exp_avg) | reinterpret_cast<uintptr_t>(exp_avg_sq)) & 15 ||
      reinterpret_cast<uintptr_t>(weight_bf16) & 7)
    return VP_ERR_UNSUPPORTED;
  constexpr int U = 8;
  const int64_t want = (n / 4 + 256 * U - 1) / (256 * U);
  const unsigned grid = static_cast<unsigned>(
      std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(device_sms()) * 8, want)));
  adam_kernel_u<U><<<grid, 256, 0, ST>>>(master, BF(weight_bf16), grad, exp_avg, exp_avg_sq, n,
                                         flags, lr, beta1, beta2, eps, weight_decay,
                                         inv_loss_scale, max_grad_norm, bias_c1, bias_c2,
                                         nullptr);
  return launch_status();
}

extern "C" int vp_adam_step_dev(float* master, void* weight_bf16, float* grad, float* exp_avg,
                                float* exp_avg_sq, int64_t n, const float* flags, float lr,
                                float beta1, float beta2, float eps, float weight_decay,
                                float max_grad_norm, const float* scaler, void* stream) {
  if (n <= 0) return VP_OK;
  if (!scaler || !flags) return VP_ERR_ARGS;
  if ((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(grad) |
       reinterpret_cast<uintptr_t>(exp_avg) | reinterpret_cast<uintptr_t>(exp_avg_sq)) & 15 ||
      reinterpret_cast<uintptr_t>(weight_bf16) & 7)
    return VP_ERR_UNSUPPORTED;
  constexpr int U = 8;
  const int64_t want = (n / 4 + 256 * U - 1) / (256 * U);
  const unsigned grid = static_cast<unsigned>(
      std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(device_sms()) * 8, want)));
  adam_kernel_u<U><<<grid, 256, 0, ST>>>(master, BF(weight_bf16), grad, exp_avg, exp_avg_sq, n,
                                         flags, lr, beta1, beta2, eps, weight_decay, 1.f,
                                         max_grad_norm, 1.f, 1.f, scaler);
  return launch_status();
}

namespace vp {
namespace {
// One thread: the dynamic loss scaler after the step (apex/Megatron
// schedule): overflow (flags[1] != 0) -> scale *= backoff (>= min_scale),
// good = 0, Adam's applied-step count unchanged (the update was skipped);
// otherwise steps += 1, good += 1 and after `window` good steps scale *=
// growth. ss[3] keeps the scale this step used (for unscaling its loss).
__global__ void loss_scaler_kernel(float* ss, const float* flags, float growth, float backoff,
                                   float window, float min_scale, float max_scale) {
  ss[3] = ss[0];
  if (flags[1] != 0.f) {
    ss[0] = fmaxf(ss[0] * backoff, min_scale);
    ss[2] = 0.f;
  } else {
    ss[1] += 1.f;
    ss[2] += 1.f;
    if (ss[2] >= window) {
      ss[0] = fminf(ss[0] * growth, max_scale);
      ss[2] = 0.f;
    }
  }
}
}  // namespace
}  // namespace vp

extern "C" int vp_loss_scaler_update(float* scaler, const float* flags, float growth,
                                     float backoff, int64_t window, float min_scale,
                                     float max_scale, void* stream) {
  if (!scaler || !flags || window <= 0 || growth < 1.f || backoff <= 0.f || backoff > 1.f)
    return VP_ERR_ARGS;
  loss_scaler_kernel<<<1, 1, 0, ST>>>(scaler, flags, growth, backoff, static_cast<float>(window),
                                      min_scale, max_scale);
  return launch_status();
}

extern "C" int vp_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream) {
  if (n <= 0) return VP_OK;
  cast_kernel<<<blocks_for(n, 256), 256, 0, ST>>>(x, BF(y), n);
  return launch_status();
}

extern "C" int vp_grad_pack_bf16(const float* x, void* y, int64_t n, void* stream) {
  if (n <= 0) return VP_OK;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 15))
    return VP_ERR_UNSUPPORTED;
  pack_bf16_kernel<<<blocks_for(n, 256 * 8), 256, 0, ST>>>(x, BF(y), n);
  return launch_status();
}

extern "C" int vp_grad_unpack_bf16(const void* x, float* y, int64_t n, void* stream) {
  if (n <= 0) return VP_OK;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 15))
    return VP_ERR_UNSUPPORTED;
  unpack_bf16_kernel<<<blocks_for(n, 256 * 8), 256, 0, ST>>>(CBF(x), y, n);
  return launch_status();
}
