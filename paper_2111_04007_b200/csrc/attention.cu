// Attention entry points (K2/K3 of DESIGN.md). The kernels live in
// attention_tc.cu (tcgen05 forward, deterministic two-kernel backward) and
// attention_bwd.cu (fused one-pass backward, head_dim 64 and 96); this file holds
// the C ABI and the delta pre-pass of the deterministic backward.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"

namespace vp {

int attention_fwd_tc(const void* qkv, void* o, float* lse, int64_t B, int64_t S, int64_t H,
                     int64_t D, int causal, float p, const uint64_t* seed, uint32_t salt,
                     const uint32_t* mask_q, cudaStream_t st);
int attention_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* delta,
                     void* dqkv, int64_t B, int64_t S, int64_t H, int64_t D, int causal,
                     float p, const uint64_t* seed, uint32_t salt, const uint32_t* mask_q,
                     const uint32_t* mask_k, cudaStream_t st);
int64_t attention_bwd_fused_ws(int64_t B, int64_t S, int64_t H, int64_t D);
bool attention_bwd_fused_ok(int64_t D);
int attention_bwd_fused(const void* qkv, const void* o, const void* dout, const float* lse,
                        void* dqkv, float* ws, int64_t B, int64_t S, int64_t H, int64_t D,
                        int causal, float* dbias, const AttnDrop& drop, cudaStream_t st);

namespace {

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

template <int D, bool CAUSAL>
int bwd_t(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
          float* delta, int64_t B, int64_t S, int64_t H, float p, const uint64_t* seed,
          uint32_t salt, const uint32_t* mask_q, const uint32_t* mask_k, cudaStream_t st) {
  const int64_t tokens = B * S;
  constexpr int RPW = 32 / (D / 8);
  const int64_t warps = (tokens * H + RPW - 1) / RPW;
  attn_delta_kernel<D><<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(o), reinterpret_cast<const __nv_bfloat16*>(dout),
      delta, tokens, static_cast<int>(S), static_cast<int>(H));
  return attention_bwd_tc(qkv, dout, lse, delta, dqkv, B, S, H, D, CAUSAL, p, seed, salt, mask_q,
                          mask_k, st);
}

}  // namespace

}  // namespace vp

using namespace vp;

extern "C" int vp_attention_fwd(const void* qkv, void* o, float* lse, int64_t batch, int64_t seq,
                                int64_t heads, int64_t head_dim, int causal, void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0) return VP_ERR_ARGS;
  return attention_fwd_tc(qkv, o, lse, batch, seq, heads, head_dim, causal, 0.f, nullptr, 0,
                          nullptr, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int vp_attention_fwd_ex(const void* qkv, void* o, float* lse, int64_t batch,
                                   int64_t seq, int64_t heads, int64_t head_dim, int causal,
                                   float p, const uint64_t* seed, uint32_t salt,
                                   const uint32_t* mask_q, void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || p < 0.f || p >= 1.f) return VP_ERR_ARGS;
  if (p > 0.f && !seed) return VP_ERR_ARGS;
  return attention_fwd_tc(qkv, o, lse, batch, seq, heads, head_dim, causal, p, seed, salt,
                          mask_q, reinterpret_cast<cudaStream_t>(stream));
}

namespace vp {
namespace {
// The keep bits of one attention call site, drawn once (K7 mask function,
// common.cuh) in both layouts (AttnDrop): CTA = (b*H + h, 128 queries), warp
// = 32 query rows, lane = one row. Per 32-key group: 16 pair hashes give the
// row's word (mask_q, coalesced over the warp's rows), a 32x32 bit
// transpose (warp_transpose32) gives 32 keys' words over the warp's rows
// (mask_k, coalesced over keys). Causal: groups above the diagonal skipped.
template <bool CAUSAL>
__global__ void __launch_bounds__(128) attn_mask_kernel(const uint64_t* __restrict__ seed,
                                                        uint32_t salt, uint32_t thr, int S,
                                                        uint32_t* __restrict__ mask_q,
                                                        uint32_t* __restrict__ mask_k) {
  const int bh = blockIdx.y;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qw = blockIdx.x * 4 + static_cast<int>(warp);   // 32-query group
  const int q = qw * 32 + static_cast<int>(lane);
  if (qw * 32 >= S) return;
  const uint32_t key = drop_key(seed, salt);
  const int words = S >> 5;
  const int kw_end = CAUSAL ? qw + 1 : words;
  const uint64_t row = (static_cast<uint64_t>(bh) * S + min(q, S - 1)) * S;
  for (int kw = 0; kw < kw_end; ++kw) {
    uint32_t w = 0;
    const uint64_t p0 = (row + static_cast<uint64_t>(kw) * 32) >> 1;
#pragma unroll
    for (int t = 0; t < 16; ++t) w |= drop_keep2(key, p0 + t, thr) << (2 * t);
    const uint64_t base = (static_cast<uint64_t>(bh) * words + kw) * S;
    if (q < S) mask_q[base + q] = w;
    const uint32_t wt = warp_transpose32(w, lane);        // key kw*32+lane over these rows
    mask_k[(static_cast<uint64_t>(bh) * words + qw) * S + kw * 32 + lane] = wt;
  }
}
}  // namespace
}  // namespace vp

extern "C" int vp_attention_dropout_mask(int64_t batch, int64_t seq, int64_t heads, int causal,
                                         float p, const uint64_t* seed, uint32_t salt,
                                         uint32_t* mask_q, uint32_t* mask_k, void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || (seq % 32) || !seed || !mask_q || !mask_k ||
      p <= 0.f || p >= 1.f)
    return VP_ERR_ARGS;
  dim3 grid(static_cast<unsigned>((seq / 32 + 3) / 4), static_cast<unsigned>(batch * heads));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t thr = drop_threshold(p);
  if (causal)
    attn_mask_kernel<true><<<grid, 128, 0, st>>>(seed, salt, thr, static_cast<int>(seq), mask_q,
                                                 mask_k);
  else
    attn_mask_kernel<false><<<grid, 128, 0, st>>>(seed, salt, thr, static_cast<int>(seq), mask_q,
                                                  mask_k);
  return launch_status();
}

extern "C" int64_t vp_attention_mask_words(int64_t batch, int64_t seq, int64_t heads) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || (seq % 32)) return 0;
  return batch * heads * seq * (seq / 32);
}

namespace {
int attn_bwd_det(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                 float* delta_ws, int64_t batch, int64_t seq, int64_t heads, int64_t head_dim,
                 int causal, float p, const uint64_t* seed, uint32_t salt, const uint32_t* mask_q,
                 const uint32_t* mask_k, cudaStream_t st) {
#define BWD(DD)                                                                              \
  return causal ? bwd_t<DD, true>(qkv, o, dout, lse, dqkv, delta_ws, batch, seq, heads, p, seed, \
                                  salt, mask_q, mask_k, st)                                   \
                : bwd_t<DD, false>(qkv, o, dout, lse, dqkv, delta_ws, batch, seq, heads, p,     \
                                   seed, salt, mask_q, mask_k, st)
  switch (head_dim) {
    case 64: BWD(64);
    case 96: BWD(96);
    case 128: BWD(128);
    default: return VP_ERR_UNSUPPORTED;
  }
#undef BWD
}
}  // namespace

// delta_ws: batch*heads*seq floats.
extern "C" int vp_attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse,
                                void* dqkv, float* delta_ws, int64_t batch, int64_t seq,
                                int64_t heads, int64_t head_dim, int causal, void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || !delta_ws) return VP_ERR_ARGS;
  return attn_bwd_det(qkv, o, dout, lse, dqkv, delta_ws, batch, seq, heads, head_dim, causal, 0.f,
                      nullptr, 0, nullptr, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int64_t vp_attention_bwd_ws_elems(int64_t batch, int64_t seq, int64_t heads,
                                             int64_t head_dim) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || head_dim <= 0) return 0;
  return attention_bwd_fused_ws(batch, seq, heads, head_dim);
}

extern "C" int vp_attention_bwd_fuses_bias(int64_t head_dim, int flags) {
  const bool det = (flags & VP_ATTN_DETERMINISTIC) || getenv("VP_ATTN_DETERMINISTIC");
  return (!det && attention_bwd_fused_ok(head_dim)) ? 1 : 0;
}

extern "C" int vp_attention_bwd_ex(const void* qkv, const void* o, const void* dout,
                                   const float* lse, void* dqkv, float* workspace,
                                   int64_t ws_elems, int64_t batch, int64_t seq, int64_t heads,
                                   int64_t head_dim, int causal, int flags, float p,
                                   const uint64_t* seed, uint32_t salt, const uint32_t* mask_q,
                                   const uint32_t* mask_k, float* dbias, void* stream) {
  if (batch <= 0 || seq <= 0 || heads <= 0 || !workspace) return VP_ERR_ARGS;
  if (p < 0.f || p >= 1.f || (p > 0.f && !seed)) return VP_ERR_ARGS;
  if (ws_elems < attention_bwd_fused_ws(batch, seq, heads, head_dim)) return VP_ERR_ARGS;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return VP_ERR_ARGS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (vp_attention_bwd_fuses_bias(head_dim, flags)) {
    const AttnDrop dr = (seq % 32) ? make_attn_drop(p, seed, salt)
                                   : make_attn_drop(p, seed, salt, mask_q, mask_k);
    if (dr.seed && (seq & 1)) return VP_ERR_UNSUPPORTED;
    return attention_bwd_fused(qkv, o, dout, lse, dqkv, workspace, batch, seq, heads, head_dim,
                               causal, dbias, dr, st);
  }
  if (dbias) return VP_ERR_UNSUPPORTED;  // bias sums are fused only into the one-pass kernel
  return attn_bwd_det(qkv, o, dout, lse, dqkv, workspace, batch, seq, heads, head_dim, causal, p,
                      seed, salt, mask_q, mask_k, st);
}
