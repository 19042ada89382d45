#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "vpipe.h"

namespace vp {

// Opt kernel `fn` into `bytes` of dynamic shared memory, once per (kernel,
// device, size) — keyed by the function pointer (a `static bool` inside a
// generic launch lambda would be shared by every kernel of the same
// signature) and by the current device (the attribute is per-device state).
inline cudaError_t smem_optin(const void* fn, int bytes) {
  struct Key { const void* fn; int dev; int bytes; };
  static std::mutex mu;
  static Key done[1024];
  static int nd = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < nd; ++i)
    if (done[i].fn == fn && done[i].dev == dev && done[i].bytes >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && nd < 1024) done[nd++] = Key{fn, dev, bytes};
  return e;
}
template <typename F>
inline cudaError_t smem_optin(F* fn, int bytes) {
  return smem_optin(reinterpret_cast<const void*>(fn), bytes);
}

// SM count of the current device (cached per device; B200: 148).
inline int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// 8 x bf16 <-> 8 x float through one 16-byte vector.
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// Counter-based hash (Philox-style mixing, 2 rounds of 64-bit multiply-xor)
// keyed by (seed, offset + element index): regenerating it in recompute
// gives the identical dropout mask.
__device__ __forceinline__ uint32_t hash_u32(uint64_t seed, uint64_t idx) {
  uint64_t x = seed ^ (idx * 0x9E3779B97F4A7C15ull);
  x ^= x >> 33;
  x *= 0xFF51AFD7ED558CCDull;
  x ^= x >> 33;
  x *= 0xC4CEB9FE1A85EC53ull;
  x ^= x >> 33;
  return static_cast<uint32_t>(x);
}

// ---------------------------------------------------------------- dropout
// K7 dropout mask, regenerated bit-for-bit by recompute and by the backward.
// The 64-bit seed of the current (step, micro-batch) is READ FROM DEVICE
// MEMORY (written by vp_set_seed before each task), so captured CUDA graphs
// replay with fresh masks; the per-call-site salt (layer, site) is static.
// Element e of a call site's tensor: bits = fmix32(key ^ lo(e/2)*A ^ hi(e/2)*B),
// its 16-bit half (low for even e, high for odd e) u; kept iff u >= thr,
// thr = round(p * 65536); kept values are scaled by 65536 / (65536 - thr).
// oracle/gpt2_fp32.py restates this function for the parity tests.
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}
__device__ __forceinline__ uint32_t drop_key(const uint64_t* seed, uint32_t salt) {
  const uint64_t s = *seed;
  return fmix32(static_cast<uint32_t>(s) ^ fmix32(static_cast<uint32_t>(s >> 32) ^ fmix32(salt)));
}
__device__ __forceinline__ uint32_t drop_bits(uint32_t key, uint64_t pair) {
  return fmix32(key ^ (static_cast<uint32_t>(pair) * 0x9E3779B1u) ^
                (static_cast<uint32_t>(pair >> 32) * 0x85EBCA77u));
}
// keep flags of elements 2*pair (bit 0) and 2*pair + 1 (bit 1)
__device__ __forceinline__ uint32_t drop_keep2(uint32_t key, uint64_t pair, uint32_t thr) {
  const uint32_t b = drop_bits(key, pair);
  return ((b & 0xFFFFu) >= thr ? 1u : 0u) | ((b >> 16) >= thr ? 2u : 0u);
}
// Elements e0 .. e0+7 (e0 even) of a call site's tensor through its mask:
// kept values scaled by 1/(1-p), dropped ones 0.
__device__ __forceinline__ void drop8(float (&f)[8], uint32_t key, int64_t e0, uint32_t thr,
                                      float scale) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t k = drop_keep2(key, static_cast<uint64_t>(e0 >> 1) + q, thr);
    f[2 * q] = (k & 1u) ? f[2 * q] * scale : 0.f;
    f[2 * q + 1] = (k & 2u) ? f[2 * q + 1] * scale : 0.f;
  }
}
inline uint32_t drop_threshold(float p) {
  const double t = static_cast<double>(p) * 65536.0 + 0.5;
  return t >= 65535.0 ? 65535u : static_cast<uint32_t>(t);
}
inline float drop_scale(uint32_t thr) { return 65536.f / static_cast<float>(65536u - thr); }

// Transpose of the 32x32 bit matrix whose row r is lane r's word: on
// return lane c holds column c (bit r = row r's bit c). Butterfly: at
// distance j lanes l, l^j swap the off-diagonal j x j bit blocks.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, uint32_t lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const uint32_t m = masks[s];
    const uint32_t o = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? (((o >> j) & m) | (x & ~m)) : ((x & m) | ((o & m) << j));
  }
  return x;
}

// Attention-probability dropout of one call site (seed == nullptr: none).
// Keep-bit masks (optional, S % 32 == 0), drawn ONCE per (layer, micro-
// batch) by vp_attention_dropout_mask — off the softmax critical path — in
// the two layouts the kernels' thread mappings read coalesced:
//   mask_q: word [((b*H + h)*(S/32) + key/32)*S + q], bit key % 32
//           (threads own query rows: forward, dQ kernel);
//   mask_k: word [((b*H + h)*(S/32) + q/32)*S + key], bit q % 32
//           (threads own key rows: the fused backward, the dK/dV kernel).
// Without them the kernels hash every element (common.cuh drop_bits).
struct AttnDrop {
  const uint64_t* seed;
  uint32_t salt;
  uint32_t thr;
  float scale;
  const uint32_t* mask_q;
  const uint32_t* mask_k;
};
inline AttnDrop make_attn_drop(float p, const uint64_t* seed, uint32_t salt,
                               const uint32_t* mask_q = nullptr,
                               const uint32_t* mask_k = nullptr) {
  if (p <= 0.f || !seed) return AttnDrop{nullptr, 0, 0, 1.f, nullptr, nullptr};
  const uint32_t thr = drop_threshold(p);
  return AttnDrop{seed, salt, thr, drop_scale(thr), mask_q, mask_k};
}

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? VP_OK : static_cast<int>(e);
}

}  // namespace vp
