"""Torch-facing wrappers of the sm_100a kernels in libvpipe.so.

Thin: each function checks dtypes/contiguity, passes ``data_ptr()`` and the
current CUDA stream to the C-ABI (include/vpipe.h) and raises on a non-zero
status. No fallback path exists: a missing library or a non-CUDA tensor is
an error.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import check, f32, i64, vp

L = _lib.lib
c_int = ctypes.c_int
u64 = ctypes.c_uint64

EPI_STORE, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESID, EPI_DGELU, EPI_ACC_F32, EPI_STORE_F32 = range(7)

_SIGS = {
    "vp_device_sm_count": [ctypes.POINTER(c_int)],
    "vp_gemm_bf16": [c_int, c_int, c_int, vp, i64, vp, i64, vp, i64, vp, vp, i64, i64, i64, i64, vp],
    "vp_layernorm_fwd": [vp, vp, vp, vp, vp, vp, i64, i64, f32, vp],
    "vp_layernorm_bwd": [vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, c_int, vp, vp],
    "vp_attention_fwd": [vp, vp, vp, i64, i64, i64, i64, c_int, vp],
    "vp_attention_bwd": [vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, c_int, vp],
    "vp_embed_fwd": [vp, vp, vp, vp, i64, i64, i64, vp],
    "vp_embed_bwd": [vp, vp, vp, vp, i64, i64, i64, vp],
    "vp_xent_fwd_bwd": [vp, vp, vp, i64, i64, f32, vp],
    "vp_bias_grad": [vp, vp, i64, i64, vp, vp],
    "vp_dropout": [vp, i64, f32, u64, u64, vp],
    "vp_add": [vp, vp, vp, i64, vp],
    "vp_grad_norm_sq": [vp, i64, vp, vp],
    "vp_adam_step": [vp, vp, vp, vp, vp, i64, vp, f32, f32, f32, f32, f32, f32, f32, f32, f32, vp],
    "vp_cast_f32_bf16": [vp, vp, i64, vp],
    "vp_ipc_get_mem_handle": [vp, vp],
    "vp_ipc_open_mem_handle": [vp, ctypes.POINTER(vp)],
    "vp_ipc_close_mem_handle": [vp],
    "vp_ipc_event_create": [ctypes.POINTER(vp), vp],
    "vp_ipc_event_open": [vp, ctypes.POINTER(vp)],
    "vp_event_destroy": [vp],
    "vp_event_record": [vp, vp],
    "vp_stream_wait_event": [vp, vp],
    "vp_event_query": [vp],
    "vp_p2p_put": [vp, vp, i64, vp],
}
for _name, _args in _SIGS.items():
    _fn = getattr(L, _name, None)
    if _fn is not None:
        _fn.argtypes = _args
        _fn.restype = c_int


def _stream(s=None):
    return (s or torch.cuda.current_stream()).cuda_stream


def _p(t):
    return None if t is None else t.data_ptr()


def _need(t, dtype, name):
    if not t.is_cuda:
        raise ValueError(f"{name}: CUDA tensor required (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")


def sm_count() -> int:
    n = c_int(0)
    check(L.vp_device_sm_count(ctypes.byref(n)), "vp_device_sm_count")
    return n.value


def gemm(a, b, out, *, a_kmajor=True, b_kmajor=True, epilogue=EPI_STORE, bias=None, aux=None,
         M=None, N=None, K=None, stream=None):
    """out[M,N] = epi(op(a) @ op(b)^T) where op(a) is [M,K] (a_kmajor: a is
    [M,K], else a is [K,M]) and op(b) is [N,K] (b_kmajor: b is [N,K], else
    [K,N]). All operands bf16 row-major with unit inner stride; out is bf16
    or fp32 (ACC_F32 / STORE_F32)."""
    _need(a, torch.bfloat16, "gemm.a")
    _need(b, torch.bfloat16, "gemm.b")
    if M is None:
        M = a.shape[0] if a_kmajor else a.shape[1]
    if K is None:
        K = a.shape[1] if a_kmajor else a.shape[0]
    if N is None:
        N = b.shape[0] if b_kmajor else b.shape[1]
    for t in (a, b, out) + ((aux,) if aux is not None else ()):
        if t.stride(-1) != 1:
            raise ValueError("gemm: inner stride must be 1")
    check(L.vp_gemm_bf16(int(a_kmajor), int(b_kmajor), epilogue, a.data_ptr(), a.stride(0),
                         b.data_ptr(), b.stride(0), out.data_ptr(), out.stride(0), _p(bias),
                         _p(aux), aux.stride(0) if aux is not None else 0, M, N, K,
                         _stream(stream)), "vp_gemm_bf16")
    return out
