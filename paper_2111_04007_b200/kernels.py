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
u32 = ctypes.c_uint32

(EPI_STORE, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESID, EPI_DGELU, EPI_ACC_F32, EPI_STORE_F32,
 EPI_RESID) = range(8)

_SIGS = {
    "vp_device_sm_count": [ctypes.POINTER(c_int)],
    "vp_gemm_bf16": [c_int, c_int, c_int, vp, i64, vp, i64, vp, i64, vp, vp, i64, i64, i64, i64, vp],
    "vp_gemm_bf16_ex": [c_int, c_int, c_int, vp, i64, vp, i64, vp, i64, vp, vp, i64, i64, i64, i64,
                        c_int, vp],
    "vp_layernorm_fwd": [vp, vp, vp, vp, vp, vp, i64, i64, f32, vp],
    "vp_layernorm_bwd": [vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, c_int, vp, vp],
    "vp_attention_fwd": [vp, vp, vp, i64, i64, i64, i64, c_int, vp],
    "vp_attention_bwd": [vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, c_int, vp],
    "vp_attention_bwd_ex": [vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, c_int, c_int, f32,
                            vp, u32, vp, vp, vp, vp],
    "vp_attention_dropout_mask": [i64, i64, i64, c_int, f32, vp, u32, vp, vp, vp],
    "vp_attention_fwd_ex": [vp, vp, vp, i64, i64, i64, i64, c_int, f32, vp, u32, vp, vp],
    "vp_attention_mask_words": [i64, i64, i64],
    "vp_set_seed": [vp, u64, vp],
    "vp_fill_f32": [vp, f32, i64, vp],
    "vp_xent_fwd_bwd_dev": [vp, vp, vp, vp, i64, i64, f32, vp, vp],
    "vp_adam_step_dev": [vp, vp, vp, vp, vp, i64, vp, f32, f32, f32, f32, f32, f32, vp, vp],
    "vp_loss_scaler_update": [vp, vp, f32, f32, i64, f32, f32, vp],
    "vp_grad_pack_bf16": [vp, vp, i64, vp],
    "vp_grad_unpack_bf16": [vp, vp, i64, vp],
    "vp_dropout_dev": [vp, i64, f32, vp, u32, vp],
    "vp_dropout_bwd": [vp, vp, i64, i64, f32, vp, u32, vp, vp, vp],
    "vp_gemm_bf16_dropout": [c_int, c_int, vp, i64, vp, i64, vp, i64, vp, vp, i64, i64, i64, i64,
                             f32, vp, u32, c_int, vp],
    "vp_attention_bwd_ws_elems": [i64, i64, i64, i64],
    "vp_attention_bwd_fuses_bias": [i64, c_int],
    "vp_layernorm_ws_elems": [i64],
    "vp_gemm_dbias_ws_elems": [i64, i64],
    "vp_gemm_bf16_dbias": [c_int, c_int, c_int, vp, i64, vp, i64, vp, i64, vp, vp, i64, i64, i64,
                           i64, vp, vp, vp],
    "vp_bias_grad_ws_elems": [i64],
    "vp_layernorm_bwd_ex": [vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, c_int, vp, vp],
    "vp_layernorm_bwd_dropout": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, f32, vp, u32, i64, i64,
                                 c_int, vp, vp],
    "vp_embed_fwd": [vp, vp, vp, vp, i64, i64, i64, vp],
    "vp_embed_bwd": [vp, vp, vp, vp, i64, i64, i64, vp],
    "vp_xent_fwd_bwd": [vp, vp, vp, vp, i64, i64, f32, vp],
    "vp_device_alloc": [i64, ctypes.POINTER(vp)],
    "vp_device_free": [vp],
    "vp_bias_grad": [vp, vp, i64, i64, vp, vp],
    "vp_embed_typed_fwd": [vp, vp, vp, vp, vp, vp, i64, i64, i64, vp],
    "vp_embed_typed_bwd": [vp, vp, vp, vp, vp, vp, i64, i64, i64, vp],
    "vp_gelu_bwd": [vp, vp, vp, i64, vp],
    "vp_dropout": [vp, i64, f32, u64, u64, vp],
    "vp_add": [vp, vp, vp, i64, vp],
    "vp_mul": [vp, vp, vp, i64, vp],
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
L.vp_attention_bwd_ws_elems.restype = ctypes.c_int64
L.vp_attention_mask_words.restype = ctypes.c_int64
L.vp_layernorm_ws_elems.restype = ctypes.c_int64
L.vp_gemm_dbias_ws_elems.restype = ctypes.c_int64
L.vp_bias_grad_ws_elems.restype = ctypes.c_int64


# Kernel launches issued through this module (the bench's gpu_launches
# claim); GEMM timing hook (CUDA events on the launching stream) used by
# bench.py to measure the dominant kernel's achieved TFLOP/s.
LAUNCHES = [0]
GEMM_TIMING = {"on": False, "records": []}


def _count(n=1):
    LAUNCHES[0] += n


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


def gemm_dbias_ws_elems(M: int, N: int) -> int:
    return int(L.vp_gemm_dbias_ws_elems(M, N))


def gemm(a, b, out, *, a_kmajor=True, b_kmajor=True, epilogue=EPI_STORE, bias=None, aux=None,
         M=None, N=None, K=None, stream=None, out_ptr=None, ldd=None, direct=False,
         dbias=None, dbias_ws=None):
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
    for t in (a, b) + tuple(x for x in (out, aux) if x is not None):
        if t.stride(-1) != 1:
            raise ValueError("gemm: inner stride must be 1")
    if out is not None:
        out_ptr, ldd = out.data_ptr(), out.stride(0)
    timing = GEMM_TIMING["on"]
    if timing:
        st = stream or torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
    if dbias is not None:
        # bias gradient (column sums of the output) fused into the epilogue
        if dbias_ws is None or dbias_ws.numel() < gemm_dbias_ws_elems(M, N):
            raise ValueError("gemm: dbias needs a workspace of gemm_dbias_ws_elems(M, N)")
        _count(2)
        check(L.vp_gemm_bf16_dbias(int(a_kmajor), int(b_kmajor), epilogue, a.data_ptr(),
                                   a.stride(0), b.data_ptr(), b.stride(0), out_ptr, ldd, _p(bias),
                                   _p(aux), aux.stride(0) if aux is not None else 0, M, N, K,
                                   dbias.data_ptr(), dbias_ws.data_ptr(), _stream(stream)),
              "vp_gemm_bf16_dbias")
    else:
        _count()
        check(L.vp_gemm_bf16_ex(int(a_kmajor), int(b_kmajor), epilogue, a.data_ptr(),
                                a.stride(0), b.data_ptr(), b.stride(0), out_ptr, ldd, _p(bias),
                                _p(aux), aux.stride(0) if aux is not None else 0, M, N, K,
                                1 if direct else 0, _stream(stream)), "vp_gemm_bf16")
    if timing:
        e1.record(st)
        GEMM_TIMING["records"].append((2 * M * N * K, e0, e1,
                                       (M, N, K, a_kmajor, b_kmajor, epilogue)))
    return out


def layernorm_fwd(x, gamma, beta, y, mean, rstd, eps=1e-5, stream=None):
    rows, cols = x.shape
    _count(1)
    check(L.vp_layernorm_fwd(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
                             mean.data_ptr(), rstd.data_ptr(), rows, cols, eps, _stream(stream)),
          "vp_layernorm_fwd")
    return y


def layernorm_ws_elems(cols: int) -> int:
    return int(L.vp_layernorm_ws_elems(cols))


def layernorm_bwd(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, workspace, accumulate=False,
                  stream=None, dsum=None):
    """dx (= or += when ``accumulate``) and dgamma/dbeta += (fp32). ``dsum``
    (optional fp32 [cols]) += the column sum of the finished dx: the bias
    gradient of a residual branch whose output gradient is dx."""
    rows, cols = x.shape
    _count(2 if cols <= 1024 else 3)
    check(L.vp_layernorm_bwd_ex(dy.data_ptr(), x.data_ptr(), gamma.data_ptr(), mean.data_ptr(),
                                rstd.data_ptr(), dx.data_ptr(), dgamma.data_ptr(),
                                dbeta.data_ptr(), _p(dsum), rows, cols, int(accumulate),
                                workspace.data_ptr(), _stream(stream)), "vp_layernorm_bwd")
    return dx


def layernorm_bwd_dropout(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, workspace, dsum, gy, p,
                          seed, salt, accumulate=False, stream=None) -> bool:
    """layernorm_bwd plus the dropped-out residual branch's gradient in the
    same pass: gy = mask(dx) (call site ``salt``, device ``seed``) and dsum
    += its column sums. Returns False (nothing launched) when this row width
    has no fused path — the caller then runs layernorm_bwd + dropout_bwd."""
    rows, cols = x.shape
    rc = L.vp_layernorm_bwd_dropout(dy.data_ptr(), x.data_ptr(), gamma.data_ptr(),
                                    mean.data_ptr(), rstd.data_ptr(), dx.data_ptr(),
                                    dgamma.data_ptr(), dbeta.data_ptr(), dsum.data_ptr(),
                                    gy.data_ptr(), p, seed.data_ptr(), salt & 0xFFFFFFFF, rows,
                                    cols, int(accumulate), workspace.data_ptr(), _stream(stream))
    if rc == _lib.VP_ERR_UNSUPPORTED:
        return False
    check(rc, "vp_layernorm_bwd_dropout")
    _count(2)
    return True


def attention_mask_words(batch, seq, heads) -> int:
    return int(L.vp_attention_mask_words(batch, seq, heads))


def attention_dropout_mask(batch, seq, heads, causal, p, seed, salt, mask_q, mask_k,
                           stream=None):
    """Draw the keep bits of one attention dropout site once, in the forward
    (``mask_q``) and backward (``mask_k``) layouts."""
    _count(1)
    check(L.vp_attention_dropout_mask(batch, seq, heads, int(causal), p, seed.data_ptr(),
                                      salt & 0xFFFFFFFF, mask_q.data_ptr(), mask_k.data_ptr(),
                                      _stream(stream)), "vp_attention_dropout_mask")


def attention_fwd(qkv, out, lse, batch, seq, heads, head_dim, causal=True, stream=None,
                  p=0.0, seed=None, salt=0, mask=None):
    """``p`` > 0: attention-probability dropout keyed by the device seed
    tensor ``seed`` (int64 [1]) and the call site's ``salt``; ``mask``: the
    site's pre-drawn keep bits (``mask_q`` of attention_dropout_mask)."""
    _count(1)
    check(L.vp_attention_fwd_ex(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), batch, seq, heads,
                                head_dim, int(causal), p, _p(seed) if p > 0 else None,
                                salt & 0xFFFFFFFF, _p(mask) if p > 0 else None, _stream(stream)),
          "vp_attention_fwd_ex")
    return out


def attention_bwd_ws_elems(batch, seq, heads, head_dim) -> int:
    return int(L.vp_attention_bwd_ws_elems(batch, seq, heads, head_dim))


def attention_bwd(qkv, out, dout, lse, dqkv, ws, batch, seq, heads, head_dim, causal=True,
                  stream=None, deterministic=False, dbias=None, p=0.0, seed=None, salt=0,
                  mask_q=None, mask_k=None):
    """dqkv = d(qkv). ``ws``: fp32 workspace of attention_bwd_ws_elems()
    elements. head_dim 64 and 96 run the fused one-pass kernel (dQ
    accumulated by TMA reduce-add); ``deterministic`` (or other head dims)
    the two-kernel path. ``dbias`` (fp32 [3*heads*head_dim]) += column sums of dqkv, fused
    on the one-pass path; returns False when the caller must sum itself."""
    need = attention_bwd_ws_elems(batch, seq, heads, head_dim)
    if ws.numel() < need or ws.dtype != torch.float32:
        raise ValueError(f"attention_bwd: workspace needs {need} fp32 elements")
    fused_bias = dbias is not None and bool(
        L.vp_attention_bwd_fuses_bias(head_dim, 1 if deterministic else 0))
    _count(3 + (1 if fused_bias else 0))
    check(L.vp_attention_bwd_ex(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                dqkv.data_ptr(), ws.data_ptr(), ws.numel(), batch, seq, heads,
                                head_dim, int(causal), 1 if deterministic else 0, p,
                                _p(seed) if p > 0 else None, salt & 0xFFFFFFFF,
                                _p(mask_q) if p > 0 else None, _p(mask_k) if p > 0 else None,
                                dbias.data_ptr() if fused_bias else None, _stream(stream)),
          "vp_attention_bwd")
    return fused_bias


def embed_fwd(ids, wte, wpe, x, batch, seq, stream=None):
    _count(1)
    check(L.vp_embed_fwd(ids.data_ptr(), wte.data_ptr(), wpe.data_ptr(), x.data_ptr(), batch, seq,
                         wte.shape[1], _stream(stream)), "vp_embed_fwd")
    return x


def embed_bwd(ids, dx, dwte, dwpe, batch, seq, stream=None):
    _count(1 if dwpe is None else 2)
    check(L.vp_embed_bwd(ids.data_ptr(), dx.data_ptr(), dwte.data_ptr(), _p(dwpe), batch, seq,
                         dx.shape[1], _stream(stream)), "vp_embed_bwd")


def embed_typed_fwd(ids, types, wte, wpe, tte, x, batch, seq, stream=None):
    _count(1)
    check(L.vp_embed_typed_fwd(ids.data_ptr(), types.data_ptr(), wte.data_ptr(), wpe.data_ptr(),
                               tte.data_ptr(), x.data_ptr(), batch, seq, wte.shape[1],
                               _stream(stream)), "vp_embed_typed_fwd")
    return x


def embed_typed_bwd(ids, types, dx, dwte, dwpe, dtte, batch, seq, stream=None):
    _count(3)
    check(L.vp_embed_typed_bwd(ids.data_ptr(), types.data_ptr(), dx.data_ptr(), dwte.data_ptr(),
                               dwpe.data_ptr(), dtte.data_ptr(), batch, seq, dx.shape[1],
                               _stream(stream)), "vp_embed_typed_bwd")


def gelu_bwd(dy, pre, dx, stream=None):
    _count(1)
    check(L.vp_gelu_bwd(dy.data_ptr(), pre.data_ptr(), dx.data_ptr(), dy.numel(), _stream(stream)),
          "vp_gelu_bwd")
    return dx


def xent_fwd_bwd(logits, labels, loss_rows, scale, loss_sum=None, stream=None, scale_dev=None):
    """``scale_dev`` (device fp32, optional): multiply ``scale`` by
    scale_dev[0] in-kernel — the dynamic loss scale."""
    rows, vocab = logits.shape
    _count(1)
    if scale_dev is not None:
        check(L.vp_xent_fwd_bwd_dev(logits.data_ptr(), labels.data_ptr(), loss_rows.data_ptr(),
                                    _p(loss_sum), rows, vocab, scale, scale_dev.data_ptr(),
                                    _stream(stream)), "vp_xent_fwd_bwd_dev")
        return loss_rows
    check(L.vp_xent_fwd_bwd(logits.data_ptr(), labels.data_ptr(), loss_rows.data_ptr(),
                            _p(loss_sum), rows, vocab, scale, _stream(stream)), "vp_xent_fwd_bwd")
    return loss_rows


def bias_grad_ws_elems(cols: int) -> int:
    """fp32 elements of the bias_grad workspace; allocate it zero-filled."""
    return int(L.vp_bias_grad_ws_elems(cols))


def bias_grad(dy, dbias, workspace, stream=None):
    rows, cols = dy.shape
    _count(1)
    check(L.vp_bias_grad(dy.data_ptr(), dbias.data_ptr(), rows, cols, workspace.data_ptr(),
                         _stream(stream)), "vp_bias_grad")


def dropout_(x, p, seed, offset, stream=None):
    if p > 0:
        _count()
    check(L.vp_dropout(x.data_ptr(), x.numel(), p, seed, offset, _stream(stream)), "vp_dropout")
    return x


def set_seed(buf, value: int, stream=None):
    """Write the current (step, micro-batch) dropout seed into the device
    buffer every dropout site reads (outside captured graphs)."""
    _count(1)
    check(L.vp_set_seed(buf.data_ptr(), value & 0xFFFFFFFFFFFFFFFF, _stream(stream)), "vp_set_seed")


def fill_f32_(x, value=0.0, stream=None):
    _need(x, torch.float32, "fill_f32_")
    _count(1)
    check(L.vp_fill_f32(x.data_ptr(), value, x.numel(), _stream(stream)), "vp_fill_f32")
    return x


def dropout_dev_(x, p, seed, salt, stream=None):
    """x *= K7 mask (device seed, static salt), in place."""
    if p <= 0:
        return x
    _count(1)
    check(L.vp_dropout_dev(x.data_ptr(), x.numel(), p, seed.data_ptr(), salt & 0xFFFFFFFF,
                           _stream(stream)), "vp_dropout_dev")
    return x


def dropout_bwd(g, gy, p, seed, salt, dbias, workspace, stream=None):
    """gy = mask(g) (the gradient of a dropped-out branch) and dbias += its
    column sums, one pass."""
    rows, cols = g.shape
    _count(1)
    check(L.vp_dropout_bwd(g.data_ptr(), gy.data_ptr(), rows, cols, p, seed.data_ptr(),
                           salt & 0xFFFFFFFF, dbias.data_ptr(), workspace.data_ptr(),
                           _stream(stream)), "vp_dropout_bwd")
    return gy


def gemm_dropout(a, b, out, bias, resid, p, seed, salt, *, stream=None, out_ptr=None, ldd=None,
                 direct=False):
    """out[M,N] = resid + dropout(a @ b^T + bias) (a [M,K], b [N,K]); the K7
    mask applied in the GEMM epilogue."""
    _need(a, torch.bfloat16, "gemm.a")
    _need(b, torch.bfloat16, "gemm.b")
    M, K = a.shape
    N = b.shape[0]
    if out is not None:
        out_ptr, ldd = out.data_ptr(), out.stride(0)
    timing = GEMM_TIMING["on"]
    if timing:
        st = stream or torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
    _count()
    check(L.vp_gemm_bf16_dropout(1, 1, a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0),
                                 out_ptr, ldd, bias.data_ptr(), resid.data_ptr(), resid.stride(0),
                                 M, N, K, p, _p(seed) if p > 0 else None, salt & 0xFFFFFFFF,
                                 1 if direct else 0, _stream(stream)), "vp_gemm_bf16_dropout")
    if timing:
        e1.record(st)
        GEMM_TIMING["records"].append((2 * M * N * K, e0, e1,
                                       (M, N, K, True, True, EPI_BIAS_RESID)))
    return out


def add(a, b, y, stream=None):
    _count(1)
    check(L.vp_add(a.data_ptr(), b.data_ptr(), y.data_ptr(), a.numel(), _stream(stream)), "vp_add")
    return y


def mul(a, b, y, stream=None):
    _count(1)
    check(L.vp_mul(a.data_ptr(), b.data_ptr(), y.data_ptr(), a.numel(), _stream(stream)), "vp_mul")
    return y


def grad_norm_sq(g, out, stream=None):
    _count(1)
    check(L.vp_grad_norm_sq(g.data_ptr(), g.numel(), out.data_ptr(), _stream(stream)),
          "vp_grad_norm_sq")


def adam_step(master, weight, grad, m, v, flags, lr, beta1, beta2, eps, weight_decay,
              inv_loss_scale, max_grad_norm, step, stream=None):
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    _count(1)
    check(L.vp_adam_step(master.data_ptr(), weight.data_ptr(), grad.data_ptr(), m.data_ptr(),
                         v.data_ptr(), master.numel(), flags.data_ptr(), lr, beta1, beta2, eps,
                         weight_decay, inv_loss_scale, max_grad_norm, bc1, bc2, _stream(stream)),
          "vp_adam_step")


def grad_pack_bf16(x, y, stream=None):
    _count(1)
    check(L.vp_grad_pack_bf16(x.data_ptr(), y.data_ptr(), x.numel(), _stream(stream)),
          "vp_grad_pack_bf16")


def grad_unpack_bf16(x, y, stream=None):
    _count(1)
    check(L.vp_grad_unpack_bf16(x.data_ptr(), y.data_ptr(), x.numel(), _stream(stream)),
          "vp_grad_unpack_bf16")


def adam_step_dev(master, weight, grad, m, v, flags, lr, beta1, beta2, eps, weight_decay,
                  max_grad_norm, scaler, stream=None):
    """Fused unscale / skip / clip / AdamW with the unscale factor and the
    bias-correction step read from the device scaler state."""
    _count(1)
    check(L.vp_adam_step_dev(master.data_ptr(), weight.data_ptr(), grad.data_ptr(), m.data_ptr(),
                             v.data_ptr(), master.numel(), flags.data_ptr(), lr, beta1, beta2, eps,
                             weight_decay, max_grad_norm, scaler.data_ptr(), _stream(stream)),
          "vp_adam_step_dev")


def loss_scaler_update(scaler, flags, growth, backoff, window, min_scale=1.0,
                       max_scale=2.0 ** 64, stream=None):
    _count(1)
    check(L.vp_loss_scaler_update(scaler.data_ptr(), flags.data_ptr(), growth, backoff, window,
                                  min_scale, max_scale, _stream(stream)), "vp_loss_scaler_update")


def cast_f32_bf16(x, y, stream=None):
    _count(1)
    check(L.vp_cast_f32_bf16(x.data_ptr(), y.data_ptr(), x.numel(), _stream(stream)),
          "vp_cast_f32_bf16")


def p2p_put(dst_ptr: int, src, nbytes=None, stream=None):
    nbytes = src.numel() * src.element_size() if nbytes is None else nbytes
    _count(1)
    check(L.vp_p2p_put(dst_ptr, src.data_ptr(), nbytes, _stream(stream)), "vp_p2p_put")


class DeviceBuffer:
    """A dedicated cudaMalloc allocation (IPC-exportable at offset 0), exposed
    to torch zero-copy through __cuda_array_interface__."""

    def __init__(self, nbytes: int):
        p = vp()
        check(L.vp_device_alloc(nbytes, ctypes.byref(p)), "vp_device_alloc")
        self.ptr = p.value
        self.nbytes = nbytes

    def tensor(self, shape, dtype=torch.bfloat16, offset_bytes=0):
        import math
        itemsize = torch.tensor([], dtype=dtype).element_size()
        n = math.prod(shape)
        assert offset_bytes + n * itemsize <= self.nbytes
        typestr = {torch.bfloat16: "<f2", torch.float32: "<f4", torch.int64: "<i8",
                   torch.uint8: "|u1"}[dtype]
        holder = self

        class _Iface:
            __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                        "data": (self.ptr + offset_bytes, False), "version": 2,
                                        "strides": None}
            _keep = holder
        t = torch.as_tensor(_Iface(), device=torch.cuda.current_device())
        if dtype == torch.bfloat16:
            t = t.view(torch.bfloat16)
        return t

    def free(self):
        if self.ptr:
            L.vp_device_free(self.ptr)
            self.ptr = 0
