"""tcgen05 GEMM (vp_gemm_bf16) vs a torch fp32 reference of the same op.
Tolerance: bf16 output rounding + fp32-accumulate order, rel-L2 <= 5e-3
(<= 1e-5 for the fp32-output epilogues)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2111_04007_b200 import kernels as K


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12)).item()


def gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def dgelu(x):
    t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)


SHAPES = [(128, 256, 64), (256, 512, 128), (1000, 776, 320), (8192, 3072, 1024),
          (4096, 1920, 1920), (384, 128, 4096), (136, 1032, 72)]


@pytest.mark.parametrize("M,N,Kd", SHAPES)
@pytest.mark.parametrize("layout", ["nt", "nn", "tn", "tt"])
def test_gemm_layouts(M, N, Kd, layout):
    torch.manual_seed(0)
    dev = "cuda"
    a_k = layout[0] == "n"
    b_k = layout[1] == "t"
    A = torch.randn(M, Kd, device=dev).bfloat16()
    B = torch.randn(N, Kd, device=dev).bfloat16()
    a = A if a_k else A.t().contiguous()
    b = B if b_k else B.t().contiguous()
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    K.gemm(a, b, out, a_kmajor=a_k, b_kmajor=b_k)
    ref = A.float() @ B.float().t()
    assert rel(out, ref) < 5e-3


def test_gemm_epilogues():
    torch.manual_seed(1)
    M, N, Kd = 512, 768, 256
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    B = (torch.randn(N, Kd, device="cuda") * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    base = A.float() @ B.float().t()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(A, B, out, epilogue=K.EPI_BIAS, bias=bias)
    assert rel(out, base + bias.float()) < 5e-3
    pre = torch.empty_like(out)
    K.gemm(A, B, out, epilogue=K.EPI_BIAS_GELU, bias=bias, aux=pre)
    # the saving forward stores gelu'(pre-activation) for the DGELU multiply
    xpre = (base + bias.float()).bfloat16().float()
    assert rel(pre, dgelu(xpre)) < 1e-2
    assert rel(out, gelu(base + bias.float())) < 1e-2
    out_only = torch.empty_like(out)  # no pre-activation output (non-saving forward)
    K.gemm(A, B, out_only, epilogue=K.EPI_BIAS_GELU, bias=bias)
    assert torch.equal(out_only, out)
    res = torch.randn(M, N, device="cuda").bfloat16()
    out2 = res.clone()
    K.gemm(A, B, out2, epilogue=K.EPI_BIAS_RESID, bias=bias, aux=out2)
    assert rel(out2, res.float() + base + bias.float()) < 5e-3
    x = torch.randn(M, N, device="cuda").bfloat16()
    K.gemm(A, B, out, epilogue=K.EPI_DGELU, aux=x)   # aux = gelu'(pre) from the forward
    assert rel(out, base * x.float()) < 5e-3
    # end to end: forward-saved derivative -> DGELU == acc * gelu'(pre)
    K.gemm(A, B, out, epilogue=K.EPI_BIAS_GELU, bias=bias, aux=pre)
    K.gemm(A, B, out_only, epilogue=K.EPI_DGELU, aux=pre)
    assert rel(out_only, base * dgelu(xpre)) < 1e-2
    acc = torch.randn(M, N, device="cuda")
    acc0 = acc.clone()
    K.gemm(A, B, acc, epilogue=K.EPI_ACC_F32)
    assert rel(acc, acc0 + base) < 1e-5
    K.gemm(A, B, acc, epilogue=K.EPI_STORE_F32)
    assert rel(acc, base) < 1e-5


def test_gemm_wgrad_shape():
    # dW[N,K] += dY^T X with T=8192 reduction (both operands MN-major).
    torch.manual_seed(2)
    T, N, Kd = 8192, 1024, 4096
    dy = torch.randn(T, N, device="cuda").bfloat16()
    x = torch.randn(T, Kd, device="cuda").bfloat16()
    dw = torch.zeros(N, Kd, device="cuda")
    K.gemm(dy, x, dw, a_kmajor=False, b_kmajor=False, epilogue=K.EPI_ACC_F32)
    ref = dy.float().t() @ x.float()
    assert rel(dw, ref) < 1e-5


@pytest.mark.parametrize("direct", [False, True])
def test_gemm_paths_agree(direct):
    # 2-CTA TMA-store path and the 1-SM direct-store path (peer-pointer
    # writes) give the same numbers for every epilogue.
    torch.manual_seed(4)
    M, N, Kd = 640, 1152, 320
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    B = (torch.randn(N, Kd, device="cuda") * 0.1).bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda").bfloat16()
    base = A.float() @ B.float().t()
    out = res.clone()
    K.gemm(A, B, out, epilogue=K.EPI_BIAS_RESID, bias=bias, aux=out, direct=direct)
    assert rel(out, res.float() + base + bias.float()) < 5e-3
    act = torch.empty_like(res)
    der = torch.empty_like(res)
    K.gemm(A, B, act, epilogue=K.EPI_BIAS_GELU, bias=bias, aux=der, direct=direct)
    xpre = (base + bias.float()).bfloat16().float()
    assert rel(act, gelu(xpre)) < 1e-2
    assert rel(der, dgelu(xpre)) < 1e-2
    dg = torch.empty_like(res)
    K.gemm(A, B, dg, epilogue=K.EPI_DGELU, aux=der, direct=direct)
    assert rel(dg, base * dgelu(xpre)) < 1e-2


@pytest.mark.parametrize("T,N,Kd", [(8192, 1024, 1024), (8192, 3072, 1024), (4096, 1920, 7680),
                                    (1000, 520, 264)])
def test_gemm_wgrad_splitk(T, N, Kd):
    # small output, long reduction -> split-K with TMA reduce-add epilogue
    torch.manual_seed(5)
    dy = torch.randn(T, N, device="cuda").bfloat16()
    x = torch.randn(T, Kd, device="cuda").bfloat16()
    dw = torch.randn(N, Kd, device="cuda")
    dw0 = dw.clone()
    K.gemm(dy, x, dw, a_kmajor=False, b_kmajor=False, epilogue=K.EPI_ACC_F32)
    assert rel(dw, dw0 + dy.float().t() @ x.float()) < 1e-5


def test_gemm_deterministic():
    torch.manual_seed(3)
    A = torch.randn(2048, 1024, device="cuda").bfloat16()
    B = torch.randn(3072, 1024, device="cuda").bfloat16()
    o1 = torch.empty(2048, 3072, device="cuda", dtype=torch.bfloat16)
    o2 = torch.empty_like(o1)
    K.gemm(A, B, o1)
    K.gemm(A, B, o2)
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("M,N", [(8192, 4096), (300, 520), (1000, 96)])
def test_gemm_fused_bias_grad(M, N):
    """DGELU dgrad with the FC1 bias gradient (column sums of the output,
    fp32 before rounding) fused into the epilogue: matches a separate column
    sum and is deterministic."""
    torch.manual_seed(2)
    Kd = 256
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    B = (torch.randn(Kd, N, device="cuda") * 0.05).bfloat16()
    x = torch.randn(M, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(K.gemm_dbias_ws_elems(M, N), device="cuda")
    db = torch.ones(N, device="cuda")
    K.gemm(A, B, out, b_kmajor=False, epilogue=K.EPI_DGELU, aux=x, dbias=db, dbias_ws=ws)
    ref = (A.float() @ B.float()) * x.float()   # aux = gelu'(pre)
    assert rel(out, ref) < 1e-2
    assert rel(db, 1 + ref.sum(0)) < 1e-3
    db2 = torch.ones(N, device="cuda")
    out2 = torch.empty_like(out)
    K.gemm(A, B, out2, b_kmajor=False, epilogue=K.EPI_DGELU, aux=x, dbias=db2, dbias_ws=ws)
    assert torch.equal(db, db2) and torch.equal(out, out2)


def test_gemm_aux_epilogue_ragged_n_many_tiles():
    """BIAS_RESID / DGELU / RESID with a ragged last N tile over many
    persistent tiles per cluster (aux-prefetch barrier phases must follow the
    chunks actually prefetched; 2.5B shapes: N = 1920, 5760)."""
    torch.manual_seed(5)
    for M, N, Kd in ((8192, 1920, 256), (8192, 5760, 128), (4096, 1920, 1920)):
        A = torch.randn(M, Kd, device="cuda").bfloat16()
        B = (torch.randn(N, Kd, device="cuda") * 0.05).bfloat16()
        bias = torch.randn(N, device="cuda").bfloat16()
        res = torch.randn(M, N, device="cuda").bfloat16()
        out = res.clone()
        K.gemm(A, B, out, epilogue=K.EPI_BIAS_RESID, bias=bias, aux=out)
        ref = res.float() + A.float() @ B.float().t() + bias.float()
        assert rel(out, ref) < 5e-3
        x = torch.randn(M, N, device="cuda").bfloat16()
        out2 = torch.empty_like(x)
        K.gemm(A, B, out2, epilogue=K.EPI_DGELU, aux=x)
        assert rel(out2, (A.float() @ B.float().t()) * x.float()) < 1e-2
