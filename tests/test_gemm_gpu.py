"""tcgen05 GEMM parity vs a torch fp32 reference of the same op (bf16 inputs)."""

import pytest
import torch

from paper_2507_10392_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _rand(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


def _gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def _gelu_grad(x):
    k0, k1 = 0.7978845608028654, 0.044715
    t = torch.tanh(k0 * (x + k1 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * k0 * (1 + 3 * k1 * x * x)


def _close(out, ref, tol=2e-2):
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    assert err / scale < tol, f"rel max err {err / scale:.3e}"


SHAPES = [(128, 128, 64), (256, 256, 128), (384, 768, 768), (200, 136, 72), (1024, 2304, 768),
          (8192, 50304 // 8, 768), (128, 64, 1024), (130, 300, 96)]


@pytest.mark.parametrize("M,N,Kd", SHAPES)
def test_gemm_tn(cuda, M, N, Kd):
    torch.manual_seed(0)
    a = _rand(M, Kd)
    b = _rand(N, Kd)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(a, b, out)
    torch.cuda.synchronize()
    _close(out, a.float() @ b.float().t())


@pytest.mark.parametrize("M,N,Kd", SHAPES)
def test_gemm_dgrad_layout(cuda, M, N, Kd):
    if N % 8:
        pytest.skip("MN-major B needs a 16-byte row pitch (TMA)")
    # out = a @ w where w is stored [K, N] (N contiguous): B operand MN-major
    torch.manual_seed(1)
    a = _rand(M, Kd)
    w = _rand(Kd, N)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(a, w, out, b_t=True)
    torch.cuda.synchronize()
    _close(out, a.float() @ w.float())


@pytest.mark.parametrize("M,N,Kd", [(128, 128, 64), (768, 2304, 1024), (3072, 768, 2048),
                                    (200, 136, 72), (64, 192, 4096)])
def test_gemm_wgrad_layout_f32_accumulate(cuda, M, N, Kd):
    # dW[M,N] += dY^T @ X with dY [K, M], X [K, N]: both MN-major, fp32 accumulate
    torch.manual_seed(2)
    dy = _rand(Kd, M)
    x = _rand(Kd, N)
    c = torch.randn(M, N, device="cuda")
    ref = c + dy.float().t() @ x.float()
    K.gemm(dy, x, c, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0)
    torch.cuda.synchronize()
    _close(c, ref, tol=1e-3)


@pytest.fixture(params=["tma", "direct"])
def epi_path(request):
    """GEMM entry for the TMA-store epilogue (default path) and for the direct-store
    epilogue (explicit tile request)."""
    if request.param == "direct":
        return lambda *a, **kw: K.gemm_tile(*a, tma_epi=False, **kw)
    return K.gemm


@pytest.mark.parametrize("M,N,Kd", [(512, 1536, 384), (200, 136, 72), (130, 328, 96),
                                    (512, 768, 2048), (1000, 2304, 2560)])
def test_gemm_epilogues(cuda, epi_path, M, N, Kd):
    torch.manual_seed(3)
    a = _rand(M, Kd)
    b = _rand(N, Kd, scale=0.05)
    bias = _rand(N)
    acc = a.float() @ b.float().t()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    epi_path(a, b, out, epilogue=K.EPI_BIAS, bias=bias)
    _close(out, acc + bias.float())
    aux = torch.empty_like(out)
    epi_path(a, b, out, epilogue=K.EPI_BIAS_GELU, bias=bias, aux=aux)
    _close(aux, acc + bias.float())
    _close(out, _gelu(aux.float()))
    r = _rand(M, N)
    epi_path(a, b, out, epilogue=K.EPI_BIAS_RESID, bias=bias, resid=r)
    _close(out, acc + bias.float() + r.float())
    epi_path(a, b, out, epilogue=K.EPI_GELU_BWD, aux=aux)
    _close(out, acc * _gelu_grad(aux.float()))
    epi_path(a, b, out, epilogue=K.EPI_BIAS_GELU_NA, bias=bias)
    _close(out, _gelu((acc + bias.float()).bfloat16().float()))
    torch.cuda.synchronize()


@pytest.mark.parametrize("M,N,Kd", [(256, 384, 512), (200, 136, 2048), (768, 768, 8192)])
def test_gemm_f32_store_and_accumulate(cuda, epi_path, M, N, Kd):
    """fp32 epilogue: beta = 0 (plain store) and beta = 1 (accumulate / split-K)."""
    torch.manual_seed(4)
    dy = _rand(Kd, M)
    x = _rand(Kd, N)
    prod = dy.float().t() @ x.float()
    c = torch.full((M, N), 7.0, device="cuda")
    epi_path(dy, x, c, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=0.0)
    torch.cuda.synchronize()
    _close(c, prod, tol=1e-3)
    c2 = torch.randn(M, N, device="cuda")
    ref = c2 + prod
    epi_path(dy, x, c2, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0)
    torch.cuda.synchronize()
    _close(c2, ref, tol=1e-3)


@pytest.mark.parametrize("raster", ["0", "1"])
@pytest.mark.parametrize("ctas", ["1", "2"])
@pytest.mark.parametrize("M,N,Kd,lay", [(1000, 392, 4096, "dgrad"), (640, 264, 2048, "tn"),
                                        (2944, 384, 1024, "wgrad")])
def test_gemm_tile_rasters(cuda, raster, ctas, M, N, Kd, lay):
    """Both tile rasters (M-fastest; N-fastest, used when A outgrows L2) and both CTA
    modes, on ragged shapes, against torch fp32 (pinned through zb_gemm_bf16_tile)."""
    tile = dict(raster=int(raster), pair=int(ctas) - 1)
    torch.manual_seed(5)
    if lay == "tn":
        a, b = _rand(M, Kd), _rand(N, Kd)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        K.gemm_tile(a, b, out, **tile)
        ref = a.float() @ b.float().t()
    elif lay == "dgrad":
        a, b = _rand(M, Kd), _rand(Kd, N)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        K.gemm_tile(a, b, out, **tile, b_t=True)
        ref = a.float() @ b.float()
    else:
        a, b = _rand(Kd, M), _rand(Kd, N)
        out = torch.full((M, N), 0.5, device="cuda")
        K.gemm_tile(a, b, out, **tile, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0)
        ref = 0.5 + a.float().t() @ b.float()
    torch.cuda.synchronize()
    _close(out, ref, tol=1e-3 if lay == "wgrad" else 2e-2)


@pytest.mark.parametrize("bn", ["256", "192"])
@pytest.mark.parametrize("M,N,Kd,lay,epi", [(512, 512, 256, "tn", 0), (1000, 768, 3072, "tn", 3),
                                            (8192, 3072, 768, "tn", 7), (1024, 1024, 2048, "dgrad", 0),
                                            (2304, 1024, 4096, "wgrad", 5), (768, 1536, 768, "tn", 2)])
def test_gemm_multicast_pairs(cuda, bn, M, N, Kd, lay, epi):
    """Two CTA pairs per cluster sharing the A tile through TMA multicast
    (pair=2), every layout and the epilogue families, vs torch fp32."""
    n_tiles = (N + int(bn) - 1) // int(bn)
    if n_tiles % 2 or (lay != "tn" and bn == "192"):
        pytest.skip("multicast pairs need an even n-tile count (MN-major B: BN 256)")
    tile = dict(pair=2, bn=int(bn))
    torch.manual_seed(7)
    bias = _rand(N, scale=0.5)
    if lay == "tn":
        a, b = _rand(M, Kd, scale=0.5), _rand(N, Kd, scale=0.5)
        ref = a.float() @ b.float().t()
        kw = {}
    elif lay == "dgrad":
        a, b = _rand(M, Kd, scale=0.5), _rand(Kd, N, scale=0.5)
        ref = a.float() @ b.float()
        kw = {"b_t": True}
    else:
        a, b = _rand(Kd, M, scale=0.5), _rand(Kd, N, scale=0.5)
        ref = a.float().t() @ b.float()
        kw = {"a_t": True, "b_t": True}
    if epi == 5:
        out = torch.full((M, N), 0.25, device="cuda")
        K.gemm_tile(a, b, out, **tile, epilogue=5, beta=1.0, **kw)
        torch.cuda.synchronize()
        _close(out, ref + 0.25, tol=1e-3)
        return
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    if epi == 0:
        K.gemm_tile(a, b, out, **tile, **kw)
        exp = ref
    elif epi == 3:
        r = _rand(M, N)
        K.gemm_tile(a, b, out, **tile, epilogue=3, bias=bias, resid=r, **kw)
        exp = ref + bias.float() + r.float()
    elif epi == 7:
        K.gemm_tile(a, b, out, **tile, epilogue=7, bias=bias, **kw)
        exp = _gelu(ref + bias.float())
    else:  # 2: pre-activation to aux, GELU to out
        aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        K.gemm_tile(a, b, out, **tile, epilogue=2, bias=bias, aux=aux, **kw)
        torch.cuda.synchronize()
        _close(aux, ref + bias.float())
        exp = _gelu(ref + bias.float())
    torch.cuda.synchronize()
    _close(out, exp)
