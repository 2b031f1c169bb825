"""NCHW convolution geometries through the C ABI (lsb_conv2d_nchw) on device
buffers, against an f64 convolution of the same inputs (strict per-element
rule).  Exercises the planar tensor-core kernel's TMA box alignment (pads
whose columns start off a 16-B boundary, conv_planar.cuh `wsh`), dilation,
large taps, ragged channel / filter counts, strided X views, and the
fallbacks when the planar preconditions fail (unaligned X rows, halos that
do not fit)."""

import pytest

import common

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

# (N, C, H, W, CO, R, S, pad_h, pad_w, dil_h, dil_w), planar kernel expected
GEOMS = [
    ((2, 16, 20, 20, 64, 3, 3, 0, 0, 1, 1), True),    # no padding: box from w = 0
    ((2, 32, 24, 24, 64, 3, 3, 2, 2, 2, 2), True),    # pad 2 (box from -4, wsh 2), dilation 2
    ((1, 8, 32, 32, 64, 7, 7, 3, 3, 1, 1), True),     # pad 3 (wsh 1), 7x7 taps
    ((3, 20, 17, 28, 40, 3, 3, 1, 1, 1, 1), True),    # 20 channels (zero-filled block), 40 filters
    ((2, 16, 16, 16, 96, 1, 1, 0, 0, 1, 1), True),    # 1x1, two filter tiles
    ((2, 16, 20, 24, 64, 3, 5, 1, 2, 1, 2), True),    # asymmetric taps / pads / dilation
    ((2, 16, 15, 15, 64, 3, 3, 1, 1, 1, 1), False),   # 15-float rows: not TMA-able -> fallback
    ((1, 16, 8, 100, 64, 3, 3, 1, 1, 1, 1), False),   # wide rows: raw box too big -> fallback
]


def _conv_f64(x, w, ph, pw, dh, dw):
    import torch.nn.functional as F
    return F.conv2d(x.double(), w.double(), padding=(ph, pw), dilation=(dh, dw))


def _run(x, w, o, geom):
    from paper_2205_00618_b200 import native
    N, C, H, W, CO, R, S, ph, pw, dh, dw = geom
    d = native.ConvDesc()
    d.N, d.C, d.H, d.W, d.CO, d.R, d.S = N, C, H, W, CO, R, S
    d.HO, d.WO = o.shape[2], o.shape[3]
    d.stride_h = d.stride_w = 1
    d.pad_h, d.pad_w, d.dil_h, d.dil_w = ph, pw, dh, dw
    d.fill = 0.0
    d.x, d.w, d.o = x.data_ptr(), w.data_ptr(), o.data_ptr()
    for i in range(4):
        d.sx[i], d.sw[i], d.so[i] = x.stride(i), w.stride(i), o.stride(i)
    d.combine, d.reduce = 1, 0     # (mul, add): program.KIND_CODE
    d.beta, d.beta_in_loop, d.n_epi = 1.0, 0, 0
    native.conv2d_nchw(d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


@pytest.mark.parametrize("algo", ["tf32x3_planar", None])
@pytest.mark.parametrize("geom,planar", GEOMS, ids=[str(g) for g, _ in GEOMS])
def test_conv_geometry(geom, planar, algo, monkeypatch):
    from paper_2205_00618_b200 import native
    native.init(0)
    if algo:
        monkeypatch.setenv("LSB_GEMM_ALGO", algo)
    else:
        monkeypatch.delenv("LSB_GEMM_ALGO", raising=False)
    N, C, H, W, CO, R, S, ph, pw, dh, dw = geom
    g = torch.Generator(device="cpu").manual_seed(sum(geom))
    x = (torch.rand(N, C, H, W, generator=g) * 2 - 1).cuda()
    w = (torch.randn(CO, C, R, S, generator=g) * (2.0 / (C * R * S)) ** 0.5).cuda()
    ref = _conv_f64(x, w, ph, pw, dh, dw)
    o = torch.full(ref.shape, float("nan"), device="cuda")
    _run(x, w, o, geom)
    got, want = o.double().cpu().numpy(), ref.cpu().numpy()
    ok = common.strict_ok(got, want)
    assert ok.all(), (float(ok.mean()), common.ref_metric(got, want))
    kind, nt = native.last_conv_kernel()
    if algo or 2 * CO * ref.shape[2] * ref.shape[3] * N * C * R * S >= 1 << 28:
        assert (kind == 2) == planar, (kind, nt)


def test_conv_strided_x_view(monkeypatch):
    """X as a view with padded rows and channels (sx = (C*H*64, H*64, 64, 1)):
    the TMA map takes the view's strides."""
    from paper_2205_00618_b200 import native
    native.init(0)
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3_planar")
    g = torch.Generator(device="cpu").manual_seed(5)
    base = (torch.rand(2, 24, 30, 64, generator=g) * 2 - 1).cuda()
    x = base[:, :20, :28, :56]
    w = (torch.randn(64, 20, 3, 3, generator=g) * 0.1).cuda()
    ref = _conv_f64(x, w, 1, 1, 1, 1)
    o = torch.full(ref.shape, float("nan"), device="cuda")
    _run(x, w, o, (2, 20, 28, 56, 64, 3, 3, 1, 1, 1, 1))
    ok = common.strict_ok(o.double().cpu().numpy(), ref.cpu().numpy())
    assert ok.all(), float(ok.mean())
    assert native.last_conv_kernel()[0] == 2


def test_conv_output_view_keeps_neighbours(monkeypatch):
    """O as a channel slice of a larger tensor: stores stay inside the view
    (the planar kernel's ragged row ends and its per-image tiles)."""
    from paper_2205_00618_b200 import native
    native.init(0)
    monkeypatch.setenv("LSB_GEMM_ALGO", "tf32x3_planar")
    g = torch.Generator(device="cpu").manual_seed(6)
    x = (torch.rand(2, 16, 24, 24, generator=g) * 2 - 1).cuda()
    w = (torch.randn(64, 16, 3, 3, generator=g) * 0.1).cuda()
    big = torch.full((2, 80, 24, 24), 7.0, device="cuda")
    o = big[:, 8:72]
    ref = _conv_f64(x, w, 1, 1, 1, 1)
    _run(x, w, o, (2, 16, 24, 24, 64, 3, 3, 1, 1, 1, 1))
    assert common.strict_ok(o.double().cpu().numpy(), ref.cpu().numpy()).all()
    assert bool((big[:, :8] == 7.0).all()) and bool((big[:, 72:] == 7.0).all())
    assert native.last_conv_kernel()[0] == 2
