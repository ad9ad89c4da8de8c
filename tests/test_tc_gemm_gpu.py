"""The tcgen05 implicit-GEMM path (fp16 shapes with 64-multiple channels,
the im2col stem, affine layers) against the oracle and the SIMT kernel."""

import ctypes as C

import numpy as np
import pytest

from oracle import nnl_oracle as O

pytestmark = pytest.mark.gpu

CONV = [  # (B, cin, cout, k, stride, pad, hw)
    (2, 64, 128, 1, 1, 0, 8),      # 1x1 s1: TMA A / TMA B
    (2, 64, 64, 3, 1, 1, 8),       # 3x3 gather, BN=64
    (3, 128, 128, 3, 2, 1, 9),     # strided 3x3, ragged M tail
    (2, 64, 256, 1, 2, 0, 10),     # 1x1 s2 (downsample)
    (2, 3, 64, 7, 2, 3, 20),       # stem: 4-channel padded gather (A / B)
    (8, 3, 64, 7, 2, 3, 64),       # stem: many k-blocks, split-K wgrad
    (3, 1, 16, 5, 1, 0, 12),       # 1 channel (LeNet conv1), ragged taps
    (2, 3, 32, 5, 2, 2, 17),       # stride 2, even pad, odd width: pair loads, no shift
    (2, 2, 16, 3, 2, 0, 15),       # stride 2, pad 0, 2 channels
    (2, 3, 24, 4, 2, 1, 12),       # even filter width (no padded tap slot)
    (2, 4, 64, 3, 1, 1, 10),       # 4 channels: no channel padding
    (2, 12, 64, 3, 1, 1, 10),      # 12 channels: explicit im2col
    (4, 256, 64, 1, 1, 0, 7),      # 1x1 reduce, 7x7 maps
    (8, 256, 512, 1, 1, 0, 14),    # 256-wide tiles
    (4, 256, 512, 1, 2, 0, 14),    # 1x1 s2 dgrad: row remap + zero fill
    (16, 128, 256, 3, 1, 1, 14),   # 3x3 gather with 256-wide tiles
    (64, 64, 128, 3, 1, 1, 20),    # > 148 work units: persistent tile loop
    (4, 64, 64, 3, 1, 1, 24),      # shared-halo tiles, last tile row past the image
    (2, 64, 64, 3, 1, 1, 56),      # shared-halo tiles at the ResNet-50 stage-1 extent
    (4, 64, 128, 3, 2, 1, 16),     # strided 3x3 dgrad: 4 parity-class GEMMs
    (2, 64, 64, 3, 1, 0, 9),       # valid (pad 0) 3x3: dgrad im2col bounding box
    (2, 128, 64, 3, 1, 1, 14),     # halo wgrad: 14x14 maps in 2x2 8x8 tiles, two channel blocks
    (3, 64, 192, 3, 1, 1, 17),     # halo wgrad: three output blocks, ragged 17x17 tiles
    (2, 512, 512, 3, 1, 1, 14),    # halo wgrad: 64 block pairs
    (2, 512, 512, 3, 1, 1, 7),     # 7x7 maps: the per-tap im2col wgrad
    (2, 16, 16, 5, 1, 0, 12),      # LeNet conv2: dgrad as a forward conv over flipped weights
    (3, 16, 32, 3, 1, 1, 9),       # same, padded
    (2, 64, 128, 1, 2, 0, 9),      # 1x1 s2 dgrad, odd extent: the zero-fill pass
]


def test_conv_backward_accumulate_mode(nnl):
    """acc=True writes q(prev + grad) (R2) on every tcgen05 path."""
    import paper_2102_06725_b200.functions as F
    _half(nnl)
    for geom in [(2, 64, 128, 1, 2, 0, 8), (2, 64, 64, 3, 1, 1, 8), (2, 128, 256, 1, 1, 0, 6),
                 (2, 64, 64, 3, 2, 1, 10), (2, 3, 64, 7, 2, 3, 20), (2, 16, 16, 5, 1, 0, 12)]:
        b, cin, cout, k, s, p, hw = geom
        rng = np.random.default_rng(k + cout)
        x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
        w = rng.uniform(-0.2, 0.2, (cout, cin, k, k)).astype(np.float32)
        bias = np.zeros(cout, np.float32)
        vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
        for v, a in zip(vs, (x, w, bias)):
            v.d = a
        y = F.convolution(*vs, stride=(s, s), pad=(p, p))
        y.forward()
        gy = O.q16(rng.uniform(-1, 1, y.shape).astype(np.float32))
        y.g = gy
        prev = [O.q16(rng.uniform(-1, 1, a.shape).astype(np.float32)) for a in (x, w, bias)]
        for v, pv in zip(vs, prev):
            v.g = pv
        node = y.parent
        node.impl.backward(node, [y.grad], [v.grad for v in vs], [True] * 3)
        ov = [O.Var(a, half=True, need_grad=True) for a in (x, w, bias)]
        oy = O.conv2d(*ov, (s, s), (p, p), True)
        gxs = oy.parent.bwd([gy], [True, True, True])
        for v, pv, want in zip(vs, prev, gxs):
            assert _rel_err(v.g, O.q16(pv + want)) < 4e-3, geom


def _half(nn):
    nn.set_default_context(nn.ExecutionContext(type_config=nn.TypeConfig.HALF))


def _rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b).max() / (np.abs(b).max() + 1e-6)


@pytest.mark.parametrize("geom", CONV)
def test_conv_tc_vs_oracle(nnl, geom):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(cin * 7 + cout + k)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.2, 0.2, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (cout,)).astype(np.float32)
    vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
    for v, a in zip(vs, (x, w, bias)):
        v.d = a
    y = F.convolution(*vs, stride=(s, s), pad=(p, p))
    gy = O.q16(rng.uniform(-1, 1, y.shape).astype(np.float32))
    before = _lib.lib().nnl_launch_count(0)
    y.forward()
    y.g = gy
    node = y.parent
    for v in vs:
        v.grad.fill(0.0)
    node.impl.backward(node, [y.grad], [v.grad for v in vs], [False] * 3)
    ov = [O.Var(a, half=True, need_grad=True) for a in (x, w, bias)]
    oy = O.conv2d(*ov, (s, s), (p, p), True)
    gxs = oy.parent.bwd([gy], [True, True, True])
    assert _rel_err(y.d, oy.value) < 4e-3
    for v, want in zip(vs, gxs):
        assert _rel_err(v.g, O.q16(want)) < 4e-3, (geom, v.shape)
    assert _lib.lib().nnl_launch_count(0) > before


def test_conv_tc_matches_simt_kernel(nnl):
    """Same inputs through both kernels (tensor cores vs SIMT fp32 accumulation)."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (2, 64, 12, 12)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (128, 64, 3, 3)).astype(np.float32)
    bias = np.zeros(128, np.float32)
    outs = []
    for tc in (1, 0):
        prev = _lib.lib().nnl_set_tc_enabled(tc)
        try:
            vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(1, 1), pad=(1, 1))
            y.forward()
            y.backward(1.0)
            outs.append([y.d, vs[0].g, vs[1].g])
        finally:
            _lib.lib().nnl_set_tc_enabled(prev)
    for a, b in zip(*outs):
        assert _rel_err(a, b) < 2e-3


@pytest.mark.parametrize("geom", [(3, 64, 64, 3, 1, 1, 9), (2, 3, 64, 7, 2, 3, 30),
                                  (4, 64, 40, 1, 1, 0, 12), (2, 64, 256, 1, 1, 0, 20)])
def test_conv_stats_epilogue(nnl, geom):
    """BN partial statistics from the conv epilogue equal column sums of the
    rounded output (3x3 gather, narrow-channel stem, ragged N, 256-wide tiles)."""
    import paper_2102_06725_b200.functions as F
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (cout, cin, k, k)).astype(np.float32)
    vs = [nnl.Variable(a.shape) for a in (x, w, np.zeros(cout, np.float32))]
    for v, a in zip(vs, (x, w, np.zeros(cout, np.float32))):
        v.d = a
    y = F.convolution(*vs, stride=(s, s), pad=(p, p))
    node = y.parent
    # the epilogue sums are centred on the consuming BN's shift K (its previous
    # batch mean): a stand-in BN node carries a ready shift
    import torch

    class _Bn:
        state = {"shift_ready": True,
                 "shift": torch.from_numpy(rng.uniform(-0.2, 0.2, cout).astype(np.float32)).cuda()}
    node.state["emit_stats"] = True
    node.state["stat_bn"] = _Bn
    node.impl.forward(node, [v.data for v in vs], [y.data])
    y.data.mark_set()
    st = y.parent.state["stats"].cpu().numpy()
    rows = y.parent.state["stat_rows"]
    assert rows > 0
    parts = st[: rows * 2 * cout].reshape(rows, 2, cout)
    kc = _Bn.state["shift"].cpu().numpy().astype(np.float64)
    yd = y.d.transpose(0, 2, 3, 1).reshape(-1, cout).astype(np.float64) - kc
    # idle rows of partial tiles must not count (as -K)
    np.testing.assert_allclose(parts[:, 0].sum(0), yd.sum(0), rtol=1e-4, atol=1e-3)
    np.testing.assert_allclose(parts[:, 1].sum(0), (yd ** 2).sum(0), rtol=1e-4, atol=1e-3)
    ov = [O.Var(a, half=True) for a in (x, w, np.zeros(cout, np.float32))]
    assert _rel_err(y.d, O.conv2d(*ov, (s, s), (p, p), True).value) < 4e-3


@pytest.mark.parametrize("dims", [(32, 128, 64), (16, 256, 1000), (256, 2048, 1000)])
def test_affine_tc_vs_oracle(nnl, dims):
    import paper_2102_06725_b200.functions as F
    _half(nnl)
    bsz, i, o = dims
    rng = np.random.default_rng(i + o)
    x = rng.uniform(-1, 1, (bsz, i)).astype(np.float32)
    w = rng.uniform(-0.05, 0.05, (i, o)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, (o,)).astype(np.float32)
    vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
    for v, a in zip(vs, (x, w, bias)):
        v.d = a
    y = F.affine(*vs)
    y.forward()
    y.backward(1.0)
    ov = [O.Var(a, half=True, need_grad=True) for a in (x, w, bias)]
    oy = O.affine(*ov, True)
    O.backward(oy, 1.0)
    assert _rel_err(y.d, oy.value) < 4e-3
    for v, o_ in zip(vs, ov):
        assert _rel_err(v.g, o_.grad) < 4e-3


def test_cta_pairs_match_single_cta(nnl):
    """256-row CTA-pair tiles (tcgen05 cta_group::2) give the same sums as
    128-row tiles: bit-identical where no split-K is involved (fprop, dgrad),
    within f32 regrouping of the split-K partials for wgrad."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (128, 256, 14, 14)).astype(np.float32)
    w = rng.uniform(-0.05, 0.05, (256, 256, 3, 3)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (256,)).astype(np.float32)
    outs = []
    for pairs in (1, 0):
        prev = _lib.lib().nnl_set_tc_pairs(pairs)
        try:
            vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(1, 1), pad=(1, 1))
            y.forward()
            y.backward(1.0)
            outs.append([y.d, vs[0].g, vs[1].g])
        finally:
            _lib.lib().nnl_set_tc_pairs(prev)
    for a, c in zip(outs[0], outs[1]):
        assert _rel_err(a, c) < 2e-3


@pytest.mark.parametrize("geom", [(64, 64, 64, 3, 1, 1, 28), (32, 64, 256, 1, 1, 0, 28),
                                  (16, 3, 64, 7, 2, 3, 112)])
def test_resident_b_matches_streamed(nnl, geom):
    """Weight-stationary tiles (whole B resident in shared memory) give the same
    bits as streaming B through the ring (fprop and dgrad need no split-K here)."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (cout,)).astype(np.float32)
    outs = []
    for resb in (1, 0):
        prev = _lib.lib().nnl_set_tc_resident_b(resb)
        try:
            vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(s, s), pad=(p, p))
            y.forward()
            y.backward(1.0)
            outs.append([y.d, vs[0].g if cin % 8 == 0 else None])
        finally:
            _lib.lib().nnl_set_tc_resident_b(prev)
    assert np.array_equal(outs[0][0], outs[1][0])
    if outs[0][1] is not None:
        assert np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("geom", [(4, 3, 64, 7, 2, 3, 40), (16, 3, 64, 7, 2, 3, 112)])
def test_stem_s2d4_matches_s2d16(nnl, geom):
    """The stem over the row-concatenated 64-channel space-to-depth tensor
    (128 B im2col rows) reduces in the same (block row, block column, slot)
    order as the 16-channel one (32 B rows): identical output and weight
    gradient bits."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (cout,)).astype(np.float32)
    outs = []
    for mode in (1, 0):
        prev = _lib.lib().nnl_set_tc_s2d4(mode)
        try:
            vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(s, s), pad=(p, p))
            y.forward()
            y.backward(1.0)
            outs.append([y.d, vs[1].g, vs[2].g])
        finally:
            _lib.lib().nnl_set_tc_s2d4(prev)
    for a, c in zip(outs[0], outs[1]):
        assert np.array_equal(a, c)


@pytest.mark.parametrize("geom", [(4, 64, 64, 3, 1, 1, 56), (8, 128, 128, 3, 1, 1, 28),
                                  (32, 64, 128, 3, 1, 1, 14), (2, 128, 64, 3, 1, 1, 32),
                                  (16, 256, 256, 3, 1, 1, 14)])
def test_spatial_tiles_match_im2col(nnl, geom):
    """Spatial pixel-box tiles (one tiled 4D TMA box per tap) against the TMA
    im2col path.  Both reduce each output in (tap, channel block) order, but
    the im2col path may split K across CTAs when the grid is small (f32
    partials summed afterwards), and wgrad sums pixels in box order: the
    results agree to f32 rounding of the accumulator."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(12)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (cout,)).astype(np.float32)
    gy = rng.uniform(-1, 1, (b, cout, hw, hw)).astype(np.float32)
    outs = []
    for mode in (2, 0):
        prev = _lib.lib().nnl_set_tc_tile4(mode)
        try:
            vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(s, s), pad=(p, p))
            y.forward()
            y.backward(1.0)
            y.g = gy
            for v in vs:
                v.grad.fill(0.0)
            y.parent.impl.backward(y.parent, [y.grad], [v.grad for v in vs], [False] * 3)
            outs.append([y.d, vs[0].g, vs[1].g])
        finally:
            _lib.lib().nnl_set_tc_tile4(prev)
    for a, c in zip(outs[0], outs[1]):
        assert _rel_err(a, c) < 2e-3


@pytest.mark.parametrize("geom,tail", [((4, 64, 128, 1, 1, 0, 16), False),
                                       ((4, 64, 64, 3, 1, 1, 16), False),
                                       ((4, 256, 64, 1, 1, 0, 16), True)])
def test_dgrad_bn_stats_epilogue(nnl, geom, tail):
    """nnl_conv2d_bwd_data_bn against nnl_conv2d_bwd_data + the BN-backward
    statistics computed here: identical gated gradient bits, column sums of
    (gy, gy*xhat) within f32 summation-order noise."""
    import torch
    from paper_2102_06725_b200 import _lib
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(5)
    dev = torch.device("cuda")
    h16 = lambda a: torch.from_numpy(O.q16(a.astype(np.float32))).to(dev).half()
    dy = h16(rng.uniform(-1, 1, (b, hw, hw, cout)))
    w = h16(rng.uniform(-0.1, 0.1, (cout, k, k, cin)))
    x = h16(rng.uniform(-2, 2, (b, hw, hw, cin)))
    gate = h16(rng.uniform(-1, 1, (b, hw, hw, cin)))
    prev = h16(rng.uniform(-1, 1, (b, hw, hw, cin)))
    mean = torch.from_numpy(rng.uniform(-0.2, 0.2, cin).astype(np.float32)).to(dev)
    istd = torch.from_numpy(rng.uniform(0.5, 1.5, cin).astype(np.float32)).to(dev)
    gam = torch.from_numpy(rng.uniform(0.5, 1.5, cin).astype(np.float32)).to(dev)
    bet = torch.from_numpy(rng.uniform(-0.5, 0.5, cin).astype(np.float32)).to(dev)
    cs = _lib.ConvShape(b, hw, hw, cin, cout, k, k, s, s, p, p, hw, hw)
    L = _lib.lib()
    ws_n = L.nnl_conv2d_workspace_size(C.byref(cs), _lib.F16, 1)
    ws = torch.empty(ws_n, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ref = prev.clone() if tail else torch.empty_like(x)
    _lib.call("nnl_conv2d_bwd_data", C.byref(cs), _lib.F16, dy.data_ptr(), w.data_ptr(),
              ref.data_ptr(), 1 if tail else 0, ws.data_ptr(), ws_n, st)
    rows = L.nnl_conv2d_bwd_data_bn_rows(C.byref(cs), _lib.F16)
    assert rows > 0
    parts = torch.zeros(rows * 2 * cin, dtype=torch.float32, device=dev)
    dx = prev.clone() if tail else torch.empty_like(x)
    out = torch.empty_like(x) if tail else None
    bf = _lib.BnBwdFuse(x.data_ptr(), gate.data_ptr() if tail else None,
                        None if tail else gam.data_ptr(), None if tail else bet.data_ptr(),
                        mean.data_ptr(), istd.data_ptr(), 0 if tail else 1, 1 if tail else 0,
                        out.data_ptr() if tail else None, parts.data_ptr())
    _lib.call("nnl_conv2d_bwd_data_bn", C.byref(cs), _lib.F16, dy.data_ptr(), w.data_ptr(),
              dx.data_ptr(), 1 if tail else 0, C.byref(bf), ws.data_ptr(), ws_n, st)
    torch.cuda.synchronize()
    g = ref.float().cpu().numpy().reshape(-1, cin)
    xf = x.float().cpu().numpy().reshape(-1, cin)
    xh = (xf - mean.cpu().numpy()) * istd.cpu().numpy()
    if tail:
        gt = (gate.float().cpu().numpy().reshape(-1, cin) > 0).astype(np.float32)
    else:
        z = O.q16(gam.cpu().numpy() * xh + bet.cpu().numpy())
        gt = (z > 0).astype(np.float32)
    gy = g * gt
    got = (out if tail else dx).float().cpu().numpy().reshape(-1, cin)
    assert np.array_equal(got, O.q16(gy + 0.0 if tail else gy))
    sums = parts.cpu().numpy().reshape(rows, 2, cin).sum(0)
    want = np.stack([gy.sum(0, dtype=np.float64), (gy * xh).sum(0, dtype=np.float64)])
    np.testing.assert_allclose(sums, want, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("geom", [(4, 64, 64, 3, 1, 1, 56), (3, 64, 64, 3, 1, 1, 24),
                                  (8, 64, 64, 3, 1, 1, 16)])
def test_halo_tiles_match_per_tap_loads(nnl, geom):
    """3x3 convolutions over one shared input halo per tile (nine descriptor views
    into it) against per-tap operand loads: same (tap, K16) MMA order, outputs
    and input gradients agree to f32 accumulation rounding (the per-tap path may
    split K on small grids)."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(14)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (cout,)).astype(np.float32)
    outs = []
    for mode in (1, 0):
        prev = _lib.lib().nnl_set_tc_halo(mode)
        try:
            vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(s, s), pad=(p, p))
            y.forward()
            y.backward(1.0)
            outs.append([y.d, vs[0].g])
        finally:
            _lib.lib().nnl_set_tc_halo(prev)
    for a, c in zip(outs[0], outs[1]):
        assert _rel_err(a, c) < 2e-3


@pytest.mark.parametrize("geom", [(4, 64, 64, 3, 1, 1, 56), (2, 3, 64, 7, 2, 3, 64),
                                  (4, 64, 256, 1, 1, 0, 28), (3, 128, 128, 1, 1, 0, 20),
                                  (2, 256, 64, 1, 1, 0, 17)])
def test_interleaved_epilogue_matches_column_split(nnl, geom):
    """Tile-interleaved 8-warp epilogues (warp groups on alternate tiles, all
    columns each) against the column-split epilogue: identical output bits
    (bias with a -0 entry: q(0 + (acc + b)) == q(acc + (b + 0))), and BN
    statistics equal up to the association of the per-CTA f32 sums."""
    import torch
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(21)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (cout,)).astype(np.float32)
    bias[0] = -0.0
    shift = torch.from_numpy(rng.uniform(-0.2, 0.2, cout).astype(np.float32)).cuda()

    class _Bn:
        state = {"shift_ready": True, "shift": shift}
    outs = []
    for mode in (1, 0):
        prev = _lib.lib().nnl_set_tc_epi_il(mode)
        try:
            vs = [nnl.Variable(a.shape) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(s, s), pad=(p, p))
            node = y.parent
            node.state["emit_stats"] = True
            node.state["stat_bn"] = _Bn
            node.impl.forward(node, [v.data for v in vs], [y.data])
            y.data.mark_set()
            rows = node.state["stat_rows"]
            st = node.state["stats"].cpu().numpy()[: rows * 2 * cout]
            outs.append((y.d.copy(), st.reshape(rows, 2, cout).astype(np.float64).sum(0)))
        finally:
            _lib.lib().nnl_set_tc_epi_il(prev)
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=1e-5, atol=1e-4)
    ov = [O.Var(a, half=True) for a in (x, w, bias)]
    assert _rel_err(outs[0][0], O.conv2d(*ov, (s, s), (p, p), True).value) < 4e-3


@pytest.mark.parametrize("geom", [(8, 128, 128, 3, 2, 1, 56), (32, 256, 256, 3, 2, 1, 28),
                                  (16, 64, 128, 3, 2, 1, 32)])
def test_strided_dgrad_spatial_classes(nnl, geom):
    """Stride-2 3x3 dgrad parity classes over spatial tiles (one tiled 4D dy box
    per class tap, TMA-stored through the class's strided 4D view of dx) against
    the TMA-im2col class GEMMs with row-remapped stores: identical dx bits (same
    tap and channel-block order), and the oracle's input gradient."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib
    _half(nnl)
    b, cin, cout, k, s, p, hw = geom
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, (b, cin, hw, hw)).astype(np.float32)
    w = rng.uniform(-0.1, 0.1, (cout, cin, k, k)).astype(np.float32)
    bias = rng.uniform(-0.5, 0.5, (cout,)).astype(np.float32)
    outs = []
    for mode in (1, 0):
        prev = _lib.lib().nnl_set_tc_tile4(mode)
        try:
            vs = [nnl.Variable(a.shape, need_grad=True) for a in (x, w, bias)]
            for v, a in zip(vs, (x, w, bias)):
                v.d = a
            y = F.convolution(*vs, stride=(s, s), pad=(p, p))
            y.forward()
            y.backward(1.0)
            outs.append(vs[0].g.copy())
        finally:
            _lib.lib().nnl_set_tc_tile4(prev)
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    ov = [O.Var(a, half=True, need_grad=True) for a in (x, w, bias)]
    oy = O.conv2d(*ov, (s, s), (p, p), True)
    gxs = oy.parent.bwd([np.ones(oy.value.shape, np.float32)], [True, False, False])
    assert _rel_err(outs[0], O.q16(gxs[0])) < 4e-3
