"""GPU parity of LPO (NEXT-2): range fit, fake quantiser (codes + proxy) bit-exact
against the oracle; the proxy render forward / backward (STE: the proxy's gradient is the master's)
with the usual bars: bit-exact binning and pixel state, images within 1e-4, gradients within
max(1e-3 |g|, 1e-6)."""
import numpy as np
import pytest
import torch

from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import make_scene, ring, rho_scene
from tests.gpu_common import describe_violations, grad_violations

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint32)


def _quant_check(layout, planes, occ, pos_bits=16, attr_bits=8, rho=False):
    dev = torch.device("cuda")
    P = torch.from_numpy(planes).to(dev)
    O = torch.from_numpy(occ).to(dev)
    spec = puv.quant_fit(layout, P, O)
    proxy, codes = puv.quantize(layout, P, O, spec, pos_bits, attr_bits, codes=True)
    torch.cuda.synchronize()
    skip = (1, 2) if rho else ()
    spec_ref = orc.quant_fit(planes, occ, skip=skip)
    assert np.array_equal(spec.cpu().numpy(), spec_ref)      # by value (+0 / -0 compare equal)
    pb = orc.FP16 if pos_bits == "fp16" else pos_bits
    bits = [0 if d in skip else (pb if d < 3 else attr_bits) for d in range(planes.shape[0])]
    codes_ref, proxy_ref = orc.quantize(planes, occ, spec_ref, bits)
    px = proxy.cpu().numpy()
    for d in range(planes.shape[0]):
        if d in skip:
            continue
        assert np.array_equal(_bits(px[d]), _bits(proxy_ref[d])), f"proxy plane {d}"
        c = codes[d].cpu()
        c = (c.view(torch.int16).numpy().astype(np.int64) & 0xFFFF) if c.dtype == torch.uint16 else c.numpy()
        assert np.array_equal(c.astype(np.uint32), codes_ref[d]), f"codes plane {d}"
    # requantising the proxy with the same range returns the same codes
    proxy2, codes2 = puv.quantize(layout, proxy, O, spec, pos_bits, attr_bits, codes=True)
    for d in range(planes.shape[0]):
        if d not in skip:
            assert torch.equal(codes2[d], codes[d]) and torch.equal(proxy2[d], proxy[d])
    return spec, proxy, proxy_ref


@pytest.mark.parametrize("pos_bits,attr_bits", [(16, 8), (12, 5), (8, 8), (16, 1), ("fp16", 8)])
def test_quantize_c2_bitexact(pos_bits, attr_bits):
    sc = make_scene(2)
    planes, occ, _ = orc.pack(sc.levels)
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    occ = occ.copy()
    occ[::7, ::5] = 0                           # holes: unoccupied texels excluded from the range
    _quant_check(layout, planes, occ, pos_bits, attr_bits)


def test_quantize_rho_paper_atlas_bitexact():
    rows, cols, place, W, H = orc.layout_paper(64, 8)
    sc = rho_scene(71, list(zip(rows.tolist(), cols.tolist())), 1, [])
    planes, occ, _ = orc.pack(sc.levels, place=place, W=W, H=H)
    lay = puv.with_rho(puv.layout_paper(64, 8, 1), (0.0, 0.0, 0.0))
    _quant_check(lay, planes, occ, rho=True)


def test_quantize_degenerate_and_empty():
    dev = torch.device("cuda")
    layout = puv.layout_for_levels([(9, 13)], 0)
    planes = np.random.default_rng(1).normal(size=(14, 9, 13)).astype(np.float32)
    planes[5] = 0.75                                   # constant plane: code 0, proxy = min
    occ = np.ones((9, 13), np.uint8)
    _, proxy, _ = _quant_check(layout, planes, occ)
    assert torch.all(proxy[5] == 0.75)
    spec = puv.quant_fit(layout, torch.from_numpy(planes).to(dev), torch.zeros((9, 13), dtype=torch.uint8,
                                                                              device=dev))
    assert spec.abs().max().item() == 0.0


@pytest.mark.parametrize("pos_bits", [16, "fp16"])
def test_lpo_render_forward_backward_c2(pos_bits):
    """C2, two views: render the GPU proxy; oracle renders its own (bit-identical) proxy; the backward
    (STE) gradient lands on the master planes and matches the oracle's backward of the proxy.
    pos_bits "fp16": positions stored as IEEE binary16 (reading Q8)."""
    sc = make_scene(2)
    views = [0, 9]
    dev = torch.device("cuda")
    planes, occ, _ = orc.pack(sc.levels)
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    spec, proxy, proxy_ref = _quant_check(layout, planes, occ, pos_bits=pos_bits)
    cams = puv.cameras([sc.cameras[v] for v in views])
    R = puv.Renderer(layout, cams, device=dev)
    O = torch.from_numpy(occ).to(dev)
    img = R.forward(proxy, O).cpu().numpy()
    dls = []
    for vi, v in enumerate(views):
        cam = sc.cameras[v]
        dbg = puv.debug_tensors(layout, cams, R.state, R.arena, vi)
        P = orc.project(proxy_ref, occ, cam)
        start, end, gids = orc.binning(P, cam)
        assert np.array_equal(dbg["keys_gid"].cpu().numpy().view(np.uint32), gids)
        ref, T, nc, _ = orc.forward(proxy_ref, occ, sc.sh_degree, cam)
        assert np.array_equal(_bits(dbg["t_final"].cpu().numpy()), _bits(T))
        assert np.array_equal(dbg["n_contrib"].cpu().numpy(), nc)
        assert np.abs(img[vi] - ref).max() <= 1e-4
        dls.append(orc.l2_loss_grad(ref, sc.target(v))[1].astype(np.float32).astype(np.float64))
    master_grad = torch.zeros((layout.planes,) + occ.shape, dtype=torch.float32, device=dev)
    R.backward(proxy, O, torch.from_numpy(np.stack(dls).astype(np.float32)).to(dev), grad=master_grad)
    torch.cuda.synchronize()
    g_ref = np.zeros(planes.shape, np.float64)
    for v, dl in zip(views, dls):
        orc.backward(proxy_ref, occ, sc.sh_degree, sc.cameras[v], dl, grad=g_ref)
    g = master_grad.cpu().numpy()
    bad = grad_violations(g, g_ref)
    assert not bad.any(), describe_violations(g, g_ref, bad)
    # the proxy render differs from the master render (quantisation is not a no-op)
    img_master = puv.Renderer(layout, cams, device=dev).forward(torch.from_numpy(planes).to(dev), O).cpu().numpy()
    assert np.abs(img_master - img).max() > 1e-4


@pytest.mark.slow
def test_lpo_c3_full_size_quantize_and_view0():
    sc = make_scene(3)
    dev = torch.device("cuda")
    planes, occ, _ = orc.pack(sc.levels)
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    spec, proxy, proxy_ref = _quant_check(layout, planes, occ)
    cams = puv.cameras(sc.cameras)
    R = puv.Renderer(layout, cams, device=dev)
    img = R.forward(proxy, torch.from_numpy(occ).to(dev))
    ref, T, nc, _ = orc.forward(proxy_ref, occ, sc.sh_degree, sc.cameras[0])
    dbg = puv.debug_tensors(layout, cams, R.state, R.arena, 0)
    assert np.array_equal(_bits(dbg["t_final"].cpu().numpy()), _bits(T))
    assert np.array_equal(dbg["n_contrib"].cpu().numpy(), nc)
    assert np.abs(img[0].cpu().numpy() - ref).max() <= 1e-4


@pytest.mark.parametrize("pos_bits", [16, "fp16"])
def test_fused_lpo_render_equals_proxy_render(pos_bits):
    """PUV_RENDER_LPO (NEXT-2 fused into K1/K7): rendering the MASTER planes with the quantiser applied
    as they are read equals rendering the materialised proxy atlas -- images, T_final, n_contrib and
    the tile lists bit for bit -- and its backward (the STE master gradient) equals the proxy
    render's backward up to fp64 atomic order.  C2, views 0 and 9, holes in the atlas."""
    sc = make_scene(2)
    views = [0, 9]
    dev = torch.device("cuda")
    planes, occ, _ = orc.pack(sc.levels)
    occ = occ.copy()
    occ[::7, ::5] = 0
    layout = puv.layout_for_levels([(lv.rows, lv.cols) for lv in sc.levels], sc.sh_degree)
    P = torch.from_numpy(planes).to(dev)
    O = torch.from_numpy(occ).to(dev)
    spec = puv.quant_fit(layout, P, O)
    proxy, _ = puv.quantize(layout, P, O, spec, pos_bits, 8)
    cams = puv.cameras([sc.cameras[v] for v in views])
    Rp = puv.Renderer(layout, cams, device=dev)
    img_p = Rp.forward(proxy, O)
    Rf = puv.Renderer(layout, cams, device=dev, lpo=(spec, pos_bits, 8))
    img_f = Rf.forward(P, O)
    torch.cuda.synchronize()
    assert torch.equal(img_p, img_f)
    for vi in range(len(views)):
        a = puv.debug_tensors(layout, cams, Rp.state, Rp.arena, vi)
        b = puv.debug_tensors(layout, cams, Rf.state, Rf.arena, vi)
        for k in ("t_final", "n_contrib", "keys_gid", "tile_start", "depth_key"):
            assert torch.equal(a[k], b[k]), k
    dL = torch.from_numpy(np.stack([sc.target(v) for v in views])).to(dev) - img_p
    g_p = Rp.backward(proxy, O, dL.contiguous())
    g_f = Rf.backward(P, O, dL.contiguous())
    torch.cuda.synchronize()
    a, b = g_p.cpu().numpy().astype(np.float64), g_f.cpu().numpy().astype(np.float64)
    assert np.abs(a).max() > 0
    assert np.all(np.abs(a - b) <= 1e-6 * np.abs(a) + 1e-12)
