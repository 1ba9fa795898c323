"""CPU checks of the C-ABI library: it loads, exports every symbol include/puv.h
declares, lays out atlases like the oracle, and rejects bad arguments before
touching the GPU (no compute calls here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import orc
from paper_2602_23040_b200 import puv
from synth.scenes import look_at

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "puv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(puv_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = puv.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert puv.version().startswith("libpuv sm_100a")


def test_struct_sizes_match_header():
    assert C.sizeof(puv.Camera) == 16 * 4 + 4 * 4 + 2 * 4 + 4 + 3 * 4
    assert C.sizeof(puv.Layout) == 5 * 4 + 16 * 5 * 4 + 4 + 3 * 4
    assert C.sizeof(puv.RenderOpts) == 16 + 8 + 2 * 4   # bg, flags, lpo_spec, lpo_pos_bits, lpo_attr_bits


@pytest.mark.parametrize("shapes", [[(64, 64)], [(512, 512), (256, 256), (128, 128)], [(1024, 1024), (1024, 512)],
                                    [(7, 5), (3, 9), (4, 4), (1, 1)]])
def test_layout_matches_oracle(shapes):
    lay = puv.layout_for_levels(shapes, 1)
    place, W, H = orc.layout_column(shapes)
    assert (lay.atlas_w, lay.atlas_h) == (W, H)
    for k in range(len(shapes)):
        assert (lay.level[k].x, lay.level[k].y, lay.level[k].rot90ccw) == tuple(place[k])
    assert lay.planes == 23


def _cams(n=2, W=64, H=48):
    return puv.cameras([look_at((3, 0, 1), (0, 0, 0), W, H, 60.0) for _ in range(n)])


def test_argument_validation_without_gpu():
    lay = puv.layout_for_levels([(16, 16)], 0)
    cams = _cams()
    sb, ah = puv.query_sizes(lay, cams, puv.opts())
    assert sb > 0 and ah > 0
    L = puv.lib()
    planes = (C.c_void_p * 14)(*([1] * 14))
    o = puv.opts()
    # state too small
    rc = L.puv_render_views(C.byref(lay), planes, None, 2, cams, C.byref(o), C.c_void_p(1), C.c_void_p(1), 16,
                            C.c_void_p(1), 16, None)
    assert rc == -6 and "state_bytes" in puv.last_error()
    # bad camera: fx <= 0
    bad = _cams()
    bad[1].fx = 0.0
    rc = L.puv_render_views(C.byref(lay), planes, None, 2, bad, C.byref(o), C.c_void_p(1), C.c_void_p(1), sb,
                            C.c_void_p(1), 16, None)
    assert rc == -5
    # non-orthonormal rotation
    bad = _cams()
    bad[0].viewmat[0] = 2.0
    rc = L.puv_render_views(C.byref(lay), planes, None, 2, bad, C.byref(o), C.c_void_p(1), C.c_void_p(1), sb,
                            C.c_void_p(1), 16, None)
    assert rc == -5 and "orthonormal" in puv.last_error()
    # mixed image sizes
    mixed = puv.cameras([look_at((3, 0, 1), (0, 0, 0), 64, 48, 60.0), look_at((3, 0, 1), (0, 0, 0), 32, 48, 60.0)])
    rc = L.puv_render_views(C.byref(lay), planes, None, 2, mixed, C.byref(o), C.c_void_p(1), C.c_void_p(1), sb,
                            C.c_void_p(1), 16, None)
    assert rc == -4
    # NULL plane
    planes0 = (C.c_void_p * 14)(*([1] * 13 + [0]))
    rc = L.puv_render_views(C.byref(lay), planes0, None, 2, cams, C.byref(o), C.c_void_p(1), C.c_void_p(1), sb,
                            C.c_void_p(1), 16, None)
    assert rc == -1
    # bad layout: D mismatch, overlap, overflow
    lay2 = puv.layout_for_levels([(16, 16), (8, 8)], 0)
    lay2.planes = 15
    assert L.puv_query_sizes(C.byref(lay2), 2, cams, None, C.byref(C.c_size_t()), C.byref(C.c_size_t())) == -4
    lay3 = puv.layout_for_levels([(16, 16), (8, 8)], 0)
    lay3.level[1].x = 4
    assert L.puv_query_sizes(C.byref(lay3), 2, cams, None, C.byref(C.c_size_t()), C.byref(C.c_size_t())) == -3
    lay4 = puv.layout_for_levels([(16, 16)], 0)
    lay4.level[0].x = 1
    assert L.puv_query_sizes(C.byref(lay4), 2, cams, None, C.byref(C.c_size_t()), C.byref(C.c_size_t())) == -3
    # layout_for_levels errors
    with pytest.raises(puv.PuvError):
        puv.layout_for_levels([(0, 4)], 0)
    with pytest.raises(puv.PuvError):
        puv.layout_for_levels([(4, 4)] * 17, 0)
    with pytest.raises(puv.PuvError):
        puv.layout_for_levels([(4, 4)], 4)


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The product package never imports the oracle; the binding fails loudly without libpuv.so."""
    pkg = os.path.join(ROOT, "paper_2602_23040_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracle's", "").lower() or f.endswith((".cu", ".cuh")), f
                assert "import oracle" not in src and "from oracle" not in src, f


@pytest.mark.parametrize("S,K", [(1024, 8), (64, 8), (32, 5), (16, 3), (16, 2), (16, 1)])
def test_paper_layout_matches_oracle(S, K):
    """puv_layout_paper (recursive right/below rule) vs the oracle's scaled SPEC.md:257 table."""
    lay = puv.layout_paper(S, K, 3)
    rows, cols, place, W, H = orc.layout_paper(S, K)
    assert (lay.atlas_w, lay.atlas_h) == (W, H)
    for k in range(K):
        a = lay.level[k]
        assert (a.rows, a.cols, a.x, a.y, a.rot90ccw) == (rows[k], cols[k], *place[k])
    assert lay.position_mode == puv.POS_XYZ and lay.planes == 59


def test_rho_layout_validation():
    lay = puv.with_rho(puv.layout_for_levels([(16, 16)], 0), (0.0, 0.0, 1.0))
    assert lay.position_mode == puv.POS_RHO and list(lay.center) == [0.0, 0.0, 1.0]
    bad = puv.with_rho(lay, (0, 0, 0))
    bad.position_mode = 7
    cams = _cams()
    assert puv.lib().puv_query_sizes(C.byref(bad), 2, cams, None, C.byref(C.c_size_t()), C.byref(C.c_size_t())) == -2
    # rho mode: plane entries 1, 2 may be NULL but the 3 ray planes (D..D+2) must be given
    sb, _ = puv.query_sizes(lay, cams, puv.opts())
    o = puv.opts()
    tab = (C.c_void_p * 17)(*([1, 0, 0] + [1] * 11 + [1, 1, 0]))
    rc = puv.lib().puv_render_views(C.byref(lay), tab, None, 2, cams, C.byref(o), C.c_void_p(1), C.c_void_p(1), sb,
                                    C.c_void_p(1), 16, None)
    assert rc == -1 and "plane 16" in puv.last_error()


def test_train_step_argument_validation_without_gpu():
    """puv_train_step / puv_train_step_host reject bad arguments before enqueueing anything (the
    uploads of the host-buffer call included): no GPU is touched here."""
    lay = puv.layout_for_levels([(16, 16)], 0)
    cams = _cams(3)
    L = puv.lib()
    o = puv.opts()
    sb, _ = puv.query_sizes(lay, puv.cameras([look_at((3, 0, 1), (0, 0, 0), 64, 48, 60.0)] * 2), o)
    planes = (C.c_void_p * 14)(*([1] * 14))
    grads = (C.c_void_p * 14)(*([1] * 14))

    def bufs(state_bytes=sb, flags=1):
        b = puv.StepBuffers()
        b.images = b.dL_dimages = b.loss = b.state = b.arena = 1
        b.overflow = b.arena_need = flags
        b.state_bytes, b.arena_bytes = state_bytes, 16
        return b

    # views_per_call 2 over 3 views: the state is sized for a 2-view chunk -> accepted by validation;
    # a 1-view state is too small
    rc = L.puv_train_step(C.byref(lay), planes, None, 3, cams, C.byref(o), C.c_void_p(1), None, 2,
                          C.byref(bufs(16)), grads, None)
    assert rc == -6
    rc = L.puv_train_step(C.byref(lay), planes, None, 3, cams, C.byref(o), C.c_void_p(1), None, 2,
                          C.byref(bufs(flags=0)), grads, None)
    assert rc == -1 and "overflow" in puv.last_error()
    bad_grads = (C.c_void_p * 14)(*([1] * 13 + [0]))
    rc = L.puv_train_step(C.byref(lay), planes, None, 3, cams, C.byref(o), C.c_void_p(1), None, 2,
                          C.byref(bufs()), bad_grads, None)
    assert rc == -1 and "grad plane 13" in puv.last_error()
    bad = _cams(3)
    bad[2].fx = -1.0    # a camera outside the first chunk is checked too
    rc = L.puv_train_step(C.byref(lay), planes, None, 3, bad, C.byref(o), C.c_void_p(1), None, 2,
                          C.byref(bufs()), grads, None)
    assert rc == -5
    up = (puv.Copy * 1)(puv.Copy(1, 1, 64))
    rc = L.puv_train_step_host(C.byref(lay), planes, None, 3, cams, C.byref(o), up, 1, C.c_void_p(1), C.c_void_p(1),
                               None, 2, C.byref(bufs(16)), grads, None, 0, None)
    assert rc == -6
    up0 = (puv.Copy * 1)(puv.Copy(0, 1, 64))
    rc = L.puv_train_step_host(C.byref(lay), planes, None, 3, cams, C.byref(o), up0, 1, C.c_void_p(1), C.c_void_p(1),
                               None, 2, C.byref(bufs()), grads, None, 0, None)
    assert rc == -1 and "upload 0" in puv.last_error()
