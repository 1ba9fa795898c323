"""ctypes wrapper of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` arms may import this module.  It shares nothing with the
CUDA path (paper_2602_23040_b200/); both consume scenes from synth/.

Functions mirror oracle/puv_oracle.c; see that file's header for the
passages of PAPER.md each follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

TILE = 16


class OrcCamera(C.Structure):
    _fields_ = [("viewmat", C.c_float * 16), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("near_plane", C.c_float), ("campos", C.c_float * 3)]


class OrcProj(C.Structure):
    _fields_ = [("visible", C.c_int32), ("depth_bits", C.c_uint32), ("x0", C.c_int32), ("x1", C.c_int32),
                ("y0", C.c_int32), ("y1", C.c_int32), ("tiles", C.c_uint32),
                ("mx", C.c_float), ("my", C.c_float), ("ha", C.c_float), ("nb", C.c_float), ("hc", C.c_float),
                ("o", C.c_float), ("t_g", C.c_float), ("clamp_x", C.c_int32), ("clamp_y", C.c_int32)]


PROJ_DTYPE = np.dtype([("visible", "<i4"), ("depth_bits", "<u4"), ("x0", "<i4"), ("x1", "<i4"),
                       ("y0", "<i4"), ("y1", "<i4"), ("tiles", "<u4"), ("mx", "<f4"), ("my", "<f4"),
                       ("ha", "<f4"), ("nb", "<f4"), ("hc", "<f4"), ("o", "<f4"), ("t_g", "<f4"),
                       ("clamp_x", "<i4"), ("clamp_y", "<i4")])
assert PROJ_DTYPE.itemsize == C.sizeof(OrcProj)


def build():
    src = os.path.join(_HERE, "puv_oracle.c")
    so = os.path.join(_HERE, "liborc.so")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return so


def lib():
    global _LIB
    if _LIB is None:
        L = C.CDLL(build())
        P = C.c_void_p
        L.orc_set_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_exp_c.restype = C.c_float
        L.orc_exp_c.argtypes = [C.c_float]
        L.orc_log_c.restype = C.c_float
        L.orc_log_c.argtypes = [C.c_float]
        L.orc_exp_c_array.argtypes = [P, P, C.c_int64]
        L.orc_log_c_array.argtypes = [P, P, C.c_int64]
        L.orc_sh_basis.argtypes = [C.c_int, P, C.c_int64, P]
        L.orc_project.argtypes = [P, C.c_int64, P, P, P]
        L.orc_bin_count.restype = C.c_int64
        L.orc_bin_count.argtypes = [C.c_int64, P]
        L.orc_bin.argtypes = [C.c_int64, P, C.c_int, C.c_int, P, P, P]
        L.orc_forward.argtypes = [P, P, C.c_int, C.c_int64, P, P, P, P, P, P, P]
        L.orc_backward.argtypes = [P, P, C.c_int, C.c_int64, P, P, P, P, P, P]
        L.orc_layout_column.argtypes = [C.c_int, P, P, P, P, P]
        L.orc_label_dynamic.argtypes = [P, C.c_int64, P, C.c_int, P, P, C.c_int, P, C.c_int64, P]
        L.orc_layout_paper.argtypes = [C.c_int, C.c_int, P, P, P, P, P]
        L.orc_ray_dirs.argtypes = [C.c_int, P, P, P, C.c_int32, C.c_int32, P, P, P]
        L.orc_positions_from_rho.argtypes = [P, P, P, P, P, C.c_int64, P, P, P]
        L.orc_rho_grad.argtypes = [P, P, P, P, P, P, C.c_int64, P]
        L.orc_quant_code.restype = C.c_uint32
        L.orc_quant_code.argtypes = [C.c_float, C.c_float, C.c_float, C.c_int]
        L.orc_dequant.restype = C.c_float
        L.orc_dequant.argtypes = [C.c_uint32, C.c_float, C.c_float, C.c_int]
        L.orc_quant_fit.argtypes = [C.c_int, P, P, C.c_int64, P]
        L.orc_quantize_plane.argtypes = [P, P, C.c_int64, C.c_float, C.c_float, C.c_int, P, P]
        L.orc_fp16_bits.restype = C.c_uint32
        L.orc_fp16_bits.argtypes = [C.c_float]
        L.orc_fp16_value.restype = C.c_float
        L.orc_fp16_value.argtypes = [C.c_uint32]
        L.orc_quantize_plane_fp16.argtypes = [P, P, C.c_int64, P, P]
        L.orc_pack.argtypes = [C.c_int, P, P, P, C.c_int, P, P, C.c_int32, C.c_int32, P, P]
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _ptr_table(arrs, ctype=C.c_void_p):
    tab = (ctype * len(arrs))(*[a.ctypes.data for a in arrs])
    return tab


def camera(cam) -> OrcCamera:
    c = OrcCamera()
    c.viewmat[:] = [float(v) for v in np.asarray(cam.viewmat, np.float32).reshape(-1)]
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.width, c.height = cam.width, cam.height
    c.near_plane = cam.near
    c.campos[:] = [float(v) for v in np.asarray(cam.campos, np.float32)]
    return c


# ----------------------------------------------------------------------------
# contract functions

def exp_c(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().orc_exp_c_array(_ptr(x), _ptr(y), x.size)
    return y


def log_c(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().orc_log_c_array(_ptr(x), _ptr(y), x.size)
    return y


def sh_basis(deg, dirs):
    dirs = np.ascontiguousarray(dirs, np.float64)
    n = dirs.shape[0]
    Y = np.empty((n, (deg + 1) ** 2), np.float64)
    lib().orc_sh_basis(deg, _ptr(dirs), n, _ptr(Y))
    return Y


# ----------------------------------------------------------------------------
# atlas

def layout_column(shapes):
    K = len(shapes)
    rows = np.array([s[0] for s in shapes], np.int32)
    cols = np.array([s[1] for s in shapes], np.int32)
    place = np.zeros((K, 3), np.int32)
    W = C.c_int32()
    H = C.c_int32()
    rc = lib().orc_layout_column(K, _ptr(rows), _ptr(cols), _ptr(place), C.byref(W), C.byref(H))
    assert rc == 0
    return place, W.value, H.value


def layout_paper(S, K):
    """(rows, cols, place (K,3), W, H) of the paper's K-level pyramid atlas."""
    rows = np.zeros(K, np.int32)
    cols = np.zeros(K, np.int32)
    place = np.zeros((K, 3), np.int32)
    W = C.c_int32()
    H = C.c_int32()
    rc = lib().orc_layout_paper(S, K, _ptr(rows), _ptr(cols), _ptr(place), C.byref(W), C.byref(H))
    assert rc == 0
    return rows, cols, place, W.value, H.value


def ray_dirs(rows, cols, place, W, H):
    """(3, H, W) fp32 ray direction of every atlas texel (0 where unplaced)."""
    out = np.zeros((3, H, W), np.float32)
    r = np.ascontiguousarray(rows, np.int32)
    c = np.ascontiguousarray(cols, np.int32)
    p = np.ascontiguousarray(place, np.int32)
    lib().orc_ray_dirs(len(r), _ptr(r), _ptr(c), _ptr(p), W, H, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]))
    return out


def positions_from_rho(rho, rays, center):
    """mu = c (+) rho (x) ray in fp32.  rho (H, W); rays (3, H, W) -> (3, H, W)."""
    rho = np.ascontiguousarray(rho, np.float32)
    rays = np.ascontiguousarray(rays, np.float32)
    c = np.asarray(center, np.float32)
    out = np.empty((3,) + rho.shape, np.float32)
    lib().orc_positions_from_rho(_ptr(rho), _ptr(rays[0]), _ptr(rays[1]), _ptr(rays[2]), _ptr(c), rho.size,
                                 _ptr(out[0]), _ptr(out[1]), _ptr(out[2]))
    return out


def rho_grad(rays, gxyz):
    """d rho = ray . d mu (fp64)."""
    rays = np.ascontiguousarray(rays, np.float32)
    g = np.ascontiguousarray(gxyz, np.float64)
    out = np.empty(rays.shape[1:], np.float64)
    lib().orc_rho_grad(_ptr(rays[0]), _ptr(rays[1]), _ptr(rays[2]), _ptr(g[0]), _ptr(g[1]), _ptr(g[2]),
                       out.size, _ptr(out))
    return out


def quant_code(x, mn, mx, bits):
    """LPO fake-quantiser code of one value (DESIGN.md §13 Q1-Q3)."""
    return int(lib().orc_quant_code(x, mn, mx, bits))


def dequant(code, mn, mx, bits):
    return float(lib().orc_dequant(code, mn, mx, bits))


def quant_fit(planes, occ, skip=()):
    """(D, 2) fp32 per-plane (min, max) over occupied texels; planes in `skip` -> (0, 0)."""
    planes = np.ascontiguousarray(planes, np.float32)
    D = planes.shape[0]
    tab = (C.c_void_p * D)(*[None if d in skip else planes[d].ctypes.data for d in range(D)])
    o = np.ascontiguousarray(occ, np.uint8) if occ is not None else None
    spec = np.empty((D, 2), np.float32)
    lib().orc_quant_fit(D, tab, None if o is None else _ptr(o), planes[0].size, _ptr(spec))
    return spec


FP16 = "fp16"   # bits value of a plane stored as IEEE binary16 (reading Q8)


def fp16_bits(x):
    """binary16 bit patterns (uint32) of fp32 values, round to nearest even (reading Q8)."""
    x = np.ascontiguousarray(x, np.float32)
    code = np.zeros(x.shape, np.uint32)
    proxy = np.zeros(x.shape, np.float32)
    lib().orc_quantize_plane_fp16(_ptr(x), None, x.size, _ptr(code), _ptr(proxy))
    return code, proxy


def quantize(planes, occ, spec, bits):
    """Per plane d with bits[d] > 0: codes (uint32) and the fp32 proxy; bits[d] == FP16: the binary16
    pattern and value; planes with bits 0 are copied through unchanged with code 0 (the unused
    planes 1, 2 of rho mode)."""
    planes = np.ascontiguousarray(planes, np.float32)
    o = np.ascontiguousarray(occ, np.uint8) if occ is not None else None
    codes = np.zeros(planes.shape, np.uint32)
    proxy = planes.copy()
    for d in range(planes.shape[0]):
        if bits[d] == 0:
            continue
        if bits[d] == FP16:
            lib().orc_quantize_plane_fp16(_ptr(planes[d]), None if o is None else _ptr(o), planes[d].size,
                                          _ptr(codes[d]), _ptr(proxy[d]))
            continue
        lib().orc_quantize_plane(_ptr(planes[d]), None if o is None else _ptr(o), planes[d].size,
                                 float(spec[d, 0]), float(spec[d, 1]), int(bits[d]), _ptr(codes[d]), _ptr(proxy[d]))
    return codes, proxy


def pack(levels, place=None, W=None, H=None):
    """levels: list of synth.scenes.Level.  Returns (planes (D,H,W) f32, occ (H,W) u8, place)."""
    shapes = [(lv.rows, lv.cols) for lv in levels]
    if place is None:
        place, W, H = layout_column(shapes)
    place = np.ascontiguousarray(place, np.int32)
    K = len(levels)
    D = levels[0].planes.shape[0]
    rows = np.array([s[0] for s in shapes], np.int32)
    cols = np.array([s[1] for s in shapes], np.int32)
    lp = [np.ascontiguousarray(lv.planes[d]) for lv in levels for d in range(D)]
    lo = [np.ascontiguousarray(lv.occ) for lv in levels]
    planes = np.empty((D, H, W), np.float32)
    occ = np.empty((H, W), np.uint8)
    ap = [planes[d] for d in range(D)]
    rc = lib().orc_pack(K, _ptr(rows), _ptr(cols), _ptr(place), D, _ptr_table(lp), _ptr_table(lo),
                        W, H, _ptr_table(ap), _ptr(occ))
    if rc != 0:
        raise ValueError(f"orc_pack failed: {rc}")
    return planes, occ, place


def pack_labels(levels, place, W, H):
    """Dynamic labels packed like the occupancy plane (mask for gradient freezing)."""
    out = np.zeros((H, W), np.uint8)
    for lv, (x, y, rot) in zip(levels, place):
        assert rot == 0
        out[y:y + lv.rows, x:x + lv.cols] = lv.labels
    return out


# ----------------------------------------------------------------------------
# projection / binning / render

def set_threads(n: int = 0) -> int:
    """OpenMP threads of the following oracle calls (n < 1: all host cores); returns the count."""
    return int(lib().orc_set_threads(int(n)))


def project(planes, occ, cam):
    D, H, W = planes.shape
    n = H * W
    pl = [np.ascontiguousarray(planes[d].reshape(-1)) for d in range(D)]
    out = np.zeros(n, PROJ_DTYPE)
    c = camera(cam)
    occ_p = _ptr(np.ascontiguousarray(occ.reshape(-1))) if occ is not None else None
    lib().orc_project(_ptr_table(pl), n, occ_p, C.byref(c), _ptr(out))
    return out


def binning(proj, cam):
    """Per-tile ranges [start, end) and concatenated gid lists, sorted by (depth_bits, gid)."""
    gx = (cam.width + TILE - 1) // TILE
    gy = (cam.height + TILE - 1) // TILE
    n = proj.shape[0]
    K = lib().orc_bin_count(n, _ptr(proj))
    start = np.zeros(gx * gy, np.uint32)
    end = np.zeros(gx * gy, np.uint32)
    gids = np.zeros(max(K, 1), np.uint32)
    rc = lib().orc_bin(n, _ptr(proj), gx, gy, _ptr(start), _ptr(end), _ptr(gids))
    assert rc == 0
    return start, end, gids[:K]


def _val_planes(planes, val):
    D = planes.shape[0]
    if val is None:
        val = planes.astype(np.float64)
    dec = [np.ascontiguousarray(planes[d].reshape(-1), np.float32) for d in range(D)]
    vl = [np.ascontiguousarray(val[d].reshape(-1), np.float64) for d in range(D)]
    return dec, vl


def forward(planes, occ, sh_degree, cam, bg=(0.0, 0.0, 0.0), val=None):
    """Returns (image (3,H,W) f64, T_final f32 (H,W), n_contrib i32 (H,W), stats dict).

    `planes` (fp32) take every decision; `val` (fp64, default = planes) gives
    the values — pass a perturbed `val` for finite differences.
    """
    D, HA, WA = planes.shape
    n = HA * WA
    dec, vl = _val_planes(planes, val)
    c = camera(cam)
    img = np.zeros((3, cam.height, cam.width), np.float64)
    T = np.zeros((cam.height, cam.width), np.float32)
    nc = np.zeros((cam.height, cam.width), np.int32)
    stats = np.zeros(3, np.int64)
    bgv = np.asarray(bg, np.float64)
    occ_p = _ptr(np.ascontiguousarray(occ.reshape(-1))) if occ is not None else None
    rc = lib().orc_forward(_ptr_table(dec), _ptr_table(vl), sh_degree, n, occ_p, C.byref(c),
                           _ptr(bgv), _ptr(img), _ptr(T), _ptr(nc), _ptr(stats))
    assert rc == 0
    return img, T, nc, {"n_vis": int(stats[0]), "K": int(stats[1]), "composited": int(stats[2])}


def backward(planes, occ, sh_degree, cam, dL_dimage, mask=None, bg=(0.0, 0.0, 0.0), val=None, grad=None):
    """Returns grad (D, H_A, W_A) f64 of L w.r.t. the texel planes (accumulated into `grad`)."""
    D, HA, WA = planes.shape
    n = HA * WA
    dec, vl = _val_planes(planes, val)
    c = camera(cam)
    if grad is None:
        grad = np.zeros((D, HA, WA), np.float64)
    gl = [grad[d].reshape(-1) for d in range(D)]
    for g in gl:
        assert g.flags.c_contiguous
    dl = np.ascontiguousarray(dL_dimage, np.float64)
    bgv = np.asarray(bg, np.float64)
    occ_p = _ptr(np.ascontiguousarray(occ.reshape(-1))) if occ is not None else None
    mask_p = _ptr(np.ascontiguousarray(mask.reshape(-1), np.uint8)) if mask is not None else None
    rc = lib().orc_backward(_ptr_table(dec), _ptr_table(vl), sh_degree, n, occ_p, C.byref(c),
                            _ptr(bgv), _ptr(dl), mask_p, _ptr_table(gl))
    assert rc == 0
    return grad


def label_dynamic(planes, occ, cams, masks, r_max=64, gids=None):
    """Supp. Alg. 1: D_i = OR_c [exists pixel p, |p-m|_inf <= r, d^2 <= 9, M_c(p)].
    masks: (n_cams, H, W) uint8.  gids: optional texel ids to label (others returned as 0)."""
    D, HA, WA = planes.shape
    n = HA * WA
    pl = [np.ascontiguousarray(planes[d].reshape(-1)) for d in range(D)]
    arr = (OrcCamera * len(cams))(*[camera(c) for c in cams])
    m = np.ascontiguousarray(masks, np.uint8)
    assert m.shape == (len(cams), cams[0].height, cams[0].width)
    labels = np.zeros(n, np.uint8)
    occ_p = _ptr(np.ascontiguousarray(occ.reshape(-1))) if occ is not None else None
    if gids is not None:
        g = np.ascontiguousarray(gids, np.int64)
        rc = lib().orc_label_dynamic(_ptr_table(pl), n, occ_p, len(cams), arr, _ptr(m), r_max, _ptr(g), g.size,
                                     _ptr(labels))
    else:
        rc = lib().orc_label_dynamic(_ptr_table(pl), n, occ_p, len(cams), arr, _ptr(m), r_max, None, 0,
                                     _ptr(labels))
    assert rc == 0
    return labels.reshape(HA, WA)


def l2_loss_grad(image, target):
    """L = 1/2 sum (I_hat - I)^2 (R11); dL/dI_hat = I_hat - I."""
    d = np.asarray(image, np.float64) - np.asarray(target, np.float64)
    return 0.5 * float(np.sum(d * d)), d
