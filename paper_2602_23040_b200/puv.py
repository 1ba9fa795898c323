"""Thin ctypes binding of libpuv (include/puv.h).  Argument marshalling only.

Every step of the render runs in the CUDA kernels of `csrc/`; this module
turns torch tensors into raw device pointers and the current CUDA stream into
a `cudaStream_t`.  There is no CPU fallback: if `libpuv.so` is missing the
import fails loudly (`RuntimeError`).

Functions keep the C names without the `puv_` prefix: layout_for_levels,
pack_atlas, unpack_levels, query_sizes, render_views, l2_loss_grad,
render_backward, check_overflow, debug_view, last_error.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# PUV_LIB: an alternative build of the same library (A/B timing of kernel variants, tools/ab_raster.py)
LIB_PATH = os.environ.get("PUV_LIB") or os.path.join(_HERE, "libpuv.so")
MAX_LEVELS = 16

_status = {0: "PUV_OK", -1: "PUV_E_INVALID_ARGUMENT", -2: "PUV_E_INVALID_CONFIG", -3: "PUV_E_LAYOUT_OVERFLOW",
           -4: "PUV_E_DIMENSION_MISMATCH", -5: "PUV_E_INVALID_CAMERA", -6: "PUV_E_WORKSPACE_TOO_SMALL",
           -7: "PUV_E_STATE_MISMATCH", -8: "PUV_E_CUDA", -9: "PUV_E_UNSUPPORTED"}


class PuvError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_status.get(code, code)}: {msg}")
        self.code = code


class Placement(C.Structure):
    _fields_ = [("rows", C.c_int32), ("cols", C.c_int32), ("x", C.c_int32), ("y", C.c_int32),
                ("rot90ccw", C.c_int32)]


class Layout(C.Structure):
    _fields_ = [("num_levels", C.c_int32), ("sh_degree", C.c_int32), ("planes", C.c_int32),
                ("atlas_w", C.c_int32), ("atlas_h", C.c_int32), ("level", Placement * MAX_LEVELS),
                ("position_mode", C.c_int32), ("center", C.c_float * 3)]


POS_XYZ, POS_RHO = 0, 1


class Camera(C.Structure):
    _fields_ = [("viewmat", C.c_float * 16), ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float),
                ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32), ("near_plane", C.c_float),
                ("campos", C.c_float * 3)]


RENDER_LPO = 1


class RenderOpts(C.Structure):
    _fields_ = [("bg", C.c_float * 3), ("flags", C.c_uint32), ("lpo_spec", C.c_void_p), ("lpo_pos_bits", C.c_int32),
                ("lpo_attr_bits", C.c_int32)]


class ViewDebug(C.Structure):
    _fields_ = [("n_visible", C.c_uint32), ("ntiles", C.c_uint32), ("tiles_x", C.c_uint32),
                ("tiles_y", C.c_uint32), ("n_keys", C.c_uint64), ("tile_start", C.c_void_p),
                ("tile_end", C.c_void_p), ("keys_gid", C.c_void_p), ("depth_key", C.c_void_p),
                ("t_final", C.c_void_p), ("n_contrib", C.c_void_p), ("grad2d", C.c_void_p),
                ("depth_order", C.c_void_p), ("n_examined", C.c_uint64), ("n_composited", C.c_uint64)]


class StepBuffers(C.Structure):
    _fields_ = [("images", C.c_void_p), ("dL_dimages", C.c_void_p), ("loss", C.c_void_p), ("overflow", C.c_void_p),
                ("arena_need", C.c_void_p), ("state", C.c_void_p), ("state_bytes", C.c_size_t),
                ("arena", C.c_void_p), ("arena_bytes", C.c_size_t)]


class Copy(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("bytes", C.c_size_t)]


NUM_STAGES = 11
STAGES = ("project", "depth_sort", "bin", "raster_fwd", "loss", "raster_bwd", "project_bwd", "pack", "label",
          "objective", "quant")


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * NUM_STAGES), ("launches", C.c_uint64 * NUM_STAGES),
                ("calls", C.c_uint64 * NUM_STAGES), ("kernel_launches", C.c_uint64)]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libpuv.so not built at {LIB_PATH}: run __graft_entry__.build() "
                               "(make -C paper_2602_23040_b200/csrc); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        P, S = C.c_void_p, C.c_int32
        L.puv_layout_for_levels.argtypes = [S, P, P, S, P]
        L.puv_pack_atlas.argtypes = [P, P, P, P, P, P]
        L.puv_unpack_levels.argtypes = [P, P, P, P]
        L.puv_query_sizes.argtypes = [P, S, P, P, P, P]
        L.puv_render_views.argtypes = [P, P, P, S, P, P, P, P, C.c_size_t, P, C.c_size_t, P]
        L.puv_l2_loss_grad.argtypes = [C.c_int64, P, P, P, P, P]
        L.puv_render_backward.argtypes = [P, P, P, S, P, P, P, P, P, C.c_size_t, P, C.c_size_t, P, P]
        L.puv_render_l2_step.argtypes = [P, P, P, S, P, P, P, P, P, P, P, P, C.c_size_t, P, C.c_size_t, P, P, P]
        L.puv_check_overflow.argtypes = [P, S, P, P, P]
        L.puv_overflow_accumulate.argtypes = [P, P, P, P]
        L.puv_train_step.argtypes = [P, P, P, S, P, P, P, P, S, P, P, P]
        L.puv_train_step_host.argtypes = [P, P, P, S, P, P, P, S, P, P, P, S, P, P, P, S, P]
        L.puv_train_step_host_atlas.argtypes = [P, P, P, P, S, P, P, P, P, P, S, P, P, P, P, P]
        L.puv_train_step_host_atlas.restype = C.c_int32
        L.puv_debug_view.argtypes = [P, S, P, P, C.c_size_t, P, S, P, P]
        L.puv_debug_contract.argtypes = [S, P, P, C.c_int64, P]
        L.puv_view_counts.argtypes = [P, S, P, P]
        L.puv_view_counts.restype = C.c_int32
        L.puv_layout_paper.argtypes = [S, S, S, P]
        L.puv_layout_paper.restype = C.c_int32
        L.puv_ray_planes.argtypes = [P, P, P]
        L.puv_ray_planes.restype = C.c_int32
        L.puv_label_workspace_bytes.argtypes = [S, S]
        L.puv_label_workspace_bytes.restype = C.c_size_t
        L.puv_label_dynamic.argtypes = [P, P, P, S, P, P, S, P, P, C.c_size_t, P]
        L.puv_label_dynamic.restype = C.c_int32
        L.puv_photo_workspace_bytes.argtypes = [S, S, S]
        L.puv_photo_workspace_bytes.restype = C.c_size_t
        L.puv_photo_loss_grad.argtypes = [S, S, S, P, P, C.c_double, P, P, P, C.c_size_t, P]
        L.puv_photo_loss_grad.restype = C.c_int32
        L.puv_reg_workspace_bytes.argtypes = []
        L.puv_reg_workspace_bytes.restype = C.c_size_t
        L.puv_reg_loss_grad.argtypes = [P, P, P, P, C.c_double, C.c_double, C.c_double, P, P, P, C.c_size_t, P]
        L.puv_reg_loss_grad.restype = C.c_int32
        L.puv_quant_fit.argtypes = [P, P, P, P, P]
        L.puv_quant_fit.restype = C.c_int32
        L.puv_quantize.argtypes = [P, P, P, P, S, S, P, P, P]
        L.puv_quantize.restype = C.c_int32
        L.puv_profile_enable.argtypes = [S]
        L.puv_profile_serial.argtypes = [S]
        L.puv_profile_timeline.argtypes = [P, S, P]
        L.puv_profile_timeline.restype = C.c_int32
        L.puv_profile_serial.restype = C.c_int32
        L.puv_profile_read.argtypes = [P, S]
        L.puv_profile_enable.restype = C.c_int32
        L.puv_profile_read.restype = C.c_int32
        L.puv_last_error.argtypes = [C.c_char_p, C.c_size_t]
        L.puv_last_error.restype = C.c_size_t
        L.puv_version.restype = C.c_char_p
        for f in ("puv_layout_for_levels", "puv_pack_atlas", "puv_unpack_levels", "puv_query_sizes",
                  "puv_render_views", "puv_l2_loss_grad", "puv_render_backward", "puv_check_overflow",
                  "puv_debug_view", "puv_debug_contract", "puv_overflow_accumulate", "puv_train_step",
                  "puv_train_step_host"):
            getattr(L, f).restype = C.c_int32
        _LIB = L
    return _LIB


def last_error() -> str:
    buf = C.create_string_buffer(1024)
    lib().puv_last_error(buf, 1024)
    return buf.value.decode()


def _ok(rc):
    if rc != 0:
        raise PuvError(rc, last_error())


def version() -> str:
    return lib().puv_version().decode()


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _ptr_table(tensors):
    return (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])


def _planes(t):
    """(D, H, W) fp32 CUDA tensor, or a sequence of D contiguous (H, W) fp32 CUDA tensors (planes may be
    shared between atlases, e.g. the constant planes of a frame sequence) -> host table of D pointers."""
    if isinstance(t, torch.Tensor):
        assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous(), "planes: contiguous fp32 CUDA (D,H,W)"
        return _ptr_table([t[d] for d in range(t.shape[0])])
    for p in t:
        assert p.is_cuda and p.dtype == torch.float32 and p.is_contiguous(), "planes: contiguous fp32 CUDA (H,W)"
    return _ptr_table(list(t))


def camera(viewmat, fx, fy, cx, cy, width, height, near, campos) -> Camera:
    c = Camera()
    c.viewmat[:] = [float(x) for x in torch.as_tensor(viewmat, dtype=torch.float32).reshape(-1).tolist()]
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    c.width, c.height, c.near_plane = int(width), int(height), float(near)
    c.campos[:] = [float(x) for x in torch.as_tensor(campos, dtype=torch.float32).reshape(-1).tolist()]
    return c


def cameras(cams) -> C.Array:
    """Sequence of objects with viewmat/fx/fy/cx/cy/width/height/near/campos (e.g. synth.scenes.Camera)."""
    arr = (Camera * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = camera(c.viewmat, c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.near, c.campos)
    return arr


def opts(bg=(0.0, 0.0, 0.0), lpo=None) -> RenderOpts:
    """Render options.  lpo = (spec, pos_bits, attr_bits): render the LPO proxy of the atlas inline
    (PUV_RENDER_LPO; spec = quant_fit's (D, 2) CUDA tensor, kept alive by the caller; pos_bits may be
    "fp16"); the backward then gives the STE gradient of the master planes."""
    o = RenderOpts()
    o.bg[:] = [float(x) for x in bg]
    o.flags = 0
    if lpo is not None:
        spec, pb, ab = lpo
        assert spec.is_cuda and spec.dtype == torch.float32 and spec.is_contiguous()
        o.flags = RENDER_LPO
        o.lpo_spec = spec.data_ptr()
        o.lpo_pos_bits = QUANT_FP16 if pb == "fp16" else int(pb)
        o.lpo_attr_bits = int(ab)
    return o


# ---------------------------------------------------------------------------------------------
# entry points (same names as the C ABI)

def layout_for_levels(shapes, sh_degree: int) -> Layout:
    K = len(shapes)
    rows = (C.c_int32 * K)(*[int(s[0]) for s in shapes])
    cols = (C.c_int32 * K)(*[int(s[1]) for s in shapes])
    out = Layout()
    _ok(lib().puv_layout_for_levels(K, rows, cols, sh_degree, C.byref(out)))
    return out


def layout_paper(S: int, K: int, sh_degree: int) -> Layout:
    """The paper's pyramid schedule + recursive atlas layout."""
    out = Layout()
    _ok(lib().puv_layout_paper(S, K, sh_degree, C.byref(out)))
    return out


def ray_planes(layout: Layout, device="cuda", stream=None) -> torch.Tensor:
    """(3, H_A, W_A) fp32 UV-ray directions of every atlas texel (for position_mode = POS_RHO)."""
    out = torch.empty((3, layout.atlas_h, layout.atlas_w), dtype=torch.float32, device=device)
    _ok(lib().puv_ray_planes(C.byref(layout), _planes(out), _stream(stream)))
    return out


def with_rho(layout: Layout, center) -> Layout:
    """A copy of `layout` in POS_RHO mode about `center`."""
    L = Layout.from_buffer_copy(layout)
    L.position_mode = POS_RHO
    L.center[:] = [float(x) for x in center]
    return L


def rho_plane_table(atlas: torch.Tensor, rays: torch.Tensor):
    """Plane table of a POS_RHO atlas: [rho, -, -, planes 3..D-1, ray x, y, z] (entries 1, 2 unused)."""
    return [atlas[0], atlas[0], atlas[0]] + [atlas[d] for d in range(3, atlas.shape[0])] + [rays[0], rays[1], rays[2]]


def pack_atlas(layout: Layout, level_planes, level_occ=None, stream=None):
    """level_planes: list of K (D, rows, cols) fp32 CUDA tensors; level_occ: list of K uint8 or None.
    Returns (atlas (D, H_A, W_A) fp32, occ (H_A, W_A) uint8)."""
    D = layout.planes
    dev = level_planes[0].device
    atlas = torch.empty((D, layout.atlas_h, layout.atlas_w), dtype=torch.float32, device=dev)
    occ = torch.empty((layout.atlas_h, layout.atlas_w), dtype=torch.uint8, device=dev)
    lp = _ptr_table([lv[d] for lv in level_planes for d in range(D)])
    lo = _ptr_table(level_occ) if level_occ is not None else None
    _ok(lib().puv_pack_atlas(C.byref(layout), lp, lo, _planes(atlas), _ptr(occ), _stream(stream)))
    return atlas, occ


def unpack_levels(layout: Layout, atlas: torch.Tensor, stream=None):
    D = layout.planes
    out = [torch.empty((D, layout.level[k].rows, layout.level[k].cols), dtype=torch.float32, device=atlas.device)
           for k in range(layout.num_levels)]
    lp = _ptr_table([lv[d] for lv in out for d in range(D)])
    _ok(lib().puv_unpack_levels(C.byref(layout), _planes(atlas), lp, _stream(stream)))
    return out


def query_sizes(layout: Layout, cams, opts_=None):
    sb, ah = C.c_size_t(), C.c_size_t()
    _ok(lib().puv_query_sizes(C.byref(layout), len(cams), cams, C.byref(opts_) if opts_ else None,
                              C.byref(sb), C.byref(ah)))
    return sb.value, ah.value


def _check_images(name, t, n_views, cams, dtype=torch.float32):
    """Image-like argument: contiguous CUDA tensor of `dtype` with n_views*3*H*W elements (the C ABI
    reads and writes that many elements at its data pointer)."""
    W, H = cams[0].width, cams[0].height
    assert isinstance(t, torch.Tensor) and t.is_cuda, f"{name}: CUDA tensor expected"
    assert t.dtype == dtype, f"{name}: {dtype} expected, got {t.dtype}"
    assert t.is_contiguous(), f"{name}: must be contiguous"
    assert t.numel() == n_views * 3 * H * W, f"{name}: {t.numel()} elements != n_views*3*H*W = {n_views * 3 * H * W}"


def _check_loss(loss):
    assert isinstance(loss, torch.Tensor) and loss.is_cuda and loss.dtype == torch.float64 and loss.numel() >= 1, \
        "loss: CUDA fp64 tensor with >= 1 element expected"


def render_views(layout, atlas, occ, cams, opts_, images, state, arena, stream=None):
    _check_images("images", images, len(cams), cams)
    _ok(lib().puv_render_views(C.byref(layout), _planes(atlas), _ptr(occ), len(cams), cams,
                               C.byref(opts_) if opts_ else None, _ptr(images), _ptr(state), state.numel(),
                               _ptr(arena), arena.numel(), _stream(stream)))


def l2_loss_grad(images, targets, dL, loss, stream=None):
    for name, t in (("images", images), ("targets", targets), ("dL", dL)):
        assert isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous(), \
            f"{name}: contiguous fp32 CUDA tensor expected"
        assert t.numel() == images.numel(), f"{name}: {t.numel()} elements != images' {images.numel()}"
    _check_loss(loss)
    _ok(lib().puv_l2_loss_grad(images.numel(), _ptr(images), _ptr(targets), _ptr(dL), _ptr(loss), _stream(stream)))


def quant_fit(layout, atlas, occ, spec=None, stream=None):
    """LPO: per-plane (min, max) over occupied texels -> (D, 2) fp32 CUDA tensor."""
    dev = atlas.device if isinstance(atlas, torch.Tensor) else atlas[0].device
    if spec is None:
        spec = torch.empty((layout.planes, 2), dtype=torch.float32, device=dev)
    _ok(lib().puv_quant_fit(C.byref(layout), _planes(atlas), _ptr(occ), _ptr(spec), _stream(stream)))
    return spec


QUANT_FP16 = 256   # pos_bits value: position planes stored as IEEE binary16 (include/puv.h, reading Q8)


def quantize(layout, atlas, occ, spec, pos_bits=16, attr_bits=8, proxy=None, codes=False, stream=None):
    """LPO fake quantiser.  Returns (proxy (D, H_A, W_A) fp32 or None, code planes list or None); code
    planes are uint8 (bits <= 8) or uint16 (bits > 8 or binary16).  proxy=False skips the proxy.
    pos_bits="fp16" (or QUANT_FP16) stores the position planes as binary16."""
    if pos_bits == "fp16":
        pos_bits = QUANT_FP16
    dev = spec.device
    shp = (layout.atlas_h, layout.atlas_w)
    rho = layout.position_mode == POS_RHO
    if proxy is None:
        proxy = torch.empty((layout.planes,) + shp, dtype=torch.float32, device=dev)
        if rho:
            proxy[1:3] = atlas[1:3] if isinstance(atlas, torch.Tensor) else 0.0
    ptab = None if proxy is False else _planes(proxy)
    code_list = None
    ctab = None
    if codes:
        code_list = []
        for d in range(layout.planes):
            bits = pos_bits if d < 3 else attr_bits
            code_list.append(torch.zeros(shp, dtype=torch.uint16 if bits > 8 else torch.uint8, device=dev))
            # (QUANT_FP16 > 8: binary16 patterns are uint16 planes)
        ctab = _ptr_table(code_list)
    _ok(lib().puv_quantize(C.byref(layout), _planes(atlas), _ptr(occ), _ptr(spec), int(pos_bits), int(attr_bits),
                           ctab, ptab, _stream(stream)))
    return (None if proxy is False else proxy), code_list


def photo_workspace_bytes(width: int, height: int, views_per_chunk: int = 1) -> int:
    return int(lib().puv_photo_workspace_bytes(width, height, views_per_chunk))


def photo_loss_grad(images, targets, dL, loss, lambda_ssim=0.2, workspace=None, stream=None):
    """L1 + SSIM photometric loss.  images/targets/dL: (V, 3, H, W) fp32 CUDA;
    loss: (1,) fp64 CUDA, overwritten.  Returns the workspace (reuse it across calls)."""
    V, _, H, W = images.shape
    for name, t in (("images", images), ("targets", targets), ("dL", dL)):
        assert isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous(), \
            f"{name}: contiguous fp32 CUDA tensor expected"
        assert tuple(t.shape) == (V, 3, H, W), f"{name}: shape {tuple(t.shape)} != {(V, 3, H, W)}"
    _check_loss(loss)
    if workspace is None:
        workspace = torch.empty(photo_workspace_bytes(W, H, min(V, 8)), dtype=torch.uint8, device=images.device)
    _ok(lib().puv_photo_loss_grad(V, W, H, _ptr(images), _ptr(targets), float(lambda_ssim), _ptr(dL), _ptr(loss),
                                  _ptr(workspace), workspace.numel(), _stream(stream)))
    return workspace


def reg_workspace_bytes() -> int:
    return int(lib().puv_reg_workspace_bytes())


def reg_loss_grad(layout, atlas, occ, grad, loss, lambda_scale=1e-4, lambda_opacity=1e-4, s_max=0.05, mask=None,
                  workspace=None, stream=None):
    """Scale + opacity regularisers; grad planes ACCUMULATED, loss overwritten."""
    dev = loss.device
    if workspace is None:
        workspace = torch.empty(reg_workspace_bytes(), dtype=torch.uint8, device=dev)
    _ok(lib().puv_reg_loss_grad(C.byref(layout), _planes(atlas), _ptr(occ), _ptr(mask), float(lambda_scale),
                                float(lambda_opacity), float(s_max), _planes(grad), _ptr(loss), _ptr(workspace),
                                workspace.numel(), _stream(stream)))
    return workspace


def render_backward(layout, atlas, occ, cams, opts_, dL, mask, state, arena, grad, stream=None):
    _check_images("dL", dL, len(cams), cams)
    _ok(lib().puv_render_backward(C.byref(layout), _planes(atlas), _ptr(occ), len(cams), cams,
                                  C.byref(opts_) if opts_ else None, _ptr(dL), _ptr(mask), _ptr(state),
                                  state.numel(), _ptr(arena), arena.numel(), _planes(grad), _stream(stream)))


def render_l2_step(layout, atlas, occ, cams, opts_, images, targets, dL, loss, mask, state, arena, grad,
                   targets_ready=None, stream=None):
    """Fused render + L2 loss gradient + backward (include/puv.h puv_render_l2_step).
    targets_ready: optional torch.cuda.Event the loss gradients wait for."""
    ev = C.c_void_p(targets_ready.cuda_event) if targets_ready is not None else None
    for name, t in (("images", images), ("targets", targets), ("dL", dL)):
        _check_images(name, t, len(cams), cams)
    _check_loss(loss)
    _ok(lib().puv_render_l2_step(C.byref(layout), _planes(atlas), _ptr(occ), len(cams), cams,
                                 C.byref(opts_) if opts_ else None, _ptr(images), _ptr(targets), _ptr(dL),
                                 _ptr(loss), _ptr(mask), _ptr(state), state.numel(), _ptr(arena), arena.numel(),
                                 _planes(grad), ev, _stream(stream)))


def label_workspace_bytes(width: int, height: int) -> int:
    return int(lib().puv_label_workspace_bytes(width, height))


def label_dynamic(layout, atlas, occ, cams, masks, r_max=64, labels=None, workspace=None, stream=None):
    """Supp. Alg. 1 flow masking.  masks: (n_cams, H, W) uint8 CUDA tensor.  Returns labels (H_A, W_A) uint8."""
    dev = masks.device
    W, H = cams[0].width, cams[0].height
    if labels is None:
        labels = torch.empty((layout.atlas_h, layout.atlas_w), dtype=torch.uint8, device=dev)
    if workspace is None:
        workspace = torch.empty(label_workspace_bytes(W, H), dtype=torch.uint8, device=dev)
    assert masks.dtype == torch.uint8 and masks.is_contiguous() and tuple(masks.shape) == (len(cams), H, W)
    _ok(lib().puv_label_dynamic(C.byref(layout), _planes(atlas), _ptr(occ), len(cams), cams, _ptr(masks), int(r_max),
                                _ptr(labels), _ptr(workspace), workspace.numel(), _stream(stream)))
    return labels


def _copies(pairs):
    """[(src_tensor, dst_tensor), ...] -> (array of puv_copy, n); bytes = src.numel() * element size."""
    arr = (Copy * max(len(pairs), 1))()
    for i, (a, b) in enumerate(pairs):
        assert a.is_contiguous() and b.is_contiguous() and a.nbytes == b.nbytes, "copy: contiguous, equal sizes"
        arr[i] = Copy(a.data_ptr(), b.data_ptr(), a.nbytes)
    return arr, len(pairs)


class StepState:
    """Device buffers of puv_train_step for chunks of `views_per_call` views (images, dL/dImage,
    loss, overflow flags, state, key arena); the arena grows on overflow (TrainStep.run)."""

    def __init__(self, layout, cams_chunk, device, arena_bytes=None, bg=(0.0, 0.0, 0.0)):
        self.opts = opts(bg)
        sb, hint = query_sizes(layout, cams_chunk, self.opts)
        W, H = cams_chunk[0].width, cams_chunk[0].height
        n = len(cams_chunk)
        self.device = torch.device(device)
        self.state = torch.empty(sb, dtype=torch.uint8, device=self.device)
        self.arena = torch.empty(arena_bytes if arena_bytes else hint, dtype=torch.uint8, device=self.device)
        self.images = torch.empty((n, 3, H, W), dtype=torch.float32, device=self.device)
        self.dL = torch.empty_like(self.images)
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.flags = torch.zeros(2, dtype=torch.int64, device=self.device)   # [overflow (u32 in low word), need]
        self.views_per_call = n

    def buffers(self) -> StepBuffers:
        b = StepBuffers()
        b.images, b.dL_dimages, b.loss = self.images.data_ptr(), self.dL.data_ptr(), self.loss.data_ptr()
        b.overflow, b.arena_need = self.flags.data_ptr(), self.flags.data_ptr() + 8
        b.state, b.state_bytes = self.state.data_ptr(), self.state.numel()
        b.arena, b.arena_bytes = self.arena.data_ptr(), self.arena.numel()
        return b

    def overflow(self):
        """(overflowed, arena bytes needed) of the last step (synchronises)."""
        f = self.flags.cpu()
        return bool(int(f[0]) & 0xFFFFFFFF), int(f[1])

    def grow(self, need):
        self.arena = torch.empty(int(need * 1.1) + 4096, dtype=torch.uint8, device=self.device)


def train_step(layout, atlas, occ, cams, targets, grad, st: StepState, mask=None, stream=None):
    """puv_train_step: grad (D planes) OVERWRITTEN with dL/dtexels over all `cams`; st.loss = L."""
    _check_images("targets", targets, len(cams), cams)
    _ok(lib().puv_train_step(C.byref(layout), _planes(atlas), _ptr(occ), len(cams), cams, C.byref(st.opts),
                             _ptr(targets), _ptr(mask), st.views_per_call, C.byref(st.buffers()), _planes(grad),
                             _stream(stream)))


def train_step_host(layout, atlas, occ, cams, targets_host, targets, grad, st: StepState, uploads=(), downloads=(),
                    mask=None, stream=None):
    """puv_train_step_host: `uploads` / `downloads` are [(host, device)] / [(device, host)] tensor
    pairs copied before / after the step; targets_host -> targets overlaps the render."""
    _check_images("targets", targets, len(cams), cams)
    assert not targets_host.is_cuda and targets_host.is_contiguous() and targets_host.numel() == targets.numel()
    up, nu = _copies(list(uploads))
    down, nd = _copies(list(downloads))
    _ok(lib().puv_train_step_host(C.byref(layout), _planes(atlas), _ptr(occ), len(cams), cams, C.byref(st.opts), up,
                                  nu, _ptr(targets_host), _ptr(targets), _ptr(mask), st.views_per_call,
                                  C.byref(st.buffers()), _planes(grad), down, nd, _stream(stream)))


def train_step_host_atlas(layout, atlas_dev, atlas_host, occ, cams, targets_host, targets, grad, grad_host, loss_host,
                          st: StepState, mask=None, stream=None):
    """puv_train_step_host_atlas: atlas_host -> atlas_dev and grad -> grad_host in texel chunks overlapping
    K1 / K7, targets_host -> targets beside the render, the loss into loss_host (all host tensors pinned,
    contiguous; atlas_host / grad_host (D, H_A, W_A) fp32, loss_host (1,) fp64)."""
    _check_images("targets", targets, len(cams), cams)
    for name, t in (("atlas_host", atlas_host), ("grad_host", grad_host), ("targets_host", targets_host)):
        assert not t.is_cuda and t.is_contiguous() and t.dtype == torch.float32, f"{name}: contiguous fp32 host"
    assert atlas_host.numel() == grad_host.numel() == layout.planes * layout.atlas_w * layout.atlas_h
    assert not loss_host.is_cuda and loss_host.dtype == torch.float64
    _ok(lib().puv_train_step_host_atlas(C.byref(layout), _planes(atlas_dev), _ptr(atlas_host), _ptr(occ), len(cams),
                                        cams, C.byref(st.opts), _ptr(targets_host), _ptr(targets), _ptr(mask),
                                        st.views_per_call, C.byref(st.buffers()), _planes(grad), _ptr(grad_host),
                                        _ptr(loss_host), _stream(stream)))


def check_overflow(state, n_views, stream=None):
    ov, need = C.c_int32(), C.c_uint64()
    _ok(lib().puv_check_overflow(_ptr(state), n_views, _stream(stream), C.byref(ov), C.byref(need)))
    return bool(ov.value), int(need.value)


def view_counts(state, view, stream=None) -> dict:
    """n_visible, K, examined, composited, overflow of one view of the last render (no list materialisation)."""
    out = (C.c_uint64 * 5)()
    _ok(lib().puv_view_counts(_ptr(state), int(view), _stream(stream), out))
    return {"n_vis": int(out[0]), "K": int(out[1]), "examined": int(out[2]), "composited": int(out[3]),
            "overflow": bool(out[4])}


def debug_view(layout, cams, state, arena, view, stream=None) -> ViewDebug:
    out = ViewDebug()
    _ok(lib().puv_debug_view(C.byref(layout), len(cams), cams, _ptr(state), state.numel(), _ptr(arena), view,
                             _stream(stream), C.byref(out)))
    return out


def profile_serial(on: bool = True):
    """Run each view's depth sort + binning on the caller's stream (serialised stage times)."""
    _ok(lib().puv_profile_serial(1 if on else 0))


def profile_timeline(max_events: int = 100000):
    """[(stage name, start ms, end ms)] of the recorded stage instances (call before profile_read(reset))."""
    buf = (C.c_double * (3 * max_events))()
    n = C.c_int32()
    _ok(lib().puv_profile_timeline(buf, max_events, C.byref(n)))
    return [(STAGES[int(buf[3 * i])], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n.value)]


def profile_enable(on: bool = True):
    _ok(lib().puv_profile_enable(1 if on else 0))


def profile_read(reset: bool = True) -> dict:
    """Per-stage device ms / kernel launches / stage instances since the last reset (syncs)."""
    p = Profile()
    _ok(lib().puv_profile_read(C.byref(p), 1 if reset else 0))
    return {"ms": {s: p.ms[i] for i, s in enumerate(STAGES)},
            "launches": {s: int(p.launches[i]) for i, s in enumerate(STAGES)},
            "calls": {s: int(p.calls[i]) for i, s in enumerate(STAGES)},
            "kernel_launches": int(p.kernel_launches)}


def kernel_launches() -> int:
    p = Profile()
    _ok(lib().puv_profile_read(C.byref(p), 0))
    return int(p.kernel_launches)


def debug_contract(op: str, x: torch.Tensor, stream=None) -> torch.Tensor:
    """exp_c / log_c of DESIGN.md R13 on a CUDA fp32 tensor (bit-equality tests)."""
    out = torch.empty_like(x)
    _ok(lib().puv_debug_contract({"exp_c": 0, "log_c": 1}[op], _ptr(x), _ptr(out), x.numel(), _stream(stream)))
    return out


def _view_of(owner: torch.Tensor, ptr, n, dtype):
    """A cloned tensor of n elements at device address `ptr` inside the uint8 buffer `owner`."""
    esz = torch.empty(0, dtype=dtype).element_size()
    if n == 0:
        return torch.empty(0, dtype=dtype, device=owner.device)
    off = int(ptr) - owner.data_ptr()
    assert 0 <= off and off + n * esz <= owner.numel(), "debug pointer outside its buffer"
    return owner[off:off + n * esz].view(dtype).clone()


def debug_tensors(layout, cams, state, arena, view):
    """Per-view binning / pixel state copied out of the state (for parity tests)."""
    d = debug_view(layout, cams, state, arena, view)
    N = layout.atlas_w * layout.atlas_h
    W, H = cams[0].width, cams[0].height
    return {
        "n_visible": d.n_visible, "ntiles": d.ntiles, "n_keys": d.n_keys,
        "n_examined": d.n_examined, "n_composited": d.n_composited,
        "tile_start": _view_of(state, d.tile_start, d.ntiles, torch.int32),
        "tile_end": _view_of(state, d.tile_end, d.ntiles, torch.int32),
        "keys_gid": _view_of(arena, d.keys_gid, d.n_keys, torch.int32),
        "depth_key": _view_of(state, d.depth_key, N, torch.int32),
        "t_final": _view_of(state, d.t_final, W * H, torch.float32).reshape(H, W),
        "n_contrib": _view_of(state, d.n_contrib, W * H, torch.int32).reshape(H, W),
        "grad2d": _view_of(state, d.grad2d, N * 9, torch.float64).reshape(N, 9),
        "depth_order": _view_of(state, d.depth_order, d.n_visible, torch.int32),
    }


# ---------------------------------------------------------------------------------------------
# convenience: a renderer that owns state + arena and grows the arena on overflow

class Renderer:
    """Owns the per-call state and key arena for a fixed (layout, cameras) signature."""

    def __init__(self, layout: Layout, cams, bg=(0.0, 0.0, 0.0), device="cuda", arena_bytes=None, lpo=None):
        self.layout = layout
        self.cams = cams
        self.opts = opts(bg, lpo)
        self.device = torch.device(device)
        sb, hint = query_sizes(layout, cams, self.opts)
        self.state = torch.empty(sb, dtype=torch.uint8, device=self.device)
        self.arena = torch.empty(arena_bytes if arena_bytes else hint, dtype=torch.uint8, device=self.device)
        W, H = cams[0].width, cams[0].height
        self.image_shape = (len(cams), 3, H, W)

    def forward(self, atlas, occ, images=None, stream=None, check=True):
        if images is None:
            images = torch.empty(self.image_shape, dtype=torch.float32, device=self.device)
        while True:
            render_views(self.layout, atlas, occ, self.cams, self.opts, images, self.state, self.arena, stream)
            if not check:
                return images
            ov, need = check_overflow(self.state, len(self.cams), stream)
            if not ov:
                return images
            self.arena = torch.empty(int(need * 1.1) + 4096, dtype=torch.uint8, device=self.device)

    def backward(self, atlas, occ, dL, grad=None, mask=None, stream=None):
        if grad is None:
            grad = (torch.zeros_like(atlas) if isinstance(atlas, torch.Tensor) else
                    torch.zeros((self.layout.planes,) + tuple(atlas[0].shape), dtype=torch.float32,
                                device=self.device))
        render_backward(self.layout, atlas, occ, self.cams, self.opts, dL, mask, self.state, self.arena, grad,
                        stream)
        return grad
