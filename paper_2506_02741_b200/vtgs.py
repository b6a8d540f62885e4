"""Thin Python binding of include/vtgs.h (argument marshalling only).

Every function named `vtgs_*` here is the C function of the same name, called through ctypes
with `tensor.data_ptr()` and the current CUDA stream.  No step of the method runs in Python:
if `libvtgs.so` is missing this module raises on import, and without a CUDA device every call
fails with VTGS_ERR_NO_DEVICE — there is no CPU fallback.

`Renderer` bundles a context with torch-allocated outputs for convenience.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# VTGS_LIB=checked loads the bounds-checked build (libvtgs_checked.so, tests/test_gpu_variants.py)
LIB_PATH = os.path.join(_HERE, "libvtgs_checked.so" if os.environ.get("VTGS_LIB") == "checked" else "libvtgs.so")
# A/B of compile-time variants (tools/gpu_lib_ab.sh): an explicit path to another in-tree build
LIB_PATH = os.environ.get("VTGS_LIB_PATH", LIB_PATH)
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2506_02741_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

VTGS_OK = 0
VTGS_ERR_INVALID_ARG = -1
VTGS_ERR_SHAPE = -2
VTGS_ERR_CAPACITY = -3
VTGS_ERR_CUDA = -4
VTGS_ERR_STATE = -5
VTGS_ERR_NO_DEVICE = -6
VTGS_GRAD_COLOR, VTGS_GRAD_OPACITY, VTGS_GRAD_RADIUS, VTGS_GRAD_POSE, VTGS_GRAD_POSITION = 1, 2, 4, 8, 16
VTGS_GRAD_DETERMINISTIC = 32
VTGS_GRAD_ATTR = VTGS_GRAD_COLOR | VTGS_GRAD_OPACITY | VTGS_GRAD_RADIUS
VTGS_GRAD_ALL = VTGS_GRAD_ATTR | VTGS_GRAD_POSE


class vtgs_intrinsics(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_float), ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class vtgs_pose(ctypes.Structure):
    _fields_ = [("q", ctypes.c_float * 4), ("t", ctypes.c_float * 3)]


class vtgs_l1_loss(ctypes.Structure):
    _fields_ = [("target_rgb", ctypes.c_void_p), ("target_depth", ctypes.c_void_p), ("vis_mask", ctypes.c_void_p),
                ("w_color", ctypes.c_float), ("w_depth", ctypes.c_float), ("color_mask_mode", ctypes.c_int32),
                ("depth_mask_mode", ctypes.c_int32), ("normalize", ctypes.c_int32), ("extra_dcolor", ctypes.c_void_p)]


class vtgs_stats(ctypes.Structure):
    _fields_ = [("n_gaussians", ctypes.c_int64), ("n_pairs", ctypes.c_int64), ("e_eval", ctypes.c_int64),
                ("e_comp", ctypes.c_int64), ("max_tile", ctypes.c_int64), ("overflow", ctypes.c_int64),
                ("launches", ctypes.c_int64)]


_c = ctypes
_P = ctypes.c_void_p
_SIGS = {
    "vtgs_abi_version": (_c.c_int32, []),
    "vtgs_measure_peaks": (_c.c_int32, [_c.c_int32, _P, _P]),
    "vtgs_create": (_c.c_int32, [_c.POINTER(_P), _c.c_int32, _c.c_int64, _c.c_int32, _c.c_int32, _c.c_int64]),
    "vtgs_destroy": (_c.c_int32, [_P]),
    "vtgs_status_string": (_c.c_char_p, [_c.c_int32]),
    "vtgs_last_error": (_c.c_char_p, [_P]),
    "vtgs_instantiate": (_c.c_int32, [_P, _P, _P, _P, _c.c_int32, vtgs_intrinsics, _P, _c.c_float, _P, _P, _P, _P]),
    "vtgs_render_fwd": (_c.c_int32, [_P, _P, _P, _c.c_int64, _P, vtgs_intrinsics, _P, _P, _P, _P]),
    "vtgs_render_bwd": (_c.c_int32, [_P, _P, _P, _P, _c.POINTER(vtgs_l1_loss), _c.c_uint32, _c.c_int64, _c.c_int64,
                                     _P, _P, _P, _P, _P, _P]),
    "vtgs_visibility_mask": (_c.c_int32, [_P, _P, _P, _P, _P, _c.c_int32, vtgs_intrinsics, _c.c_float, _P, _P, _P]),
    "vtgs_visibility_counts": (_c.c_int32, [_P, _P, _P, _P, _P, _c.c_int32, vtgs_intrinsics, _c.c_float, _P, _P, _P]),
    "vtgs_densify": (_c.c_int32, [_P, _P, _P, _P, vtgs_intrinsics, _P, _c.c_float, _P, _c.c_float, _P, _P, _P, _P]),
    "vtgs_ssim_loss": (_c.c_int32, [_P, _P, _P, _c.c_int32, _c.c_int32, _c.c_float, _P, _P, _P]),
    "vtgs_keyframe_pose_grad": (_c.c_int32, [_P, _P, _P, _P, _c.c_int32, _c.c_int64, _P, _P]),
    "vtgs_pose_adam_step": (_c.c_int32, [_P, _P, _P, _P, _c.c_float, _c.c_float, _P]),
    "vtgs_get_stats": (_c.c_int32, [_P, _c.POINTER(vtgs_stats), _P]),
    "vtgs_check": (_c.c_int32, [_P, _P]),
    "vtgs_set_profiling": (_c.c_int32, [_P, _c.c_int32]),
    "vtgs_set_work_counters": (_c.c_int32, [_P, _c.c_int32]),
    "vtgs_get_profile": (_c.c_int32, [_P, _P, _P, _P]),
    "vtgs_export_tiles": (_c.c_int32, [_P, _P, _P, _c.c_int64, _c.POINTER(_c.c_int64), _P]),
    "vtgs_step_host": (_c.c_int32, [_P, _P, _P, _c.c_int64, _P, vtgs_intrinsics, _P, _P, _c.c_float, _c.c_float,
                                    _c.c_int32, _c.c_int32, _c.c_int32, _c.c_uint32, _c.c_int64, _c.c_int64,
                                    _P, _P, _P, _P, _P, _P, _P, _P]),
    "vtgs_step_host_sensor": (_c.c_int32, [_P, _P, _P, _c.c_int64, _P, vtgs_intrinsics, _P, _P, _c.c_float,
                                           _c.c_float, _c.c_float, _c.c_int32, _c.c_int32, _c.c_int32, _c.c_uint32,
                                           _c.c_int64, _c.c_int64, _P, _P, _P, _P, _P, _P, _P, _P]),
}
EXPORTED = tuple(_SIGS)
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


class VtgsError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        self.status = status
        msg = vtgs_status_string(status).decode()
        super().__init__(f"vtgs status {status} ({msg}){': ' + detail if detail else ''}")


def _ok(status: int, ctx=None):
    if status != VTGS_OK:
        detail = vtgs_last_error(ctx).decode() if ctx else ""
        raise VtgsError(status, detail)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensors passed to vtgs must be contiguous")
    return t.data_ptr()


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def intrinsics(intr) -> vtgs_intrinsics:
    return vtgs_intrinsics(float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy), int(intr.width),
                           int(intr.height))


def pose_tensor(poses, device) -> torch.Tensor:
    """(…, 7) (w, x, y, z, tx, ty, tz) → contiguous float32 device tensor = vtgs_pose[…]."""
    return torch.as_tensor(poses, dtype=torch.float32).reshape(-1, 7).contiguous().to(device)


class Renderer:
    """One vtgs context (scratch for one in-flight forward/backward) on one device."""

    def __init__(self, device: int, max_gaussians: int, max_width: int, max_height: int, max_pairs: int = 0):
        self.device = torch.device("cuda", device)
        h = ctypes.c_void_p()
        _ok(vtgs_create(ctypes.byref(h), int(device), int(max_gaussians), int(max_width), int(max_height),
                        int(max_pairs)))
        self.ctx = h
        self.max_gaussians = max_gaussians

    def close(self):
        if getattr(self, "ctx", None):
            vtgs_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- (1)
    def instantiate(self, depth: torch.Tensor, rgb: torch.Tensor, kf_poses: torch.Tensor, intr,
                    opacity: Optional[torch.Tensor] = None, opacity_default: float = 0.5,
                    out=None, stream=None, n_valid: Optional[torch.Tensor] = None):
        """(1) view-tied Gaussians of K keyframes → (pos_rad, col_opa); `n_valid` (int64 [1] device,
        optional) receives the valid-slot count."""
        K = depth.shape[0]
        N = K * intr.width * intr.height
        pos_rad, col_opa = out if out is not None else (
            torch.empty((N, 4), dtype=torch.float32, device=self.device),
            torch.empty((N, 4), dtype=torch.float32, device=self.device))
        _ok(vtgs_instantiate(self.ctx, _ptr(depth), _ptr(rgb), _ptr(kf_poses), K, intrinsics(intr), _ptr(opacity),
                             float(opacity_default), _ptr(pos_rad), _ptr(col_opa), _ptr(n_valid), _stream(stream)),
            self.ctx)
        return pos_rad, col_opa

    # --- (2)-(4)
    def render_fwd(self, pos_rad: torch.Tensor, col_opa: torch.Tensor, view: torch.Tensor, intr, out=None,
                   stream=None, N: Optional[int] = None):
        H, W = intr.height, intr.width
        if out is None:
            out = (torch.empty((H, W, 3), dtype=torch.float32, device=self.device),
                   torch.empty((H, W), dtype=torch.float32, device=self.device),
                   torch.empty((H, W), dtype=torch.float32, device=self.device))
        color, depth, sil = out
        n = pos_rad.shape[0] if N is None else N
        _ok(vtgs_render_fwd(self.ctx, _ptr(pos_rad), _ptr(col_opa), n, _ptr(view), intrinsics(intr), _ptr(color),
                            _ptr(depth), _ptr(sil), _stream(stream)), self.ctx)
        return color, depth, sil

    # --- (5)
    def render_bwd(self, want: int, d_col_opa=None, d_radius=None, d_pose=None, dL_dcolor=None, dL_ddepth=None,
                   dL_dsil=None, loss: Optional[dict] = None, learn: Sequence[int] = (0, 1 << 62),
                   loss_out=None, stream=None, d_position=None):
        lp = None
        if loss is not None:
            L = vtgs_l1_loss(_ptr(loss["target_rgb"]), _ptr(loss["target_depth"]), _ptr(loss.get("vis_mask")),
                             float(loss.get("w_color", 1.0)), float(loss.get("w_depth", 1.0)),
                             int(loss.get("color_mask_mode", 0)), int(loss.get("depth_mask_mode", 0)),
                             int(loss.get("normalize", 0)), _ptr(loss.get("extra_dcolor")))
            lp = ctypes.byref(L)
        _ok(vtgs_render_bwd(self.ctx, _ptr(dL_dcolor), _ptr(dL_ddepth), _ptr(dL_dsil), lp, int(want), int(learn[0]),
                            int(learn[1]), _ptr(d_col_opa), _ptr(d_radius), _ptr(d_position), _ptr(d_pose),
                            _ptr(loss_out), _stream(stream)), self.ctx)

    def visibility_mask(self, depth: torch.Tensor, pose: torch.Tensor, ref_depth: torch.Tensor,
                        ref_poses: torch.Tensor, intr, tol: float = 0.01, mask=None, stream=None):
        """Visibility of a frame's back-projected pixels to reference views → uint8 [H, W]."""
        H, W = depth.shape
        R = ref_poses.reshape(-1, 7).shape[0]
        if mask is None:
            mask = torch.empty((H, W), dtype=torch.uint8, device=self.device)
        _ok(vtgs_visibility_mask(self.ctx, _ptr(depth), _ptr(pose), _ptr(ref_depth), _ptr(ref_poses), R,
                                 intrinsics(intr), float(tol), _ptr(mask), None, _stream(stream)), self.ctx)
        return mask

    def visibility_counts(self, depth: torch.Tensor, pose: torch.Tensor, ref_depth: torch.Tensor,
                          ref_poses: torch.Tensor, intr, tol: float = 0.01, stream=None):
        """Per-candidate visible-point counts of a frame → (int64 [R] device, int64 [1]
        device valid-pixel count)."""
        R = ref_poses.reshape(-1, 7).shape[0]
        counts = torch.empty(R, dtype=torch.int64, device=self.device)
        n_valid = torch.empty(1, dtype=torch.int64, device=self.device)
        _ok(vtgs_visibility_counts(self.ctx, _ptr(depth), _ptr(pose), _ptr(ref_depth), _ptr(ref_poses), R,
                                   intrinsics(intr), float(tol), _ptr(counts), _ptr(n_valid), _stream(stream)), self.ctx)
        return counts, n_valid

    def densify(self, depth: torch.Tensor, rgb: torch.Tensor, pose: torch.Tensor, intr, silhouette: torch.Tensor,
                pos_rad_out: torch.Tensor, col_opa_out: torch.Tensor, threshold: float = 0.5, opacity=None,
                opacity_default: float = 0.5, stream=None) -> int:
        """Regular-frame densification: returns the number of new Gaussians
        written to pos_rad_out / col_opa_out (synchronises the stream to read it)."""
        n = torch.zeros(1, dtype=torch.int64, device=self.device)
        _ok(vtgs_densify(self.ctx, _ptr(depth), _ptr(rgb), _ptr(pose), intrinsics(intr), _ptr(silhouette),
                         float(threshold), _ptr(opacity), float(opacity_default), _ptr(pos_rad_out), _ptr(col_opa_out),
                         _ptr(n), _stream(stream)), self.ctx)
        return int(n.item())

    def ssim_loss(self, color: torch.Tensor, target_rgb: torch.Tensor, tau: float = 0.2, d_color=None,
                  loss_out=None, stream=None):
        """SSIM term τ·L_S of Eq. 2: d_color += dL/dcolor, loss_out = τ·L_S."""
        H, W = color.shape[0], color.shape[1]
        _ok(vtgs_ssim_loss(self.ctx, _ptr(color), _ptr(target_rgb), int(W), int(H), float(tau), _ptr(d_color),
                           _ptr(loss_out), _stream(stream)), self.ctx)

    def keyframe_pose_grad(self, pos_rad: torch.Tensor, d_position: torch.Tensor, kf_poses: torch.Tensor,
                           slots_per_kf: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Head-frame bundle adjustment: dL/d(keyframe pose) [K, 7]."""
        K = kf_poses.reshape(-1, 7).shape[0]
        if out is None:
            out = torch.empty((K, 7), dtype=torch.float32, device=self.device)
        _ok(vtgs_keyframe_pose_grad(self.ctx, _ptr(pos_rad), _ptr(d_position), _ptr(kf_poses), K, int(slots_per_kf),
                                    _ptr(out), _stream(stream)), self.ctx)
        return out

    def pose_adam_step(self, pose: torch.Tensor, d_pose: torch.Tensor, state: torch.Tensor, lr_rot: float,
                       lr_trans: float, stream=None):
        _ok(vtgs_pose_adam_step(self.ctx, _ptr(pose), _ptr(d_pose), _ptr(state), float(lr_rot), float(lr_trans),
                                _stream(stream)), self.ctx)

    def stats(self, stream=None) -> dict:
        s = vtgs_stats()
        st = vtgs_get_stats(self.ctx, ctypes.byref(s), _stream(stream))
        d = {k: int(getattr(s, k)) for k, _ in vtgs_stats._fields_}
        if st not in (VTGS_OK, VTGS_ERR_CAPACITY):
            _ok(st, self.ctx)
        return d

    STAGES = ("project_count", "scan_tiles", "emit_pairs", "tile_sort", "composite_fwd", "l1_count",
              "composite_bwd", "pose_finalize", "instantiate", "pose_adam", "keyframe_pose_grad", "ssim",
              "densify", "visibility")

    def set_work_counters(self, enable: bool):
        _ok(vtgs_set_work_counters(self.ctx, int(bool(enable))), self.ctx)

    def set_profiling(self, enable: bool):
        _ok(vtgs_set_profiling(self.ctx, int(bool(enable))), self.ctx)

    def profile(self, stream=None) -> dict:
        """{stage: (ms summed since the last call, launches)}; synchronous; resets."""
        import numpy as np
        ms = np.zeros(len(self.STAGES), dtype=np.float64)
        cnt = np.zeros(len(self.STAGES), dtype=np.int64)
        _ok(vtgs_get_profile(self.ctx, ms.ctypes.data, cnt.ctypes.data, _stream(stream)), self.ctx)
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.STAGES)}

    def check(self, stream=None):
        _ok(vtgs_check(self.ctx, _stream(stream)), self.ctx)

    def export_tiles(self, intr, stream=None):
        import numpy as np
        T = ((intr.width + 15) // 16) * ((intr.height + 15) // 16)
        start = np.zeros(T + 1, dtype=np.int64)
        P = ctypes.c_int64()
        _ok(vtgs_export_tiles(self.ctx, start.ctypes.data, None, 0, ctypes.byref(P), _stream(stream)), self.ctx)
        gid = np.zeros(max(P.value, 1), dtype=np.int32)
        _ok(vtgs_export_tiles(self.ctx, start.ctypes.data, gid.ctypes.data, P.value, ctypes.byref(P),
                              _stream(stream)), self.ctx)
        return start, gid[:P.value]

    def step_host(self, pos_rad, col_opa, view_host, intr, target_rgb_host, target_depth_host, w_color, w_depth,
                  color_mask_mode, depth_mask_mode, normalize, want, learn, out, d_col_opa, d_radius,
                  d_pose_host=None, stream=None) -> float:
        """End-to-end step with HOST targets / pose (numpy float32 arrays or pinned CPU tensors)."""
        color, depth, sil = out
        loss = ctypes.c_float()
        vp = view_host if isinstance(view_host, torch.Tensor) else torch.as_tensor(view_host, dtype=torch.float32)
        _ok(vtgs_step_host(self.ctx, _ptr(pos_rad), _ptr(col_opa), pos_rad.shape[0], _ptr(vp), intrinsics(intr),
                           _ptr(target_rgb_host), _ptr(target_depth_host), float(w_color), float(w_depth),
                           int(color_mask_mode), int(depth_mask_mode), int(normalize), int(want), int(learn[0]),
                           int(learn[1]), _ptr(color), _ptr(depth), _ptr(sil), _ptr(d_col_opa), _ptr(d_radius),
                           ctypes.addressof(loss), _ptr(d_pose_host), _stream(stream)), self.ctx)
        return float(loss.value)


    def step_host_sensor(self, pos_rad, col_opa, view_host, intr, rgb8_host, depth16_host, depth_scale, w_color,
                         w_depth, color_mask_mode, depth_mask_mode, normalize, want, learn, out, d_col_opa, d_radius,
                         d_pose_host=None, stream=None) -> float:
        """step_host with the frame as a sensor delivers it: HOST uint8 RGB [H, W, 3] and uint16 depth
        [H, W] (metres = value · depth_scale), widened to fp32 on the device (vtgs_step_host_sensor)."""
        color, depth, sil = out
        loss = ctypes.c_float()
        vp = view_host if isinstance(view_host, torch.Tensor) else torch.as_tensor(view_host, dtype=torch.float32)
        for t, dt in ((rgb8_host, torch.uint8), (depth16_host, torch.uint16)):
            if isinstance(t, torch.Tensor) and (t.dtype != dt or t.is_cuda or not t.is_contiguous()):
                raise VtgsError(VTGS_ERR_INVALID_ARG, f"step_host_sensor: expected a contiguous host {dt} tensor")
        _ok(vtgs_step_host_sensor(self.ctx, _ptr(pos_rad), _ptr(col_opa), pos_rad.shape[0], _ptr(vp),
                                  intrinsics(intr), _ptr(rgb8_host), _ptr(depth16_host), float(depth_scale),
                                  float(w_color), float(w_depth), int(color_mask_mode), int(depth_mask_mode),
                                  int(normalize), int(want), int(learn[0]), int(learn[1]), _ptr(color), _ptr(depth),
                                  _ptr(sil), _ptr(d_col_opa), _ptr(d_radius), ctypes.addressof(loss),
                                  _ptr(d_pose_host), _stream(stream)), self.ctx)
        return float(loss.value)


def measure_peaks(device: int = 0):
    """Measured FP32 FMA peak (TFLOP/s) and MUFU ex2 throughput (ops/s) of `device` (vtgs_measure_peaks)."""
    f, x = ctypes.c_double(), ctypes.c_double()
    _ok(vtgs_measure_peaks(int(device), ctypes.byref(f), ctypes.byref(x)), None)
    return f.value, x.value
