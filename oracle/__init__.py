"""CPU oracle for the view-tied splatting hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import this package.  The product package `paper_2506_02741_b200`
never imports it, and it never imports the product package: the two share no code.

This module is argument marshalling (numpy ↔ ctypes) around `oracle/vtgs_oracle.c`, whose
header lists what each function computes and which PAPER.md / SPEC.md passage it follows.
`mode="f32"` takes every decision in fp32 (the kernel's precision) and
accumulates values in fp64; `mode="f64"` is fp64 throughout (finite-difference pins).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "vtgs_oracle.c"), os.path.join(_HERE, "oracle_impl.inc")]
_LIB_PATH = os.path.join(_HERE, "libvtgs_oracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_I32 = ctypes.POINTER(ctypes.c_int32)
_U8 = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    stale = not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB_PATH) for s in _SRC)
    if force or stale:
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
               _SRC[0], "-o", _LIB_PATH + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        for m in ("f32", "f64"):
            f = getattr(lib, f"or_instantiate_{m}")
            f.restype = ctypes.c_int64
            f.argtypes = [_D, _D, _D, ctypes.c_int, _D, ctypes.c_int, ctypes.c_int, _D, ctypes.c_double, _D, _D]
            f = getattr(lib, f"or_project_{m}")
            f.restype = None
            f.argtypes = [_D, ctypes.c_int64, _D, _D, ctypes.c_int, ctypes.c_int, _D, _D, _I32, _I32]
            f = getattr(lib, f"or_tile_lists_{m}")
            f.restype = ctypes.c_int64
            f.argtypes = [_D, ctypes.c_int64, _D, _D, ctypes.c_int, ctypes.c_int, _I64, _I64, ctypes.c_int64]
            f = getattr(lib, f"or_render_{m}")
            f.restype = ctypes.c_int
            f.argtypes = [_D, _D, ctypes.c_int64, _D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                          _D, _D, _D, _D, _I32, _I32, _I64, _U8, ctypes.POINTER(ctypes.c_uint64), _I32]
            f = getattr(lib, f"or_render_bwd_{m}")
            f.restype = ctypes.c_int
            f.argtypes = [_D, _D, ctypes.c_int64, _D, _D, ctypes.c_int, ctypes.c_int, _D, _D, _D, _D, _D, _D, _D, _D, _D, _D,
                          _D]
            f = getattr(lib, f"or_visibility_{m}")
            f.restype = ctypes.c_int64
            f.argtypes = [_D, _D, _D, _D, ctypes.c_int, _D, ctypes.c_int, ctypes.c_int, ctypes.c_double, _U8]
            f = getattr(lib, f"or_keyframe_pose_grad_{m}")
            f.restype = None
            f.argtypes = [_D, _D, ctypes.c_int, _D, ctypes.c_int, ctypes.c_int, _D, _D]
        f = lib.or_densify_f32
        f.restype = ctypes.c_int64
        f.argtypes = [_D, _D, _D, _D, ctypes.c_int, ctypes.c_int, _D, ctypes.c_double, _D, ctypes.c_double, _D, _D]
        f = lib.or_pose_adam
        f.restype = None
        f.argtypes = [_D, _D, _D, ctypes.c_double, ctypes.c_double]
        f = lib.or_ssim_loss
        f.restype = ctypes.c_double
        f.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_double, _D, _D]
        f = lib.or_l1_upstream
        f.restype = ctypes.c_double
        f.argtypes = [_D, _D, _D, _D, _D, _U8, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                      ctypes.c_int, ctypes.c_int, ctypes.c_int, _D, _D, _D, _I32, ctypes.c_double, _D]
        _lib = lib
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a, t=_D):
    return None if a is None else a.ctypes.data_as(t)


def _intr(intr) -> np.ndarray:
    return _d([intr.fx, intr.fy, intr.cx, intr.cy])


def instantiate(depth, rgb, poses, intr, opacity=None, opacity_default=0.5, mode="f32"):
    """(a1) depth [K,H,W], rgb [K,H,W,3], poses [K,7] → pos_rad [N,4], col_opa [N,4], n_valid."""
    lib = _load()
    depth = _d(depth)
    K, H, W = depth.shape
    rgb, poses = _d(rgb), _d(poses).reshape(K, 7)
    opa = None if opacity is None else _d(opacity)
    N = K * H * W
    pos_rad = np.zeros((N, 4))
    col_opa = np.zeros((N, 4))
    n = getattr(lib, f"or_instantiate_{mode}")(_p(depth), _p(rgb), _p(poses), K, _p(_intr(intr)), W, H,
                                                _p(opa), float(opacity_default), _p(pos_rad), _p(col_opa))
    return pos_rad, col_opa, int(n)


def project(pos_rad, view, intr, mode="f32"):
    """(a2) → dict(proj [N,4] (u,v,z,σ), xc [N,3], rect [N,4] (x0,y0,x1,y1), status [N])."""
    lib = _load()
    pos_rad = _d(pos_rad).reshape(-1, 4)
    N = pos_rad.shape[0]
    proj = np.zeros((N, 4))
    xc = np.zeros((N, 3))
    rect = np.zeros((N, 4), dtype=np.int32)
    status = np.zeros(N, dtype=np.int32)
    getattr(lib, f"or_project_{mode}")(_p(pos_rad), N, _p(_d(view)), _p(_intr(intr)), intr.width, intr.height,
                                       _p(proj), _p(xc), _p(rect, _I32), _p(status, _I32))
    return {"proj": proj, "xc": xc, "rect": rect, "status": status}


def tile_lists(pos_rad, view, intr, mode="f32"):
    """(a3) → (tile_start [T+1] int64, gid [P] int64)."""
    lib = _load()
    pos_rad = _d(pos_rad).reshape(-1, 4)
    N = pos_rad.shape[0]
    ntiles = ((intr.width + 15) // 16) * ((intr.height + 15) // 16)
    start = np.zeros(ntiles + 1, dtype=np.int64)
    fn = getattr(lib, f"or_tile_lists_{mode}")
    P = fn(_p(pos_rad), N, _p(_d(view)), _p(_intr(intr)), intr.width, intr.height, _p(start, _I64), None, 0)
    if P < 0:
        raise MemoryError("oracle tile lists")
    gid = np.zeros(max(P, 1), dtype=np.int64)
    fn(_p(pos_rad), N, _p(_d(view)), _p(_intr(intr)), intr.width, intr.height, _p(start, _I64), _p(gid, _I64), P)
    return start, gid[:P]


def render(pos_rad, col_opa, view, intr, rows=None, mode="f32", want_tainted=False, extra_flags=None):
    """(a4) → dict(color [H,W,3], depth, sil, T_final, n_comp, flags [H,W] (bool), flag_bits [H,W]
    (1: α decision near-tie, 2: T cut-off near-tie, 4: caller-flagged), stats (E_eval,
    E_comp, P), trace [H,W] (hash of every per-pixel decision), tainted [N] bool or None).
    `rows=(r0, r1)` renders only those rows; `extra_flags` [H,W] marks further pixels flagged
    (their Gaussians are tainted too)."""
    lib = _load()
    pos_rad = _d(pos_rad).reshape(-1, 4)
    col_opa = _d(col_opa).reshape(-1, 4)
    N = pos_rad.shape[0]
    W, H = intr.width, intr.height
    r0, r1 = (0, H) if rows is None else rows
    color = np.zeros((H, W, 3))
    depth = np.zeros((H, W))
    sil = np.zeros((H, W))
    T_final = np.ones((H, W))
    n_comp = np.zeros((H, W), dtype=np.int32)
    flags = np.zeros((H, W), dtype=np.int32)
    stats = np.zeros(3, dtype=np.int64)
    tainted = np.zeros(max(N, 1), dtype=np.uint8) if want_tainted else None
    trace = np.zeros((H, W), dtype=np.uint64)
    ext = None if extra_flags is None else np.ascontiguousarray(np.asarray(extra_flags, dtype=np.int32))
    rc = getattr(lib, f"or_render_{mode}")(_p(pos_rad), _p(col_opa), N, _p(_d(view)), _p(_intr(intr)), W, H, r0, r1,
                                           _p(color), _p(depth), _p(sil), _p(T_final), _p(n_comp, _I32),
                                           _p(flags, _I32), _p(stats, _I64), _p(tainted, _U8),
                                           _p(trace, ctypes.POINTER(ctypes.c_uint64)), _p(ext, _I32))
    if rc:
        raise MemoryError("oracle render")
    if ext is not None:
        flags |= (ext != 0).astype(np.int32) << 2
    return {"color": color, "depth": depth, "sil": sil, "T_final": T_final, "n_comp": n_comp,
            "flags": flags.astype(bool), "flag_bits": flags, "stats": stats, "trace": trace,
            "tainted": None if tainted is None else tainted[:N].astype(bool)}


def render_bwd(pos_rad, col_opa, view, intr, gC=None, gD=None, gS=None, mode="f32", want_allow=False):
    """(a5) → dict(d_col_opa [N,4], d_radius [N], d_pose [7], d_geom [N,4] (du,dv,dσ,dz),
    d_abs [N,5] (Σ of |per-pixel contributions| to dc0..2, do, dr), d_pos [N,3] (dL/dX_w), d_pos_abs [N,3]
    (its Σ|terms|)[, d_allow [N,8] (T cut-off near-tie allowance: dc0..2, do, dr, dX_w)])."""
    lib = _load()
    pos_rad = _d(pos_rad).reshape(-1, 4)
    col_opa = _d(col_opa).reshape(-1, 4)
    N = pos_rad.shape[0]
    W, H = intr.width, intr.height
    gC = None if gC is None else _d(gC).reshape(H, W, 3)
    gD = None if gD is None else _d(gD).reshape(H, W)
    gS = None if gS is None else _d(gS).reshape(H, W)
    d_col_opa = np.zeros((max(N, 1), 4))
    d_rad = np.zeros(max(N, 1))
    d_pose = np.zeros(7)
    d_geom = np.zeros((max(N, 1), 4))
    d_abs = np.zeros((max(N, 1), 5))
    d_pos = np.zeros((max(N, 1), 3))
    d_pos_abs = np.zeros((max(N, 1), 3))
    d_allow = np.zeros((max(N, 1), 8)) if want_allow else None
    rc = getattr(lib, f"or_render_bwd_{mode}")(_p(pos_rad), _p(col_opa), N, _p(_d(view)), _p(_intr(intr)), W, H,
                                               _p(gC), _p(gD), _p(gS), _p(d_col_opa), _p(d_rad), _p(d_pose),
                                               _p(d_geom), _p(d_abs), _p(d_pos), _p(d_pos_abs), _p(d_allow))
    if rc:
        raise MemoryError("oracle render_bwd")
    out = {"d_col_opa": d_col_opa[:N], "d_radius": d_rad[:N], "d_pose": d_pose, "d_geom": d_geom[:N],
           "d_abs": d_abs[:N], "d_pos": d_pos[:N], "d_pos_abs": d_pos_abs[:N]}
    if want_allow:
        out["d_allow"] = d_allow[:N]
    return out


def keyframe_pose_grad(depth, poses, intr, d_pos, mode="f64"):
    """Head-frame bundle adjustment: dL/d(keyframe pose) [K,7] (dq 4, dt 3) from the
    keyframes' depth [K,H,W], poses [K,7] and dL/dX_w per slot [K*H*W,3]."""
    lib = _load()
    depth = _d(depth)
    K, H, W = depth.shape
    poses = _d(poses).reshape(K, 7)
    d_pos = _d(d_pos).reshape(K * H * W, 3)
    out = np.zeros((K, 7))
    getattr(lib, f"or_keyframe_pose_grad_{mode}")(_p(depth), _p(poses), K, _p(_intr(intr)), W, H, _p(d_pos),
                                                  _p(out))
    return out



# L1 sign near-tie band: the kernel's fp32 render differs from the oracle's fp64 values by
# ≤ 1.3e-6 on every config measured; a residual within L1_BAND of 0 may take
# the other side of sgn on the GPU.
L1_BAND = 1e-5


def l1_upstream(color, depth, sil, target_rgb, target_depth, vis=None, w_color=1.0, w_depth=0.5,
                color_mask_mode=0, depth_mask_mode=0, normalize=0, band=L1_BAND, want_flip=False):
    """Masked L1 of Eq. 1 / Eq. 2 (no SSIM) → (loss, gC [H,W,3], gD, gS, flags[, flip [H,W,4]]).
    `flip`: per near-tie (pixel, component) the largest upstream change the other sgn branch
    could cause (see or_l1_upstream)."""
    lib = _load()
    C, D, S = _d(color), _d(depth), _d(sil)
    tC, tD = _d(target_rgb), _d(target_depth)
    H, W = D.shape
    v = None if vis is None else np.ascontiguousarray(np.asarray(vis, dtype=np.uint8))
    gC = np.zeros((H, W, 3))
    gD = np.zeros((H, W))
    gS = np.zeros((H, W))
    fl = np.zeros((H, W), dtype=np.int32)
    flip = np.zeros((H, W, 4)) if want_flip else None
    loss = lib.or_l1_upstream(_p(C), _p(D), _p(S), _p(tC), _p(tD), _p(v, _U8), H * W, float(w_color),
                              float(w_depth), int(color_mask_mode), int(depth_mask_mode), int(normalize),
                              _p(gC), _p(gD), _p(gS), _p(fl, _I32), float(band), _p(flip))
    if want_flip:
        return float(loss), gC, gD, gS, fl.astype(bool), flip
    return float(loss), gC, gD, gS, fl.astype(bool)


def ssim_loss(render_rgb, target_rgb, tau=0.2, want_map=False):
    """SSIM term of Eq. 2: (τ·(1 − mean SSIM), dL/d render [H,W,3][, SSIM map])."""
    lib = _load()
    x, y = _d(render_rgb), _d(target_rgb)
    H, W, _ = x.shape
    grad = np.zeros((H, W, 3))
    smap = np.zeros((H, W, 3)) if want_map else None
    loss = lib.or_ssim_loss(_p(x), _p(y), W, H, float(tau), _p(grad), _p(smap))
    return (loss, grad, smap) if want_map else (loss, grad)


def densify(depth, rgb, pose, intr, sil, threshold=0.5, opacity=None, opacity_default=0.5):
    """Regular-frame densification: new Gaussians at valid pixels with S < threshold,
    row-major → (pos_rad [M,4], col_opa [M,4])."""
    lib = _load()
    depth = _d(depth)
    H, W = depth.shape
    rgb, sil = _d(rgb), _d(sil)
    opa = None if opacity is None else _d(opacity)
    pr = np.zeros((H * W, 4))
    co = np.zeros((H * W, 4))
    n = lib.or_densify_f32(_p(depth), _p(rgb), _p(_d(pose)), _p(_intr(intr)), W, H, _p(sil), float(threshold), _p(opa),
                           float(opacity_default), _p(pr), _p(co))
    return pr[:n], co[:n]


def visibility(depth, pose, ref_depth, ref_poses, intr, tol=0.01, mode="f32"):
    """Visibility mask of a frame (depth [H,W] at pose) to reference views (ref_depth [R,H,W],
    ref_poses [R,7]); union over the references → bool [H,W]."""
    lib = _load()
    depth = _d(depth)
    H, W = depth.shape
    ref_depth = _d(ref_depth).reshape(-1, H, W)
    R = ref_depth.shape[0]
    ref_poses = _d(ref_poses).reshape(R, 7)
    mask = np.zeros((H, W), dtype=np.uint8)
    getattr(lib, f"or_visibility_{mode}")(_p(depth), _p(_d(pose)), _p(ref_depth), _p(ref_poses), R, _p(_intr(intr)),
                                          W, H, float(tol), _p(mask, _U8))
    return mask.astype(bool)


def pose_adam(pose, grad, state, lr_rot, lr_trans):
    """One Adam step on a pose, fp64: returns (new pose [7], new state [15]); the
    state holds m[7], v[7], step (zeros = fresh)."""
    lib = _load()
    p = _d(pose).copy()
    st = _d(state).copy()
    lib.or_pose_adam(_p(p), _p(_d(grad)), _p(st), float(lr_rot), float(lr_trans))
    return p, st


def visibility_counts(depth, pose, cand_depth, cand_poses, intr, tol=0.01):
    """Per-candidate visible-point counts of a frame: for each candidate view r alone, the
    number of valid pixels of `depth` (at `pose`) visible to it (the or_visibility test with one
    reference) → (counts [R] int, n_valid)."""
    cand_depth = _d(cand_depth).reshape(-1, *np.shape(depth))
    cand_poses = _d(cand_poses).reshape(-1, 7)
    counts = [int(visibility(depth, pose, cand_depth[r:r + 1], cand_poses[r:r + 1], intr, tol).sum())
              for r in range(cand_depth.shape[0])]
    d = np.asarray(depth, dtype=np.float32)
    return counts, int(((d > 0) & np.isfinite(d)).sum())


def select_sections(counts, n_valid, cand_section, gamma, n_sections=3):
    """P:180 / S:382-387: candidates with visible fraction > γ; the most-front (earliest) 3 distinct
    sections containing one of them; none → the most recent section."""
    kept = [i for i in range(len(counts)) if n_valid > 0 and counts[i] / n_valid > gamma]
    secs = sorted(set(int(cand_section[i]) for i in kept))[:n_sections]
    return secs if secs else [max(int(s) for s in cand_section)]


def track(pos_rad, col_opa, intr, rgb, depth, init_pose, iterations, lr_rot, lr_trans, w_color=0.5, w_depth=1.0,
          vis=None):
    """Tracking of one frame (Eq. 1): `iterations` × (render at the pose → masked L1 of
    Eq. 1 with W = valid ∧ S > 0.99 ∧ vis, mean form → pose gradient → one Adam step).
    Decisions in fp32 (f32 mode); the pose is rounded to fp32 after every step (it is an fp32
    parameter).  Returns (pose [7], losses [iterations]) — losses[i] is the loss at the i-th
    iterate, before its step."""
    pose = np.asarray(init_pose, dtype=np.float32).astype(np.float64).reshape(7)
    st = np.zeros(15)
    losses = []
    for _ in range(iterations):
        img = render(pos_rad, col_opa, pose, intr)
        loss, gC, gD, gS, _ = l1_upstream(img["color"], img["depth"], img["sil"], rgb, depth, vis, w_color, w_depth,
                                          1, 1, 1)
        g = render_bwd(pos_rad, col_opa, pose, intr, gC, gD, gS)
        losses.append(loss)
        pose, st = pose_adam(pose, g["d_pose"], st, lr_rot, lr_trans)
        pose = pose.astype(np.float32).astype(np.float64)
    return pose, np.array(losses)
