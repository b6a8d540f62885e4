"""Helpers shared by the GPU parity tests (test infrastructure; may call the oracle)."""
from __future__ import annotations

import numpy as np

import oracle


def gpu_instantiate(R, cfg, device="cuda"):
    """Instantiate cfg's keyframes on the GPU through the C ABI → (pos_rad, col_opa) tensors."""
    import torch
    from paper_2506_02741_b200 import vtgs
    depth = torch.from_numpy(cfg.depth_stack()).to(device)
    rgb = torch.from_numpy(cfg.rgb_stack()).to(device)
    poses = vtgs.pose_tensor(cfg.pose_stack(), device)
    opa = torch.from_numpy(cfg.opacity).to(device)
    return R.instantiate(depth, rgb, poses, cfg.intr, opa)


def oracle_instantiate(cfg, mode="f32"):
    pr, co, n = oracle.instantiate(cfg.depth_stack(), cfg.rgb_stack(), cfg.pose_stack(), cfg.intr, cfg.opacity,
                                   mode=mode)
    return pr, co


def view32(pose) -> np.ndarray:
    """The fp32 pose both sides receive."""
    return np.asarray(pose, dtype=np.float32).astype(np.float64)


FP32_SUM_FLOOR = 16 * 2.0 ** -24


def close(gpu: np.ndarray, ref: np.ndarray, rtol=1e-3, atol=1e-5, absum=None, stats=None):
    """Elementwise 'within rtol relative OR atol absolute' (north_star gradient bar).

    `absum` (oracle: Σ of |per-pixel contributions| of each sum) enables the fp32 summation
    floor of DESIGN.md §3 reading R23: an element whose sum cancels by κ = Σ|t|/|ref| ≫ 1e3
    cannot be resolved to 1e-3 relative by ANY fp32 evaluation; it passes if
    |Δ| ≤ 16·2⁻²⁴·Σ|t|.  `stats` (dict) receives how many elements needed that clause."""
    err = np.abs(gpu - ref)
    ok = err <= np.maximum(atol, rtol * np.abs(ref))
    if absum is not None:
        floor_ok = err <= FP32_SUM_FLOOR * absum
        if stats is not None:
            stats["floor_only"] = int((floor_ok & ~ok).sum())
            stats["n"] = int(ok.size)
        ok = ok | floor_ok
    return ok


def report(name, ok: np.ndarray, gpu, ref):
    bad = np.argwhere(~ok)
    msg = f"{name}: {int((~ok).sum())} / {ok.size} outside tolerance"
    if len(bad):
        i = tuple(bad[0])
        msg += f"; first at {i}: gpu={gpu[i]!r} oracle={ref[i]!r}"
    return msg
