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


def flip_allowance(opr, oco, view, intr, flip):
    """Per-Gaussian allowance for the L1 loss's sgn near-ties: for each upstream
    component c (3 colour channels, depth) the oracle's backward run on the flip weights of c
    alone gives Σ_p |Δg_c(p)|·|∂(gradient)/∂g_c(p)| in its Σ|terms| outputs — an upper bound on
    how much the gradient of each Gaussian can move when the kernel's fp32 render puts a near-tie
    residual on the other side of 0.  → dict(d_col_opa [N,4], d_radius [N], d_pos [N,3])."""
    H, W = intr.height, intr.width
    N = opr.reshape(-1, 4).shape[0]
    out = {"d_col_opa": np.zeros((N, 4)), "d_radius": np.zeros(N), "d_pos": np.zeros((N, 3))}
    for c in range(4):
        fc = flip[..., c]
        if not fc.any():
            continue
        gC = np.zeros((H, W, 3))
        gD = np.zeros((H, W))
        if c < 3:
            gC[..., c] = fc
        else:
            gD[:] = fc
        g = oracle.render_bwd(opr, oco, view, intr, gC, gD, None)
        out["d_col_opa"] += g["d_abs"][:, :4]
        out["d_radius"] += g["d_abs"][:, 4]
        out["d_pos"] += g["d_pos_abs"]
    return out


# Parity exclusions (tainted by a decision flag, or passing only through the sgn allowance) are
# reported by every gradient check and capped at this fraction of the Gaussians.
EXCLUDED_CAP = 5e-3


def combine_allow(g, flip_allow=None):
    """The per-Gaussian allowance of a gradient check: the oracle's T cut-off near-tie allowance
    (render_bwd(..., want_allow=True)["d_allow"]) plus, for a fused L1 loss, the sgn near-tie
    allowance (flip_allowance).  → dict(d_col_opa [N,4], d_radius [N], d_pos [N,3])."""
    al = g["d_allow"]
    out = {"d_col_opa": al[:, :4].copy(), "d_radius": al[:, 4].copy(), "d_pos": al[:, 5:8].copy()}
    if flip_allow is not None:
        for k in out:
            out[k] += flip_allow[k]
    return out


def check_grads(vt, want, dco, drad, dpose, g, tainted, allow=None, learn=None, name="", cap=EXCLUDED_CAP,
                floor_cap=(5, 1e-5)):
    """North_star gradient bar on every Gaussian: within 1e-3 relative or 1e-5 absolute, or the
    fp32 summation floor of a cancelling sum (R23, counted and capped), or — only for Gaussians
    at a near-tie the kernel may decide the other way (T cut-off, L1 sgn) — within that
    near-tie's allowance plus the bar.  Gaussians evaluated at a pixel with an α-decision
    near-tie are excluded (tainted).  Excluded + allowance-only Gaussians are printed and must
    stay below `cap` of the Gaussians with a gradient.  Returns the counts."""
    N = len(tainted)
    keep = ~tainted
    if learn is not None:
        lo, hi = learn
        idx = np.arange(N)
        outside = (idx < lo) | (idx >= hi)
        assert not dco[outside].any() and not drad[outside].any()
        keep &= ~outside
    touched = (np.abs(g["d_abs"]).sum(1) > 0)
    allow_only = np.zeros(N, dtype=bool)

    def _one(label, gpu, ref, absum, al):
        st = {}
        ok = close(gpu, ref, absum=absum, stats=st)
        if al is not None:   # the near-tie's largest effect, plus the ordinary bar on the rest
            a_ok = np.abs(gpu - ref) <= al + np.maximum(1e-5, 1e-3 * np.abs(ref))
            extra = a_ok & ~ok
            ok = ok | a_ok
            if extra.ndim > 1:
                extra = extra.any(1)
            allow_only[np.nonzero(keep)[0][extra]] = True
        assert ok.all(), report(label, ok, gpu, ref)
        assert st["floor_only"] <= floor_cap[0] + floor_cap[1] * st["n"], (label, st)

    if want & (vt.VTGS_GRAD_COLOR | vt.VTGS_GRAD_OPACITY):
        _one("d_col_opa", dco[keep], g["d_col_opa"][keep], g["d_abs"][keep, :4],
             None if allow is None else allow["d_col_opa"][keep])
    if want & vt.VTGS_GRAD_RADIUS:
        _one("d_radius", drad[keep], g["d_radius"][keep], g["d_abs"][keep, 4],
             None if allow is None else allow["d_radius"][keep])
    n_t = int((tainted & touched).sum())
    n_a = int(allow_only.sum())
    n_touched = max(int(touched.sum()), 1)
    frac = (n_t + n_a) / n_touched
    print(f"[parity {name}] Gaussians with a gradient: {n_touched}; tainted (decision near-tie): {n_t}; "
          f"sgn-allowance only: {n_a}; excluded fraction {frac:.2e} (cap {cap:.0e})")
    assert frac <= cap, f"{name}: excluded fraction {frac:.3e} > {cap}"
    if want & vt.VTGS_GRAD_POSE and dpose is not None:
        ref = g["d_pose"]
        err = np.linalg.norm(dpose - ref)
        assert err <= 1e-3 * np.linalg.norm(ref), f"d_pose gpu={dpose} oracle={ref}"
    return {"touched": n_touched, "tainted": n_t, "allow_only": n_a, "frac": frac}
