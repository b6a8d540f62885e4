#!/usr/bin/env python
"""Offline model of the compositing kernels' lane utilisation (design tool, uses the oracle).

For a sample of 8×4 sub-tiles of config 2 it builds the sub-lists, each pixel's candidate
entries (rect ∋ pixel ∧ d² ≤ 9σ²) and its termination position, then reports, for several
batch-window sizes W, the warp iterations Σ_windows max_lanes(#candidates in window) against
the ideal Σ_lanes #candidates / 32.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
from synth.scenes import cached_config  # noqa: E402


def main(n_sub=200, seed=0):
    cfg = cached_config(2)
    intr = cfg.intr
    pr, co, _ = oracle.instantiate(cfg.depth_stack(), cfg.rgb_stack(), cfg.pose_stack(), intr, cfg.opacity)
    view = np.asarray(cfg.views[0], dtype=np.float32).astype(np.float64)
    start, gid = oracle.tile_lists(pr, view, intr)
    p = oracle.project(pr, view, intr)
    proj, rect = p["proj"], p["rect"]
    ntx = (intr.width + 15) // 16
    T = len(start) - 1
    rng = np.random.default_rng(seed)
    Ws = [32, 256, 320, 384, 448, 512, 100000]
    it = {W: 0 for W in Ws}
    Hs = []
    ring = {H: 0 for H in Hs}
    ideal = 0
    cands = []
    for _ in range(n_sub):
        t = rng.integers(T)
        s = rng.integers(8)
        ty, tx = divmod(int(t), ntx)
        sx, sy = tx * 16 + (s & 1) * 8, ty * 16 + (s >> 1) * 4
        lst = gid[start[t]:start[t + 1]]
        r = rect[lst]
        ov = (r[:, 0] <= sx + 7) & (r[:, 2] >= sx) & (r[:, 1] <= sy + 3) & (r[:, 3] >= sy)
        sub = lst[ov]
        if len(sub) == 0:
            continue
        u, v, z, sg = proj[sub].T
        rr = rect[sub]
        o = co[sub, 3]
        bits = np.zeros((32, len(sub)), dtype=bool)
        for lane in range(32):
            x, y = sx + (lane & 7), sy + (lane >> 3)
            if x >= intr.width or y >= intr.height:
                continue
            inr = (rr[:, 0] <= x) & (rr[:, 2] >= x) & (rr[:, 1] <= y) & (rr[:, 3] >= y)
            d2 = (x - u) ** 2 + (y - v) ** 2
            el = inr & (d2 <= 9 * sg * sg)
            a = np.minimum(o * np.exp(-0.5 * d2 / (sg * sg)), 0.999)
            Tcur = 1.0
            for k in np.nonzero(el)[0]:
                bits[lane, k] = True
                if a[k] < 1 / 255:
                    continue
                Tn = Tcur * (1 - a[k])
                if Tn < 1e-4:
                    break
                Tcur = Tn
        n_l = bits.sum(1)
        ideal += n_l.sum() / 32
        cands.append(n_l.mean())
        for W in Ws:
            for b0 in range(0, len(sub), W):
                it[W] += bits[:, b0:b0 + W].sum(1).max()
        # ring of two halves of H entries: a lane may run ahead into the next half; a half is
        # refilled once every unfinished lane has left it
        seqs = [list(np.nonzero(bits[l])[0]) for l in range(32)]
        for H in Hs:
            ptr = [0] * 32
            steps = 0
            while True:
                live = [l for l in range(32) if ptr[l] < len(seqs[l])]
                if not live:
                    break
                lo = min(seqs[l][ptr[l]] for l in live) // H
                limit = (lo + 2) * H
                moved = False
                for l in live:
                    if seqs[l][ptr[l]] < limit:
                        ptr[l] += 1
                        moved = True
                steps += 1
            ring[H] += steps
    print(f"mean candidates/pixel {np.mean(cands):.1f}; ideal warp-iterations {ideal:.0f}")
    for W in Ws:
        print(f"W={W:6d}: warp-iterations {it[W]:8d}  lane efficiency {ideal / it[W]:.2f}")
    for H in Hs:
        print(f"ring 2x{H}: warp-iterations {ring[H]:8d}  lane efficiency {ideal / ring[H]:.2f}")


if __name__ == "__main__":
    main()
