#!/usr/bin/env python
"""Offline model (design tool, uses the oracle): lane utilisation of 'balanced lock-step'
batches — per 32-entry batch of a region's list, the region's pixels (with their candidate
counts in the batch) are split into 32 contiguous lane ranges by prefix sums; the warp runs
max-over-lanes(Σ candidates) iterations plus one state swap per (lane, pixel)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
from synth.scenes import cached_config  # noqa: E402


def main(n_tiles=60, seed=0):
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
    res = {}
    for (RW, RH) in [(8, 4), (16, 8), (16, 16)]:
        ideal = it = sw = 0
        for _ in range(n_tiles):
            t = int(rng.integers(T))
            ty, tx = divmod(t, ntx)
            ox = tx * 16 + (rng.integers(16 // RW) * RW if RW < 16 else 0)
            oy = ty * 16 + (rng.integers(16 // RH) * RH if RH < 16 else 0)
            lst = gid[start[t]:start[t + 1]]
            r = rect[lst]
            ov = (r[:, 0] <= ox + RW - 1) & (r[:, 2] >= ox) & (r[:, 1] <= oy + RH - 1) & (r[:, 3] >= oy)
            sub = lst[ov]
            if len(sub) == 0:
                continue
            u, v, z, sg = proj[sub].T
            rr = rect[sub]
            o = co[sub, 3]
            npx = RW * RH
            bits = np.zeros((npx, len(sub)), dtype=bool)
            for pi in range(npx):
                x, y = ox + pi % RW, oy + pi // RW
                if x >= intr.width or y >= intr.height:
                    continue
                inr = (rr[:, 0] <= x) & (rr[:, 2] >= x) & (rr[:, 1] <= y) & (rr[:, 3] >= y)
                d2 = (x - u) ** 2 + (y - v) ** 2
                el = inr & (d2 <= 9 * sg * sg)
                a = np.minimum(o * np.exp(-0.5 * d2 / (sg * sg)), 0.999)
                Tc = 1.0
                for k in np.nonzero(el)[0]:
                    bits[pi, k] = True
                    if a[k] < 1 / 255:
                        continue
                    Tn = Tc * (1 - a[k])
                    if Tn < 1e-4:
                        break
                    Tc = Tn
            ideal += bits.sum() / 32
            for b0 in range(0, len(sub), 32):
                c = bits[:, b0:b0 + 32].sum(1)
                tot = c.sum()
                if tot == 0:
                    continue
                if npx == 32:
                    it += c.max()
                    continue
                # contiguous split of pixels into 32 lanes by prefix sums
                pre = np.cumsum(c) - c
                owner = np.minimum(31, (pre * 32) // max(tot, 1))
                load = np.bincount(owner, weights=c, minlength=32)
                it += load.max()
                sw += np.bincount(owner[c > 0], minlength=32).max()
        res[(RW, RH)] = (ideal, it, sw)
        print(f"region {RW}x{RH}: lane efficiency {ideal / it:.2f}; max pixel switches per lane/batch summed {sw} "
              f"(vs iterations {it:.0f})")


if __name__ == "__main__":
    main()
