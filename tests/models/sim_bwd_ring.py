#!/usr/bin/env python
"""Offline model of the backward's phase-1 lane utilisation (design tool, uses the oracle).

Same sample of sub-tiles of config 2 as tests/models/sim_batches.py (shape sw × 32/sw, argv[2]).  Per pixel the phase-1
candidates are the entries at sub-list positions < its `last` whose rect and 3σ disc contain it,
walked back to front.  Compared: the lock-step walk per 32-entry batch (today's k_composite_bwd)
and a ring of 32-entry batches whose (pixel, entry) pair storage is a circular buffer of C pairs
(at most R batches resident): a lane walks across batch boundaries at its own pace; a batch is
released (its phase 2 run) once every live lane has passed it.  Reported: warp steps of phase 1,
lane efficiency = Σ candidates / 32 / steps, and the pair count per batch (phase-2 work).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
from synth.scenes import cached_config  # noqa: E402


def main(n_sub=300, seed=0, sw=8):
    sh = 32 // sw   # sub-tile shape sw × sh (4×8 built; 8×4 the round-1 shape; 2×16 modelled)
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
    confs = [(R, C) for R in (4,) for C in (1 << 20,)]
    steps = {c: 0 for c in confs}
    lock = 0
    wins = [(2, 1024), (4, 1024), (4, 2048), (8, 2048)]
    lockw = {w: 0 for w in wins}
    ideal = 0.0
    pairs_per_batch = []
    for _ in range(n_sub):
        t = rng.integers(T)
        s = rng.integers(8)
        ty, tx = divmod(int(t), ntx)
        sx, sy = tx * 16 + (s % (16 // sw)) * sw, ty * 16 + (s // (16 // sw)) * sh
        lst = gid[start[t]:start[t + 1]]
        r = rect[lst]
        ov = (r[:, 0] <= sx + sw - 1) & (r[:, 2] >= sx) & (r[:, 1] <= sy + sh - 1) & (r[:, 3] >= sy)
        sub = lst[ov]
        if len(sub) == 0:
            continue
        u, v, z, sg = proj[sub].T
        rr = rect[sub]
        o = co[sub, 3]
        bits = np.zeros((32, len(sub)), dtype=bool)
        for lane in range(32):
            x, y = sx + (lane % sw), sy + (lane // sw)
            if x >= intr.width or y >= intr.height:
                continue
            inr = (rr[:, 0] <= x) & (rr[:, 2] >= x) & (rr[:, 1] <= y) & (rr[:, 3] >= y)
            d2 = (x - u) ** 2 + (y - v) ** 2
            el = inr & (d2 <= 9 * sg * sg)
            a = np.minimum(o * np.exp(-0.5 * d2 / (sg * sg)), 0.999)
            Tcur = 1.0
            last = 0
            for k in np.nonzero(el)[0]:
                if a[k] < 1 / 255:
                    continue
                Tn = Tcur * (1 - a[k])
                if Tn < 1e-4:
                    break
                Tcur = Tn
                last = k + 1
            bits[lane, :last] = el[:last]
        n = bits.shape[1]
        nb = (n + 31) // 32
        wmax = max([np.nonzero(bits[l])[0].max() + 1 if bits[l].any() else 0 for l in range(32)])
        nb = (wmax + 31) // 32
        ideal += bits.sum() / 32
        bp = [int(bits[:, 32 * b:32 * b + 32].sum()) for b in range(nb)]
        pairs_per_batch += bp
        for b in range(nb):
            lock += bits[:, 32 * b:32 * b + 32].sum(1).max()
        # lock-step over windows of up to 4 batches whose pairs fit in C (back to front)
        for (Wn, Cw) in wins:
            b = nb - 1
            while b >= 0:
                lo_b, tot = b, bp[b]
                while b - (lo_b - 1) < Wn and lo_b - 1 >= 0 and tot + bp[lo_b - 1] <= Cw:
                    lo_b -= 1
                    tot += bp[lo_b]
                lockw[(Wn, Cw)] += bits[:, 32 * lo_b:32 * b + 32].sum(1).max()
                b = lo_b - 1
        # back to front: batch order nb-1 .. 0 ; per lane sequence of (batch) of its candidates
        seqs = [[k // 32 for k in np.nonzero(bits[l])[0][::-1]] for l in range(32)]
        for (R, C) in confs:
            ptr = [0] * 32
            built = []   # resident batches (descending index), oldest first
            nextb = nb - 1
            st = 0
            while True:
                live = [l for l in range(32) if ptr[l] < len(seqs[l])]
                if not live:
                    break
                # release batches every live lane has passed (lane's current batch < batch)
                cur_min_b = max(seqs[l][ptr[l]] for l in live)   # highest batch still needed
                built = [b for b in built if b <= cur_min_b]
                # build while room
                while nextb >= 0 and len(built) < R and sum(bp[b] for b in built) + bp[nextb] <= C:
                    built.append(nextb)
                    nextb -= 1
                lowest = min(built) if built else nb
                for l in live:
                    if seqs[l][ptr[l]] >= lowest:
                        ptr[l] += 1
                st += 1
            steps[(R, C)] += st
    print(f"ideal warp steps {ideal:.0f}; lock-step per batch {lock}  eff {ideal / lock:.2f}")
    pb = np.array(pairs_per_batch)
    print(f"pairs per batch: mean {pb.mean():.0f}  p99 {np.percentile(pb, 99):.0f}  max {pb.max()}")
    for w in wins:
        print(f"lock-step window <= {w[0]} batches, <= {w[1]} pairs: steps {lockw[w]:8d}  eff {ideal / lockw[w]:.2f}")
    for c in confs:
        print(f"ring R={c[0]:2d} C={c[1]:5d}: steps {steps[c]:8d}  eff {ideal / steps[c]:.2f}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 300, 0, int(sys.argv[2]) if len(sys.argv) > 2 else 8)
