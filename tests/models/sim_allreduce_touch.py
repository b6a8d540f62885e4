"""Offline check of the keyframe-chunked sparse all-reduce on config 5: which keyframes
each of the 16 mapping views touches (any slot visible, oracle projection), and the union over each
rank's view shard at N = 2, 4, 8 -- the chunks no rank touches are the only ones the sparse
all-reduce could skip."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
from synth.scenes import make_config
from paper_2506_02741_b200.mapping import shard_views
cfg = make_config(5, 0); intr = cfg.intr
pr, co, _ = oracle.instantiate(cfg.depth_stack(), cfg.rgb_stack(), cfg.pose_stack(), intr, cfg.opacity)
K = cfg.K; spk = intr.width * intr.height
touched = []
for vi, v in enumerate(cfg.views[:16]):
    view = np.asarray(v, dtype=np.float32).astype(np.float64)
    p = oracle.project(pr, view, intr)
    vis = p["status"] != 0
    kt = np.array([vis[k * spk:(k + 1) * spk].any() for k in range(K)])
    frac = np.array([vis[k * spk:(k + 1) * spk].mean() for k in range(K)])
    touched.append(kt)
    print(vi, "keyframes touched", kt.sum(), "visible slots", vis.mean().round(3), flush=True)
T = np.array(touched)
for n in (2, 4, 8):
    union = np.zeros(K, bool)
    for r in range(n):
        u = T[shard_views(len(cfg.views), n, r)].any(0)
        union |= u
    print("N", n, "union of touched keyframes", union.sum(), "of", K)
