#!/usr/bin/env python
"""Dump one config's forward outputs (colour, depth, silhouette, T_final-free) to an npz — a
debugging aid for comparing kernel variants (VTGS_FWD=...) offline against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_02741_b200 import vtgs  # noqa: E402
from synth.scenes import cached_config  # noqa: E402


def main(which=2, out="gpurun_out/fwd.npz"):
    cfg = cached_config(which)
    R = vtgs.Renderer(0, cfg.n_slots, cfg.intr.width, cfg.intr.height)
    dev = "cuda"
    pr, co = R.instantiate(torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev),
                           vtgs.pose_tensor(cfg.pose_stack(), dev), cfg.intr, torch.from_numpy(cfg.opacity).to(dev))
    v = vtgs.pose_tensor(np.asarray(cfg.views[0], dtype=np.float32).astype(np.float64), dev)
    C, D, S = R.render_fwd(pr, co, v, cfg.intr)
    torch.cuda.synchronize()
    st = R.stats()
    np.savez_compressed(out, color=C.cpu().numpy(), depth=D.cpu().numpy(), sil=S.cpu().numpy(),
                        e_eval=st["e_eval"], e_comp=st["e_comp"])
    print(out, st)


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2])
