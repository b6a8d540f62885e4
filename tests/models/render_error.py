#!/usr/bin/env python
"""Measure the GPU render's deviation from the oracle (design tool, GPU + oracle).

For configs 1-3 it renders the config's view through the C ABI and with the oracle and prints,
over the pixels the oracle does not flag, max |ΔC|, |ΔD|, |ΔS| and the flag counts by kind
(bit 1: α decision near-tie, bit 2: T cut-off near-tie).  The max |ΔC|, |ΔD| bound how far the
kernel's L1 residual can sit from the oracle's — the basis of oracle.L1_BAND.
Usage: python tests/models/render_error.py [configs...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2506_02741_b200 import vtgs  # noqa: E402
from synth.scenes import cached_config  # noqa: E402
from vtgs_testlib import gpu_instantiate, oracle_instantiate, view32  # noqa: E402


def main(which_list):
    out = {}
    for which in which_list:
        cfg = cached_config(which)
        R = vtgs.Renderer(0, cfg.n_slots, cfg.intr.width, cfg.intr.height)
        pr, co = gpu_instantiate(R, cfg)
        v = view32(cfg.views[0])
        C, D, S = R.render_fwd(pr, co, vtgs.pose_tensor(v, "cuda"), cfg.intr)
        torch.cuda.synchronize()
        opr, oco = oracle_instantiate(cfg)
        ref = oracle.render(opr, oco, v, cfg.intr)
        ok = ~ref["flags"]
        dC = np.abs(C.cpu().numpy().astype(np.float64) - ref["color"])[ok]
        dD = np.abs(D.cpu().numpy().astype(np.float64) - ref["depth"])[ok]
        dS = np.abs(S.cpu().numpy().astype(np.float64) - ref["sil"])[ok]
        st = R.stats()
        rec = {"max_dC": float(dC.max()), "max_dD": float(dD.max()), "max_dS": float(dS.max()),
               "p999_dC": float(np.quantile(dC, 0.999)), "flagged_px": int(ref["flags"].sum()),
               "flag_alpha": int(((ref["flag_bits"] & 1) != 0).sum()), "flag_T": int(((ref["flag_bits"] & 2) != 0).sum()),
               "px": int(ref["flags"].size), "e_comp_gpu": st["e_comp"], "e_comp_oracle": int(ref["stats"][1]),
               "e_eval_gpu": st["e_eval"], "e_eval_oracle": int(ref["stats"][0])}
        out[which] = rec
        print(which, json.dumps(rec), flush=True)
    return out


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3])
