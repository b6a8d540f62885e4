"""Ad-hoc GPU diagnostic (not collected by pytest): gradient error vs conditioning."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from synth.scenes import cached_config
from vtgs_testlib import gpu_instantiate, oracle_instantiate, view32
from paper_2506_02741_b200 import vtgs as vt

for which in (1, 2, 3):
    cfg = cached_config(which)
    R = vt.Renderer(0, cfg.n_slots, cfg.intr.width, cfg.intr.height)
    pr, co = gpu_instantiate(R, cfg)
    v = view32(cfg.views[0])
    vv = vt.pose_tensor(v, "cuda")
    out = R.render_fwd(pr, co, vv, cfg.intr)
    H, W = cfg.intr.height, cfg.intr.width
    rng = np.random.default_rng(which)
    gC = rng.normal(size=(H, W, 3)).astype(np.float32)
    gD = rng.normal(size=(H, W)).astype(np.float32)
    gS = rng.normal(size=(H, W)).astype(np.float32)
    dco = torch.zeros((cfg.n_slots, 4), device="cuda"); drad = torch.zeros(cfg.n_slots, device="cuda")
    dp = torch.zeros(7, device="cuda")
    R.render_bwd(vt.VTGS_GRAD_ALL, d_col_opa=dco, d_radius=drad, d_pose=dp, dL_dcolor=torch.from_numpy(gC).cuda(),
                 dL_ddepth=torch.from_numpy(gD).cuda(), dL_dsil=torch.from_numpy(gS).cuda())
    torch.cuda.synchronize()
    opr, oco = oracle_instantiate(cfg)
    ref = oracle.render(opr, oco, v, cfg.intr, want_tainted=True)
    g = oracle.render_bwd(opr, oco, v, cfg.intr, gC, gD, gS)
    keep = ~ref["tainted"]
    print(f"config {which}: pose gpu {dp.cpu().numpy()} oracle {g['d_pose']}", flush=True)
    a = np.concatenate([dco.cpu().numpy().astype(np.float64), drad.cpu().numpy()[:, None]], 1)[keep]
    b = np.concatenate([g["d_col_opa"], g["d_radius"][:, None]], 1)[keep]
    ab = g["d_abs"][keep]
    for j, name in enumerate(["dc0", "dc1", "dc2", "do", "dr"]):
        err = np.abs(a[:, j] - b[:, j])
        bar = np.maximum(1e-5, 1e-3 * np.abs(b[:, j]))
        bad = err > bar
        rel_to_abs = err / np.maximum(ab[:, j], 1e-30)
        print(f"  {name}: bad {bad.sum()}/{len(err)}  max err/Σ|terms| {rel_to_abs.max():.3e}  "
              f"p99.99 {np.quantile(rel_to_abs, 0.9999):.3e}  bad with err/Σ|t|>2e-6: {(bad & (rel_to_abs > 2e-6)).sum()}",
              flush=True)
        if bad.any():
            kappa = ab[bad, j] / np.maximum(np.abs(b[bad, j]), 1e-30)
            print(f"     bad: err/Σ|t| quantiles {np.quantile(rel_to_abs[bad], [0.5, 0.9, 0.99, 1.0])}, "
                  f"cancellation Σ|t|/|ref| quantiles {np.quantile(kappa, [0.01, 0.5, 0.9])}", flush=True)
    print(f"  flagged px {ref['flags'].sum()}  tainted {ref['tainted'].sum()}", flush=True)
