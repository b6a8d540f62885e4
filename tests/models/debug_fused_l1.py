#!/usr/bin/env python
"""Debug aid (GPU + oracle): the fused-L1 config-2 backward's outliers — for each Gaussian outside
the gradient bar, the residual signs (GPU render vs oracle render) and flags in its 7×7 window."""
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
from vtgs_testlib import close, flip_allowance, gpu_instantiate, oracle_instantiate, view32  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = cached_config(which)
intr = cfg.intr
R = vtgs.Renderer(0, cfg.n_slots, intr.width, intr.height)
pr, co = gpu_instantiate(R, cfg)
v = view32(cfg.views[0])
vt_ = vtgs.pose_tensor(v, "cuda")
C, D, S = R.render_fwd(pr, co, vt_, intr)
tg = cfg.targets[0]
wc, wd = cfg.loss_weights
dco = torch.zeros((cfg.n_slots, 4), device="cuda")
drad = torch.zeros(cfg.n_slots, device="cuda")
R.render_bwd(vtgs.VTGS_GRAD_ATTR, d_col_opa=dco, d_radius=drad, loss=dict(
    target_rgb=torch.from_numpy(tg.rgb).cuda(), target_depth=torch.from_numpy(tg.depth).cuda(), w_color=wc,
    w_depth=wd))
torch.cuda.synchronize()
Cg, Dg = C.cpu().numpy().astype(np.float64), D.cpu().numpy().astype(np.float64)
opr, oco = oracle_instantiate(cfg)
img = oracle.render(opr, oco, v, intr, want_tainted=True)
loss, gC, gD, gS, lfl, flip = oracle.l1_upstream(img["color"], img["depth"], img["sil"], tg.rgb, tg.depth, None, wc,
                                                 wd, 0, 0, 0, want_flip=True)
g = oracle.render_bwd(opr, oco, v, intr, gC, gD, gS)
allow = flip_allowance(opr, oco, v, intr, flip)
a = dco.cpu().numpy().astype(np.float64)
keep = ~img["tainted"]
ok = close(a, g["d_col_opa"], absum=g["d_abs"][:, :4]) | (np.abs(a - g["d_col_opa"]) <= allow["d_col_opa"])
bad = np.nonzero(~ok.all(1) & keep)[0]
print("outliers", len(bad), "flip px", int(lfl.sum()), "flagged px", int(img["flags"].sum()))
p = oracle.project(opr, v, intr)
sgn_g = np.sign(Cg - tg.rgb)
sgn_o = np.sign(img["color"] - tg.rgb)
sgnD_g = np.sign(Dg - tg.depth) * (tg.depth > 0)
sgnD_o = np.sign(img["depth"] - tg.depth) * (tg.depth > 0)
mism = (sgn_g != sgn_o).any(2) | (sgnD_g != sgnD_o)
print("sign mismatches (gpu vs oracle render):", int(mism.sum()), "of which flagged:", int((mism & lfl).sum()),
      "at decision-flagged px:", int((mism & img["flags"]).sum()))
ys, xs = np.nonzero(mism & ~lfl & ~img["flags"])
for y, x in list(zip(ys, xs))[:10]:
    print(" unflagged mismatch px", (x, y), "C gpu", Cg[y, x], "C or", img["color"][y, x], "tC", tg.rgb[y, x],
          "D gpu", Dg[y, x], "D or", img["depth"][y, x], "tD", tg.depth[y, x])
for gid in bad[:5]:
    u, vv = p["proj"][gid, :2]
    print("gid", gid, "gpu", a[gid], "or", g["d_col_opa"][gid], "allow", allow["d_col_opa"][gid], "uv", u, vv)
