#!/usr/bin/env python
"""One pass of every kernel family for compute-sanitizer (memcheck / racecheck / initcheck /
synccheck): instantiate, forward (+ work counters), fused-L1 mapping backward (attribute +
deterministic merge), pose-only tracking backward, position + keyframe-pose backward, SSIM,
visibility counts, densify, pose Adam — on config `argv[1]` (1 or 2)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_02741_b200 import vtgs  # noqa: E402
from synth.scenes import make_config  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "1"
if arg == "long":   # 60,000 Gaussians in a 40×36 image: tile lists > 16,384 (chunked sort paths)
    from synth.scenes import Config, Frame, Intrinsics
    rng = np.random.Generator(np.random.PCG64([7, 3]))
    W_, H_ = 40, 36
    intr_ = Intrinsics(30.0, 30.0, (W_ - 1) / 2, (H_ - 1) / 2, W_, H_)
    depth = rng.uniform(1.0, 4.0, size=(1, H_, W_)).astype(np.float32)
    kf = Frame(depth[0], rng.random((H_, W_, 3)).astype(np.float32), np.array([1.0, 0, 0, 0, 0, 0, 0]))
    kfs = [kf] * 40
    cfg = Config("long", intr_, kfs, rng.uniform(0.01, 0.2, (40, H_, W_)).astype(np.float32),
                 [np.array([1.0, 0, 0, 0, 0.01, 0, 0])], [kf], (0.8, 1.0), "mapping", 0)
    which = "long"
else:
    which = int(arg)
    cfg = make_config(which)
intr = cfg.intr
H, W = intr.height, intr.width
N = cfg.n_slots
dev = "cuda"
R = vtgs.Renderer(0, N + H * W, W, H)
nv = torch.zeros(1, dtype=torch.int64, device=dev)
kfp = vtgs.pose_tensor(cfg.pose_stack(), dev)
pr = torch.zeros((N + H * W, 4), device=dev)
co = torch.zeros((N + H * W, 4), device=dev)
R.instantiate(torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev), kfp, intr,
              torch.from_numpy(cfg.opacity).to(dev), out=(pr[:N], co[:N]), n_valid=nv)
view = vtgs.pose_tensor(np.asarray(cfg.views[0], dtype=np.float32), dev)
tg = cfg.targets[0]
L = dict(target_rgb=torch.from_numpy(tg.rgb).to(dev), target_depth=torch.from_numpy(tg.depth).to(dev),
         w_color=cfg.loss_weights[0], w_depth=cfg.loss_weights[1])
dco = torch.zeros((N, 4), device=dev)
drad = torch.zeros(N, device=dev)
dpos = torch.zeros((N, 4), device=dev)
dpose = torch.zeros(7, device=dev)
loss = torch.zeros(1, device=dev)
C, D, S = R.render_fwd(pr[:N], co[:N], view, intr, N=N)
R.render_bwd(vtgs.VTGS_GRAD_ATTR, d_col_opa=dco, d_radius=drad, loss=L, loss_out=loss)
R.render_bwd(vtgs.VTGS_GRAD_ATTR | vtgs.VTGS_GRAD_DETERMINISTIC, d_col_opa=dco, d_radius=drad, loss=L)
R.render_bwd(vtgs.VTGS_GRAD_POSE, d_pose=dpose, loss=dict(L, color_mask_mode=1, depth_mask_mode=1, normalize=1))
R.render_bwd(vtgs.VTGS_GRAD_POSITION | vtgs.VTGS_GRAD_POSE, d_position=dpos, d_pose=dpose,
             dL_dcolor=torch.randn((H, W, 3), device=dev), dL_ddepth=torch.randn((H, W), device=dev))
kf = R.keyframe_pose_grad(pr[:N], dpos, kfp, H * W)
dss = torch.zeros((H, W, 3), device=dev)
R.ssim_loss(C, L["target_rgb"], 0.2, d_color=dss)
R.visibility_counts(L["target_depth"], view, torch.from_numpy(cfg.depth_stack()).to(dev), kfp, intr)
R.visibility_mask(L["target_depth"], view, torch.from_numpy(cfg.depth_stack()[:1]).to(dev), kfp[:1], intr)
n_new = R.densify(L["target_depth"], L["target_rgb"], view, intr, S, pr[N:], co[N:])
state = torch.zeros(16, device=dev)
R.pose_adam_step(view, dpose, state, 0.002, 0.002)
torch.cuda.synchronize()
R.check()
print(f"sanitize pass ok: config {which}, n_valid {int(nv.item())}, loss {loss.item():.4f}, densified {n_new}")
