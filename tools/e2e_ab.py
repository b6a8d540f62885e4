"""Probe: the e2e step through vtgs_step_host (fp32 targets) vs vtgs_step_host_sensor (uint8 RGB +
uint16 depth), alternated, wall time per step (the bench's e2e method)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_02741_b200 import vtgs
from synth.scenes import make_config
cfg = make_config(2, 0)
dev = torch.device("cuda", 0)
N = cfg.n_slots
R = vtgs.Renderer(0, N, cfg.intr.width, cfg.intr.height)
pr, co = R.instantiate(torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev),
                       vtgs.pose_tensor(cfg.pose_stack(), dev), cfg.intr, torch.from_numpy(cfg.opacity).to(dev))
R.set_work_counters(False)
kf = cfg.keyframes[2]
hv = torch.from_numpy(np.asarray(kf.pose, dtype=np.float32).reshape(7).copy()).pin_memory()
hr, hd = torch.from_numpy(kf.rgb).pin_memory(), torch.from_numpy(kf.depth).pin_memory()
sc = np.float32(1 / 5000)
sr = torch.from_numpy(np.clip(np.rint(kf.rgb * 255), 0, 255).astype(np.uint8)).pin_memory()
sd = torch.from_numpy(np.clip(np.rint(kf.depth / sc), 0, 65535).astype(np.uint16)).pin_memory()
H, W = cfg.intr.height, cfg.intr.width
out = (torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev), torch.empty((H, W), device=dev))
g = torch.zeros(5 * N, device=dev)
d_co, d_r = g[:4 * N].view(N, 4), g[4 * N:]
want = vtgs.VTGS_GRAD_ATTR
def f32():
    g.zero_()
    R.step_host(pr, co, hv, cfg.intr, hr, hd, 0.8, 1.0, 0, 0, 0, want, (0, N), out, d_co, d_r)
def sen():
    g.zero_()
    R.step_host_sensor(pr, co, hv, cfg.intr, sr, sd, float(sc), 0.8, 1.0, 0, 0, 0, want, (0, N), out, d_co, d_r)
def t(fn, n=100):
    for _ in range(20): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3 / n
for rep in range(3):
    print(f"rep {rep}: fp32 {t(f32):.3f} ms  sensor {t(sen):.3f} ms")
