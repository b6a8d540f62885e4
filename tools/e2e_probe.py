"""Probe: where the end-to-end (vtgs_step_host, host buffers) step spends its wall time."""
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
H, W = cfg.intr.height, cfg.intr.width
out = (torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev), torch.empty((H, W), device=dev))
d_co = torch.zeros((N, 4), device=dev); d_r = torch.zeros(N, device=dev)
want = vtgs.VTGS_GRAD_ATTR
def step():
    return R.step_host(pr, co, hv, cfg.intr, hr, hd, 0.8, 1.0, 0, 0, 0, want, (0, N), out, d_co, d_r)
for _ in range(3): step()
torch.cuda.synchronize()
n = 30
t0 = time.perf_counter()
for _ in range(n): step()
t1 = time.perf_counter()
print(f"step_host wall {1e3 * (t1 - t0) / n:.3f} ms/step")
# host-side cost of one call when the GPU is idle vs the device time
ts = []
for _ in range(n):
    a = time.perf_counter(); step(); ts.append(time.perf_counter() - a)
print(f"per-call wall median {1e3 * np.median(ts):.3f} ms")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(); step(); ev[1].record(); torch.cuda.synchronize()
print(f"device time of one call {ev[0].elapsed_time(ev[1]):.3f} ms")
grads = torch.zeros(5 * N, device=dev)
d_co2, d_r2 = grads[:4 * N].view(N, 4), grads[4 * N:]
def step2():
    grads.zero_()
    return R.step_host(pr, co, hv, cfg.intr, hr, hd, 0.8, 1.0, 0, 0, 0, want, (0, N), out, d_co2, d_r2)
for _ in range(5): step2()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n): step2()
torch.cuda.synchronize()
print(f"zero + step_host wall {1e3 * (time.perf_counter() - t0) / n:.3f} ms/step")
