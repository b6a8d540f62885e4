"""Probe: config 2 mapping step eager vs captured in one CUDA graph (launch gaps), device events."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_02741_b200 import vtgs
from paper_2506_02741_b200.mapping import BatchedMapper
from synth.scenes import make_config
cfg = make_config(2, 0)
dev = torch.device("cuda", 0)
R = vtgs.Renderer(0, cfg.n_slots, cfg.intr.width, cfg.intr.height)
pr, co = R.instantiate(torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev),
                       vtgs.pose_tensor(cfg.pose_stack(), dev), cfg.intr, torch.from_numpy(cfg.opacity).to(dev))
kf = cfg.keyframes[2]
m = BatchedMapper(R, pr, co, cfg.intr, [vtgs.pose_tensor(np.asarray(kf.pose, dtype=np.float32), dev)],
                  [dict(rgb=torch.from_numpy(kf.rgb).to(dev), depth=torch.from_numpy(kf.depth).to(dev))], 0.8, 1.0)
R.set_work_counters(False)
s = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, device=dev)
def timeit(fn, n=50):
    ts = []
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s)
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts)
with torch.cuda.stream(s):
    for _ in range(3): m.step(allreduce=False)
    torch.cuda.synchronize()
    eager = timeit(lambda: m.step(allreduce=False))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        m.step(allreduce=False)
    g.replay(); torch.cuda.synchronize()
    graph = timeit(g.replay)
    lg = m.loss.clone(); m.step(allreduce=False); torch.cuda.synchronize()
print(f"eager {eager:.4f} ms  graph {graph:.4f} ms  (loss eager {m.loss.item():.4f} graph {lg.item():.4f})")
with torch.cuda.stream(s):
    R.set_profiling(True); R.profile()
    prof_on = timeit(lambda: m.step(allreduce=False))
    R.set_profiling(False); R.profile()
    prof_off = timeit(lambda: m.step(allreduce=False))
print(f"eager with per-kernel events {prof_on:.4f} ms, without {prof_off:.4f} ms")
