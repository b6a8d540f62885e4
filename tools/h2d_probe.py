"""Probe: pinned host→device copy bandwidth of the e2e leg's 13 MB of targets, alone and while the
mapping step's kernels run (is the upload hidden under projection / sort / forward?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
dev = torch.device("cuda", 0)
n = 1200 * 680 * 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device=dev)
for _ in range(5):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"H2D {n * 4 / 1e6:.1f} MB: {ms:.3f} ms = {n * 4 / ms / 1e6:.1f} GB/s")
