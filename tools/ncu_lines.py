#!/usr/bin/env python
"""Per-CUDA-source-line instruction and stall shares of one kernel launch in an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]
skip = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                               "--launch-skip", skip, "--launch-count", "1"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
res, fname, h = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < len(h) or r[0] in ("",) or r[2] != "-":
        continue
    ie, ist, ith = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Thread Instructions Executed")
    pon = h.index("Predicated-On Thread Instructions Executed")
    try:
        res.append((int(r[ie]), int(r[ist]), int(r[ith]), int(r[pon]), fname, r[0], r[1][:70]))
    except ValueError:
        pass
tot = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
print(f"warp-instr {tot:.3e}  predicated-on thread-instr / warp-instr {sum(x[3] for x in res) / tot:.1f}")
for x in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{x[0] / tot * 100:5.1f}% i {x[1] / ts * 100:5.1f}% st  on {x[3] / max(x[0], 1):4.1f} {x[4]}:{x[5]} {x[6]}")
