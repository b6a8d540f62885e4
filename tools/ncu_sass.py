#!/usr/bin/env python
"""Per-SASS-instruction execution counts of one kernel from an ncu report (hot loops)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 80
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                              text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]
ie, ia, iss, src = h.index("Instructions Executed"), h.index("Avg. Threads Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
data = []
for r in rows[i0 + 1:]:
    if len(r) < len(h) or not r[0].startswith("0x"):
        continue
    data.append((int(r[ie] or 0), float(r[ia] or 0), int(r[iss] or 0), r[src].strip()))
tot = sum(d[0] for d in data); ts = sum(d[2] for d in data) or 1
print(f"total warp-instr {tot:.3e}")
mx = max(d[0] for d in data)
for n, a, s, t in data:
    if n >= mx * 0.02:
        print(f"{n:>11d} {a:5.1f} {100*s/ts:5.1f}%  {t[:90]}")
