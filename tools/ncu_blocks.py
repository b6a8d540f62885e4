#!/usr/bin/env python
"""Group the SASS of one kernel in an ncu report into straight-line blocks (equal execution
counts) and list the heaviest blocks by instructions and by stall samples."""
import csv, io, subprocess, sys
rep, idx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 18
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                               "--launch-skip", str(idx), "--launch-count", "1"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
i0 = starts[0]
end = starts[1] if len(starts) > 1 else len(rows)
h = rows[i0]
ie, ia, src, ss = h.index("Instructions Executed"), h.index("Avg. Threads Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ie] or 0), float(r[ia] or 0), int(r[ss] or 0), r[src].strip()) for r in rows[i0 + 1:end]
        if len(r) == len(h) and r[0].startswith("0x")]
blocks, cur = [], None
for k, (n, a, s, t) in enumerate(data):
    if cur and cur[0] == n:
        cur[2] += 1; cur[3].append(t); cur[4] += s
    else:
        cur = [n, a, 1, [t], s, k]; blocks.append(cur)
tot = sum(d[0] for d in data); tots = sum(d[2] for d in data) or 1
print("total warp-instr", tot)
for n, a, c, ss_, st, k in sorted(blocks, key=lambda b: -(b[0] * b[2] + b[4] * tot / tots))[:top]:
    print(f"@{k:5d} {n:>10d} x{c:3d} = {n * c / tot * 100:5.1f}% instr {st / tots * 100:5.1f}% stall thr={a:4.1f}  {ss_[0][:40]} .. {ss_[-1][:30]}")
