#!/usr/bin/env python
"""Summarise an ncu report: key throughput metrics, stall breakdown, hottest source lines.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--source] [--kernel REGEX]
"""
import argparse
import csv
import io
import re
import subprocess

KEYS = [
    "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--source", action="store_true")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    hdr, rows = raw(a.rep)
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        if a.kernel and not re.search(a.kernel, name):
            continue
        print(f"== {name}")
        for k in KEYS:
            if k in hdr:
                print(f"   {k:60s} {r[hdr.index(k)]}")
        st = [(h, r[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        st = sorted(((h, float(v or 0)) for h, v in st), key=lambda x: -x[1])
        print("   stalls (warps per issue-active cycle):",
              ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for h, v in st[:8]))
    if a.source:
        out = subprocess.check_output(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda"]
                                      + (["-k", a.kernel] if a.kernel else []), text=True, stderr=subprocess.DEVNULL)
        rows = list(csv.reader(io.StringIO(out)))
        if not rows:
            return
        h = rows[0]
        def col(name):
            for i, x in enumerate(h):
                if x.startswith(name):
                    return i
            return None
        ci = col("Warp Stall Sampling (All")
        src = col("Source")
        line = col("#")
        if ci is None:
            print(h)
            return
        data = []
        for r in rows[1:]:
            try:
                data.append((float(r[ci] or 0), r[line] if line is not None else "", r[src][:110]))
            except (ValueError, IndexError):
                pass
        tot = sum(d[0] for d in data) or 1
        for v, ln, s in sorted(data, key=lambda x: -x[0])[:a.top]:
            print(f"   {100 * v / tot:5.1f}%  {ln:>5}  {s}")


if __name__ == "__main__":
    main()
