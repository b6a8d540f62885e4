#!/usr/bin/env python
"""Collect one round's evidence from gpurun_out/ into profiles/: the bench lines, the launch list,
the ncu report's per-kernel summary, the DRAM traffic per kernel (profiles/traffic.json) and a
markdown summary.   python tools/round_summary.py TAG [--out r02]"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
NAMES = {"k_project_count": "project_count", "k_emit_pairs": "emit_pairs", "k_tile_sort_bucket": "tile_sort",
         "k_composite_fwd_ring": "composite_fwd", "k_composite_bwd": "composite_bwd", "k_scan_tiles": "scan_tiles",
         "k_loss_finalize": "loss_finalize"}


def last_json(path):
    try:
        with open(path) as f:
            return json.loads(f.read().strip().splitlines()[-1])
    except Exception:
        return None


def ncu_rows(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--out", default="r02")
    a = ap.parse_args()
    t, o = a.tag, a.out
    files = {"bench": f"{t}_bench.json", "reference": f"{t}_reference.json", "tracking": f"{t}_tracking.json",
             "bench_ssim": f"{t}_bench_ssim.json", "bench_config4": f"{t}_bench_config4.json",
             "bench_config5": f"{t}_bench_config5.json"}
    lines = {}
    for k, fn in files.items():
        src = os.path.join(G, fn)
        if os.path.exists(src):
            shutil.copy(src, os.path.join(P, f"{o}_{k}.json"))
            lines[k] = last_json(src)
    for fn in (f"{t}_launches.csv", f"{t}_render_error.log", f"{t}_lscpu.txt"):
        src = os.path.join(G, fn)
        if os.path.exists(src):
            shutil.copy(src, os.path.join(P, fn.replace(t, o)))
    rep = os.path.join(G, f"{t}_kernels.ncu-rep")
    kern = []
    traffic = {}
    if os.path.exists(rep):
        shutil.copy(rep, os.path.join(P, f"{o}_kernels.ncu-rep"))
        h, rows = ncu_rows(rep)
        seen = set()
        for r in rows:
            name = r[h.index("Kernel Name")]
            short = next((v for k, v in NAMES.items() if k in name), None)
            if short is None or short in seen:
                continue
            seen.add(short)
            get = lambda c: float(r[h.index(c)]) if c in h and r[h.index(c)] else float("nan")
            rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
            kern.append((short, name[:60], get("gpu__time_duration.sum"), get("smsp__inst_executed.sum"),
                         get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                         get("sm__warps_active.avg.pct_of_peak_sustained_active"), rd, wr,
                         get("launch__registers_per_thread")))
            # ncu reports MB (1e6 bytes) for dram__bytes_*.sum in this capture's units
            traffic[short] = {"bytes": int(round((rd + wr) * 1e6)), "source": f"profiles/{o}_kernels.ncu-rep"}
    wl = (lines.get("bench") or {}).get("config", {}).get("workload", "config2_mapping_1200x680_K5")
    tj_path = os.path.join(P, "traffic.json")
    tj = json.load(open(tj_path)) if os.path.exists(tj_path) else {}
    if traffic:
        tj[wl] = traffic
        tj["_doc"] = ("DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum, bytes) from one ncu "
                      "--set full --clock-control none capture of the bench step's kernels; bench.py copies the "
                      "dominant kernel's figure into roofline.traffic and sums them for path_floor.step_dram_bytes_ncu.")
        with open(tj_path, "w") as f:
            json.dump(tj, f, indent=1)
    md = [f"# Round 2 evidence ({o}, gpurun tag {t})", ""]
    b = lines.get("bench")
    if b:
        md += [f"**Config 2 mapping step**: {b['ms_per_step']:.4f} ms = {b['value']:.1f} Mpix/s = "
               f"{b['gaussians_per_s'] / 1e9:.2f} G Gaussians/s (fp32), clocks {b.get('clocks')}",
               f"- roofline (dominant kernel {b['roofline']['kernel']}): {b['roofline']['achieved']:.2f} "
               f"{b['roofline']['unit']} of {b['roofline']['peak']:.1f} = **{b['roofline']['frac']:.4f}** "
               f"({b['roofline']['peak_source']}); of nominal {b['roofline'].get('frac_of_nominal', float('nan')):.4f}",
               f"- path floor: {b['path_floor']['t_floor_ms'] * 1e3:.1f} µs → the step runs at "
               f"{b['path_floor']['frac']:.3f} of it; step DRAM (ncu) {b['path_floor'].get('step_dram_bytes_ncu')} B = "
               f"{b['path_floor'].get('dram_over_algorithmic')} × the algorithmic bytes",
               (f"- e2e ({b['e2e'].get('api', 'vtgs_step_host')}): {b['e2e']['value']:.1f} Mpix/s"
                + (f"; fp32 targets ({b['e2e']['fp32_targets']['api']}): {b['e2e']['fp32_targets']['value']:.1f} Mpix/s"
                   if b['e2e'].get('fp32_targets') else "")) if b.get("e2e") else "",
               f"- cpu_baseline: {json.dumps(b.get('cpu_baseline'))}",
               f"- peaks: {json.dumps(b.get('peaks'))}",
               f"- context scratch: {b.get('context_scratch_bytes', 0) / 1e9:.2f} GB", "",
               "| stage | ms / launch | bound | achieved | frac |", "|---|---|---|---|---|"]
        for k, v in b["stages"].items():
            md.append(f"| {k} | {v['ms_per_launch']:.4f} | {v.get('bound', '')} | "
                      f"{v.get('achieved', float('nan')):.2f} {v.get('unit', '')} | {v.get('frac') or ''} |")
        md.append("")
    for k in ("tracking", "bench_ssim", "bench_config4", "bench_config5", "reference"):
        x = lines.get(k)
        if x:
            rf = x.get("roofline") or {}
            md.append(f"- **{k}**: {x.get('ms_per_step', float('nan')):.3f} ms/step, {x['value']:.2f} {x['unit']}"
                      + (f", roofline {rf.get('kernel')} {rf.get('frac', float('nan')):.4f}" if rf else "")
                      + (f", scratch {x.get('context_scratch_bytes', 0) / 1e9:.2f} GB" if x.get("context_scratch_bytes") else ""))
    if kern:
        md += ["", "ncu (`--set full --clock-control none`, cold L2 per launch):", "",
               "| kernel | µs | warp instr | issue active % | warps active % | DRAM read MB | DRAM write MB | regs |",
               "|---|---|---|---|---|---|---|---|"]
        for s, n, us, ins, ia, wa, rd, wr, rg in kern:
            md.append(f"| {s} | {us:.1f} | {ins / 1e6:.1f}M | {ia:.1f} | {wa:.1f} | {rd:.1f} | {wr:.1f} | {rg:.0f} |")
    with open(os.path.join(P, f"{o}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
