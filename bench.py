#!/usr/bin/env python
"""bench.py — fwd+bwd render throughput of the view-tied splatting hot path on B200.

Metric (BASELINE.json): "fwd+bwd render Mpix/s & Gaussians/s at 1/2/4/8 B200; fraction of
roofline".  One STEP = one pass of the whole hot path over one batch of synthetic input:
projection + tile binning + per-tile sort + compositing (forward), the fused masked-L1 loss,
and the reverse-order backward to colour / opacity / radius gradients, per rank one
1200×680 view of BASELINE.json configs[1] (5 keyframes, 4.08M view-tied Gaussians), plus —
for N > 1 — the NCCL all-reduce of the 5N fp32 gradient buffer over NVLink (batched mapping,
SURVEY.md §8(e)).  Weak scaling: every rank renders one view per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config 2]

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the reference arm of
this tier) on a bounded row band of the same workload.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fwd+bwd render Mpix/s & Gaussians/s at 1/2/4/8 B200; fraction of roofline"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0        # B200_PROFILING.md fallback
SM_COUNT = 148
PROFILE_EVERY = 10   # per-kernel CUDA events ride on every 10th timed step (each event pair costs ≈ 2.7 µs of stream time)
FP32_LANES_PER_SM = 128
# Algorithmic work per unit: FP32 flops per (pixel, Gaussian)
# evaluation in the forward and per composited pair in the backward (an FMA counts 2).
FLOPS_PER_EVAL_FWD = 20.0
FLOPS_PER_COMP_BWD = 60.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="vtgs", choices=["vtgs", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-run", action="store_true", help="short run for ncu (no clocks / cpu baseline)")
    ap.add_argument("--ssim", type=float, default=0.0,
                    help="add Eq. 2's SSIM term with this weight tau (0.2 in the paper) to the mapping step")
    ap.add_argument("--no-graph", action="store_true", help="run every timed step eagerly (no CUDA graph)")
    ap.add_argument("--deterministic", action="store_true",
                    help="mapping: attribute gradients merged deterministically (VTGS_GRAD_DETERMINISTIC)")
    ap.add_argument("--streams", type=int, default=0,
                    help="renderer contexts / CUDA streams the views of a step alternate over "
                         "(0 = 2 for the batched configs 4 / 5, 1 otherwise)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region.  The sampler process
    starts before the warm-up (nvidia-smi needs ~0.1-0.3 s to produce its first line); mark()
    brackets the timed region on the host clock and only samples stamped inside it (±25 ms) are
    kept; a region shorter than the sampling period keeps the sample nearest to it instead."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None
        self.region = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark_start(self):
        self.region = [time.time(), None]

    def mark_stop(self):
        if self.region:
            self.region[1] = time.time()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if self.region and self.region[1] is not None:
            time.sleep(0.12)   # let the sample after the region arrive
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        note = None
        if self.region and self.region[1] is not None and rows:
            t0, t1 = self.region
            inside = [r for r in rows if t0 - 0.025 <= r[0] <= t1 + 0.025]
            if not inside:
                mid = 0.5 * (t0 + t1)
                inside = [min(rows, key=lambda r: abs(r[0] - mid))]
                note = f"timed region {1e3 * (t1 - t0):.0f} ms < sampling period: nearest sample"
            rows = inside
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for n, v in zip(names, r[3]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        out = {"sm_mhz": statistics.median([r[1] for r in rows]) if rows else None,
               "sm_max_mhz": max(r[2] for r in rows) if rows else None,
               "reasons": sorted(reasons), "samples": len(rows)}
        if note:
            out["note"] = note
        return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------------------
# reference arm / cpu_baseline: the CPU oracle as it stands, on a bounded row band
# ----------------------------------------------------------------------------------------
def oracle_step(cfg, state, view, rows):
    import oracle
    pr, co = state
    tg = cfg.targets[0]
    wc, wd = cfg.loss_weights
    r0, r1 = rows
    img = oracle.render(pr, co, view, cfg.intr, rows=rows)
    loss, gC, gD, gS, _ = oracle.l1_upstream(img["color"], img["depth"], img["sil"], tg.rgb, tg.depth, None,
                                              wc, wd, 0, 0, 0)
    band = np.zeros(img["depth"].shape, dtype=bool)
    band[r0:r1] = True
    gC[~band] = 0.0
    gD[~band] = 0.0
    g = oracle.render_bwd(pr, co, view, cfg.intr, gC, gD, gS)
    return loss, g


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def set_oracle_threads(n: int):
    """The oracle's OpenMP thread count (oracle/vtgs_oracle.c: rows / row bands in parallel)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass
    os.environ["OMP_NUM_THREADS"] = str(n)


def time_oracle(cfg, steps, warmup, rows, threads=1, state=None):
    """Seconds per oracle step (render + L1 + backward of `rows` of view 0) with `threads` OpenMP
    threads, and the pixels per step.  `state` = the oracle's instantiated (pos_rad, col_opa)."""
    import oracle
    if state is None:
        pr, co, _ = oracle.instantiate(cfg.depth_stack(), cfg.rgb_stack(), cfg.pose_stack(), cfg.intr, cfg.opacity)
        state = (pr, co)
    set_oracle_threads(threads)
    view = np.asarray(cfg.views[0], dtype=np.float32).astype(np.float64)
    for _ in range(warmup):
        oracle_step(cfg, state, view, rows)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle_step(cfg, state, view, rows)
    dt = (time.perf_counter() - t0) / max(steps, 1)
    px = (rows[1] - rows[0]) * cfg.intr.width
    return dt, px


def cpu_baseline_runs(cfg, repeats=3):
    """The oracle as it stands on the host: one whole step of the view (all rows), median of
    `repeats` runs on all host cores and on 1 core."""
    import oracle
    pr, co, _ = oracle.instantiate(cfg.depth_stack(), cfg.rgb_stack(), cfg.pose_stack(), cfg.intr, cfg.opacity)
    rows = (0, cfg.intr.height)
    ncores = host_cores()
    res = {}
    for label, th in (("all_cores", ncores), ("one_core", 1)):
        ts = [time_oracle(cfg, 1, 0, rows, th, (pr, co))[0] for _ in range(repeats)]
        res[label] = {"cores": th, "seconds_median": statistics.median(ts), "seconds": ts}
    set_oracle_threads(ncores)
    return res, rows[1] * cfg.intr.width


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from synth.scenes import make_config
    cfg = make_config(args.config, args.seed)
    rows = (0, cfg.intr.height)   # the whole view, every step
    ncores = host_cores()
    dt, px = time_oracle(cfg, args.steps, args.warmup, rows, threads=ncores)
    mpix = px / dt / 1e6
    sample = (f"the whole view 0 ({px} px) per step: projection + tile lists of all {cfg.n_slots} slots, render, "
              f"L1, backward (oracle/vtgs_oracle.c, -O2, OpenMP on {ncores} host cores, {cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": mpix, "unit": "Mpix/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 decisions / f64 values", "data": "synthetic",
        "config": workload_config(cfg, args),
        "gaussians_per_s": cfg.n_slots * (px / (cfg.intr.width * cfg.intr.height)) / dt,
        "cpu_baseline": {"value": mpix, "unit": "Mpix/s", "cores": ncores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": mpix, "unit": "Mpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def measured_traffic(workload, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            return json.load(f)[workload][kernel]["bytes"]
    except (OSError, KeyError, ValueError):
        return None


class RendererGroup:
    """The bench's view of the k renderer contexts a mapping step alternates its views over
    (BatchedMapper): calls that configure go to every context; the work counters are those of the
    context that rendered the step's last view (the single-context meaning: the last forward's);
    launches and per-kernel profiles are summed."""

    def __init__(self, rs):
        self.rs = list(rs)
        self.last = None   # index of the context that renders the last view (set by the caller)

    def __getattr__(self, name):   # everything else (instantiate, step_host, ...) on context 0
        return getattr(self.rs[0], name)

    def set_work_counters(self, on):
        for r in self.rs:
            r.set_work_counters(on)

    def set_profiling(self, on):
        for r in self.rs:
            r.set_profiling(on)

    def stats(self):
        ss = [r.stats() for r in self.rs]
        d = dict(ss[self.last if self.last is not None else -1])
        d["launches"] = sum(x["launches"] for x in ss)
        d["overflow"] = max(x["overflow"] for x in ss)
        return d

    def profile(self):
        ps = [r.profile() for r in self.rs]
        return {k: (sum(p[k][0] for p in ps), sum(p[k][1] for p in ps)) for k in ps[0]}


def context_scratch_bytes(N, P, W, H):
    """Device scratch a vtgs context allocates (csrc/abi.cu vtgs_create): per slot proj 16 + rect 8
    + thresholds 8 B; per pair keys / values / fallback-sort scratch 21 B + 8 sub-lists and masks
    64 B; per pixel T, last, SSIM factors, staging ≈ 60 B."""
    tiles = ((W + 15) // 16) * ((H + 15) // 16)
    return int(32 * N + 85 * P + 60 * W * H + 12 * 4 * (P // 2048 + tiles + 1) + 16 * 8 * 16 * tiles)


def workload_config(cfg, args, n_views=1, views_per_rank=1):
    return {"workload": f"config{args.config}_{cfg.name}_{cfg.intr.width}x{cfg.intr.height}_K{cfg.K}",
            "n_gaussians": cfg.n_slots, "image": [cfg.intr.width, cfg.intr.height], "views_per_step": n_views,
            "views_per_rank": views_per_rank,
            "loss": f"{cfg.loss_weights[0]}*L1(C) + {cfg.loss_weights[1]}*U*L1(D)"
                    + (f" + {args.ssim}*L_S(C)" if getattr(args, "ssim", 0.0) > 0 else "") + ", sum form",
            "grads": "colour, opacity, radius" + (" (deterministic int64 merge)" if getattr(args, "deterministic", False)
                                                   else ""), "seed": args.seed,
            "l2": "flushed between timed steps (256 MiB write outside the step events)",
            "parallelism": f"dp{args.gpus} (view-sharded mapping, one NCCL all-reduce of the 5N fp32 gradient buffer per step)"}


# ----------------------------------------------------------------------------------------
# the product arm
# ----------------------------------------------------------------------------------------
def run_tracking(args):
    """Config 3 (BASELINE.json configs[2]): one STEP = tracking one frame = 40 iterations of
    forward + fused masked-L1 (Eq. 1, W mask, mean form) + pose backward + device Adam, captured in
    one CUDA graph.  Tracking a single view does not shard: with N ranks every rank tracks its own
    replica (no collective) and `value` counts all ranks' pixels ("replicas only")."""
    import torch
    import torch.distributed as dist
    from paper_2506_02741_b200 import vtgs
    from synth.scenes import make_config
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = make_config(3, args.seed)
    W, H = cfg.intr.width, cfg.intr.height
    N = cfg.n_slots
    iters = cfg.extra["iterations"]
    R = vtgs.Renderer(local, N, W, H)
    pr, co = R.instantiate(torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev),
                           vtgs.pose_tensor(cfg.pose_stack(), dev), cfg.intr, torch.from_numpy(cfg.opacity).to(dev))
    tg = cfg.targets[0]
    L = dict(target_rgb=torch.from_numpy(tg.rgb).to(dev), target_depth=torch.from_numpy(tg.depth).to(dev),
             w_color=cfg.loss_weights[0], w_depth=cfg.loss_weights[1], color_mask_mode=1, depth_mask_mode=1,
             normalize=1)
    init = vtgs.pose_tensor(np.asarray(cfg.views[0], dtype=np.float32), dev)
    pose = init.clone()
    state = torch.zeros(16, device=dev)
    dp = torch.zeros(7, device=dev)
    loss = torch.zeros(1, device=dev)
    out = (torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev), torch.empty((H, W), device=dev))
    s = torch.cuda.Stream()

    def body(stream):
        for _ in range(iters):
            R.render_fwd(pr, co, pose, cfg.intr, out=out, stream=stream)
            R.render_bwd(vtgs.VTGS_GRAD_POSE, d_pose=dp, loss=L, loss_out=loss, stream=stream)
            R.pose_adam_step(pose, dp, state, cfg.extra["lr_rot"], cfg.extra["lr_trans"], stream=stream)

    with torch.cuda.stream(s):           # warm-up (eager) before capture
        body(s)
    torch.cuda.synchronize()
    st = R.stats()                        # work counters of the last iteration's forward (diagnostics)
    R.set_work_counters(False)            # off in the captured loop
    fp32_meas, ex2_meas = vtgs.measure_peaks(local)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        body(s)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    clocks = ClockSampler(local)
    clocks.start()                        # before the warm-up: nvidia-smi's first line takes a while
    for _ in range(max(args.warmup, 1)):
        pose.copy_(init); state.zero_(); g.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    cur = torch.cuda.current_stream()
    for i in range(args.steps):
        flush.fill_(float(i))
        pose.copy_(init)
        state.zero_()
        ev[i][0].record(cur)
        g.replay()
        ev[i][1].record(cur)
    torch.cuda.synchronize()
    clocks.mark_stop()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    px = ws * iters * W * H
    gt = cfg.extra["gt_pose"]
    pf = pose.cpu().numpy()[0].astype(np.float64)
    # per-kernel shares from an eager profiled frame (events cannot be recorded inside the graph)
    R.set_profiling(True)
    R.profile()
    pose.copy_(init); state.zero_()
    body(torch.cuda.current_stream())
    prof = R.profile()
    R.set_profiling(False)
    # roofline of the dominant kernel (per launch = one iteration): the pose backward, FP32-bound
    peaks, _ = load_peaks()
    per = {k: v[0] / v[1] for k, v in prof.items() if v[1]}
    work = {"composite_fwd": FLOPS_PER_EVAL_FWD * st["e_eval"], "composite_bwd": FLOPS_PER_COMP_BWD * st["e_comp"]}
    dom = max(work, key=lambda k: per.get(k, 0.0))
    ach = work[dom] / (per[dom] * 1e-3) / 1e12
    roofline = {"kernel": dom, "bound": "alu", "achieved": ach, "peak": fp32_meas, "unit": "TFLOP/s",
                "frac": ach / fp32_meas, "traffic": measured_traffic(f"config3_tracking_{W}x{H}_K{cfg.K}", dom),
                "peak_source": "measured: FP32 FMA-chain microbenchmark in this process (vtgs_measure_peaks)"}
    if rank == 0:
        line = {"metric": METRIC, "value": px / (ms * 1e-3) / 1e6, "unit": "Mpix/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"config3_tracking_{W}x{H}_K{cfg.K}", "n_gaussians": N,
                           "iterations_per_step": iters, "graph": True, "loss": "0.5*W*L1(C) + 1.0*W*L1(D), mean",
                           "l2": "flushed between timed steps", "parallelism": f"replicas x{ws}"},
                "gaussians_per_s": ws * iters * N / (ms * 1e-3),
                "tracking": {"t_err_init_m": float(np.linalg.norm(np.asarray(cfg.views[0])[4:] - gt[4:])),
                             "t_err_final_m": float(np.linalg.norm(pf[4:] - gt[4:]))},
                "stages_eager_frame_ms": {k: v[0] for k, v in prof.items() if v[1]},
                "roofline": roofline,
                "work_per_iteration": {"n_pairs": st["n_pairs"], "e_eval": st["e_eval"], "e_comp": st["e_comp"]},
                "peaks": {"fp32_tflops_measured": fp32_meas, "ex2_per_s_measured": ex2_meas,
                          "hbm_gbs": peaks.get("hbm_gbs")},
                "clocks": clk, "gpu_launches": int(args.steps * sum(v[1] for v in prof.values()))}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 3:
        return run_tracking(args)
    import torch
    import torch.distributed as dist
    from paper_2506_02741_b200 import vtgs
    from synth.scenes import make_config

    ws, rank, local = dist_env()
    if args.gpus > 1 and ws == 1:
        print("for --gpus > 1 launch with torchrun (one rank per GPU)", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = make_config(args.config, args.seed)
    W, H = cfg.intr.width, cfg.intr.height
    N = cfg.n_slots
    # config 5 (40 keyframes, 32.6M slots): one view needs ≤ 0.72 pairs per slot (23.5M), so the
    # context holds N pairs — its scratch stays under 4 GB; the others take the default 2N
    max_pairs = N + 262144 if args.config == 5 else 0
    n_streams = args.streams or (2 if args.config in (4, 5) else 1)
    R_list = [vtgs.Renderer(local, N, W, H, max_pairs=max_pairs) for _ in range(n_streams)]
    R = RendererGroup(R_list)
    scratch_bytes = context_scratch_bytes(N, max_pairs or 2 * N + 262144, W, H)
    # the section's Gaussians: every rank instantiates the same keyframes (no broadcast needed)
    pr, co = R.instantiate(torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev),
                           vtgs.pose_tensor(cfg.pose_stack(), dev), cfg.intr, torch.from_numpy(cfg.opacity).to(dev))
    # this rank's views.  Config 2 (the N = 1 headline): one view per rank — keyframe 2's at N = 1,
    # keyframe (2 + rank) mod K with more ranks (weak scaling).  Configs 4 / 5: the config's batch of
    # views sharded over the ranks (strong scaling; BASELINE.json configs[3], configs[4]).
    from paper_2506_02741_b200.mapping import BatchedMapper, shard_views
    if args.config == 2:
        kf = [(2 + rank) % cfg.K]
        views_np = [np.asarray(cfg.keyframes[k].pose, dtype=np.float32) for k in kf]
        tgts = [cfg.keyframes[k] for k in kf]
        n_views_total = ws
        scaling = "weak"
    else:
        mine = shard_views(len(cfg.views), ws, rank)
        views_np = [np.asarray(cfg.views[k], dtype=np.float32) for k in mine]
        tgts = [cfg.targets[k] for k in mine]
        n_views_total = len(cfg.views)
        scaling = "strong"
    R.last = (len(views_np) - 1) % n_streams
    view_np = views_np[0]
    tgt = tgts[0]
    wc, wd = cfg.loss_weights
    mapper = BatchedMapper(R_list, pr, co, cfg.intr, [vtgs.pose_tensor(v, dev) for v in views_np],
                           [dict(rgb=torch.from_numpy(t.rgb).to(dev), depth=torch.from_numpy(t.depth).to(dev))
                            for t in tgts], wc, wd, w_ssim=args.ssim, deterministic=args.deterministic)
    grads = mapper.grads.flat
    d_co, d_r = mapper.grads.d_col_opa, mapper.grads.d_radius
    out = mapper.out
    loss_out = mapper.loss
    want = vtgs.VTGS_GRAD_ATTR
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step(serial=False):
        mapper.step(allreduce=ws > 1, serial=serial)

    # measured roofline denominators of the ALU-bound kernels (FMA chain, MUFU ex2), this process
    fp32_meas, ex2_meas = vtgs.measure_peaks(local)
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    # (1) instantiation (a1), timed on its own: it runs once per keyframe, not per step
    d_depth, d_rgb = torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev)
    d_kf, d_opa = vtgs.pose_tensor(cfg.pose_stack(), dev), torch.from_numpy(cfg.opacity).to(dev)
    pr_i, co_i = torch.empty_like(pr), torch.empty_like(co)
    for _ in range(3):
        R.instantiate(d_depth, d_rgb, d_kf, cfg.intr, d_opa, out=(pr_i, co_i))
    inst_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in inst_ev:
        flush_inst = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev).fill_(1.0)
        a.record(stream)
        R.instantiate(d_depth, d_rgb, d_kf, cfg.intr, d_opa, out=(pr_i, co_i))
        b.record(stream)
    torch.cuda.synchronize()
    inst_ms = statistics.median(a.elapsed_time(b) for a, b in inst_ev)
    del pr_i, co_i, flush_inst, d_depth, d_rgb

    clocks = ClockSampler(local) if not args.profile_run else None
    if clocks:
        clocks.start()                    # before the warm-up: nvidia-smi's first line takes a while
    if args.profile_run:                  # ncu captures the first launches: make them the timed kernels
        R.set_work_counters(False)
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    st = R.stats()                                         # work counters of the (identical) warm-up steps
    assert st["overflow"] == 0, "tile-pair capacity exceeded"
    R.set_work_counters(False)                             # diagnostics only: off in the timed region

    # one CUDA graph of the whole step (launch-only: no host sync inside), replayed in the timed
    # region; the every-10th profiled steps run eagerly (per-kernel events).  N > 1 steps stay
    # eager (the NCCL all-reduce is not captured).
    graph, per_step_launches = None, 0
    if ws == 1 and not args.no_graph:
        R.set_profiling(False)
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            step()
        torch.cuda.synchronize()
        l0 = R.stats()["launches"]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            step()
        per_step_launches = R.stats()["launches"] - l0
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()

    # ---------------- timed region
    R.set_profiling(True)
    R.profile()                                            # reset
    launches0 = R.stats()["launches"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.mark_start()
    replays = 0
    for i in range(args.steps):
        flush.fill_(float(i))                               # evict L2 between steps (not timed)
        prof_i = i % PROFILE_EVERY == 0
        R.set_profiling(prof_i)                             # per-kernel events on every 10th step
        ev[i][0].record(stream)
        if graph is not None and not prof_i:
            graph.replay()
            replays += 1
        else:   # the profiled steps run their views serially: per-kernel events need no overlap
            step(serial=prof_i)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.mark_stop()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    launches = R.stats()["launches"] - launches0 + replays * per_step_launches
    prof = R.profile()
    R.set_profiling(False)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(sum(step_ms) / len(step_ms))
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    px_per_step = n_views_total * W * H
    value = px_per_step / (ms_max * 1e-3) / 1e6
    gps = n_views_total * N / (ms_max * 1e-3)

    # ---------------- roofline of the dominant kernel (event-timed inside the timed region)
    stats = dict(R.stats(), e_eval=st["e_eval"], e_comp=st["e_comp"])
    peaks, peak_src = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_nominal = sm_count * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12    # TFLOP/s at max clock
    fp32_peak, ex2_peak = fp32_meas, ex2_meas
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    per_launch = {k: (v[0] / v[1] if v[1] else 0.0) for k, v in prof.items()}
    P = stats["n_pairs"]
    HW = W * H
    # algorithmic work per launch
    work = {
        "project_count": ("hbm", (16 + 16 + 8) * N),                 # pos_rad in, proj + rect out
        "emit_pairs": ("hbm", 24 * N + 8 * P),                       # proj + rect in, (key, gid) out
        "tile_sort": ("hbm", 12 * P),                                # (key, gid) in, gid out
        "composite_fwd": ("alu", FLOPS_PER_EVAL_FWD * stats["e_eval"]),
        "composite_bwd": ("alu", FLOPS_PER_COMP_BWD * stats["e_comp"]),
        "ssim": ("hbm", 36 * HW / 3),                                # per launch (3 launches / view): x, y in, dL/dx out
    }
    stage_json = {}
    for k, (ms_k, cnt) in prof.items():
        if cnt == 0:
            continue
        e = {"ms_per_launch": per_launch[k], "launches": cnt, "share": ms_k / max(sum(v[0] for v in prof.values()), 1e-9)}
        if k in work:
            bound, units = work[k]
            if bound == "hbm":
                ach = units / (per_launch[k] * 1e-3) / 1e9
                e.update(bound="hbm", achieved=ach, unit="GB/s", frac=ach / hbm_peak)
            else:
                ach = units / (per_launch[k] * 1e-3) / 1e12
                e.update(bound="alu", achieved=ach, unit="TFLOP/s", frac=ach / fp32_peak)
        stage_json[k] = e
    inst_bytes = 52.0 * N   # depth 4 + rgb 12 + opacity 4 in, pos_rad 16 + col_opa 16 out per slot
    stage_json["instantiate"] = {"ms_per_launch": inst_ms, "launches": 10, "share": None,
                                 "note": "timed separately (once per keyframe, not in the step), L2 flushed",
                                 "bound": "hbm", "achieved": inst_bytes / (inst_ms * 1e-3) / 1e9, "unit": "GB/s",
                                 "frac": inst_bytes / (inst_ms * 1e-3) / 1e9 / hbm_peak}
    dom = max((k for k in stage_json if k in work), key=lambda k: stage_json[k]["share"])
    d = stage_json[dom]
    roofline = {"kernel": dom, "bound": d["bound"], "achieved": d["achieved"],
                "peak": hbm_peak if d["bound"] == "hbm" else fp32_peak, "unit": d["unit"], "frac": d["frac"],
                "traffic": measured_traffic(workload_config(cfg, args)["workload"], dom),
                "peak_source": (f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)" if d["bound"] == "hbm" else
                                f"measured: FP32 FMA-chain microbenchmark in this process (vtgs_measure_peaks); "
                                f"nominal {sm_count} SMs x {FP32_LANES_PER_SM} lanes x 2 x {sm_max:.0f} MHz = "
                                f"{fp32_nominal:.1f} TFLOP/s"),
                "frac_of_nominal": d["achieved"] / (hbm_peak if d["bound"] == "hbm" else fp32_nominal)}
    # the whole step against SURVEY §8(d)'s floors, per view: bytes 32 N (state) + 20 N (gradients)
    # + 24 P (pairs written and read) + 68 HW (images, targets, saved T / last, re-reads); flops
    # 20 E_eval + 60 E_comp; t_floor = max(bytes / HBM peak, flops / FP32 peak)
    n_views_rank = len(views_np)
    path_bytes = n_views_rank * (52.0 * N + 24.0 * P + 68.0 * HW)
    path_flops = n_views_rank * (FLOPS_PER_EVAL_FWD * stats["e_eval"] + FLOPS_PER_COMP_BWD * stats["e_comp"])
    t_floor_ms = max(path_bytes / (hbm_peak * 1e9), path_flops / (fp32_peak * 1e12)) * 1e3
    # whole-step DRAM traffic measured by ncu (profiles/traffic.json, sum over the step's kernels)
    step_dram = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f).get(workload_config(cfg, args)["workload"])
        if tj:
            step_dram = float(sum(v["bytes"] for v in tj.values()))
    except (OSError, ValueError, KeyError, TypeError):
        pass
    path_floor = {"bytes": path_bytes, "flops": path_flops, "t_floor_ms": t_floor_ms,
                  "frac": t_floor_ms / ms_max, "ex2": n_views_rank * (stats["e_eval"] + stats["e_comp"]),
                  "t_ex2_ms": n_views_rank * (stats["e_eval"] + stats["e_comp"]) / ex2_peak * 1e3,
                  "step_dram_bytes_ncu": step_dram,
                  "dram_over_algorithmic": (step_dram / (path_bytes / n_views_rank)) if step_dram else None}
    peaks_json = {"fp32_tflops_measured": fp32_meas, "ex2_per_s_measured": ex2_meas,
                  "fp32_tflops_nominal": fp32_nominal, "hbm_gbs": hbm_peak, "hbm_source": peak_src}

    # ---------------- e2e: the same step through the C-ABI with HOST buffers.  Headline: the frame
    # as an RGB-D sensor (and the paper's datasets) delivers it — 8-bit RGB, 16-bit depth (metres =
    # value / 5000) — uploaded as 5 B/px and widened on the device (vtgs_step_host_sensor); also
    # timed: the same step with fp32 host targets (16 B/px, vtgs_step_host).
    e2e = None
    if not args.profile_run:
        depth_scale = np.float32(1.0 / 5000.0)
        h_views = [torch.from_numpy(v.reshape(7).copy()).pin_memory() for v in views_np]
        h_tg = [(torch.from_numpy(t.rgb).pin_memory(), torch.from_numpy(t.depth).pin_memory()) for t in tgts]
        h_sn = [(torch.from_numpy(np.clip(np.rint(t.rgb * 255.0), 0, 255).astype(np.uint8)).pin_memory(),
                 torch.from_numpy(np.clip(np.rint(t.depth / depth_scale), 0, 65535).astype(np.uint16)).pin_memory())
                for t in tgts]

        def e2e_run(sensor):
            def one_step():
                grads.zero_()
                for hv, (hr, hd), (sr, sd) in zip(h_views, h_tg, h_sn):
                    if sensor:
                        R.step_host_sensor(pr, co, hv, cfg.intr, sr, sd, float(depth_scale), wc, wd, 0, 0, 0, want,
                                           (0, N), out, d_co, d_r)
                    else:
                        R.step_host(pr, co, hv, cfg.intr, hr, hd, wc, wd, 0, 0, 0, want, (0, N), out, d_co, d_r)
                if ws > 1:
                    dist.all_reduce(grads)
                    torch.cuda.synchronize()
            for _ in range(max(args.warmup, 20)):   # fresh pinned buffers and an idle host: let them settle
                one_step()
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                one_step()
            torch.cuda.synchronize()
            e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
            te = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            if ws > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            return float(te.item())

        e_ms = e2e_run(True)
        f_ms = e2e_run(False)
        e2e = {"value": px_per_step / (e_ms * 1e-3) / 1e6, "unit": "Mpix/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(sum(sr.numel() + sd.numel() * 2 + 28 for sr, sd in h_sn)),
               "d2h_bytes_per_step": 4 * len(h_sn),
               "api": "vtgs_step_host_sensor (host uint8 RGB + uint16 depth + pose in, host loss out)",
               "fp32_targets": {"value": px_per_step / (f_ms * 1e-3) / 1e6, "ms_per_step": f_ms,
                                "h2d_bytes_per_step": int(sum(hr.numel() * 4 + hd.numel() * 4 + 28 for hr, hd in h_tg)),
                                "api": "vtgs_step_host (host fp32 RGB-D + pose in, host loss out)"}}

    # ---------------- cpu baseline (oracle as it stands, bounded sample, rank 0, N=1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile_run:
        runs, px = cpu_baseline_runs(cfg)
        allc, one = runs["all_cores"], runs["one_core"]
        cpu = {"value": px / allc["seconds_median"] / 1e6, "unit": "Mpix/s", "cores": allc["cores"], "kind": "oracle",
               "sample": f"one whole step of the same view ({px} px): projection + tile lists of all {N} slots, "
                         f"render, L1, backward (oracle/vtgs_oracle.c, -O2, OpenMP); median of 3 runs",
               "cpu_model": cpu_model(), "seconds_median": allc["seconds_median"],
               "one_core": {"value": px / one["seconds_median"] / 1e6, "seconds_median": one["seconds_median"],
                            "cores": 1}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mpix/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded procedural rooms, ray-cast RGB-D; stands in for Replica/TUM/ScanNet)",
            "config": dict(workload_config(cfg, args, n_views_total, len(views_np)),
                           streams=f"{n_streams} renderer context(s) / CUDA stream(s), views alternating"),
            "gaussians_per_s": gps,
            "roofline": roofline,
            "path_floor": path_floor,
            "peaks": peaks_json,
            "stages": stage_json,
            "stage_timing": f"CUDA events around every kernel on every {PROFILE_EVERY}th timed step ({(args.steps + PROFILE_EVERY - 1) // PROFILE_EVERY} of {args.steps}, run eagerly"
                            + (", views serially on one context's stream" if n_streams > 1 else "") + "), on the launching stream",
            "graph": (f"the other {replays} timed steps replay one captured CUDA graph of the step ({per_step_launches} launches)"
                      if graph is not None else "eager"),
            "work": {"n_pairs": P, "e_eval": stats["e_eval"], "e_comp": stats["e_comp"], "max_tile": stats["max_tile"]},
            "context_scratch_bytes": scratch_bytes,          # per renderer context
            "contexts": n_streams,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": int(launches),
            "loss": float(loss_out.sum().item()),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
