#!/bin/bash
# One round's measurement evidence (run on the GPU box via gpurun, from the repo root): bench
# lines (product arm with cpu_baseline, reference arm, tracking, SSIM, configs 4 / 5), the render
# error vs the oracle, the ncu launch list of the bench command and one `ncu --set full` capture of
# the step's kernels.  Outputs under gpurun_out/ with the TAG prefix.
set -x
TAG=${1:-r02}
cd $GRAFT_REPO_ROOT
nvidia-smi > gpurun_out/${TAG}_nvidia_smi.txt 2>&1; lscpu > gpurun_out/${TAG}_lscpu.txt 2>&1
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_reference.json 2>> gpurun_out/${TAG}_bench.err
python bench.py --config 3 --steps 20 --warmup 3 > gpurun_out/${TAG}_tracking.json 2>> gpurun_out/${TAG}_bench.err
python bench.py --ssim 0.2 --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_ssim.json 2>> gpurun_out/${TAG}_bench.err
python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_config4.json 2>> gpurun_out/${TAG}_bench.err
python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_config5.json 2>> gpurun_out/${TAG}_bench.err
python tests/models/render_error.py 1 2 3 > gpurun_out/${TAG}_render_error.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --profile-run --no-cpu-baseline > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_project_count|k_emit_pairs|k_tile_sort_bucket|k_composite_fwd_ring|k_composite_bwd|k_loss_finalize|k_scan_tiles" -c 9 \
    -o gpurun_out/${TAG}_kernels -f python bench.py --steps 1 --warmup 1 --profile-run --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out
