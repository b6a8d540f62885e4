#!/bin/bash
# One round's measurement evidence (run on the GPU box via gpurun, from the repo root):
# bench lines (product arm, reference arm, tracking config), the ncu launch list of the bench
# command and one `ncu --set full` capture of the step's kernels.  Outputs under gpurun_out/.
set -x
TAG=${1:-r01b}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.json 2>> gpurun_out/${TAG}_bench.err
python bench.py --config 3 --steps 20 --warmup 3 > gpurun_out/${TAG}_tracking.json 2>> gpurun_out/${TAG}_bench.err
python bench.py --ssim 0.2 --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_ssim.json 2>> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --profile-run > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_project_count|k_emit_pairs|k_tile_sort_bucket|k_composite_fwd_ring|k_composite_bwd" -c 8 \
    -o gpurun_out/${TAG}_kernels -f python bench.py --steps 1 --warmup 1 --profile-run > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out
