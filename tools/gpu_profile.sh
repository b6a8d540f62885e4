# ncu evidence for one build (gpurun): launch list of the bench step + one --set full capture of
# the step's kernels; outputs under gpurun_out/ (TAG prefix)
cd $GRAFT_REPO_ROOT
TAG=${1:-p}
KREGEX=${2:-"k_project_count|k_emit_pairs|k_tile_sort_bucket|k_composite_fwd_ring|k_composite_bwd"}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --profile-run --no-cpu-baseline > gpurun_out/${TAG}_ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -c 8 \
    -o gpurun_out/${TAG}_kernels -f python bench.py --steps 1 --warmup 1 --profile-run --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
