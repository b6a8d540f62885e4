cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
for v in 0 41 81 82 162; do
  VTGS_BWD_RING=$v timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/ring_$v.json 2> gpurun_out/ring_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ring_$v.json')); s=d['stages']; print('$v', round(d['ms_per_step'],4), 'bwd', round(s['composite_bwd']['ms_per_launch'],4), 'fwd', round(s['composite_fwd']['ms_per_launch'],4))"
done
