# A/B the tracking frame (config 3) under several values of one environment variable
cd $GRAFT_REPO_ROOT
VAR=$1; shift
for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/trk_$v.json 2> gpurun_out/trk_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/trk_$v.json').read().strip().splitlines()[-1]); print('$VAR=$v', round(d['ms_per_step'],3), round(d['stages_eager_frame_ms']['composite_bwd'],3), d['tracking']['t_err_final_m'])"
done
