# A/B the step under several values of one environment variable: gpu_ab_env.sh VAR v1 v2 ...
cd $GRAFT_REPO_ROOT
VAR=$1; shift
for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); s=d['stages']; print('$VAR=$v', round(d['ms_per_step'],4), {k: round(x['ms_per_launch'],4) for k,x in s.items()})"
done
