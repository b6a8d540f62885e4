# quick check (gpurun): config-2 bench line + a pytest selection ($2, a -k expression)
cd $GRAFT_REPO_ROOT
TAG=$1
timeout 300 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], {k: round(v['ms_per_launch'], 4) for k, v in d['stages'].items()})"
if [ -n "$2" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu -k "$2" > gpurun_out/${TAG}_tests.log 2>&1
  tail -2 gpurun_out/${TAG}_tests.log
fi
