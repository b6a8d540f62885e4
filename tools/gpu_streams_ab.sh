# configs 4 / 5: views alternating over 1 vs 2 renderer contexts / streams (gpurun)
cd $GRAFT_REPO_ROOT
for c in 4 5; do
  for k in ${KS:-1 2}; do
    timeout 600 python bench.py --config $c --streams $k --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/st_c${c}_k$k.json 2> gpurun_out/st_c${c}_k$k.err
    python -c "
import json; d=json.loads(open('gpurun_out/st_c${c}_k$k.json').read().strip().splitlines()[-1]); print('config $c streams $k', round(d['ms_per_step'],3), round(d['value'],1), d['e2e']['value'] if d.get('e2e') else None)"
  done
done
