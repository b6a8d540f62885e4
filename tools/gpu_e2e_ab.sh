# A/B of prebuilt library variants on the e2e leg (vtgs_step_host_sensor) of the config-2 bench line (gpurun):
#   bash tools/gpu_e2e_ab.sh TAG lib1.so lib2.so …   (each variant twice, alternating)
cd $GRAFT_REPO_ROOT
TAG=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  out=gpurun_out/${TAG}_$(basename $lib .so)_$rep
  VTGS_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 100 > $out.json 2> $out.err
  python -c "
import json; d=json.loads(open('$out.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$lib', round(d['ms_per_step'],4), 'e2e', round(e['value'],1), round(e['ms_per_step'],4), 'fp32', round(e['fp32_targets']['value'],1))"
done
done
