# A/B of prebuilt library variants (gpurun): VTGS_LIB_PATH points the binding at each .so in turn
cd $GRAFT_REPO_ROOT
TAG=$1; shift
for lib in "$@"; do
  VTGS_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/${TAG}_$(basename $lib .so).json 2> gpurun_out/${TAG}_$(basename $lib .so).err
  python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_$(basename $lib .so).json').read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],4), {k: round(v['ms_per_launch'],4) for k, v in d['stages'].items()})"
done
