# A/B of prebuilt library variants with extra bench.py arguments (gpurun):
#   bash tools/gpu_lib_ab_args.sh TAG "--ssim 0.2" lib1.so lib2.so …
# Each variant is run twice, alternating, so a drifting box shows up as a spread.
cd $GRAFT_REPO_ROOT
TAG=$1; ARGS=$2; shift 2
for rep in 1 2; do
for lib in "$@"; do
  out=gpurun_out/${TAG}_$(basename $lib .so)_$rep
  VTGS_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 60 $ARGS > $out.json 2> $out.err
  python -c "
import json; d=json.loads(open('$out.json').read().strip().splitlines()[-1]); st=d.get('stages') or {k: {'ms_per_launch': v} for k, v in d.get('stages_eager_frame_ms', {}).items()}; print('$lib', round(d['ms_per_step'],4), {k: round(v['ms_per_launch'],4) for k, v in st.items()})"
done
done
