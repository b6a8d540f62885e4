# A/B of a kernel-variant environment variable on the config-2 bench step (gpurun)
cd $GRAFT_REPO_ROOT
TAG=$1; VAR=$2; shift 2
for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/${TAG}_${VAR}_${v}.json 2> gpurun_out/${TAG}_${VAR}_${v}.err
done
echo done
