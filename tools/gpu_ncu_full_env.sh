# ncu --set full of one launch of the kernels matching $1 with env var $2 set to each of the rest
cd $GRAFT_REPO_ROOT
K=$1; VAR=$2; shift 2
for v in "$@"; do
  env $VAR=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
    -o gpurun_out/full_${VAR}_$v -f python bench.py --steps 1 --warmup 1 --profile-run > gpurun_out/ncu_${VAR}_$v.log 2>&1
  tail -1 gpurun_out/ncu_${VAR}_$v.log
done
