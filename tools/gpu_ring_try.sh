# Try a kernel variant: A/B bench against the default, then the backward parity tests under it (gpurun)
cd $GRAFT_REPO_ROOT
TAG=$1; VAR=$2; VAL=$3
env $VAR=0 timeout 300 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/${TAG}_base.json 2> gpurun_out/${TAG}_base.err
env $VAR=$VAL timeout 300 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/${TAG}_var.json 2> gpurun_out/${TAG}_var.err
env $VAR=$VAL timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "backward or loss or deterministic or mapping or ssim or step_host or edge" > gpurun_out/${TAG}_tests.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log
