# SSIM kernels: parity tests + the --ssim bench line (gpurun)
cd $GRAFT_REPO_ROOT
TAG=$1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "ssim" > gpurun_out/${TAG}_tests.log 2>&1
tail -2 gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --no-cpu-baseline --steps 60 --ssim 0.2 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stages']['ssim'])"
