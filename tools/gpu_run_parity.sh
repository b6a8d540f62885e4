# GPU parity run (gpurun): smoke, the GPU test suite, a bench line; logs under gpurun_out/
cd $GRAFT_REPO_ROOT
TAG=${1:-g}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 3000 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=15 ${PYTEST_K} > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo done
