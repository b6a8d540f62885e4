# compute-sanitizer evidence (gpurun): one tool per run; logs under gpurun_out/
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
: > gpurun_out/san_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_step.py 1 > gpurun_out/san_${tool}_c1.log 2>&1
  echo "$tool config1 rc=$?" >> gpurun_out/san_summary.txt
done
timeout 900 $CS --tool racecheck --error-exitcode 9 python tools/sanitize_step.py long > gpurun_out/san_racecheck_long.log 2>&1
echo "racecheck long-lists rc=$?" >> gpurun_out/san_summary.txt
timeout 1500 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_step.py 2 > gpurun_out/san_memcheck_c2.log 2>&1
echo "memcheck config2 rc=$?" >> gpurun_out/san_summary.txt
echo done
