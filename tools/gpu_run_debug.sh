cd $GRAFT_REPO_ROOT
timeout 900 python tests/models/debug_fused_l1.py 2 > gpurun_out/g2_debug.log 2>&1
free -g > gpurun_out/g2_host.txt; nproc >> gpurun_out/g2_host.txt; lscpu | head -20 >> gpurun_out/g2_host.txt
echo done
