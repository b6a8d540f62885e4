# ncu --set full of the SSIM kernels of one --ssim bench step (gpurun)
cd $GRAFT_REPO_ROOT
TAG=$1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssim -c 3 \
  -o gpurun_out/${TAG}_ssim -f python bench.py --steps 1 --warmup 1 --profile-run --ssim 0.2 > gpurun_out/${TAG}_ssim_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ssim_ncu.log
