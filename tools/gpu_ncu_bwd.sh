# ncu --set full of one backward launch per ring variant given as args (run on the GPU box)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  VTGS_BWD_RING=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_composite_bwd" -c 1 \
    -o gpurun_out/bwd_$v -f python bench.py --steps 1 --warmup 1 --profile-run > gpurun_out/ncu_bwd_$v.log 2>&1
  tail -2 gpurun_out/ncu_bwd_$v.log
done
