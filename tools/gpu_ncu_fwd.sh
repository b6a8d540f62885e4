# ncu metrics of the forward ring at several depths (VTGS_FWD = R), run on the GPU box
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_pred_on.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers
for v in "$@"; do
  echo "== VTGS_FWD=$v"
  VTGS_FWD=$v timeout 600 ncu --metrics $M --clock-control none -k regex:"k_composite_fwd" -c 1 \
    python bench.py --steps 1 --warmup 1 --profile-run 2>&1 | grep -E "^\s+(gpu__|smsp__|sm__|l1tex|launch)" 
done
