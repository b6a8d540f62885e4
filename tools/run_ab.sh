ncu --set full --clock-control none --import-source on \
    -k regex:"k_project_count|k_emit_pairs|k_tile_sort_bucket|k_composite_fwd_ring|k_composite_bwd" -c 8 \
    -o gpurun_out/r01c_kernels -f python bench.py --steps 1 --warmup 1 --profile-run > gpurun_out/r01c_ncu_full.log 2>&1
