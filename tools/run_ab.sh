for ki in 2 6 8; do
  cp tools/ab_libs/libvtgs_k$ki.so paper_2506_02741_b200/libvtgs.so
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python - <<PY
import json; d=json.load(open("gpurun_out/b.json")); s=d["stages"]
print("$ki", round(d["ms_per_step"],4), round(s["composite_fwd"]["ms_per_launch"],4))
PY
done
