for v in 4 8 16; do
  VTGS_FWD=$v python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/fwd_$v.json 2>gpurun_out/fwd_$v.err
  python - <<PY
import json; d=json.load(open("gpurun_out/fwd_$v.json")); s=d["stages"]
print("$v", round(d["ms_per_step"],4), round(s["composite_fwd"]["ms_per_launch"],4))
PY
done
