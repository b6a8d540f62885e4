python -m pytest tests -m gpu -x -q -k "backward or loss or deterministic or tracking or step_host or position or pretrack" 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -30
for v in 1; do
VTGS_BWD_POSE=$v python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/t$v.json 2>gpurun_out/t$v.err
python - <<PY
import json; d=json.load(open("gpurun_out/t$v.json"))
print("$v", round(d["ms_per_step"],3), d["tracking"], {k: round(v,3) for k,v in d["stages_eager_frame_ms"].items()})
PY
done
