python -m pytest tests -m gpu -x -q -k "step_host" 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -30
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
python - <<PY
import json; d=json.load(open("gpurun_out/b.json")); s=d["stages"]
print(round(d["ms_per_step"],4), d["value"], d["e2e"])
PY
