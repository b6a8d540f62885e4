python -m pytest tests -m gpu -x -q -k "tile or forward" 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -30
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
python - <<PY
import json; d=json.load(open("gpurun_out/b.json")); s=d["stages"]
print(round(d["ms_per_step"],4), {k: round(v["ms_per_launch"],4) for k,v in s.items()})
PY
