python -m pytest tests -m gpu -x -q -k "ssim or mapping_objective" 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -30
python bench.py --ssim 0.2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bs.json 2>gpurun_out/bs.err
python - <<PY
import json; d=json.load(open("gpurun_out/bs.json")); s=d["stages"]
print(round(d["ms_per_step"],4), {k: round(v["ms_per_launch"],4) for k,v in s.items()})
PY
