python -m pytest tests -m gpu -x -q -k "tile or forward or sort" 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -30
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4.json 2>gpurun_out/c4.err
timeout 1500 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5.json 2>gpurun_out/c5.err
python - <<PY
import json
for f in ("b", "c4", "c5"):
    try:
        d=json.load(open(f"gpurun_out/{f}.json")); s=d["stages"]
        print(f, round(d["value"],1), d["unit"], round(d["ms_per_step"],3), {k: round(v["ms_per_launch"],4) for k,v in s.items()})
    except Exception as e:
        print(f, "failed", e)
PY
