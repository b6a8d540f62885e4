# ncu launch list (gpu__time_duration.sum) of one bench step of config $1 (run on the GPU box)
cd $GRAFT_REPO_ROOT
C=${1:-2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c$C.csv \
  python bench.py --config $C --steps 1 --warmup 1 --profile-run > gpurun_out/launches_c$C.log 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/launches_c$C.csv")) if len(r)>10]
h=rows[0]; ik=h.index("Kernel Name"); iv=h.index("Metric Value"); iid=h.index("ID")
for r in rows[1:]: print(r[iid], r[ik][:70], r[iv])
PY
