#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/picu_launches.csv python bench_pic.py --workload uniform --steps 1 --warmup 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/picu_launches.csv")))
h = None
for r in rows:
    if "Kernel Name" in r:
        h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if "lbx" in d["Kernel Name"]:
            print(d["Kernel Name"][:60], d["Metric Value"])
PY
timeout 900 python bench_lb.py --emulate 8 --physics pic --replicas 128 --steps 60 --speed 0.3 --drift 0.3 --exchange p2p > gpurun_out/lb_pic.json 2> gpurun_out/lb_pic.err; echo "lb pic rc=$?"; tail -3 gpurun_out/lb_pic.err; cat gpurun_out/lb_pic.json
