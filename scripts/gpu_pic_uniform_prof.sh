#!/bin/bash
# Uniform-plasma PIC (SURVEY 8d roofline case), in-place mode: per-kernel
# launch list (time + DRAM bytes) of one step, and the bench numbers.
mkdir -p gpurun_out
timeout 300 python bench_pic.py --workload uniform --modes ${MODES:-push_deposit_inplace} --steps 6 --warmup 2 > gpurun_out/picu_bench.json 2> gpurun_out/picu_bench.err
python -c "import json; d=json.load(open('gpurun_out/picu_bench.json')); print({k: (v['ms'], v['ms_per_step']) for k, v in d.items() if isinstance(v, dict)})"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/picu_launches.csv python bench_pic.py --workload uniform --modes ${MODES:-push_deposit_inplace} --steps 1 --warmup 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/picu_launches.csv")) if len(r) > 10]
hdr = rows[0]
iN, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iID = hdr.index("ID")
k = {}
for r in rows[1:]:
    k.setdefault(r[iID], {"name": r[iN][:60]})[r[iM]] = r[iV]
for i, d in list(k.items())[-14:]:
    print(i, d["name"], d.get("gpu__time_duration.sum"), d.get("dram__bytes_read.sum"),
          d.get("dram__bytes_write.sum"), d.get("smsp__inst_executed.sum"))
PY
