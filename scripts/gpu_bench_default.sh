#!/bin/bash
start=$(date +%s)
timeout 900 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; echo "bench rc=$? secs=$(( $(date +%s) - start ))"
python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/r2j_bench.json') if l.startswith('{')][-1]
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['pic']['ms_per_step'], d['pic']['frac_of_hbm'], d['pic']['first_step_frac_of_hbm'], d['c2_native']['us_per_step'], d['clocks'])"
