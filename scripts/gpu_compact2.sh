#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/cp2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cp2_pytest.log
for v in ""; do
LBX_VARIANT=$v timeout 600 python scripts/compaction_probe.py 3 > gpurun_out/cp2_bench_$v.json 2>&1; echo "bench $v rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/cp2_bench_$v.json').read().strip().splitlines()[-1]); print(d['compaction_gbs'], d['frac_of_hbm'], [round(r['compaction_ms'],3) for r in d['steps']])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cp2_launches.csv python scripts/compaction_probe.py 2 > gpurun_out/cp2_launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compact_move -s 1 -c 1 -o gpurun_out/cp2_full python scripts/compaction_probe.py 2 > gpurun_out/cp2_full.log 2>&1; echo "ncu full rc=$?"
