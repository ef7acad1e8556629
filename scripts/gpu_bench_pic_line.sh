#!/bin/bash
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-native > gpurun_out/bpl.json 2> gpurun_out/bpl.err; echo rc=$?; tail -3 gpurun_out/bpl.err
python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/bpl.json') if l.startswith('{')][-1]; print(d['value'], d['pic'])"
