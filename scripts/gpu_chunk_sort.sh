#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pic.py tests/test_gpu_pic_fast.py -q -x > gpurun_out/cs_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/cs_pytest.log
timeout 900 python bench_pic.py --steps 20 --warmup 3 --resort 10 --modes push_deposit_fast,push_deposit_fast_resort,push_deposit_resort,push_deposit_inplace > gpurun_out/cs_c2.json 2>&1; echo "c2 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/cs_c2.json').read().strip().splitlines()[-1])
for k,v in d.items():
    if isinstance(v,dict): print(k, round(v['ms'],3), round(v['ms_pipelined'],3), round(v['frac_of_hbm_peak_pipelined'],3), v['ms_per_step'][:12])"
for s in 0 7; do
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pic_pipe_kernel" -s $s -c 1 python bench_pic.py --steps 8 --warmup 0 --resort 100 --modes push_deposit_fast_resort > gpurun_out/cs_$s.txt 2>&1; echo "s=$s"; grep -E "gpu__time|inst_executed|issue_active|op_red|dram__bytes" gpurun_out/cs_$s.txt
done
