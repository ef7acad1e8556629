#!/bin/bash
# Final verification after the round-2-end kernel trims: all GPU tests,
# smoke, bench (both arms), ncu of the PIC kernels.  Outputs -> gpurun_out/r2k_*
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2k_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2k_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2k_smoke.log
timeout 900 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "bench rc=$?"; grep '^{' gpurun_out/r2k_bench.json | tail -1 | head -c 600; echo
timeout 900 python bench.py --impl reference > gpurun_out/r2k_bench_ref.json 2> gpurun_out/r2k_bench_ref.err; echo "ref rc=$?"; grep '^{' gpurun_out/r2k_bench_ref.json | tail -1 | head -c 300; echo
for m in push_deposit_fast_resort_noclock push_deposit_resort_noclock push_deposit_esk3_resort_noclock; do
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none -k regex:"pic_pipe_kernel|pic_esk_kernel" -c 1 python bench_pic.py --steps 1 --warmup 0 --modes $m > gpurun_out/r2k_ncu_$m.txt 2>&1; echo "== $m"; grep -E "gpu__time|inst_executed|issue_active|dram__bytes|registers" gpurun_out/r2k_ncu_$m.txt
done
