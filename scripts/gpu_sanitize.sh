#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over CI-sized cases of
# every kernel family: fused push/bin/compaction, drop-in AoS path + host
# pipeline, PIC (quad/direct, in place/sorted, cell sort), native loop graph replay, multi-GPU exchange (p2p and
# collectives, thread ranks).  Summaries -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CASES_K='tests/test_gpu_kernels.py -k "fixture or known_answer or empty or (fused_step_matches_oracle and 300001) or non_power or (host_pipeline and 5000)"'
CASES_P='tests/test_gpu_pic.py -k "first_step or (multi_step and clustered-quad) or sorted_mode_matches_oracle"'
CASES_D='tests/test_gpu_dist.py -k "mini-2 and p2p"'
CASES_E='tests/test_gpu_3d.py tests/test_gpu_pic.py -k "3d or hole_filling or (multi_step and direct) or gpuclock or timers"'
CASES_R='tests/test_gpu_runs.py -k "(timers and not cupti) or gpuclock or (graph_replay and mini)"'
CASES_S='tests/test_gpu_pic.py -k "periodic_cell_sort or share_a_state or reused_buffers or tiled"'
# round 2: pipelined tolerance kernel, Esirkepov, count/scan/move compaction
CASES_F='tests/test_gpu_pic_fast.py -k "quad or tiled or large_sparse"'
CASES_Q='tests/test_gpu_pic_esirkepov.py -k "first_step or absorbing"'
CASES_C='tests/test_gpu_kernels.py -k "compaction_large_shift or (fused_step_matches_oracle and 300001)"'
CASES_X='tests/test_gpu_pic.py -k "quad and not sorted"'
CASES_Y='tests/test_gpu_dist.py -k "esirkepov"'
for tool in ${SAN_TOOLS:-memcheck racecheck synccheck}; do
  for grp in ${SAN_GROUPS:-K P D E R S F Q C X}; do   # (Y: memcheck / synccheck only; racecheck of thread ranks stalls the tool)
    eval cases=\$CASES_$grp
    eval timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --target-processes all \
      python -m pytest $cases -x -q -p no:cacheprovider > gpurun_out/sanitize_${tool}_$grp.log 2>&1
    echo "$tool $grp rc=$?  $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_${tool}_$grp.log | tr '\n' ' ' | cut -c1-200)"
  done
done
