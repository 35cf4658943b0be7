# ncu instruction/issue/pipe counters for one production fill per library build:
#   gpurun -- bash tools/ncu_ab.sh build/variants/a.so ...
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,dram__bytes_write.sum,dram__bytes_read.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum
for lib in "$@"; do
  echo "== $lib"
  ZF_LIB=$lib ncu --clock-control none -k regex:fill_ctr_kernel -c 2 --metrics $M --csv python tools/prof_fill.py normal 28 1 2>/dev/null | grep -v "^==PROF" | tail -n +1
done
