#!/bin/bash
# ncu summaries of the streaming kernels next to k_coop: the row LSE and the
# plan materialization of the D2 solve (late-stage launches), and the
# on-the-fly pair kernel's product and log-sum-exp passes at n = 65536
# (FP64-pipe utilisation) -> gpurun_out/streams_ncu.txt.
mkdir -p gpurun_out
out=gpurun_out/streams_ncu.txt; : > $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum
python tools/profile_step.py > /dev/null || exit 1
echo "=== D2 solve (n=4096): k_lse_rows launch 160, k_materialize launch 40" >> $out
ncu --metrics $M --clock-control none -k regex:k_lse_rows --launch-skip 160 -c 1 python tools/profile_step.py 2>/dev/null | grep -E "k_lse|  [a-z]" >> $out
ncu --metrics $M --clock-control none -k regex:k_materialize --launch-skip 40 -c 1 python tools/profile_step.py 2>/dev/null | grep -E "k_mat|  [a-z]" >> $out
echo "=== pair kernel, n = 65536 3-D points (d5_pass order: MAXD, row LSE, row DOT, col LSE)" >> $out
python tools/d5_pass.py 65536 > /dev/null
ncu --metrics $M --clock-control none -k regex:k_pair -c 4 python tools/d5_pass.py 65536 2>/dev/null | grep -E "k_pair|  [a-z]" >> $out
