#!/bin/bash
# One `ncu --set full` capture of k_coop per plan mode of the D2 L2^2 solve
# (launch 12: dense ring, 30: global CSR/CSC, 40: shared CSR/CSC), summarised
# into gpurun_out/kcoop_modes_ncu.txt (copied to profiles/ after review).
mkdir -p gpurun_out
python tools/profile_step.py > /dev/null || exit 1
out=gpurun_out/kcoop_modes_ncu.txt; : > $out
for pair in "12:mode0_ring" "30:mode3_global_sparse" "40:mode2_smem_sparse"; do
  skip=${pair%%:*}; name=${pair##*:}
  ncu --set full --clock-control none --import-source on -k regex:k_coop --launch-skip $skip -c 1 \
      -o gpurun_out/kcoop_$name python tools/profile_step.py > /dev/null 2>&1
  echo "=== $name (k_coop launch $skip of the solve)" >> $out
  ncu -i gpurun_out/kcoop_$name.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h = rows[0]; r = rows[2]
for m in ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
          'lts__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
          'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
          'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
          'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread']:
    if m in h: print(f'  {m:62s} {r[h.index(m)]:>18s} {rows[1][h.index(m)]}')
" >> $out
  python tools/ncu_source.py gpurun_out/kcoop_$name.ncu-rep 12 2>/dev/null | head -30 >> $out
done
