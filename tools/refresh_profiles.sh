#!/bin/bash
# Re-measure everything profiles/ holds for the D2 headline (run on the GPU box;
# outputs land in gpurun_out/, copied into profiles/ by hand after review):
#   bench line, ncu launch list, per-launch k_coop profile, host gaps, k_coop DRAM.
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/profile_step.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
python tools/launch_profile.py > gpurun_out/kcoop_launch_profile.txt 2>&1
python tools/gap_trace.py > gpurun_out/host_gaps_full.txt 2>&1
grep -A40 "^solve" gpurun_out/host_gaps_full.txt > gpurun_out/host_gaps.txt
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_coop --csv --log-file gpurun_out/kcoop_dram.csv \
    python tools/profile_step.py > /dev/null 2>&1
