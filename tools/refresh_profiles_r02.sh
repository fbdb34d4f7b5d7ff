#!/bin/bash
# Round-2 refresh of profiles/ (run on the GPU box; outputs in gpurun_out/):
# the bench line as the driver runs it, the reference arm, the ncu launch list
# of the bench command, per-launch k_coop profile, per-mode ncu captures and
# the k_coop DRAM traffic.  Each ncu pass only after the plain run exited 0.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err || exit 1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_reference.json 2> gpurun_out/r02_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/r02_launches.csv > gpurun_out/r02_launches_summary.txt
timeout 300 python tools/launch_profile.py > gpurun_out/r02_kcoop_launch_profile.txt 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_coop --csv --log-file gpurun_out/kcoop_dram.csv \
    python tools/profile_step.py > /dev/null 2>&1
timeout 900 bash tools/ncu_kcoop_modes.sh
timeout 300 python tools/idle_profile.py > gpurun_out/r02_idle_profile.txt 2>/dev/null
timeout 300 python tools/host_stalls.py 150 > gpurun_out/r02_host_stalls.txt 2>&1
echo refresh-done
