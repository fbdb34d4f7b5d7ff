#!/bin/bash
# Per-kernel total GPU time of one D2 solve (ncu launch list), for the in-tree
# library and each build/ab/*.so:  tools/kernel_times.sh [regex]
re=${1:-.}
run() {
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$re" --csv \
      --log-file gpurun_out/kt_$1.csv python tools/profile_step.py > /dev/null 2>&1
  echo "=== $1"; python tools/ncu_launches.py gpurun_out/kt_$1.csv | head -12
}
mkdir -p gpurun_out
python tools/profile_step.py > /dev/null
run intree
for so in build/ab/*.so; do n=$(basename $so .so); OTN_LIB_AB=$so run $n; done
