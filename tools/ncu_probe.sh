#!/bin/bash
# ncu metrics of one probe launch (tools/probe_one.py) for the in-tree library and
# each build/ab/*.so:  tools/ncu_probe.sh <what> <masked> <log2 gamma> [metrics]
what=$1; masked=$2; lg=$3
metrics=${4:-gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum}
for so in "" build/ab/*.so; do
  n=$(OTN_LIB_AB=$so python tools/probe_one.py $what $masked $lg | awk '/coop_launches_before_probe/{print $2}')
  echo "=== ${so:-in-tree} probe what=$what masked=$masked lg=$lg (skip $n)"
  OTN_LIB_AB=$so ncu --clock-control none -k regex:k_coop -s $n -c 1 --metrics $metrics \
      python tools/probe_one.py $what $masked $lg 2>&1 | grep -E "^\s+(gpu__|smsp__|lts__|sm__|l1tex__)"
done
