#!/bin/bash
# Full ncu capture (with source) of one probe launch: tools/ncu_probe_full.sh <what> <masked> <lg> <out>
what=$1; masked=$2; lg=$3; out=$4
n=$(python tools/probe_one.py $what $masked $lg | awk '/coop_launches_before_probe/{print $2}')
ncu --set full --import-source on --clock-control none -k regex:k_coop -s $n -c 1 -f -o $out \
    python tools/probe_one.py $what $masked $lg > /dev/null 2>&1
echo "captured $out (skip $n)"
