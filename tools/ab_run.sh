#!/bin/bash
# Run a timing tool against the in-tree library and each build/ab/*.so, interleaved twice.
#   tools/ab_run.sh "python tools/probe.py grid:64:l2sq:0 16"
cmd=$1
for round in 1 2; do
  echo "=== in-tree (round $round)"; $cmd 2>&1 | tail -${TAIL:-4}
  for so in build/ab/*.so; do
    echo "=== $so (round $round)"; OTN_LIB_AB=$so $cmd 2>&1 | tail -${TAIL:-4}
  done
done
