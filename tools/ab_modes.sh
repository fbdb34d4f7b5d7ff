#!/bin/bash
# A/B of the column-block sparse mode (kPlanDual) against kPlanSparse on the
# D2 headline: per-mode launch profile and whole-solve time, each build.
set -x
for nd in 0 1; do
  OTN_NO_DUAL=$nd python tools/launch_profile.py grid:64:l2sq:0 2>&1 | tail -6
  OTN_NO_DUAL=$nd python tools/quick_time.py 2>&1 | tail -6
done
