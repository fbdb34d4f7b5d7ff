#!/bin/bash
# A/B of the column-block sparse kernel (k_coop<true>, kPlanDual; OTN_DUAL=1)
# against the classic kernel on the D2 headline: per-mode launch profile and
# whole-solve time.
set -x
for d in 0 1; do
  OTN_DUAL=$d timeout 300 python tools/launch_profile.py grid:64:l2sq:0 2>&1 | tail -8
  OTN_DUAL=$d timeout 300 python tools/quick_time.py 2>&1 | tail -6
done
