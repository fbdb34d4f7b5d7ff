#!/bin/bash
# A/B of the row LSE: bitwise comparison of outputs and pass times, the
# in-tree library against build/ab/libotn_$1.so (tools/build_ab.sh).
OTN_LIB_AB=build/ab/libotn_$1.so timeout 120 python tools/lse_ring_check.py gpurun_out/lse_a.npz
timeout 120 python tools/lse_ring_check.py gpurun_out/lse_b.npz
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/lse_a.npz"), np.load("gpurun_out/lse_b.npz")
print("bitwise identical:", all(np.array_equal(a[k], b[k]) for k in a.files),
      [k for k in a.files if not np.array_equal(a[k], b[k])])
PY
echo "== A ($1)"; OTN_LIB_AB=build/ab/libotn_$1.so timeout 300 python tools/lse_bench.py 2>&1 | tail -6
echo "== B (in-tree)"; timeout 300 python tools/lse_bench.py 2>&1 | tail -6
