"""Device cost construction for the D3 pixel sets (n = 4096, d = 784):
otn_pixel_cost time (pack + u8 tensor-core GEMM + normalize) from device
point sets, against the host's numpy evaluation of the same cost."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_02067_b200 import problems  # noqa: E402

n, d = 4096, 784
X, Y = problems.pixel_points(n, d, 0)
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
for _ in range(3):
    problems.pixel_cost_device(Xd, Yd)
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    problems.pixel_cost_device(Xd, Yd)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
gop = 2.0 * n * n * d / 1e9
print(f"otn_pixel_cost n={n} d={d}: {ms * 1e3:.1f} us per cost (incl. the host sync), "
      f"GEMM {gop:.1f} GOP -> {gop / ms:.1f} TOP/s if the GEMM took it all")
t0 = time.perf_counter()
problems.dense_points_problem(n, d, 0, "pixel")
print(f"host numpy (incl. the point generation): {(time.perf_counter() - t0) * 1e3:.0f} ms, "
      f"{os.cpu_count()} cores")
