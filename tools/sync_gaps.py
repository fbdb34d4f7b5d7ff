"""GPU idle caused by host turnaround, from the host side: after every
blocking C-ABI call (one that waited for the GPU, so the stream is drained)
the GPU idles until the host's next call enqueues work.  Sums that time per
(blocking call -> next call) pair over one D2 solve (diagnostic).

    python tools/sync_gaps.py [block_us]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200 import _device  # noqa: E402

block_us = float(sys.argv[1]) if len(sys.argv) > 1 else 25.0
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
orig = _device.Context.call
log = []


def traced(self, name, *args):
    t0 = time.perf_counter()
    r = orig(self, name, *args)
    log.append((name, t0, time.perf_counter()))
    return r


_device.Context.call = traced
for rep in range(3):
    log.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
agg = {}
total = 0.0
for (a, s0, e0), (b, s1, e1) in zip(log, log[1:]):
    if (e0 - s0) * 1e6 < block_us:
        continue                                   # a did not wait: the GPU still had work
    gap = (s1 - e0) * 1e6
    total += gap
    v = agg.setdefault((a, b), [0.0, 0])
    v[0] += gap
    v[1] += 1
print(f"solve {wall * 1e3:.2f} ms, {len(log)} calls; host turnaround after blocking calls "
      f"(GPU idle, plus the next call's enqueue latency): {total / 1e3:.2f} ms")
for (a, b), (us, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:16]:
    print(f"  {a:>22s} -> {b:<22s} {us / 1e3:7.3f} ms {c:5d}  ({us / c:6.1f} us each)")

# one stage boundary as the host sees it: the calls between two Newton steps
# of different stages, with the host time before each call and its duration
idx = [i for i, (n, _, _) in enumerate(log) if n == "otn_newton_step"]
best = max(range(1, len(idx)), key=lambda k: idx[k] - idx[k - 1])
i0, i1 = idx[best - 1], idx[best]
print(f"the stretch with the most calls between two otn_newton_step calls: {(log[i1][1] - log[i0][2]) * 1e6:.0f} us, "
      f"{i1 - i0 - 1} calls in between")
for k in range(i0, i1 + 1):
    n, s, e = log[k]
    gap = (s - log[k - 1][2]) * 1e6 if k > i0 else 0.0
    print(f"   +{gap:6.1f} us host, {n:<24s} {(e - s) * 1e6:7.1f} us in the call")
