"""Where does the GPU sit idle during one D2 solve?  Records a CUDA event
before and after every C-ABI call and reports, per call name, the idle time
between the previous call's last GPU work and the next call's first
(diagnostic: the events themselves add a little overhead)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200 import _device  # noqa: E402

p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
recs = []
orig = _device.Context.call


import time  # noqa: E402
import traceback  # noqa: E402


def traced(self, name, *args):
    host_t = time.perf_counter()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    r = orig(self, name, *args)
    b.record()
    recs.append((name, a, b, host_t, time.perf_counter(),
                 "".join(traceback.format_stack(limit=6)[:-1]) if name == "otn_rebalance_cols" else ""))
    return r


_device.Context.call = traced
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
e1.record()
torch.cuda.synchronize()
total = e0.elapsed_time(e1)
idle_before = collections.defaultdict(float)
busy = collections.defaultdict(float)
count = collections.Counter()
prev_end = e0
prev_name = "start"
worst = []
prev_host_end = None
for name, a, b, h0, h1, stk in recs:
    gap = prev_end.elapsed_time(a)
    if name == "otn_rebalance_cols":
        worst.append((gap, h0 - (prev_host_end or h0), prev_name, stk))
    prev_host_end = h1
    idle_before[(prev_name, name)] += max(gap, 0.0)
    busy[name] += a.elapsed_time(b)
    count[name] += 1
    prev_end, prev_name = b, name
worst.sort(key=lambda w: -w[0])
for g, hd, pn, stk in worst[:3]:
    print(f"gap {g:.3f} ms, host {hd * 1e3:.3f} ms after {pn}; stack:\n{stk}")
tail = prev_end.elapsed_time(e1)
print(f"solve {total:.2f} ms; sum of call spans {sum(busy.values()):.2f} ms; "
      f"gaps {sum(idle_before.values()) + tail:.2f} ms (tail {tail:.2f})")
print("largest gap sources (previous call -> next call): ms total, count")
pairs = collections.Counter()
for (pn, nn), ms in idle_before.items():
    pairs[(pn, nn)] = ms
for (pn, nn), ms in pairs.most_common(14):
    print(f"  {pn:>20s} -> {nn:<20s} {ms:7.2f} ms")
print("call spans (GPU time between the call's events): ms, count")
for name, ms in sorted(busy.items(), key=lambda kv: -kv[1]):
    print(f"  {name:<22s} {ms:8.2f} ms  {count[name]}")
