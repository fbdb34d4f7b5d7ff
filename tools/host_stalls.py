"""Host-side stalls inside one D2 solve: the longest host intervals between
two consecutive C-ABI calls (the GPU idles through them when its queue is
empty), with the Python stack of the call that ended each (diagnostic).

    python tools/host_stalls.py [threshold_us]
"""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200 import _device  # noqa: E402

thr = float(sys.argv[1]) if len(sys.argv) > 1 else 200.0
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
orig = _device.Context.call
state = {"last": None, "last_name": "start"}
stalls = []
pairs = {}


def traced(self, name, *args):
    t = time.perf_counter()
    if state["last"] is not None:
        key = (state["last_name"], name)
        v = pairs.setdefault(key, [0.0, 0])
        v[0] += (t - state["last"]) * 1e6
        v[1] += 1
    if state["last"] is not None and (t - state["last"]) * 1e6 > thr:
        stalls.append(((t - state["last"]) * 1e6, state["last_name"], name,
                       "".join(traceback.format_stack(limit=7)[:-1])))
    r = orig(self, name, *args)
    state["last"] = time.perf_counter()
    state["last_name"] = name
    return r


_device.Context.call = traced
torch.cuda.synchronize()
for rep in range(3):
    stalls.clear()
    pairs.clear()
    state["last"] = None
    t0 = time.perf_counter()
    ot.mdot(dp, 2.0 ** 5, 2.0 ** 16)
    torch.cuda.synchronize()
    print(f"solve {rep}: {(time.perf_counter() - t0) * 1e3:.2f} ms wall, "
          f"{len(stalls)} host intervals > {thr:.0f} us, total {sum(s[0] for s in stalls) / 1e3:.2f} ms")
tot = sum(v[0] for v in pairs.values())
print(f"host time between calls (last solve): {tot / 1e3:.2f} ms over {sum(v[1] for v in pairs.values())} intervals")
for (a, b), (us, c) in sorted(pairs.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"  {a:>22s} -> {b:<22s} {us / 1e3:7.3f} ms {c:5d}  ({us / c:6.1f} us each)")
for us, a, b, stk in sorted(stalls, reverse=True)[:6]:
    print(f"--- {us:.0f} us between {a} and {b}:\n{stk}")
