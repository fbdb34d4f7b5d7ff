"""GPU idle time inside one solve, from a CUPTI kernel trace (torch.profiler):
kernel / memcpy / memset intervals on the device, the gaps between them, and
the largest gap sources by (previous op -> next op) name (diagnostic; CUPTI
adds far less overhead than per-call events).

    python tools/idle_profile.py [spec] [log2 gamma_f]
"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "grid:64:l2sq:0"
gf = 2.0 ** (int(sys.argv[2]) if len(sys.argv) > 2 else 16)
p = ot.workload(spec)
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0 ** 5, gf)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ot.mdot(dp, 2.0 ** 5, gf)
    torch.cuda.synchronize()


def short(name):
    name = name.replace("void ", "").replace("otn::", "")
    return name.split("(")[0][:40]


ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"),
            key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
gaps = collections.defaultdict(float)
cnt = collections.Counter()
per_kernel = collections.defaultdict(float)
end = ev[0].time_range.start
prev = "start"
for e in ev:
    g = e.time_range.start - end
    if g > 0:
        gaps[(prev, short(e.name))] += g
        cnt[(prev, short(e.name))] += 1
    end = max(end, e.time_range.end)
    prev = short(e.name)
    per_kernel[short(e.name)] += e.time_range.end - e.time_range.start
print(f"{spec} gamma_f={gf:g}: first-to-last {span / 1e3:.2f} ms, device busy {busy / 1e3:.2f} ms, "
      f"idle {(span - busy) / 1e3:.2f} ms over {len(ev)} device ops")
print("largest idle sources (previous op -> next op): ms total, count")
for k, v in sorted(gaps.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {k[0]:>40s} -> {k[1]:<40s} {v / 1e3:7.3f} {cnt[k]:5d}")
print("largest single gaps (us): position in the op sequence, prev -> next")
single = []
end = ev[0].time_range.start
for i, e in enumerate(ev):
    g = e.time_range.start - end
    if g > 0 and i > 0:
        single.append((g, i, short(ev[i - 1].name), short(e.name),
                       (e.time_range.start - ev[0].time_range.start) / 1e3))
    end = max(end, e.time_range.end)
for g, i, a, b, t in sorted(single, reverse=True)[:12]:
    print(f"  {g:8.1f}  #{i:5d} at {t:7.2f} ms  {a} -> {b}")
print("device time per op: ms")
for k, v in sorted(per_kernel.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {k:<40s} {v / 1e3:8.3f}")
