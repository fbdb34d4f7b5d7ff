import time, collections, sys
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2504_02067_b200 as ot
from paper_2504_02067_b200 import driver, dual, projector, _device
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0**5, 2.0**16)
acc = collections.defaultdict(float); cnt = collections.Counter()
def wrap(obj, name, label):
    f = getattr(obj, name)
    def w(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); acc[label] += time.perf_counter() - t0; cnt[label] += 1; return r
    setattr(obj, name, w)
wrap(dual.DualState, "_snapshot", "snapshot")
wrap(dual.DualState, "_extrapolate", "extrapolate")
wrap(dual.DualState, "set_targets", "set_targets")
wrap(_device.Context, "upload_rows_async", "upload_rows_async")
wrap(driver, "smooth_marginals", "smooth_marginals")
wrap(dual.DualState, "scale_rows_to_target", "scale_rows")
wrap(dual.DualState, "_grad_norm_l1_deferred", "gn_deferred")
wrap(dual.DualState, "rebalance_columns", "rebalance")
wrap(driver, "adjust_schedule", "adjust_schedule")
wrap(_device.Context, "call", "ctx.call(all)")
torch.cuda.synchronize()
t0 = time.perf_counter(); ot.mdot(dp, 2.0**5, 2.0**16); torch.cuda.synchronize(); T = time.perf_counter() - t0
print(f"total {T*1e3:.1f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{k:22s} {v*1e3:8.3f} ms  {cnt[k]:4d}  {v/cnt[k]*1e6:8.1f} us/call")
