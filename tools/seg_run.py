"""Per-segment cycle breakdown of the CG iteration per plan mode (CTA 0):
    python tools/make_seg_build.py && OTN_LIB_AB=build/ab/libotn_seg.so python tools/seg_run.py"""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2504_02067_b200 as ot
from paper_2504_02067_b200 import _lib
lib = _lib.load()
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
ot.mdot(dp, 2.0**5, 2.0**16)
buf = (ctypes.c_ulonglong * 48)()
lib.otn_dbg_seg(buf)
sol = ot.mdot(dp, 2.0**5, 2.0**16)
lib.otn_dbg_seg(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 12).astype(float)
names = ["loop top", "a2_sums", "rz reduce_end", "a2_tail", "pq reduce_begin", "phase B",
         "pq reduce_end", "vector updates", "stage_x", "phase A", "rz reduce_begin", "-"]
hv = {0: 414, 2: 2025, 3: 658}
for m in (0, 2, 3):
    tot = a[m].sum()
    print(f"mode {m}: total {tot/1.965e3/1e3:.2f} ms  ({tot/1.965e3/hv[m]:.2f} us per hvp approx)")
    for i, nm in enumerate(names[:11]):
        print(f"   {nm:18s} {a[m][i]/1.965e3/hv[m]:7.2f} us/it")

# per-CTA balance: work between exchanges vs wait inside them (thread 0 of every CTA)
if hasattr(lib, "otn_dbg_cta"):
    ot.mdot(dp, 2.0**5, 2.0**16)
    cb = (ctypes.c_ulonglong * 3072)()
    lib.otn_dbg_cta(cb)
    sol = ot.mdot(dp, 2.0**5, 2.0**16)
    lib.otn_dbg_cta(cb)
    c = np.frombuffer(cb, dtype=np.uint64).reshape(3, 4, 256).astype(float)[:, :, :148]
    for m in (0, 2, 3):
        work, wait, nex = c[0][m], c[1][m], c[2][m]
        if nex.max() == 0:
            continue
        ne = nex.max()
        w = work / ne / 1.965e3
        t = wait / ne / 1.965e3
        print(f"mode {m}: {int(ne)} exchanges; work per exchange interval us: mean {w.mean():.2f} "
              f"max {w.max():.2f} (CTA {int(w.argmax())}) min {w.min():.2f}; wait mean {t.mean():.2f} "
              f"min {t.min():.2f}")
        print("   slowest CTAs:", [(int(i), round(float(w[i]), 2)) for i in np.argsort(-w)[:6]])
