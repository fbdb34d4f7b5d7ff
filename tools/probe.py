"""Time the persistent solver's building blocks on a real D2 plan (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402
from paper_2504_02067_b200._device import vptr  # noqa: E402

p = ot.workload(sys.argv[1] if len(sys.argv) > 1 else "grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
NAMES = ["grid.sync", "grid_reduce<2>", "phase A", "phase B", "A+sync+A2+sync", "full HVP"]
for lg in [int(a) for a in (sys.argv[2:] or ["10", "16"])]:
    st = ot.mdot(dp, 2.0 ** 5, 2.0 ** lg).final_state
    s = ot.DiscountedSystem.from_state(st)
    k = s._ctx
    x = torch.randn(k.ld, dtype=torch.float64, device="cuda")
    out = k.vec()
    # streaming geometry the kernel derives from the mask (64-column segments)
    m = s._mask.cpu().numpy().view(np.uint64)
    nnz = m[: k.n, -1].astype(np.int64)
    m = m[: k.n, :-1]
    mw = m.shape[1]
    G = 148
    tot, wmax, nchs = 0, 0, []
    for b in range(G):
        r0, r1 = b * k.n // G, (b + 1) * k.n // G
        for ti in range(mw):
            bits = m[r0:r1, ti]
            nz = bits[bits != 0]
            if not len(nz):
                continue
            lo = np.array([(int(x) & -int(x)).bit_length() - 1 for x in nz]) * 64
            hi = np.array([int(x).bit_length() for x in nz]) * 64
            tot += int((hi - lo).sum())
            W = int(hi.max() - lo.min())
            wmax = max(wmax, W)
            nchs.append((W + 1023) // 1024)
    print(f"gamma=2^{lg} masked plan: span bytes {tot * 8 / 2**20:.1f} MiB, max window {wmax}, "
          f"nch histogram {np.bincount(nchs, minlength=5)[1:].tolist()}, nnz {int(nnz.sum())} "
          f"(max row {int(nnz.max())})", flush=True)
    k.call("otn_probe", vptr(s._P), vptr(s._mask), vptr(s._cP), vptr(s._rP), vptr(x), vptr(out), 0, 1)
    lay = np.zeros(G + 2, dtype=np.int32)
    k.call("otn_coop_layout", lay.ctypes.data)
    rows = np.diff(lay[: G + 1])
    cta_nnz = np.add.reduceat(nnz, lay[:G]) if rows.min() > 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    k.call("otn_probe", vptr(s._P), vptr(s._mask), vptr(s._cP), vptr(s._rP), vptr(x), vptr(out), 0, 1)
    e1.record()
    e1.synchronize()
    print(f"   mode {int(lay[G + 1])}  rows/CTA min {rows.min()} max {rows.max()}  nnz/CTA max "
          f"{None if cta_nnz is None else int(cta_nnz.max())}  launch+stage "
          f"{e0.elapsed_time(e1) * 1e3:.1f}us", flush=True)
    for mask in (s._mask, None):
        row = []
        for what in range(6):
            reps = 400
            def go():
                k.call("otn_probe", vptr(s._P), vptr(mask), vptr(s._cP), vptr(s._rP), vptr(x),
                       vptr(out), what, reps)
            go()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            go()
            e1.record()
            e1.synchronize()
            row.append(e0.elapsed_time(e1) / reps * 1e3)
        print(f"gamma=2^{lg} {'masked' if mask is not None else 'dense '}: " +
              "  ".join(f"{n} {t:6.2f}us" for n, t in zip(NAMES, row)), flush=True)
