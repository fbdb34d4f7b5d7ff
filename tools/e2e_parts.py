"""Where the end-to-end (host numpy problem) time goes (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_02067_b200 as ot  # noqa: E402

p = ot.workload("grid:64:l2sq:0")
dev = torch.device("cuda", 0)
pinned = torch.empty(p.C.shape, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = p.C
for name, src in (("pageable", p.C), ("pinned", pinned.numpy())):
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = torch.from_numpy(src).to(dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(f"H2D {name}: {(t1 - t0) * 1e3:.1f} ms", flush=True)
for _ in range(2):
    t0 = time.perf_counter()
    h = d.cpu().numpy()
    t1 = time.perf_counter()
print(f"D2H pageable (.cpu()): {(t1 - t0) * 1e3:.1f} ms")
hp = torch.empty(p.C.shape, dtype=torch.float64, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hp.copy_(d)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
print(f"D2H pinned: {(t1 - t0) * 1e3:.1f} ms")
for name, prob in (("host pageable", p), ("host pinned", ot.Problem(C=pinned.numpy(), r=p.r, c=p.c))):
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ot.mdot(prob, 2.0 ** 5, 2.0 ** 16)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(f"mdot {name}: {(t1 - t0) * 1e3:.1f} ms", flush=True)
