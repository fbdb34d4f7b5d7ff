import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_02067_b200 as ot
from paper_2504_02067_b200._device import vptr
p = ot.workload("grid:64:l2sq:0")
dp = ot.Problem(C=torch.from_numpy(p.C).cuda(), r=p.r, c=p.c)
st = ot.mdot(dp, 2.0 ** 5, 2.0 ** int(sys.argv[1])).final_state
s = ot.DiscountedSystem.from_state(st)
k = s._ctx
x = torch.randn(k.ld, dtype=torch.float64, device="cuda")
out = k.vec()
for rep in range(3):
    k.call("otn_probe", vptr(s._P), vptr(s._mask), vptr(s._cP), vptr(s._rP), vptr(x), vptr(out), 2, 50)
torch.cuda.synchronize()
d = out.cpu().numpy()[: 148 * 4].reshape(148, 4)
print("cols: max-thread cycles, its entries, its columns, E")
order = np.argsort(-d[:, 0])
for b in order[:10]:
    print(b, d[b].astype(int).tolist())
print("median", np.median(d, axis=0).astype(int).tolist())
