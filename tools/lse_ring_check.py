"""Row LSE outputs on fixed inputs (ragged and full n, with and without the
trial direction), written to an .npz: run once per OTN_LSE_RING setting and
compare the files bit for bit (diagnostic for the cp.async ring variant)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_02067_b200._device import Context, vptr  # noqa: E402

out = {}
rng = np.random.default_rng(5)
for n in (4096, 1000, 300):
    k = Context.get(n, torch.device("cuda", 0))
    C = torch.zeros((n, k.ld), dtype=torch.float64, device="cuda")
    C[:, :n] = torch.from_numpy(rng.random((n, n)) * 50).cuda()
    for lg in (0, 6, 12):
        inner = k.vec(); inner[:n] = torch.from_numpy(rng.standard_normal(n) * 2.0 ** lg).cuda()
        d = k.vec(); d[:n] = torch.from_numpy(rng.standard_normal(n)).cuda()
        outer = k.vec(); outer[:n] = torch.from_numpy(rng.standard_normal(n)).cuda()
        for with_d in (False, True):
            o = k.vec()
            if with_d:   # symmetric trial sums: the row kernel with a direction term
                k.call("otn_trial_cols", vptr(C), 1, -(2.0 ** lg) / 50, vptr(outer), vptr(d),
                       vptr(inner), vptr(d), 0.37, vptr(o), None)
            else:
                k.call("otn_lse_rows", vptr(C), -(2.0 ** lg) / 50, vptr(outer), vptr(inner),
                       vptr(o))
            torch.cuda.synchronize()
            out[f"n{n}_g{lg}_d{int(with_d)}"] = o[:n].cpu().numpy()
np.savez(sys.argv[1], **out)
print("wrote", sys.argv[1], len(out))
