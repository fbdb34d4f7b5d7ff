import sys, time, ctypes
sys.path.insert(0, '.')
import torch
from paper_2504_02067_b200 import _lib
from paper_2504_02067_b200._device import Context, vptr
k = Context.get(4096, torch.device("cuda", 0))
a = k.vec(); b = k.vec(); out = k.vec()
N = 20000
for mode in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if mode == 0:
        for _ in range(N):
            k.call("otn_vec", _lib.VEC_ADD, 0.0, vptr(a), vptr(b), None, None, vptr(out))
    else:
        f = k.lib.otn_vec; h = k.h; pa, pb, po = vptr(a), vptr(b), vptr(out)
        for _ in range(N):
            f(h, _lib.VEC_ADD, 0.0, pa, pb, None, None, po)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / N * 1e6
    print(["ctx.call", "raw ctypes"][mode], f"{dt:.2f} us/call")
