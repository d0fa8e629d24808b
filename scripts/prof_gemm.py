"""Profiling driver: runs one GEMM configuration a few times (for ncu / timing).
usage: prof_gemm.py M N K [checked=1] [iters=5] [tiling]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
checked = int(sys.argv[4]) if len(sys.argv) > 4 else 1
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 5
if len(sys.argv) > 6:
    os.environ["ABFTLP_GEMM_TILING"] = sys.argv[6]
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
a = torch.randint(0, 256, (m, k), dtype=torch.int32, device=dev).to(torch.uint8)
b = torch.randint(-128, 128, (k, n), dtype=torch.int32, device=dev).to(torch.int8)
w = C.c_void_p()
L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
c = torch.zeros((m, n), dtype=torch.int32, device=dev)
cs = torch.zeros(m, dtype=torch.int32, device=dev)
fl = torch.zeros(m, dtype=torch.uint8, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
for _ in range(iters):
    if checked:
        L.call("abftlp_gemm_checked", vp(a), m, k, w, vp(c), n, vp(cs), 1, vp(fl), vp(err), None, st)
    else:
        L.call("abftlp_gemm_unchecked", vp(a), m, k, w, vp(c), n, st)
torch.cuda.synchronize()
ref = (a[:4].double() @ b.double()).round().long()
assert torch.equal(c[:4].long(), ref), "mismatch"
print("ok", int(err.item()))
