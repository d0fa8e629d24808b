"""One grouped launch of the D5 MLP share at G=8 (for ncu): 9 problems m=8192, (k, n/8)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
m = 8192
keep = []
probs = (L.GemmProblem * 9)()
q = 0
for k in (512, 1024, 2048):
    for n in (512 // G, 1024 // G, 2048 // G):
        b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev)
        a = torch.randint(0, 256, (m, k), dtype=torch.uint8, device=dev)
        w = C.c_void_p()
        L.call("abftlp_gemm_encode", vp(b), k, n, n, st, C.byref(w))
        c, cs, fl, er = (torch.empty((m, n), dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int32, device=dev),
                         torch.empty(m, dtype=torch.uint8, device=dev), torch.zeros(1, dtype=torch.int32, device=dev))
        keep += [b, a, c, cs, fl, er]
        probs[q] = L.GemmProblem(a.data_ptr(), m, k, w.value, c.data_ptr(), n, cs.data_ptr(), 1, fl.data_ptr(), er.data_ptr())
        q += 1
grp = C.c_void_p()
L.call("abftlp_gemm_group_create", probs, 9, 1, C.byref(grp))
for _ in range(4):
    L.call("abftlp_gemm_group_run", grp, st)
torch.cuda.synchronize()
print("ok")
