"""Profiling driver for the grouped G2 launch: `nb` runs of m=256 k=4096 n=4096 against one encoded weight in
ONE abftlp_gemm_checked_batched launch, repeated `iters` times (for ncu / timing).
usage: prof_grouped.py [nb=100] [checked=1] [iters=4]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_00130_b200 import _lib as L  # noqa: E402

M, N, K = 256, 4096, 4096
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 100
checked = int(sys.argv[2]) if len(sys.argv) > 2 else 1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
dev = torch.device("cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
b = torch.empty((K, N), dtype=torch.int8, device=dev)
L.call("abftlp_generate", vp(b), K * N, 20260823, 1000, 0, 1, 0.0, 0.0, 0, st)
w = C.c_void_p()
L.call("abftlp_gemm_encode", vp(b), K, N, N, st, C.byref(w))
a = torch.empty((nb, M, K), dtype=torch.uint8, device=dev)
L.call("abftlp_generate", vp(a), nb * M * K, 20260823, 0, 0, 0, 0.0, 0.0, 0, st)
c = torch.empty((nb, M, N), dtype=torch.int32, device=dev)
cs = torch.empty((nb, M), dtype=torch.int32, device=dev)
fl = torch.empty((nb, M), dtype=torch.uint8, device=dev)
err = torch.zeros(nb, dtype=torch.int32, device=dev)
for _ in range(iters):
    if checked:
        L.call("abftlp_gemm_checked_batched", vp(a), nb, M, K, M * K, w, vp(c), N, M * N, vp(cs), 1, M, vp(fl), M,
               vp(err), None, st)
    else:
        L.call("abftlp_gemm_unchecked_batched", vp(a), nb, M, K, M * K, w, vp(c), N, M * N, st)
torch.cuda.synchronize()
ref = (a[nb - 1, :4].double() @ b.double()).round().long()
assert torch.equal(c[nb - 1, :4].long(), ref), "mismatch"
assert int(err.sum().item()) == 0
print("ok")
