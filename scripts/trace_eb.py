"""Per-warp timeline of the EmbeddingBag async kernel (debug instrumentation abftlp_debug_eb_trace).
usage: trace_eb.py E3|E4 [checked=1]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import runpy  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "E4"
checked = sys.argv[2] if len(sys.argv) > 2 else "1"
sys.argv = ["prof_eb.py", cfg, checked, "3"]
from paper_2103_00130_b200 import _lib as L  # noqa: E402
tr = torch.zeros(16 * 148 * 64, dtype=torch.int64, device="cuda")
L.lib.abftlp_debug_eb_trace.argtypes = [C.c_void_p]
L.lib.abftlp_debug_eb_trace(C.c_void_p(tr.data_ptr()))
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_eb.py"), run_name="__main__")
L.lib.abftlp_debug_eb_trace(None)
t = tr.cpu().numpy().reshape(-1, 16)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = lambda c: (t[:, c][t[:, c] > 0] - t0) / 1000.0  # noqa: E731
print(f"warps {len(t)}, bags/warp mean {t[:, 14].mean():.2f} max {t[:, 14].max()}")
for name, c in (("start", 0), ("bag0 begin", 1), ("bag0 first chunk", 2), ("bag0 end", 3), ("bag1 begin", 4),
                ("bag1 first chunk", 5), ("bag1 end", 6), ("bag2 end", 9), ("warp end", 13)):
    v = rel(c)
    if len(v):
        print(f"  {name:18s} n={len(v):5d} min {v.min():6.2f} med {np.median(v):6.2f} p90 {np.percentile(v, 90):6.2f} max {v.max():6.2f} us")
d = (t[:, 3] - t[:, 1]) / 1000.0
print(f"  bag0 duration: med {np.median(d):.2f} p90 {np.percentile(d, 90):.2f} max {d.max():.2f} us")
d2 = (t[:, 2] - t[:, 1]) / 1000.0
print(f"  bag0 begin->first chunk: med {np.median(d2):.2f} p90 {np.percentile(d2, 90):.2f} max {d2.max():.2f} us")
