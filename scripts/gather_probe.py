"""Random-row gather roofline probe: time torch index_select of N random 64-B / 32-B / 128-B records from
a table far larger than L2 (the E4 access pattern), L2 flushed between reps."""
import torch

dev = torch.device("cuda")
fb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for rec_bytes, rows in ((32, 8_000_000), (64, 8_000_000), (128, 4_000_000)):
    tab = torch.randint(0, 2**31 - 1, (rows, rec_bytes // 4), dtype=torch.int32, device=dev)
    for n in (310_000, 1_240_000):
        idx = torch.randint(0, rows, (n,), device=dev)
        ts = []
        for r in range(6):
            fb.add_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = tab.index_select(0, idx)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        t = sorted(ts[1:])[len(ts[1:]) // 2]
        print(f"rec {rec_bytes:4d} B x {n:8d} random rows of {rows}: {t:7.1f} us  -> {n*rec_bytes/t/1e3:7.1f} GB/s useful, {n/t:6.1f} rows/ns")
    del tab
