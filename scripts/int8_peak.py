"""Measured int8 tensor roof on this B200, two ways, each burst and sustained:

  * cuBLASLt int8 (torch._int_mm, s8 x s8 -> s32) at 8192^3, random operands: best of 10 CUDA-event timings
    (burst, the method MEASURED_PEAKS.json uses for bf16) and back to back for 4 s (sustained);
  * the tcgen05 issue-rate microbenchmark (scripts/int8_peak_tc.cu): cta_group::2 kind::i8 M=256 N=256 on every
    CTA pair, random operands in shared memory (no memory traffic): the tensor pipe's own rate.

SM clocks are sampled with nvidia-smi during each leg. Writes one JSON object (stdout and argv[1] if given);
bench.py reads the committed copy under profiles/r*/int8_peak.json.
"""
import json
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent


class Smi:
    def __init__(self):
        self.s = []
        self.p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                                   "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                  stderr=subprocess.DEVNULL, text=True)
        threading.Thread(target=self._r, daemon=True).start()

    def _r(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                self.s.append((float(parts[0]), float(parts[1]), parts[2]))
            except (ValueError, IndexError):
                pass

    def mark(self):
        return len(self.s)

    def summary(self, i0):
        xs = self.s[i0:]
        busy = [x for x in xs if x[1] > 300] or xs
        if not busy:
            return {}
        return {"sm_mhz_median": statistics.median(x[0] for x in busy), "power_w_max": max(x[1] for x in busy),
                "power_cap_samples": sum(1 for x in busy if x[2].lower().startswith("active")), "samples": len(busy)}


def main():
    smi = Smi()
    time.sleep(0.5)
    n = 8192
    a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    i0 = smi.mark()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    cub_burst = 2 * n ** 3 / best / 1e9
    c_burst = smi.summary(i0)
    i0 = smi.mark()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cnt = 0
    while time.perf_counter() - t0 < 4.0:
        for _ in range(10):
            torch._int_mm(a, b)
        cnt += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    cub_sus = 2 * n ** 3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
    c_sus = smi.summary(i0)
    del a, b
    torch.cuda.empty_cache()
    time.sleep(1.0)

    exe = REPO / "scripts" / "bin" / "int8_peak_tc"
    i0 = smi.mark()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    tc = json.loads(r.stdout.strip().splitlines()[-1])
    c_tc = smi.summary(i0)
    smi.p.terminate()
    out = {
        "cublas_i8_burst_tops": cub_burst, "cublas_i8_sustained_tops": cub_sus,
        "cublas_clocks": {"burst": c_burst, "sustained": c_sus},
        **tc, "tcgen05_clocks": c_tc,
        "gpu": torch.cuda.get_device_name(0),
        "how": "cuBLASLt int8 torch._int_mm 8192^3 random s8 (burst: best of 10 CUDA-event timings; sustained: back to back "
               ">= 4 s); tcgen05 microbenchmark scripts/int8_peak_tc.cu (cta_group::2 kind::i8 256x256x32 on all CTA "
               "pairs, random shared-memory operands; burst: best of 5 single ~5 ms launches; sustained: >= 4 s)",
    }
    out["int8_peak_burst_tops"] = max(cub_burst, out["tcgen05_i8_burst_tops"])
    out["int8_peak_sustained_tops"] = max(cub_sus, out["tcgen05_i8_sustained_tops"])
    s = json.dumps(out, indent=1)
    print(s)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(s + "\n")


if __name__ == "__main__":
    main()
