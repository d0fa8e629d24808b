"""Measured int8 tensor peak via cuBLASLt (torch._int_mm), same method as MEASURED_PEAKS.json's bf16 entry."""
import torch, json
n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
for _ in range(3):
    torch._int_mm(a, b)
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
x = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
for _ in range(3): x @ x
bb = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x @ x; e1.record(); torch.cuda.synchronize()
    bb = min(bb, e0.elapsed_time(e1))
print(json.dumps({"int8_tops_cublas_best_of_10": 2 * n**3 / best / 1e9, "bf16_tflops_best_of_10": 2 * n**3 / bb / 1e9}))
