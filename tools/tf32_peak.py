"""Measure the TF32 tensor peak on this box the way MEASURED_PEAKS.json measures bf16
(BASELINE.md section 4 / SURVEY 8(d) "Peaks"): torch.matmul on fp32 8192^3 with
allow_tf32, best of 10 (burst) and back to back for 4 s (sustained).  cuBLAS is used
here only as a measuring stick for the roofline denominator, never on the product path.

  python tools/tf32_peak.py > profiles/r02_tf32_peak.json
"""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
c = torch.empty(n, n, device="cuda")
flop = 2.0 * n ** 3
for _ in range(5):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = flop / (best * 1e-3) / 1e12
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        torch.matmul(a, b, out=c)
    cnt += 20
    torch.cuda.synchronize()
e1.record(); e1.synchronize()
sus = flop * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
# which kernel cuBLAS picked (name only) for the record
print(json.dumps({"tf32_tflops_burst": round(burst, 1), "tf32_tflops_sustained": round(sus, 1),
                  "how": "torch.matmul fp32 8192^3, allow_tf32=True: best of 10 (burst), back to back 4 s (sustained)",
                  "gpu": torch.cuda.get_device_name(), "torch": torch.__version__}))
