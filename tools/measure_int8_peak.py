"""Measure the dense int8 tensor-core peak on this B200 with cuBLASLt
(torch._int_mm, int8 x int8 -> int32, 8192^3), best of 10, CUDA events.
Writes profiles/int8_peak.json, the roofline denominator for the kernels that
run on tcgen05 kind::i8."""
import datetime
import json
import os

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
tops = 2 * n ** 3 / (best / 1e3) / 1e12
out = {"int8_tops": tops, "best_ms": best, "n": n, "how": "torch._int_mm (cuBLASLt) 8192^3 best of 10",
       "when": datetime.datetime.now(datetime.timezone.utc).isoformat(), "gpu": torch.cuda.get_device_name()}
os.makedirs(os.path.join(REPO, "profiles"), exist_ok=True)
json.dump(out, open(os.path.join(REPO, "profiles", "int8_peak.json"), "w"), indent=1)
print(json.dumps(out))
