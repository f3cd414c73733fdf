"""Sweep the host-entry split (PNN_HOST_DMA_IN / _OUT, PNN_HOST_THREADS,
PNN_HOST_PANELS) of pnn_matmul_host on config 1 (4096^3, posit(8,0) + (16,1)),
pinned uint64 Tensor storage, wall clock per call (best of 5).  One
subprocess per setting (the library reads the knobs once)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, time, json, numpy as np, torch
sys.path.insert(0, '.')
from paper_2105_00053_b200 import _native
L = _native.lib()
torch.set_num_threads(1)
M = N = K = 4096
res = {}
for (n, es) in [(8, 0), (16, 1)]:
    rng = np.random.default_rng(0)
    A = torch.from_numpy(rng.integers(0, (1 << n) - 1, (M, K)).astype(np.int64)).pin_memory()
    B = torch.from_numpy(rng.integers(0, (1 << n) - 1, (K, N)).astype(np.int64)).pin_memory()
    C = torch.empty((M, N), dtype=torch.int64).pin_memory()
    ts = []
    for _ in range(6):
        t0 = time.perf_counter()
        _native.check(L.pnn_matmul_host(n, es, A.data_ptr(), B.data_ptr(), C.data_ptr(), M, K, N))
        ts.append(time.perf_counter() - t0)
    res[f"{n},{es}"] = 1e3 * min(ts[1:])
print(json.dumps(res))
"""


def run(env):
    r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, cwd=REPO,
                       env=dict(os.environ, **{k: str(v) for k, v in env.items()}), timeout=600)
    if r.returncode:
        return {"error": r.stderr[-500:]}
    if r.stderr.strip():
        print(r.stderr.strip()[-3000:], file=sys.stderr, flush=True)
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    settings = []
    base = {"PNN_HOST_DMA_IN": 0.3, "PNN_HOST_DMA_OUT": 0.3, "PNN_HOST_THREADS": 16, "PNN_HOST_PANELS": 4}
    settings.append(dict(base, PNN_HOST_DMA_IN=0, PNN_HOST_DMA_OUT=0))
    for fi in (0.2, 0.3, 0.4, 0.5):
        settings.append(dict(base, PNN_HOST_DMA_IN=fi))
    for fo in (0.0, 0.2, 0.4, 0.5):
        settings.append(dict(base, PNN_HOST_DMA_OUT=fo))
    for th in (8, 12, 14):
        settings.append(dict(base, PNN_HOST_THREADS=th))
    for pn in (2, 8):
        settings.append(dict(base, PNN_HOST_PANELS=pn))
    if len(sys.argv) > 1:
        settings = [json.loads(a) for a in sys.argv[1:]]
    for s in settings:
        r = run(s)
        tot = r.get("8,0", 0) + r.get("16,1", 0)
        print(json.dumps({"env": s, "ms": r, "total_ms": round(tot, 3)}), flush=True)


if __name__ == "__main__":
    main()
