#!/usr/bin/env python
"""Benchmark: exact posit-quire MAC/s on BASELINE config 1.

Workload (BASELINE.json configs[1]): C = round(A.B) with A, B 4096x4096 packed
posit codes drawn uniformly over all non-NaR codes from a seed, exact quire
accumulation -- once in posit(8,0), then repeated in posit(16,1).  One "step"
is that whole config-1 pass (both GEMMs, 2 x 4096^3 exact posit MACs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun): the GEMM microbench does not shard (SURVEY.md §8e "replicas
only"); every rank runs the full workload on its own GPU, value = all ranks'
MACs / max-over-ranks device time.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libpnn_ref.so, the unmodified reference built from its sources)
with every host thread, on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

M = N = K = 4096
FORMATS = [(8, 0), (16, 1)]
METRIC = "exact posit-quire MAC/s"
UNIT = "posit-MAC/s"
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def workload_config(world: int) -> dict:
    """The `config` both arms print (ours and --impl reference): the same workload."""
    return {"workload": "BASELINE config 1: exact quire GEMM C=round(A.B), "
                        "M=N=K=4096, posit(8,0) then posit(16,1)",
            "M": M, "N": N, "K": K, "formats": ["posit(8,0)", "posit(16,1)"],
            "l2": "flushed between timed steps (512 MiB write, untimed)",
            "parallelism": f"replicas x{world}"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-train", action="store_true", help="skip the CNN training images/s leg")
    return p.parse_args()


def rank_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def gen_codes(fmt, seed):
    """Uniform over all non-NaR codes of the format (config 1)."""
    n, _ = fmt
    rng = np.random.default_rng(seed)
    nar = 1 << (n - 1)
    A = rng.integers(0, (1 << n) - 1, (M, K), dtype=np.int64)
    B = rng.integers(0, (1 << n) - 1, (K, N), dtype=np.int64)
    A += A >= nar  # skip the NaR pattern: map [0, 2^n - 1) onto non-NaR codes
    B += B >= nar
    return A.astype(np.uint64), B.astype(np.uint64)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def int8_peak(L=None):
    """Dense int8 tensor-pipe peak (TOPS) measured on this GPU: the tcgen05
    kind::i8 probe (pnn_probe_int8_peak: back-to-back 128x256x32 MMAs from
    shared memory on every SM, CUDA events), else profiles/int8_peak.json
    (cuBLASLt int8 GEMM), else 2x the measured bf16 burst figure."""
    if L is not None:
        tops, ms = C.c_double(), C.c_double()
        if L.pnn_probe_int8_peak(20000, C.byref(tops), C.byref(ms)) == 0:
            return tops.value, (f"measured tensor-pipe ceiling: tcgen05 kind::i8 probe, 148 SMs x "
                                f"20000 MMAs 128x256x32, {ms.value:.2f} ms")
    p = os.path.join(REPO, "profiles", "int8_peak_cublaslt.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["int8_tops"], f"measured cuBLASLt int8 GEMM (torch._int_mm 8192^3, {d.get('when', '')})"
    mp = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        return 2 * json.load(open(mp))["bf16_tflops"], "2x MEASURED_PEAKS bf16_tflops (int8 = fp8 rate)"
    return 2 * 1590.0, "2x fallback bf16 1.59 PFLOP/s (B200_PROFILING.md)"


_REF_CACHE = {}


def ncu_traffic(kernel_prefix: str):
    """DRAM bytes (read + write) per launch of the kernel from the committed
    `ncu --set full` capture summaries (profiles/ncu_full_r02.json, else r01)."""
    for name in ("ncu_full_r02.json", "ncu_full_r01.json"):
        p = os.path.join(REPO, "profiles", name)
        if not os.path.exists(p):
            continue
        for rep, ks in json.load(open(p)).items():
            for k in ks:
                if k["kernel"].startswith(kernel_prefix) and "dram_traffic_bytes" in k:
                    return {"bytes_per_launch": k["dram_traffic_bytes"], "source": f"profiles/{name}:{rep}"}
    return None


def run_cpu_reference_sample(rows: int, threads: int, cols: int = N):
    """Reference matmul (oracle/_ref, unmodified reference) on the first
    rows x cols outputs of the config-1 GEMM (full K = 4096 dot length)."""
    from oracle import bind

    ref = bind.Reference()
    total_macs, total_t = 0, 0.0
    for fmt in FORMATS:
        key = (fmt, rows, cols)
        if key not in _REF_CACHE:
            A, B = gen_codes(fmt, seed=2105 + fmt[0])
            _REF_CACHE[key] = (np.ascontiguousarray(A[:rows]), np.ascontiguousarray(B[:, :cols]))
        A, B = _REF_CACHE[key]
        t, _ = ref.time_matmul(fmt[0], fmt[1], A, B, threads)
        total_macs += rows * K * cols
        total_t += t
    return total_macs / total_t, total_t


TRAIN_PER_GPU_BATCH = 1024


def run_training(args, rank, world, dev, dist):
    """Second half of the BASELINE metric: CIFAR-shape CNN training images/s
    (configs 3/4: stages fwd posit(8,1), grads posit(12,1), loss/optimizer
    posit(16,1), all with quires), weak scaling at 1024 images per GPU.  One
    GPU replays a CUDA-graph-captured step; N > 1 runs the data-parallel step
    (raw quire words -> 60-bit lanes -> one NCCL all-reduce -> round once).
    Device time (CUDA events) of K steps after W warm-ups, max over ranks."""
    import torch

    from paper_2105_00053_b200 import codec, dp, nn, ops

    st = nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161)
    B = TRAIN_PER_GPU_BATCH
    rng = np.random.default_rng(3 + rank)  # this rank's shard of the synthetic global batch
    x = codec.from_float64_device(rng.uniform(-1.0, 1.0, (B, 3, 32, 32)), st.forward)
    lab = torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).to(dev)
    model = nn.cifar_cnn(st, seed=7)
    loss_fn = nn.CrossEntropyLoss(st)
    opt = nn.SGD(model.params(), 1.0 / 16, st)
    gb = B * world
    if world == 1:
        g = nn.GraphedTrainStep(model, loss_fn, opt, x, lab, B, warmup=1)
    else:  # the data-parallel step, NCCL all-reduce of quire lanes inside the graph
        reducer = dp.QuireAllReduce(model.params(), st.gradient)
        g = nn.GraphedTrainStep(model, loss_fn, opt, x, lab, gb, warmup=1,
                                step_fn=lambda: dp.dp_train_step(model, loss_fn, opt, reducer, x, lab, gb))
    graphed = True
    try:
        g.step()  # eager warm-up
        g.step()  # capture + first replay
        one = g.step
    except Exception:  # capture unsupported here: same step, eager
        graphed = False
        torch.cuda.synchronize(dev)
        one = g.step_fn
    steps = max(5, min(args.steps, 50))
    for _ in range(max(args.warmup, 3)):
        one()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        one()
    b.record()
    torch.cuda.synchronize(dev)
    t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
    if dist:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / steps
    out = {"workload": "BASELINE config 3/4 CIFAR-shape CNN (conv 3-32-32-pool-64-64-pool, "
                       "Linear 4096-512-10) full SGD step, fwd posit(8,1), grad posit(12,1), "
                       "loss/optimizer posit(16,1), quires everywhere",
           "metric": "CNN training images/s", "value": gb / (ms / 1000.0), "unit": "images/s",
           "ms_per_step": ms, "global_batch": gb, "per_gpu_batch": B, "steps": steps,
           "scaling": "weak", "cuda_graph": graphed,
           "parallelism": f"dp{world}" + (" (quire-lane NCCL all-reduce)" if world > 1 else ""),
           "data": "synthetic uniform [-1,1) images, uniform labels (seeded per rank)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import bind

        if bind.reference_available():
            import importlib.util

            spec = importlib.util.spec_from_file_location("bench_train", os.path.join(REPO, "tools", "bench_train.py"))
            bt = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(bt)
            from oracle.step import CIFAR_CNN, oracle_step

            threads = os.cpu_count() or 1
            Bc = 16
            xc = codec.to_host(x[:Bc])
            labc = lab[:Bc].cpu().numpy()
            params0 = [(codec.to_host(l.w.master), codec.to_host(l.b.master))
                       for l in nn.cifar_cnn(st, seed=7).layers if isinstance(l, nn.Conv2d)]
            std = {k: (getattr(st, k).nbits, getattr(st, k).es)
                   for k in ("forward", "backward", "gradient", "optimizer", "loss")}
            t0 = time.perf_counter()
            oracle_step(bt.HybridRef(threads), CIFAR_CNN, std, params0, xc, labc, 1.0 / 16, Bc)
            tc = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": Bc / tc, "unit": "images/s", "cores": threads,
                                   "kind": "reference",
                                   "sample": f"one SGD step of the same CNN at batch {Bc}: reference "
                                             f"tensor kernels (oracle/_ref) + restated elementwise, "
                                             f"{tc:.1f} s"}
    return out


def run_reference_impl(args):
    rank, _, world = rank_info()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rows, cols = max(16, threads), 1024  # >= one row per worker (ThreadPool splits rows)
    for _ in range(min(args.warmup, 3)):
        run_cpu_reference_sample(rows, threads, cols)
    vals, tsum = [], 0.0
    for _ in range(args.steps):
        v, t = run_cpu_reference_sample(rows, threads, cols)
        vals.append(v)
        tsum += t
    value = float(np.mean(vals))
    sample = (f"outputs [0:{rows}, 0:{cols}] of the 4096^3 GEMM (full K=4096 quire dots) per "
              f"format (8,0),(16,1) = {2 * rows * K * cols / 1e9:.3f} G exact MACs per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tsum / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int (posit codes)",
        "data": "synthetic (seeded uniform non-NaR codes)",
        "config": workload_config(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample + " (reference ThreadPool row split)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_impl(args)
    import torch

    from paper_2105_00053_b200 import _native, ops

    rank, local, world = rank_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    L = _native.lib()

    # ---- inputs resident in HBM (seeded, identical on every rank) ----
    data = {}
    for fmt in FORMATS:
        cfg = ops.PositConfig(*fmt)
        A, B = gen_codes(fmt, seed=2105 + fmt[0])
        dA = torch.from_numpy(A.astype(cfg.np_code_dtype)).to(dev)
        dB = torch.from_numpy(B.astype(cfg.np_code_dtype)).to(dev)
        dC = torch.empty((M, N), dtype=cfg.code_dtype, device=dev)
        ws = torch.empty(ops.quire_gemm_workspace(cfg, M, N, K), dtype=torch.uint8, device=dev)
        data[fmt] = (cfg, A, B, dA, dB, dC, ws)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        for fmt in FORMATS:
            cfg, _, _, dA, dB, dC, ws = data[fmt]
            _native.check(L.pnn_quire_gemm(cfg.nbits, cfg.es, dA.data_ptr(), dB.data_ptr(),
                                           dC.data_ptr(), M, N, K, ws.data_ptr(), ws.numel(), sptr))

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, L2 flushed (untimed) between steps ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    macs_per_step = len(FORMATS) * M * N * K
    value = world * args.steps * macs_per_step / (t_ms / 1000.0)

    # ---- per-kernel device times (CUDA events on the launch stream) ----
    per_fmt = {}
    for fmt in FORMATS:
        cfg, _, _, dA, dB, dC, ws = data[fmt]
        reps = []
        for _ in range(3):
            flush.fill_(1)
            ms = (C.c_float * 3)()
            _native.check(L.pnn_quire_gemm_profiled(cfg.nbits, cfg.es, dA.data_ptr(), dB.data_ptr(),
                                                    dC.data_ptr(), M, N, K, ws.data_ptr(), ws.numel(),
                                                    sptr, ms))
            reps.append(list(ms))
        pack, mma, fin = (float(np.mean([r[i] for r in reps])) for i in range(3))
        per_fmt[fmt] = {"pack_ms": pack, "mma_ms": mma, "finalize_ms": fin,
                        "total_ms": pack + mma + fin,
                        "posit_mac_per_s": M * N * K / ((pack + mma + fin) / 1000.0)}
    # dominant kernel: the tcgen05 MMA kernel of the slowest format
    dom = max(FORMATS, key=lambda f: per_fmt[f]["mma_ms"])
    ncfg = data[dom][0]
    D = {8: 2, 16: 8}[ncfg.nbits] if ncfg.es <= 1 else None
    int8_ops = 2.0 * M * N * K * D * D  # algorithmic int8 ops per launch (D^2 digit MMAs / MAC)
    achieved = int8_ops / (per_fmt[dom]["mma_ms"] / 1000.0) / 1e12
    peak, peak_src = int8_peak(L)
    traffic = ncu_traffic(f"quire_gemm_tc_kernel<{D}, {4 if ncfg.nbits > 8 else 1}, "
                          f"{'unsigned short' if ncfg.nbits > 8 else 'unsigned char'}")

    # ---- e2e through the reference-facing host API (uint64 Tensor storage) ----
    e2e = None
    if not args.no_e2e:
        host = {}
        for fmt in FORMATS:
            cfg, A, B = data[fmt][:3]
            pa = torch.from_numpy(A.view(np.int64)).pin_memory()
            pb = torch.from_numpy(B.view(np.int64)).pin_memory()
            pc = torch.empty((M, N), dtype=torch.int64).pin_memory()
            host[fmt] = (cfg, pa, pb, pc)

        def e2e_step():
            for fmt in FORMATS:
                cfg, pa, pb, pc = host[fmt]
                _native.check(L.pnn_matmul_host(cfg.nbits, cfg.es, pa.data_ptr(), pb.data_ptr(),
                                                pc.data_ptr(), M, K, N))

        # torch's own CPU worker threads (used by pin_memory above) must not spin
        # against the library's host pool inside the timed region
        torch.set_num_threads(1)
        for _ in range(3):
            e2e_step()
        e_steps = max(1, min(args.steps, 10))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        te = time.perf_counter() - t0
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
        # spot-check the e2e result against the device path
        for fmt in FORMATS:
            cfg, pa, pb, pc = host[fmt]
            dC = data[fmt][5]
            assert (pc[:64].numpy().astype(np.uint64) == dC[:64].cpu().numpy().astype(np.uint64)).all()
        e2e = {"value": world * e_steps * macs_per_step / te, "unit": UNIT,
               "h2d_bytes_per_step": sum(2 * M * K * 8 for _ in FORMATS),
               "d2h_bytes_per_step": sum(M * N * 8 for _ in FORMATS),
               "path": "pnn_matmul_host: uint64 code arrays (reference Tensor storage, pinned) -> "
                       "host-thread AVX-512 narrow to packed codes, chunked H2D overlapped -> quire GEMM -> "
                       "chunked D2H overlapped with host-thread widen (streaming stores); wall clock (bound by host "
                       "memory traffic of the 8-byte-per-code storage)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import bind

        if bind.reference_available():
            threads = os.cpu_count() or 1
            rows = 128
            v, tcpu = run_cpu_reference_sample(rows, threads)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"rows 0..{rows - 1} of A x full B (4096x4096), posit(8,0) and (16,1): "
                             f"{2 * rows * K * N / 1e9:.2f} G exact MACs in {tcpu:.1f} s "
                             f"(oracle/_ref/libpnn_ref.so matmul, ThreadPool({threads}))"}

    training = None
    if not args.no_train:
        try:  # the config-1 line above must survive a failure of the training leg
            training = run_training(args, rank, world, dev, dist)
        except Exception as e:  # noqa: BLE001
            training = {"metric": "CNN training images/s", "error": f"{type(e).__name__}: {e}"[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8 digit MMA -> exact int quire",
            "data": "synthetic (seeded uniform over non-NaR codes)",
            "config": workload_config(world),
            "per_format": {f"posit({f[0]},{f[1]})": per_fmt[f] for f in FORMATS},
            "roofline": {"bound": "tensor", "kernel": f"quire_gemm_tc_kernel posit({dom[0]},{dom[1]})",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak,
                         "traffic": traffic["bytes_per_launch"] if traffic else None,
                         "traffic_unit": "bytes/launch (dram read+write, ncu --set full)",
                         "traffic_source": traffic["source"] if traffic else None,
                         "note": f"int8 tensor ops (2/MAC) on tcgen05 kind::i8, {D}x{D} digit "
                                 f"MMAs per posit MAC; peak = {peak_src}"},
            # per step: 2 packs + MMA kernel per format, + the posit(16,1) 4-digit variant
            # (launched, exits on the device flag); profiles/launches_r02_bench.json
            "gpu_launches": args.steps * (len(FORMATS) * 3 + 1),
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        if training:
            line["training"] = training
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
