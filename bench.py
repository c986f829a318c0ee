#!/usr/bin/env python
"""Benchmark of the butterfly merge (BASELINE.json metric: params merged/sec).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N=1 workload: BASELINE config 2 — one 1B-parameter pipeline stage, 16 miners,
fp32 wire values, redundancy 2, on one B200 (the largest single-GPU config; the
reference's own CPU-runnable config 1 is a parity-test case).  A "step" is one
merge round: reduce every shard over the alive replicas (fp64 sequential
accumulation), compare redundant copies, adopt, scatter back in place into all
16 replicas.  Inputs are 64 GB of replicas, far larger than the 126 MB L2, so
no flush is needed between steps.

One JSON line on rank 0 (see DESIGN.md §Measurement for every field).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "params merged/sec (GB/s) at 1/2/4/8 B200 vs HBM/NVLink roofline and CPU ref"
UNIT = "params/s"

CONFIGS = {
    # name: (miners, params, dtype, redundancy, deceptive)
    "c1": (8, 10_000_000, "fp32", 2, 0),
    "c2": (16, 1_000_000_000, "fp32", 2, 0),
    "c3": (64, 1_000_000_000, "fp32", 2, 0),
    "c4": (32, 1_750_000_000, "bf16", 3, 0),
    "c5": (64, 1_000_000_000, "fp32", 2, 6),
}
WORKLOAD = {
    "c1": "reference default: butterfly merge 8 miners x 10M fp32, r=2",
    "c2": "1B-param stage, 16 miners fp32, r=2, 1 B200 (BASELINE config 2)",
    "c3": "1B-param stage, 64 miners across the GPUs, r=2 (BASELINE config 3)",
    "c4": "14B model / 8 stages: 1.75B-param stage, 32 miners bf16 (fp32 acc), r=3 (BASELINE config 4)",
    "c5": "1B-param stage, 64 miners, 6 deceptive (noise), r=2 (BASELINE config 5)",
}


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self._t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------


def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc  # test infrastructure: timed here only as the CPU baseline

    return orc


def cpu_sample(cfg, p_cpu: int, reps: int = 2):
    """Time the C oracle (restatement of run_all_reduce) with all host threads."""
    import numpy as np

    orc = _oracle()
    n, _, dtype, r, _ = cfg
    threads = orc.threads_available()
    rng = np.random.default_rng(0)
    if dtype == "bf16":
        replicas = [(rng.uniform(-1, 1, p_cpu).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
                    for _ in range(n)]
        odt = orc.BF16
    else:
        replicas = [rng.uniform(-1, 1, p_cpu).astype(np.float32) for _ in range(n)]
        odt = orc.F32
    assign, bounds = orc.plan(n, p_cpu, 0, r=r)
    orc.merge(replicas, assign, bounds, dtype=odt, threads=threads)  # warm
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        orc.merge(replicas, assign, bounds, dtype=odt, threads=threads)
        best = min(best, time.perf_counter() - t)
    return p_cpu / best, threads, best


# ---------------------------------------------------------------------------
# device path
# ---------------------------------------------------------------------------


def make_replicas(n, P, dtype, dev, seed=0):
    import torch

    g = torch.Generator(device=dev)
    out = []
    for m in range(n):
        g.manual_seed(seed + m)
        t = torch.empty(P, dtype=torch.float32, device=dev)
        t.uniform_(-1.0, 1.0, generator=g)
        out.append(t.to(torch.bfloat16) if dtype == "bf16" else t)
    return out


def deceptive_set(n, k, seed=0):
    import numpy as np

    return sorted(int(x) for x in np.random.default_rng(seed).choice(n, k, replace=False)) if k else []


def run_device(cfg, args, dev):
    import torch

    from paper_2507_17766_b200 import _lib as L
    from paper_2507_17766_b200.device import ButterflyMerge, Corruption, DevicePlan

    n, P, dtype, r, k_bad = cfg
    reps = make_replicas(n, P, dtype, dev)
    plan = DevicePlan(n, P, 0, redundancy=r, device=dev)
    corr = {m: Corruption.noise(2.0, (0x5EED, m)) for m in deceptive_set(n, k_bad)}
    job = ButterflyMerge(reps, plan, corruptions=corr, scatter_back=True, want_merged=False)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        job.run(L.PHASE_REDUCE)
        job.run(L.PHASE_FINISH)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            ev[3 * k].record(stream)
            job.run(L.PHASE_REDUCE)
            ev[3 * k + 1].record(stream)
            job.run(L.PHASE_FINISH)
            ev[3 * k + 2].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    reduce_ms = [ev[3 * k].elapsed_time(ev[3 * k + 1]) for k in range(args.steps)]
    finish_ms = [ev[3 * k + 1].elapsed_time(ev[3 * k + 2]) for k in range(args.steps)]
    status = job.status.cpu()
    info = {
        "total_ms": total_ms,
        "reduce_ms": statistics.mean(reduce_ms),
        "finish_ms": statistics.mean(finish_ms),
        "launches": job.launches_per_run() * args.steps,
        "clocks": clk.summary(),
        "n_alive": len(job.alive),
        "disagreement_shards": int((status == L.DISAGREEMENT).sum()),
        "flagged": int(job.flagged.sum().item()),
    }
    del job, reps
    torch.cuda.empty_cache()
    return info


def run_e2e(cfg, args, dev, p_e2e):
    """Same metric through the drop-in API (butterfly.run_all_reduce) from pinned host fp64 payloads."""
    import numpy as np
    import torch

    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200.simkernel import BlobStore

    n, _, _, r, _ = cfg
    if r != 2:
        return None
    payloads = {}
    g = torch.Generator()
    for m in range(n):
        g.manual_seed(1000 + m)
        t = torch.empty(p_e2e, dtype=torch.float64, pin_memory=True)
        t.uniform_(-1.0, 1.0, generator=g)
        payloads[m] = t.numpy()
    plan = bf.plan_shards(bf.enumerate_pairs(n), p_e2e, bf.BYTES_PER_WEIGHT, 0)
    for _ in range(max(1, min(args.warmup, 2))):
        res = bf.run_all_reduce(BlobStore(), payloads, plan)
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 5))
    t = time.perf_counter()
    for _ in range(steps):
        res = bf.run_all_reduce(BlobStore(), payloads, plan)
    dt = (time.perf_counter() - t) / steps
    assert res.merged.shape == (p_e2e,)
    S = plan.n_shards
    return {
        "value": p_e2e / dt,
        "unit": UNIT,
        "h2d_bytes_per_step": n * p_e2e * 8 + S * 2 * 4 + n,
        "d2h_bytes_per_step": p_e2e * 8 + S + n * n * 8 + n + S * 4,
        "params": p_e2e,
        "ms_per_step": dt * 1e3,
        "path": "paper_2507_17766_b200.butterfly.run_all_reduce(BlobStore(), fp64 pinned host payloads, plan)",
    }


def traffic_from_profiles(config_name):
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(f.read_text()).get(config_name)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--e2e-params", type=int, default=1 << 27)
    ap.add_argument("--cpu-params", type=int, default=1 << 25)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        from paper_2507_17766_b200 import multigpu

        return multigpu.bench_main(args, rank, world)
    name = args.config or "c2"
    cfg = CONFIGS[name]
    n, P, dtype, r, k_bad = cfg

    if args.impl == "reference":
        per_step = []
        threads = None
        for _ in range(args.warmup):
            cpu_sample(cfg, args.cpu_params, reps=1)
        for _ in range(args.steps):
            v, threads, secs = cpu_sample(cfg, args.cpu_params, reps=1)
            per_step.append(secs)
        value = args.cpu_params / statistics.mean(per_step)
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(per_step) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if dtype == "fp32" else "f32",
            "data": "synthetic uniform(-1,1) replicas",
            "config": {"workload": WORKLOAD[name], "miners": n, "params": args.cpu_params, "redundancy": r,
                       "sampled_from_params": P},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"oracle/bfly_oracle.c run_all_reduce restatement, {n} miners x "
                                       f"{args.cpu_params} params {dtype}, one merge per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    import torch

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    info = run_device(cfg, args, dev)
    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    t_step = info["total_ms"] / args.steps / 1e3
    value = P / t_step
    esize = 2 if dtype == "bf16" else 4
    alg_bytes = (info["n_alive"] + n) * P * esize  # read every alive replica once, write every replica once
    achieved = alg_bytes / (info["reduce_ms"] / 1e3) / 1e9
    e2e = None if args.no_e2e else run_e2e(cfg, args, dev, args.e2e_params)
    cpu = None
    if not args.no_cpu:
        v, threads, secs = cpu_sample(cfg, args.cpu_params)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"oracle/bfly_oracle.c (C restatement of run_all_reduce, OpenMP), {n} miners x "
                         f"{args.cpu_params} params {dtype}, best of 2 ({secs:.3f} s)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if dtype == "fp32" else "f32",
        "data": "synthetic uniform(-1,1) replicas (torch Philox, seed = miner index)",
        "config": {"workload": WORKLOAD[name], "miners": n, "params": P, "replica_dtype": dtype,
                   "redundancy": r, "deceptive": k_bad, "parallelism": "single GPU",
                   "l2": "inputs (%.0f GB) >> 126 MB L2, no flush" % (n * P * esize / 1e9)},
        "GBps": alg_bytes / t_step / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic_from_profiles(name),
                     "kernel": "k_reduce (+k_fill_nan, k_classify in the same event window)",
                     "algorithmic_bytes": alg_bytes, "kernel_ms": info["reduce_ms"],
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
        "finish_ms": info["finish_ms"],
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": info["launches"],
        "clocks": info["clocks"],
        "disagreement_shards": info["disagreement_shards"],
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
