#!/usr/bin/env python
"""Benchmark of the butterfly merge (BASELINE.json metric: params merged/sec (GB/s)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c1..c5]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

Workload.  N=1 (default): BASELINE config 2 — 16 miner replicas of one 1B-parameter
pipeline stage (fp32 wire values) on one B200, redundancy 2.  N>1 (default): config 3
— the north star — 64 miners of a 1B stage spread over the N GPUs in contiguous blocks
(64/N per GPU: strong scaling; N=8 is 8 miners per GPU).  ``--config c2`` keeps 16
miners per GPU at any N (weak scaling); c5 is c3 (c2 at N=1) with 6 noise-deceptive
miners; c4 is one 1.75B bf16 r=3 stage per GPU; c1 the reference default (8 x 10M).

A "step" is one merge round: every shard is reduced over the alive replicas (fp64
sequential accumulation in miner order, bit-identical to the reference), redundant
copies are compared, and the adopted slices are scattered back in place into every
replica.  Inputs are 32-128 GB per GPU, far larger than the 126 MB L2: no flush.

``value`` is the whole-job merge bandwidth in GB/s: the algorithmic bytes over all GPUs
(every alive replica read once + every replica written once, 4 B per parameter) divided
by the round time (max over ranks).  P / t (params merged per second) is beside it.
Multi-GPU lines carry SURVEY §8(d)'s roofline (HBM bytes per GPU at the measured copy
peak, NVLink bytes h(G-1)Ps + (G-1)/G Ps at 900 GB/s per direction) and the NVLink bytes
the GPUs' own counters (NVML) saw during the timed rounds.
"""

from __future__ import annotations

import argparse
import json
import math
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
UNIT = "GB/s"
NVLINK_SPEC_GBPS = 900.0  # per direction per GPU (NVLink 5; PAPER.md:177 cites 900 GB/s)

# name: miners, whether the count is per GPU (weak) or for the whole job (strong),
# params, replica dtype, redundancy, deceptive miners
CONFIGS = {
    "c1": dict(miners=8, per_gpu=False, params=10_000_000, dtype="fp32", r=2, bad=0),
    "c2": dict(miners=16, per_gpu=True, params=1_000_000_000, dtype="fp32", r=2, bad=0),
    "c3": dict(miners=64, per_gpu=False, params=1_000_000_000, dtype="fp32", r=2, bad=0),
    "c4": dict(miners=32, per_gpu=True, params=1_750_000_000, dtype="bf16", r=3, bad=0),
    "c5": dict(miners=64, per_gpu=False, params=1_000_000_000, dtype="fp32", r=2, bad=6),
}
WORKLOAD = {
    "c1": "reference default: 8 miners x 10M fp32, r=2 (BASELINE config 1)",
    "c2": "1B-param stage, 16 miners per B200 fp32, r=2 (BASELINE config 2 at N=1; weak scaling)",
    "c3": "1B-param stage, 64 miners fp32 in contiguous blocks over N B200s (64/N per GPU), r=2 "
          "(BASELINE config 3, the north star; strong scaling)",
    "c4": "14B model / 8 stages: one 1.75B-param stage per GPU, 32 miners bf16 (fp32 acc), r=3 (BASELINE config 4)",
    "c5": "adversarial 1B-param stage: 64 miners over N GPUs (16 on one GPU), 6 noise-deceptive, r=2 "
          "(BASELINE config 5)",
}
BYTES = {"fp32": 4, "bf16": 2}


def resolve_config(name, world):
    """(name, miners per GPU, total miners, params, dtype, r, deceptive)."""
    if name is None:
        name = "c2" if world == 1 else "c3"
    c = CONFIGS[name]
    if c["per_gpu"]:
        n_local, n = c["miners"], c["miners"] * world
    elif world == 1:
        n = 16 if name in ("c3", "c5") else c["miners"]  # 64 x 4 GB does not fit one GPU
        n_local = n
    else:
        n = c["miners"]
        if n % world:
            raise SystemExit(f"{name}: {n} miners do not split over {world} GPUs")
        n_local = n // world
    return name, n_local, n, c["params"], c["dtype"], c["r"], c["bad"]


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=lambda: self.lines.extend(ln.strip() for ln in self.proc.stdout),
                                       daemon=True)
            self._t.start()
            time.sleep(0.2)
        except FileNotFoundError:
            self.proc = None
        return self

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
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            reasons.update(nm for nm, v in zip(self.NAMES, parts[2:]) if v.lower() == "active")
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


class NVLinkCounter:
    """NVLink bytes this GPU sent and received, from its own counters (NVML field values
    summed over all links): read before and after the timed rounds."""

    # (tx field, rx field, bytes per unit): NVLINK_COUNT_XMIT/RCV_BYTES, else the older
    # NVLINK_THROUGHPUT_DATA_TX/RX counters (KiB)
    FIELDS = ((202, 204, 1), (138, 139, 1024))
    ALL_LINKS = 0xFFFFFFFF

    def __init__(self, index: int):
        self.ok, self.why = False, None
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(index)
            self.field = None
            for tx, rx, unit in self.FIELDS:
                if self._read_fields(tx, rx) is not None:
                    self.field = (tx, rx, unit)
                    break
            self.ok = self.field is not None
            if not self.ok:
                self.why = "NVML NVLink byte counters unavailable on this GPU/driver"
        except Exception as e:  # no NVML: reported, not fatal
            self.why = f"NVML: {e}"

    def _read_fields(self, tx, rx):
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, [(tx, self.ALL_LINKS), (rx, self.ALL_LINKS)])
        if any(v.nvmlReturn != 0 for v in vals):
            return None
        return [int(v.value.ullVal) for v in vals]

    def read(self):
        if not self.ok:
            return None
        tx, rx, unit = self.field
        v = self._read_fields(tx, rx)
        return None if v is None else (v[0] * unit, v[1] * unit)


# ---------------------------------------------------------------------------
# CPU timing: the reference itself (baseline/_ref) and its C restatement (oracle/)
# ---------------------------------------------------------------------------


REF_DIR = ROOT / "baseline" / "_ref"


def reference_sample(n, p_cpu, reps, warmup=1):
    """Time the unmodified reference, iota_sim.butterfly.run_all_reduce (butterfly.py:161-295)
    from baseline/_ref, on fp64 payloads with a fresh BlobStore per call: a list of seconds
    per call (None when the reference is not installed)."""
    if not (REF_DIR / "iota_sim").is_dir():
        return None
    sys.path.insert(0, str(REF_DIR))
    import numpy as np
    from iota_sim import butterfly as ref
    from iota_sim.simkernel import BlobStore as RefStore

    rng = np.random.default_rng(0)  # the reference tests' recipe (tests/test_butterfly.py:106-108)
    payloads = {m: rng.uniform(-1.0, 1.0, p_cpu) for m in range(n)}
    plan = ref.plan_shards(ref.enumerate_pairs(n), p_cpu, ref.BYTES_PER_WEIGHT, 0)
    for _ in range(warmup):
        ref.run_all_reduce(RefStore(), payloads, plan)
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        ref.run_all_reduce(RefStore(), payloads, plan)
        times.append(time.perf_counter() - t)
    return times


def reference_params(n, params):
    """The bounded sample of the workload the Python reference merges per step: P_cpu =
    2^24 at 16 miners, scaled down with the miner count so a step stays
    ~3 s, and never more than the workload itself (config 1 runs in full)."""
    p = min(params, 1 << 24, max(1 << 20, (1 << 28) // max(n, 1)))
    return params if params <= 10_000_000 else p


def cpu_env():
    return {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default")}



def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc  # test infrastructure: timed here only as the CPU baseline

    return orc


def cpu_sample(n, p_cpu, dtype, r, fp64_payloads: bool, reps: int = 1):
    """Time the C oracle (restatement of run_all_reduce) with all host threads.
    Returns (seconds per merge, threads)."""
    import numpy as np

    orc = _oracle()
    threads = orc.threads_available()
    rng = np.random.default_rng(0)
    if dtype == "bf16":
        replicas = [(rng.uniform(-1, 1, p_cpu).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
                    for _ in range(n)]
        odt = orc.BF16
    elif fp64_payloads:
        replicas = [rng.uniform(-1, 1, p_cpu) for _ in range(n)]
        odt = orc.F64WIRE
    else:
        replicas = [rng.uniform(-1, 1, p_cpu).astype(np.float32) for _ in range(n)]
        odt = orc.F32
    assign, bounds = orc.plan(n, p_cpu, 0, r=r)
    orc.merge(replicas, assign, bounds, dtype=odt, threads=threads)  # warm
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        orc.merge(replicas, assign, bounds, dtype=odt, threads=threads)
        times.append(time.perf_counter() - t)
    return times, threads


def merge_bytes(n_miners, params, esize):
    """Algorithmic bytes of one round: each replica read once and written once."""
    return 2 * n_miners * params * esize


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


def timed_rounds(step, args, dev, nvlink=None):
    """W untimed rounds, then K rounds between CUDA events on the current stream (and the
    GPU's NVLink byte counters read on both sides, when given)."""
    import torch

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nvl = None
    with ClockSampler(dev.index or 0) as clk:
        if torch.distributed.is_initialized():
            torch.distributed.barrier()
        torch.cuda.synchronize()
        c0 = nvlink.read() if nvlink is not None else None
        t0.record(stream)
        kernel_ms = [step(timed=True) for _ in range(args.steps)]
        t1.record(stream)
        torch.cuda.synchronize()
        c1 = nvlink.read() if nvlink is not None else None
        if c0 is not None and c1 is not None:
            nvl = (c1[0] - c0[0], c1[1] - c0[1])
        if torch.distributed.is_initialized():
            torch.distributed.barrier()
    return t0.elapsed_time(t1), kernel_ms, clk.summary(), nvl


def run_single(cfg, args, dev):
    import torch

    from paper_2507_17766_b200 import _lib as L
    from paper_2507_17766_b200.device import ButterflyMerge, Corruption, DevicePlan

    name, _, n, P, dtype, r, k_bad = cfg
    reps = make_replicas(n, P, dtype, dev)
    plan = DevicePlan(n, P, 0, redundancy=r, device=dev)
    corr = {m: Corruption.noise(2.0, (0x5EED, m)) for m in deceptive_set(n, k_bad)}
    job = ButterflyMerge(reps, plan, corruptions=corr, scatter_back=True, want_merged=False)
    events = []

    def step(timed=False):
        if not timed:
            job.run()
            return None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        job.run(L.PHASE_REDUCE)
        b.record()
        job.run(L.PHASE_FINISH)
        events.append((a, b))
        return None

    total_ms, _, clocks, _ = timed_rounds(step, args, dev)
    torch.cuda.synchronize()
    reduce_ms = statistics.mean(a.elapsed_time(b) for a, b in events)
    status = job.status.cpu()
    info = dict(total_ms=total_ms, reduce_ms=reduce_ms, launches=job.launches_per_run() * args.steps,
                clocks=clocks, n_alive=len(job.alive), disagreement=int((status == L.DISAGREEMENT).sum()),
                flagged=int(job.flagged.sum().item()))
    resident = run_e2e_resident(job, args)
    del job, reps
    torch.cuda.empty_cache()
    return info, resident


def run_e2e_resident(job, args):
    """Device-resident API end to end: per round the host sends the round's control
    inputs (failure mask, corruption table; pinned -> device) and reads back the
    round's result (status, flags, agreement matrix) — weights stay in HBM."""
    import torch

    failed_h = job._failed.cpu().pin_memory()
    corr_h = job._corr.cpu().pin_memory()
    outs = [torch.empty_like(t, device="cpu").pin_memory() for t in (job.status, job.flagged, job.entries)]
    steps = max(1, min(args.steps, 10))
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        job._failed.copy_(failed_h, non_blocking=True)
        job._corr.copy_(corr_h, non_blocking=True)
        job.run()
        for o, d in zip(outs, (job.status, job.flagged, job.entries)):
            o.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / steps
    h2d = failed_h.numel() + corr_h.numel()
    d2h = sum(o.numel() * o.element_size() for o in outs)
    return dt, h2d, d2h


def e2e_params(n, params, requested):
    """Parameters per payload of the end-to-end leg: the workload's own when the host can
    hold n fp64 payloads (pinned) with room to spare, else the largest power of two that
    fits (stated in the line)."""
    if requested:
        return requested, "requested"
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    need = n * params * 8
    if need * 1.6 < avail:
        return params, "the workload's full size"
    p = 1 << 27
    while p * 2 * n * 8 * 1.6 < avail and p * 2 <= params:
        p *= 2
    return p, f"host RAM {avail / 2**30:.0f} GiB holds {n} x {p} fp64 payloads, not {n} x {params}"


def run_e2e(n, r, args, dev, p_e2e, why):
    """The drop-in API (butterfly.run_all_reduce) on fp64 payloads in host memory: the
    fp32 wire conversion + H2D of every payload and the D2H of the merged vector are
    inside every step."""
    import torch

    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200.simkernel import BlobStore

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
    del res
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 5))
    t = time.perf_counter()
    for _ in range(steps):
        res = bf.run_all_reduce(BlobStore(), payloads, plan)
        del res
    dt = (time.perf_counter() - t) / steps
    S = plan.n_shards
    return {
        "value": merge_bytes(n, p_e2e, 4) / dt / 1e9,
        "unit": UNIT,
        "h2d_bytes_per_step": n * p_e2e * 4 + S * 2 * 4 + n + n * 32,
        "d2h_bytes_per_step": p_e2e * 8 + S + n * n * 8 + n + S * 4,
        "params": p_e2e,
        "params_why": why,
        "params_merged_per_s": p_e2e / dt,
        "ms_per_step": dt * 1e3,
        "path": "paper_2507_17766_b200.butterfly.run_all_reduce(BlobStore(), {miner: fp64 payload in pinned "
                "host memory}, plan) -> MergeResult (merged fp64 copied back)",
        "bound": "host: %.1f GB of fp64 payloads converted to the fp32 wire on host threads, %.1f GB H2D"
                 % (n * p_e2e * 8 / 1e9, n * p_e2e * 4 / 1e9),
    }


def contract_roofline(n, n_local, world, P, esize, hbm_peak, r=2):
    """per GPU B_HBM = 2 n_g P s; NVLink bytes into a GPU
    B_NVL = h (G-1) P s + (G-1)/G P s with h = 1 - C(N - N/G, r) / C(N, r); t_roof = max."""
    b_hbm = 2 * n_local * P * esize
    if world == 1:
        return dict(b_hbm=b_hbm, b_nvl=0.0, t_roof=b_hbm / (hbm_peak * 1e9), bound="hbm", h=0.0)
    h = 1.0 - math.comb(n - n // world, r) / math.comb(n, r)
    b_nvl = h * (world - 1) * P * esize + (world - 1) / world * P * esize
    t_h, t_n = b_hbm / (hbm_peak * 1e9), b_nvl / (NVLINK_SPEC_GBPS * 1e9)
    return dict(b_hbm=b_hbm, b_nvl=b_nvl, t_roof=max(t_h, t_n), bound="hbm" if t_h >= t_n else "nvlink", h=h)


def run_multi(cfg, args, rank, world):
    import torch
    import torch.distributed as dist

    from paper_2507_17766_b200.device import Corruption, DevicePlan
    from paper_2507_17766_b200.multigpu import ShardedButterflyMerge

    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    name, n_local, n, P, dtype, r, k_bad = cfg
    reps = make_replicas(n_local, P, dtype, dev, seed=rank * n_local)
    plan = DevicePlan(n, P, 0, redundancy=r, device=dev)
    bad = deceptive_set(n, k_bad)
    corr = {m: Corruption.noise(2.0, (0x5EED, m)) for m in bad}
    tuning = json.loads(args.ring_tuning) if args.ring_tuning else None
    job = ShardedButterflyMerge(reps, plan, corruptions=corr, chunk=args.chunk, fuse_stats=args.fuse_stats,
                                ring_tuning=tuning)
    nvcount = NVLinkCounter(local_rank)
    phases = None
    if args.timing:  # one extra round with CUDA events between the phases (diagnostics, untimed)
        job.timing = True
        job.run()
        phases = {k: round(v, 3) for k, v in job.timings.items()}
        job.timing = False

    def step(timed=False):
        job.run()
        return None

    total_ms, _, clocks, nvl = timed_rounds(step, args, dev, nvlink=nvcount)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    t_step = total_ms / args.steps / 1e3
    esize = BYTES[dtype]
    # measured NVLink bytes per round: max over ranks of what a GPU received / sent
    meas = torch.tensor([-1.0, -1.0] if nvl is None else [float(nvl[1]), float(nvl[0])], dtype=torch.float64,
                        device=dev)
    dist.all_reduce(meas, op=dist.ReduceOp.MAX)
    nb = job.bytes_per_round()
    impl_nvl = torch.tensor([nb["nvlink_in"]], dtype=torch.float64, device=dev)
    dist.all_reduce(impl_nvl, op=dist.ReduceOp.MAX)
    lt = torch.tensor([job.launches_per_run() * args.steps], dtype=torch.int64, device=dev)
    dist.all_reduce(lt)  # every rank's kernels: the whole job's launches
    launches = int(lt.item())
    disagree = int((job.status == 2).sum().item())
    e2e = None if args.no_e2e else run_e2e_multi(n_local, n, r, args, dev, rank, world, plan_seed=0)
    if rank == 0:
        peaks = _peaks()
        hbm_peak = peaks.get("hbm_gbs", 6550.0)
        alg = merge_bytes(n, P, esize)
        value = alg / t_step / 1e9
        roof = contract_roofline(n, n_local, world, P, esize, hbm_peak, r)
        if roof["bound"] == "hbm":
            achieved, peak, unit_peak = roof["b_hbm"] / t_step / 1e9, hbm_peak, "HBM copy peak (MEASURED_PEAKS.json)"
        else:
            achieved, peak, unit_peak = roof["b_nvl"] / t_step / 1e9, NVLINK_SPEC_GBPS, "NVLink 5 spec per direction"
        impl_t = max(roof["b_hbm"] / (hbm_peak * 1e9), float(impl_nvl.item()) / (NVLINK_SPEC_GBPS * 1e9))
        rx, tx = float(meas[0].item()), float(meas[1].item())
        measured = None if rx < 0 else {
            "rx_bytes_per_round": rx / args.steps, "tx_bytes_per_round": tx / args.steps,
            "rx_GBps": rx / args.steps / t_step / 1e9, "tx_GBps": tx / args.steps / t_step / 1e9,
            "rx_frac_of_spec": rx / args.steps / t_step / 1e9 / NVLINK_SPEC_GBPS,
            "source": "NVML NVLink byte counters (all links) read before/after the timed rounds; max over ranks"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "weak" if CONFIGS[name]["per_gpu"] else "strong",
            "vs_baseline": None, "dtype": "f64" if dtype == "fp32" else "f32",
            "data": "synthetic uniform(-1,1) replicas (torch Philox, seed = miner index)",
            "config": {"workload": WORKLOAD[name], "config": name, "miners": n, "miners_per_gpu": n_local,
                       "params": P, "replica_dtype": dtype, "redundancy": r, "deceptive": len(bad),
                       "parallelism": (f"miners in contiguous blocks over {world} GPUs; one persistent kernel per "
                                       f"GPU (k_ring): fp64 running sums chained rank to rank tile by tile through "
                                       f"TMA bulk stores into IPC-mapped peer inboxes over NVLink, final values "
                                       f"relayed round the ring" if job.fused else
                                       f"miners in contiguous blocks over {world} GPUs; chunked ring: fp64 running "
                                       f"sums chained rank to rank (TMA bulk stores into IPC-mapped peer inboxes, "
                                       f"up to {args.chunk}-element chunks), final vector relayed round the ring"),
                       "l2": "inputs %.2f GB per GPU >> 126 MB L2, no flush" % (n_local * P * esize / 1e9)},
            "params_merged_per_s": P / t_step,
            "roofline": {"bound": roof["bound"], "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": unit_peak,
                         "kernel": ("whole round per GPU (k_ring: one persistent kernel)" if job.fused else
                                    "whole round per GPU (chain / reduce / fan-out kernels + NVLink ring)"),
                         "contract": "SURVEY §8(d): t_roof = max(2 n_g P s / BW_HBM, "
                                     "(h (G-1) P s + (G-1)/G P s) / 900 GB/s)",
                         "t_roof_ms": roof["t_roof"] * 1e3, "h": roof["h"],
                         "hbm_bytes_per_gpu": roof["b_hbm"], "nvlink_bytes_in_per_gpu": roof["b_nvl"],
                         "impl": {"nvlink_bytes_in_per_gpu": float(impl_nvl.item()),
                                  "note": "this implementation's exchange: fp64 running sums (8 B/param) into every "
                                          "rank > 0 plus the final vector (s B/param) into every rank < last, "
                                          "which keeps the reference's summation order bit for bit",
                                  "t_roof_ms": impl_t * 1e3, "frac": impl_t / t_step}},
            "nvlink_measured": measured if measured else {"unavailable": nvcount.why},
            "e2e": e2e, "cpu_baseline": None, "gpu_launches": launches, "clocks": clocks,
            "disagreement_shards": disagree,
        }
        if phases:
            line["phases_ms_rank0"] = phases
        print(json.dumps(line))
    if phases and rank == world - 1:
        print(f"[rank {rank}] phases (ms): " + json.dumps(phases), file=sys.stderr, flush=True)
    job.close()
    dist.barrier()
    dist.destroy_process_group()


def run_e2e_multi(n_local, n, r, args, dev, rank, world, plan_seed=0):
    """Multi-GPU end to end through the public API: every step each rank uploads its
    miners' fp64 payloads from pinned host memory (bfly_upload_wire: fp32 wire
    conversion on host threads + H2D), runs ShardedButterflyMerge, and reads the
    round's results (status, flags, agreement matrix) back to the host.  Time is the
    max over ranks."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2507_17766_b200 import _lib as L
    from paper_2507_17766_b200.device import DevicePlan, _stream_handle
    from paper_2507_17766_b200.multigpu import ShardedButterflyMerge

    P = min(args.e2e_params or (1 << 26), 1 << 26)
    host = []
    g = torch.Generator()
    for i in range(n_local):
        g.manual_seed(1000 + rank * n_local + i)
        host.append(torch.empty(P, dtype=torch.float64, pin_memory=True).uniform_(-1.0, 1.0, generator=g))
    wire = [torch.empty(P, dtype=torch.float32, device=dev) for _ in range(n_local)]
    h_ptrs = (ctypes.c_void_p * n_local)(*[t.data_ptr() for t in host])
    d_ptrs = (ctypes.c_void_p * n_local)(*[t.data_ptr() for t in wire])
    threads = max(1, (os.cpu_count() or world) // world)
    plan = DevicePlan(n, P, plan_seed, redundancy=r, device=dev)
    job = ShardedButterflyMerge(wire, plan, chunk=min(args.chunk, 1 << 24))
    outs = [torch.empty_like(t, device="cpu").pin_memory() for t in (job.status, job.flagged, job.entries)]

    def step():
        L.check(L.lib().bfly_upload_wire(h_ptrs, n_local, P, d_ptrs, threads, 0, _stream_handle()))
        job.run()
        for o, d in zip(outs, (job.status, job.flagged, job.entries)):
            o.copy_(d, non_blocking=True)
        torch.cuda.synchronize()

    step()
    dist.barrier()
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = torch.tensor([(time.perf_counter() - t0) / steps], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    dt = float(dt.item())
    job.close()
    return {"value": merge_bytes(n, P, 4) / dt / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": n_local * P * 4, "d2h_bytes_per_step": sum(o.numel() * o.element_size() for o in outs),
            "params": P, "ms_per_step": dt * 1e3,
            "path": "per rank: bfly_upload_wire(fp64 pinned host payloads) + ShardedButterflyMerge.run() + results D2H",
            "bound": "host memory / PCIe of each rank"}


def run_stages(cfg, args, rank, world):
    """Config 4: one pipeline stage per GPU; stages merge independently
    (orchestrator.py:596-597 loops over layers), so N GPUs run N independent
    merges — replicas only, no exchange.  Timing is the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan

    distributed = world > 1
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    _, n, _, P, dtype, r, _ = cfg
    reps = make_replicas(n, P, dtype, dev, seed=1000 * rank)
    plan = DevicePlan(n, P, rank, redundancy=r, device=dev)
    job = ButterflyMerge(reps, plan, scatter_back=True)

    def step(timed=False):
        job.run()

    total_ms, _, clocks, _ = timed_rounds(step, args, dev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t.item()) / args.steps / 1e3
    if rank == 0:
        esize = BYTES[dtype]
        alg = world * merge_bytes(n, P, esize)
        hbm_peak = _peaks().get("hbm_gbs", 6550.0)
        line = {
            "metric": METRIC, "value": alg / t_step / 1e9, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic uniform(-1,1) bf16 replicas (torch Philox)",
            "config": {"workload": WORKLOAD["c4"], "config": "c4", "miners_per_stage": n, "params_per_stage": P,
                       "stages": world, "replica_dtype": dtype, "redundancy": r,
                       "parallelism": "one stage per GPU (replicas only)",
                       "l2": "inputs %.2f GB per GPU >> 126 MB L2, no flush" % (n * P * esize / 1e9)},
            "params_merged_per_s": world * P / t_step,
            "roofline": {"bound": "hbm", "achieved": merge_bytes(n, P, esize) / t_step / 1e9, "peak": hbm_peak,
                         "unit": "GB/s", "frac": merge_bytes(n, P, esize) / t_step / 1e9 / hbm_peak,
                         "traffic": None, "kernel": "whole merge round per GPU"},
            "e2e": None, "cpu_baseline": None, "gpu_launches": job.launches_per_run() * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line))
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(cfg, args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path,
    iota_sim.butterfly.run_all_reduce from baseline/_ref (unmodified, installed with the
    base contract's pip command), timed on this host for a bounded sample of the same
    workload (same miner count, P_cpu parameters), one merge per step.  Its C restatement
    (oracle/, all host threads) is timed beside it and reported as a labelled second
    figure.  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    name, _, n, P, dtype, r, k_bad = cfg
    esize = BYTES[dtype]
    p_cpu = args.cpu_params or reference_params(n, P)
    times = reference_sample(n, p_cpu, reps=args.steps, warmup=args.warmup) if r == 2 and dtype == "fp32" else None
    port_times, port_threads = cpu_sample(n, p_cpu, dtype, r, dtype == "fp32", reps=max(1, min(args.steps, 5)))
    port = {"value": merge_bytes(n, p_cpu, esize) / statistics.mean(port_times) / 1e9, "unit": UNIT,
            "cores": port_threads, "kind": "port", "ms_per_step": statistics.mean(port_times) * 1e3,
            "sample": f"oracle/bfly_oracle.c: C restatement of run_all_reduce (OpenMP, {port_threads} threads), "
                      f"{n} miners x {p_cpu} params as fp64 payloads -> fp32 wire -> fp64 mean"}
    if times is not None:
        t_step = statistics.mean(times)
        value = merge_bytes(n, p_cpu, esize) / t_step / 1e9
        kind, cores = "reference", 1
        sample = (f"iota_sim.butterfly.run_all_reduce (baseline/_ref, unmodified; numpy, 1 effective core) on "
                  f"{n} fp64 payloads x {p_cpu} params (of the workload's {P}), fresh BlobStore per step; "
                  f"best {min(times) * 1e3:.0f} ms")
    else:  # bf16 / r = 3 (config 4): no reference implementation exists; the port is the arm
        t_step = statistics.mean(port_times)
        value, kind, cores = port["value"], "port", port_threads
        sample = port["sample"] + " (no reference implementation of this extension config)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak" if CONFIGS[name]["per_gpu"] else "strong", "vs_baseline": None,
        "dtype": "f64" if dtype == "fp32" else "f32", "data": "synthetic uniform(-1,1) payloads",
        "config": {"workload": WORKLOAD[name], "config": name, "miners": n, "params": p_cpu,
                   "sampled_from_params": P, "redundancy": r, "deceptive": k_bad},
        "params_merged_per_s": p_cpu / t_step,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                         "host": cpu_env()},
        "port": port,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 on one GPU, c3 (the north star) on several")
    ap.add_argument("--params", type=int, default=None, help="override the stage size")
    ap.add_argument("--chunk", type=int, default=1 << 24)
    ap.add_argument("--e2e-params", type=int, default=None, help="default: the workload's size if host RAM allows")
    ap.add_argument("--cpu-params", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--timing", action="store_true", help="multi-GPU: per-phase times of one extra round")
    ap.add_argument("--fuse-stats", action="store_true", help="multi-GPU: pair statistics inside k_ring")
    ap.add_argument("--ring-tuning", default=None, help='multi-GPU experiments, e.g. \'{"slots": 12, "lag": 2}\'')
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    cfg = list(resolve_config(args.config, world))
    if args.params:
        cfg[3] = args.params
    cfg = tuple(cfg)
    name = cfg[0]
    if args.impl == "reference":
        return run_reference(cfg, args, rank, world)
    if name == "c4":
        return run_stages(cfg, args, rank, world)
    if world > 1:
        return run_multi(cfg, args, rank, world)

    import torch

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    _, _, n, P, dtype, r, k_bad = cfg
    info, resident = run_single(cfg, args, dev)
    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs", 6550.0)
    t_step = info["total_ms"] / args.steps / 1e3
    esize = BYTES[dtype]
    alg = (info["n_alive"] + n) * P * esize  # read every alive replica once, write every replica once
    value = alg / t_step / 1e9
    if k_bad:  # corrupted shards are finished by k_stats/k_apply: the round is the unit
        kernel_ms, kernel_name = t_step * 1e3, "whole merge round (k_reduce + k_stats + k_decide + k_apply)"
    else:
        kernel_ms, kernel_name = info["reduce_ms"], "k_reduce (event window also holds k_fill_nan + k_classify, < 10 us)"
    achieved = alg / (kernel_ms / 1e3) / 1e9
    e2e = None
    if not args.no_e2e:
        p_e2e, why = e2e_params(n, P, args.e2e_params)
        e2e = run_e2e(n, r, args, dev, p_e2e, why)
    cpu = None
    if not args.no_cpu:
        p_cpu = args.cpu_params or reference_params(n, P)
        ref_times = reference_sample(n, p_cpu, reps=2) if r == 2 and dtype == "fp32" else None
        port_times, threads = cpu_sample(n, p_cpu, dtype, r, False, reps=2)
        port = {"value": merge_bytes(n, p_cpu, esize) / min(port_times) / 1e9, "unit": UNIT, "cores": threads,
                "kind": "port", "ms_per_step": min(port_times) * 1e3,
                "sample": f"oracle/bfly_oracle.c (C restatement of run_all_reduce, OpenMP {threads} threads) on "
                          f"host-resident {dtype} replicas, {n} miners x {p_cpu} params, best of 2"}
        if ref_times:
            secs = min(ref_times)
            cpu = {"value": merge_bytes(n, p_cpu, esize) / secs / 1e9, "unit": UNIT, "cores": 1, "kind": "reference",
                   "params_merged_per_s": p_cpu / secs,
                   "sample": f"iota_sim.butterfly.run_all_reduce (baseline/_ref, unmodified; 1 effective core) on "
                             f"{n} fp64 payloads x {p_cpu} params, best of 2 ({secs * 1e3:.0f} ms per merge)",
                   "host": cpu_env(), "port": port}
        else:
            cpu = port
    rt, h2d, d2h = resident
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if dtype == "fp32" else "f32",
        "data": "synthetic uniform(-1,1) replicas (torch Philox, seed = miner index)",
        "config": {"workload": WORKLOAD[name], "config": name, "miners": n, "params": P, "replica_dtype": dtype,
                   "redundancy": r, "deceptive": k_bad, "parallelism": "single GPU",
                   "l2": "inputs %.2f GB >> 126 MB L2, no flush" % (n * P * esize / 1e9)},
        "params_merged_per_s": P / t_step,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic_from_profiles(name),
                     "kernel": kernel_name, "algorithmic_bytes_per_launch": alg, "kernel_ms": kernel_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
        "e2e": e2e,
        "e2e_resident": {"value": alg / rt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "ms_per_step": rt * 1e3,
                         "path": "device.ButterflyMerge.run() on HBM-resident replicas; per step H2D of the "
                                 "failure mask + corruption table, D2H of status/flags/agreement matrix"},
        "cpu_baseline": cpu,
        "gpu_launches": info["launches"],
        "clocks": info["clocks"],
        "disagreement_shards": info["disagreement"],
    }
    print(json.dumps(line))


def traffic_from_profiles(config_name):
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(f.read_text()).get(config_name)
    except Exception:
        return None


if __name__ == "__main__":
    main()
