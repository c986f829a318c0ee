"""Shared body of the multi-GPU merge tests: one rank's side of a case, checked bit for
bit against the oracle.  Run either by torchrun workers (one process per GPU, NCCL,
DistComm) or by ``multigpu.run_loopback`` (every rank a thread on ONE GPU, LoopbackComm:
the same kernels and host logic, so the driver's 1-GPU box tests the ring too)."""

from __future__ import annotations

import numpy as np
import torch

import oracle as orc
from _golden import assert_entries_close, assert_same_floats

KINDS = {1: "add", 2: "scale", 3: "noise", 4: "noise_add"}


def case_data(case) -> dict:
    """Replicas, fallback and the oracle's answer for a case (identical on every rank)."""
    counts, P, seed = case["counts"], case["P"], case["seed"]
    n = sum(counts)
    rng = np.random.default_rng(7)
    data = (rng.uniform(-1, 1, (n, P)) * 10.0 ** rng.integers(-4, 4, (n, 1))).astype(np.float32)
    r = case.get("r", 2)
    bf16 = case.get("bf16", False)
    if bf16:
        data = (data.view(np.uint32) >> 16).astype(np.uint16)
    for m, e, v in case.get("poison", ()):
        data[m][e] = {"nan": np.nan, "inf": np.inf, "-inf": -np.inf}[v]
    fails = tuple(case["failures"])
    specs = {int(k): tuple(v) for k, v in case["corr"].items()}
    fb = rng.uniform(-2, 2, P) if case["fallback"] else None
    assign, bounds = orc.plan(n, P, seed, r=r)
    want = orc.merge(list(data), assign, bounds, failures=fails, corruptions=specs, fallback=fb,
                     dtype=orc.BF16 if bf16 else orc.F32)
    if fb is None and case.get("poison"):
        # multi-GPU: a fast shard whose mean is not finite falls back after the relay has
        # overwritten the lowest alive replica, so without a fallback it takes NaN (bfly.h)
        cls_fast = [all(m in fails or m not in specs for m in assign[s]) and any(m not in fails for m in assign[s])
                    for s in range(len(assign))]
        for s in range(len(assign)):
            if cls_fast[s] and want["status"][s] != 0:
                want["merged"][bounds[s]:bounds[s + 1]] = np.nan
    return dict(data=data, want=want, fb=fb, specs=specs, fails=fails, r=r, bf16=bf16, n=n, P=P, seed=seed,
                counts=counts, bounds=bounds)


def run_rank(case, d, rank, comm, dev) -> int:
    """Rank `rank`'s side of the case: build its replicas and the job, run the rounds,
    compare merged / own replicas / status / flags / entries with the oracle."""
    from paper_2507_17766_b200.device import Corruption, DevicePlan
    from paper_2507_17766_b200.multigpu import ShardedButterflyMerge

    data, want, counts, P = d["data"], d["want"], d["counts"], d["P"]
    off = sum(counts[:rank])
    if d["bf16"]:
        local = [torch.from_numpy(data[off + i].view(np.int16).copy()).to(dev).view(torch.bfloat16)
                 for i in range(counts[rank])]
    else:
        local = [torch.from_numpy(data[off + i].copy()).to(dev) for i in range(counts[rank])]
    plan = DevicePlan(d["n"], P, d["seed"], redundancy=d["r"], device=dev)
    corr = {m: Corruption(KINDS[s[0]], s[1], (s[2], s[3]) if len(s) > 2 else (0, 0)) for m, s in d["specs"].items()}
    fb = d["fb"]
    job = ShardedButterflyMerge(local, plan, failures=d["fails"], corruptions=corr,
                                fallback=None if fb is None else torch.from_numpy(fb).to(dev),
                                chunk=case["chunk"], want_merged=True, comm=comm,
                                executor=case.get("executor", "auto"), fuse_stats=case.get("fuse_stats", False))
    if "fused" in case:
        assert job.fused == case["fused"], (job.fused, case["fused"])
    orig = [t.clone() for t in local]
    try:
        for rnd in range(case.get("rounds", 1)):
            if rnd:  # refill the replicas in place: the next round reuses slots and flags
                for t, o in zip(local, orig):
                    t.copy_(o)
            job.run()
            torch.cuda.current_stream(dev).synchronize()
            assert_same_floats(job.merged.cpu().numpy(), want["merged"])
            if not d["bf16"]:
                for t in local:
                    assert_same_floats(t.cpu().numpy(), want["merged"].astype(np.float32))
            else:
                bits = np.array([orc.lib().orc_f32_to_bf16(float(v)) for v in want["merged"][:4099].astype(np.float32)],
                                dtype=np.uint16)
                for t in local:
                    assert np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16)[:4099], bits)
            assert np.array_equal(job.status.cpu().numpy(), want["status"])
            assert np.array_equal(job.flagged.cpu().numpy(), want["flagged"])
            assert_entries_close(job.entries.cpu().numpy(), want["entries"])
    finally:
        job.close()
    return int(job.fused)


def fuzz_case(case_idx: int, world: int) -> dict:
    """A seeded random case of the multi-GPU fuzz (identical on every rank)."""
    rng = np.random.default_rng(1000 + case_idx)
    counts = [int(x) for x in rng.integers(1, 6, world)]
    n = sum(counts)
    r = 3 if (n >= 4 and rng.random() < 0.3) else 2
    S = {2: n * (n - 1) // 2, 3: n * (n - 1) * (n - 2) // 6}[r]
    kind = ["fp32", "bf16", "fp64"][int(rng.integers(0, 3))]
    P = int(rng.choice([2 * S + int(rng.integers(0, 50)), int(rng.integers(2 * S, 200_000)),
                        int(rng.integers(200_000, 2_500_000))]))
    fails = sorted(int(x) for x in rng.choice(n, int(rng.integers(0, r)), replace=False))
    corr = {}
    if rng.random() < 0.15:
        m = int(rng.choice([x for x in range(n) if x not in fails]))
        corr[m] = (orc.ADD, 0.5)
    seed = int(rng.integers(0, 2**31))
    # round 2: noise-deceptive miners (shared keys = colluders) and the stats warps
    # (fuse_stats), from their own stream so the earlier cases keep their draws
    rng2 = np.random.default_rng(5000 + case_idx)
    fuse_stats = bool(rng2.random() < 0.4)
    if rng2.random() < 0.3:
        # one amplitude per case: two pure-noise copies of one key with different amplitudes
        # would be exactly proportional, a cosine of 1 up to the summation order (a tie
        # numpy's own order decides)
        amp = float(rng2.choice([1e-9, 0.5, 2.0]))
        alive = [x for x in range(n) if x not in fails and x not in corr]
        for m in rng2.choice(alive, min(len(alive), int(rng2.integers(1, 3))), replace=False):
            kind3 = int(rng2.choice([orc.NOISE, orc.NOISE_ADD]))
            corr[int(m)] = (kind3, amp, 77, int(rng2.integers(0, 2)))
    data = (rng.uniform(-1, 1, (n, P)) * 10.0 ** rng.integers(-3, 3, (n, 1))).astype(np.float32)
    if kind == "bf16":
        data = (data.view(np.uint32) >> 16).astype(np.uint16)
        odt = orc.BF16
    elif kind == "fp64":
        data = rng.uniform(-1, 1, (n, P)) * 10.0 ** rng.integers(-3, 3, (n, 1))
        odt = orc.F64WIRE
    else:
        odt = orc.F32
    assign, bounds = orc.plan(n, P, seed, r=r)
    want = orc.merge(list(data), assign, bounds, failures=tuple(fails), corruptions=corr, dtype=odt)
    return dict(counts=counts, n=n, r=r, kind=kind, P=P, fails=fails, corr=corr, seed=seed, data=data, want=want,
                rounds=int(rng.integers(1, 4)), fuse_stats=fuse_stats)


def fuzz_rank(c, rank, comm, dev) -> int:
    from paper_2507_17766_b200.device import Corruption, DevicePlan
    from paper_2507_17766_b200.multigpu import ShardedButterflyMerge

    counts, data, want, kind = c["counts"], c["data"], c["want"], c["kind"]
    off = sum(counts[:rank])
    if kind == "bf16":
        local = [torch.from_numpy(data[off + i].view(np.int16).copy()).to(dev).view(torch.bfloat16)
                 for i in range(counts[rank])]
    else:
        local = [torch.from_numpy(data[off + i].copy()).to(dev) for i in range(counts[rank])]
    orig = [t.clone() for t in local]
    plan = DevicePlan(c["n"], c["P"], c["seed"], redundancy=c["r"], device=dev)
    dcorr = {m: Corruption(KINDS[s[0]], s[1], (s[2], s[3]) if len(s) > 2 else (0, 0)) for m, s in c["corr"].items()}
    job = ShardedButterflyMerge(local, plan, failures=c["fails"], corruptions=dcorr, chunk=1 << 18, want_merged=True,
                                comm=comm, fuse_stats=c["fuse_stats"])
    try:
        for rnd in range(c["rounds"]):
            if rnd:
                for t, o in zip(local, orig):
                    t.copy_(o)
            job.run()
            torch.cuda.current_stream(dev).synchronize()
            tag = (f"counts {counts}, P {c['P']}, r {c['r']}, {kind}, fails {c['fails']}, corr {list(c['corr'])}, "
                   f"fused {job.fused}, fuse_stats {c['fuse_stats']}, round {rnd}")
            try:
                assert_same_floats(job.merged.cpu().numpy(), want["merged"])
                if kind == "bf16":
                    bits = np.array([orc.lib().orc_f32_to_bf16(float(v))
                                     for v in want["merged"][:3000].astype(np.float32)], dtype=np.uint16)
                    for t in local:
                        assert np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16)[:3000], bits)
                elif kind == "fp32":
                    for t in local:
                        assert_same_floats(t.cpu().numpy(), want["merged"].astype(np.float32))
                else:
                    for t in local:
                        assert_same_floats(t.cpu().numpy(), want["merged"])
                assert np.array_equal(job.status.cpu().numpy(), want["status"])
                assert np.array_equal(job.flagged.cpu().numpy(), want["flagged"])
                assert_entries_close(job.entries.cpu().numpy(), want["entries"])
            except AssertionError as e:
                raise AssertionError(tag + ": " + str(e)) from None
    finally:
        job.close()
    return int(job.fused)


# ---------------------------------------------------------------------------
# full-size ring: 16 miners x 1e9 fp32 per rank, 6 noise-deceptive miners
# ---------------------------------------------------------------------------

def fullsize_case(world: int, n_local: int = 16, P: int = 1_000_000_000, seed: int = 4) -> dict:
    n = world * n_local
    bad = sorted(int(x) for x in np.random.default_rng(1).choice(n, 6, replace=False))
    assign, bounds = orc.plan(n, P, seed)
    special = [s for s in range(len(assign)) if set(assign[s]) & set(bad)]
    fast = [s for s in range(len(assign)) if s not in special]
    rng = np.random.default_rng(6)
    sample = sorted(set(rng.choice(special, 5, replace=False).tolist()) |
                    set(rng.choice(fast, 3, replace=False).tolist()) | {0, len(assign) - 1})
    return dict(world=world, n_local=n_local, n=n, P=P, seed=seed, bad=bad, keys={m: (0xC5, m) for m in bad},
                amp=2.0, assign=assign, bounds=bounds, special=special, sample=sample)


def fullsize_rank(c, rank, comm, dev) -> dict:
    """One rank's side: its replicas (seeded per miner), snapshots of the sampled shards,
    one round, the sampled shards of its first and last replica afterwards."""
    from paper_2507_17766_b200.device import Corruption, DevicePlan
    from paper_2507_17766_b200.multigpu import ShardedButterflyMerge

    bounds, P = c["bounds"], c["P"]
    g = torch.Generator(device=dev)
    reps = []
    for i in range(c["n_local"]):
        g.manual_seed(rank * c["n_local"] + i)
        reps.append(torch.empty(P, dtype=torch.float32, device=dev).uniform_(-1, 1, generator=g))
    before = {s: [r[bounds[s]:bounds[s + 1]].cpu().numpy() for r in reps] for s in c["sample"]}
    plan = DevicePlan(c["n"], P, c["seed"], device=dev)
    job = ShardedButterflyMerge(reps, plan, comm=comm,
                                corruptions={m: Corruption.noise(c["amp"], c["keys"][m]) for m in c["bad"]})
    job.run()
    torch.cuda.current_stream(dev).synchronize()
    after = {s: [reps[0][bounds[s]:bounds[s + 1]].cpu().numpy(), reps[-1][bounds[s]:bounds[s + 1]].cpu().numpy()]
             for s in c["sample"]}
    out = dict(fused=job.fused, status=job.status.cpu().numpy(), flagged=job.flagged.cpu().numpy(),
               entries=job.entries.cpu().numpy(), before=before, after=after)
    job.close()
    return out


def fullsize_check(c, res) -> None:
    """Closed forms (C(n,2) - C(n-6,2) disagreements, every miner flagged) on every rank,
    and the sampled shards re-decided with the oracle's primitives from the snapshots:
    the sequential fp64 mean in miner order, each assignee's copy (noise keyed by the
    global element index), agreement, adoption or the lowest alive replica's values."""
    n, assign, bounds, special = c["n"], c["assign"], c["bounds"], c["special"]
    k = n - len(c["bad"])
    for out in res:
        assert out["fused"]
        assert int((out["status"] == orc.DISAGREEMENT).sum()) == n * (n - 1) // 2 - k * (k - 1) // 2 == len(special)
        assert np.array_equal(np.flatnonzero(out["status"] == orc.DISAGREEMENT), np.array(special))
        assert int(out["flagged"].sum()) == n
    for s in c["sample"]:
        lo, hi = int(bounds[s]), int(bounds[s + 1])
        snap = [x for out in res for x in out["before"][s]]  # miners 0..n-1 in rank order
        acc = np.zeros(hi - lo)
        for m in range(n):
            acc = acc + snap[m].astype(np.float64)
        mean = acc / n
        i, j = (int(x) for x in assign[s])
        copy = {x: (orc.noise_values(*c["keys"][x], c["amp"], lo, hi) if x in c["bad"] else mean) for x in (i, j)}
        score = orc.agreement(copy[i], copy[j])
        want = (copy[min(i, j)] if score == 1.0 else snap[0].astype(np.float64)).astype(np.float32)
        for out in res:
            assert out["status"][s] == (orc.MERGED if score == 1.0 else orc.DISAGREEMENT), s
            assert abs(out["entries"][i, j] - score) <= 1e-12, s
            for got in out["after"][s]:
                assert_same_floats(got, want)
