"""Seeded fuzz of the multi-GPU merge against the oracle: random miner counts per rank,
payload lengths (partial last tiles, lengths below one tile per lane), redundancy 2/3,
fp32 / bf16 / fp64 replicas, failures (fewer than r, so the persistent ring kernel
k_ring runs; a few cases with corruptions take the chunked ring), several rounds per
case with the replicas refilled in place (slot rings and monotonic flags carry over).
Every rank checks merged values, its own replicas, status, flags and entries bit for
bit (entries <= 1e-12).  One torchrun job runs every case; needs >= 2 GPUs."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import os, sys, json
import numpy as np, torch, torch.distributed as dist
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/oracle", sys.argv[1] + "/tests"]
import oracle as orc
from _golden import assert_same_floats, assert_entries_close
from paper_2507_17766_b200.device import DevicePlan, Corruption
from paper_2507_17766_b200.multigpu import ShardedButterflyMerge
n_cases = int(sys.argv[2])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
fused_seen = 0
for case in range(n_cases):
    rng = np.random.default_rng(1000 + case)  # identical on every rank
    counts = [int(x) for x in rng.integers(1, 6, world)]
    n = sum(counts)
    r = 3 if (n >= 4 and rng.random() < 0.3) else 2
    S = {2: n * (n - 1) // 2, 3: n * (n - 1) * (n - 2) // 6}[r]
    kind = ["fp32", "bf16", "fp64"][int(rng.integers(0, 3))]
    P = int(rng.choice([2 * S + int(rng.integers(0, 50)), int(rng.integers(2 * S, 200_000)),
                        int(rng.integers(200_000, 2_500_000))]))
    fails = sorted(int(x) for x in rng.choice(n, int(rng.integers(0, r)), replace=False))
    corr = {}
    if rng.random() < 0.15:  # a corrupted miner: the round takes the chunked ring
        m = int(rng.choice([x for x in range(n) if x not in fails]))
        corr[m] = (orc.ADD, 0.5)
    seed = int(rng.integers(0, 2**31))
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
    off = sum(counts[:rank])
    if kind == "bf16":
        local = [torch.from_numpy(data[off + i].view(np.int16).copy()).to(dev).view(torch.bfloat16)
                 for i in range(counts[rank])]
    else:
        local = [torch.from_numpy(data[off + i].copy()).to(dev) for i in range(counts[rank])]
    orig = [t.clone() for t in local]
    plan = DevicePlan(n, P, seed, redundancy=r, device=dev)
    dcorr = {m: Corruption.add(a) for m, (_, a) in corr.items()}
    job = ShardedButterflyMerge(local, plan, failures=fails, corruptions=dcorr, chunk=1 << 18, want_merged=True)
    fused_seen += int(job.fused)
    rounds = int(rng.integers(1, 4))
    for rnd in range(rounds):
        if rnd:
            for t, o in zip(local, orig):
                t.copy_(o)
        job.run()
        torch.cuda.synchronize()
        tag = f"case {case} (counts {counts}, P {P}, r {r}, {kind}, fails {fails}, corr {list(corr)}, fused {job.fused}, round {rnd})"
        try:
            assert_same_floats(job.merged.cpu().numpy(), want["merged"])
            if kind == "bf16":
                bits = np.array([orc.lib().orc_f32_to_bf16(float(v)) for v in want["merged"][:3000].astype(np.float32)],
                                dtype=np.uint16)
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
            raise AssertionError(tag + ": " + str(e))
    job.close()
    dist.barrier()
assert fused_seen >= n_cases // 2, fused_seen
dist.destroy_process_group()
print("rank", rank, "ok", fused_seen, "fused of", n_cases)
'''


@pytest.mark.parametrize("world", [2, 4])
def test_multigpu_fuzz(world, tmp_path):
    import torch

    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(28500 + os.getpid() % 1000 + world), str(script),
           str(ROOT), "24" if world == 2 else "12"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
