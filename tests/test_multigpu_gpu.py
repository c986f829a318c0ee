"""Multi-GPU merge (NCCL chain) against the oracle: bit-exact merged values,
status, flags and agreement entries on every rank.  Needs >= 2 GPUs; launched
as torchrun workers from the test (one process per GPU)."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
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
case = json.loads(sys.argv[2])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
counts, P, seed = case["counts"], case["P"], case["seed"]
n = sum(counts)
rng = np.random.default_rng(7)
data = (rng.uniform(-1, 1, (n, P)) * 10.0 ** rng.integers(-4, 4, (n, 1))).astype(np.float32)
r = case.get("r", 2)
bf16 = case.get("bf16", False)
if bf16:
    data = (data.view(np.uint32) >> 16).astype(np.uint16)
fails = tuple(case["failures"])
specs = {int(k): tuple(v) for k, v in case["corr"].items()}
fb = rng.uniform(-2, 2, P) if case["fallback"] else None
assign, bounds = orc.plan(n, P, seed, r=r)
want = orc.merge(list(data), assign, bounds, failures=fails, corruptions=specs, fallback=fb,
                 dtype=orc.BF16 if bf16 else orc.F32)
off = sum(counts[:rank])
if bf16:
    local = [torch.from_numpy(data[off + i].view(np.int16).copy()).to(dev).view(torch.bfloat16)
             for i in range(counts[rank])]
else:
    local = [torch.from_numpy(data[off + i].copy()).to(dev) for i in range(counts[rank])]
plan = DevicePlan(n, P, seed, redundancy=r, device=dev)
kinds = {1: "add", 2: "scale", 3: "noise", 4: "noise_add"}
corr = {m: Corruption(kinds[s[0]], s[1], (s[2], s[3]) if len(s) > 2 else (0, 0)) for m, s in specs.items()}
job = ShardedButterflyMerge(local, plan, failures=fails, corruptions=corr,
                            fallback=None if fb is None else torch.from_numpy(fb).to(dev),
                            chunk=case["chunk"], want_merged=True)
if "fused" in case:
    assert job.fused == case["fused"], (job.fused, case["fused"])
orig = [t.clone() for t in local]
for rnd in range(case.get("rounds", 1)):
    if rnd:  # refill the replicas in place: the next round reuses slots and flags
        for t, o in zip(local, orig):
            t.copy_(o)
    job.run()
    torch.cuda.synchronize()
    assert_same_floats(job.merged.cpu().numpy(), want["merged"])
    if not bf16:
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
dist.barrier()
dist.destroy_process_group()
print("rank", rank, "ok")
'''

CASES = [
    {"counts": [4, 4], "P": 1_000_003, "seed": 3, "failures": [], "corr": {}, "fallback": False, "chunk": 65536},
    {"counts": [3, 5], "P": 777_777, "seed": 9, "failures": [0, 6], "corr": {"2": [3, 1.0, 5, 6], "7": [1, 0.5]},
     "fallback": False, "chunk": 4096 * 7},
    {"counts": [2, 6], "P": 300_001, "seed": 4, "failures": [1, 2], "corr": {"5": [3, 2.0, 1, 1], "6": [3, 2.0, 1, 1]},
     "fallback": True, "chunk": 4096},
    {"counts": [3, 2, 4], "P": 500_009, "seed": 6, "failures": [4], "corr": {"1": [1, 0.5]}, "fallback": False,
     "chunk": 4096 * 9},
    {"counts": [4, 3], "P": 350_003, "seed": 8, "failures": [2], "corr": {"5": [3, 1.0, 2, 2]}, "fallback": True,
     "chunk": 65536, "bf16": True},
    {"counts": [3, 4], "P": 35 * 2000 + 3, "seed": 10, "failures": [0], "corr": {"6": [3, 1.0, 4, 4]},
     "fallback": False, "chunk": 8192, "r": 3},
    # ramped chunk sizes (1M/16 .. 1M .. 1M/16, multigpu.chunk_edges), fallback values in chunk groups
    {"counts": [3, 3], "P": 5_000_011, "seed": 12, "failures": [4], "corr": {"1": [3, 2.0, 9, 9], "5": [1, 0.0]},
     "fallback": False, "chunk": 1 << 20},
    {"counts": [2, 2, 2, 2], "P": 6_000_007, "seed": 13, "failures": [], "corr": {"3": [3, 1.0, 2, 3]},
     "fallback": False, "chunk": 1 << 20},
    # persistent single-kernel ring (bfly_ring_fused): every shard fast; several rounds
    # reuse the slot rings and the monotonic flags; partial last tiles; uneven lanes
    {"counts": [4, 4], "P": 3_000_017, "seed": 21, "failures": [], "corr": {}, "fallback": False,
     "chunk": 1 << 20, "fused": True, "rounds": 8},
    {"counts": [3, 5], "P": 2_345_679, "seed": 22, "failures": [6], "corr": {}, "fallback": False,
     "chunk": 1 << 20, "fused": True, "rounds": 2},
    {"counts": [2, 3, 2], "P": 1_234_567, "seed": 23, "failures": [0], "corr": {}, "fallback": False,
     "chunk": 1 << 20, "fused": True, "rounds": 2},
    {"counts": [2, 2, 2, 2], "P": 4_000_037, "seed": 24, "failures": [], "corr": {}, "fallback": False,
     "chunk": 1 << 20, "fused": True, "rounds": 8},
    {"counts": [3, 3], "P": 1_500_007, "seed": 25, "failures": [1], "corr": {}, "fallback": False,
     "chunk": 1 << 20, "bf16": True, "fused": True, "rounds": 2},
    {"counts": [2, 3], "P": 10 * 3000 + 7, "seed": 26, "failures": [3, 4], "corr": {}, "fallback": False,
     "chunk": 8192, "r": 3, "fused": True, "rounds": 2},
    {"counts": [1, 2], "P": 9_001, "seed": 27, "failures": [], "corr": {}, "fallback": False,
     "chunk": 8192, "fused": True, "rounds": 4},
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['counts']}_P{c['P']}")
def test_sharded_merge_matches_oracle(case, tmp_path):
    import json

    import torch

    if torch.cuda.device_count() < len(case["counts"]):
        pytest.skip(f"needs {len(case['counts'])} GPUs")
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={len(case['counts'])}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000), str(script), str(ROOT),
           json.dumps(case)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
