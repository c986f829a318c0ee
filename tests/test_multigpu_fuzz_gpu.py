"""Seeded fuzz of the multi-GPU merge against the oracle: random miner counts per rank,
payload lengths (partial last tiles, lengths below one tile per lane), redundancy 2/3,
fp32 / bf16 / fp64 replicas, failures (fewer than r, so the persistent ring kernel
k_ring runs; a few cases with corruptions take the chunked ring), several rounds per
case with the replicas refilled in place (slot rings and monotonic flags carry over).
Every rank checks merged values, its own replicas, status, flags and entries bit for
bit (entries <= 1e-12).  Runs as a single-device loopback (ranks as threads on one GPU)
and, given enough GPUs, as one torchrun job per world size."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import os, sys
import torch, torch.distributed as dist
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/oracle", sys.argv[1] + "/tests"]
from _multigpu_cases import fuzz_case, fuzz_rank
from paper_2507_17766_b200.multigpu import DistComm
n_cases = int(sys.argv[2])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
comm = DistComm()
fused_seen = 0
for case in range(n_cases):
    c = fuzz_case(case, world)
    try:
        fused_seen += fuzz_rank(c, rank, comm, dev)
    except AssertionError as e:
        raise AssertionError(f"case {case}: {e}") from None
    dist.barrier()
assert fused_seen >= n_cases // 2, fused_seen
dist.destroy_process_group()
print("rank", rank, "ok", fused_seen, "fused of", n_cases)
'''


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_multigpu_fuzz_loopback(world, cuda_device):
    """The same seeded cases with every rank a thread on ONE GPU (multigpu.run_loopback)."""
    from _multigpu_cases import fuzz_case, fuzz_rank

    from paper_2507_17766_b200.multigpu import run_loopback

    n_cases = {2: 24, 3: 12, 4: 12, 8: 6}[world] * int(os.environ.get("BFLY_FUZZ_SCALE", "1"))  # soak: > 1
    fused_seen = 0
    for case in range(n_cases):
        c = fuzz_case(case, world)
        try:
            fused = run_loopback(world, lambda rank, comm: fuzz_rank(c, rank, comm, cuda_device), device=cuda_device)
        except AssertionError as e:
            raise AssertionError(f"case {case}: {e}") from None
        fused_seen += fused[0]
    assert fused_seen >= n_cases // 2, fused_seen


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
