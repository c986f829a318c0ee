"""Multi-GPU merge against the oracle: bit-exact merged values, own replicas, status,
flags and agreement entries on every rank.

Every case runs twice: as a single-device LOOPBACK (every rank a thread on one GPU,
multigpu.run_loopback: the same k_ring / chunked-ring kernels and host logic, the
persistent ring as one cooperative launch of G x L CTAs) — so the driver's 1-GPU box
checks the multi-GPU path — and, given >= G GPUs, as torchrun workers (one process per
GPU, NCCL + CUDA IPC)."""

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
import torch, torch.distributed as dist
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/oracle", sys.argv[1] + "/tests"]
from _multigpu_cases import case_data, run_rank
from paper_2507_17766_b200.multigpu import DistComm
case = json.loads(sys.argv[2])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
run_rank(case, case_data(case), rank, DistComm(), dev)
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
    # adversarial (config 5 pattern at reduced size): noise-deceptive miners on every rank,
    # persistent ring with predicted outcomes + FINISH on the last rank
    {"counts": [4, 4, 4, 4], "P": 2_000_039, "seed": 28, "failures": [],
     "corr": {"1": [3, 2.0, 24301, 1], "6": [3, 2.0, 24301, 6], "9": [3, 2.0, 24301, 9], "15": [3, 2.0, 24301, 15]},
     "fallback": False, "chunk": 1 << 20, "fused": True, "rounds": 2},
    # eight ranks (config 3's G = 8 layout at reduced size): honest and adversarial
    {"counts": [2] * 8, "P": 1_500_007, "seed": 33, "failures": [], "corr": {}, "fallback": False,
     "chunk": 1 << 20, "fused": True, "rounds": 3},
    {"counts": [2] * 8, "P": 1_200_011, "seed": 34, "failures": [5],
     "corr": {"1": [3, 2.0, 24301, 1], "9": [3, 2.0, 24301, 9], "14": [3, 2.0, 24301, 14]},
     "fallback": False, "chunk": 1 << 20, "fused": True, "rounds": 2},
    # the same with the pair statistics accumulated inside k_ring (fuse_stats)
    {"counts": [3, 5], "P": 2_000_029, "seed": 32, "failures": [],
     "corr": {"1": [3, 2.0, 24301, 1], "6": [3, 2.0, 24301, 6], "7": [1, 0.0]},
     "fallback": False, "chunk": 1 << 20, "fused": True, "rounds": 2, "fuse_stats": True},
    {"counts": [4, 4, 4, 4], "P": 2_000_039, "seed": 35, "failures": [3],
     "corr": {"1": [3, 2.0, 24301, 1], "6": [4, 2.0, 24301, 6], "9": [4, 0.5, 7, 7], "15": [4, 0.5, 7, 7]},
     "fallback": False, "chunk": 1 << 20, "fused": True, "rounds": 3, "fuse_stats": True},
    {"counts": [3, 3, 3], "P": 1_800_017, "seed": 36, "failures": [],
     "corr": {"2": [4, 2.0, 11, 2], "4": [4, 1e-9, 11, 4]}, "fallback": False, "chunk": 1 << 20, "bf16": True,
     "fused": True, "rounds": 2, "fuse_stats": True},
    # non-finite weights (a diverged miner): fast shards with NaN / Inf means are
    # disagreements decided after the exchange and re-broadcast
    {"counts": [3, 3], "P": 600_011, "seed": 29, "failures": [], "corr": {}, "fallback": True,
     "chunk": 1 << 20, "fused": True, "rounds": 2, "poison": [[0, 17, "nan"], [4, 300_000, "inf"], [5, 599_999, "-inf"]]},
    {"counts": [2, 2, 2], "P": 400_009, "seed": 30, "failures": [], "corr": {}, "fallback": False,
     "chunk": 1 << 20, "fused": True, "poison": [[1, 5, "nan"], [3, 200_000, "inf"]]},
    {"counts": [3, 3], "P": 300_007, "seed": 31, "failures": [2], "corr": {}, "fallback": True,
     "chunk": 65536, "executor": "chunked", "poison": [[0, 17, "nan"], [4, 150_000, "inf"]]},
]


def _ids(c):
    return f"{c['counts']}_P{c['P']}"


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_loopback_merge_matches_oracle(case, cuda_device):
    """Every rank of the case as a thread on ONE GPU (LoopbackComm)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from _multigpu_cases import case_data, run_rank

    from paper_2507_17766_b200.multigpu import run_loopback

    d = case_data(case)
    world = len(case["counts"])
    fused = run_loopback(world, lambda rank, comm: run_rank(case, d, rank, comm, cuda_device), device=cuda_device)
    assert len(set(fused)) == 1


@pytest.mark.parametrize("case", CASES, ids=_ids)
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


WORKER_FULL = r'''
import os, sys
import torch, torch.distributed as dist
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/oracle", sys.argv[1] + "/tests"]
from _multigpu_cases import fullsize_case, fullsize_check, fullsize_rank
from paper_2507_17766_b200.multigpu import DistComm
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
case = fullsize_case(world)
out = fullsize_rank(case, rank, DistComm(), dev)
allres = [None] * world
dist.gather_object(out, allres if rank == 0 else None, dst=0)
if rank == 0:
    fullsize_check(case, allres)
    print("FULLSIZE OK")
dist.barrier()
dist.destroy_process_group()
'''


def test_sharded_full_size(tmp_path):
    """Config 5's pattern at full size on 4 GPUs (16 miners x 1e9 fp32 per GPU, 64 miners,
    6 noise-deceptive), one process per GPU: closed forms on every rank and sampled shards
    against the oracle (the 2-rank loopback twin is in test_gpu_fullsize.py)."""
    import torch

    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    import gc

    gc.collect()
    torch.cuda.empty_cache()  # this process's cached blocks (earlier tests) back to the driver
    for d in range(4):
        if torch.cuda.mem_get_info(d)[0] < 80 * 2**30:
            pytest.skip(f"GPU {d} has < 80 GB free")
    script = tmp_path / "worker_full.py"
    script.write_text(WORKER_FULL)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr", "127.0.0.1", "--master-port", str(29400 + os.getpid() % 1000), str(script), str(ROOT)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    err = r.stderr[r.stderr.find("Traceback"):][:4000] if "Traceback" in r.stderr else r.stderr[-3000:]
    assert r.returncode == 0 and "FULLSIZE OK" in r.stdout, r.stdout[-2000:] + err
