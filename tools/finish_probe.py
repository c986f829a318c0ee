"""Config 5's multi-GPU layout on ONE device (loopback ranks): per-phase times of the
last rank's FINISH (k_stats / k_decide / k_apply after the persistent ring), so the
kernels can be profiled with ncu (`--kernel-name regex:k_stats`).

    python tools/finish_probe.py [world] [miners_per_rank] [P] [deceptive] [rounds] [fuse]
"""
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.environ.get("BFLY_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_17766_b200.device import Corruption, DevicePlan  # noqa: E402
from paper_2507_17766_b200.multigpu import ShardedButterflyMerge, run_loopback  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n_local = int(sys.argv[2]) if len(sys.argv) > 2 else 16
P = int(float(sys.argv[3])) if len(sys.argv) > 3 else 250_000_000
k_bad = int(sys.argv[4]) if len(sys.argv) > 4 else 6
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 5
fuse = len(sys.argv) > 6 and sys.argv[6] == "fuse"
dev = torch.device("cuda", 0)
n = n_local * world
bad = sorted(int(x) for x in np.random.default_rng(0).choice(n, k_bad, replace=False)) if k_bad else []


def body(rank, comm):
    g = torch.Generator(device=dev)
    reps = []
    for i in range(n_local):
        g.manual_seed(rank * n_local + i)
        reps.append(torch.empty(P, dtype=torch.float32, device=dev).uniform_(-1, 1, generator=g))
    plan = DevicePlan(n, P, 0, device=dev)
    job = ShardedButterflyMerge(reps, plan, comm=comm, fuse_stats=fuse,
                                corruptions={m: Corruption.noise(2.0, (0x5EED, m)) for m in bad})
    job.run()
    job.timing = True
    acc = {}
    for _ in range(rounds):
        job.run()
        for k, v in job.timings.items():
            acc.setdefault(k, []).append(v)
    out = {k: round(float(np.median(v)), 3) for k, v in acc.items()}
    fused = job.fused
    job.close()
    return {"rank": rank, "fused": fused, "ms": out}


res = run_loopback(world, body, device=dev)
print(json.dumps({"fuse_stats": fuse, "world": world, "n": n, "P": P, "deceptive": bad, "phases": res}))
