"""Per-phase times of multi-GPU merge rounds, averaged over rounds (CUDA events between
the phases of ShardedButterflyMerge.run, timing mode): which phase of a round a change
moved.  Works with any build of the package (A/B: point ROOT at another checkout).

    torchrun --nproc-per-node 4 tools/phase_probe.py [ROOT] [miners_per_gpu] [deceptive] [rounds] [fuse]
"""
import json
import os
import sys

root = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.abspath(root))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17766_b200.device import Corruption, DevicePlan  # noqa: E402
from paper_2507_17766_b200.multigpu import ShardedButterflyMerge  # noqa: E402

n_local = int(sys.argv[2]) if len(sys.argv) > 2 else 16
k_bad = int(sys.argv[3]) if len(sys.argv) > 3 else 6
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 10
fuse = len(sys.argv) > 5 and sys.argv[5] == "fuse"
P = 1_000_000_000
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
n = n_local * world
g = torch.Generator(device=dev)
reps = []
for i in range(n_local):
    g.manual_seed(rank * n_local + i)
    reps.append(torch.empty(P, dtype=torch.float32, device=dev).uniform_(-1, 1, generator=g))
plan = DevicePlan(n, P, 0, device=dev)
bad = sorted(int(x) for x in np.random.default_rng(0).choice(n, k_bad, replace=False)) if k_bad else []
job = ShardedButterflyMerge(reps, plan, fuse_stats=fuse, corruptions={m: Corruption.noise(2.0, (0x5EED, m)) for m in bad})
for _ in range(3):
    job.run()
torch.cuda.synchronize()
job.timing = True
acc = {}
for _ in range(rounds):
    dist.barrier()
    job.run()
    for k, v in job.timings.items():
        acc.setdefault(k, []).append(v)
out = {k: round(float(np.median(v)), 3) for k, v in acc.items()}
allp = [None] * world
dist.all_gather_object(allp, out)
if rank == 0:
    print(json.dumps({"root": root, "fuse_stats": fuse, "fused": job.fused, "median_ms_per_phase_by_rank": allp}))
dist.barrier()
dist.destroy_process_group()
