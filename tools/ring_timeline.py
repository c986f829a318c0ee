"""Per-op completion times of one multi-GPU round (chunked executor issued from Python, debug=3).

    torchrun --nproc-per-node 4 tools/ring_timeline.py [--params 1e9] [--bad 6] [--miners-per-gpu 16]

Writes gpurun_out/timeline_rank{g}.json: [[kind, stream, chunk, ms], ...] for the third
round (two warm-up rounds first).
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from bench import deceptive_set, make_replicas  # noqa: E402
from paper_2507_17766_b200.device import Corruption, DevicePlan  # noqa: E402
from paper_2507_17766_b200.multigpu import ShardedButterflyMerge  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--params", type=float, default=1e9)
ap.add_argument("--bad", type=int, default=6)
ap.add_argument("--miners-per-gpu", type=int, default=16)
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
P, nl = int(a.params), a.miners_per_gpu
n = nl * world
local = make_replicas(nl, P, "fp32", dev, seed=rank * nl)
plan = DevicePlan(n, P, 0, device=dev)
corr = {m: Corruption.noise(2.0, (0x5EED, m)) for m in deceptive_set(n, a.bad)}
job = ShardedButterflyMerge(local, plan, corruptions=corr, executor="chunked", debug=3)
for _ in range(3):
    job.run()
tl = [[op[0], op[1], op[2], ms] for op, ms in job.timeline()]
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
(out / f"timeline_rank{rank}.json").write_text(json.dumps(tl))
dist.barrier()
dist.destroy_process_group()
