"""Run one small multi-GPU merge with the ring watchdog on (debug=1: the watchdog of the chunked executor)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17766_b200.device import DevicePlan  # noqa: E402
from paper_2507_17766_b200.multigpu import ShardedButterflyMerge  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096 * 8 + 5
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 4096 * 2
nloc = int(sys.argv[3]) if len(sys.argv) > 3 else 3
local = [torch.rand(P, device=dev) for _ in range(nloc)]
plan = DevicePlan(nloc * world, P, 0, device=dev)
job = ShardedButterflyMerge(local, plan, chunk=chunk, executor="chunked", debug=1)
print(f"[rank {rank}] K={job.K} debug={job.debug}", flush=True)
for r in range(3):
    job.run()
    torch.cuda.synchronize()
    print(f"[rank {rank}] round {r} ok", flush=True)
dist.barrier()
dist.destroy_process_group()
