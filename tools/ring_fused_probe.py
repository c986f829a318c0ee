"""Diagnostics of the persistent multi-GPU ring (k_ring, csrc/bfly_ring.cu).

    torchrun --nproc-per-node G tools/ring_fused_probe.py [P] [miners_per_gpu] [profile]

Times a few rounds with CUDA events (max over ranks) and prints, per rank, the
share of the kernel's cycles each role spent waiting (mean over CTAs):
loader (replica stage free, upstream ready flag, acc stage free), compute (acc
tile, out stage free, replica stage full), storer (out tile, downstream free
flag, stage read-out, landing), relay loader (ready flag, stage free), relay
storer (stage full, downstream free flag, read-out, landing).
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2507_17766_b200.device import DevicePlan  # noqa: E402
from paper_2507_17766_b200.multigpu import ShardedButterflyMerge  # noqa: E402

NAMES = ["ld.rep_empty", "ld.schedule", "ld.ready_flag+acc_empty", "-", "cmp.acc_full", "cmp.out_empty", "cmp.rep_full",
         "total_cycles", "st.out_full", "st.free_flag", "st.read", "st.landed", "rl.ready_flag", "rl.rel_empty", "-",
         "-", "rs.rel_full", "rs.free_flag", "rs.read", "rs.landed", "t_start", "t_end", "-", "-"]


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
    n_local = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    g = torch.Generator(device=dev)
    reps = []
    for i in range(n_local):
        g.manual_seed(rank * n_local + i)
        reps.append(torch.empty(P, dtype=torch.float32, device=dev).uniform_(-1, 1, generator=g))
    plan = DevicePlan(n_local * world, P, 0, device=dev)
    job = ShardedButterflyMerge(reps, plan)
    assert job.fused
    profile = len(sys.argv) > 3 and sys.argv[3] == "profile"
    prof = torch.zeros(job.lanes * 24, dtype=torch.int64, device=dev) if profile else None
    if profile:  # the descriptor's diagnostics buffer (bfly.h d_profile)
        job._fdesc.d_profile = prof.data_ptr()
    for _ in range(2):
        job.run()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    rounds = 3
    ev[0].record()
    for _ in range(rounds):
        job.run()
    ev[1].record()
    torch.cuda.synchronize()
    ms = torch.tensor([ev[0].elapsed_time(ev[1]) / rounds], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    out = {"rank": rank, "round_ms": round(float(ms.item()), 3), "lanes": job.lanes}
    if profile:
        a = prof.cpu().numpy().view(np.uint64).reshape(job.lanes, 24).astype(np.float64)
        tot = a[:, 7].mean()
        out["kernel_ms_at_1.9GHz"] = round(tot / 1.9e6, 3)
        out["wait_share"] = {NAMES[k]: round(a[:, k].mean() / tot, 3) for k in range(24)
                             if NAMES[k] not in ("-", "total_cycles", "t_start", "t_end")}
        ts, te = a[:, 20], a[:, 21]
        out["cta_ms"] = {"start_skew": round((ts.max() - ts.min()) / 1e6, 3),
                         "span": round((te.max() - ts.min()) / 1e6, 3),
                         "mean_dur": round((te - ts).mean() / 1e6, 3), "max_dur": round((te - ts).max() / 1e6, 3),
                         "end_skew": round((te.max() - te.min()) / 1e6, 3)}
        dur = (te - ts) / 1e6
        order = np.argsort(dur)
        out["lane_ms_pct"] = [round(float(np.percentile(dur, q)), 2) for q in (0, 10, 50, 90, 100)]
        out["slowest_lanes"] = [(int(c), int(a[c, 22]), round(float(dur[c]), 2)) for c in order[-6:]]
        out["fastest_lanes"] = [(int(c), int(a[c, 22]), round(float(dur[c]), 2)) for c in order[:4]]
    for r in range(world):
        if r == rank:
            print(json.dumps(out), flush=True)
        dist.barrier()
    job.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
