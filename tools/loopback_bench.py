"""Time (and, under ncu, capture) the persistent ring in single-device loopback: G ranks
of n_local miners each, all on cuda:0, one cooperative k_ring_loop launch per round.

    python tools/loopback_bench.py G n_local P [rounds] [deceptive]

Prints the round time and the algorithmic bytes of the round on this one device: every
replica read once and written once (2 * G * n_local * P * 4), plus what crosses the
"NVLink" inboxes (fp64 running sums into ranks > 0, final values into ranks < last),
which in loopback stays in this GPU's L2 / HBM.
"""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import torch  # noqa: E402

from paper_2507_17766_b200.device import Corruption, DevicePlan  # noqa: E402
from paper_2507_17766_b200.multigpu import ShardedButterflyMerge, run_loopback  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_local = int(sys.argv[2]) if len(sys.argv) > 2 else 8
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 27
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 5
k_bad = int(sys.argv[5]) if len(sys.argv) > 5 else 0
dev = torch.device("cuda", 0)
n = G * n_local


def body(rank, comm):
    g = torch.Generator(device=dev)
    reps = []
    for i in range(n_local):
        g.manual_seed(rank * n_local + i)
        reps.append(torch.empty(P, dtype=torch.float32, device=dev).uniform_(-1, 1, generator=g))
    plan = DevicePlan(n, P, 0, device=dev)
    import numpy as np

    bad = sorted(int(x) for x in np.random.default_rng(0).choice(n, k_bad, replace=False)) if k_bad else []
    job = ShardedButterflyMerge(reps, plan, corruptions={m: Corruption.noise(2.0, (0x5EED, m)) for m in bad},
                                comm=comm)
    assert job.fused
    cur = torch.cuda.current_stream(dev)
    job.run()
    cur.synchronize()
    comm.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(cur)
    for _ in range(rounds):
        job.run()
    ev[1].record(cur)
    cur.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / rounds
    job.close()
    return ms


t = time.time()
ms = max(run_loopback(G, body, device=dev))
alg = 2 * n * P * 4
inbox = (G - 1) * P * 8 + (G - 1) * P * 4
print(f"loopback G={G} n_local={n_local} P={P} deceptive={k_bad}: {ms:.3f} ms/round; replica bytes "
      f"{alg / 1e9:.2f} GB -> {alg / ms / 1e6:.0f} GB/s; inbox bytes {inbox / 1e9:.2f} GB "
      f"(wall {time.time() - t:.1f} s)")
