"""Round time of a small merge (config 1: 8 miners x 10M fp32) issued kernel by kernel vs
replayed from a CUDA graph (ButterflyMerge.capture()).  One GPU."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import make_replicas  # noqa: E402
from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan  # noqa: E402

dev = torch.device("cuda:0")
for n, P in ((8, 10_000_000), (8, 1_000_000), (16, 100_000)):
    reps = make_replicas(n, P, "fp32", dev)
    job = ButterflyMerge(reps, DevicePlan(n, P, 0, device=dev))
    for mode in ("launches", "graph"):
        if mode == "graph":
            job.capture()
        for _ in range(10):
            job.run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(100):
            job.run()
        b.record()
        torch.cuda.synchronize()
        print(f"{n} miners x {P}: {mode:8s} {a.elapsed_time(b) / 100 * 1e3:8.1f} us per round", flush=True)
