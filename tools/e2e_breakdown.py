"""Where does the drop-in (host payload) merge spend its time?  One GPU."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2507_17766_b200 import butterfly as bf  # noqa: E402
from paper_2507_17766_b200.simkernel import BlobStore  # noqa: E402

n, P = 16, 1 << 27
dev = torch.device("cuda:0")
host = [torch.empty(P, dtype=torch.float64, pin_memory=True).uniform_(-1, 1) for _ in range(n)]
print("pinned:", host[0].is_pinned(), "numpy view pinned:", torch.from_numpy(host[0].numpy()).is_pinned())
dst = [torch.empty(P, dtype=torch.float64, device=dev) for _ in range(n)]
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    for h, d in zip(host, dst):
        d.copy_(torch.from_numpy(h.numpy()), non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"H2D {n*P*8/1e9:.1f} GB in {dt*1e3:.1f} ms = {n*P*8/dt/1e9:.1f} GB/s")
out = torch.empty(P, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter(); out.copy_(dst[0], non_blocking=True); torch.cuda.synchronize()
print(f"D2H pinned {P*8/1e9:.2f} GB {1e3*(time.perf_counter()-t):.1f} ms")
t = time.perf_counter(); x = dst[0].cpu(); print(f"D2H pageable {1e3*(time.perf_counter()-t):.1f} ms")
payloads = {m: host[m].numpy() for m in range(n)}
plan = bf.plan_shards(bf.enumerate_pairs(n), P, 4, 0)
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    res = bf.run_all_reduce(BlobStore(), payloads, plan)
    print(f"run_all_reduce {1e3*(time.perf_counter()-t):.1f} ms")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile(); pr.enable(); res = bf.run_all_reduce(BlobStore(), payloads, plan); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
