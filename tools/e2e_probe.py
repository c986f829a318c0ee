"""Drop-in e2e (butterfly.run_all_reduce on fp64 payloads in pinned host memory) for a few
upload staging block sizes and thread counts: ms per round and GB/s (the bench's e2e
definition).    python tools/e2e_probe.py [P] [blocks,...] [threads,...]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2507_17766_b200 import butterfly as bf  # noqa: E402
from paper_2507_17766_b200.simkernel import BlobStore  # noqa: E402

n = 16
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
blocks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1 << 19]
threads = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
payloads = {}
g = torch.Generator()
for m in range(n):
    g.manual_seed(1000 + m)
    payloads[m] = torch.empty(P, dtype=torch.float64, pin_memory=True).uniform_(-1, 1, generator=g).numpy()
plan = bf.plan_shards(bf.enumerate_pairs(n), P, 4, 0)
for block in blocks:
    for th in threads:
        bf._UPLOAD_BLOCK, bf._UPLOAD_THREADS = block, th
        bf.run_all_reduce(BlobStore(), payloads, plan)
        t = time.perf_counter()
        for _ in range(3):
            bf.run_all_reduce(BlobStore(), payloads, plan)
        dt = (time.perf_counter() - t) / 3
        print(f"block {block:8d} threads {th:3d}: {dt * 1e3:8.1f} ms  {2 * n * P * 4 / dt / 1e9:6.1f} GB/s", flush=True)
