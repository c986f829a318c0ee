"""One launch of each hot kernel on one GPU, for ncu captures.

    python tools/prof_kernels.py
k_reduce (16 replicas x 2^26 fp32, all shards honest), k_chain with TMA bulk stores
(16 x 2^24 into a local fp64 buffer), k_fanout (2^24 fp32 into 16 replicas), and the
special-shard kernels k_stats / k_apply (6 of 16 miners deceptive, 2^26).
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import deceptive_set, make_replicas  # noqa: E402
from paper_2507_17766_b200 import _lib as L  # noqa: E402
from paper_2507_17766_b200.device import ButterflyMerge, Corruption, DevicePlan, _stream_handle  # noqa: E402

dev = torch.device("cuda:0")
lib = L.lib()
P = 1 << 26
reps = make_replicas(16, P, "fp32", dev)
plan = DevicePlan(16, P, 0, device=dev)
ButterflyMerge(reps, plan).run()
C = 1 << 24
tab = torch.tensor([t.data_ptr() for t in reps], dtype=torch.int64, device=dev)
out = torch.empty(C, dtype=torch.float64, device=dev)
L.check(lib.bfly_chain_step(tab.data_ptr(), 16, 0, None, out.data_ptr(), 0, C, _stream_handle()))
fin = torch.rand(C, device=dev)
views = torch.tensor([t.data_ptr() for t in reps], dtype=torch.int64, device=dev)
L.check(lib.bfly_fanout(fin.data_ptr(), views.data_ptr(), 16, C * 4, _stream_handle()))
corr = {m: Corruption.noise(2.0, (0x5EED, m)) for m in deceptive_set(16, 6)}
ButterflyMerge(reps, plan, corruptions=corr).run()
torch.cuda.synchronize()
print("ok")
