"""Small driver for ncu captures of the merge kernels (one GPU).

    python tools/prof_merge.py --miners 16 --params 67108864 --runs 3 [--dtype fp32|bf16] [--r 2] [--bad 0]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import deceptive_set, make_replicas  # noqa: E402
from paper_2507_17766_b200.device import ButterflyMerge, Corruption, DevicePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--miners", type=int, default=16)
ap.add_argument("--params", type=int, default=1 << 26)
ap.add_argument("--dtype", default="fp32")
ap.add_argument("--r", type=int, default=2)
ap.add_argument("--bad", type=int, default=0)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--merged", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda:0")
reps = make_replicas(a.miners, a.params, a.dtype, dev)
plan = DevicePlan(a.miners, a.params, 0, redundancy=a.r, device=dev)
corr = {m: Corruption.noise(2.0, (0x5EED, m)) for m in deceptive_set(a.miners, a.bad)}
job = ButterflyMerge(reps, plan, corruptions=corr, want_merged=a.merged)
for _ in range(a.runs):
    job.run()
torch.cuda.synchronize()
print("ok", a)
