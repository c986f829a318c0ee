"""Sweep k_reduce variants (replicas in flight U, min CTAs/SM, grid size) on one GPU.

    make tune && python tools/tune_reduce.py [--miners 16] [--params 1000000000] [--deceptive 6]
Prints one JSON line per variant: ms per launch and GB/s of algorithmic traffic.
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import make_replicas  # noqa: E402
from paper_2507_17766_b200 import _lib as L  # noqa: E402
from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan, _stream_handle  # noqa: E402

VARIANTS = {0: (4, 1, 'auto'), 1: (4, 2, 1), 2: (8, 1, 1), 3: (8, 2, 1), 4: (4, 3, 1), 5: (16, 1, 1), 6: (2, 4, 1),
            7: (4, 1, 1)}
VARIANTS_BF16 = {0: (4, 1, 'auto'), 1: (4, 2, 1), 2: (8, 1, 1), 3: (2, 2, 1), 4: (4, 3, 1), 5: (2, 3, 1),
                 6: (2, 4, 1), 7: (4, 1, 1)}

ap = argparse.ArgumentParser()
ap.add_argument("--miners", type=int, default=16)
ap.add_argument("--params", type=int, default=1_000_000_000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"])
ap.add_argument("--r", type=int, default=2)
ap.add_argument("--deceptive", type=int, default=0, help="noise-deceptive miners (config 5: 6)")
a = ap.parse_args()
tune = ctypes.CDLL(str(ROOT / "build" / "libbfly_tune.so"))
tune.bfly_tune_reduce.argtypes = [ctypes.POINTER(L.MergeArgs), ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda:0")
reps = make_replicas(a.miners, a.params, a.dtype, dev)
plan = DevicePlan(a.miners, a.params, 0, redundancy=a.r, device=dev)
corr = {}
if a.deceptive:
    import numpy as np

    from paper_2507_17766_b200.device import Corruption
    bad = sorted(int(x) for x in np.random.default_rng(0).choice(a.miners, a.deceptive, replace=False))
    corr = {m: Corruption.noise(2.0, (0x5EED, m)) for m in bad}
job = ButterflyMerge(reps, plan, corruptions=corr)
job.run()
torch.cuda.synchronize()
args = job._args
args.phase = L.PHASE_REDUCE
alg = 2 * a.miners * a.params * (2 if a.dtype == "bf16" else 4)
for v, (U, minb, outer) in (VARIANTS_BF16 if a.dtype == "bf16" else VARIANTS).items():
    for gps in (1, 2, 4, 8, 16):
        rc = tune.bfly_tune_reduce(ctypes.byref(args), v, gps, _stream_handle())
        if rc:
            print(json.dumps({"variant": v, "error": rc}))
            continue
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(a.reps):
            tune.bfly_tune_reduce(ctypes.byref(args), v, gps, _stream_handle())
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / a.reps
        print(json.dumps({"U": U, "min_ctas": minb, "outer_unroll": outer, "grid_per_sm": gps, "ms": round(ms, 3),
                          "GBps": round(alg / ms / 1e6, 1)}), flush=True)
