"""Host->device upload of fp64 payloads as fp32 wire values (bfly_upload_wire): block /
ring / thread sweep, then the drop-in run_all_reduce end to end.  One GPU.

    python tools/upload_probe.py [--miners 16] [--log2p 27]
"""
import argparse
import ctypes
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2507_17766_b200 import _lib as L  # noqa: E402
from paper_2507_17766_b200 import butterfly as bf  # noqa: E402
from paper_2507_17766_b200.device import _stream_handle  # noqa: E402
from paper_2507_17766_b200.simkernel import BlobStore  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--miners", type=int, default=16)
ap.add_argument("--log2p", type=int, default=27)
a = ap.parse_args()
n, P = a.miners, 1 << a.log2p
dev = torch.device("cuda:0")
host = [torch.empty(P, dtype=torch.float64, pin_memory=True).uniform_(-1, 1) for _ in range(n)]
wire = [torch.empty(P, dtype=torch.float32, device=dev) for _ in range(n)]
h_ptrs = (ctypes.c_void_p * n)(*[h.data_ptr() for h in host])
d_ptrs = (ctypes.c_void_p * n)(*[w.data_ptr() for w in wire])
gb = n * P * 4 / 1e9
print(f"cpus {os.cpu_count()} miners {n} P 2^{a.log2p}: {gb:.2f} GB fp32 wire", flush=True)
for threads in (os.cpu_count(),):
    for block in (1 << 19,):
        for ring in (3,):
            os.environ["BFLY_UPLOAD_BLOCK"] = str(block)
            os.environ["BFLY_UPLOAD_RING"] = str(ring)
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize()
                t = time.perf_counter()
                L.check(L.lib().bfly_upload_wire(h_ptrs, n, P, d_ptrs, threads, _stream_handle()))
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t)
            print(f"threads {threads:2d} block {block:8d} ring {ring}: {best * 1e3:7.1f} ms  "
                  f"{gb / best:6.1f} GB/s wire", flush=True)
for every in ("0", "8", "5", "4", "3"):
    os.environ["BFLY_UPLOAD_RAW_EVERY"] = every
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        L.check(L.lib().bfly_upload_wire(h_ptrs, n, P, d_ptrs, 0, _stream_handle()))
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    ok = all(torch.equal(w.cpu(), h.float()) for w, h in zip(wire[:3], host[:3]))
    print(f"raw every {every}: {best * 1e3:7.1f} ms  {gb / best:6.1f} GB/s wire  exact {ok}", flush=True)

ok = all(torch.equal(w.cpu(), h.float()) for w, h in zip(wire[:2], host[:2]))
print("values exact:", ok)
os.environ.pop("BFLY_UPLOAD_BLOCK")
os.environ.pop("BFLY_UPLOAD_RING")
payloads = {m: host[m].numpy() for m in range(n)}
os.environ.pop("BFLY_UPLOAD_RAW_EVERY")
plan = bf.plan_shards(bf.enumerate_pairs(n), P, 4, 0)
for _ in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = bf.run_all_reduce(BlobStore(), payloads, plan)
    print(f"run_all_reduce {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
