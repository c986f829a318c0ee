"""Cost of the last rank's remote store: k_reduce over a 16M-element chunk (16 replicas,
fp64 running sums in) scattering into the 16 replicas plus one more target that is
(a) a local buffer, (b) a buffer on another GPU (peer access over NVLink), (c) absent.
Needs 2 GPUs.

    python tools/remote_store_probe.py
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan  # noqa: E402

C, n = 1 << 24, 16
P = 4 * C
d0, d1 = torch.device("cuda:0"), torch.device("cuda:1")
rt = ctypes.CDLL("libcudart.so.12")
torch.cuda.set_device(d0)
torch.zeros(1, device=d1)
torch.zeros(1, device=d0)
rc = rt.cudaDeviceEnablePeerAccess(1, 0)
print("peer access enable rc", rc, "can access", torch.cuda.can_device_access_peer(0, 1), flush=True)
reps = [torch.rand(P, device=d0) for _ in range(n)]
plan = DevicePlan(2 * n, P, 0, device=d0)
job = ButterflyMerge([None] * n + reps, plan, remote_sum=True, n_div=2 * n, scatter_back=True)
acc = torch.rand(C, dtype=torch.float64, device=d0)
local_out = torch.empty(C, device=d0)
remote_out = torch.empty(C, device=d1)


def table(extra):
    ptrs = [t.data_ptr() for t in reps]
    return torch.tensor(ptrs + ([extra] if extra is not None else []), dtype=torch.int64, device=d0)


cases = {"local extra target": table(local_out.data_ptr() - C * 4),  # biased by -begin (chunk 1)
         "remote extra target": table(remote_out.data_ptr() - C * 4),
         "no extra target": table(None)}
for name, tab in cases.items():
    for _ in range(3):
        job.reduce_range(0, C, acc_in=acc, dst_table=(tab.data_ptr(), tab.numel()))
        job.reduce_range(C, 2 * C, acc_in=acc, dst_table=(tab.data_ptr(), tab.numel()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        job.reduce_range(C, 2 * C, acc_in=acc, dst_table=(tab.data_ptr(), tab.numel()))
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10:.3f} ms per 16M-element chunk", flush=True)
