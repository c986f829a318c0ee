"""A middle rank's per-chunk work on one GPU: the chain step (16 replicas + fp64 sums in
-> fp64 sums out) and the relay fan-out (one fp32 chunk -> 16 replicas + one inbox),
alone and concurrently on two streams, with 256-bit stores vs TMA bulk stores.

    python tools/fanout_probe.py [--chunk 16777216]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2507_17766_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chunk", type=int, default=1 << 24)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
C, n = a.chunk, 16
dev = torch.device("cuda:0")
lib = L.lib()
reps = [torch.rand(C * 4, device=dev) for _ in range(n)]  # replicas (4 chunks each, rotate)
acc_in = torch.rand(C, dtype=torch.float64, device=dev)
acc_out = torch.empty(C, dtype=torch.float64, device=dev)
fin = torch.rand(C, device=dev)
inbox = torch.empty(C, device=dev)
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()


def tables(j):
    src = torch.tensor([t.data_ptr() + j * C * 4 for t in reps], dtype=torch.int64, device=dev)
    dst = torch.tensor([t.data_ptr() + ((j + 2) % 4) * C * 4 for t in reps] + [inbox.data_ptr()],
                       dtype=torch.int64, device=dev)
    return src, dst


tabs = [tables(j) for j in range(4)]


def chain(j, st):
    L.check(lib.bfly_chain_step(tabs[j][0].data_ptr(), n, 0, acc_in.data_ptr(), acc_out.data_ptr(), 0, C,
                                st.cuda_stream))


def fanout(j, st):
    L.check(lib.bfly_fanout(fin.data_ptr(), tabs[j][1].data_ptr(), n + 1, C * 4, st.cuda_stream))


def timed(fn):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.reps):
        fn(i % 4)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


chain_b = (n * 4 + 16) * C
fan_b = (4 + (n + 1) * 4) * C
for bulk, cap in ((0, 0), (1, 0), (0, 296), (0, 444), (0, 592), (0, 888)):
    L.check(lib.bfly_set_fanout_bulk(bulk))
    L.check(lib.bfly_set_max_ctas(cap))
    cur = torch.cuda.current_stream()
    tc = timed(lambda j: chain(j, cur))
    tf = timed(lambda j: fanout(j, cur))

    def both(j):
        sA.wait_stream(cur)
        sB.wait_stream(cur)
        chain(j, sA)
        fanout((j + 1) % 4, sB)
        cur.wait_stream(sA)
        cur.wait_stream(sB)

    tb = timed(both)
    print(f"fanout_bulk={bulk} max_ctas={cap}: chain {tc:.3f} ms ({chain_b / tc / 1e6:.0f} GB/s)  fanout {tf:.3f} ms "
          f"({fan_b / tf / 1e6:.0f} GB/s)  both concurrently {tb:.3f} ms ({(chain_b + fan_b) / tb / 1e6:.0f} GB/s)",
          flush=True)
