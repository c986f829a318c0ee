"""Kernel-level cost of storing into a peer GPU's memory (2 GPUs, one process per GPU).

    torchrun --nproc-per-node 2 tools/peer_bw.py
Times bfly_chain_step (16 replicas x 16M fp32 -> 16M fp64 sums) writing locally vs into
the other GPU, and bfly_fanout (16M fp32 into 16 replicas) with and without an extra
peer destination, while the other GPU runs the same kernels.
"""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17766_b200 import _lib as L  # noqa: E402

rank = int(os.environ["RANK"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
lib = L.lib()
C = 1 << 24
reps = [torch.rand(C, device=dev) for _ in range(16)]
tab = torch.tensor([t.data_ptr() for t in reps], dtype=torch.int64, device=dev)
base = ctypes.c_void_p()
h = (ctypes.c_uint8 * 64)()
L.check(lib.bfly_ipc_alloc(C * 8 * 2, ctypes.byref(base), h))
hs = [None, None]
dist.all_gather_object(hs, bytes(h))
p = ctypes.c_void_p()
L.check(lib.bfly_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(hs[1 - rank]), ctypes.byref(p)))
peer = p.value
local_out = torch.empty(C, dtype=torch.float64, device=dev)
fin = torch.rand(C, device=dev)
s = torch.cuda.current_stream().cuda_stream


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


res = {}
res["chain->local"] = timeit(lambda: lib.bfly_chain_step(tab.data_ptr(), 16, 0, None, local_out.data_ptr(), 0, C, s))
res["chain->peer"] = timeit(lambda: lib.bfly_chain_step(tab.data_ptr(), 16, 0, None, peer, 0, C, s))
res["chain(acc_in)->peer"] = timeit(lambda: lib.bfly_chain_step(tab.data_ptr(), 16, 0, local_out.data_ptr(), peer,
                                                                0, C, s))
lib.bfly_set_chain_bulk(1)
res["bulk chain->local"] = timeit(lambda: lib.bfly_chain_step(tab.data_ptr(), 16, 0, None, local_out.data_ptr(), 0, C, s))
res["bulk chain->peer"] = timeit(lambda: lib.bfly_chain_step(tab.data_ptr(), 16, 0, None, peer, 0, C, s))
res["bulk chain(acc_in)->peer"] = timeit(lambda: lib.bfly_chain_step(tab.data_ptr(), 16, 0, local_out.data_ptr(),
                                                                     peer, 0, C, s))
lib.bfly_set_chain_bulk(0)
ft = torch.tensor([t.data_ptr() for t in reps], dtype=torch.int64, device=dev)
ftp = torch.tensor([t.data_ptr() for t in reps] + [peer], dtype=torch.int64, device=dev)
res["fanout 16 local"] = timeit(lambda: lib.bfly_fanout(fin.data_ptr(), ft.data_ptr(), 16, C * 4, s))
res["fanout 16 local + peer"] = timeit(lambda: lib.bfly_fanout(fin.data_ptr(), ftp.data_ptr(), 17, C * 4, s))
if rank == 0:
    for k, v in res.items():
        print(f"{k:28s} {v:.3f} ms", flush=True)

# pipeline: chain into a local slot, copy-engine push to the peer on a side stream
xs = torch.cuda.Stream(device=dev)
outs = [torch.empty(C, dtype=torch.float64, device=dev) for _ in range(2)]
ev_chain = [torch.cuda.Event() for _ in range(2)]
ev_copy = [torch.cuda.Event() for _ in range(2)]
for e in ev_copy:
    e.record()
cur = torch.cuda.current_stream()


def pipeline(n=20):
    for k in range(n):
        j = k % 2
        cur.wait_event(ev_copy[j])
        lib.bfly_chain_step(tab.data_ptr(), 16, 0, None, outs[j].data_ptr(), 0, C, cur.cuda_stream)
        ev_chain[j].record(cur)
        xs.wait_event(ev_chain[j])
        lib_rt.cudaMemcpyAsync(ctypes.c_void_p(peer + (k % 2) * 0), ctypes.c_void_p(outs[j].data_ptr()),
                               ctypes.c_size_t(C * 8), 3, ctypes.c_void_p(xs.cuda_stream))
        ev_copy[j].record(xs)
    cur.wait_stream(xs)


import glob  # noqa: E402
rt = glob.glob(str(Path(torch.__file__).parent / "lib" / "libcudart*.so*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*")
lib_rt = ctypes.CDLL(rt[0])
dist.barrier()
torch.cuda.synchronize()
for _ in range(2):
    pipeline(4)
torch.cuda.synchronize()
dist.barrier()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
pipeline(20)
b.record()
torch.cuda.synchronize()
if rank == 0:
    print(f"{'chain->local + CE push':28s} {a.elapsed_time(b) / 20:.3f} ms per chunk", flush=True)
dist.barrier()
dist.destroy_process_group()
