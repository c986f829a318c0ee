"""Step-by-step check of the multi-GPU peer primitives, with a host watchdog.

    torchrun --nproc-per-node 2 tools/peer_probe.py
Each step prints ok/FAIL; a stream that does not finish within the deadline is
reported and the process exits (no hang).
"""
import ctypes
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_17766_b200 import _lib as L  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
lib = L.lib()


def log(*a):
    print(f"[rank {rank}]", *a, flush=True)


def wait_stream(s, what, deadline=20.0):
    t = time.time()
    while not s.query():
        if time.time() - t > deadline:
            log(f"FAIL: {what}: stream did not finish in {deadline}s")
            sys.stdout.flush()
            os._exit(3)
        time.sleep(0.01)
    log(f"ok: {what} ({time.time() - t:.3f}s)")


base = ctypes.c_void_p()
h = (ctypes.c_uint8 * 64)()
L.check(lib.bfly_ipc_alloc(1 << 20, ctypes.byref(base), h))
handles = [None] * world
dist.all_gather_object(handles, bytes(h))
peer = {}
for r, hh in enumerate(handles):
    if r == rank:
        continue
    p = ctypes.c_void_p()
    rc = lib.bfly_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(hh), ctypes.byref(p))
    log("ipc_open", r, "rc", rc, lib.bfly_last_error().decode())
    peer[r] = p.value
dist.barrier()
other = 1 - rank
s = torch.cuda.current_stream()

# 1. flag write into the peer region, wait locally
flag_local = base.value + 4096
flag_peer = peer[other] + 4096
if rank == 0:
    L.check(lib.bfly_stream_write_value(flag_peer, 7, s.cuda_stream))
    wait_stream(s, "write_value to peer")
else:
    L.check(lib.bfly_stream_wait_value(flag_local, 7, s.cuda_stream))
    wait_stream(s, "wait_value on local flag written by peer")
dist.barrier()

# 2. kernel stores into the peer region (fanout), then a flag
src = torch.arange(1024, dtype=torch.float32, device=dev) + 1000 * rank
tab = torch.tensor([peer[other] + 8192], dtype=torch.int64, device=dev)
L.check(lib.bfly_fanout(src.data_ptr(), tab.data_ptr(), 1, 4096, s.cuda_stream))
L.check(lib.bfly_stream_write_value(peer[other] + 4100, 11, s.cuda_stream))
L.check(lib.bfly_stream_wait_value(base.value + 4100, 11, s.cuda_stream))
wait_stream(s, "peer store + flag round trip")
got = torch.empty(1024, dtype=torch.float32, device=dev)
L.check(lib.bfly_fanout(base.value + 8192, torch.tensor([got.data_ptr()], dtype=torch.int64, device=dev).data_ptr(),
                        1, 4096, s.cuda_stream))
torch.cuda.synchronize()
want = torch.arange(1024, dtype=torch.float32, device=dev) + 1000 * other
log("peer data correct:", bool(torch.equal(got, want)))

# 3. chain step writing fp64 sums into the peer
reps = [torch.rand(1 << 16, device=dev) for _ in range(3)]
rt = torch.tensor([t.data_ptr() for t in reps], dtype=torch.int64, device=dev)
L.check(lib.bfly_chain_step(rt.data_ptr(), 3, 0, None, peer[other] + 65536, 0, 1 << 16, s.cuda_stream))
L.check(lib.bfly_stream_write_value(peer[other] + 4104, 13, s.cuda_stream))
L.check(lib.bfly_stream_wait_value(base.value + 4104, 13, s.cuda_stream))
wait_stream(s, "chain into peer + flag")
dist.barrier()
dist.destroy_process_group()
log("done")
