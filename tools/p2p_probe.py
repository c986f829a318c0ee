"""NVLink transfer probes (2+ GPUs).

    python tools/p2p_probe.py ce                 # one process: copy-engine peer copies
    torchrun --nproc-per-node 2 tools/p2p_probe.py nccl   # NCCL send/recv, alone and under load
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402


def ce():
    n = torch.cuda.device_count()
    for size_mb in (64, 256, 1024):
        a = torch.empty(size_mb << 20, dtype=torch.uint8, device="cuda:0")
        b = torch.empty(size_mb << 20, dtype=torch.uint8, device="cuda:1")
        for _ in range(3):
            b.copy_(a)
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        t = time.perf_counter()
        for _ in range(10):
            b.copy_(a)
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        dt = (time.perf_counter() - t) / 10
        print(f"CE peer copy {size_mb} MB: {size_mb / 1024 / dt:.1f} GiB/s", flush=True)
    print("peer access 0->1:", torch.cuda.can_device_access_peer(0, 1), "gpus", n)


def nccl():
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2507_17766_b200 import _lib as L
    from bench import make_replicas

    reps = make_replicas(16, 1 << 26, "fp32", dev)
    out = torch.empty(1 << 26, dtype=torch.float64, device=dev)
    from paper_2507_17766_b200.multigpu import CudaOps

    ops = CudaOps()
    for mb in (32, 128, 512):
        x = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
        for load in (False, True):
            for cap in ((0, 132) if load else (0,)):
                L.lib().bfly_set_max_ctas(cap)
                dist.barrier(); torch.cuda.synchronize()
                t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
                t0.record()
                for _ in range(10):
                    if load:
                        ops.chain(reps, None, out, 0, 1 << 26)
                    w = dist.batch_isend_irecv([dist.P2POp(dist.isend if rank == 0 else dist.irecv, x, 1 - rank)])
                    for ww in w:
                        ww.wait()
                t1.record(); torch.cuda.synchronize()
                ms = t0.elapsed_time(t1) / 10
                if rank == 0:
                    print(f"NCCL send {mb} MB load={load} cap={cap}: {ms:.3f} ms/iter -> {mb / 1024 / (ms / 1e3):.1f} GiB/s",
                          flush=True)
        L.lib().bfly_set_max_ctas(0)
    # the compute alone
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(10):
        ops.chain(reps, None, out, 0, 1 << 26)
    t1.record(); torch.cuda.synchronize()
    if rank == 0:
        print(f"chain kernel alone (16 x 256 MB): {t0.elapsed_time(t1) / 10:.3f} ms", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    {"ce": ce, "nccl": nccl}[sys.argv[1]]()
