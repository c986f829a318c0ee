"""Diagnose a single-device loopback ring round step by step (events polled with a
deadline): which of launch / check / broadcast completes."""
import faulthandler
import os
import sys
import time

faulthandler.dump_traceback_later(45, exit=True)

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, ROOT + "/oracle", ROOT + "/tests"]
import torch  # noqa: E402

from _multigpu_cases import fuzz_case  # noqa: E402
from paper_2507_17766_b200 import multigpu as mg  # noqa: E402
from paper_2507_17766_b200.device import DevicePlan  # noqa: E402

dev = torch.device("cuda", 0)
world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cases = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
VERBOSE = len(cases) == 1


def wait(ev, what, rank, deadline=30):
    t = time.time()
    while not ev.query():
        if time.time() - t > deadline:
            print(f"[{rank}] STUCK at {what}", flush=True)
            return False
        time.sleep(0.01)
    if VERBOSE:
        print(f"[{rank}] done {what} in {time.time() - t:.3f}s", flush=True)
    return True


def body(rank, comm):
    counts, data = c["counts"], c["data"]
    kind = c["kind"]
    off = sum(counts[:rank])
    if kind == "bf16":
        local = [torch.from_numpy(data[off + i].view(np.int16).copy()).to(dev).view(torch.bfloat16)
                 for i in range(counts[rank])]
    else:
        local = [torch.from_numpy(data[off + i].copy()).to(dev) for i in range(counts[rank])]
    from paper_2507_17766_b200.device import Corruption
    dcorr = {m: Corruption.add(a) for m, (_, a) in c["corr"].items()}
    plan = DevicePlan(c["n"], c["P"], c["seed"], redundancy=c["r"], device=dev)
    job = mg.ShardedButterflyMerge(local, plan, failures=c["fails"], corruptions=dcorr, chunk=1 << 18,
                                   want_merged=True, comm=comm, debug=int(os.environ.get("PROBE_DEBUG", "0")))
    print(f"[{rank}] fused={job.fused} lanes={getattr(job, 'lanes', None)}", flush=True)
    cur = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event()
    e0.record(cur)
    ok = wait(e0, "setup", rank)
    # one full round, every transport step polled
    real_bcast, real_launch = comm.broadcast, comm.launch_fused

    def bcast(t, src):
        real_bcast(t, src)
        e = torch.cuda.Event()
        e.record(torch.cuda.current_stream(dev))
        wait(e, f"broadcast {tuple(t.shape)} from {src}", rank)

    def launch(d, dv):
        real_launch(d, dv)
        e = torch.cuda.Event()
        e.record(torch.cuda.current_stream(dev))
        wait(e, "launch_fused", rank)

    comm.broadcast, comm.launch_fused = bcast, launch
    if job.is_last:
        real_run = job.job.run

        def run(*a, **k):
            out = real_run(*a, **k)
            e = torch.cuda.Event()
            e.record(torch.cuda.current_stream(dev))
            wait(e, f"job.run{a}", rank)
            return out

        job.job.run = run
    job.run()
    e2 = torch.cuda.Event()
    e2.record(cur)
    ok = wait(e2, "round", rank) and ok
    for _ in range(c["rounds"] - 1):
        job.run()
        e2 = torch.cuda.Event()
        e2.record(cur)
        ok = wait(e2, "round", rank) and ok
    job.close()
    return ok


import numpy as np  # noqa: E402

for case in cases:
    c = fuzz_case(case, world)
    print("case", case, c["counts"], c["kind"], c["P"], c["r"], c["fails"], c["corr"], flush=True)
    print(mg.run_loopback(world, body, device=dev, timeout=60), flush=True)
