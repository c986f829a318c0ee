"""Host-side schedule of the multi-GPU merge (paper_2507_17766_b200/multigpu.py)
over gloo on CPU, world sizes 2 and 3.

The per-rank compute is replaced by a CPU stand-in with the same contract as
the CUDA ops (fp64 running sums continued across ranks, last rank divides and
scatters back); the chunked send/recv chain, the result broadcast and the
fan-out run for real.  Every rank must end with the bit-exact sequential mean
(the reference's order, butterfly.py:156-158) of all alive miners' replicas.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class CpuJob:
    def __init__(self, replicas, plan, *, failures, corruptions, fallback, fallback_src, scatter_back, want_merged,
                 tolerance, n_div):
        self.reps = replicas
        self.resident = [m for m, t in enumerate(replicas) if t is not None]
        self.local_alive = [m for m in self.resident if m not in failures]
        self.n_div = n_div
        P = int(next(t for t in replicas if t is not None).numel())
        n, S = plan.n_miners, plan.n_shards
        self.mean = torch.empty(P, dtype=torch.float64)
        self.status = torch.zeros(S, dtype=torch.uint8)
        self.flagged = torch.zeros(n, dtype=torch.uint8)
        self.source = torch.zeros(S, dtype=torch.int32)
        self.entries = torch.full((n, n), float("nan"), dtype=torch.float64)
        self.merged = torch.empty(P, dtype=torch.float64) if want_merged else None
        self.started = False

    def reduce_range(self, b, e, acc_in=None):
        if b == 0:
            self.started = True
        acc = acc_in.clone() if acc_in is not None else torch.zeros(e - b, dtype=torch.float64)
        for m in self.local_alive:
            acc = acc + self.reps[m][b:e].double()
        self.mean[b:e] = acc / self.n_div
        for m in self.resident:  # scatter-back of the chunk, like k_reduce
            self.reps[m][b:e] = self.mean[b:e].float()

    def run(self, phase):
        assert self.started
        if self.merged is not None:
            self.merged.copy_(self.mean)
        self.entries.fill_(1.0)


class CpuOps:
    def chain(self, src, acc_in, acc_out, b, e):
        acc = acc_in.clone() if acc_in is not None else torch.zeros(e - b, dtype=torch.float64)
        for x in src:
            acc = acc + x[b:e].double()
        acc_out.copy_(acc)

    def fanout(self, src, dsts):
        for d in dsts:
            d.copy_(src)

    def gather_ranges(self, full, packed, ranges):
        for lo, hi, off in ranges.tolist():
            packed[off:off + hi - lo] = full[lo:hi]

    def scatter_ranges(self, packed, dsts, ranges):
        for lo, hi, off in ranges.tolist():
            for d in dsts:
                d[lo:hi] = packed[off:off + hi - lo]

    def make_job(self, replicas, plan, **kw):
        return CpuJob(replicas, plan, **kw)


class Plan:
    def __init__(self, n, P):
        import oracle as orc

        self.n_miners, self.n_shards, self.redundancy, self.payload_len = n, n * (n - 1) // 2, 2, P
        self.assign = orc.plan(n, P, 11)[0]


def _all_miners(n, P):
    rng = np.random.default_rng(42)
    return (rng.uniform(-1, 1, (n, P)) * 10.0 ** rng.integers(-5, 5, (n, 1))).astype(np.float32)


def _worker(rank, world, port, counts, P, failures, chunk, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_17766_b200.multigpu import ShardedButterflyMerge

        n = sum(counts)
        data = _all_miners(n, P)
        off = sum(counts[:rank])
        local = [torch.from_numpy(data[off + i].copy()) for i in range(counts[rank])]
        job = ShardedButterflyMerge(local, Plan(n, P), failures=failures, chunk=chunk, ops=CpuOps(),
                                    want_merged=True)
        for _ in range(2):  # a second round starts from identical replicas (a fixed point)
            job.run()
        alive = [m for m in range(n) if m not in failures]
        acc = np.zeros(P)
        for m in alive:
            acc = acc + data[m].astype(np.float64)
        first = (acc / len(alive)).astype(np.float32).astype(np.float64)
        acc2 = np.zeros(P)
        for _ in alive:
            acc2 = acc2 + first
        want = (acc2 / len(alive))
        ok = all(np.array_equal(t.numpy(), want.astype(np.float32)) for t in local)
        ok = ok and np.array_equal(job.merged.numpy(), want)
        ok = ok and bool(torch.all(job.entries == 1.0))
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("counts,P,failures,chunk", [
    ((3, 2), 20_000, (), 4096),
    ((2, 2, 3), 12_289, (1, 4), 4096),
    ((1, 4), 8192 * 3, (0,), 8192),
])
def test_sharded_chain_schedule_gloo(counts, P, failures, chunk):
    world = len(counts)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), counts, P, failures, chunk, out), nprocs=world, join=True)
    assert [out[r] for r in range(world)] == [1] * world
