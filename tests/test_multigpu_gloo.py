"""Host-side pieces of the multi-GPU merge over gloo on CPU (world sizes 2, 3).

The data path (peer-memory chain + relay) is verified by the schedule simulator
(tests/test_ringsched.py) and, on GPUs, by tests/test_multigpu_gpu.py.  Here the
collective plumbing that surrounds it runs for real on CPU tensors: the
late-shard ranges and their pack/broadcast/scatter, and the packed broadcast
of the per-shard results from the last rank.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as orc

        from paper_2507_17766_b200.multigpu import pack_results, special_ranges, unpack_results

        n, P, last = 9, 4000, world - 1
        assign, bounds = orc.plan(n, P, 3)
        failures, corrupted = {1, 4}, {6}
        runs = special_ranges(assign, P, failures, corrupted)
        # brute force: a shard is late iff no survivor, or a corrupted survivor
        late = np.zeros(P, dtype=bool)
        for s, mem in enumerate(assign):
            surv = [m for m in mem if m not in failures]
            if not surv or any(m in corrupted for m in surv):
                late[bounds[s]:bounds[s + 1]] = True
        mask = np.zeros(P, dtype=bool)
        for lo, hi in runs:
            assert not mask[lo:hi].any()
            mask[lo:hi] = True
        ok = np.array_equal(mask, late) and all(runs[i][1] < runs[i + 1][0] for i in range(len(runs) - 1))

        # packed late-shard values travel from the last rank and land in every replica
        rng = np.random.default_rng(rank)
        local = [torch.from_numpy(rng.uniform(-1, 1, P).astype(np.float32)) for _ in range(2)]
        final = torch.from_numpy(np.random.default_rng(99).uniform(-1, 1, P).astype(np.float32))
        packed = (torch.cat([final[lo:hi] for lo, hi in runs]) if rank == last
                  else torch.empty(int(mask.sum()), dtype=torch.float32))
        dist.broadcast(packed, src=last)
        off = 0
        for lo, hi in runs:
            for t in local:
                t[lo:hi] = packed[off:off + hi - lo]
            off += hi - lo
        m = torch.from_numpy(mask)
        ok = ok and all(torch.equal(t[m], final[m]) for t in local)

        # per-shard results: pack on the last rank, broadcast, unpack everywhere
        S = len(assign)
        g = torch.Generator().manual_seed(5)
        want = (torch.rand((n, n), generator=g, dtype=torch.float64),
                torch.randint(-1, n, (S,), generator=g, dtype=torch.int32),
                torch.randint(0, 3, (S,), generator=g, dtype=torch.uint8),
                torch.randint(0, 2, (n,), generator=g, dtype=torch.uint8))
        buf = torch.empty(8 * n * n + 4 * S + S + n, dtype=torch.uint8)
        if rank == last:
            pack_results(*want, buf)
        dist.broadcast(buf, src=last)
        got = (torch.empty((n, n), dtype=torch.float64), torch.empty(S, dtype=torch.int32),
               torch.empty(S, dtype=torch.uint8), torch.empty(n, dtype=torch.uint8))
        unpack_results(buf, *got)
        ok = ok and all(torch.equal(a, b) for a, b in zip(got, want))
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_multigpu_host_collectives_gloo(world):
    out = mp.get_context("spawn").Manager().dict()  # no fork of a multi-threaded process
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert [out[r] for r in range(world)] == [1] * world


def test_loopback_comm_exchanges_between_threads():
    """The single-device loopback transport (multigpu.LoopbackComm): every rank's thread
    sees every rank's object in rank order; min-reductions agree; a failing rank breaks
    the others' barriers instead of hanging them."""
    import threading

    from paper_2507_17766_b200.multigpu import LoopbackComm, LoopbackGroup

    world = 4
    group = LoopbackGroup(world, timeout=30)
    out = [None] * world

    def body(rank):
        comm = LoopbackComm(group, rank)
        got = comm.all_gather_object(("rank", rank))
        low = comm.all_reduce_min(10 - rank, None)
        comm.barrier()
        again = comm.all_gather_object(rank * rank)
        out[rank] = (got, low, again)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for rank in range(world):
        got, low, again = out[rank]
        assert got == [("rank", r) for r in range(world)]
        assert low == 10 - (world - 1)
        assert again == [r * r for r in range(world)]

    group = LoopbackGroup(2, timeout=30)
    errs = [None, None]

    def bad(rank):
        comm = LoopbackComm(group, rank)
        try:
            if rank == 1:
                group.barrier.abort()  # what run_loopback does when a rank raises
                return
            comm.barrier()
        except threading.BrokenBarrierError as e:
            errs[rank] = e

    ts = [threading.Thread(target=bad, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    assert isinstance(errs[0], threading.BrokenBarrierError)
