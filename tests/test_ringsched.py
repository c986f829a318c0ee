"""CPU simulation of the multi-GPU merge schedule (paper_2507_17766_b200/ringsched.py).

Every rank's two streams execute their op lists under random interleavings:
waits block until the flag reaches the value (wrap-safe >=), kernels move real
numbers with numpy exactly as the CUDA kernels do (fp64 running sums in miner
order, divide on the last rank, fp32 scatter-back, relay).  The simulation
asserts that no stream ever deadlocks, that every consumer reads the chunk it
expects, that no producer overwrites an inbox slot before it was consumed, that
no rank's replicas are overwritten before its chain read them, and that every
replica ends bit-identical to the sequential fp64 mean (the reference order).
"""

import random

import numpy as np
import pytest

from paper_2507_17766_b200 import ringsched as rs


class Rank:
    def __init__(self, g, replicas, NB, C):
        self.g = g
        self.rep = [r.copy() for r in replicas]
        self.acc_in = [None] * NB  # (tag, array)
        self.acc_consumed = [True] * NB
        self.fin_in = [None] * NB
        self.fin_consumed = [True] * NB
        self.flags = {f: [0] * NB for f in rs.FLAGS}
        self.final_written = set()


def simulate(G, counts, P, C, NB, rounds, failures=(), seed=0, start_round=0, late=False):
    rng = random.Random(seed)
    n = sum(counts)
    data_rng = np.random.default_rng(seed)
    allrep = (data_rng.uniform(-1, 1, (n, P)) * 10.0 ** data_rng.integers(-6, 6, (n, 1))).astype(np.float32)
    offs = [sum(counts[:g]) for g in range(G)]
    ranks = [Rank(g, [allrep[offs[g] + i] for i in range(counts[g])], NB, C) for g in range(G)]
    alive = [m for m in range(n) if m not in failures]
    K = -(-P // C)
    Z = G - 1
    if start_round:  # flags as left by the rounds before: each slot's last occupant
        start = start_round * K
        for rk in ranks:
            for f in rs.FLAGS:
                for slot_i in range(NB):
                    last = max(i for i in range(start - NB, start) if i % NB == slot_i)
                    rk.flags[f][slot_i] = (last + 1) & 0xFFFFFFFF

    def bounds(k):
        return k * C, min((k + 1) * C, P)

    def local_alive(g):
        return [ranks[g].rep[m - offs[g]] for m in alive if offs[g] <= m < offs[g] + counts[g]]

    for r in range(start_round, start_round + rounds):
        current = [np.array([ranks[g].rep[i] for i in range(counts[g])]) for g in range(G)]
        everyone = np.concatenate(current)
        acc = np.zeros(P)
        for m in alive:
            acc = acc + everyone[m].astype(np.float64)
        want = (acc / len(alive)).astype(np.float32)
        queues = {}
        for g in range(G):
            ops = rs.round_ops(g, G, K, NB, r, late)
            for st in ("C", "R", "F"):
                queues[(g, st)] = [o for o in ops if o[1] == st]
            ranks[g].final_written = set()
        while any(queues.values()):
            runnable = []
            for key, q in queues.items():
                if not q:
                    continue
                op = q[0]
                if op[0] == "wait":
                    _, _, flag, s, v = op
                    if not rs.geq(ranks[key[0]].flags[flag][s], v):
                        continue
                runnable.append(key)
            assert runnable, f"deadlock: heads {[(k, q[0]) for k, q in queues.items() if q]}"
            key = rng.choice(runnable)
            g = key[0]
            op = queues[key].pop(0)
            me = ranks[g]
            kind = op[0]
            if kind == "wait":
                continue
            if kind == "write":
                _, _, peer, flag, s, v = op
                ranks[peer].flags[flag][s] = v
            elif kind == "chain":
                _, _, k, s, dst = op
                b, e = bounds(k)
                assert k not in me.final_written, "chain read a replica chunk already overwritten"
                if g > 0:
                    tag, a = me.acc_in[s]
                    assert tag == (r, k) and not me.acc_consumed[s], "chain read the wrong chunk"
                    a = a.copy()
                    me.acc_consumed[s] = True
                else:
                    a = np.zeros(e - b)
                for x in local_alive(g):
                    a = a + x[b:e].astype(np.float64)
                assert ranks[dst].acc_consumed[s], "acc slot overwritten before it was consumed"
                ranks[dst].acc_in[s] = ((r, k), a)
                ranks[dst].acc_consumed[s] = False
            elif kind == "reduce":
                _, _, k, s, fin_rank = op
                b, e = bounds(k)
                tag, a = me.acc_in[s]
                assert tag == (r, k) and not me.acc_consumed[s]
                a = a.copy()
                me.acc_consumed[s] = True
                for x in local_alive(g):
                    a = a + x[b:e].astype(np.float64)
                mean32 = (a / len(alive)).astype(np.float32)
                for x in me.rep:
                    x[b:e] = mean32
                me.final_written.add(k)
                assert ranks[fin_rank].fin_consumed[s], "fin slot overwritten before it was consumed"
                # with late shards the chunk is incomplete until "finish" runs
                ranks[fin_rank].fin_in[s] = ((r, k, "partial" if late else "final"), mean32.copy())
                ranks[fin_rank].fin_consumed[s] = False
            elif kind == "finish":
                _, _, k, s, fin_rank = op
                tag, f = ranks[fin_rank].fin_in[s]
                assert tag == (r, k, "partial"), "finish saw the wrong chunk"
                ranks[fin_rank].fin_in[s] = ((r, k, "final"), f)
            elif kind == "fanout":
                _, _, k, s, fwd = op
                b, e = bounds(k)
                tag, f = me.fin_in[s]
                assert tag[:2] == (r, k) and not me.fin_consumed[s], "fanout read the wrong chunk"
                assert tag[2] == "final", "fanout relayed a chunk whose late shards were not finished"
                for x in me.rep:
                    x[b:e] = f
                me.final_written.add(k)
                if fwd is not None:
                    assert ranks[fwd].fin_consumed[s]
                    ranks[fwd].fin_in[s] = (tag, f.copy())
                    ranks[fwd].fin_consumed[s] = False
                me.fin_consumed[s] = True
        for g in range(G):
            for x in ranks[g].rep:
                assert np.array_equal(x, want), f"rank {g} round {r}: wrong merged values"


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("K_chunks,NB", [(1, 2), (2, 2), (5, 3), (17, 3), (9, 2)])
@pytest.mark.parametrize("late", [False, True])
def test_schedule_completes_and_is_exact(G, K_chunks, NB, late):
    counts = [2 + (g % 3) for g in range(G)]
    C = 64
    P = C * K_chunks - (7 if K_chunks > 1 else 0)
    for seed in range(3):
        simulate(G, counts, P, C, NB, rounds=2, failures=(1,), seed=seed, late=late)


def test_flag_wraparound():
    # rounds near 2^32 / K: flag values wrap, waits must stay correct
    K = 4
    r0 = (0xFFFFFFFF // K) - 1
    simulate(3, [2, 1, 2], 4 * 32, 32, 2, rounds=3, seed=5, start_round=r0)
    simulate(3, [2, 1, 2], 4 * 32, 32, 2, rounds=3, seed=6, start_round=r0, late=True)


def test_waits_reference_earlier_work_only():
    # every wait on rank g is satisfied by a write another rank issues for the same or an earlier chunk
    for G in (2, 4, 8):
        for g in range(G):
            for op in rs.round_ops(g, G, 6, 3, 0):
                if op[0] == "wait":
                    assert op[4] <= 6


def test_rejects_single_rank_and_one_slot():
    with pytest.raises(ValueError):
        rs.round_ops(0, 1, 4, 2, 0)
    with pytest.raises(ValueError):
        rs.round_ops(0, 2, 4, 1, 0)


@pytest.mark.parametrize("G", [2, 3, 5, 8])
@pytest.mark.parametrize("K,NB,r", [(1, 2, 0), (7, 3, 0), (7, 3, 5), (13, 2, 2), (4, 3, (1 << 32) // 4 - 1)])
@pytest.mark.parametrize("late", [False, True])
def test_native_executor_issues_the_same_ops(G, K, NB, r, late):
    """bfly_ring_round (C++) generates its ops with bfly_ring_ops' generator; it must
    equal ringsched.round_ops, the schedule the simulator above verifies."""
    import ctypes

    from paper_2507_17766_b200 import _lib

    kinds = {"wait": 0, "write": 1, "chain": 2, "reduce": 3, "fanout": 4, "finish": 5}
    streams = {"C": 0, "R": 1, "F": 2}
    for g in range(G):
        want = []
        for op in rs.round_ops(g, G, K, NB, r, late):
            kind, st = op[0], op[1]
            if kind == "wait":
                row = (kinds[kind], streams[st], g, rs.FLAGS.index(op[2]), op[3], -1, op[4])
            elif kind == "write":
                row = (kinds[kind], streams[st], op[2], rs.FLAGS.index(op[3]), op[4], -1, op[5])
            else:
                peer = -1 if op[4] is None else op[4]
                row = (kinds[kind], streams[st], peer, -1, op[3], op[2], 0)
            want.append(row)
        buf = (ctypes.c_int32 * (7 * 16 * K))()
        n = _lib.lib().bfly_ring_ops(g, G, K, NB, r & 0xFFFFFFFF, int(late), buf, 16 * K)
        got = [tuple(buf[7 * i:7 * i + 7]) for i in range(n)]
        got = [(a, b, c, d, e, (f if a >= 2 else -1), (h & 0xFFFFFFFF if a < 2 else 0)) for a, b, c, d, e, f, h in got]
        want = [(a, b, c, d, e, f, h & 0xFFFFFFFF) for a, b, c, d, e, f, h in want]
        assert got == want, (g, G, K, NB, r)


@pytest.mark.parametrize("P,chunk", [(10**9, 1 << 24), (4096 * 8 + 5, 8192), (6_000_007, 1 << 20), (1 << 20, 1 << 20),
                                     (50_000_000, 1 << 22), (3, 4096)])
def test_chunk_edges_cover_the_payload(P, chunk):
    """multigpu.chunk_edges: contiguous cover of [0, P), every chunk fits an inbox slot,
    inner edges on 4096-element (k_reduce tile) boundaries, ramps mirror each other."""
    from paper_2507_17766_b200.multigpu import chunk_edges

    for ramp in (False, True):
        e = chunk_edges(P, chunk, ramp=ramp)
        sizes = [b - a for a, b in zip(e, e[1:])]
        assert e[0] == 0 and e[-1] == P and all(0 < x <= chunk for x in sizes)
        assert all(x % 4096 == 0 for x in e[1:-1])
        if ramp and sizes[0] < chunk:
            head = [x for x in sizes[:4] if x < chunk]
            assert sizes[-len(head):][::-1][1:] == head[1:]  # mirrored (the last one absorbs the tail)
