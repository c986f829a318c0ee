"""Per-rank operation lists of one multi-GPU merge round (pure host logic).

The multi-GPU merge (multigpu.py) moves data by storing straight into the
neighbouring GPU's inbox from inside the kernels (peer memory over NVLink) and
orders GPUs with 32-bit flags written and awaited by the streams themselves.
This module decides *what* each rank issues, in which stream and order; the
CUDA executor (multigpu.py) and the CPU simulator (tests/test_ringsched.py)
both consume these lists, so the schedule is verified without a GPU.

Ranks g = 0..Z (Z = G-1).  Chunk k of round r is the (r*K + k)-th chunk the
ring carries; it uses inbox slot s = (r*K + k) % NB and flag value
v = r*K + k + 1 (monotonic across rounds, so flags never need resetting and the
previous occupant of slot s always carries v - NB; waits use the wrap-safe
">=" of cuStreamWaitValue32).

chain (stream "C"), rank g < Z:
    [g>0] wait acc_ready[s] >= v            running sums of chunk k arrived from g-1
    [v>NB] wait acc_free[s] >= v-NB         g+1 has consumed the previous chunk in its slot s
    chain k -> g+1.acc_in[s]                fp64 sum continued over my replicas, stored remotely
    write g+1.acc_ready[s] = v
    [g>0] write g-1.acc_free[s] = v         my slot s may be refilled
last rank Z (stream "C"):
    wait acc_ready[s] >= v ; [v>NB] wait fin_free[s] >= v-NB
    reduce k -> own replicas + 0.fin_in[s]  divide, scatter back, push the final chunk
    write 0.fin_ready[s] = v ; write Z-1.acc_free[s] = v
  with late shards (corrupted / lost) the chunk's shards are decided before the
  final chunk is released, on stream "F" so the next reduce is not held up:
    C: ... reduce k ; write reduced[s] = v (own) ; write Z-1.acc_free[s] = v
    F: wait reduced[s] >= v ; finish k ; write 0.fin_ready[s] = v
relay (stream "R"), ranks 0..Z-1, ring Z -> 0 -> 1 -> ... -> Z-1:
    wait fin_ready[s] >= v ; [succ and v>NB] wait fin_free[s] >= v-NB
    fanout k: fin_in[s] -> my replicas (+ succ.fin_in[s])
    [succ] write succ.fin_ready[s] = v ; write pred.fin_free[s] = v

Every wait names an event of the same or an earlier chunk further up the chain
or the ring, so the lists cannot deadlock (checked exhaustively by the tests).

The chain kernel writes the running sums into the next GPU's inbox through TMA
bulk stores from shared memory: measured on B200 (16 replicas x 16M elements),
plain SM stores into peer memory stretched the kernel from 0.19 to 0.32 ms, a
local write + copy-engine push pipeline cost 0.23 ms per chunk, the bulk stores
0.21 ms with no extra HBM traffic (tools/peer_bw.py, profiles/).
"""

from __future__ import annotations

FLAGS = ("acc_ready", "acc_free", "fin_ready", "fin_free", "reduced")


def relay_pred(g: int, Z: int) -> int:
    return Z if g == 0 else g - 1


def relay_succ(g: int, Z: int):
    return g + 1 if g + 1 < Z else None


def value(round_index: int, K: int, k: int) -> int:
    return (round_index * K + k + 1) & 0xFFFFFFFF


def slot(round_index: int, K: int, k: int, NB: int) -> int:
    return (round_index * K + k) % NB


def chunk_ops(g: int, G: int, K: int, NB: int, round_index: int, k: int, late: bool = False) -> list:
    """Ops of rank g for chunk k of one round (stream "C" ops, then stream "R" ops):
    ("wait", stream, flag, slot, value)         wait on a flag in MY region
    ("write", stream, peer, flag, slot, value)   write a flag in peer's region
    ("chain", stream, k, slot, dst_rank)
    ("reduce", stream, k, slot, fin_rank)
    ("finish", stream, k, slot, fin_rank)      late shards of chunk k (``late`` only)
    ("fanout", stream, k, slot, fwd_rank|None)
    """
    if G < 2:
        raise ValueError("the ring schedule needs at least 2 ranks")
    if NB < 2:
        raise ValueError("need at least 2 inbox slots")
    Z = G - 1
    s = slot(round_index, K, k, NB)
    v = value(round_index, K, k)
    first_use = round_index * K + k < NB  # slot never filled before
    prev = (v - NB) & 0xFFFFFFFF
    ops = []
    if g < Z:
        if g > 0:
            ops.append(("wait", "C", "acc_ready", s, v))
        if not first_use:
            ops.append(("wait", "C", "acc_free", s, prev))
        ops.append(("chain", "C", k, s, g + 1))
        ops.append(("write", "C", g + 1, "acc_ready", s, v))
        if g > 0:
            ops.append(("write", "C", g - 1, "acc_free", s, v))
        succ, pred = relay_succ(g, Z), relay_pred(g, Z)
        ops.append(("wait", "R", "fin_ready", s, v))
        if succ is not None and not first_use:
            ops.append(("wait", "R", "fin_free", s, prev))
        ops.append(("fanout", "R", k, s, succ))
        if succ is not None:
            ops.append(("write", "R", succ, "fin_ready", s, v))
        ops.append(("write", "R", pred, "fin_free", s, v))
    else:
        ops.append(("wait", "C", "acc_ready", s, v))
        if not first_use:
            ops.append(("wait", "C", "fin_free", s, prev))
        ops.append(("reduce", "C", k, s, 0))
        if late:
            ops.append(("write", "C", g, "reduced", s, v))
            ops.append(("write", "C", Z - 1, "acc_free", s, v))
            ops.append(("wait", "F", "reduced", s, v))
            ops.append(("finish", "F", k, s, 0))
            ops.append(("write", "F", 0, "fin_ready", s, v))
        else:
            ops.append(("write", "C", 0, "fin_ready", s, v))
            ops.append(("write", "C", Z - 1, "acc_free", s, v))
    return ops


def round_ops(g: int, G: int, K: int, NB: int, round_index: int, late: bool = False) -> list:
    """All ops of rank g for one round, chunk by chunk (see chunk_ops).

    The executor issues them chunk by chunk and keeps at most a few chunks in
    flight per stream: a host that enqueued far ahead could block inside a
    launch on a stream stalled at a wait, before issuing the other stream's ops
    the wait depends on."""
    return [op for k in range(K) for op in chunk_ops(g, G, K, NB, round_index, k, late)]


def geq(flag_value: int, v: int) -> bool:
    """cuStreamWaitValue32 GEQ: (int32)(flag - v) >= 0."""
    d = (flag_value - v) & 0xFFFFFFFF
    return d < 0x80000000
