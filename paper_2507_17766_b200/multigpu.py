"""Multi-GPU butterfly merge: one process per GPU on one NVLink 5 / NVSwitch node,
miners partitioned in contiguous blocks over the ranks of the default group.

The reference merges a layer's N miner payloads in one process
(butterfly.py:216-240).  Its reduction order — a fp64 sum over the alive miners
in ascending index order, then one divide (mean_reducer, :156-158) — is what
makes the result reproducible, so the cross-GPU exchange keeps it exactly:

1. **chain** — rank 0 sums its alive replicas into fp64 running sums; the
   chain kernel (``bfly_chain_step``) stores them *directly into rank 1's inbox*
   over NVLink (TMA bulk stores from shared memory); rank 1 continues the same sum over its replicas and stores into
   rank 2, and so on.  The payload is cut into chunks, so all ranks stream
   concurrently (chunk k on rank g while chunk k+1 is on rank g-1);
2. **finish** — the last rank completes the sum, divides and scatters back into
   its replicas (``bfly_merge`` REDUCE with ``d_acc_in``), and the same kernel
   stores the final chunk into rank 0's inbox; after the last chunk it
   classifies, compares the redundant copies of corrupted shards and adopts or
   falls back (FINISH);
3. **relay** — rank 0 fans the final chunk out into its replicas and, in the
   same kernel (``bfly_fanout``), into rank 1's inbox, which does the same for
   rank 2, … (ring last -> 0 -> 1 -> … -> last-1).

Transfers are stores issued by the compute kernels into IPC-mapped peer memory
(no copy kernels, no staging); cross-GPU ordering uses 32-bit flags written and
awaited by the CUDA streams themselves (``bfly_stream_write_value`` /
``bfly_stream_wait_value``: front-end waits, no SM spins).  The op lists come
from ``ringsched.round_ops``, which the CPU simulator in tests/ verifies.
NCCL is used only for setup (IPC handles) and for the small end-of-round
broadcasts (per-shard results, late-decided shards).

Bytes received over NVLink per rank per round: 8 B x P of running sums (ranks >
0) plus s x P of the final vector (ranks < last).  The merged vector is
bit-identical to the single-GPU (and reference) result.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from . import errors
from . import ringsched as rs
from .device import ButterflyMerge, _DTYPES, _stream_handle

NB = 3  # inbox slots per ring of the chunked executor
WINDOW = 4  # chunks the host may run ahead of the GPUs per stream
FUSED_NB = 10  # slots per lane of the persistent ring (more spill the inboxes out of L2)


# ---------------------------------------------------------------------------
# communication: torch.distributed across processes, or threads on one device
# ---------------------------------------------------------------------------


class DistComm:
    """One process per GPU (torch.distributed, NCCL): the production transport.  Peer
    memory is shared through CUDA IPC handles; the persistent ring is one cooperative
    launch per GPU."""

    loopback = False

    def __init__(self):
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def all_gather_object(self, obj) -> list:
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def all_reduce_min(self, x: int, dev) -> int:
        t = torch.tensor([int(x)], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return int(t.item())

    def barrier(self):
        dist.barrier()

    def broadcast(self, t: torch.Tensor, src: int):
        dist.broadcast(t, src=src)

    def share_region(self, base: int, handle: bytes, dev) -> dict:
        """rank -> this process's mapping of every rank's region."""
        handles = self.all_gather_object(bytes(handle))
        peer = {}
        with torch.cuda.device(dev):
            for r, h in enumerate(handles):
                if r == self.rank:
                    peer[r] = base
                    continue
                p = ctypes.c_void_p()
                L.check(L.lib().bfly_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(h), ctypes.byref(p)))
                peer[r] = p.value
        dist.barrier()
        return peer

    def close_region(self, peer: dict, base: int, dev):
        lib = L.lib()
        with torch.cuda.device(dev):
            for r, p in peer.items():
                if r != self.rank:
                    lib.bfly_ipc_close(ctypes.c_void_p(p))
            lib.bfly_ipc_free(ctypes.c_void_p(base))

    def export_tensor(self, t: torch.Tensor):
        return _ipc_export(t)

    def map_tensor(self, token, dev) -> int:
        handle, off = token
        return _ipc_map(handle, dev) + off

    def unmap_tensor(self, token):
        _ipc_unmap(token[0])

    def launch_fused(self, desc, dev):
        with torch.cuda.device(dev):
            L.check(L.lib().bfly_ring_fused(ctypes.byref(desc), _stream_handle()))


class LoopbackGroup:
    """State shared by the ranks of a single-device loopback ring (one thread each)."""

    def __init__(self, world: int, timeout: float = 300.0):
        if not 2 <= world <= 8:
            raise errors.InvalidArgumentError("loopback rings have 2..8 ranks")
        self.world = world
        self.barrier = threading.Barrier(world, timeout=timeout)
        self.slots = [None] * world


class LoopbackComm:
    """G ranks of the ring as G threads of ONE process on ONE device (each with its own
    CUDA stream): collectives are exchanges between the threads, peer memory is plain
    device memory, and the persistent ring's G kernels become ONE cooperative launch of
    G x L CTAs (bfly_ring_fused_loopback).  The kernels, the protocol and every line of
    ShardedButterflyMerge above the transport are the multi-GPU ones — so the ring is
    parity-tested and profiled on a single GPU."""

    loopback = True

    def __init__(self, group: LoopbackGroup, rank: int):
        self.group, self.rank, self.world = group, rank, group.world

    def _exchange(self, obj) -> list:
        g = self.group
        g.barrier.wait()
        g.slots[self.rank] = obj
        g.barrier.wait()
        out = list(g.slots)
        g.barrier.wait()
        return out

    def all_gather_object(self, obj) -> list:
        return self._exchange(obj)

    def all_reduce_min(self, x: int, dev) -> int:
        return min(self._exchange(int(x)))

    def barrier(self):
        self.group.barrier.wait()

    def broadcast(self, t: torch.Tensor, src: int):
        cur = torch.cuda.current_stream(t.device)
        if self.rank == src:
            ev = torch.cuda.Event()
            ev.record(cur)
            slots = self._exchange((t, ev))
            done = self._exchange(None)
            for d in done:
                if d is not None:
                    cur.wait_event(d)  # the readers' copies finish before src writes t again
            return
        slots = self._exchange(None)
        src_t, ev = slots[src]
        cur.wait_event(ev)
        t.copy_(src_t)
        mine = torch.cuda.Event()
        mine.record(cur)
        self._exchange(mine)

    def share_region(self, base: int, handle: bytes, dev) -> dict:
        return dict(enumerate(self._exchange(base)))

    def close_region(self, peer: dict, base: int, dev):
        self.barrier()  # no rank frees its region while another's kernel may still use it
        torch.cuda.synchronize(dev)
        self.barrier()
        with torch.cuda.device(dev):
            L.lib().bfly_ipc_free(ctypes.c_void_p(base))

    def export_tensor(self, t: torch.Tensor):
        return t.data_ptr()

    def map_tensor(self, token, dev) -> int:
        return int(token)

    def unmap_tensor(self, token):
        pass

    def launch_fused(self, desc, dev):
        """Rank 0 launches every rank's lanes once all ranks' preceding work is queued."""
        cur = torch.cuda.current_stream(dev)
        ready = torch.cuda.Event()
        ready.record(cur)
        got = self._exchange((desc, ready))
        err, done = None, None
        if self.rank == 0:
            for _, ev in got:
                cur.wait_event(ev)
            arr = (L.RingFusedDesc * self.world)()
            for g, (d, _) in enumerate(got):
                arr[g] = d
            with torch.cuda.device(dev):
                rc = L.lib().bfly_ring_fused_loopback(arr, self.world, _stream_handle())
            if rc != L.OK:
                err = (rc, L.lib().bfly_last_error().decode(errors="replace"))
            done = torch.cuda.Event()
            done.record(cur)
        res = self._exchange((err, done))
        err, done = res[0]
        if err is not None:
            raise RuntimeError(f"loopback ring launch failed ({err[0]}): {err[1]}")
        cur.wait_event(done)


def run_loopback(world: int, fn, device=None, timeout: float = 300.0) -> list:
    """Run ``fn(rank, comm)`` for every rank of a ``world``-rank ring on ``world`` threads
    of this process, all on one CUDA device (each thread on its own stream), and return
    the per-rank results.  The first exception of any rank is re-raised (the others'
    collectives are aborted)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    group = LoopbackGroup(world, timeout)
    results, failures = [None] * world, [None] * world

    def body(rank):
        try:
            torch.cuda.set_device(dev)
            L.check(L.lib().bfly_preload())  # no lazy kernel load while the ranks' streams wait on each other
            with torch.cuda.stream(L.own_stream(dev, role=("loopback", rank))):
                results[rank] = fn(rank, LoopbackComm(group, rank))
                torch.cuda.current_stream(dev).synchronize()
        except BaseException as e:  # noqa: BLE001 - re-raised in the caller
            failures[rank] = e
            group.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"bfly-loopback-{r}") for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = [e for e in failures if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if first or any(failures):
        raise first[0] if first else next(e for e in failures if e is not None)
    return results


def special_ranges(assign: np.ndarray, P: int, failures: set, corrupted: set) -> list:
    """Element runs [lo, hi) of the shards decided only after the reduction: a
    surviving assignee is corrupted, or every assignee failed (butterfly.py:248-273)."""
    S = assign.shape[0]
    base, rem = divmod(P, S)
    runs = []
    for s in range(S):
        surv = [m for m in assign[s] if m not in failures]
        if surv and not any(m in corrupted for m in surv):
            continue
        lo = s * base + min(s, rem)
        hi = lo + base + (1 if s < rem else 0)
        if runs and runs[-1][1] == lo:
            runs[-1][1] = hi
        else:
            runs.append([lo, hi])
    return runs


CLS_FAST, CLS_SPECIAL, CLS_LOST = 0, 1, 2
PRED_NONE, PRED_MEAN, PRED_FALLBACK = 0, 1, 2


def classify_host(assign: np.ndarray, failures: set, corrupted: set, n_alive: int):
    """Host restatement of k_classify (csrc/bfly_merge.cu) for a chained reduce: per shard
    the class (fast / special / lost) and the predicted outcome of special and lost shards
    (an honest majority adopts the mean; no majority among >= 2 survivors falls back; a
    lone corrupted survivor has no prediction)."""
    S = assign.shape[0]
    cls = np.zeros(S, dtype=np.uint8)
    pred = np.zeros(S, dtype=np.uint8)
    for s in range(S):
        surv = [int(m) for m in assign[s] if int(m) not in failures]
        if not surv or n_alive == 0:
            cls[s], pred[s] = CLS_LOST, PRED_FALLBACK
        elif any(m in corrupted for m in surv):
            cls[s] = CLS_SPECIAL
            nh = sum(1 for m in surv if m not in corrupted)
            pred[s] = PRED_MEAN if 2 * nh > len(surv) else (PRED_FALLBACK if len(surv) >= 2 else PRED_NONE)
    return cls, pred


def mispredicted_shards(special_ids: np.ndarray, pred: np.ndarray, source: np.ndarray,
                        corr_kind: np.ndarray) -> np.ndarray:
    """The special / lost shards whose decision differs from k_classify's prediction, as
    k_apply judges it (csrc/bfly_merge.cu): a fallback outcome is as predicted when the
    prediction was the fallback, an adopted copy when the prediction was the mean and the
    adopted assignee is honest.  The persistent ring re-broadcasts exactly these."""
    pr = pred[special_ids]
    src = source[special_ids]
    honest_src = corr_kind[np.maximum(src, 0)] == 0
    as_pred = np.where(src < 0, pr == PRED_FALLBACK, (pr == PRED_MEAN) & honest_src)
    return special_ids[~as_pred]


def pack_results(entries, source, status, flagged, out):
    """entries | source | status | flagged into one byte buffer (8-byte aligned parts first)."""
    parts = [entries.reshape(-1).view(torch.uint8), source.view(torch.uint8), status.view(torch.uint8),
             flagged.view(torch.uint8)]
    out.copy_(torch.cat([p.to(out.device) for p in parts]))


def unpack_results(buf, entries, source, status, flagged):
    n, S = entries.shape[0], status.numel()
    buf = buf.to(entries.device)
    o = 8 * n * n
    entries.copy_(buf[:o].view(torch.float64).reshape(n, n))
    source.copy_(buf[o:o + 4 * S].view(torch.int32))
    o += 4 * S
    status.copy_(buf[o:o + S])
    flagged.copy_(buf[o + S:o + S + n])


_IPC_MAPS = {}  # IPC handle -> [mapped base, users]: a process maps an allocation once


def _ipc_export(t: torch.Tensor) -> tuple:
    """(IPC handle of the allocation holding t, byte offset of t in it)."""
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_uint64()
    with torch.cuda.device(t.device):
        L.check(L.lib().bfly_ipc_export(t.data_ptr(), h, ctypes.byref(off)))
    return bytes(h), int(off.value)


def _ipc_map(handle: bytes, dev) -> int:
    ent = _IPC_MAPS.get(handle)
    if ent is None:
        p = ctypes.c_void_p()
        with torch.cuda.device(dev):
            L.check(L.lib().bfly_ipc_open((ctypes.c_uint8 * 64).from_buffer_copy(handle), ctypes.byref(p)))
        ent = _IPC_MAPS[handle] = [p.value, 0]
    ent[1] += 1
    return ent[0]


def _ipc_unmap(handle: bytes):
    ent = _IPC_MAPS.get(handle)
    if ent is not None:
        ent[1] -= 1
        if ent[1] == 0:
            L.lib().bfly_ipc_close(ctypes.c_void_p(ent[0]))
            del _IPC_MAPS[handle]


def chunk_edges(P: int, chunk: int, ramp: bool = True) -> list:
    """Element boundaries of the pipelined chunks.  Full chunks of `chunk` elements, but
    with `ramp` the first and last few halve down to chunk/16: the ring's fill (the first
    chunk crosses every rank before the last one can reduce it) and drain (the last
    chunk's relay) then cost a few small steps instead of 2(G-1) full ones."""
    ramp_sizes = [chunk >> j for j in (4, 3, 2, 1) if (chunk >> j) >= (1 << 16) and (chunk >> j) % 4096 == 0]
    if not ramp or not ramp_sizes or P < 2 * sum(ramp_sizes) + 2 * chunk:
        sizes = [chunk] * (P // chunk) + ([P % chunk] if P % chunk else [])
    else:
        mid = P - 2 * sum(ramp_sizes)
        tail = mid % 4096  # keeps every inner boundary on a 4096-element (tile) edge
        mid -= tail
        body = [chunk] * (mid // chunk) + ([mid % chunk] if mid % chunk else [])
        sizes = ramp_sizes + body + ramp_sizes[::-1]
        sizes[-1] += tail
    edges = [0]
    for x in sizes:
        edges.append(edges[-1] + x)
    return edges


class _Region:
    """Layout of one rank's IPC region: NB fp64 running-sum slots, NB final-vector
    slots, and the flag arrays of ringsched (uint32 x NB each)."""

    def __init__(self, chunk: int, esize: int):
        def align(x):
            return (x + 255) & ~255

        self.acc = 0
        self.fin = align(NB * chunk * 8)
        self.flags = align(self.fin + NB * chunk * esize)
        self.total = align(self.flags + len(rs.FLAGS) * NB * 4)
        self.chunk, self.esize = chunk, esize

    def acc_slot(self, base: int, s: int) -> int:
        return base + self.acc + s * self.chunk * 8

    def fin_slot(self, base: int, s: int) -> int:
        return base + self.fin + s * self.chunk * self.esize

    def flag(self, base: int, name: str, s: int) -> int:
        return base + self.flags + (rs.FLAGS.index(name) * NB + s) * 4


class ShardedButterflyMerge:
    """One merge round over miners spread across the ranks of the default group.

    local        this rank's replicas (contiguous 1-D CUDA tensors of length P,
                 one dtype); rank g holds global miners [offset_g, offset_g + len).
    plan         the shard plan (DevicePlan or any object with .assign/.n_miners/
                 .n_shards/.redundancy/.payload_len), identical on every rank.
    failures / corruptions / fallback / tolerance: as ButterflyMerge, global indices.
    chunk        elements per pipelined chunk (multiple of 4096).
    comm         the transport: DistComm() (default, one process per GPU) or a
                 LoopbackComm (ranks as threads on one device, see run_loopback).
    executor     "auto" (the persistent ring whenever it applies) or "chunked".
    per_chunk_finish  chunked ring: the last rank decides each chunk's special shards
                 before relaying it (False: all after the ring; diagnostics).
    fuse_stats   persistent ring: the last rank's idle relay warps compute the special
                 shards' pair statistics during the ring (tiles offered through a
                 shared-memory queue), instead of k_stats after the kernel on every SM.
                 Off by default: FINISH shrinks 1.4 -> 0.3 ms but the queue slows the
                 last rank's compute warps (4 GPUs: a net loss; 2 GPUs: a gain).
    ring_tuning  persistent ring experiments: {"slots": inbox slots per lane (default
                 FUSED_NB), "lag": publication lag 1..3, "pub_every": publish every k-th
                 step} (bfly.h; defaults are the measured best).
    debug / timing    diagnostics of the chunked ring (per-op watchdog, timeline) and
                 per-phase CUDA-event times of a round (``.timings``).
    """

    def __init__(self, local: list, plan, *, failures=(), corruptions=None, fallback=None,
                 want_merged: bool = False, tolerance: float = 1e-6, chunk: int = 1 << 24, comm=None,
                 executor: str = "auto", per_chunk_finish: bool = True, debug: int = 0, timing: bool = False,
                 fuse_stats: bool = False, ring_tuning: dict | None = None):
        self.comm = comm if comm is not None else DistComm()
        self.fuse_stats = bool(fuse_stats)
        self.ring_tuning = dict(ring_tuning or {})
        self.rank = self.comm.rank
        self.world = G = self.comm.world
        if executor not in ("auto", "chunked"):
            raise errors.InvalidArgumentError(f"unknown executor {executor!r}")
        if not local:
            raise errors.InvalidArgumentError("every rank must hold at least one miner")
        self.local = list(local)
        self.dev = local[0].device
        if self.dev.type != "cuda":
            raise RuntimeError("the multi-GPU merge runs on CUDA devices (no CPU fallback)")
        self.P = int(local[0].numel())
        self.esize = local[0].element_size()
        self.dtype = _DTYPES[local[0].dtype]
        if chunk % 4096:
            raise errors.InvalidArgumentError("chunk must be a multiple of 4096 elements")
        self.chunk = int(min(chunk, ((self.P + 4095) // 4096) * 4096))  # inbox slot size
        self.edges = chunk_edges(self.P, self.chunk, ramp=G > 1)
        self.K = len(self.edges) - 1
        self.counts = [int(c) for c in self.comm.all_gather_object(len(local))]
        self.offset = sum(self.counts[: self.rank])
        self.n = sum(self.counts)
        if self.n != plan.n_miners:
            raise errors.ShapeError(f"plan expects {plan.n_miners} miners, ranks hold {self.n}")
        failures = set(int(m) for m in failures)
        self.failures = failures
        self.alive = [m for m in range(self.n) if m not in failures]
        mine = range(self.offset, self.offset + len(local))
        self.local_alive = [self.local[m - self.offset] for m in mine if m not in failures]
        self.plan = plan
        self.want_merged = want_merged
        self.is_last = self.rank == G - 1
        self.plan_r = int(getattr(plan, "redundancy", 2))
        self._round = 0
        self.debug = int(debug)
        self.timing = bool(timing)  # per-phase ms in .timings
        self.timings = {}
        self._tables = []  # keeps the device pointer tables alive
        self._peer = None

        corrupted = {m for m in (corruptions or {}) if m not in failures}
        assign = plan.assign.cpu().numpy() if hasattr(plan.assign, "cpu") else np.asarray(plan.assign)
        runs = special_ranges(assign, self.P, failures, corrupted) if (corrupted or len(failures) >= 2) else []
        # The last rank finishes a chunk's late (corrupted / lost) shards right after
        # reducing it, before the final chunk enters the relay, so only shards that
        # straddle a chunk boundary are finished after the ring and broadcast late.
        self._finish_ranges, straddlers = self._chunk_shard_ranges(plan.n_shards)
        self.straddlers = straddlers
        self._straddle_dev = torch.tensor(straddlers, dtype=torch.int32, device=self.dev)
        self._per_chunk_finish = bool(per_chunk_finish)
        # fallback values come from the lowest alive miner when no fallback is given; when
        # that replica lives on another rank the last rank reads it in place over NVLink
        # (IPC-mapped): chunk k of it is only overwritten by the relay, which starts after
        # the last rank has reduced and finished chunk k
        self._needs_fb = bool(fallback is None and self.alive and runs)
        self.fb_owner, self._fb_buf, self._fb_ptr, self._fb_handle = None, None, None, None
        if self._needs_fb:
            m0 = self.alive[0]
            self.fb_owner = next(r for r in range(G) if sum(self.counts[: r + 1]) > m0)
        # The persistent ring (one kernel per GPU, csrc/bfly_ring.cu) runs every round whose
        # shards are >= 2 elements long and whose replicas are 16-byte aligned on every rank.
        # Corrupted / lost shards ride along with k_classify's predicted outcome and are
        # decided after the kernel; it needs that no decision can end in fallback values
        # the relay has already overwritten: the fallback is given, or the lowest alive
        # replica is not on the last rank and no special shard has an honest majority
        # (only such a shard could, with non-finite means, fall back unpredicted).
        self._cls, self._pred = classify_host(assign, failures, corrupted, len(self.alive))
        self._special_ids = np.flatnonzero(self._cls != CLS_FAST)
        # fast shards: the other ranks apply the last rank's non-finite decisions on device
        self._fast_mask = torch.from_numpy((self._cls == CLS_FAST).astype(np.uint8)).to(self.dev)
        self._fallback = None if fallback is None else fallback.to(self.dev, torch.float64).contiguous()
        honest_major = bool(np.any((self._cls == CLS_SPECIAL) & (self._pred == PRED_MEAN)))
        self.fused = bool(G > 1 and self.P // plan.n_shards >= 2 and executor == "auto"
                          and not (self._needs_fb and (self.fb_owner == G - 1 or honest_major)))
        if self.fused:
            self.fused = bool(self.comm.all_reduce_min(int(all(t.data_ptr() % 16 == 0 for t in self.local)),
                                                       self.dev))
        self._corr_kind = np.zeros(self.n, dtype=np.int32)
        for m, c in (corruptions or {}).items():
            self._corr_kind[int(m)] = int(c.code()) if hasattr(c, "code") else 1
        late = ([] if self.fused else
                [r for r in runs if any(r[0] < b < r[1] for b in self._chunk_starts())]
                if G > 1 and self._per_chunk_finish else runs)
        self.late_runs = late
        self.special_runs = late  # kept name: ranges broadcast after the ring
        self._late_set = self._range_set(late) if late else None
        if G > 1 and self._needs_fb and self.fb_owner != G - 1:
            info = self.comm.export_tensor(local[m0 - self.offset]) if self.rank == self.fb_owner else None
            infos = self.comm.all_gather_object(info)
            if self.is_last:
                self._fb_handle = infos[self.fb_owner]
                self._fb_ptr = self.comm.map_tensor(self._fb_handle, self.dev)
                if late:  # shards straddling chunk edges finish after the relay: copy theirs first
                    self._fb_buf = torch.empty_like(local[0])

        self.job = None
        if self.is_last:
            reps = [None] * self.n
            for i, t in enumerate(local):
                reps[self.offset + i] = t
            fb_src = None
            if self._needs_fb:
                fb_src = self._fb_ptr if self._fb_ptr is not None else reps[self.alive[0]]
            self.job = ButterflyMerge(reps, plan, remote_sum=G > 1, n_div=len(self.alive), failures=failures,
                                      corruptions=corruptions, fallback=fallback, fallback_src=fb_src,
                                      scatter_back=True, want_merged=want_merged, tolerance=tolerance)
            # shards decided after the exchange (non-finite means) cannot read the lowest
            # alive replica any more: the relay has overwritten it (bfly.h fallback_gone)
            self.job._args.fallback_gone = int(G > 1)
        # last rank: late shards possible (corrupted survivors, or shards whose assignees
        # all failed) -> each chunk's are finished on the late-shard stream
        self._late_mode = bool(self.is_last and self.job.needs_finish() and self._per_chunk_finish)
        S, n = plan.n_shards, self.n
        self._res = torch.empty(8 * n * n + 4 * S + S + n, dtype=torch.uint8, device=self.dev)
        self.status = torch.empty(S, dtype=torch.uint8, device=self.dev)
        self.flagged = torch.empty(n, dtype=torch.uint8, device=self.dev)
        self.source = torch.empty(S, dtype=torch.int32, device=self.dev)
        self.entries = torch.empty((n, n), dtype=torch.float64, device=self.dev)
        self.merged = torch.empty(self.P, dtype=torch.float64, device=self.dev) if want_merged else None
        self._src_table = self._table(self.local_alive) if self.local_alive else None
        self._local_table = self._table(self.local)
        self._fb_table = self._table([self._fb_buf]) if self._fb_buf is not None else None
        if self.fused:
            self._late_mode = False  # (r = 3) every shard's FINISH runs after the kernel
            self._setup_fused()
        elif G > 1:
            self._setup_ring()

    # -- late shards -------------------------------------------------------------
    def _chunk_starts(self):
        return self.edges[1:-1]

    def _chunk_shard_ranges(self, S: int):
        """Per chunk k, the shards lying entirely inside it ([s_begin, s_end)), and the
        shards that straddle a chunk boundary."""
        base, rem = divmod(self.P, S)

        def start(s):
            return s * base + min(s, rem)

        def shard_of(e):
            big = rem * (base + 1)
            return e // (base + 1) if e < big else rem + (e - big) // base

        ranges, straddle = [], []
        for k in range(self.K):
            b, e = self._bounds(k)
            s0 = shard_of(b)
            if start(s0) < b:
                s0 += 1
            s1 = shard_of(e - 1)
            if start(s1 + 1) > e:  # start(S) == P, so s1 + 1 <= S is always valid
                s1 -= 1
            ranges.append((s0, max(s0, s1 + 1)))
            if k > 0 and start(shard_of(b)) < b:
                straddle.append(shard_of(b))
        return ranges, sorted(set(straddle))

    @staticmethod
    def _packed_offsets(runs):
        offs, off = [], 0
        for lo, hi in runs:
            off += (lo - off) % 16  # same 32-byte alignment on both sides (vector copies)
            offs.append(off)
            off += hi - lo
        return offs, off

    def _range_set(self, runs):
        """Device table {lo, hi, packed offset} + packed buffer for element runs."""
        offs, off = self._packed_offsets(runs)
        tab = [(lo, hi, o) for (lo, hi), o in zip(runs, offs)]
        return (torch.tensor(tab, dtype=torch.int64, device=self.dev),
                torch.empty(off, dtype=self.local[0].dtype, device=self.dev))

    # -- peer-memory ring ------------------------------------------------------
    def _table(self, ptrs) -> torch.Tensor:
        t = torch.tensor([p if isinstance(p, int) else p.data_ptr() for p in ptrs], dtype=torch.int64).to(self.dev)
        self._tables.append(t)
        return t

    def _open_region(self, total: int):
        """Allocate this rank's region (zeroed, IPC-exportable) and map every other rank's."""
        lib = L.lib()
        base = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * 64)()
        with torch.cuda.device(self.dev):
            L.check(lib.bfly_ipc_alloc(total, ctypes.byref(base), handle))
        self._base = base.value
        self._peer = self.comm.share_region(self._base, bytes(handle), self.dev)
        self._peer_arr = (ctypes.c_uint64 * self.world)(*[self._peer[r] for r in range(self.world)])

    def _setup_fused(self):
        """The persistent single-kernel ring (bfly_ring_fused, csrc/bfly_ring.cu)."""
        lib = L.lib()
        lanes = int(lib.bfly_ring_fused_lanes(self.dtype))
        if self.comm.loopback:  # every rank's lanes share this one device
            lanes //= self.world
        self.lanes = self.comm.all_reduce_min(lanes, self.dev)  # every rank deals tiles to the same lanes
        if self.lanes < 1:
            raise RuntimeError("fused ring: no co-resident lanes on this device")
        o = [ctypes.c_int64() for _ in range(3)]
        nb = self.ring_tuning.get("slots", FUSED_NB)
        L.check(lib.bfly_ring_fused_layout(self.lanes, nb, self.dtype, *[ctypes.byref(x) for x in o]))
        self._open_region(o[2].value)
        d = L.RingFusedDesc()
        d.rank, d.world, d.lanes, d.nb, d.dtype = self.rank, self.world, self.lanes, nb, self.dtype
        d.lag = int(self.ring_tuning.get("lag", 0))
        d.pub_every = int(self.ring_tuning.get("pub_every", 0))
        d.n_src, d.n_dst, d.n_div = len(self.local_alive), len(self.local), len(self.alive)
        d.payload_len = self.P
        d.peer_base = ctypes.cast(self._peer_arr, ctypes.c_void_p)
        d.d_src = self._src_table.data_ptr() if self._src_table is not None else None
        d.d_dst = self._local_table.data_ptr()
        if self.is_last:
            d.d_merged = self.job.merged.data_ptr() if self.job.merged is not None else None
            # fuse_stats: the kernel's stats warps compute the special shards' pair
            # statistics per k_ring tile (FINISH then covers only the rest: shard edges,
            # tiles the queue could not take, r = 3)
            self.job._args.stat_tile = int(lib.bfly_ring_fused_stat_tile(self.dtype)) if self.fuse_stats else 0
            d.merge_args = ctypes.pointer(self.job._args)
            d.special = int(len(self._special_ids) > 0)
        self._fdesc = d

    def _setup_ring(self):
        self.layout = lay = _Region(self.chunk, self.esize)
        self._open_region(lay.total)
        self._relay = L.own_stream(self.dev, role=("relay", self.rank))
        # last rank: per-chunk late shards, high priority so a chunk's decision does not queue
        # behind the next chunk's reduce CTAs (the relay waits for it)
        self._late = L.own_stream(self.dev, priority=-1, role=("late", self.rank))
        Z = self.world - 1
        g = self.rank
        # per (chunk, slot) scatter-back tables: the last rank pushes the final chunk
        # into rank 0's inbox (pointer biased by -begin: k_reduce indexes globally);
        # relay ranks fan out into their replicas and the successor's inbox
        self._reduce_tables, self._fan_tables = {}, {}
        for k in range(self.K):
            b = self.edges[k]
            for s in range(NB):
                if self.is_last:
                    fin0 = lay.fin_slot(self._peer[0], s) - b * self.esize
                    self._reduce_tables[k, s] = self._table(self.local + [fin0])
                else:
                    succ = rs.relay_succ(g, Z)
                    views = [t.data_ptr() + b * self.esize for t in self.local]
                    if succ is not None:
                        views.append(lay.fin_slot(self._peer[succ], s))
                    self._fan_tables[k, s] = self._table(views)
        # descriptor of the native executor (bfly_ring_round)
        d = L.RingDesc()
        d.rank, d.world, d.k_chunks, d.nb = g, self.world, self.K, NB
        d.payload_len, d.chunk, d.dtype, d.esize = self.P, self.chunk, self.dtype, self.esize
        self._edge_arr = (ctypes.c_int64 * (self.K + 1))(*self.edges)
        d.chunk_edges = ctypes.cast(self._edge_arr, ctypes.c_void_p)
        d.peer_base = ctypes.cast(self._peer_arr, ctypes.c_void_p)
        d.off_acc, d.off_fin, d.off_flags = lay.acc, lay.fin, lay.flags
        d.d_src_table = self._src_table.data_ptr() if self._src_table is not None else None
        d.n_src = len(self.local_alive)
        d.window = WINDOW
        if self.is_last:
            self._red_arr = (ctypes.c_uint64 * (self.K * NB))(
                *[self._reduce_tables[k, s].data_ptr() for k in range(self.K) for s in range(NB)])
            d.reduce_tables = ctypes.cast(self._red_arr, ctypes.c_void_p)
            d.reduce_n = len(self.local) + 1
            d.merge_args = ctypes.pointer(self.job._args)
            if self._late_mode:
                self._fin_arr = (ctypes.c_int64 * (2 * self.K))(*[x for r in self._finish_ranges for x in r])
                d.finish_ranges = ctypes.cast(self._fin_arr, ctypes.c_void_p)
        else:
            self._fan_arr = (ctypes.c_uint64 * (self.K * NB))(
                *[self._fan_tables[k, s].data_ptr() for k in range(self.K) for s in range(NB)])
            d.fan_tables = ctypes.cast(self._fan_arr, ctypes.c_void_p)
            d.fan_n = len(self.local) + (1 if rs.relay_succ(g, Z) is not None else 0)
        self._desc = d

    def close(self):
        """Release the peer regions (a collective: every rank calls it)."""
        if self._peer:
            torch.cuda.synchronize(self.dev)
            self.comm.close_region(self._peer, self._base, self.dev)
            if self._fb_handle is not None:
                self.comm.unmap_tensor(self._fb_handle)
                self._fb_handle = None
            self._peer = None

    def __del__(self):
        try:
            if not self.comm.loopback:  # (a loopback close is a collective of the threads)
                self.close()
        except Exception:
            pass

    def _bounds(self, k):
        return self.edges[k], self.edges[k + 1]

    def _issue(self, op):
        lib, lay = L.lib(), self.layout
        kind, st = op[0], op[1]
        stream = {"C": _stream_handle(), "R": self._relay.cuda_stream, "F": self._late.cuda_stream}[st]
        if kind == "wait":
            _, _, flag, s, v = op
            L.check(lib.bfly_stream_wait_value(lay.flag(self._base, flag, s), v, stream))
        elif kind == "write":
            _, _, peer, flag, s, v = op
            L.check(lib.bfly_stream_write_value(lay.flag(self._peer[peer], flag, s), v, stream))
        elif kind == "chain":
            _, _, k, s, dst = op
            b, e = self._bounds(k)
            acc_in = lay.acc_slot(self._base, s) if self.rank > 0 else None
            src = self._src_table.data_ptr() if self._src_table is not None else None
            L.check(lib.bfly_chain_step(src, len(self.local_alive), self.dtype, acc_in,
                                        lay.acc_slot(self._peer[dst], s), b, e, stream))
        elif kind == "reduce":
            _, _, k, s, _fin_rank = op
            b, e = self._bounds(k)
            tab = self._reduce_tables[k, s]
            self.job.reduce_range(b, e, acc_in=lay.acc_slot(self._base, s), dst_table=(tab.data_ptr(), tab.numel()))
        elif kind == "finish":
            _, _, k, s, _fin_rank = op
            tab = self._reduce_tables[k, s]
            s0, s1 = self._finish_ranges[k]
            with torch.cuda.stream(self._late):
                self.job.run_finish_range(s0, s1, dst_table=(tab.data_ptr(), tab.numel()))
        elif kind == "fanout":
            _, _, k, s, _fwd = op
            b, e = self._bounds(k)
            tab = self._fan_tables[k, s]
            L.check(lib.bfly_fanout(lay.fin_slot(self._base, s), tab.data_ptr(), tab.numel(), (e - b) * self.esize,
                                    stream))

    def _host_wait(self, events, deadline: float = 120.0):
        import time

        t0 = time.time()
        while not all(e.query() for e in events):
            if time.time() - t0 > deadline:
                raise RuntimeError("multi-GPU ring made no progress for %.0f s" % deadline)
            time.sleep(20e-6)

    def _watch(self, marks, deadline: float = 30.0):
        """Debug aid (BFLY_DEBUG_RING=1): wait for every op with a deadline and report
        the first op each stream is stuck at, with this rank's flag values."""
        import sys
        import time

        t0 = time.time()
        while not all(ev.query() for _, ev in marks):
            if time.time() - t0 > deadline:
                stuck = {}
                for op, ev in marks:
                    if not ev.query() and op[1] not in stuck:
                        stuck[op[1]] = op
                flags = torch.empty(len(rs.FLAGS) * NB, dtype=torch.int32, device=self.dev)
                side = L.own_stream(self.dev, role=("watch", self.rank))
                with torch.cuda.stream(side):
                    L.lib().bfly_fanout(self._base + self.layout.flags,
                                        self._table([flags]).data_ptr(), 1, 4 * len(rs.FLAGS) * NB, side.cuda_stream)
                side.synchronize()
                print(f"[rank {self.rank}] ring stuck after {deadline}s: {stuck}; flags "
                      f"{dict(zip(rs.FLAGS, flags.view(len(rs.FLAGS), NB).tolist()))}", file=sys.stderr, flush=True)
                raise RuntimeError("multi-GPU ring did not complete")
            time.sleep(0.005)

    def _copy_ranges(self, rset, full, table, n_dst, scatter):
        ranges, packed = rset
        L.check(L.lib().bfly_copy_ranges(full, packed.data_ptr(), table, n_dst, ranges.data_ptr(), ranges.shape[0],
                                         self.esize, scatter, _stream_handle()))

    # -- one round -------------------------------------------------------------
    def run(self) -> "ShardedButterflyMerge":
        G, g = self.world, self.rank
        last = G - 1
        cur = torch.cuda.current_stream(self.dev)
        tm = [] if self.timing else None

        def mark(name):
            if tm is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(cur)
                tm.append((name, ev))

        mark("start")
        if self.debug == 3:  # timeline: every op's completion time from here (tools/ring_timeline.py)
            self._t0 = torch.cuda.Event(enable_timing=True)
            self._t0.record(cur)
        if G == 1:
            for k in range(self.K):
                b, e = self._bounds(k)
                self.job.reduce_range(b, e)
        elif self.fused:
            self._fdesc.round_index = self._round
            self.comm.launch_fused(self._fdesc, self.dev)
        else:
            # fallback values (the lowest alive miner's replica) for the late shards: packed
            # before the relay overwrites that replica, sent while the ring runs
            self._relay.wait_stream(cur)
            self._late.wait_stream(cur)
            if self._fb_buf is not None:  # straddling late ranges' fallback values, before any relay
                self._copy_ranges(self._late_set, self._fb_ptr, None, 0, 0)
                self._copy_ranges(self._late_set, None, self._fb_table.data_ptr(), 1, 1)
            mark("fallback")
            marks, window = [], []
            if not self.debug:  # native executor: the whole round issued from C++
                self._desc.stream_c = _stream_handle()
                self._desc.stream_r = self._relay.cuda_stream
                self._desc.stream_f = self._late.cuda_stream
                with torch.cuda.device(self.dev):
                    L.check(L.lib().bfly_ring_round(ctypes.byref(self._desc), self._round & 0xFFFFFFFF))
            for k in range(self.K if self.debug else 0):  # debug: the same ops issued from Python
                for op in rs.chunk_ops(g, G, self.K, NB, self._round, k, self._late_mode):
                    self._issue(op)
                    if self.debug:
                        ev = torch.cuda.Event(enable_timing=self.debug == 3)
                        ev.record({"C": cur, "R": self._relay, "F": self._late}[op[1]])
                        marks.append((op, ev))
                # bounded run-ahead: never more than WINDOW chunks queued per stream
                done = (torch.cuda.Event(), torch.cuda.Event())
                done[0].record(cur)
                done[1].record(self._relay)
                window.append(done)
                if len(window) > WINDOW:
                    self._host_wait(window.pop(0))
            if self.debug == 1:
                self._watch(marks)
            self._marks = marks
            cur.wait_stream(self._relay)
            cur.wait_stream(self._late)
        self._round += 1
        mark("ring")

        # finish the shards that straddle chunk boundaries, then distribute the
        # per-shard results and those shards' final values
        if self.is_last:
            if G == 1:
                self.job.run(L.PHASE_FINISH)
            elif self.job.needs_finish() and not self._late_mode:
                if self._fb_buf is not None:
                    self.job._args.d_fallback_src = self._fb_buf.data_ptr()
                self.job.run(L.PHASE_FINISH)
                self.job._args.d_fallback_src = self._fb_ptr if self._fb_ptr is not None else self.job._args.d_fallback_src
            elif self.fused:  # every shard fast: only a non-finite mean can still fall back
                self.job.run(L.PHASE_CHECK)
            elif self.job.needs_finish() and self.straddlers:
                a = self.job._args
                if self._fb_buf is not None:  # the owner's replica may hold relayed values by now
                    a.d_fallback_src = self._fb_buf.data_ptr()
                try:
                    self.job.run_finish_list(self._straddle_dev)
                finally:
                    a.d_fallback_src = self._fb_ptr if self._fb_ptr is not None else a.d_fallback_src
            pack_results(self.job.entries, self.job.source, self.job.status, self.job.flagged, self._res)
            if self.special_runs:
                self._copy_ranges(self._late_set, self.local[0].data_ptr(), None, 0, 0)
        mark("finish")
        if G > 1:
            self.comm.broadcast(self._res, src=last)
            mark("results")
            if self.special_runs:
                self.comm.broadcast(self._late_set[1], src=last)
                mark("late_bcast")
                if not self.is_last:
                    self._copy_ranges(self._late_set, None, self._local_table.data_ptr(), len(self.local), 1)
                mark("late_scatter")
            if self.want_merged:
                if self.is_last:
                    self.merged.copy_(self.job.merged)
                self.comm.broadcast(self.merged, src=last)
        elif self.want_merged:
            self.merged.copy_(self.job.merged)
        unpack_results(self._res, self.entries, self.source, self.status, self.flagged)
        if G > 1 and not self.is_last:
            # fast shards the last rank decided a disagreement (non-finite means): the
            # fallback (or NaN) into this rank's replicas, on the device
            L.check(L.lib().bfly_fill_shards(self.status.data_ptr(), self._fast_mask.data_ptr(),
                                             self._fallback.data_ptr() if self._fallback is not None else None,
                                             self._local_table.data_ptr(), len(self.local), self.dtype, self.P,
                                             self.plan.n_shards, _stream_handle()))
        if G > 1 and self.fused and len(self._special_ids):
            self._rebroadcast_mispredicted()
        mark("end")
        if tm is not None:
            torch.cuda.synchronize(self.dev)
            self.timings = {b[0]: a[1].elapsed_time(b[1]) for a, b in zip(tm, tm[1:])}
        if self.debug == 2 and G > 1:
            self._watch(self._marks)
        return self

    def _rebroadcast_mispredicted(self):
        """Persistent ring: the relayed tiles of special / lost shards carried the predicted
        outcome; the shards FINISH decided otherwise (k_apply rewrote them on the last rank)
        are sent to the other ranks and scattered into their replicas.  Every rank reads
        the same per-shard results, so they agree on the list without communicating.
        (Fast shards decided a disagreement — non-finite means — need no data: every rank
        writes the fallback itself, bfly_fill_shards.)"""
        mis = mispredicted_shards(self._special_ids, self._pred, self.source.cpu().numpy(), self._corr_kind)
        self.mispredicted = len(mis)
        if not len(mis):
            return
        base, rem = divmod(self.P, self.plan.n_shards)
        runs = []
        for sh in mis.tolist():
            lo = sh * base + min(sh, rem)
            hi = lo + base + (1 if sh < rem else 0)
            if runs and runs[-1][1] == lo:
                runs[-1][1] = hi
            else:
                runs.append([lo, hi])
        rset = self._range_set(runs)
        if self.is_last:
            self._copy_ranges(rset, self.local[0].data_ptr(), None, 0, 0)
        self.comm.broadcast(rset[1], src=self.world - 1)
        if not self.is_last:
            self._copy_ranges(rset, None, self._local_table.data_ptr(), len(self.local), 1)

    def timeline(self) -> list:
        """BFLY_DEBUG_RING=3: (op, ms after the round started) for every op of the last
        round, once it has completed."""
        torch.cuda.synchronize(self.dev)
        return [(op, self._t0.elapsed_time(ev)) for op, ev in self._marks]

    def launches_per_run(self) -> int:
        """Our kernels per round on this rank (bench.py gpu_launches); the re-broadcast of
        mispredicted shards (none in the benchmarked rounds) is not counted."""
        # FINISH: k_nonfinite, k_stats, k_decide, [k_entries3], k_apply; CHECK: k_nonfinite
        fin = 4 + (1 if self.plan_r > 2 else 0)
        if self.world == 1:
            return 2 + self.K + (fin if self.job.needs_finish() else 1)
        if self.fused:  # k_ring; the last rank adds k_fill_nan, k_classify and FINISH or CHECK,
            # the others k_fill_shards
            return 3 + (fin if self.job.needs_finish() else 1) if self.is_last else 2
        if self.is_last:
            n = 2 + self.K + 1  # k_fill_nan + k_classify, one k_reduce per chunk, k_nonfinite (last chunk)
            if self._late_mode:
                n += fin * sum(1 for b, e in self._finish_ranges if e > b)
                n += fin if self.straddlers else 0
            n += 2 if self._fb_buf is not None else 0  # straddlers' fallback ranges: gather + scatter
            n += 1 if self.special_runs else 0  # late ranges packed for the broadcast
            return n
        # k_chain + k_fanout per chunk, [late ranges scattered], k_fill_shards
        return 2 * self.K + (1 if self.special_runs else 0) + 1

    def bytes_per_round(self) -> dict:
        """Algorithmic HBM and NVLink bytes of this rank for one round."""
        s = self.esize
        hbm = (len(self.local_alive) + len(self.local)) * self.P * s
        nvl_in = (8 * self.P if self.rank > 0 else 0) + (s * self.P if not self.is_last else 0)
        return {"hbm": hbm, "nvlink_in": nvl_in}
