"""Multi-GPU butterfly merge: one process per GPU (torch.distributed, NCCL over
NVLink 5 / NVSwitch), miners partitioned in contiguous blocks over the ranks.

The reference merges a layer's N miner payloads in one process
(butterfly.py:216-240).  Its reduction order — a fp64 sum over the alive miners
in ascending index order, then one divide (mean_reducer, :156-158) — is what
makes the result reproducible, so the cross-GPU exchange keeps it exactly:

1. **chain** — rank 0 sums its alive replicas into a fp64 running sum and sends
   it to rank 1, which continues the same sum over its own replicas, and so on
   (``bfly_chain_step``); the payload is cut into chunks so all ranks stream
   concurrently (chunk k on rank g overlaps chunk k+1 arriving from rank g-1);
2. **finish** — the last rank completes the sum, divides, classifies shards,
   compares the redundant copies of corrupted shards and adopts or falls back
   (``bfly_merge`` with ``d_acc_in``), scattering back into its own replicas;
3. **distribute** — as soon as the last rank has reduced chunk k, chunk k of
   the final vector travels a relay ring (last -> 0 -> 1 -> ...), each rank
   fanning it out into its replicas (``bfly_fanout``) and forwarding it,
   overlapping the chain of later chunks.
   Shards decided only after the chain (corrupted or lost ones) are packed,
   broadcast and scattered once more (``bfly_copy_ranges``), together with the
   per-shard results (status, agreement entries, flags).

The merged vector is bit-identical to the single-GPU (and reference) result.
NVLink bytes received per rank per round: 8 B x P of running sums (ranks > 0)
plus s x P of the final vector (ranks < G-1).  All transfers are NCCL
send/recv on ONE communicator, grouped per step of a systolic schedule (see
``run``) so that every rank issues them in the same global order.

``ops`` abstracts the per-rank compute so the host-side schedule can be tested
on CPU over gloo (tests/test_multigpu_gloo.py); the default is the CUDA library.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from . import errors
from .device import ButterflyMerge, _DTYPES, _ptr_table, _stream_handle


class CudaOps:
    """Per-rank compute through libbfly (current CUDA stream)."""

    def __init__(self):
        self._tables = {}

    def chain(self, src: list, acc_in, acc_out, begin: int, end: int):
        table = self._table(src)
        dtype = _DTYPES[src[0].dtype] if src else L.F32
        L.check(L.lib().bfly_chain_step(table.data_ptr() if table is not None else None, len(src), dtype,
                                        acc_in.data_ptr() if acc_in is not None else None, acc_out.data_ptr(),
                                        begin, end, _stream_handle()))

    def fanout(self, src, dsts: list):
        if not dsts:
            return
        table = self._table(dsts)
        L.check(L.lib().bfly_fanout(src.data_ptr(), table.data_ptr(), len(dsts), src.numel() * src.element_size(),
                                    _stream_handle()))

    def gather_ranges(self, full, packed, ranges):
        L.check(L.lib().bfly_copy_ranges(full.data_ptr(), packed.data_ptr(), None, 0, ranges.data_ptr(),
                                         ranges.shape[0], full.element_size(), 0, _stream_handle()))

    def scatter_ranges(self, packed, dsts, ranges):
        table = self._table(dsts)
        L.check(L.lib().bfly_copy_ranges(None, packed.data_ptr(), table.data_ptr(), len(dsts), ranges.data_ptr(),
                                         ranges.shape[0], packed.element_size(), 1, _stream_handle()))

    def make_job(self, replicas, plan, **kw):
        return ButterflyMerge(replicas, plan, remote_sum=True, **kw)

    def _table(self, tensors):
        if not tensors:
            return None
        key = tuple(t.data_ptr() for t in tensors)
        t = self._tables.get(key)
        if t is None:
            t = self._tables[key] = _ptr_table(tensors, tensors[0].device)
        return t


def _special_ranges(assign: np.ndarray, P: int, failures: set, corrupted: set) -> list:
    """Element runs [lo, hi) of the shards decided after the chain: some surviving
    assignee is corrupted, or every assignee failed (butterfly.py:248-273)."""
    S = assign.shape[0]
    base, rem = divmod(P, S)
    runs = []
    for s in range(S):
        members = assign[s]
        surv = [m for m in members if m not in failures]
        if surv and not any(m in corrupted for m in surv):
            continue
        lo = s * base + min(s, rem)
        hi = lo + base + (1 if s < rem else 0)
        if runs and runs[-1][1] == lo:
            runs[-1][1] = hi
        else:
            runs.append([lo, hi])
    return runs


class ShardedButterflyMerge:
    """One merge round over miners spread across the ranks of the default group.

    local        this rank's replicas (1-D tensors of equal length P); rank g holds
                 the global miners [offset_g, offset_g + len(local)) in order.
    plan         the shard plan (DevicePlan or any object with .assign/.n_miners/
                 .n_shards/.redundancy/.payload_len); identical on every rank.
    failures / corruptions / fallback / tolerance: as ButterflyMerge, with global
                 miner indices.
    chunk        elements per pipelined chain message (multiple of 4096).
    """

    def __init__(self, local: list, plan, *, failures=(), corruptions=None, fallback=None,
                 want_merged: bool = False, tolerance: float = 1e-6, chunk: int = 1 << 24, ops=None):
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.ops = ops or CudaOps()
        if not local:
            raise errors.InvalidArgumentError("every rank must hold at least one miner")
        self.local = list(local)
        self.dev = local[0].device
        self.cuda = self.dev.type == "cuda"
        self.P = int(local[0].numel())
        if chunk % 4096:
            raise errors.InvalidArgumentError("chunk must be a multiple of 4096 elements")
        self.chunk = int(chunk)
        cd = self._comm_dev()
        counts = [torch.zeros(1, dtype=torch.int64, device=cd) for _ in range(self.world)]
        dist.all_gather(counts, torch.tensor([len(local)], dtype=torch.int64, device=cd))
        self.counts = [int(c.item()) for c in counts]
        self.offset = sum(self.counts[: self.rank])
        self.n = sum(self.counts)
        if self.n != plan.n_miners:
            raise errors.ShapeError(f"plan expects {plan.n_miners} miners, ranks hold {self.n}")
        G = self.world
        failures = set(int(m) for m in failures)
        self.failures = failures
        self.alive = [m for m in range(self.n) if m not in failures]
        mine = range(self.offset, self.offset + len(local))
        self.local_alive = [self.local[m - self.offset] for m in mine if m not in failures]
        self.plan = plan
        self.want_merged = want_merged
        self.is_last = self.rank == G - 1
        nb = 3
        clen = min(self.chunk, self.P)
        f64 = dict(dtype=torch.float64, device=self.dev)
        self._inb = [torch.empty(clen, **f64) for _ in range(nb)] if self.rank > 0 else []
        self._outb = [torch.empty(clen, **f64) for _ in range(nb)] if not self.is_last else []
        self._stage = ([torch.empty(clen, dtype=local[0].dtype, device=self.dev) for _ in range(nb)]
                       if not self.is_last else [])
        corrupted = {m for m in (corruptions or {}) if m not in failures}
        assign = plan.assign.cpu().numpy() if hasattr(plan.assign, "cpu") else np.asarray(plan.assign)
        runs = _special_ranges(assign, self.P, failures, corrupted) if (corrupted or len(failures) >= 2) else []
        self.special_runs = runs
        if runs:
            tab = []
            off = 0
            for lo, hi in runs:
                tab.append((lo, hi, off))
                off += hi - lo
            self._ranges = torch.tensor(tab, dtype=torch.int64, device=self.dev)
            self._packed = torch.empty(off, dtype=local[0].dtype, device=self.dev)
        # fallback values come from the lowest alive miner when no fallback is given
        self.fb_owner = None
        self._fb_buf = None
        self._needs_fb = bool(fallback is None and self.alive and runs)
        if self._needs_fb:
            m0 = self.alive[0]
            self.fb_owner = next(r for r in range(G) if sum(self.counts[: r + 1]) > m0)
            if self.is_last and self.fb_owner != self.rank:
                self._fb_buf = torch.empty_like(local[0])
        self.job = None
        if self.is_last:
            reps = [None] * self.n
            for i, t in enumerate(local):
                reps[self.offset + i] = t
            fb_src = None
            if self._needs_fb:
                fb_src = self._fb_buf if self._fb_buf is not None else reps[self.alive[0]]
            self.job = self.ops.make_job(reps, plan, failures=failures, corruptions=corruptions, fallback=fallback,
                                         fallback_src=fb_src, scatter_back=True, want_merged=want_merged,
                                         tolerance=tolerance, n_div=len(self.alive))
        S, n = plan.n_shards, self.n
        self._res_bytes = 8 * n * n + 4 * S + S + n  # entries | source | status | flagged (aligned)
        self.status = torch.empty(S, dtype=torch.uint8, device=self.dev)
        self.flagged = torch.empty(n, dtype=torch.uint8, device=self.dev)
        self.source = torch.empty(S, dtype=torch.int32, device=self.dev)
        self.entries = torch.empty((n, n), dtype=torch.float64, device=self.dev)
        self.merged = torch.empty(self.P, **f64) if want_merged else None

    def _comm_dev(self):
        return self.dev if dist.get_backend() == "nccl" else torch.device("cpu")

    def _chunks(self):
        return [(b, min(b + self.chunk, self.P)) for b in range(0, self.P, self.chunk)]

    # -- one round -----------------------------------------------------------
    def _step_ops(self, t: int, K: int):
        """P2P operations of global step t on this rank (see the schedule in run())."""
        g, Z = self.rank, self.world - 1  # Z: last rank
        nb = 3
        ops = []

        def chunk(c):
            b, e = c * self.chunk, min((c + 1) * self.chunk, self.P)
            return e - b

        if g >= 1:  # running sums of chunk c arrive from g-1
            c = t - 2 * g + 1
            if 0 <= c < K:
                ops.append(dist.P2POp(dist.irecv, self._inb[c % nb][: chunk(c)], g - 1))
        if g < Z:  # ... and leave for g+1 one step after they were computed
            c = t - 2 * g - 1
            if 0 <= c < K:
                ops.append(dist.P2POp(dist.isend, self._outb[c % nb][: chunk(c)], g + 1))
        if g == Z and Z > 0:  # final chunk c enters the relay ring Z -> 0 -> 1 -> ... -> Z-1
            c = t - 2 * Z - 1
            if 0 <= c < K:
                b = c * self.chunk
                ops.append(dist.P2POp(dist.isend, self.local[0][b:b + chunk(c)], 0))
        if g < Z:
            c = t - 2 * Z - 1 - g
            if 0 <= c < K:
                ops.append(dist.P2POp(dist.irecv, self._stage[c % nb][: chunk(c)], Z if g == 0 else g - 1))
            c = t - 2 * Z - 2 - g
            if g + 1 < Z and 0 <= c < K:
                ops.append(dist.P2POp(dist.isend, self._stage[c % nb][: chunk(c)], g + 1))
        return ops

    def run(self) -> "ShardedButterflyMerge":
        """One merge round.

        Systolic schedule on ONE communicator (every rank issues its NCCL work in
        the same global step order, so nothing can deadlock across communicators):
        rank g computes chain chunk c at step c + 2g and sends it at step c + 2g + 1,
        while it computes chunk c + 1; the last rank Z reduces chunk c at step c + 2Z
        and starts chunk c of the final vector round the relay ring Z -> 0 -> ... ->
        Z-1 at step c + 2Z + 1; rank g fans chunk c out into its replicas and
        forwards it one step after receiving it.  Communication of step t (NCCL
        stream) overlaps computation of step t (current stream).
        """
        g, G = self.rank, self.world
        Z = G - 1  # last rank
        K = len(self._chunks())
        nb = 3
        T = K + 3 * Z + 1 if G > 1 else K
        # fallback values (the lowest alive miner's replica) for the late shards,
        # moved before the fan-out below overwrites that replica
        if self._needs_fb and self.fb_owner != Z:
            if g == self.fb_owner:
                self.ops.gather_ranges(self.local[self.alive[0] - self.offset], self._packed, self._ranges)
                dist.send(self._packed, dst=Z)
            elif self.is_last:
                dist.recv(self._packed, src=self.fb_owner)
                self.ops.scatter_ranges(self._packed, [self._fb_buf], self._ranges)
        pending = []
        for t in range(T):
            for w in pending:  # data received at step t-1 is needed now
                w.wait()
            ops = self._step_ops(t, K) if G > 1 else []
            pending = dist.batch_isend_irecv(ops) if ops else []
            c = t - 2 * g  # chain / reduce
            if 0 <= c < K:
                b, e = c * self.chunk, min((c + 1) * self.chunk, self.P)
                acc_in = self._inb[c % nb][: e - b] if g > 0 else None
                if self.is_last:
                    self.job.reduce_range(b, e, acc_in=acc_in)
                else:
                    self.ops.chain(self.local_alive, acc_in, self._outb[c % nb][: e - b], b, e)
            c = t - 2 * Z - 2 - g  # fan-out of the final vector
            if g < Z and 0 <= c < K:
                b, e = c * self.chunk, min((c + 1) * self.chunk, self.P)
                self.ops.fanout(self._stage[c % nb][: e - b], [x[b:e] for x in self.local])
        for w in pending:
            w.wait()

        last = Z

        # finish on the last rank, then the per-shard results and the late shards
        res = torch.empty(self._res_bytes, dtype=torch.uint8, device=self._comm_dev())
        if self.is_last:
            self.job.run(L.PHASE_FINISH)
            parts = [self.job.entries.reshape(-1).view(torch.uint8), self.job.source.view(torch.uint8),
                     self.job.status.view(torch.uint8), self.job.flagged.view(torch.uint8)]
            res.copy_(torch.cat([p.to(res.device) for p in parts]))
            if self.special_runs:
                self.ops.gather_ranges(self.local[0], self._packed, self._ranges)
        if G > 1:
            dist.broadcast(res, src=last)
            if self.special_runs:
                dist.broadcast(self._packed, src=last)
                if not self.is_last:
                    self.ops.scatter_ranges(self._packed, self.local, self._ranges)
            if self.want_merged:
                if self.is_last:
                    self.merged.copy_(self.job.merged)
                dist.broadcast(self.merged, src=last)
        elif self.want_merged:
            self.merged.copy_(self.job.merged)
        self._unpack(res)
        return self

    def _unpack(self, res):
        S, n = self.plan.n_shards, self.n
        res = res.to(self.dev)
        o = 8 * n * n
        self.entries.copy_(res[:o].view(torch.float64).reshape(n, n))
        self.source.copy_(res[o:o + 4 * S].view(torch.int32))
        o += 4 * S
        self.status.copy_(res[o:o + S])
        self.flagged.copy_(res[o + S:o + S + n])

    def launches_per_run(self) -> int:
        """Our kernels per round on this rank (bench.py gpu_launches)."""
        k = len(self._chunks())
        if self.is_last:
            fin = self.job.launches_per_run() - 3  # setup + finish kernels beyond the per-chunk reduces
            return k + 2 + fin + (1 if self.special_runs else 0)
        return 2 * k + (1 if self.special_runs else 0)

    def bytes_per_round(self) -> dict:
        """Algorithmic HBM and NVLink bytes of this rank for one round."""
        s = self.local[0].element_size()
        hbm = (len(self.local_alive) + len(self.local)) * self.P * s
        nvl_in = (8 * self.P if self.rank > 0 else 0) + (s * self.P if not self.is_last else 0)
        return {"hbm": hbm, "nvlink_in": nvl_in}
