"""Device-native butterfly merge: replicas resident in HBM, merged in place.

This is the B200 form of the reference's merge round (run_all_reduce,
butterfly.py:161-295) plus the orchestrator's adoption of the merged weights
by every miner (orchestrator.py:581-590): one call reduces every shard over
the alive replicas, checks the redundant copies, and scatters the adopted
slices back into each miner's own parameter buffer.

* ``DevicePlan``       — the GPU index map (plan_shards, butterfly.py:84-114)
* ``Corruption``       — GPU-native deceptive-miner descriptors (butterfly.py:232-233)
* ``ButterflyMerge``   — a prepared merge over fixed replicas; ``run()`` issues
                         the kernels on the current stream (CUDA-graph capturable)
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import errors


def _stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the butterfly merge runs on a CUDA device; none is visible (no CPU fallback)")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def n_shards(n_miners: int, redundancy: int = 2) -> int:
    return int(L.lib().bfly_n_shards(n_miners, redundancy))


class DevicePlan:
    """Shard plan built on the device by k_plan (bit-identical to plan_shards).

    ``assign`` is an int32 [S, r] tensor of ascending miner indices per shard and
    ``perm`` the int64 shard -> combination-rank permutation (Generator.permutation,
    simkernel.py:237-238).  Bounds are closed-form (butterfly.py:101-107).
    """

    def __init__(self, n_miners: int, payload_len: int, seed: int, redundancy: int = 2, device=None,
                 stream=None):
        dev = _require_cuda(device)
        self.n_miners, self.redundancy, self.payload_len, self.seed = n_miners, redundancy, payload_len, seed
        S = n_shards(n_miners, redundancy) if n_miners >= redundancy >= 2 else 0
        self.n_shards = S
        self.assign = torch.empty((max(S, 1), redundancy), dtype=torch.int32, device=dev)
        self.perm = torch.empty(max(S, 1), dtype=torch.int64, device=dev)
        k0, k1 = L.philox_key(seed, "shard-plan")
        with torch.cuda.device(dev):
            L.check(L.lib().bfly_plan_device(n_miners, redundancy, payload_len, k0, k1, self.perm.data_ptr(),
                                             self.assign.data_ptr(), _stream_handle(stream)))
        self.assign = self.assign[:S]
        self.perm = self.perm[:S]

    @classmethod
    def from_assignment(cls, assignment, n_miners: int, payload_len: int, device=None) -> "DevicePlan":
        """Upload a host plan (e.g. a ShardPlan's assignment tuples)."""
        dev = _require_cuda(device)
        self = cls.__new__(cls)
        a = np.asarray(assignment, dtype=np.int32)
        self.n_miners, self.redundancy, self.payload_len, self.seed = n_miners, a.shape[1], payload_len, None
        self.n_shards = a.shape[0]
        self.assign = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self.perm = None
        return self

    def bounds(self) -> np.ndarray:
        S, P = self.n_shards, self.payload_len
        base, rem = divmod(P, S)
        idx = np.arange(S + 1, dtype=np.int64)
        return idx * base + np.minimum(idx, rem)


@dataclass(frozen=True)
class Corruption:
    """A deceptive assignee's transformation of its shard reduction, applied on the GPU.

    kinds: "add" (mean + a), "scale" (mean * a), "noise" (a * (2u - 1)) and
    "noise_add" (mean + a * (2u - 1)), where u is word e of Philox4x64-10 keyed
    by ``key`` for global element e — counter-based, so miners sharing a key
    (colluders) produce identical copies.

    Portability of the decision: the reference adopts a pair of copies when
    ``agreement == 1.0``, which holds when max|a - b| <= tolerance OR when the clamped
    cosine rounds to exactly 1.0.  The second clause depends on the order of the dot
    products (the reference's BLAS ddot; fixed-order trees here), so for copies (nearly)
    parallel to the honest mean — a positive ``scale``, an ``add`` tiny against the mean,
    one noise key at two amplitudes — the GPU and the reference may decide differently.
    Decisions are bit-exact for corruptions that move the copy off that direction
    (``noise``, ``noise_add`` / ``add`` beyond the tolerance, a negative ``scale``).
    """

    kind: str
    a: float
    key: tuple = (0, 0)

    _KINDS = {"add": L.CORR_ADD, "scale": L.CORR_SCALE, "noise": L.CORR_NOISE, "noise_add": L.CORR_NOISE_ADD}

    def code(self) -> int:
        try:
            return self._KINDS[self.kind]
        except KeyError:
            raise errors.InvalidArgumentError(f"unknown corruption kind {self.kind!r}") from None

    def struct(self) -> L.Corruption:
        return L.Corruption(self.code(), 0, float(self.a), int(self.key[0]), int(self.key[1]))

    @staticmethod
    def add(c: float) -> "Corruption":
        return Corruption("add", c)

    @staticmethod
    def scale(c: float) -> "Corruption":
        return Corruption("scale", c)

    @staticmethod
    def noise(amp: float, key) -> "Corruption":
        return Corruption("noise", amp, tuple(key))

    @staticmethod
    def noise_add(amp: float, key) -> "Corruption":
        return Corruption("noise_add", amp, tuple(key))


_DTYPES = {torch.float32: L.F32, torch.bfloat16: L.BF16, torch.float64: L.F64WIRE}


def _ptr_table(tensors, dev) -> torch.Tensor:
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64).to(dev)


def corruption_table(n: int, corruptions: dict | None, host_kinds=()) -> bytes:
    table = (L.Corruption * n)()
    for m, c in (corruptions or {}).items():
        table[m] = c.struct()
    for m in host_kinds:
        table[m] = L.Corruption(L.CORR_HOST, 0, 0.0, 0, 0)
    return bytes(table)


class ButterflyMerge:
    """One prepared merge round over device-resident replicas.

    replicas     list of N entries in miner-index order (the reference's
                 sorted(payloads), butterfly.py:189): contiguous 1-D CUDA tensors
                 (float32 wire values, bfloat16, or float64 payloads rounded to the
                 fp32 wire on load).  None marks a failed miner or — with
                 ``remote_sum`` — a miner resident on another GPU.
    plan         DevicePlan (or any object with .assign [S, r] int32 CUDA tensor).
    failures     miner indices that dropped before upload (butterfly.py:167,203).
    corruptions  {miner index: Corruption}; ``host_miners`` lists miners whose
                 copies the caller supplies to ``run(host_copies=...)``.
    fallback     optional fp64 [P] CUDA tensor (butterfly.py:169,268-273).
    fallback_src replica supplying fallback values when ``fallback`` is None
                 (default: the lowest alive resident replica).
    scatter_back write the adopted slices into every resident replica in place.
    want_merged  also produce the fp64 merged vector (MergeResult.merged).
    keep_means   keep special-shard means in a separate workspace (read back by
                 the drop-in shim for the store's lazy blobs).
    remote_sum   multi-GPU chain: the running sums of the miners on earlier GPUs
                 arrive through ``reduce_range(acc_in=...)`` and the mean divides
                 by ``n_div`` = alive miners on all GPUs.
    """

    def __init__(self, replicas, plan, *, failures=(), corruptions=None, host_miners=(), fallback=None,
                 fallback_src=None, scatter_back: bool = True, want_merged: bool = False,
                 keep_means: bool = False, tolerance: float = 1e-6, remote_sum: bool = False,
                 n_div: int | None = None):
        n = len(replicas)
        if n != plan.n_miners:
            raise errors.ShapeError(f"plan expects {plan.n_miners} payloads, got {n}")
        failures = set(int(m) for m in failures)
        present = [t for t in replicas if t is not None]
        if not remote_sum and any(t is None for m, t in enumerate(replicas) if m not in failures):
            raise errors.InvalidArgumentError("only failed miners may be passed as None")
        if not present:
            raise errors.InvalidArgumentError("no replica tensors given")
        dev = present[0].device
        if dev.type != "cuda":
            raise RuntimeError("replicas must be CUDA tensors (no CPU fallback)")
        lengths = {int(t.numel()) for t in present}
        if len(lengths) != 1:
            raise errors.ShapeError(f"payload lengths differ: {sorted(lengths)}")
        (P,) = lengths
        if P != plan.payload_len:
            raise errors.ShapeError(f"plan covers {plan.payload_len} elements but payloads have {P}")
        dtypes = {t.dtype for t in present}
        if len(dtypes) != 1 or next(iter(dtypes)) not in _DTYPES:
            raise errors.InvalidArgumentError(f"replicas must share one of {list(_DTYPES)}; got {dtypes}")
        for t in present:
            if not t.is_contiguous() or t.device != dev:
                raise errors.InvalidArgumentError("replicas must be contiguous and on one device")
        if fallback is not None and int(fallback.numel()) != P:
            raise errors.ShapeError("fallback length does not match payloads")
        self.n, self.P, self.dev = n, P, dev
        self.r = plan.redundancy
        self.S = plan.n_shards
        self.dtype = _DTYPES[next(iter(dtypes))]
        self.elem_size = next(iter(dtypes)).itemsize
        self.alive = [m for m in range(n) if m not in failures]
        self.local_alive = [m for m in self.alive if replicas[m] is not None]
        self.resident = [m for m in range(n) if replicas[m] is not None]
        self.replicas = list(replicas)
        self.plan = plan
        self.remote_sum = remote_sum
        self.n_div = int(n_div) if n_div is not None else len(self.alive)

        self._src = _ptr_table([replicas[m] for m in self.local_alive], dev) if self.local_alive else None
        self._dst = _ptr_table([replicas[m] for m in self.resident], dev) if scatter_back else None
        failed = np.zeros(n, dtype=np.uint8)
        for m in failures:
            failed[m] = 1
        self._failed = torch.from_numpy(failed).to(dev)
        self._corr = torch.frombuffer(bytearray(corruption_table(n, corruptions, host_miners)),
                                      dtype=torch.uint8).to(dev)
        self.fallback = None if fallback is None else fallback.to(dev, torch.float64).contiguous()
        self.fallback_src = fallback_src
        self.status = torch.empty(self.S, dtype=torch.uint8, device=dev)
        self.entries = torch.empty((n, n), dtype=torch.float64, device=dev)
        self.flagged = torch.empty(n, dtype=torch.uint8, device=dev)
        self.source = torch.empty(self.S, dtype=torch.int32, device=dev)
        self.merged = torch.empty(P, dtype=torch.float64, device=dev) if want_merged else None
        self.special = bool({m for m in (corruptions or {}) if m not in failures}) or bool(host_miners)
        # a shard is lost only if all of its r assignees failed
        self.maybe_lost = len(failures) >= self.r
        self.means = (torch.empty(P, dtype=torch.float64, device=dev)
                      if self.special and (keep_means or not want_merged) else None)
        if self.means is None and self.merged is None:  # never written without special shards
            self.means = torch.empty(1, dtype=torch.float64, device=dev)
        scratch_bytes = int(L.lib().bfly_merge_scratch_bytes(n, self.r, P))
        self._scratch = torch.empty(max(scratch_bytes, 1), dtype=torch.uint8, device=dev)

        a = L.MergeArgs()
        a.n_miners, a.redundancy, a.payload_len, a.n_shards = n, self.r, P, self.S
        a.dtype, a.n_alive = self.dtype, len(self.local_alive)
        a.d_assign = plan.assign.data_ptr()
        a.d_src = self._src.data_ptr() if self._src is not None else None
        a.d_failed = self._failed.data_ptr()
        a.d_corr = self._corr.data_ptr()
        a.d_dst = self._dst.data_ptr() if self._dst is not None else None
        a.n_dst = len(self.resident) if scatter_back else 0
        a.d_fallback = self.fallback.data_ptr() if self.fallback is not None else None
        a.d_merged = self.merged.data_ptr() if self.merged is not None else None
        a.d_ws = self.means.data_ptr() if self.means is not None else None
        a.d_status = self.status.data_ptr()
        a.d_entries = self.entries.data_ptr()
        a.d_flagged = self.flagged.data_ptr()
        a.d_source = self.source.data_ptr()
        a.d_scratch = self._scratch.data_ptr()
        a.scratch_bytes = scratch_bytes
        a.tolerance = float(tolerance)
        a.n_div = self.n_div
        a.d_fallback_src = (None if fallback_src is None else
                            fallback_src if isinstance(fallback_src, int) else fallback_src.data_ptr())
        self._args = a
        self._host_copies = None
        self._acc_in = None
        self._graph = None  # CUDA graph of one round (capture())

    def set_fallback(self, fallback: torch.Tensor | None) -> "ButterflyMerge":
        """Replace the fp64 fallback vector (butterfly.py:169,268-273) for later phases."""
        if fallback is not None and int(fallback.numel()) != self.P:
            raise errors.ShapeError("fallback length does not match payloads")
        self.fallback = None if fallback is None else fallback.to(self.dev, torch.float64).contiguous()
        self._args.d_fallback = self.fallback.data_ptr() if self.fallback is not None else None
        return self

    def _call(self, stream):
        with torch.cuda.device(self.dev):
            L.check(L.lib().bfly_merge(ctypes.byref(self._args), _stream_handle(stream)))

    def run(self, phase: int = L.PHASE_ALL, host_copies: torch.Tensor | None = None, stream=None) -> "ButterflyMerge":
        """Issue the merge kernels on ``stream`` (default: current stream). Asynchronous."""
        if self.remote_sum and phase not in (L.PHASE_FINISH, L.PHASE_CHECK):
            raise errors.InvalidArgumentError("a chained merge reduces through reduce_range(acc_in=...)")
        if host_copies is not None:
            self._host_copies = host_copies
            self._args.d_host_copies = host_copies.data_ptr()
        requested = phase
        if phase == L.PHASE_FINISH and not self.needs_finish():
            phase = L.PHASE_CHECK  # every shard is fast: only non-finite means can fall back
        if phase == L.PHASE_ALL and not self.needs_finish():
            phase = L.PHASE_REDUCE  # every shard fast: k_classify wrote their results (REDUCE checks means)
        self._args.phase = phase
        self._args.d_acc_in = None
        self._args.elem_begin = self._args.elem_end = 0
        if self._graph is not None and requested == L.PHASE_ALL and host_copies is None:
            self._replay(stream)
        else:
            self._call(stream)
        return self

    def capture(self) -> "ButterflyMerge":
        """Record one whole round (phase ALL) as a CUDA graph; later ``run()`` calls replay
        it — one launch instead of 4-8, which matters for small payloads.  The graph
        reads the same buffers each replay, so the replicas may be refilled in place
        between rounds; the plan, failures and corruptions are fixed at construction."""
        if self.remote_sum:
            raise errors.InvalidArgumentError("a chained merge is issued chunk by chunk; capture the single-GPU job")
        self._graph = None
        self.run()  # warm-up outside the capture (function attributes, lazy module loading)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
            self._args.phase = L.PHASE_ALL if self.needs_finish() else L.PHASE_REDUCE
            self._call(None)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        self._graph = g
        return self

    def _replay(self, stream):
        if stream is None:
            self._graph.replay()
            return
        with torch.cuda.stream(stream):
            self._graph.replay()

    def reduce_range(self, begin: int, end: int, acc_in=None, stream=None, dst_table: tuple | None = None):
        """REDUCE elements [begin, end) — call with begin == 0 first in every round.

        ``acc_in`` holds the running fp64 sums of the miners on earlier GPUs (a
        float64 tensor covering [begin, end), or a raw device pointer into peer
        memory).  ``dst_table`` = (device pointer, count) overrides the
        scatter-back targets for this call (the multi-GPU last rank adds the next
        GPU's inbox, biased by -begin, so the final chunk is pushed over NVLink)."""
        if isinstance(acc_in, torch.Tensor):
            if acc_in.dtype != torch.float64 or acc_in.numel() < end - begin:
                raise errors.ShapeError("acc_in must be float64 covering [begin, end)")
            self._acc_in = acc_in
            acc_in = acc_in.data_ptr()
        self._args.phase = L.PHASE_REDUCE
        self._args.d_acc_in = acc_in if acc_in else None
        self._args.elem_begin, self._args.elem_end = int(begin), int(end)
        saved = (self._args.d_dst, self._args.n_dst)
        if dst_table is not None:
            self._args.d_dst, self._args.n_dst = dst_table
        try:
            self._call(stream)
        finally:
            self._args.d_dst, self._args.n_dst = saved
        return self

    def run_finish_list(self, shards: torch.Tensor, stream=None):
        """FINISH for the shards listed in ``shards`` (int32 device tensor) only."""
        if shards.numel() == 0 or not self.needs_finish():
            return self
        a = self._args
        a.phase = L.PHASE_FINISH
        a.d_shard_list, a.n_shard_list = shards.data_ptr(), int(shards.numel())
        try:
            self._call(stream)
        finally:
            a.d_shard_list, a.n_shard_list = None, 0
        return self

    def run_finish_range(self, shard_begin: int, shard_end: int, stream=None, dst_table: tuple | None = None):
        """FINISH (compare, decide, adopt / fall back, scatter back) for shards
        [shard_begin, shard_end) only."""
        if shard_end <= shard_begin or not self.needs_finish():
            return self
        a = self._args
        saved = (a.d_dst, a.n_dst)
        a.phase = L.PHASE_FINISH
        a.shard_begin, a.shard_end = int(shard_begin), int(shard_end)
        if dst_table is not None:
            a.d_dst, a.n_dst = dst_table
        try:
            self._call(stream)
        finally:
            a.d_dst, a.n_dst = saved
            a.shard_begin = a.shard_end = 0
        return self

    def needs_finish(self) -> bool:
        # r = 3: a pair's entry is the minimum over the shards it shares (k_entries3)
        return self.special or self.maybe_lost or self.r > 2

    def fast_shards(self) -> np.ndarray:
        """Shards with >= 1 surviving assignee, none of them corrupted (k_classify's kFast)."""
        assign = self.plan.assign.cpu().numpy()
        failed = self._failed.cpu().numpy().astype(bool)
        kinds = self._corr_kinds()
        alive = ~failed[assign]
        corrupt = (kinds[assign] != L.CORR_NONE) & alive
        return np.flatnonzero(alive.any(axis=1) & ~corrupt.any(axis=1))

    def _corr_kinds(self) -> np.ndarray:
        raw = self._corr.cpu().numpy().tobytes()
        size = ctypes.sizeof(L.Corruption)
        return np.array([int.from_bytes(raw[m * size:m * size + 4], "little", signed=True) for m in range(self.n)],
                        dtype=np.int32)

    def nonfinite_shards(self) -> np.ndarray:
        """Fast shards decided a disagreement because their mean is NaN / Inf somewhere
        (k_nonfinite; the reference's agreement of two NaN copies is NaN,
        butterfly.py:127-133,255).  Reads the status back (synchronises)."""
        fast = self.fast_shards()
        status = self.status.cpu().numpy()
        return fast[status[fast] != L.MERGED]

    # number of our kernels one run() launches (reported by bench.py as gpu_launches)
    def launches_per_run(self) -> int:
        # k_fill_nan, k_classify, [k_reduce], k_nonfinite + [k_stats, k_decide, [k_entries3], k_apply]
        fin = (3 + (1 if self.r > 2 else 0)) if self.needs_finish() else 0
        return 3 + (1 if self.local_alive or self.remote_sum else 0) + fin
