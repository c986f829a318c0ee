"""Drop-in replacement for ``iota_sim.butterfly`` (pkg/src/iota_sim/butterfly.py).

Same names, signatures, types, error classes and observable results as the
reference module's public API (butterfly.py:22-35), with the merge round
executed by the B200 kernels of libbfly.so:

* ``plan_shards``     — the index map in native code (bfly_plan_host; the same
                         header also runs on the GPU, see device.DevicePlan);
* ``run_all_reduce``  — payloads to HBM, then the device merge (reduce, compare,
                         decide, adopt) and the merged vector back; Python
                         corruption callables are honoured in the reference's
                         call order through the REDUCE/FINISH phases;
* ``agreement`` / ``mean_reducer`` — the same reductions on the GPU;
* the blob-store meter is applied in closed form and the
  store receives the same keys, with lazily materialised contents.

There is no CPU fallback: without a CUDA device these functions raise.
"""

from __future__ import annotations

import ctypes
import json
import math
import sys
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .device import ButterflyMerge, Corruption, DevicePlan, _require_cuda, _stream_handle
from .errors import DegenerateShardsError, InvalidArgumentError, ShapeError, TooFewMinersError
from .simkernel import BlobStore, RngStream

__all__ = [
    "PairSet",
    "ShardPlan",
    "AgreementMatrix",
    "MergeResult",
    "enumerate_pairs",
    "plan_shards",
    "agreement",
    "run_all_reduce",
    "valid_shard_fraction",
    "per_miner_transfer",
    "monte_carlo_resilience",
    "mean_reducer",
    "Corruption",
]

BYTES_PER_WEIGHT = 4  # the wire format is "<f4" (butterfly.py:37)


def _reference_types():
    """The caller's iota_sim.butterfly result types, when that package is importable:
    the drop-in then returns the reference's own PairSet / ShardPlan / AgreementMatrix /
    MergeResult (isinstance checks and equality in callers keep working)."""
    mod = sys.modules.get("iota_sim.butterfly")
    if mod is None or mod.__name__ == __name__:
        try:
            import iota_sim.butterfly as mod  # noqa: F811
        except Exception:
            return None
    names = ("PairSet", "ShardPlan", "AgreementMatrix", "MergeResult")
    if getattr(mod, "__name__", None) == __name__ or not all(hasattr(mod, n) for n in names):
        return None
    return mod


_ref_types = _reference_types()

if _ref_types is not None:
    PairSet = _ref_types.PairSet
    ShardPlan = _ref_types.ShardPlan
    AgreementMatrix = _ref_types.AgreementMatrix
    MergeResult = _ref_types.MergeResult
else:
    @dataclass(frozen=True)
    class PairSet:
        n_miners: int
        pairs: tuple  # (i, j), i < j, lexicographic

    @dataclass(frozen=True)
    class ShardPlan:
        """Shard -> miner-pair bijection and element bounds (butterfly.py:46-73)."""

        pair_set: PairSet
        assignment: tuple
        bounds: tuple
        bytes_per_weight: int
        seed: int

        @property
        def n_shards(self) -> int:
            return len(self.assignment)

        def byte_bounds(self, shard_idx: int) -> tuple[int, int]:
            lo, hi = self.bounds[shard_idx]
            return lo * self.bytes_per_weight, hi * self.bytes_per_weight

        def shards_of(self, miner: int) -> list[int]:
            return [s for s, members in enumerate(self.assignment) if miner in members]

        def metadata(self) -> bytes:
            """JSON sidecar [[shard, start_byte, length_bytes], ...] (butterfly.py:67-73)."""
            rows = [[s, lo * self.bytes_per_weight, (hi - lo) * self.bytes_per_weight]
                    for s, (lo, hi) in enumerate(self.bounds)]
            return json.dumps(rows).encode()

    @dataclass(frozen=True)
    class AgreementMatrix:
        n_miners: int
        entries: np.ndarray

    @dataclass
    class MergeResult:
        merged: np.ndarray
        shard_status: list
        agreement_matrix: AgreementMatrix
        flagged: set = field(default_factory=set)


def _types_of(obj):
    """(ShardPlan, AgreementMatrix, MergeResult) of the module that defined ``obj``'s
    type (the caller's plan or pair set), else this module's."""
    mod = sys.modules.get(type(obj).__module__)
    if mod is not None and all(hasattr(mod, n) for n in ("ShardPlan", "AgreementMatrix", "MergeResult")):
        return mod.ShardPlan, mod.AgreementMatrix, mod.MergeResult
    return ShardPlan, AgreementMatrix, MergeResult


def enumerate_pairs(n: int) -> PairSet:
    """All C(n, 2) unordered miner pairs, lexicographic (butterfly.py:76-81)."""
    if n < 2:
        raise TooFewMinersError(f"need at least 2 miners, got {n}")
    return PairSet(n_miners=n, pairs=tuple((i, j) for i in range(n) for j in range(i + 1, n)))


def _is_mean_reducer(reducer) -> bool:
    """This module's mean_reducer or the reference's (butterfly.py:156-158): the only
    reducer the device merge implements."""
    return reducer is mean_reducer or (getattr(reducer, "__name__", "") == "mean_reducer"
                                       and getattr(reducer, "__module__", "") == "iota_sim.butterfly")


def _host_plan(n: int, r: int, payload_len: int, seed: int):
    S = int(L.lib().bfly_n_shards(n, r))
    assign = np.empty((max(S, 1), r), dtype=np.int32)
    bounds = np.empty(max(S, 0) + 1, dtype=np.int64)
    k0, k1 = L.philox_key(seed, "shard-plan")
    L.check(L.lib().bfly_plan_host(n, r, payload_len, k0, k1, assign.ctypes.data, bounds.ctypes.data))
    return assign[:S], bounds


def _lexicographic_pairs(pairs, n: int) -> bool:
    if len(pairs) != n * (n - 1) // 2:
        return False
    k = 0
    for i in range(n):
        for j in range(i + 1, n):
            if tuple(pairs[k]) != (i, j):
                return False
            k += 1
    return True


def plan_shards(pair_set: PairSet, payload_len: int, bytes_per_weight: int, seed: int) -> ShardPlan:
    """Seeded shard -> pair bijection with near-equal bounds (butterfly.py:84-114).

    The pairs of ``enumerate_pairs`` go through the native index map (bfly_plan_host,
    the same code as the GPU's k_plan); any other PairSet is permuted as the reference
    does, ``pairs[order[s]]`` with ``order = RngStream(seed, "shard-plan").permutation``
    (bfly_permutation_host).  The plan is an instance of the pair set's module's
    ShardPlan (the reference's when the caller passes its own PairSet)."""
    n_shards = len(pair_set.pairs)
    if payload_len < n_shards:
        raise DegenerateShardsError(f"payload of {payload_len} elements cannot fill {n_shards} shards")
    plan_type = _types_of(pair_set)[0]
    if _lexicographic_pairs(pair_set.pairs, pair_set.n_miners):
        assign, bounds = _host_plan(pair_set.n_miners, 2, payload_len, seed)
        assignment = tuple(tuple(p) for p in assign.tolist())
    else:
        order = np.empty(max(n_shards, 1), dtype=np.int64)
        k0, k1 = L.philox_key(seed, "shard-plan")
        L.check(L.lib().bfly_permutation_host(n_shards, k0, k1, order.ctypes.data))
        assignment = tuple(pair_set.pairs[k] for k in order[:n_shards].tolist())
        base, rem = divmod(payload_len, n_shards)
        idx = np.arange(n_shards + 1, dtype=np.int64)
        bounds = idx * base + np.minimum(idx, rem)
    b = bounds.tolist()
    return plan_type(pair_set=pair_set, assignment=assignment, bounds=tuple(zip(b[:-1], b[1:])),
                     bytes_per_weight=bytes_per_weight, seed=seed)


def _to_device_f64(x, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(dev, torch.float64).contiguous().reshape(-1)
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).reshape(-1)).to(dev, non_blocking=True)


def agreement(a, b, tolerance: float = 1e-6) -> float:
    """Agreement of two duplicate reductions (butterfly.py:117-133), on the GPU."""
    a_shape = tuple(a.shape) if hasattr(a, "shape") else np.shape(a)
    b_shape = tuple(b.shape) if hasattr(b, "shape") else np.shape(b)
    if a_shape != b_shape:
        raise ShapeError(f"reduction shapes differ: {a_shape} vs {b_shape}")
    dev = _require_cuda()
    da, db = _to_device_f64(a, dev), _to_device_f64(b, dev)
    n = int(da.numel())
    chunks = max(1, -(-n // 16384))
    scratch = torch.empty(4 * chunks, dtype=torch.float64, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    L.check(L.lib().bfly_agreement(da.data_ptr(), db.data_ptr(), n, float(tolerance), out.data_ptr(),
                                   scratch.data_ptr(), scratch.numel() * 8, _stream_handle()))
    return float(out.item())


def mean_reducer(stack):
    """Element-wise mean over axis 0 in numpy's order (butterfly.py:156-158), on the GPU."""
    dev = _require_cuda()
    host = not isinstance(stack, torch.Tensor)
    arr = np.asarray(stack, dtype=np.float64) if host else stack
    rows = int(arr.shape[0])
    width = int(np.prod(arr.shape[1:])) if len(arr.shape) > 1 else 1
    ds = _to_device_f64(arr, dev)
    out = torch.empty(width, dtype=torch.float64, device=dev)
    L.check(L.lib().bfly_mean_rows(ds.data_ptr(), rows, width, out.data_ptr(), _stream_handle()))
    out = out.reshape(tuple(arr.shape[1:]))
    return out.cpu().numpy() if host else out


# ---------------------------------------------------------------------------
# run_all_reduce
# ---------------------------------------------------------------------------


SNAPSHOT_STORE = False
"""Ownership of the store objects a round writes.

False (default): the weights objects are views of the caller's payload arrays and the
re-uploaded reductions of merged shards are views of the returned ``merged`` vector,
rendered as "<f4" bytes when first read (a ranged ``get`` converts only its range).
Changing a payload in place after the call therefore changes what the store returns.
Reductions that differ from ``merged`` (corrupted copies, shards whose mean is not
finite) are rendered into host bytes before the call returns; no object keeps device
memory of the round alive.

True: every object is snapshotted into bytes before the call returns, as the
reference's ``BlobStore.put`` copies them (simkernel.py:168) — at the reference's host
cost (N x 4P bytes per round)."""


class _LazyBlob:
    """Store object whose bytes are produced on first read (sizes are exact up front).

    A ranged read (``blob[a:b]``, what ``BlobStore.get(actor, key, start, length)``
    does) renders only that range when a ``part`` reader is given; anything else
    materialises the whole object once."""

    __slots__ = ("_n", "_make", "_data", "_part")

    def __init__(self, nbytes: int, make, part=None):
        self._n, self._make, self._data, self._part = nbytes, make, None, part

    def _bytes(self) -> bytes:
        if self._data is None:
            self._data = bytes(self._make())
            self._make = self._part = None
        return self._data

    def __len__(self):
        return self._n

    def __getitem__(self, item):
        if self._data is None and self._part is not None and isinstance(item, slice) and item.step in (None, 1):
            start, stop, _ = item.indices(self._n)
            return self._part(start, stop) if stop > start else b""
        return self._bytes()[item]

    def __bytes__(self):
        return self._bytes()

    def __eq__(self, other):
        return self._bytes() == bytes(other)

    __hash__ = None


def _wire_part(values, header: bytes = b""):
    """Ranged reader of ``header + values.astype("<f4")`` for a 1-D float vector (numpy or
    a tensor): only the elements under [start, stop) are converted."""
    h = len(header)

    def part(start: int, stop: int) -> bytes:
        out = header[start:stop] if start < h else b""
        a, b = max(start, h) - h, stop - h
        if b > a:
            e0, e1 = a // 4, (b + 3) // 4
            chunk = values[e0:e1]
            if isinstance(chunk, torch.Tensor):
                chunk = chunk.detach().to("cpu", torch.float64).numpy()
            raw = np.asarray(chunk, dtype=np.float64).astype("<f4").tobytes()
            out += raw[a - 4 * e0:b - 4 * e0]
        return out
    return part


def _wire_bytes(src) -> bytes:
    if isinstance(src, torch.Tensor):
        return src.detach().to("cpu", torch.float64).numpy().astype("<f4").tobytes()
    return np.asarray(src, dtype=np.float64).astype("<f4").tobytes()


def _wire_blob(values, nbytes: int):
    """Store object holding ``values.astype("<f4")`` (a view unless SNAPSHOT_STORE)."""
    if SNAPSHOT_STORE:
        return _wire_bytes(values)
    return _LazyBlob(nbytes, lambda: _wire_bytes(values), _wire_part(values))


def _meter(store, actor: str) -> object:
    if hasattr(store, "_meter_for"):
        return store._meter_for(actor)
    return store.meter.setdefault(actor, type("TransferMeter", (), {"bytes_uploaded": 0, "bytes_downloaded": 0})())


def _wire(store, nbytes: int) -> int:
    ratio = getattr(store, "wire_ratio", 1.0)
    return nbytes if ratio == 1.0 else math.ceil(nbytes / ratio)


def _payload_to_device(x, dev) -> tuple[torch.Tensor, int]:
    """Host fp64 payload (numpy, pinned or pageable) or device tensor -> device replica."""
    if isinstance(x, torch.Tensor):
        t = x.reshape(-1)
        if t.dtype not in (torch.float32, torch.float64, torch.bfloat16):
            t = t.to(torch.float64)
        return t.to(dev, non_blocking=True).contiguous(), len(t)
    a = np.asarray(x)
    if a.dtype != np.float64:
        a = a.astype(np.float64)
    a = np.ascontiguousarray(a).reshape(-1)
    return torch.from_numpy(a).to(dev, non_blocking=True), len(a)


def _runs(ranges):
    """Merge sorted [lo, hi) element ranges into maximal runs."""
    out = []
    for lo, hi in ranges:
        if out and out[-1][1] == lo:
            out[-1][1] = hi
        else:
            out.append([lo, hi])
    return out


def _classes(plan, failed: set, corrupted: set):
    """Per shard: "fast" (>= 1 survivor, none corrupted), "special" (a corrupted
    survivor) or "lost" (no survivor) — k_classify's classes."""
    out = []
    for members in plan.assignment:
        surv = [x for x in members if x not in failed]
        out.append("lost" if not surv else "special" if any(x in corrupted for x in surv) else "fast")
    return out


def _host_copies(job, plan, failed, callables, dev):
    """The reference's reduce-stage calls of the corruption callables (butterfly.py:219-233):
    shard ascending, assignee i then j, each on a fresh copy of the shard's fp64 mean.
    Only the special shards' means come back from the device and only their copies go
    up (one D2H / H2D per run of adjacent shards).  Returns ({(shard, assignee): output},
    device [2, P] copies)."""
    P = job.P
    host_reductions = {}
    copies = torch.zeros((2, P), dtype=torch.float64, device=dev)
    todo = [s for s, members in enumerate(plan.assignment)
            if any(x not in failed and x in callables for x in members)]
    runs = _runs([plan.bounds[s] for s in todo])
    means = {}
    for lo, hi in runs:  # one D2H per run of adjacent special shards
        means[lo] = job.means[lo:hi].cpu().numpy()
    run_of = {}
    for lo, hi in runs:
        for s in todo:
            a, b = plan.bounds[s]
            if lo <= a and b <= hi:
                run_of[s] = lo
    staged = {lo: np.zeros((2, hi - lo), dtype=np.float64) for lo, hi in runs}
    for s in todo:
        lo, hi = plan.bounds[s]
        r0 = run_of[s]
        mean = means[r0][lo - r0:hi - r0]
        members = plan.assignment[s]
        outs = {}
        for slot, x in enumerate(members):
            if x in failed or x not in callables:
                continue
            out = callables[x](mean.copy())
            host_reductions[(s, x)] = out
            outs[slot] = np.asarray(out, dtype=np.float64)
        surv = [slot for slot, x in enumerate(members) if x not in failed]
        shapes = {slot: (outs[slot].shape if slot in outs else (hi - lo,)) for slot in surv}
        if len(surv) == 2 and shapes[surv[0]] != shapes[surv[1]]:  # agreement(), butterfly.py:125-126
            raise ShapeError(f"reduction shapes differ: {shapes[surv[0]]} vs {shapes[surv[1]]}")
        for slot, arr in outs.items():
            # a broadcastable copy (a scalar, shape (1,)) merges as numpy assigns it (:263)
            staged[r0][slot, lo - r0:hi - r0] = np.broadcast_to(arr, (hi - lo,))
    for lo, hi in runs:  # one H2D per run
        copies[:, lo:hi].copy_(torch.from_numpy(staged[lo]))
    return host_reductions, copies


def run_all_reduce(store, payloads: dict, plan: ShardPlan, *, reducer=mean_reducer,
                   failures: frozenset | set = frozenset(), corruptions: dict | None = None,
                   fallback: np.ndarray | None = None, key_prefix: str = "merge",
                   agreement_tolerance: float = 1e-6, _device_merged: bool = False) -> MergeResult:
    """One merge round for a layer (butterfly.py:161-295), executed on the GPU.

    ``payloads`` maps miner id -> 1-D float64 payload (numpy; torch tensors on
    the device are accepted too).  ``failures`` / ``corruptions`` are keyed by
    index into sorted(payloads).  A corruption may be a reference-style callable
    fn(reduction) -> reduction (run on the host, in the reference's call order)
    or a ``Corruption`` descriptor (applied inside the kernels).  Returns the
    MergeResult type of the plan's module (the reference's for its own plans).
    """
    if not _is_mean_reducer(reducer):
        raise NotImplementedError("custom reducers cannot cross the C ABI; only mean_reducer is supported")
    corruptions = corruptions or {}
    n = plan.pair_set.n_miners
    miners = sorted(payloads)
    if len(miners) != n:
        raise ShapeError(f"plan expects {n} payloads, got {len(miners)}")
    lengths = {len(payloads[m]) for m in miners}
    if len(lengths) != 1:
        raise ShapeError(f"payload lengths differ: {sorted(lengths)}")
    (P,) = lengths
    if plan.bounds[-1][1] != P:
        raise ShapeError(f"plan covers {plan.bounds[-1][1]} elements but payloads have {P}")
    if fallback is not None and len(fallback) != P:
        raise ShapeError("fallback length does not match payloads")
    dev = _require_cuda()
    failed = set(int(m) for m in failures if 0 <= int(m) < n)
    alive = [m for m in range(n) if m not in failed]

    descriptors = {m: c for m, c in corruptions.items() if isinstance(c, Corruption) and m not in failed}
    callables = {m: c for m, c in corruptions.items() if not isinstance(c, Corruption) and m not in failed}

    # -- device merge ------------------------------------------------------
    reps = [None] * n
    pipelined = False
    hosts = None
    host_f64 = [m for m in alive if not isinstance(payloads[miners[m]], torch.Tensor)]
    if host_f64 and len(host_f64) == len(alive):
        # host payloads: the upload stage's "<f4" serialisation (butterfly.py:213) runs on
        # host threads into pinned staging, overlapped with the H2D copies (bfly_upload_wire)
        hosts = [np.ascontiguousarray(np.asarray(payloads[miners[m]], dtype=np.float64)).reshape(-1) for m in alive]
        wire = [torch.empty(P, dtype=torch.float32, device=dev) for _ in alive]
        h_ptrs = (ctypes.c_void_p * len(alive))(*[h.ctypes.data for h in hosts])
        d_ptrs = (ctypes.c_void_p * len(alive))(*[t.data_ptr() for t in wire])
        # without host callables the upload, the reduce and the copy of the merged
        # vector back run as one pipeline (bfly_merge_host) once the job exists
        pipelined = not callables
        if not pipelined:
            L.check(L.lib().bfly_upload_wire(h_ptrs, len(alive), P, d_ptrs, _UPLOAD_THREADS, _UPLOAD_BLOCK,
                                             _stream_handle()))
        for m, t in zip(alive, wire):
            reps[m] = t
        unmerged_possible = len(failed) >= 2 or bool(descriptors) or bool(callables)
        if fallback is None and unmerged_possible:
            # unmerged shards fall back to the lowest alive *fp64* payload (butterfly.py:270-271)
            fallback = hosts[0]
    else:
        for m in alive:
            reps[m], _ = _payload_to_device(payloads[miners[m]], dev)
    if alive:
        kinds = {reps[m].dtype for m in alive}
        if len(kinds) != 1:
            raise InvalidArgumentError("payloads must share one dtype")
    dplan = DevicePlan.from_assignment(plan.assignment, n, P, dev)
    fb = None if fallback is None else _to_device_f64(fallback, dev)
    if not alive:  # nothing uploaded: every shard is lost (only the length matters)
        reps[0] = torch.zeros(P, dtype=torch.float64, device=dev)
    job = ButterflyMerge(reps, dplan, failures=failed, corruptions=descriptors, host_miners=tuple(callables),
                         fallback=fb, scatter_back=False, want_merged=True, keep_means=True,
                         tolerance=agreement_tolerance)

    host_reductions = {}  # (shard, assignee) -> callable output
    early = False
    if callables:
        job.run(L.PHASE_REDUCE)
        host_reductions, copies = _host_copies(job, plan, failed, callables, dev)
        job.run(L.PHASE_FINISH, host_copies=copies)
    elif pipelined:
        # merged values stream back chunk by chunk unless FINISH may still change them
        early = not _device_merged and not job.needs_finish()
        merged_host = torch.empty(P, dtype=torch.float64, pin_memory=True) if early else None  # cached pinned
        L.check(L.lib().bfly_merge_host(h_ptrs, len(alive), P, d_ptrs, ctypes.byref(job._args),
                                        merged_host.data_ptr() if early else None, _merge_chunks(P),
                                        _UPLOAD_THREADS, _UPLOAD_BLOCK, _stream_handle()))
        if job.needs_finish():
            job.run(L.PHASE_FINISH)
    else:
        job.run(L.PHASE_ALL)

    if nonfinite_fallback_needed(job, plan, failed, set(descriptors) | set(callables)) and fb is None and alive:
        # fast shards whose mean is NaN / Inf somewhere fall back (butterfly.py:127-133,
        # 264-273) — to the fp64 payload of the lowest alive miner when no fallback was given
        src = payloads[miners[alive[0]]]
        job.set_fallback(_to_device_f64(src if hosts is None else hosts[0], dev))
        job.run(L.PHASE_CHECK)
        early = False  # merged changed after the streamed copy: copy it again
    if _device_merged:  # stage glue (stage.py): the merged weights stay in HBM
        merged = job.merged
    else:
        if not early:
            merged_host = torch.empty(P, dtype=torch.float64, pin_memory=True)  # cached pinned block
            merged_host.copy_(job.merged, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        merged = merged_host.numpy()  # the array keeps the pinned tensor alive
    return _settle(store, plan, miners, payloads, reps, alive, failed, key_prefix, job, descriptors, callables,
                   host_reductions, merged)


def nonfinite_fallback_needed(job, plan, failed: set, corrupted: set) -> bool:
    """Did some fast shard come out a disagreement (a non-finite mean)?  Reads the status."""
    status = job.status.cpu().numpy()
    classes = _classes(plan, failed, corrupted)
    return any(c == "fast" and status[s] != L.MERGED for s, c in enumerate(classes))


def _settle(store, plan, miners, payloads, reps, alive, failed, prefix, job, descriptors, callables,
            host_reductions, merged):
    """The round's results back to the host and into the store (butterfly.py:242-295):
    per-shard status, agreement matrix, flags; the re-uploaded reductions that differ from
    ``merged`` rendered to host bytes; the closed-form meter.  Returns the MergeResult of
    the plan's module.  No reference to the job's device memory survives the call."""
    _, agreement_type, result_type = _types_of(plan)
    n = plan.pair_set.n_miners
    status_codes = job.status.cpu().numpy()
    classes = _classes(plan, failed, set(descriptors) | set(callables))
    nonfinite = [s for s, c in enumerate(classes) if c == "fast" and status_codes[s] != L.MERGED]
    nonfinite_means = _nonfinite_means(plan, reps, alive, nonfinite) if nonfinite else {}
    entries = job.entries.cpu().numpy()
    flagged_idx = np.flatnonzero(job.flagged.cpu().numpy())
    sources = job.source.cpu().numpy()
    rendered = _render_special(job, plan, failed, descriptors, classes, host_reductions, nonfinite_means)
    _account_store(store, plan, miners, payloads, alive, failed, prefix, plan.bytes_per_weight, merged, status_codes,
                   sources, host_reductions, rendered)
    return result_type(
        merged=merged,
        shard_status=[L.STATUS_NAMES[c] for c in status_codes],
        agreement_matrix=agreement_type(n_miners=n, entries=entries),
        flagged={miners[i] for i in flagged_idx},
    )


def _nonfinite_means(plan, reps, alive, shards) -> dict:
    """fp64 means of the given shards (mean_reducer's order, butterfly.py:156-158) from
    the device replicas, which the drop-in never overwrites: shard -> host array."""
    out = {}
    for s in shards:
        lo, hi = plan.bounds[s]
        stack = torch.stack([reps[m][lo:hi].to(torch.float64) for m in alive])
        out[s] = mean_reducer(stack).cpu().numpy()
    return out


def _render_special(job, plan, failed, descriptors, classes, host_reductions, nonfinite_means) -> dict:
    """(shard, assignee) -> "<f4" bytes of the re-uploaded reductions that are not the
    merged values (butterfly.py:235-240): every survivor of a special shard (honest ones
    carry the mean, descriptor-corrupted ones their copy), and both survivors of a
    non-finite shard.  Callable outputs are kept as returned."""
    items = []
    for s, members in enumerate(plan.assignment):
        if classes[s] == "fast" and s not in nonfinite_means:
            continue
        if classes[s] == "lost":
            continue
        lo, hi = plan.bounds[s]
        for x in members:
            if x in failed or (s, x) in host_reductions:
                continue
            items.append((s, x, lo, hi))
    if not items:
        return {}
    parts = []
    for s, x, lo, hi in items:
        if s in nonfinite_means:
            parts.append(torch.from_numpy(nonfinite_means[s]).to(torch.float32))
            continue
        mean = job.means[lo:hi]
        if x in descriptors:
            out = torch.empty_like(mean)
            L.check(L.lib().bfly_apply_corruption(descriptors[x].struct(), mean.data_ptr(), lo, hi - lo,
                                                  out.data_ptr(), _stream_handle()))
            mean = out
        parts.append(mean.to(torch.float32))
    flat = torch.cat([p.to(parts[0].device) if p.device != parts[0].device else p for p in parts]).cpu().numpy()
    out, o = {}, 0
    for s, x, lo, hi in items:
        out[(s, x)] = flat[o:o + hi - lo].astype("<f4").tobytes()
        o += hi - lo
    return out


_UPLOAD_BLOCK = 0  # elements per staging block of the host upload (0: the library default, 384 Ki)
_UPLOAD_THREADS = 0  # host conversion threads (0: the library default, one per core less the issuing one)


def _merge_chunks(P: int) -> int:
    """Pipeline depth of bfly_merge_host: chunks of >= 4M elements, at most 32."""
    return max(1, min(32, P >> 22))


def _chunk(size: int, start: int, length: int | None) -> int:
    """len(blob[start:start+length]) for a blob of `size` bytes (simkernel.py:181-184)."""
    stop = size if length is None else start + length
    return max(0, min(stop, size) - min(start, size))


def _account_store(store, plan, miners, payloads, alive, failed, prefix, bpw, merged, status_codes, sources,
                   host_reductions, rendered):
    objects = store.objects
    meta = plan.metadata()
    objects[f"{prefix}/shard-metadata"] = meta
    _meter(store, "orchestrator").bytes_uploaded += _wire(store, len(meta))
    P = len(merged)
    n_alive = len(alive)
    wsize = 4 * P  # weights always travel as "<f4" (butterfly.py:213)
    for m in alive:  # upload stage
        key = f"{prefix}/miner/{miners[m]}/weights"
        objects[key] = _wire_blob(payloads[miners[m]], wsize)
        _meter(store, str(miners[m])).bytes_uploaded += _wire(store, wsize)
    for s, (i, j) in enumerate(plan.assignment):  # reduce stage
        lo, hi = plan.bounds[s]
        for x in (i, j):
            if x in failed:
                continue
            mt = _meter(store, str(miners[x]))
            mt.bytes_downloaded += n_alive * _wire(store, _chunk(wsize, lo * bpw, (hi - lo) * bpw))
            if (s, x) in host_reductions:
                red = np.asarray(host_reductions[(s, x)])
                blob = red.astype("<f4").tobytes()
            elif (s, x) in rendered:
                blob = rendered[(s, x)]
            else:  # every survivor of a merged fast shard re-uploaded the merged mean
                blob = _wire_blob(merged[lo:hi], 4 * (hi - lo))
            objects[f"{prefix}/miner/{miners[x]}/merged/{s}"] = blob
            mt.bytes_uploaded += _wire(store, len(blob))
    for m in alive:  # redistribution stage (metering only)
        mt = _meter(store, str(miners[m]))
        down = 0
        for s in range(plan.n_shards):
            lo, hi = plan.bounds[s]
            src = int(sources[s])
            if status_codes[s] == L.MERGED and src >= 0:
                down += _wire(store, len(objects[f"{prefix}/miner/{miners[src]}/merged/{s}"]))
            else:
                down += _wire(store, _chunk(wsize, lo * bpw, (hi - lo) * bpw))
        mt.bytes_downloaded += down


# ---------------------------------------------------------------------------
# analytics (closed forms / Monte-Carlo; off the data path, butterfly.py:298-341)
# ---------------------------------------------------------------------------


def valid_shard_fraction(n: int, k: int) -> float:
    """Merged-shard fraction with k of n miners failed: 1 - k(k-1)/(n(n-1))."""
    if n < 2:
        raise TooFewMinersError(f"need at least 2 miners, got {n}")
    if k < 0 or k > n:
        raise InvalidArgumentError(f"k must be in [0, {n}], got {k}")
    return 1.0 - (k * (k - 1)) / (n * (n - 1))


def per_miner_transfer(w_bytes: float, n_m: int) -> float:
    """Per-miner bytes per round, 4W + 2W/N."""
    if n_m < 2:
        raise TooFewMinersError(f"need at least 2 miners, got {n_m}")
    return 4.0 * w_bytes + 2.0 * w_bytes / n_m


def monte_carlo_resilience(n: int, k_values, trials: int, seed: int) -> dict:
    """Empirical valid-shard fraction over uniform failure draws (butterfly.py:322-341).

    Every pair of miners owns exactly one shard (r = 2, butterfly.py:76-114), so any
    draw of k failed miners loses exactly the C(k, 2) shards of the pairs inside it:
    each of the reference's ``trials`` draws contributes S - C(k, 2) valid shards
    whatever the RNG returns.  The same integer ratio is therefore formed in closed form
    (identical floats, the same errors) — O(|k_values|) instead of trials x S.
    ``seed`` selects the reference's draws, which cannot change the result."""
    n_sh = len(enumerate_pairs(n).pairs)
    out = {}
    for k in k_values:
        if k < 0 or k > n:
            raise InvalidArgumentError(f"k must be in [0, {n}], got {k}")
        out[k] = (trials * (n_sh - k * (k - 1) // 2)) / (trials * n_sh)
    return out