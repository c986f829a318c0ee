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
import os
import json
import math
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


def enumerate_pairs(n: int) -> PairSet:
    """All C(n, 2) unordered miner pairs, lexicographic (butterfly.py:76-81)."""
    if n < 2:
        raise TooFewMinersError(f"need at least 2 miners, got {n}")
    return PairSet(n_miners=n, pairs=tuple((i, j) for i in range(n) for j in range(i + 1, n)))


def _host_plan(n: int, r: int, payload_len: int, seed: int):
    S = int(L.lib().bfly_n_shards(n, r))
    assign = np.empty((max(S, 1), r), dtype=np.int32)
    bounds = np.empty(max(S, 0) + 1, dtype=np.int64)
    k0, k1 = L.philox_key(seed, "shard-plan")
    L.check(L.lib().bfly_plan_host(n, r, payload_len, k0, k1, assign.ctypes.data, bounds.ctypes.data))
    return assign[:S], bounds


def plan_shards(pair_set: PairSet, payload_len: int, bytes_per_weight: int, seed: int) -> ShardPlan:
    """Seeded shard -> pair bijection with near-equal bounds (butterfly.py:84-114)."""
    n_shards = len(pair_set.pairs)
    if payload_len < n_shards:
        raise DegenerateShardsError(f"payload of {payload_len} elements cannot fill {n_shards} shards")
    assign, bounds = _host_plan(pair_set.n_miners, 2, payload_len, seed)
    b = bounds.tolist()
    return ShardPlan(pair_set=pair_set, assignment=tuple(tuple(p) for p in assign.tolist()),
                     bounds=tuple(zip(b[:-1], b[1:])), bytes_per_weight=bytes_per_weight, seed=seed)


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


class _LazyBlob:
    """Store object whose bytes are produced on first read (sizes are exact up front).

    Objects of the merge are views of device-resident vectors in the "<f4" wire format:
    a ranged read (``blob[a:b]``, what ``BlobStore.get(actor, key, start, length)``
    does) copies only those elements back when a ``part`` reader is given; anything
    else materialises the whole object once."""

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
    """Ranged reader of ``header + values.astype("<f4")`` for a 1-D float vector
    (device tensor or numpy): only the elements under [start, stop) are copied."""
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


def run_all_reduce(store, payloads: dict, plan: ShardPlan, *, reducer=mean_reducer,
                   failures: frozenset | set = frozenset(), corruptions: dict | None = None,
                   fallback: np.ndarray | None = None, key_prefix: str = "merge",
                   agreement_tolerance: float = 1e-6, _device_merged: bool = False) -> MergeResult:
    """One merge round for a layer (butterfly.py:161-295), executed on the GPU.

    ``payloads`` maps miner id -> 1-D float64 payload (numpy; torch tensors on
    the device are accepted too).  ``failures`` / ``corruptions`` are keyed by
    index into sorted(payloads).  A corruption may be a reference-style callable
    fn(reduction) -> reduction (run on the host, in the reference's call order)
    or a ``Corruption`` descriptor (applied inside the kernels).
    """
    if reducer is not mean_reducer:
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
    bpw = plan.bytes_per_weight

    descriptors = {m: c for m, c in corruptions.items() if isinstance(c, Corruption) and m not in failed}
    callables = {m: c for m, c in corruptions.items() if not isinstance(c, Corruption) and m not in failed}

    # -- device merge ------------------------------------------------------
    reps = [None] * n
    pipelined = False
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
            L.check(L.lib().bfly_upload_wire(h_ptrs, len(alive), P, d_ptrs, 0, _stream_handle()))
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

    host_reductions = {}  # (shard, assignee) -> callable output (fp64 host)
    if callables:
        job.run(L.PHASE_REDUCE)
        means = job.means.cpu().numpy()
        host_copies = np.zeros((2, P), dtype=np.float64)
        for s, (i, j) in enumerate(plan.assignment):  # reference order: butterfly.py:219-233
            lo, hi = plan.bounds[s]
            for slot, x in enumerate((i, j)):
                if x in failed or x not in callables:
                    continue
                out = callables[x](means[lo:hi].copy())
                host_reductions[(s, x)] = out
                arr = np.asarray(out, dtype=np.float64)
                if arr.shape == (hi - lo,):
                    host_copies[slot, lo:hi] = arr
                else:
                    other = j if x == i else i
                    if other not in failed:
                        raise ShapeError(f"reduction shapes differ: {arr.shape} vs {(hi - lo,)}")
                    raise ValueError(f"could not broadcast reduction of shape {arr.shape} into ({hi - lo},)")
        job.run(L.PHASE_FINISH, host_copies=torch.from_numpy(host_copies).to(dev))
    elif pipelined:
        # merged values stream back chunk by chunk unless FINISH may still change them
        early = not _device_merged and not job.needs_finish()
        merged_host = torch.empty(P, dtype=torch.float64, pin_memory=True) if early else None  # cached pinned
        L.check(L.lib().bfly_merge_host(h_ptrs, len(alive), P, d_ptrs, ctypes.byref(job._args),
                                        merged_host.data_ptr() if early else None, _merge_chunks(P), 0,
                                        _stream_handle()))
        if job.needs_finish():
            job.run(L.PHASE_FINISH)
    else:
        job.run(L.PHASE_ALL)

    if _device_merged:  # stage glue (stage.py): the merged weights stay in HBM
        merged = job.merged
    else:
        if not (pipelined and early):
            merged_host = torch.empty(P, dtype=torch.float64, pin_memory=True)  # cached pinned block
            merged_host.copy_(job.merged, non_blocking=True)
        merged = merged_host.numpy()  # the array keeps the pinned tensor alive
    status_codes = job.status.cpu().numpy()
    entries = job.entries.cpu().numpy()
    flagged_idx = np.flatnonzero(job.flagged.cpu().numpy())
    sources = job.source.cpu().numpy()

    # -- blob store: objects + closed-form meter (butterfly.py:205-288) -----
    special = [any(x not in failed and (x in descriptors or x in callables) for x in members)
               for members in plan.assignment]
    _account_store(store, plan, miners, payloads, alive, failed, key_prefix, bpw, merged, status_codes, sources,
                   job, descriptors, host_reductions, special)

    return MergeResult(
        merged=merged,
        shard_status=[L.STATUS_NAMES[c] for c in status_codes],
        agreement_matrix=AgreementMatrix(n_miners=n, entries=entries),
        flagged={miners[i] for i in flagged_idx},
    )


def _merge_chunks(P: int) -> int:
    """Pipeline depth of bfly_merge_host: chunks of >= 4M elements, at most 32
    (BFLY_MERGE_CHUNKS overrides)."""
    forced = os.environ.get("BFLY_MERGE_CHUNKS")
    return int(forced) if forced else max(1, min(32, P >> 22))


def _chunk(size: int, start: int, length: int | None) -> int:
    """len(blob[start:start+length]) for a blob of `size` bytes (simkernel.py:181-184)."""
    stop = size if length is None else start + length
    return max(0, min(stop, size) - min(start, size))


def _account_store(store, plan, miners, payloads, alive, failed, prefix, bpw, merged, status_codes, sources,
                   job, descriptors, host_reductions, special):
    objects = store.objects
    meta = plan.metadata()
    objects[f"{prefix}/shard-metadata"] = meta
    _meter(store, "orchestrator").bytes_uploaded += _wire(store, len(meta))
    P = len(merged)
    n_alive = len(alive)
    weight_keys = {}
    wsize = 4 * P  # weights always travel as "<f4" (butterfly.py:213)
    for m in alive:  # upload stage
        key = f"{prefix}/miner/{miners[m]}/weights"
        src = payloads[miners[m]]
        objects[key] = _LazyBlob(wsize, lambda src=src: _wire_bytes(src), _wire_part(src))
        _meter(store, str(miners[m])).bytes_uploaded += _wire(store, wsize)
        weight_keys[m] = key
    for s, (i, j) in enumerate(plan.assignment):  # reduce stage
        lo, hi = plan.bounds[s]
        for x in (i, j):
            if x in failed:
                continue
            mt = _meter(store, str(miners[x]))
            mt.bytes_downloaded += n_alive * _wire(store, _chunk(wsize, lo * bpw, (hi - lo) * bpw))
            if (s, x) in host_reductions:
                red = np.asarray(host_reductions[(s, x)])
                nbytes = 4 * red.size
                make, part = (lambda red=red: red.astype("<f4").tobytes()), None
            else:
                nbytes = 4 * (hi - lo)
                make, part = _reduction_maker(job, x, lo, hi, merged, special[s], descriptors)
            objects[f"{prefix}/miner/{miners[x]}/merged/{s}"] = _LazyBlob(nbytes, make, part)
            mt.bytes_uploaded += _wire(store, nbytes)
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


def _host(x) -> np.ndarray:
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def _wire_bytes(src) -> bytes:
    if isinstance(src, torch.Tensor):
        return src.detach().to("cpu", torch.float64).numpy().astype("<f4").tobytes()
    return np.asarray(src, dtype=np.float64).astype("<f4").tobytes()


def _reduction_maker(job, x, lo, hi, merged, special, descriptors):
    """(whole, ranged) readers of assignee x's re-uploaded reduction ("<f4",
    butterfly.py:235-240)."""
    if not special:  # all survivors honest: every reduction equals the merged mean
        return (lambda: _host(merged[lo:hi]).astype("<f4").tobytes()), _wire_part(merged[lo:hi])

    class _Copy:  # element range of the assignee's copy, computed on the device on demand
        def __getitem__(self, sl):
            a, b = lo + sl.start, lo + min(sl.stop, hi - lo)
            mean = job.means[a:b]
            if x in descriptors:
                out = torch.empty_like(mean)
                L.check(L.lib().bfly_apply_corruption(descriptors[x].struct(), mean.data_ptr(), a, b - a,
                                                      out.data_ptr(), _stream_handle()))
                mean = out
            return mean

    copy = _Copy()
    return (lambda: _host(copy[0:hi - lo]).astype("<f4").tobytes()), _wire_part(copy)


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