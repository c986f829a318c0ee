"""ctypes front end of the CPU oracle (oracle/bfly_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, as the checker or as the
timed CPU restatement of the reference.  The product package never imports it.

Every function cites the reference code it restates; the C file holds the
algorithm.  ``philox_key`` uses hashlib exactly like simkernel.py:203-205.
"""

from __future__ import annotations

import ctypes
import math
import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "_build" / "liboracle.so"

MERGED, LOST, DISAGREEMENT = 0, 1, 2
STATUS_NAMES = ("merged", "lost", "disagreement")
F32, BF16, F64WIRE = 0, 1, 2
NONE, ADD, SCALE, NOISE, NOISE_ADD = 0, 1, 2, 3, 4


class Corruption(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("a", ctypes.c_double),
        ("key0", ctypes.c_uint64),
        ("key1", ctypes.c_uint64),
    ]


def build() -> Path:
    """Compile liboracle.so with the committed Makefile (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        L = ctypes.CDLL(str(_SO))
        i32, i64, u64, dbl, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        L.orc_permutation.argtypes = [u64, u64, i64, vp]
        L.orc_philox_raw.argtypes = [u64, u64, i64, vp]
        L.orc_n_combinations.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_n_combinations.restype = i64
        L.orc_plan.argtypes = [ctypes.c_int, ctypes.c_int, i64, u64, u64, vp, vp]
        L.orc_agreement.argtypes = [vp, vp, i64, dbl]
        L.orc_agreement.restype = dbl
        L.orc_merge.argtypes = [ctypes.c_int, ctypes.c_int, i64, i64, vp, vp, ctypes.c_int, vp, vp, vp,
                                vp, dbl, vp, vp, vp, vp, vp, ctypes.c_int]
        L.orc_f32_to_bf16.argtypes = [ctypes.c_float]
        L.orc_f32_to_bf16.restype = ctypes.c_uint16
        _lib = L
    return _lib


def philox_key(seed: int, stream_id: str) -> tuple[int, int]:
    """_philox_key (simkernel.py:203-205)."""
    d = hashlib.sha256(f"{int(seed)}\x1f{stream_id}".encode()).digest()
    return int.from_bytes(d[0:8], "little"), int.from_bytes(d[8:16], "little")


def permutation(seed: int, n: int, stream_id: str = "shard-plan") -> np.ndarray:
    """RngStream(seed, stream_id).permutation(n) (simkernel.py:216-219,237-238)."""
    k0, k1 = philox_key(seed, stream_id)
    out = np.empty(n, dtype=np.int64)
    lib().orc_permutation(k0, k1, n, out.ctypes.data)
    return out


def philox_raw(key0: int, key1: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    lib().orc_philox_raw(key0, key1, n, out.ctypes.data)
    return out


def n_shards(n: int, r: int = 2) -> int:
    return int(lib().orc_n_combinations(n, r))


def plan(n: int, payload_len: int, seed: int, r: int = 2):
    """plan_shards (butterfly.py:84-114) -> (assign[S, r] int32, bounds[S+1] int64)."""
    S = n_shards(n, r) if n >= r else 0
    assign = np.empty((max(S, 1), r), dtype=np.int32)
    bounds = np.empty(max(S, 0) + 1, dtype=np.int64)
    k0, k1 = philox_key(seed, "shard-plan")
    rc = lib().orc_plan(n, r, payload_len, k0, k1, assign.ctypes.data, bounds.ctypes.data)
    if rc == 1:
        raise ValueError("too few miners")
    if rc == 2:
        raise ValueError("degenerate shards")
    return assign[:S], bounds


def agreement(a, b, tolerance: float = 1e-6) -> float:
    """agreement (butterfly.py:117-133), sequential dot products."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape
    return float(lib().orc_agreement(a.ctypes.data, b.ctypes.data, a.size, tolerance))


def corruption_table(n: int, corr: dict | None):
    """{miner index: (kind, a[, key0, key1])} -> ctypes array of n descriptors."""
    table = (Corruption * n)()
    for m, spec in (corr or {}).items():
        kind, a = spec[0], spec[1]
        k0, k1 = (spec[2], spec[3]) if len(spec) > 2 else (0, 0)
        table[m] = Corruption(kind, 0, a, k0, k1)
    return table


def merge(replicas, assign, bounds, *, failures=(), corruptions=None, fallback=None,
          tolerance: float = 1e-6, dtype: int = F32, threads: int = 0):
    """run_all_reduce (butterfly.py:161-295) on wire-value replicas.

    replicas: list of N 1-D arrays (float32, uint16 bf16 bits, or float64 payloads
    for F64WIRE).  Returns dict(merged, status, entries, flagged, source).
    """
    n = len(replicas)
    S, r = assign.shape
    P = int(bounds[-1])
    reps = [np.ascontiguousarray(x) for x in replicas]
    ptrs = (ctypes.c_void_p * n)(*[x.ctypes.data for x in reps])
    failed = np.zeros(n, dtype=np.uint8)
    for m in failures:
        failed[m] = 1
    table = corruption_table(n, corruptions)
    fb = None if fallback is None else np.ascontiguousarray(fallback, dtype=np.float64)
    merged = np.empty(P, dtype=np.float64)
    status = np.empty(S, dtype=np.uint8)
    entries = np.empty((n, n), dtype=np.float64)
    flagged = np.empty(n, dtype=np.uint8)
    source = np.empty(S, dtype=np.int32)
    a = np.ascontiguousarray(assign, dtype=np.int32)
    bnd = np.ascontiguousarray(bounds, dtype=np.int64)
    lib().orc_merge(n, r, P, S, a.ctypes.data, bnd.ctypes.data, dtype, ptrs, failed.ctypes.data,
                    ctypes.addressof(table), None if fb is None else fb.ctypes.data, tolerance,
                    merged.ctypes.data, status.ctypes.data, entries.ctypes.data, flagged.ctypes.data,
                    source.ctypes.data, threads)
    return dict(merged=merged, status=status, entries=entries, flagged=flagged, source=source)


def noise_values(key0: int, key1: int, amp: float, start: int, stop: int) -> np.ndarray:
    """The NOISE descriptor's values on elements [start, stop) — numpy form of
    orc_noise: word e of Philox(key).random_raw, mapped to amp * (2u - 1)."""
    bg = np.random.Philox(key=np.array([key0, key1], dtype=np.uint64))
    bg.advance(start // 4)  # word e lives in the 4-word block e // 4 (no need to draw the words before it)
    raw = bg.random_raw(stop - (start // 4) * 4)[start % 4:]
    unit = (raw >> np.uint64(11)).astype(np.float64) * (1.0 / 4503599627370496.0) - 1.0
    return amp * unit


def threads_available() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- validator replay checks
# (test infrastructure like the rest of this module)


def cosine_similarity(a, b) -> float:
    """validator.cosine_similarity (validator.py:33-46): a.b / (|a| |b|) with |x| =
    sqrt(x.x); two zero vectors -> 1.0, exactly one zero vector -> 0.0."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    with np.errstate(all="ignore"):
        na, nb = math.sqrt(float(np.dot(a, a))), math.sqrt(float(np.dot(b, b)))
        if na == 0.0 and nb == 0.0:
            return 1.0
        if na == 0.0 or nb == 0.0:
            return 0.0
        return float(np.dot(a, b)) / (na * nb)


def replay_check(recomputed, reported, policy) -> float:
    """validator._check (validator.py:148-167) for policy = (cosine_threshold,
    magnitude_low, magnitude_high, max_rel_deviation): the cosine, or 0.0 when it is
    below the threshold, when the norm ratio leaves the band (only if |rec| > 0), or
    when the largest deviation relative to max(|rec|, 1) exceeds the limit."""
    thr, lo, hi, max_rel = policy
    rec = np.asarray(recomputed, dtype=np.float64)
    rep = np.asarray(reported, dtype=np.float64)
    sim = cosine_similarity(rec, rep)
    if sim < thr:
        return 0.0
    with np.errstate(all="ignore"):
        n_rec, n_rep = math.sqrt(float(np.dot(rec, rec))), math.sqrt(float(np.dot(rep, rep)))
        if n_rec > 0.0 and not (lo <= n_rep / n_rec <= hi):
            return 0.0
        dev = np.abs(rec - rep) / np.maximum(np.abs(rec), 1.0)
        worst = float(np.max(dev)) if dev.size else 0.0
    if worst > max_rel:
        return 0.0
    return sim
