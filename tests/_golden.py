"""Loader for the fixtures written by tests/golden/make_golden.py (from the live reference)."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
STATUS = ("merged", "lost", "disagreement")


def merge_cases():
    return json.loads((GOLDEN / "merge_cases.json").read_text())


def load_case(meta):
    """-> (meta, arrays, payloads[N, P] fp64 in sorted-id order)."""
    arr = dict(np.load(GOLDEN / f"merge_{meta['name']}.npz"))
    if "payloads" in arr:
        payloads = arr["payloads"]
    else:  # regenerate with the reference's recipe (tests/test_butterfly.py:106-108)
        rng = np.random.default_rng(meta["payload_seed"])
        rows = [rng.uniform(-1.0, 1.0, meta["P"]) for _ in range(meta["n"])]
        order = sorted(range(meta["n"]), key=lambda m: (str(m) if meta["id_kind"] == "str" else m))
        payloads = np.stack([rows[m] for m in order])
    wire = payloads.astype(np.float32)
    assert hashlib.sha256(wire.tobytes()).hexdigest() == meta["payload_sha256"], "payload drift"
    return meta, arr, payloads


def corruption_specs(meta):
    return {int(k): tuple(v) for k, v in meta["corruptions"].items()}


def plans():
    return np.load(GOLDEN / "plans.npz")


def agreement_cases():
    return json.loads((GOLDEN / "agreement.json").read_text())


def lex_pairs(n):
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def assert_same_floats(a, b):
    """Bit-exact equality with NaN == NaN."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    same = (a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))
    if not same.all():
        idx = np.flatnonzero(~same.ravel())[:5]
        raise AssertionError(f"{(~same).sum()} of {a.size} differ, e.g. at {idx}: "
                             f"{a.ravel()[idx]} vs {b.ravel()[idx]}")


def assert_entries_close(a, b, atol=1e-12):
    a = np.asarray(a)
    b = np.asarray(b)
    assert np.array_equal(np.isnan(a), np.isnan(b)), "NaN pattern differs"
    m = ~np.isnan(a)
    assert np.all(np.abs(a[m] - b[m]) <= atol), np.max(np.abs(a[m] - b[m]))
