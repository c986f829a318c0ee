"""Pin the CPU oracle (oracle/bfly_oracle.c) to the reference's own outputs.

The fixtures under tests/golden/ were produced by running iota_sim itself
(tests/golden/make_golden.py).  CPU only.
"""

import numpy as np
import pytest

import oracle as orc
from _golden import (
    agreement_cases,
    assert_entries_close,
    assert_same_floats,
    corruption_specs,
    lex_pairs,
    load_case,
    merge_cases,
    plans,
)


def test_seed_24_kat():
    # tests/test_butterfly.py:37-40 / PAPER.md:225
    assign, _ = orc.plan(3, 9, 24)
    assert [tuple(p) for p in assign] == [(1, 2), (0, 2), (0, 1)]


def test_plans_match_reference():
    g = plans()
    seeds = [int(s) for s in g["seeds"]]
    checked = 0
    for n in (2, 3, 4, 5, 7, 8, 10, 16, 32, 50, 64):
        pairs = lex_pairs(n)
        for seed in seeds:
            ranks = g[f"n{n}_s{seed}"]
            assign, _ = orc.plan(n, len(pairs) + 3, seed)
            assert [tuple(p) for p in assign] == [pairs[k] for k in ranks], (n, seed)
            checked += 1
    assert checked >= 400


@pytest.mark.parametrize("key", ["b_n3_P10", "b_n3_P9", "b_n8_P1000", "b_n8_P10000001", "b_n10_P45",
                                 "b_n10_P89", "b_n64_P2017"])
def test_bounds_match_reference(key):
    ref = plans()[key]
    n, P = (int(x[1:]) for x in key.split("_")[1:])
    _, bounds = orc.plan(n, P, 0)
    assert np.array_equal(bounds, ref)


def test_permutation_matches_numpy_directly():
    # numpy is the pinned third-party dependency behind RngStream.permutation
    for seed in (0, 1, 24, 2**63 - 1):
        for n in (1, 2, 28, 120, 2016, 4960, 70_000):
            key = np.array(orc.philox_key(seed, "shard-plan"), dtype=np.uint64)
            want = np.random.Generator(np.random.Philox(key=key)).permutation(n)
            assert np.array_equal(orc.permutation(seed, n), want), (seed, n)


def test_philox_raw_matches_numpy():
    k = (0x243F6A8885A308D3, 0x13198A2E03707344)
    want = np.random.Philox(key=np.array(k, dtype=np.uint64)).random_raw(1001)
    assert np.array_equal(orc.philox_raw(*k, 1001), want)


def test_agreement_matches_reference():
    for c in agreement_cases():
        got = orc.agreement(np.array(c["a"]), np.array(c["b"]), c["tol"])
        want = c["value"]
        if np.isnan(want):
            assert np.isnan(got)
        else:
            assert abs(got - want) <= 1e-12
            assert (got == 1.0) == (want == 1.0)


@pytest.mark.parametrize("meta", merge_cases(), ids=lambda m: m["name"])
def test_merge_matches_reference(meta):
    meta, arr, payloads = load_case(meta)
    n, P = meta["n"], meta["P"]
    assign, bounds = orc.plan(n, P, meta["seed"])
    assert np.array_equal(assign, arr["assignment"])
    out = orc.merge(list(payloads), assign, bounds, failures=meta["failures"],
                    corruptions=corruption_specs(meta), fallback=arr.get("fallback"),
                    tolerance=meta["tol"], dtype=orc.F64WIRE)
    assert_same_floats(out["merged"], arr["merged"])
    assert np.array_equal(out["status"], arr["status"])
    assert np.array_equal(np.flatnonzero(out["flagged"]), arr["flagged"])
    assert_entries_close(out["entries"], arr["entries"])


def test_oracle_threads_deterministic():
    rng = np.random.default_rng(0)
    reps = [rng.uniform(-1, 1, 5000).astype(np.float32) for _ in range(9)]
    assign, bounds = orc.plan(9, 5000, 3)
    a = orc.merge(reps, assign, bounds, corruptions={2: (orc.ADD, 1.0)}, threads=1)
    b = orc.merge(reps, assign, bounds, corruptions={2: (orc.ADD, 1.0)}, threads=4)
    for k in ("merged", "status", "entries", "flagged"):
        assert_same_floats(a[k], b[k])
