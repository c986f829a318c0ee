"""Golden fixtures for the validator's replay checks, from the REFERENCE.

Calls iota_sim.validator._check / cosine_similarity (read-only /root/reference,
validator.py:33-46,148-167) on recomputed/reported activation pairs — honest replays,
float noise at several magnitudes, rescaled and sign-flipped reports, zero vectors,
NaN / inf entries, large entries (relative deviation scale), lengths 1 .. 4097 — under
the default ReplayPolicy and two custom ones, and records every similarity.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_validator_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from iota_sim.validator import ReplayPolicy, _check, cosine_similarity  # noqa: E402

OUT = Path(__file__).resolve().parent

POLICIES = [
    ReplayPolicy(),
    ReplayPolicy(cosine_threshold=0.99, magnitude_low=0.9, magnitude_high=1.1, max_rel_deviation=1e-3),
    ReplayPolicy(cosine_threshold=-1.0, magnitude_low=0.0, magnitude_high=float("inf"), max_rel_deviation=float("inf")),
]


def pairs():
    rng = np.random.default_rng(2507)
    for n in (1, 2, 7, 24, 64, 1000, 4097):
        a = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-3, 4)
        yield a, a.copy()                                        # exact replay
        for eps in (1e-15, 1e-12, 1e-10, 1e-8, 1e-5, 1e-2):
            yield a, a + rng.normal(0, eps, n) * np.maximum(np.abs(a), 1.0)
        yield a, a * 1.0005                                      # inside the magnitude band
        yield a, a * 1.002                                       # outside it
        yield a, -a                                              # anti-parallel
        yield a, rng.uniform(-1, 1, n)                           # unrelated
        yield a, a * 3.0 + 1e-9
    yield np.zeros(5), np.zeros(5)
    yield np.zeros(5), np.ones(5)
    yield np.ones(5), np.zeros(5)
    yield np.array([1e200, -1e200, 3.0]), np.array([1e200, -1e200, 3.0])   # overflowing norms
    yield np.array([1.0, np.nan, 2.0]), np.array([1.0, 2.0, 2.0])
    yield np.array([1.0, 2.0, 2.0]), np.array([1.0, np.inf, 2.0])
    big = np.array([1e6, -2e6, 5e5, 7.0])
    yield big, big * (1 + 5e-10)
    yield big, big + np.array([0.0, 0.0, 0.0, 1e-8])
    yield big, big + np.array([0.0, 0.0, 0.0, 1e-9])


def main():
    arrays, cases = {}, []
    for i, (a, b) in enumerate(pairs()):
        arrays[f"a{i}"], arrays[f"b{i}"] = a, b
        with np.errstate(all="ignore"):
            cos = cosine_similarity(a, b)
            sims = [_check(a, b, p) for p in POLICIES]
        cases.append({"i": i, "cos": cos, "sims": sims})
    pol = [[p.cosine_threshold, p.magnitude_low, p.magnitude_high, p.max_rel_deviation] for p in POLICIES]
    (OUT / "validator_checks.json").write_text(json.dumps({"policies": pol, "cases": cases}, indent=0))
    np.savez_compressed(OUT / "validator_checks.npz", **arrays)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
