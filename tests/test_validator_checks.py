"""Validator replay checks against fixtures from the reference's own
validator._check / cosine_similarity (tests/golden/make_validator_golden.py)."""

import json

import numpy as np
import pytest

from _golden import GOLDEN

import oracle as orc


def _cases():
    d = json.loads((GOLDEN / "validator_checks.json").read_text())
    arr = np.load(GOLDEN / "validator_checks.npz")
    return d["policies"], [(arr[f"a{c['i']}"], arr[f"b{c['i']}"], c["cos"], c["sims"]) for c in d["cases"]]


def _same(got, want, tol=1e-12):
    if np.isnan(want):
        return np.isnan(got)
    if np.isinf(want):
        return got == want
    return abs(got - want) <= tol


def test_oracle_matches_reference_checks():
    policies, cases = _cases()
    for a, b, cos, sims in cases:
        assert _same(orc.cosine_similarity(a, b), cos)
        for p, want in zip(policies, sims):
            assert _same(orc.replay_check(a, b, p), want), (p, want)


@pytest.mark.gpu
def test_gpu_checks_match_reference(cuda_device):
    from paper_2507_17766_b200 import validator as v

    policies, cases = _cases()
    recs = [a for a, _, _, _ in cases]
    reps = [b for _, b, _, _ in cases]
    for k, p in enumerate(policies):
        pol = v.ReplayPolicy(*p)
        got = v.check_batch(recs, reps, pol)
        for (a, b, cos, sims), g in zip(cases, got):
            if abs(cos - p[0]) <= 1e-12:  # cosine on the threshold: the decision depends on the
                assert _same(g, cos) or g == 0.0  # dot-product order (e.g. -a vs a at threshold -1)
                continue
            assert _same(g, sims[k]), (k, len(a), g, sims[k])
    for a, b, cos, _ in cases[:12]:
        assert _same(v.cosine_similarity(a, b), cos)
        assert _same(v.check(a, b), orc.replay_check(a, b, policies[0]))


@pytest.mark.gpu
def test_gpu_check_shapes(cuda_device):
    from paper_2507_17766_b200 import validator as v
    from paper_2507_17766_b200.errors import ShapeError

    with pytest.raises(ShapeError):
        v.check(np.ones(3), np.ones(4))
    with pytest.raises(ShapeError):
        v.cosine_similarity(np.ones(0), np.ones(0))
    with pytest.raises(ShapeError):
        v.check_batch([np.ones(3)], [])
    assert v.check_batch([], []).shape == (0,)
