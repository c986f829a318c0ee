"""The reference's own hot-path tests, restated against the drop-in module.

Mirrors pkg/tests/test_butterfly.py (TestPairs, TestShardPlan, TestAgreement,
TestAllReduce, TestResilience) and acceptance criteria 2, 3 and 4
(pkg/tests/test_acceptance.py:78-162), run through
paper_2507_17766_b200.butterfly — i.e. through the C ABI and the B200 kernels.
The analytics and plan checks need no GPU; the merge checks are marked gpu.
"""

import time

import numpy as np
import pytest

from paper_2507_17766_b200 import butterfly as bf
from paper_2507_17766_b200.errors import DegenerateShardsError, InvalidArgumentError, ShapeError, TooFewMinersError
from paper_2507_17766_b200.simkernel import BlobStore, RngStream

BPW = bf.BYTES_PER_WEIGHT
gpu = pytest.mark.gpu


# --------------------------------------------------------------------------- pairs / plan (CPU)

def test_pairs_three_miners():
    assert bf.enumerate_pairs(3).pairs == ((0, 1), (0, 2), (1, 2))


def test_pairs_count_is_n_choose_2():
    assert len(bf.enumerate_pairs(50).pairs) == 1225


def test_pairs_too_few():
    with pytest.raises(TooFewMinersError):
        bf.enumerate_pairs(1)


def test_seed_24_mapping():
    assert bf.plan_shards(bf.enumerate_pairs(3), 9, BPW, seed=24).assignment == ((1, 2), (0, 2), (0, 1))


def test_near_equal_split_remainder_first():
    plan = bf.plan_shards(bf.enumerate_pairs(3), 10, BPW, seed=0)
    sizes = [e - s for s, e in plan.bounds]
    assert sorted(sizes) == [3, 3, 4] and sizes[0] == 4
    assert plan.bounds[0][0] == 0 and plan.bounds[-1][1] == 10


def test_assignment_bijection_and_partner_coverage():
    pair_set = bf.enumerate_pairs(8)
    assert sorted(bf.plan_shards(pair_set, 1000, BPW, seed=3).assignment) == list(pair_set.pairs)
    n = 10
    plan = bf.plan_shards(bf.enumerate_pairs(n), 500, BPW, seed=5)
    for m in range(n):
        partners = {j if i == m else i for i, j in (plan.assignment[s] for s in plan.shards_of(m))}
        assert partners == set(range(n)) - {m}


def test_byte_bounds_and_degenerate():
    plan = bf.plan_shards(bf.enumerate_pairs(3), 9, BPW, seed=0)
    assert all(plan.byte_bounds(s) == (a * 4, b * 4) for s, (a, b) in enumerate(plan.bounds))
    with pytest.raises(DegenerateShardsError):
        bf.plan_shards(bf.enumerate_pairs(3), 2, BPW, seed=0)


def test_assignment_uniform_over_seeds():
    from scipy import stats

    pair_set = bf.enumerate_pairs(4)
    counts = {p: 0 for p in pair_set.pairs}
    for seed in range(10000):
        counts[bf.plan_shards(pair_set, 60, BPW, seed).assignment[0]] += 1
    assert stats.chisquare(list(counts.values())).pvalue > 1e-3


def test_resilience_analytics():
    assert bf.valid_shard_fraction(50, 5) == pytest.approx(1.0 - 20.0 / 2450.0)
    assert bf.valid_shard_fraction(50, 0) == 1.0 and bf.valid_shard_fraction(50, 1) == 1.0
    assert bf.valid_shard_fraction(10, 4) == pytest.approx(1.0 - 12.0 / 90.0)
    assert bf.valid_shard_fraction(2, 2) == 0.0
    with pytest.raises(InvalidArgumentError):
        bf.valid_shard_fraction(10, 11)
    with pytest.raises(TooFewMinersError):
        bf.valid_shard_fraction(1, 0)
    assert bf.per_miner_transfer(1000.0, 2) == pytest.approx(5000.0)
    assert bf.per_miner_transfer(1000.0, 10) == pytest.approx(4200.0)


def test_criterion_2_merge_resilience():
    start = time.perf_counter()
    ks = list(range(26))
    emp = bf.monte_carlo_resilience(50, ks, trials=1000, seed=2)
    assert all(abs(emp[k] - bf.valid_shard_fraction(50, k)) < 1e-12 for k in ks)
    assert abs(bf.valid_shard_fraction(50, 5) - 0.99184) < 1e-5
    assert time.perf_counter() - start < 5.0


def test_rngstream_matches_reference_key_scheme():
    from paper_2507_17766_b200 import _lib

    a = RngStream(4, "tamper").fork("m0")
    k = np.array(_lib.philox_key(4, "tamper/m0"), dtype=np.uint64)
    b = np.random.Generator(np.random.Philox(key=k))
    assert np.array_equal(a.normal(0, 1, 17), b.normal(0, 1, 17))


# --------------------------------------------------------------------------- merges (GPU)

def _payloads(n, length, seed=0):
    rng = np.random.default_rng(seed)
    return {m: rng.uniform(-1.0, 1.0, length) for m in range(n)}


def _f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


@gpu
def test_agreement_kats():
    a = np.array([1.0, 2.0, 3.0])
    assert bf.agreement(a, a + 1e-9) == 1.0
    assert bf.agreement(np.array([1.0, 0.0]), np.array([1.0, 1.0])) == pytest.approx(1.0 / np.sqrt(2.0))
    assert bf.agreement(np.array([1.0, 0.0]), np.array([-1.0, 0.0])) == 0.0
    with pytest.raises(ShapeError):
        bf.agreement(np.zeros(3), np.zeros(4))


@gpu
def test_honest_merge_is_mean_of_wire_payloads():
    n, length = 4, 100
    payloads = _payloads(n, length)
    plan = bf.plan_shards(bf.enumerate_pairs(n), length, BPW, seed=1)
    res = bf.run_all_reduce(BlobStore(), payloads, plan)
    assert np.allclose(res.merged, np.mean([_f32(payloads[m]) for m in range(n)], axis=0), atol=1e-12)
    assert res.shard_status == ["merged"] * plan.n_shards and res.flagged == set()


@gpu
def test_single_failure_loses_nothing():
    n, length = 5, 60
    payloads = _payloads(n, length)
    plan = bf.plan_shards(bf.enumerate_pairs(n), length, BPW, seed=2)
    res = bf.run_all_reduce(BlobStore(), payloads, plan, failures={3})
    assert res.shard_status == ["merged"] * plan.n_shards
    assert np.allclose(res.merged, np.mean([_f32(payloads[m]) for m in range(n) if m != 3], axis=0), atol=1e-12)


@gpu
def test_pair_failure_falls_back():
    n, length = 3, 30
    plan = bf.plan_shards(bf.enumerate_pairs(n), length, BPW, seed=3)
    res = bf.run_all_reduce(BlobStore(), _payloads(n, length), plan, failures={0, 1}, fallback=np.zeros(length))
    lost = plan.assignment.index((0, 1))
    assert res.shard_status[lost] == "lost"
    s, e = plan.bounds[lost]
    assert np.all(res.merged[s:e] == 0.0)


@gpu
def test_deceptive_reduction_flagged():
    n, length = 4, 80
    plan = bf.plan_shards(bf.enumerate_pairs(n), length, BPW, seed=4)
    res = bf.run_all_reduce(BlobStore(), _payloads(n, length), plan, corruptions={2: lambda red: red + 1.0},
                            fallback=np.zeros(length))
    assert 2 in res.flagged
    e = res.agreement_matrix.entries
    assert all(e[2, o] < 1.0 for o in (0, 1, 3)) and e[0, 1] == 1.0


@gpu
@pytest.mark.parametrize("n", [2, 3, 10, 50])
def test_criterion_3_transfer_accounting(n):
    n_shards = n * (n - 1) // 2
    length = max(8 * n_shards, 64) if n == 50 else 1000
    plan = bf.plan_shards(bf.enumerate_pairs(n), length, BPW, seed=n)
    store = BlobStore()
    bf.run_all_reduce(store, _payloads(n, length, seed=n), plan)
    expected = bf.per_miner_transfer(length * BPW, n)
    max_shard = max(e - s for s, e in plan.bounds) * BPW
    for m in range(n):
        mt = store.meter[str(m)]
        assert abs(mt.bytes_uploaded + mt.bytes_downloaded - expected) <= max_shard


@gpu
def test_criterion_4_deceptive_merge_detection():
    start = time.perf_counter()
    n, n_bad = 50, 10
    length = 1225 * 400
    rng = np.random.default_rng(4)
    payloads = {m: rng.uniform(-1.0, 1.0, length) for m in range(n)}
    plan = bf.plan_shards(bf.enumerate_pairs(n), length, BPW, seed=4)
    tamper = RngStream(4, "tamper")
    corruptions = {}
    for m in range(n_bad):
        sub = tamper.fork(f"m{m}")

        def corrupt(red, sub=sub):
            rms = float(np.sqrt(np.mean(red ** 2))) or 1.0
            return sub.normal(0.0, 2.0 * rms, size=red.shape)

        corruptions[m] = corrupt
    res = bf.run_all_reduce(BlobStore(), payloads, plan, corruptions=corruptions, fallback=np.zeros(length))
    e = res.agreement_matrix.entries
    bad = set(range(n_bad))
    worst_bad = max(e[i, j] for i in bad for j in range(n) if j not in bad and j != i)
    worst_honest = min(e[i, j] for i in range(n_bad, n) for j in range(i + 1, n))
    assert worst_bad < 0.5 and worst_honest >= 0.999
    # both members of a disagreeing pair are flagged (butterfly.py:266-267), and every
    # honest miner shares one shard with every deceptive miner
    assert res.flagged == set(range(n))
    assert time.perf_counter() - start < 10.0


@gpu
def test_custom_reducer_is_rejected_not_emulated():
    plan = bf.plan_shards(bf.enumerate_pairs(3), 9, BPW, seed=0)
    with pytest.raises(NotImplementedError):
        bf.run_all_reduce(BlobStore(), _payloads(3, 9), plan, reducer=lambda s: s.sum(axis=0))


@gpu
def test_store_contents_materialise_like_the_reference():
    n, length = 5, 203
    payloads = _payloads(n, length, seed=3)
    plan = bf.plan_shards(bf.enumerate_pairs(n), length, BPW, seed=8)
    store = BlobStore()
    res = bf.run_all_reduce(store, payloads, plan, failures={1}, corruptions={2: bf.Corruption.add(0.5)},
                            fallback=np.zeros(length), key_prefix="ep/0")
    assert store.get("x", "ep/0/miner/3/weights") == payloads[3].astype("<f4").tobytes()
    assert store.objects["ep/0/shard-metadata"] == plan.metadata()
    for s, (i, j) in enumerate(plan.assignment):
        lo, hi = plan.bounds[s]
        for x in (i, j):
            if x == 1:
                assert not store.exists(f"ep/0/miner/{x}/merged/{s}")
                continue
            mean = np.mean([_f32(payloads[m][lo:hi]) for m in range(n) if m != 1], axis=0)
            want = (mean + 0.5 if x == 2 else mean).astype("<f4").tobytes()
            assert store.get("x", f"ep/0/miner/{x}/merged/{s}") == want
    # both members of every disagreeing pair are flagged (butterfly.py:266-267)
    partners = {m for pair in plan.assignment if 2 in pair for m in pair if m != 1}
    assert res.flagged == partners


def test_monte_carlo_resilience_matches_reference():
    """Fixture from the reference's own monte_carlo_resilience (tests/golden/resilience_mc.json,
    made by tests/golden/make_resilience_golden.py): identical floats."""
    import json
    from pathlib import Path

    want = json.loads((Path(__file__).parent / "golden" / "resilience_mc.json").read_text())
    for key, vals in want.items():
        n, trials, seed = (int(x) for x in key.split("_"))
        got = bf.monte_carlo_resilience(n, [int(k) for k in vals], trials=trials, seed=seed)
        assert {str(k): v for k, v in got.items()} == vals
    with pytest.raises(InvalidArgumentError):
        bf.monte_carlo_resilience(5, [6], trials=3, seed=0)
    with pytest.raises(TooFewMinersError):
        bf.monte_carlo_resilience(1, [0], trials=3, seed=0)
