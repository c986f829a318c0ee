"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference's own golden outputs.  Bit-exact for plans, merged values, status and
flags; agreement entries within 1e-12 (the reference's dot products go through
BLAS ddot, whose summation order is unspecified — SURVEY F4)."""

import numpy as np
import pytest

import oracle as orc
from _golden import (
    assert_entries_close,
    assert_same_floats,
    corruption_specs,
    lex_pairs,
    load_case,
    merge_cases,
    plans,
)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KIND = {orc.ADD: "add", orc.SCALE: "scale", orc.NOISE: "noise", orc.NOISE_ADD: "noise_add"}


def _descriptors(specs):
    from paper_2507_17766_b200.device import Corruption

    out = {}
    for m, spec in specs.items():
        key = (spec[2], spec[3]) if len(spec) > 2 else (0, 0)
        out[m] = Corruption(KIND[spec[0]], spec[1], key)
    return out


# --------------------------------------------------------------------------- plan


def test_device_plan_matches_reference(cuda_device):
    from paper_2507_17766_b200.device import DevicePlan

    g = plans()
    for n in (2, 3, 4, 5, 7, 8, 10, 16, 32, 50, 64):
        pairs = lex_pairs(n)
        for seed in [int(s) for s in g["seeds"]]:
            dp = DevicePlan(n, len(pairs) + 3, seed, device=cuda_device)
            got = [tuple(p) for p in dp.assign.cpu().numpy().tolist()]
            assert got == [pairs[k] for k in g[f"n{n}_s{seed}"]], (n, seed)


@pytest.mark.parametrize("n,r,seed", [(64, 2, 0), (100, 2, 7), (362, 2, 3), (32, 3, 1), (50, 3, 2**63 - 1)])
def test_device_plan_matches_oracle_large(cuda_device, n, r, seed):
    from paper_2507_17766_b200.device import DevicePlan

    S = orc.n_shards(n, r)
    dp = DevicePlan(n, S + 11, seed, redundancy=r, device=cuda_device)
    want, bounds = orc.plan(n, S + 11, seed, r=r)
    assert np.array_equal(dp.assign.cpu().numpy(), want)
    assert np.array_equal(dp.bounds(), bounds)


# --------------------------------------------------------------------------- drop-in vs reference goldens


def _noise_callable(spec, plan, m, failures):
    k0, k1, amp, add = spec[2], spec[3], spec[1], spec[0] == orc.NOISE_ADD
    spans = [plan.bounds[s] for s, pair in enumerate(plan.assignment) if m in pair and m not in failures]
    state = {"k": 0}

    def fn(red):
        lo, hi = spans[state["k"]]
        state["k"] += 1
        noise = orc.noise_values(k0, k1, amp, lo, hi)
        return red + noise if add else noise

    return fn


@pytest.mark.parametrize("mode", ["callables", "descriptors"])
@pytest.mark.parametrize("meta", merge_cases(), ids=lambda m: m["name"])
def test_dropin_matches_reference(cuda_device, meta, mode):
    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200.simkernel import BlobStore

    meta, arr, payloads = load_case(meta)
    n, P = meta["n"], meta["P"]
    ids = meta["ids"] if meta["id_kind"] == "str" else list(range(n))
    pl = bf.plan_shards(bf.enumerate_pairs(n), P, bf.BYTES_PER_WEIGHT, meta["seed"])
    assert np.array_equal(np.array(pl.assignment), arr["assignment"])
    specs = corruption_specs(meta)
    if mode == "descriptors":
        corr = _descriptors(specs)
    else:
        corr = {}
        for m, spec in specs.items():
            if spec[0] == orc.ADD:
                corr[m] = lambda red, a=spec[1]: red + a
            elif spec[0] == orc.SCALE:
                corr[m] = lambda red, a=spec[1]: red * a
            else:
                corr[m] = _noise_callable(spec, pl, m, set(meta["failures"]))
    store = BlobStore()
    store.wire_ratio = meta["wire_ratio"]
    res = bf.run_all_reduce(store, {ids[k]: payloads[k] for k in range(n)}, pl,
                            failures=frozenset(meta["failures"]), corruptions=corr,
                            fallback=arr.get("fallback"), agreement_tolerance=meta["tol"])
    assert_same_floats(res.merged, arr["merged"])
    assert res.shard_status == [("merged", "lost", "disagreement")[c] for c in arr["status"]]
    assert res.flagged == {ids[k] for k in arr["flagged"]}
    assert_entries_close(res.agreement_matrix.entries, arr["entries"])
    meter = {a: [m.bytes_uploaded, m.bytes_downloaded] for a, m in store.meter.items()}
    assert meter == meta["meter"]
    assert list(meter) == list(meta["meter"])  # actor first-appearance order
    assert len(store.objects) == meta["n_objects"]


# --------------------------------------------------------------------------- device merge vs oracle


def _random_case(rng, n, P, r=2, dtype="f32"):
    if dtype == "bf16":
        bits = (rng.uniform(-1, 1, (n, P)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        return [bits[m] for m in range(n)]
    if dtype == "f64":
        return [rng.uniform(-1, 1, P) * 10.0 ** rng.integers(-3, 3) for _ in range(n)]
    x = rng.uniform(-1, 1, (n, P)) * (10.0 ** rng.integers(-6, 6, (n, 1)))
    return [x[m].astype(np.float32) for m in range(n)]


def _to_torch(reps, dtype, dev):
    if dtype == "bf16":
        return [torch.from_numpy(r.view(np.int16).copy()).to(dev).view(torch.bfloat16) for r in reps]
    return [torch.from_numpy(r.copy()).to(dev) for r in reps]


CASES = [
    # n, P, r, dtype, failures, corruptions, fallback
    (2, 1, 2, "f32", (), {}, False),
    (3, 3, 2, "f32", (), {}, False),
    (4, 17, 2, "f32", (1,), {}, True),
    (8, 28, 2, "f32", (), {}, False),            # width-1 shards
    (8, 45, 2, "f32", (2,), {3: (orc.ADD, 0.5)}, False),
    (12, 66 * 2 + 7, 2, "f32", (0, 5), {1: (orc.NOISE, 2.0, 11, 12), 7: (orc.SCALE, -2.0)}, True),
    (16, 1 << 16, 2, "f32", (), {}, False),
    (16, (1 << 16) + 13, 2, "f32", (3,), {4: (orc.NOISE_ADD, 1e-3, 5, 6), 9: (orc.ADD, 1e-7)}, True),
    (33, 200_003, 2, "f32", (1, 2, 30), {5: (orc.NOISE, 1.0, 1, 2), 6: (orc.NOISE, 1.0, 1, 2)}, False),
    (130, 8386, 2, "f32", (), {}, False),        # width-1 with > 128 alive (pairwise recursion)
    (5, 4099, 2, "f64", (4,), {0: (orc.ADD, 1.0)}, False),
    (9, 36 * 100 + 5, 2, "bf16", (2,), {1: (orc.ADD, 0.25)}, True),
    (6, 20 * 50 + 3, 3, "f32", (1,), {2: (orc.NOISE, 1.0, 3, 4)}, True),
    (7, 35 * 40 + 1, 3, "f32", (), {0: (orc.NOISE, 1.0, 8, 8), 3: (orc.NOISE, 1.0, 8, 8)}, False),
    (10, 120 * 64 + 9, 3, "bf16", (4, 5), {6: (orc.SCALE, -1.0)}, True),
]


# Shards of many k_reduce tiles: the reduce writes each special shard's predicted outcome
# and accumulates its pair statistics itself (r = 2); mispredictions (a zero `add`, a unit
# `scale`, colluders sharing a noise key all agree) are rewritten by k_apply.
LONG_CASES = [
    (4, (1 << 20) + 77, 2, "f32", (), {1: (orc.NOISE, 2.0, 5, 6)}, False),
    (6, (1 << 20) + 5, 2, "f32", (0,), {2: (orc.ADD, 0.0), 3: (orc.SCALE, 1.0), 4: (orc.NOISE, 1.0, 7, 7),
                                        5: (orc.NOISE, 1.0, 7, 7)}, True),
    (6, (1 << 20) + 5, 2, "f32", (), {2: (orc.ADD, 0.0), 4: (orc.NOISE, 1.0, 7, 7), 5: (orc.NOISE, 1.0, 7, 7)},
     False),
    (5, (1 << 19) + 11, 2, "bf16", (), {1: (orc.NOISE_ADD, 0.01, 3, 4)}, True),
    (4, (1 << 18) + 3, 2, "f64", (3,), {2: (orc.SCALE, 2.0)}, False),
    (7, 35 * 4096 + 3, 3, "f32", (1,), {2: (orc.NOISE, 1.0, 3, 4)}, True),   # r=3: predicted means
    (7, 35 * 4096 + 3, 3, "f32", (), {2: (orc.NOISE, 1.0, 3, 4), 4: (orc.ADD, 0.0)}, False),
]


@pytest.mark.parametrize("keep_means", [False, True], ids=["ws_in_merged", "ws_apart"])
@pytest.mark.parametrize("case", LONG_CASES, ids=lambda c: f"n{c[0]}_P{c[1]}_r{c[2]}_{c[3]}")
def test_device_merge_long_shards_match_oracle(cuda_device, case, keep_means):
    test_device_merge_matches_oracle(cuda_device, case, keep_means)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c[0]}_P{c[1]}_r{c[2]}_{c[3]}")
def test_device_merge_matches_oracle(cuda_device, case, keep_means=False):
    from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan

    n, P, r, dtype, failures, specs, use_fb = case
    rng = np.random.default_rng(n * 1000 + P)
    reps = _random_case(rng, n, P, r, dtype)
    fb = rng.uniform(-5, 5, P) if use_fb else None
    seed = int(rng.integers(0, 2**63))
    plan = DevicePlan(n, P, seed, redundancy=r, device=cuda_device)
    assign, bounds = orc.plan(n, P, seed, r=r)
    assert np.array_equal(plan.assign.cpu().numpy(), assign)
    odt = {"f32": orc.F32, "bf16": orc.BF16, "f64": orc.F64WIRE}[dtype]
    want = orc.merge(reps, assign, bounds, failures=failures, corruptions=specs, fallback=fb, dtype=odt)

    dreps = _to_torch(reps, dtype, cuda_device)
    job = ButterflyMerge(dreps, plan, failures=failures, corruptions=_descriptors(specs),
                         fallback=None if fb is None else torch.from_numpy(fb).to(cuda_device),
                         scatter_back=True, want_merged=True, keep_means=keep_means)
    job.run()
    torch.cuda.synchronize()
    assert_same_floats(job.merged.cpu().numpy(), want["merged"])
    assert np.array_equal(job.status.cpu().numpy(), want["status"])
    assert np.array_equal(job.flagged.cpu().numpy(), want["flagged"])
    assert_entries_close(job.entries.cpu().numpy(), want["entries"])
    # scatter-back: every miner now holds the merged vector rounded to its dtype
    m32 = want["merged"].astype(np.float32)
    for t in dreps:
        if dtype == "f32":
            assert_same_floats(t.cpu().numpy(), m32)
        elif dtype == "f64":
            assert_same_floats(t.cpu().numpy(), want["merged"])
        else:
            bits = np.array([orc.lib().orc_f32_to_bf16(float(v)) for v in m32[:257]], dtype=np.uint16)
            assert np.array_equal(t.view(torch.int16).cpu().numpy().view(np.uint16)[:257], bits)


@pytest.mark.parametrize("use_fb", [True, False], ids=["fallback", "no_fallback"])
@pytest.mark.parametrize("r", [2, 3])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
def test_device_merge_nonfinite(cuda_device, dtype, r, use_fb):
    """NaN / +-Inf weights (a diverged miner): a fast shard whose mean is not
    finite has identical NaN-scoring copies (butterfly.py:127-133), so it is a
    disagreement with every survivor flagged and the fallback adopted (:255,264-273);
    a lone survivor still merges its (NaN) mean.  Status, flags and entries are exact;
    values are exact with a fallback.  Without one, the scatter-back has already
    overwritten the lowest alive replica in place, so such shards take NaN."""
    from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan

    n, P = 7, (35 if r == 3 else 21) * 300 + 5
    rng = np.random.default_rng(99 + r)
    reps = _random_case(rng, n, P, r, dtype)
    poison = [(2, 100, "nan"), (5, 2000, "inf"), (0, 2000, "-inf"), (3, 4000, "nan"), (4, 5000, "nan"),
              (6, P - 1, "inf")]
    for m, e, v in poison:
        if dtype == "bf16":
            reps[m][e] = {"nan": 0x7FC0, "inf": 0x7F80, "-inf": 0xFF80}[v]
        else:
            reps[m][e] = float(v)
    failures = (4,)
    specs = {1: (orc.ADD, 0.5)}
    fb = rng.uniform(-5, 5, P) if use_fb else None
    seed = 1234 + r
    plan = DevicePlan(n, P, seed, redundancy=r, device=cuda_device)
    assign, bounds = orc.plan(n, P, seed, r=r)
    odt = {"f32": orc.F32, "bf16": orc.BF16, "f64": orc.F64WIRE}[dtype]
    want = orc.merge(reps, assign, bounds, failures=failures, corruptions=specs, fallback=fb, dtype=odt)
    dreps = _to_torch(reps, dtype, cuda_device)
    job = ButterflyMerge(dreps, plan, failures=failures, corruptions=_descriptors(specs),
                         fallback=None if fb is None else torch.from_numpy(fb).to(cuda_device),
                         scatter_back=True, want_merged=True)
    job.run()
    torch.cuda.synchronize()
    assert np.array_equal(job.status.cpu().numpy(), want["status"])
    assert np.array_equal(job.flagged.cpu().numpy(), want["flagged"])
    assert_entries_close(job.entries.cpu().numpy(), want["entries"])
    nonfin = job.nonfinite_shards()
    assert len(nonfin) >= 1  # the poison hit fast shards with >= 2 survivors
    expect = want["merged"].copy()
    if fb is None:
        for s in nonfin:
            expect[bounds[s]:bounds[s + 1]] = np.nan
    assert_same_floats(job.merged.cpu().numpy(), expect)
    if dtype == "f32":
        for t in dreps:
            assert_same_floats(t.cpu().numpy(), expect.astype(np.float32))


def test_agreement_and_mean_reducer_gpu(cuda_device):
    from _golden import agreement_cases

    from paper_2507_17766_b200 import butterfly as bf

    for c in agreement_cases():
        got = bf.agreement(np.array(c["a"]), np.array(c["b"]), c["tol"])
        if np.isnan(c["value"]):
            assert np.isnan(got)
        else:
            assert abs(got - c["value"]) <= 1e-12 and (got == 1.0) == (c["value"] == 1.0)
    rng = np.random.default_rng(5)
    for rows, width in ((1, 1), (7, 1), (9, 1), (200, 1), (3, 5), (64, 1001)):
        x = (rng.uniform(-1, 1, (rows, width)) * 10.0 ** rng.integers(-8, 8, (rows, width)))
        assert_same_floats(bf.mean_reducer(x), x.mean(axis=0))


@pytest.mark.parametrize("with_bad", [False, True], ids=["honest", "failures_and_corruptions"])
def test_pipelined_host_merge_matches_oracle(cuda_device, monkeypatch, with_bad):
    """bfly_merge_host with several chunks (small staging blocks): the upload, the
    per-chunk reduce and the per-chunk copy back agree with the oracle bit for bit."""
    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200.device import Corruption
    from paper_2507_17766_b200.simkernel import BlobStore

    monkeypatch.setattr(bf, "_UPLOAD_BLOCK", 4096)
    monkeypatch.setattr(bf, "_merge_chunks", lambda P: 7)
    n, P = 6, 100_003
    rng = np.random.default_rng(77)
    payloads = [rng.uniform(-1, 1, P) * 10.0 ** rng.integers(-3, 3) for _ in range(n)]
    plan = bf.plan_shards(bf.enumerate_pairs(n), P, bf.BYTES_PER_WEIGHT, 5)
    failures = (4,) if with_bad else ()
    specs = {1: (orc.NOISE, 1.0, 3, 4)} if with_bad else {}
    corr = {m: Corruption(KIND[s[0]], s[1], (s[2], s[3])) for m, s in specs.items()}
    res = bf.run_all_reduce(BlobStore(), {f"m{k}": payloads[k] for k in range(n)}, plan,
                            failures=frozenset(failures), corruptions=corr)
    assign = np.array(plan.assignment, dtype=np.int32)
    bounds = np.array([b for b, _ in plan.bounds] + [P], dtype=np.int64)
    want = orc.merge(payloads, assign, bounds, failures=failures, corruptions=specs, dtype=orc.F64WIRE)
    assert_same_floats(res.merged, want["merged"])
    assert res.shard_status == [("merged", "lost", "disagreement")[c] for c in want["status"]]


def test_store_objects_ranged_reads_gpu(cuda_device):
    """Every store object of a merge with a device-corrupted assignee: ranged reads
    (copied back range by range from HBM) equal slices of the whole object."""
    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200.device import Corruption
    from paper_2507_17766_b200.simkernel import BlobStore

    n, P = 5, 10_007
    rng = np.random.default_rng(5)
    payloads = {f"m{k}": rng.uniform(-1, 1, P) for k in range(n)}
    plan = bf.plan_shards(bf.enumerate_pairs(n), P, bf.BYTES_PER_WEIGHT, 9)
    store = BlobStore()
    bf.run_all_reduce(store, payloads, plan, corruptions={2: Corruption.noise(1.0, (4, 5))})
    for key, obj in store.objects.items():
        if not isinstance(obj, bf._LazyBlob):
            continue
        size = len(obj)
        cuts = [(0, 5), (3, 9), (size // 3, size // 3 + 101), (size - 6, size)]
        parts = [obj[a:b] for a, b in cuts]
        whole = bytes(obj)
        assert len(whole) == size
        for (a, b), got in zip(cuts, parts):
            assert got == whole[a:b], (key, a, b)


def test_captured_round_replays_match_oracle(cuda_device):
    """ButterflyMerge.capture(): one round as a CUDA graph; replays over replicas refilled
    in place give the oracle's results every round (corrupted and failed miners included)."""
    from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan

    n, P, seed = 6, (1 << 18) + 3, 11
    specs = {2: (orc.NOISE, 1.0, 3, 4)}
    plan = DevicePlan(n, P, seed, device=cuda_device)
    assign, bounds = orc.plan(n, P, seed)
    dreps = [torch.empty(P, dtype=torch.float32, device=cuda_device) for _ in range(n)]
    job = ButterflyMerge(dreps, plan, failures=(4,), corruptions=_descriptors(specs), want_merged=True)
    rng = np.random.default_rng(5)
    for rnd in range(4):
        reps = [rng.uniform(-1, 1, P).astype(np.float32) for _ in range(n)]
        for t, r in zip(dreps, reps):
            t.copy_(torch.from_numpy(r))
        if rnd == 1:
            job.capture()  # the capture's warm-up ran this round already; replay it again
            for t, r in zip(dreps, reps):
                t.copy_(torch.from_numpy(r))
        job.run()
        torch.cuda.synchronize()
        want = orc.merge(reps, assign, bounds, failures=(4,), corruptions=specs)
        assert_same_floats(job.merged.cpu().numpy(), want["merged"])
        assert np.array_equal(job.status.cpu().numpy(), want["status"])
        assert np.array_equal(job.flagged.cpu().numpy(), want["flagged"])
        assert_same_floats(dreps[0].cpu().numpy(), want["merged"].astype(np.float32))


def test_store_snapshot_and_no_device_references(cuda_device, monkeypatch):
    """Store ownership: by default the objects are views of the caller's payloads
    and of the returned merged vector — no object keeps the round's device memory alive;
    with SNAPSHOT_STORE every object is bytes when the call returns (simkernel.py:168)."""
    import gc
    import weakref

    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200.device import ButterflyMerge, Corruption
    from paper_2507_17766_b200.simkernel import BlobStore

    n, P = 5, 10_007
    rng = np.random.default_rng(8)
    payloads = {f"m{k}": rng.uniform(-1, 1, P) for k in range(n)}
    plan = bf.plan_shards(bf.enumerate_pairs(n), P, bf.BYTES_PER_WEIGHT, 3)
    jobs = []
    real_init = ButterflyMerge.__init__

    def spy(self, *a, **k):
        real_init(self, *a, **k)
        jobs.append(weakref.ref(self))

    monkeypatch.setattr(ButterflyMerge, "__init__", spy)
    store = BlobStore()
    res = bf.run_all_reduce(store, payloads, plan, corruptions={1: Corruption.noise(1.0, (2, 3))})
    gc.collect()
    assert jobs and all(j() is None for j in jobs), "a store object keeps the device job alive"
    want = {k: bytes(v) for k, v in store.objects.items()}
    monkeypatch.setattr(bf, "SNAPSHOT_STORE", True)
    store2 = BlobStore()
    res2 = bf.run_all_reduce(store2, payloads, plan, corruptions={1: Corruption.noise(1.0, (2, 3))})
    assert all(isinstance(v, bytes) for v in store2.objects.values())
    payloads["m0"][:] = 0.0  # the caller reuses its buffer: the snapshot does not change
    assert {k: bytes(v) for k, v in store2.objects.items()} == want
    assert_same_floats(res.merged, res2.merged)
