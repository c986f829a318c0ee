"""Randomised parity: 150 device merges with random miner counts, lengths (incl. width-1
and multi-tile shards), redundancy, dtype, failures, corruption kinds / amplitudes /
shared keys (colluders), fallback or not, scatter-back — each bit-exact against the
oracle (merged, scatter-back, status, flags; agreement entries within 1e-12)."""

import os

import numpy as np
import pytest

from _golden import assert_entries_close, assert_same_floats

import oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KIND = {orc.ADD: "add", orc.SCALE: "scale", orc.NOISE: "noise", orc.NOISE_ADD: "noise_add"}


def _case(seed):
    rng = np.random.default_rng(seed)
    r = 3 if rng.random() < 0.25 else 2
    n = int(rng.integers(r, 14 if r == 3 else 40))
    S = orc.n_shards(n, r)
    width = int(rng.choice([1, 2, 7, 300, 2500, 6000]))
    P = max(S, S * width + int(rng.integers(0, S)))
    dtype = str(rng.choice(["f32", "f32", "bf16", "f64"]))
    nfail = int(rng.integers(0, max(1, n // 3)))
    failures = tuple(sorted(int(x) for x in rng.choice(n, nfail, replace=False))) if nfail else ()
    specs = {}
    for m in rng.choice(n, int(rng.integers(0, max(1, n // 4) + 1)), replace=False):
        kind = int(rng.choice([orc.ADD, orc.SCALE, orc.NOISE, orc.NOISE_ADD]))
        # Amplitudes keep every agreement decision away from cosine == 1.0 within rounding:
        # copies that are (nearly) parallel — a positive scale, two scales of one sign, an
        # offset tiny against a mean of up to 1e6 — decide `score == 1.0` by the dot-product
        # order (the reference's BLAS included): the documented non-portable case.
        key = int(rng.integers(0, 3))  # small key space: colluders share keys
        if kind == orc.NOISE:  # one amplitude per key: shared keys give identical copies,
            amp = (1e-3, 0.5, 2.0)[key]  # not parallel ones
        elif kind == orc.NOISE_ADD:
            amp = (1e-9, 2.0, 50.0)[key]
        elif kind == orc.ADD:  # identical, decided by max|a-b| <= tol, or far from parallel
            amp = float(rng.choice([0.0, 1e-9, 2.0, 50.0]))
        else:  # scale: a zero copy or the mean's mirror image
            amp = float(rng.choice([0.0, -1.0]))
        specs[int(m)] = (kind, amp, key, key + 1)
    return n, P, r, dtype, failures, specs, bool(rng.random() < 0.5), int(rng.integers(0, 2**63))


def _reps(rng, n, P, dtype):
    if dtype == "bf16":
        bits = (rng.uniform(-1, 1, (n, P)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        return [bits[m] for m in range(n)]
    if dtype == "f64":
        return [rng.uniform(-1, 1, P) * 10.0 ** rng.integers(-3, 3) for _ in range(n)]
    x = rng.uniform(-1, 1, (n, P)) * (10.0 ** rng.integers(-6, 6, (n, 1)))
    return [x[m].astype(np.float32) for m in range(n)]


# BFLY_FUZZ_SEEDS extends the range for a soak run (profiles/r02_fuzz_soak.log)
@pytest.mark.parametrize("seed", range(int(os.environ.get("BFLY_FUZZ_SEEDS", "150"))))
def test_random_merge_matches_oracle(cuda_device, seed):
    from paper_2507_17766_b200.device import ButterflyMerge, Corruption, DevicePlan

    n, P, r, dtype, failures, specs, use_fb, plan_seed = _case(seed)
    rng = np.random.default_rng(10_000 + seed)
    reps = _reps(rng, n, P, dtype)
    fb = rng.uniform(-5, 5, P) if use_fb else None
    plan = DevicePlan(n, P, plan_seed, redundancy=r, device=cuda_device)
    assign, bounds = orc.plan(n, P, plan_seed, r=r)
    assert np.array_equal(plan.assign.cpu().numpy(), assign)
    odt = {"f32": orc.F32, "bf16": orc.BF16, "f64": orc.F64WIRE}[dtype]
    want = orc.merge(reps, assign, bounds, failures=failures, corruptions=specs, fallback=fb, dtype=odt)
    if dtype == "bf16":
        dreps = [torch.from_numpy(x.view(np.int16).copy()).to(cuda_device).view(torch.bfloat16) for x in reps]
    else:
        dreps = [torch.from_numpy(x.copy()).to(cuda_device) for x in reps]
    corr = {m: Corruption(KIND[s[0]], s[1], (s[2], s[3])) for m, s in specs.items()}
    job = ButterflyMerge(dreps, plan, failures=failures, corruptions=corr,
                         fallback=None if fb is None else torch.from_numpy(fb).to(cuda_device),
                         want_merged=True, keep_means=bool(seed % 2))
    job.run()
    torch.cuda.synchronize()
    assert_same_floats(job.merged.cpu().numpy(), want["merged"])
    assert np.array_equal(job.status.cpu().numpy(), want["status"])
    assert np.array_equal(job.flagged.cpu().numpy(), want["flagged"])
    assert_entries_close(job.entries.cpu().numpy(), want["entries"])
    if dtype == "f32":
        assert_same_floats(dreps[-1].cpu().numpy(), want["merged"].astype(np.float32))
    elif dtype == "f64":
        assert_same_floats(dreps[-1].cpu().numpy(), want["merged"])
