"""Full-size checks at BASELINE.json's configs.

* Config 1 (the reference's default, 8 miners x 10M fp32, r=2) runs in full through the
  drop-in API and is compared with the CPU oracle bit for bit (merged, status, flags).
* Config 2 (16 miners x 1e9 fp32) is too large for the oracle, so it is checked through
  size-independent properties: sampled elements equal the sequential fp64 mean recomputed
  from the original replicas, every replica ends identical, every shard merged, and a
  second merge round is a fixed point (the mean of identical fp32 values is exact).
* Config 5 (16 x 1e9, 6 noise-deceptive) and config 4 (32 x 1.75e9 bf16, r = 3, a failed
  and an adding miner) at full size: sampled shards re-decided by the oracle, every
  shard's status / flags against the closed form or the oracle's decisions.
* The persistent multi-GPU ring at full size as two loopback ranks on one GPU.
"""

import numpy as np
import pytest

import oracle as orc
from _golden import assert_entries_close, assert_same_floats

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_hbm():
    """Free HBM after handing the earlier tests' cached blocks back to the driver."""
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0]


def test_config1_full_size_matches_oracle(cuda_device):
    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200.simkernel import BlobStore

    n, P = 8, 10_000_000
    rng = np.random.default_rng(0)
    payloads = {m: rng.uniform(-1.0, 1.0, P) for m in range(n)}
    plan = bf.plan_shards(bf.enumerate_pairs(n), P, bf.BYTES_PER_WEIGHT, 0)
    res = bf.run_all_reduce(BlobStore(), payloads, plan, failures={3}, corruptions={5: bf.Corruption.add(0.25)})
    assign, bounds = orc.plan(n, P, 0)
    want = orc.merge([payloads[m] for m in range(n)], assign, bounds, failures=(3,),
                     corruptions={5: (orc.ADD, 0.25)}, dtype=orc.F64WIRE, threads=orc.threads_available())
    assert_same_floats(res.merged, want["merged"])
    assert res.shard_status == [orc.STATUS_NAMES[c] for c in want["status"]]
    assert res.flagged == set(np.flatnonzero(want["flagged"]).tolist())
    assert_entries_close(res.agreement_matrix.entries, want["entries"])


def test_config2_full_size_properties(cuda_device):
    from paper_2507_17766_b200.device import ButterflyMerge, DevicePlan

    free = _free_hbm()
    n, P = 16, 1_000_000_000
    if free < (2 * n + 4) * P * 4:
        pytest.skip("needs ~140 GB of free HBM")
    g = torch.Generator(device=cuda_device)
    reps = []
    for m in range(n):
        g.manual_seed(m)
        reps.append(torch.empty(P, dtype=torch.float32, device=cuda_device).uniform_(-1, 1, generator=g))
    idx = torch.from_numpy(np.random.default_rng(1).integers(0, P, 200_000)).to(cuda_device)
    before = torch.stack([r[idx] for r in reps]).double().cpu().numpy()  # (n, samples)
    plan = DevicePlan(n, P, 0, device=cuda_device)
    job = ButterflyMerge(reps, plan)
    job.run()
    torch.cuda.synchronize()
    acc = np.zeros(before.shape[1])
    for m in range(n):
        acc = acc + before[m]
    want = (acc / n).astype(np.float32)
    assert np.array_equal(reps[0][idx].cpu().numpy(), want)
    for r in reps[1:]:
        assert torch.equal(r[idx], reps[0][idx])
    assert int((job.status != 0).sum()) == 0 and int(job.flagged.sum()) == 0
    snap = reps[7][idx].clone()
    job.run()  # fixed point: merging identical replicas changes nothing
    torch.cuda.synchronize()
    assert torch.equal(reps[7][idx], snap)
    assert torch.equal(reps[3][: 1 << 20], reps[12][: 1 << 20])


def test_config5_full_size_sampled_shards(cuda_device):
    """Config 5 at full size: 16 miners x 1e9 fp32, 6 noise-deceptive
    miners (the bench's pattern: np.random.default_rng(0).choice(16, 6), noise amplitude 2
    keyed per miner).  Sampled shards — deceptive and honest ones — are snapshotted before
    the round and re-decided with the oracle's primitives (butterfly.py:216-273): the
    sequential fp64 mean in miner order, each assignee's copy (noise keyed by the global
    element index, orc.noise_values), orc.agreement, adoption or the lowest alive
    replica's values.  merged, status, entries and scatter-back must match bit for bit
    (entries <= 1e-12); the closed forms C(16,2) - C(10,2) = 75 disagreements and
    every miner flagged (each honest miner shares a shard with each deceptive one) hold."""
    from paper_2507_17766_b200.device import ButterflyMerge, Corruption, DevicePlan

    free = _free_hbm()
    n, P, amp = 16, 1_000_000_000, 2.0
    if free < (n + 6) * P * 4:
        pytest.skip("needs ~90 GB of free HBM")
    bad = sorted(int(x) for x in np.random.default_rng(0).choice(n, 6, replace=False))
    keys = {m: (0x5EED, m) for m in bad}
    g = torch.Generator(device=cuda_device)
    reps = []
    for m in range(n):
        g.manual_seed(m)
        reps.append(torch.empty(P, dtype=torch.float32, device=cuda_device).uniform_(-1, 1, generator=g))
    plan = DevicePlan(n, P, 0, device=cuda_device)
    assign, bounds = orc.plan(n, P, 0)
    assert np.array_equal(plan.assign.cpu().numpy(), assign)
    special = [s for s in range(len(assign)) if set(assign[s]) & set(bad)]
    fast = [s for s in range(len(assign)) if s not in special]
    rng = np.random.default_rng(5)
    sample = sorted(set(rng.choice(special, 6, replace=False).tolist()) |
                    set(rng.choice(fast, 3, replace=False).tolist()) | {0, len(assign) - 1})
    snap = {s: [r[bounds[s]:bounds[s + 1]].cpu().numpy() for r in reps] for s in sample}
    job = ButterflyMerge(reps, plan, corruptions={m: Corruption.noise(amp, keys[m]) for m in bad},
                         scatter_back=True, want_merged=True)
    job.run()
    torch.cuda.synchronize()
    status = job.status.cpu().numpy()
    entries = job.entries.cpu().numpy()
    assert int((status == orc.DISAGREEMENT).sum()) == 75 == len(special)
    assert np.array_equal(np.flatnonzero(status == orc.DISAGREEMENT), np.array(special))
    assert int(job.flagged.sum()) == n
    for s in sample:
        lo, hi = int(bounds[s]), int(bounds[s + 1])
        acc = np.zeros(hi - lo)
        for m in range(n):  # numpy's mean order: sequential fp64 sum in miner order, one divide
            acc = acc + snap[s][m].astype(np.float64)
        mean = acc / n
        i, j = (int(x) for x in assign[s])
        copy = {x: (orc.noise_values(*keys[x], amp, lo, hi) if x in bad else mean) for x in (i, j)}
        score = orc.agreement(copy[i], copy[j])
        want = copy[min(i, j)] if score == 1.0 else snap[s][0].astype(np.float64)
        assert status[s] == (orc.MERGED if score == 1.0 else orc.DISAGREEMENT), s
        assert abs(entries[i, j] - score) <= 1e-12 and entries[i, j] == entries[j, i], s
        assert_same_floats(job.merged[lo:hi].cpu().numpy(), want)
        assert_same_floats(reps[n - 1][lo:hi].cpu().numpy(), want.astype(np.float32))


def _bf16_rne(x32):
    """fp32 -> bf16 bits, round to nearest even (finite values)."""
    u = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def test_config4_full_size_sampled_shards(cuda_device):
    """Config 4 at full size: one stage of 32 miners x 1.75e9 bf16 parameters, r = 3 (the
    extension), with one failed miner and one miner adding 0.5 to its copies, so 465 of
    the 4960 shards are special and take the r = 3 majority rule through k_stats / k_decide
    at full scale.  Sampled shards are re-decided by the oracle on their own slices (a
    one-shard plan over the 32 miners' slices gives exactly that shard's decision, since an
    `add` corruption does not depend on the element index): status, the adopted source and
    the bf16 scatter-back bit for bit; status and flags of every shard against the oracle
    on the same assignment (no majority where the failed miner leaves the deceptive one
    with a single honest partner: both flagged)."""
    from paper_2507_17766_b200.device import ButterflyMerge, Corruption, DevicePlan

    free = _free_hbm()
    n, P, r = 32, 1_750_000_000, 3
    if free < n * P * 2 + 20 * P:
        pytest.skip("needs ~150 GB of free HBM")
    failed, bad, amp = 11, 7, 0.5
    g = torch.Generator(device=cuda_device)
    reps = []
    for m in range(n):
        g.manual_seed(100 + m)
        reps.append(torch.empty(P, dtype=torch.bfloat16, device=cuda_device).uniform_(-1, 1, generator=g))
    plan = DevicePlan(n, P, 3, redundancy=r, device=cuda_device)
    assign, bounds = orc.plan(n, P, 3, r=r)
    assert np.array_equal(plan.assign.cpu().numpy(), assign)
    special = [s for s in range(len(assign)) if bad in assign[s] or failed in assign[s]]
    fast = [s for s in range(len(assign)) if s not in special]
    rng = np.random.default_rng(9)
    sample = sorted(set(rng.choice(special, 6, replace=False).tolist()) |
                    set(rng.choice(fast, 3, replace=False).tolist()) | {0, len(assign) - 1})
    snap = {s: [r_[bounds[s]:bounds[s + 1]].view(torch.int16).cpu().numpy().view(np.uint16) for r_ in reps]
            for s in sample}
    job = ButterflyMerge(reps, plan, failures=(failed,), corruptions={bad: Corruption.add(amp)},
                         scatter_back=True, want_merged=False)
    job.run()
    torch.cuda.synchronize()
    status = job.status.cpu().numpy()
    source = job.source.cpu().numpy()
    # the flags follow from the per-shard decisions alone: the oracle on the same assignment
    # with 64 elements per shard (honest copies agree exactly; the +0.5 copy never does —
    # unlike one-element shards, whose cosine is always +-1)
    w = 64
    tiny = [np.random.default_rng(m).uniform(-1, 1, w * len(assign)).astype(np.float32) for m in range(n)]
    small = orc.merge(tiny, assign, np.arange(len(assign) + 1) * w, failures=(failed,),
                      corruptions={bad: (orc.ADD, amp)}, dtype=orc.F32)
    assert np.array_equal(job.flagged.cpu().numpy(), small["flagged"])
    assert np.array_equal(status, small["status"])
    for s in sample:
        lo, hi = int(bounds[s]), int(bounds[s + 1])
        want = orc.merge(snap[s], np.asarray([assign[s]], dtype=np.int32), np.asarray([0, hi - lo]),
                         failures=(failed,), corruptions={bad: (orc.ADD, amp)}, dtype=orc.BF16)
        assert status[s] == want["status"][0], s
        assert source[s] == want["source"][0], s
        bits = _bf16_rne(want["merged"].astype(np.float32))
        spot = [0, (hi - lo) // 2, hi - lo - 1]
        assert [int(orc.lib().orc_f32_to_bf16(float(want["merged"][k]))) for k in spot] == bits[spot].tolist()
        for m in (0, bad, failed, n - 1):  # scatter-back into every replica, the failed one included
            got = reps[m][lo:hi].view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(got, bits), (s, m)


def test_ring_loopback_two_ranks_full_size(cuda_device):
    """The persistent multi-GPU ring at full size on ONE GPU: 2 loopback ranks x 16 miners
    x 1e9 fp32 (32 miners, 496 shards), 6 noise-deceptive miners — config 5's pattern over
    two ranks.  k_ring streams 64 GB per rank through ~976k tiles (the schedule ring and
    the step counters wrap many times); the last rank predicts, finishes and re-broadcasts.
    Closed forms and sampled shards against the oracle (_multigpu_cases.fullsize_check);
    tests/test_multigpu_gpu.py runs the same case as 4 torchrun ranks on a 4-GPU box."""
    from _multigpu_cases import fullsize_case, fullsize_check, fullsize_rank

    from paper_2507_17766_b200.multigpu import run_loopback

    case = fullsize_case(world=2)
    if _free_hbm() < (case["n"] + 4) * case["P"] * 4:
        pytest.skip("needs ~145 GB of free HBM")
    res = run_loopback(2, lambda rank, comm: fullsize_rank(case, rank, comm, cuda_device), device=cuda_device,
                       timeout=600.0)
    fullsize_check(case, res)
