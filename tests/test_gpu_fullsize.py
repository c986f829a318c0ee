"""Full-size checks at BASELINE.json's configs.

* Config 1 (the reference's default, 8 miners x 10M fp32, r=2) runs in full through the
  drop-in API and is compared with the CPU oracle bit for bit (merged, status, flags).
* Config 2 (16 miners x 1e9 fp32) is too large for the oracle, so it is checked through
  size-independent properties: sampled elements equal the sequential fp64 mean recomputed
  from the original replicas, every replica ends identical, every shard merged, and a
  second merge round is a fixed point (the mean of identical fp32 values is exact).
"""

import numpy as np
import pytest

import oracle as orc
from _golden import assert_entries_close, assert_same_floats

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


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

    free, _ = torch.cuda.mem_get_info()
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
