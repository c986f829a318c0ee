"""Host restatement of k_classify (multigpu.classify_host), which decides whether a
multi-GPU round can run as one persistent kernel and which shards must be
re-broadcast afterwards, checked against the oracle's decisions: fast shards are
merged from their lowest survivor, lost shards are lost, and a predicted outcome is
the reference's decision whenever the corrupted copies disagree with everything."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import oracle as orc  # noqa: E402

from paper_2507_17766_b200.multigpu import (  # noqa: E402
    CLS_FAST, CLS_LOST, CLS_SPECIAL, PRED_FALLBACK, PRED_MEAN, PRED_NONE, classify_host)

STATUS_MERGED, STATUS_LOST, STATUS_DISAGREE = 0, 1, 2


@pytest.mark.parametrize("seed", range(12))
def test_classify_host_matches_oracle_decisions(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 12))
    r = 3 if (seed % 3 == 0 and n >= 4) else 2
    P = int(rng.integers(40 * n * n, 80 * n * n))
    fails = set(int(x) for x in rng.choice(n, int(rng.integers(0, 3)), replace=False))
    alive = [m for m in range(n) if m not in fails]
    bad = set(int(x) for x in rng.choice(alive, min(len(alive), int(rng.integers(1, 3))), replace=False))
    # independent noise per corrupted miner: copies never agree with anything
    specs = {m: (orc.NOISE, 3.0, 1000 + m, 7) for m in bad}
    reps = [rng.uniform(-1, 1, P).astype(np.float32) for _ in range(n)]
    assign, bounds = orc.plan(n, P, seed, r=r)
    want = orc.merge(reps, assign, bounds, failures=tuple(sorted(fails)), corruptions=specs,
                     fallback=np.zeros(P))
    cls, pred = classify_host(assign, fails, bad, len(alive))
    for s in range(assign.shape[0]):
        surv = [int(m) for m in assign[s] if int(m) not in fails]
        if cls[s] == CLS_FAST:
            assert want["status"][s] == STATUS_MERGED and want["source"][s] == min(surv)
        elif cls[s] == CLS_LOST:
            assert not surv and want["status"][s] == STATUS_LOST and pred[s] == PRED_FALLBACK
        else:
            assert cls[s] == CLS_SPECIAL
            if pred[s] == PRED_MEAN:  # an honest majority adopts its (identical) copies
                assert want["status"][s] == STATUS_MERGED and int(want["source"][s]) not in bad
            elif pred[s] == PRED_FALLBACK:  # no majority among >= 2 survivors
                assert len(surv) >= 2 and want["status"][s] == STATUS_DISAGREE and want["source"][s] == -1
            else:  # a lone corrupted survivor: adopted, so no prediction of the fallback
                assert pred[s] == PRED_NONE and surv == [s_ for s_ in surv if s_ in bad] and len(surv) == 1
                assert want["status"][s] == STATUS_MERGED


def test_mispredicted_shards_are_the_unpredictable_ones():
    """Colluders sharing a noise key agree, so their shard adopts a corrupted copy
    although no majority was predicted; a lone corrupted survivor is adopted without a
    prediction.  Exactly those shards are re-broadcast after the persistent ring."""
    from paper_2507_17766_b200.multigpu import mispredicted_shards

    n, P, seed = 9, 9 * 8 * 40, 5
    rng = np.random.default_rng(3)
    reps = [rng.uniform(-1, 1, P).astype(np.float32) for _ in range(n)]
    fails = {0}
    bad = {3, 4, 1}  # 3 and 4 collude (one key); 0 failed, so shards (0, 1/3/4) keep a lone corrupted survivor
    specs = {3: (orc.NOISE, 2.0, 11, 11), 4: (orc.NOISE, 2.0, 11, 11), 1: (orc.NOISE, 2.0, 99, 1)}
    assign, bounds = orc.plan(n, P, seed)
    want = orc.merge(reps, assign, bounds, failures=tuple(fails), corruptions=specs, fallback=np.zeros(P))
    cls, pred = classify_host(assign, fails, bad, n - len(fails))
    kind = np.zeros(n, dtype=np.int32)
    for m in bad:
        kind[m] = 3
    special = np.flatnonzero(cls != CLS_FAST)
    mis = set(mispredicted_shards(special, pred, want["source"].astype(np.int64), kind).tolist())
    expect = set()
    for s in range(assign.shape[0]):
        pair = {int(x) for x in assign[s]}
        if pair == {3, 4} or (0 in pair and len(pair & bad) == 1):
            expect.add(s)
    assert mis == expect
