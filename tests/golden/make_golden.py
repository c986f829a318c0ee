"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports iota_sim from /root/reference/pkg/src and records, for seeded
inputs, what the reference itself returns:

* plans.npz         — plan_shards assignments (as lexicographic pair ranks) for
                      many (N, seed), incl. the seed-24 KAT (tests/test_butterfly.py:37-40)
                      and seeds >= 2**63; plus bounds for ragged P;
* merge_*.npz       — run_all_reduce outputs (merged, status, entries, flagged,
                      per-actor meter) for edge cases: failures, fallbacks, lost
                      shards, width-1 shards (numpy pairwise order), additive /
                      noise / colluding corruptions, string miner ids, wire_ratio;
* agreement.json    — agreement() values incl. the clamped cosine and NaN cases.

Corruptions are numpy callables with the exact semantics of the descriptor
kinds in include/bfly.h; NOISE draws word e of Philox(key).random_raw for
global element e, so a callable that is handed only the reduction tracks its
position through the reference's own call order (shard ascending, butterfly.py:219-233).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from iota_sim import butterfly  # noqa: E402
from iota_sim.simkernel import BlobStore  # noqa: E402

OUT = Path(__file__).resolve().parent
ADD, SCALE, NOISE, NOISE_ADD = 1, 2, 3, 4


def lex_rank(n, pair):
    i, j = pair
    return i * (2 * n - i - 1) // 2 + (j - i - 1)


def make_plans():
    rows = {}
    seeds = list(range(0, 40)) + [24, 123456789012345678, 2**63 - 1, 2**63, 2**64 + 5, 10**30]
    for n in (2, 3, 4, 5, 7, 8, 10, 16, 32, 50, 64):
        S = n * (n - 1) // 2
        for seed in seeds:
            plan = butterfly.plan_shards(butterfly.enumerate_pairs(n), S + 3, 4, seed)
            rows[f"n{n}_s{seed}"] = np.array([lex_rank(n, p) for p in plan.assignment], dtype=np.int32)
    bounds = {}
    for n, P in ((3, 10), (3, 9), (8, 1000), (8, 10_000_001), (10, 45), (10, 89), (64, 2017)):
        plan = butterfly.plan_shards(butterfly.enumerate_pairs(n), P, 4, 0)
        bounds[f"b_n{n}_P{P}"] = np.array([plan.bounds[0][0]] + [e for _, e in plan.bounds], dtype=np.int64)
    np.savez_compressed(OUT / "plans.npz", seeds=np.array([str(s) for s in seeds]), **rows, **bounds)


class NoiseCallable:
    """Descriptor NOISE / NOISE_ADD as a reference corruption callable."""

    def __init__(self, key0, key1, amp, add, spans):
        self.key = np.array([key0, key1], dtype=np.uint64)
        self.amp, self.add, self.spans, self.k = amp, add, list(spans), 0

    def __call__(self, red):
        start, stop = self.spans[self.k]
        self.k += 1
        assert len(red) == stop - start
        raw = np.random.Philox(key=self.key).random_raw(stop)[start:stop]
        unit = (raw >> np.uint64(11)).astype(np.float64) * (1.0 / 4503599627370496.0) - 1.0
        noise = self.amp * unit
        return red + noise if self.add else noise


def spans_for(plan, miner, failures):
    return [plan.bounds[s] for s, pair in enumerate(plan.assignment) if miner in pair and miner not in failures]


def run_case(name, n, P, seed, *, payload_seed=0, failures=(), corr=None, fallback=None,
             ids=None, wire_ratio=1.0, tol=1e-6, store_payloads=True, poison=()):
    rng = np.random.default_rng(payload_seed)
    payloads_arr = [rng.uniform(-1.0, 1.0, P) for _ in range(n)]
    for m, e, v in poison:  # a diverged miner: NaN / +-Inf weights (fp64, so also on the wire)
        payloads_arr[m][e] = v
    ids = ids if ids is not None else list(range(n))
    payloads = {ids[m]: payloads_arr[m] for m in range(n)}
    sorted_ids = sorted(payloads)
    plan = butterfly.plan_shards(butterfly.enumerate_pairs(n), P, 4, seed)
    corr = corr or {}
    callables = {}
    for m, spec in corr.items():
        kind, a = spec[0], spec[1]
        if kind == ADD:
            callables[m] = lambda red, a=a: red + a
        elif kind == SCALE:
            callables[m] = lambda red, a=a: red * a
        else:
            callables[m] = NoiseCallable(spec[2], spec[3], a, kind == NOISE_ADD, spans_for(plan, m, failures))
    fb = None
    if fallback == "zeros":
        fb = np.zeros(P)
    elif fallback == "ramp":
        fb = np.linspace(-3.0, 3.0, P)
    store = BlobStore()
    store.wire_ratio = wire_ratio
    res = butterfly.run_all_reduce(store, payloads, plan, failures=frozenset(failures),
                                   corruptions=callables, fallback=fb, agreement_tolerance=tol)
    status = np.array([("merged", "lost", "disagreement").index(s) for s in res.shard_status], dtype=np.uint8)
    flagged = np.array(sorted(sorted_ids.index(k) for k in res.flagged), dtype=np.int32)
    meter = {a: [m.bytes_uploaded, m.bytes_downloaded] for a, m in store.meter.items()}
    wire = np.stack([_wire(sorted_ids, payloads, k) for k in range(n)])
    meta = dict(name=name, n=n, P=P, seed=seed, payload_seed=payload_seed, failures=list(failures),
                corruptions={str(k): list(v) for k, v in corr.items()}, fallback=fallback,
                ids=[str(i) for i in sorted_ids], id_kind="str" if isinstance(ids[0], str) else "int",
                wire_ratio=wire_ratio, tol=tol, meter=meter, n_objects=len(store.objects),
                poison=[[int(m), int(e), repr(float(v))] for m, e, v in poison],
                objects_sha256=hashlib.sha256("\n".join(sorted(store.objects)).encode()).hexdigest(),
                payload_sha256=hashlib.sha256(wire.tobytes()).hexdigest(),
                store_payloads=store_payloads)
    arrays = dict(merged=res.merged, status=status, entries=res.agreement_matrix.entries,
                  flagged=flagged, assignment=np.array(plan.assignment, dtype=np.int32))
    if store_payloads:
        arrays["payloads"] = np.stack([payloads[k] for k in sorted_ids])
    if fb is not None:
        arrays["fallback"] = fb
    np.savez_compressed(OUT / f"merge_{name}.npz", **arrays)
    return meta


def _wire(sorted_ids, payloads, k):
    return payloads[sorted_ids[k]].astype(np.float32)


def make_merges():
    K = (0x243F6A8885A308D3, 0x13198A2E03707344)
    K2 = (0xA4093822299F31D0, 0x082EFA98EC4E6C89)
    cases = [
        run_case("honest_n4", 4, 100, 1),
        run_case("fail1_n5", 5, 60, 2, failures=(3,)),
        run_case("pairfail_n3", 3, 30, 3, failures=(0, 1), fallback="zeros"),
        run_case("pairfail_nofb_n3", 3, 31, 3, failures=(0, 1)),
        run_case("allfail_n3", 3, 12, 7, failures=(0, 1, 2)),
        run_case("add_n4", 4, 80, 4, corr={2: (ADD, 1.0)}, fallback="zeros"),
        run_case("add_tol_edge_n5", 5, 50, 9, corr={1: (ADD, 1e-6), 3: (ADD, 1.0000001e-6)}, fallback="ramp"),
        run_case("noise_n10", 10, 10 * 45 + 7, 11, corr={0: (NOISE, 2.0, *K), 5: (NOISE_ADD, 0.5, *K2)},
                 fallback="ramp"),
        run_case("collude_n8", 8, 28 * 20 + 3, 12, corr={1: (NOISE, 1.0, *K), 2: (NOISE, 1.0, *K)},
                 fallback="zeros"),
        run_case("corrupt_partner_failed_n6", 6, 150, 13, failures=(2,), corr={4: (ADD, 0.25)}),
        run_case("mixed_n12", 12, 66 * 13 + 5, 14, failures=(3, 7), corr={0: (ADD, -0.5), 9: (NOISE, 3.0, *K2)},
                 fallback="ramp"),
        run_case("width1_n8", 8, 40, 5),
        run_case("width1_n20", 20, 200, 6, failures=(4,)),
        run_case("width1_n130", 130, 8386, 8, store_payloads=False),
        run_case("strids_n11", 11, 55 * 3 + 1, 15,
                 ids=[f"m0.{k}" for k in range(11)], corr={2: (ADD, 2.0)}, failures=(5,)),
        run_case("wire_ratio_n6", 6, 15 * 7 + 2, 16, wire_ratio=3.7, failures=(1,)),
        run_case("meter_n2", 2, 1000, 2),
        run_case("meter_n3", 3, 1000, 3),
        run_case("meter_n10", 10, 1000, 10),
        run_case("meter_n50", 50, 9800, 50, store_payloads=False),
        run_case("crit4_small_n50", 50, 1225 * 16, 4, payload_seed=4,
                 corr={m: (NOISE, 1.5, K[0] + m, K[1]) for m in range(10)}, fallback="zeros",
                 store_payloads=False),
        # non-finite weights: identical NaN copies score NaN, so the shard
        # is a disagreement, both assignees are flagged and the fallback is used
        run_case("nonfinite_nofb_n5", 5, 53, 17, poison=[(2, 7, np.nan), (0, 30, np.inf), (4, 44, -np.inf)]),
        run_case("nonfinite_fb_n6", 6, 15 * 9 + 4, 18, failures=(1,), fallback="ramp",
                 poison=[(0, e, np.nan) for e in range(0, 139, 9)] + [(3, 11, np.inf), (5, 11, -np.inf)]),
        run_case("nonfinite_corrupt_n7", 7, 21 * 6 + 1, 19, corr={3: (ADD, 0.5)}, failures=(6,),
                 poison=[(4, e, np.inf) for e in range(2, 127, 11)]),
    ]
    (OUT / "merge_cases.json").write_text(json.dumps(cases, indent=1))


def make_agreement():
    vecs = []
    rng = np.random.default_rng(3)
    cases = [
        ([1.0, 2.0, 3.0], [1.0 + 1e-9, 2.0 + 1e-9, 3.0 + 1e-9]),
        ([1.0, 0.0], [1.0, 1.0]),
        ([1.0, 0.0], [-1.0, 0.0]),
        ([0.0, 0.0], [1.0, 0.0]),
        ([1.0, float("nan")], [1.0, 2.0]),
        ([], []),
        (list(rng.uniform(-1, 1, 1000)), list(rng.uniform(-1, 1, 1000))),
    ]
    base = rng.uniform(-1, 1, 4097)
    cases.append((list(base), list(base + 2e-6)))
    cases.append((list(base), list(base + 5e-7)))
    for a, b in cases:
        vecs.append(dict(a=a, b=b, tol=1e-6, value=butterfly.agreement(np.array(a), np.array(b), 1e-6)))
    (OUT / "agreement.json").write_text(json.dumps(vecs))


if __name__ == "__main__":
    make_plans()
    make_agreement()
    make_merges()
    print("golden fixtures written to", OUT)
