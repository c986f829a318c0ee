"""The C ABI (include/bfly.h): library loads, exports every declared symbol,
struct layouts agree with ctypes, and the host-side entry points (no GPU
needed) match the reference: SHA-256 keys, the host index map, error codes."""

import ctypes
import hashlib
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle as orc
from _golden import lex_pairs, plans

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "bfly.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(bfly_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2507_17766_b200 import _lib

    L = _lib.lib()
    declared = _declared()
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.bfly_version().decode().startswith("bfly ")
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib._SO)], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", nm), name


def test_struct_layout_matches_header(tmp_path):
    from paper_2507_17766_b200 import _lib

    src = tmp_path / "layout.c"
    fields = [f for f, _ in _lib.MergeArgs._fields_]
    rfields = [f for f, _ in _lib.RingDesc._fields_]
    body = "\n".join(f'  printf("{f} %zu\\n", offsetof(bfly_merge_args_t, {f}));' for f in fields)
    body += "\n" + "\n".join(f'  printf("ring.{f} %zu\\n", offsetof(bfly_ring_desc_t, {f}));' for f in rfields)
    body += '\n  printf("rsize %zu\\n", sizeof(bfly_ring_desc_t));'
    ffields = [f for f, _ in _lib.RingFusedDesc._fields_]
    body += "\n" + "\n".join(f'  printf("fused.{f} %zu\\n", offsetof(bfly_ring_fused_desc_t, {f}));'
                             for f in ffields)
    body += '\n  printf("fsize %zu\\n", sizeof(bfly_ring_fused_desc_t));'
    src.write_text(f"""#include <stdio.h>
#include <stddef.h>
#include "bfly.h"
int main(void) {{
  printf("size %zu\\n", sizeof(bfly_merge_args_t));
  printf("csize %zu\\n", sizeof(bfly_corruption_t));
{body}
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    assert int(out["size"]) == ctypes.sizeof(_lib.MergeArgs)
    assert int(out["csize"]) == ctypes.sizeof(_lib.Corruption)
    for f in fields:
        assert int(out[f]) == getattr(_lib.MergeArgs, f).offset, f
    assert int(out["rsize"]) == ctypes.sizeof(_lib.RingDesc)
    for f in rfields:
        assert int(out["ring." + f]) == getattr(_lib.RingDesc, f).offset, f
    assert int(out["fsize"]) == ctypes.sizeof(_lib.RingFusedDesc)
    for f in ffields:
        assert int(out["fused." + f]) == getattr(_lib.RingFusedDesc, f).offset, f


def test_fused_ring_layout():
    """Region of the persistent ring (bfly_ring_fused_layout): per lane NB running-sum
    slots (one tile at accumulator width), NB final-vector slots (one tile at replica
    width), the five 64-bit flag arrays, the step counts and the tile counter; every part
    256-byte aligned."""
    from paper_2507_17766_b200 import _lib

    lib = _lib.lib()
    # a tile is 4 KB of every replica: 1024 fp32 / 2048 bf16 / 512 fp64 elements; every
    # slot starts with a 16-byte header (the tile id, -1 = the lane's last step)
    def align(x):
        return (x + 255) // 256 * 256

    for dtype, acc_b, fin_b in ((_lib.F32, 16 + 1024 * 8, 16 + 4096), (_lib.BF16, 16 + 2048 * 4, 16 + 4096),
                                (_lib.F64WIRE, 16 + 512 * 8, 16 + 4096)):
        o = [ctypes.c_int64() for _ in range(3)]
        _lib.check(lib.bfly_ring_fused_layout(148, 4, dtype, *[ctypes.byref(x) for x in o]))
        off_fin, off_flags, total = (x.value for x in o)
        assert off_fin == align(148 * 4 * acc_b)
        assert off_flags == align(off_fin + 148 * 4 * fin_b)
        # flags, the persisted step counts of both lane sides, rank 0's tile counter, the
        # tile schedule rank 0 writes ahead (512 words per lane)
        assert total == align(align(align(align(off_flags + 5 * 148 * 8) + 2 * 148 * 8) + 8) + 512 * 148 * 8)
    with pytest.raises(Exception):
        _lib.check(lib.bfly_ring_fused_layout(148, 1, _lib.F32, *[ctypes.byref(ctypes.c_int64()) for _ in range(3)]))


@pytest.mark.parametrize("seed", [0, 1, 24, 2**63 - 1, 2**64 + 5, -7, 10**30])
def test_philox_key_matches_hashlib(seed):
    from paper_2507_17766_b200 import _lib

    for stream in ("shard-plan", "root/epoch0/plan/sync/L0", "resilience"):
        d = hashlib.sha256(f"{seed}\x1f{stream}".encode()).digest()
        want = (int.from_bytes(d[:8], "little"), int.from_bytes(d[8:16], "little"))
        assert _lib.philox_key(seed, stream) == want


def test_host_plan_matches_reference_goldens():
    from paper_2507_17766_b200 import butterfly as bf

    g = plans()
    for n in (2, 3, 4, 5, 7, 8, 10, 16, 32, 50, 64):
        pairs = lex_pairs(n)
        for seed in [int(s) for s in g["seeds"]]:
            plan = bf.plan_shards(bf.enumerate_pairs(n), len(pairs) + 3, 4, seed)
            assert list(plan.assignment) == [pairs[k] for k in g[f"n{n}_s{seed}"]]


@pytest.mark.parametrize("n,r", [(6, 3), (32, 3), (200, 2), (400, 2)])
def test_host_plan_matches_oracle_r3_and_large(n, r):
    from paper_2507_17766_b200 import butterfly as bf

    S = orc.n_shards(n, r)
    assign, bounds = bf._host_plan(n, r, S * 3 + 1, 99)
    want, wb = orc.plan(n, S * 3 + 1, 99, r=r)
    assert np.array_equal(assign, want) and np.array_equal(bounds, wb)


def test_error_mapping():
    from paper_2507_17766_b200 import butterfly as bf
    from paper_2507_17766_b200 import errors

    with pytest.raises(errors.TooFewMinersError):
        bf.enumerate_pairs(1)
    with pytest.raises(errors.DegenerateShardsError):
        bf.plan_shards(bf.enumerate_pairs(3), 2, 4, 0)
    with pytest.raises(errors.TooFewMinersError):
        bf._host_plan(1, 2, 10, 0)
    with pytest.raises(errors.DegenerateShardsError):
        bf._host_plan(4, 2, 5, 0)
    assert bf.valid_shard_fraction(50, 5) == pytest.approx(1.0 - 20.0 / 2450.0)
    with pytest.raises(errors.InvalidArgumentError):
        bf.valid_shard_fraction(10, 11)


def test_plan_metadata_and_helpers():
    from paper_2507_17766_b200 import butterfly as bf

    plan = bf.plan_shards(bf.enumerate_pairs(3), 10, 4, 0)
    assert [e - s for s, e in plan.bounds] == [4, 3, 3]
    assert plan.byte_bounds(1) == (16, 28)
    assert plan.metadata() == b"[[0, 0, 16], [1, 16, 12], [2, 28, 12]]"
    assert sorted(s for m in range(3) for s in plan.shards_of(m)) == [0, 0, 1, 1, 2, 2]


def test_fused_ring_rejects_bad_descriptors():
    """bfly_ring_fused validates its descriptor before any CUDA call (so this runs
    without a GPU): ring size, slots, ranks beyond the schedule ring, a last rank
    without an alive miner, special shards without the merge arguments."""
    from paper_2507_17766_b200 import _lib, errors

    lib = _lib.lib()
    peers = (ctypes.c_uint64 * 17)(*[0x10000 * (r + 1) for r in range(17)])

    def call(**kw):
        d = _lib.RingFusedDesc()
        d.rank, d.world, d.lanes, d.nb, d.dtype = 0, 2, 148, 10, _lib.F32
        d.n_src = d.n_dst = 0
        d.n_div = 4
        d.payload_len = 1 << 20
        d.peer_base = ctypes.cast(peers, ctypes.c_void_p)
        for k, v in kw.items():
            setattr(d, k, v)
        _lib.check(lib.bfly_ring_fused(ctypes.byref(d), None))

    with pytest.raises(errors.InvalidArgumentError):
        call(world=1)
    with pytest.raises(errors.InvalidArgumentError):
        call(nb=1)
    with pytest.raises(errors.InvalidArgumentError):
        call(rank=1, n_div=0)  # the last rank divides by the alive miners
    with pytest.raises(errors.InvalidArgumentError):
        call(rank=1, special=1)  # special shards need the merge arguments
    with pytest.raises(NotImplementedError):
        call(world=17)
    with pytest.raises(NotImplementedError):
        call(world=8, nb=70)  # 7 x (8 + 70) + 1 > 512 schedule words per lane


def test_round2_entry_points_check_arguments_before_cuda():
    """The round-2 entry points reject bad arguments with the mapped status before any
    CUDA call (so on a machine without a GPU too)."""
    import ctypes

    from paper_2507_17766_b200 import _lib as L

    lib = L.lib()
    descs = (L.RingFusedDesc * 2)()
    assert lib.bfly_ring_fused_loopback(descs, 1, None) == L.E_INVALID_ARG  # world < 2
    assert lib.bfly_ring_fused_loopback(descs, 9, None) == L.E_INVALID_ARG  # world > 8
    descs[0].rank, descs[1].rank = 0, 0  # rank 1 mislabelled
    descs[0].world = descs[1].world = 2
    assert lib.bfly_ring_fused_loopback(descs, 2, None) == L.E_INVALID_ARG
    assert b"disagree" in lib.bfly_last_error()
    assert lib.bfly_fill_shards(None, None, None, None, 1, L.F32, 100, 10, None) == L.E_INVALID_ARG
    assert lib.bfly_permutation_host(-1, 0, 0, None) == L.E_INVALID_ARG
    out = (ctypes.c_int64 * 5)()
    assert lib.bfly_permutation_host(5, 1, 2, out) == L.OK
    assert sorted(out) == [0, 1, 2, 3, 4]
    assert lib.bfly_ring_fused_stat_tile(L.F64WIRE) == 0
    assert lib.bfly_ring_fused_stat_tile(L.F32) % 1024 == 0
    out_s = ctypes.c_void_p()
    assert lib.bfly_stream_create(0, None) == L.E_INVALID_ARG


def test_plan_shards_custom_pair_set_matches_reference():
    """A caller-built PairSet (a subset of pairs, another order) is permuted as the
    reference permutes it, pairs[order[s]] (butterfly.py:98-100)."""
    import importlib

    import pytest

    try:
        ref = importlib.import_module("iota_sim.butterfly")
    except ImportError:
        pytest.skip("the reference (baseline/_ref) is not installed")
    from paper_2507_17766_b200 import butterfly as bf

    for pairs, P, seed in [(((0, 1), (2, 3), (0, 2)), 30, 5), (((3, 4), (0, 1), (1, 4), (0, 3), (2, 3)), 101, 2**63 + 7),
                           (tuple((i, j) for i in range(6) for j in range(i + 1, 6))[::-1], 77, 11)]:
        ps = ref.PairSet(6, pairs)
        want = ref.plan_shards(ps, P, 4, seed)
        got = bf.plan_shards(ps, P, 4, seed)
        assert got.assignment == want.assignment and got.bounds == want.bounds
        assert type(got) is type(want)
