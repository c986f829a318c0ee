"""Store objects of the merge are lazily materialised views of (device) vectors in the
"<f4" wire format: a ranged BlobStore.get copies only that range back and returns the
same bytes as slicing the fully materialised object (simkernel.py:174-186)."""

import numpy as np

from paper_2507_17766_b200 import butterfly as bf
from paper_2507_17766_b200.simkernel import BlobStore


def test_ranged_reads_equal_full_materialisation():
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, 1001) * 1e3
    calls = []

    def part(a, b):
        calls.append((a, b))
        return bf._wire_part(v)(a, b)

    full = v.astype("<f4").tobytes()
    lazy = bf._LazyBlob(len(full), lambda: full, part)
    store = BlobStore()
    store.objects["k"] = lazy
    for start, length in [(0, 1), (1, 7), (3, 4), (15, 17), (16, 0), (len(full) - 3, None), (0, None),
                          (len(full) + 5, 3), (2, 10_000)]:
        got = store.get("actor", "k", start, length)
        want = full[start:] if length is None else full[start:start + length]
        assert got == want, (start, length)
    assert calls and lazy._data is None  # never materialised whole
    assert store.meter["actor"].bytes_downloaded == sum(
        len(full[s:] if n is None else full[s:s + n]) for s, n in
        [(0, 1), (1, 7), (3, 4), (15, 17), (16, 0), (len(full) - 3, None), (0, None), (len(full) + 5, 3),
         (2, 10_000)])
    assert bytes(lazy) == full and len(lazy) == len(full)


def test_snapshot_store_copies_at_round_end(monkeypatch):
    """SNAPSHOT_STORE: objects are bytes when written (the reference's put copies,
    simkernel.py:168); by default they are views of the caller's vector."""
    v = np.linspace(-1, 1, 37)
    lazy = bf._wire_blob(v, 4 * v.size)
    assert isinstance(lazy, bf._LazyBlob)
    monkeypatch.setattr(bf, "SNAPSHOT_STORE", True)
    snap = bf._wire_blob(v, 4 * v.size)
    assert isinstance(snap, bytes) and snap == v.astype("<f4").tobytes()
    v[3] = 123.0  # the caller mutates its payload after the round
    assert snap == np.linspace(-1, 1, 37).astype("<f4").tobytes()
    assert bytes(lazy)[12:16] == np.float32(123.0).tobytes()  # documented aliasing of the view
