"""Store objects of the merge are lazily materialised views of (device) vectors in the
"<f4" wire format: a ranged BlobStore.get copies only that range back and returns the
same bytes as slicing the fully materialised object (simkernel.py:174-186)."""

import struct

import numpy as np
import pytest

from paper_2507_17766_b200 import butterfly as bf
from paper_2507_17766_b200.simkernel import BlobStore


@pytest.mark.parametrize("header", [b"", struct.pack("<iiii", 3, 7, 5, 0)])
def test_ranged_reads_equal_full_materialisation(header):
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, 1001) * 1e3
    calls = []

    def part(a, b):
        calls.append((a, b))
        return bf._wire_part(v, header)(a, b)

    full = header + v.astype("<f4").tobytes()
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
