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


def test_lone_qualifier_blob_has_the_serialized_header():
    """A layer with one qualifying miner publishes serialize_weights' header + "<f4" weights
    (orchestrator.py:528-540, model.py:147-154); ranged reads span the header boundary."""
    import struct

    from paper_2507_17766_b200 import stage
    from paper_2507_17766_b200.simkernel import BlobStore

    import torch

    w = torch.linspace(-2, 2, 23, dtype=torch.float64)  # (HBM in the stage; the CPU works the same)
    layer = stage.StageLayer(roster=[stage.RosterEntry("a"), stage.RosterEntry("b")], weights={"a": w},
                             synced=w, layer_index=3, shape=(1, 22))
    store = BlobStore()
    stage._lone_blob(store, "p", layer, "a", w, layer.roster, 3, w.numel())
    full = struct.pack("<iiii", 3, 22, 1, 0) + w.numpy().astype("<f4").tobytes()
    blob = store.objects["p/miner/a/weights"]
    for a, b in [(0, 5), (10, 21), (16, 20), (3, len(full)), (0, len(full))]:
        assert blob[a:b] == full[a:b], (a, b)
    assert bytes(blob) == full
    assert store.meter["a"].bytes_uploaded == len(full) and store.meter["b"].bytes_downloaded == len(full)
