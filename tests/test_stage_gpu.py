"""Merge-stage glue (stage.py) against the reference orchestrator's own merge stages.

tests/golden/make_stage_golden.py recorded, from a 3-epoch reference scenario (4
layers of miners incl. deceptive, dropout, lazy and a joiner; compressed + sync
stages), every `_merge_stage` call's inputs and outputs.  Replaying each stage on
device-resident weights must give bit-identical new global weights, every miner's
weights after adoption, identical per-actor meters and the same stage duration — with
the deceptive miners' GPU noise or the orchestrator's own numpy callables (host path),
and with the stage's layers launched as one CUDA graph or one by one.
"""

import json

import numpy as np
import pytest

from _golden import GOLDEN, assert_same_floats

torch = pytest.importorskip("torch")


def _records():
    return json.loads((GOLDEN / "stage_merges.json").read_text())


def test_stage_dropouts_match_reference():
    from paper_2507_17766_b200.stage import RosterEntry, stage_dropouts

    for rec in _records():
        roster = [RosterEntry(m["id"], m["active"], m["batches"], m["kind"], m["tamper"],
                              0.5 if m["kind"] == "dropout" else 0.0)
                  for L in rec["layers"] for m in L["roster"]]
        assert sorted(stage_dropouts(rec["seed"], rec["epoch"], rec["stage"], roster)) == rec["dropped"]


@pytest.mark.gpu
@pytest.mark.parametrize("deceptive,graph", [("noise", True), ("noise", False), ("reference", True)])
def test_stage_merges_match_reference(cuda_device, deceptive, graph):
    from paper_2507_17766_b200.simkernel import BlobStore, TransferMeter
    from paper_2507_17766_b200.stage import RosterEntry, StageLayer, merge_stage

    arr = np.load(GOLDEN / "stage_merges.npz")
    for idx, rec in enumerate(_records()):
        layers = []
        for L, lay in enumerate(rec["layers"]):
            roster = [RosterEntry(m["id"], m["active"], m["batches"], m["kind"], m["tamper"]) for m in lay["roster"]]
            weights = {}
            for m in lay["roster"]:
                key = f"s{idx}_L{L}_in_{m['id']}"
                weights[m["id"]] = torch.from_numpy(arr[key]).to(cuda_device) if key in arr else None
            synced = torch.from_numpy(arr[f"s{idx}_L{L}_synced"]).to(cuda_device)
            layers.append(StageLayer(roster=roster, weights=weights, synced=synced, layer_index=L))
        store = BlobStore()
        for actor, (up, down) in rec["meter_before"].items():
            store.meter[actor] = TransferMeter(up, down)
        dur = merge_stage(store, layers, seed=rec["seed"], epoch=rec["epoch"], stage_label=rec["stage"],
                          compressed=rec["compressed"], b_min=rec["b_min"], compression_ratio=rec["ratio"],
                          bandwidth_bps=rec["bandwidth_bps"], dropped=set(rec["dropped"]),
                          deceptive=deceptive, graph=graph)
        for L, layer in enumerate(layers):
            assert_same_floats(layer.synced.cpu().numpy(), arr[f"s{idx}_L{L}_global"])
            for m in rec["layers"][L]["roster"]:
                key = f"s{idx}_L{L}_out_{m['id']}"
                if key in arr:
                    assert_same_floats(layer.weights[m["id"]].cpu().numpy(), arr[key])
        meter = {a: [m.bytes_uploaded, m.bytes_downloaded] for a, m in store.meter.items()}
        assert meter == rec["meter_after"], (idx, rec["stage"])
        assert dur == rec["clock_advance"] or abs(dur - rec["clock_advance"]) < 1e-12
