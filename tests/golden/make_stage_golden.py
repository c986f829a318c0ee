"""Golden fixtures for the orchestrator's merge glue, from the REFERENCE.

Runs a small reference scenario (iota_sim.orchestrator, read-only /root/reference) and
records, for every merge stage (`_merge_stage`, orchestrator.py:592-606), its inputs
(rosters, qualifying miners' local weights, the synced weights, dropped miners,
compression) and its outputs (the new global weights per layer, every miner's local
weights after adoption, the per-actor meter deltas, the clock advance).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_stage_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from iota_sim import orchestrator as orch  # noqa: E402
from iota_sim.orchestrator import HonestyProfile, ScenarioConfig  # noqa: E402

OUT = Path(__file__).resolve().parent


def flat(w):
    return None if w is None else np.concatenate([w.matrix.ravel(), w.bias])


def main():
    H = HonestyProfile()
    cfg = ScenarioConfig(
        dims=(6, 24, 24, 3),
        miners=(
            (H, H, HonestyProfile(kind="deceptive", tamper_scale=2.0), H),
            (H, HonestyProfile(kind="dropout", p_fail=0.5), H, H, H),
            (H, HonestyProfile(kind="lazy", skip_probability=0.3), H),
        ),
        seed=7,
        epochs=3,
        b_min=2,
        compressed_stages_per_epoch=1,
        compression_ratio=8.0,
        joins=((1, H),),
    )
    records = []
    arrays = {}
    orig = orch._ScenarioRun._merge_stage

    def spy(self, epoch, stage_label, compressed):
        idx = len(records)
        dropped = self._stage_dropouts(epoch, stage_label)  # deterministic fork, same as inside
        before = {a: [m.bytes_uploaded, m.bytes_downloaded] for a, m in self.store.meter.items()}
        t0 = self.clock.now
        rec = dict(epoch=epoch, stage=stage_label, compressed=compressed, dropped=sorted(dropped),
                   seed=self.config.seed, b_min=self.config.b_min, ratio=self.config.compression_ratio,
                   bandwidth_bps=self.network.bandwidth_bps, layers=[])
        for layer in range(self.config.n_layers):
            roster = [dict(id=m.miner_id, active=m.active, batches=m.batches_done, kind=m.profile.kind,
                           tamper=m.profile.tamper_scale) for m in self.rosters[layer]]
            rec["layers"].append(dict(roster=roster))
            arrays[f"s{idx}_L{layer}_synced"] = flat(self.global_layers[layer])
            for m in self.rosters[layer]:
                w = flat(self.local.get(m.miner_id))
                if w is not None:
                    arrays[f"s{idx}_L{layer}_in_{m.miner_id}"] = w
        rec["meter_before"] = before
        orig(self, epoch, stage_label, compressed)
        after = {a: [m.bytes_uploaded, m.bytes_downloaded] for a, m in self.store.meter.items()}
        rec["meter_after"] = after
        rec["clock_advance"] = self.clock.now - t0
        for layer in range(self.config.n_layers):
            arrays[f"s{idx}_L{layer}_global"] = flat(self.global_layers[layer])
            for m in self.rosters[layer]:
                w = flat(self.local.get(m.miner_id))
                if w is not None:
                    arrays[f"s{idx}_L{layer}_out_{m.miner_id}"] = w
        records.append(rec)

    orch._ScenarioRun._merge_stage = spy
    try:
        orch.run_scenario(cfg)
    finally:
        orch._ScenarioRun._merge_stage = orig
    np.savez_compressed(OUT / "stage_merges.npz", **arrays)
    (OUT / "stage_merges.json").write_text(json.dumps(records, indent=1))
    print(len(records), "merge stages recorded")


if __name__ == "__main__":
    main()
