"""Merge-stage glue on device-resident per-layer weights.

Restates the orchestrator's merge stage — ``_merge_stage`` / ``_merge_layer``
(orchestrator.py:519-606) and the dropout draw it relies on (``_stage_dropouts``,
:371-377) — for miners whose per-layer weights live in HBM as flat fp64 tensors
(the reference's miners hold float64 weights; the merge reads them as the fp32
wire, butterfly.py:213).  Per layer:

* qualifying miners = active, batches_done >= b_min, not dropped (:521-524);
* none -> the synced weights stand; one -> the lone miner's weights are published
  and copied (:528-540); two or more -> the butterfly merge on the GPU with the
  plan seed drawn exactly as the orchestrator does
  (``RngStream(seed, "scenario").fork(f"epoch{e}/plan/{stage}/L{layer}").integers(0, 2**63)``,
  :546-548), ``fallback = synced`` (:569), and the merged-weights blob served to
  non-participants (:575-579);
* adoption: a sync stage makes the merged weights the new global weights and every
  roster miner (joiners included) copies them and becomes active; a compressed stage
  updates the qualifying miners only (:581-590);
* the stage takes as long as its busiest actor's metered bytes (:599-606), with
  ``wire_ratio`` = the compression ratio during compressed stages (:594).

Deceptive miners corrupt their shard reductions with GPU noise (``Corruption.noise``
with amplitude tamper_scale x rms of the layer's synced weights) instead of numpy's
``normal(0, tamper_scale * rms(reduction))``.  Merged weights, statuses, meters and
durations are unaffected — the orchestrator never injects failures into the merge
(:567), so a shard with a deceptive assignee always has two survivors that disagree
and falls back to the synced weights; only the agreement cosines differ.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import butterfly as bf
from .device import Corruption
from .simkernel import RngStream

_HEADER = struct.Struct("<iiii")  # serialize_weights header (model.py:147)


@dataclass
class RosterEntry:
    miner_id: str
    active: bool = True
    batches_done: int = 0
    kind: str = "honest"  # honest | dropout | deceptive | lazy (orchestrator.py:56-104)
    tamper_scale: float = 1.0
    p_fail: float = 0.0


@dataclass
class StageLayer:
    """One pipeline layer: its roster, every miner's flat fp64 weights in HBM (None for
    a joiner that has not synchronised yet) and the last globally synced weights."""

    roster: list
    weights: dict
    synced: torch.Tensor
    layer_index: int = 0
    shape: tuple = field(default=(0, 0))  # (d_out, d_in) of the weight matrix, for the blob header


def stage_dropouts(seed: int, epoch: int, stage_label: str, miners: list) -> set:
    """Miners that fail this stage (orchestrator.py:371-377): one uniform draw per
    active dropout-profile miner, in roster order, from the forked stream."""
    rng = RngStream(seed, "scenario").fork(f"epoch{epoch}/dropout/{stage_label}")
    dropped = set()
    for m in miners:
        if m.active and m.kind == "dropout" and rng.random() < m.p_fail:
            dropped.add(m.miner_id)
    return dropped


def _wire(store, nbytes: int) -> int:
    return nbytes if store.wire_ratio == 1.0 else math.ceil(nbytes / store.wire_ratio)


def _merge_layer(store, layer: StageLayer, seed: int, epoch: int, stage_label: str, b_min: int, dropped: set):
    roster = [m for m in layer.roster if m.active]
    qualifying = [m for m in roster if m.batches_done >= b_min and m.miner_id not in dropped]
    L = layer.layer_index
    prefix = f"epoch/{epoch}/layer/{L}/{stage_label}"
    synced = layer.synced
    P = synced.numel()
    if not qualifying:
        merged = synced
    elif len(qualifying) == 1:
        lone = qualifying[0].miner_id
        merged = layer.weights[lone]
        d_out, d_in = layer.shape if layer.shape != (0, 0) else (1, P - 1)
        nbytes = _HEADER.size + 4 * P  # serialize_weights(...) without optimizer state (model.py:150-154)

        def blob(w=merged, L=L, d_in=d_in, d_out=d_out):
            return _HEADER.pack(L, d_in, d_out, 0) + w.detach().cpu().numpy().astype("<f4").tobytes()

        store.objects[f"{prefix}/miner/{lone}/weights"] = bf._LazyBlob(
            nbytes, blob, bf._wire_part(merged, _HEADER.pack(L, d_in, d_out, 0)))
        bf._meter(store, lone).bytes_uploaded += _wire(store, nbytes)
        for m in roster:
            if m.miner_id != lone:
                bf._meter(store, m.miner_id).bytes_downloaded += _wire(store, nbytes)
    else:
        ids = sorted(m.miner_id for m in qualifying)
        index_of = {mid: i for i, mid in enumerate(ids)}
        payloads = {mid: layer.weights[mid] for mid in ids}
        plan_seed = int(RngStream(seed, "scenario").fork(f"epoch{epoch}/plan/{stage_label}/L{L}").integers(0, 2**63))
        plan = bf.plan_shards(bf.enumerate_pairs(len(ids)), P, bf.BYTES_PER_WEIGHT, plan_seed)
        rms = float(torch.sqrt(torch.mean(synced.double() ** 2)).item()) or 1.0
        corruptions = {}
        for m in qualifying:
            if m.kind == "deceptive":
                key = tuple(int(x) for x in RngStream(seed, "scenario").fork(
                    f"epoch{epoch}/tamper/{stage_label}/L{L}/{m.miner_id}").integers(0, 2**63, size=2))
                corruptions[index_of[m.miner_id]] = Corruption.noise(m.tamper_scale * rms * math.sqrt(3.0), key)
        res = bf.run_all_reduce(store, payloads, plan, failures=frozenset(), corruptions=corruptions,
                                fallback=synced, key_prefix=prefix, _device_merged=True)
        merged = res.merged
        # non-participants copy the consolidated merged state (orchestrator.py:575-579)
        key = f"{prefix}/merged-weights"
        store.objects[key] = bf._LazyBlob(4 * P, lambda w=merged: w.detach().cpu().numpy().astype("<f4").tobytes(),
                                          bf._wire_part(merged))
        bf._meter(store, "orchestrator").bytes_uploaded += _wire(store, 4 * P)
        for m in roster:
            if m.miner_id not in index_of:
                bf._meter(store, m.miner_id).bytes_downloaded += _wire(store, 4 * P)
    if stage_label.startswith("sync"):
        layer.synced = merged.clone()
        for m in layer.roster:
            layer.weights[m.miner_id] = layer.synced.clone()
            m.active = True
    else:
        for m in qualifying:
            layer.weights[m.miner_id] = merged.clone()
    return merged


def merge_stage(store, layers: list, *, seed: int, epoch: int, stage_label: str, compressed: bool, b_min: int,
                compression_ratio: float = 1.0, bandwidth_bps: float = 100e6, dropped: set | None = None) -> float:
    """One merge stage over every layer (orchestrator.py:592-606); returns the stage
    duration in seconds (the busiest actor's moved bytes over the link bandwidth)."""
    before = {a: (m.bytes_uploaded, m.bytes_downloaded) for a, m in store.meter.items()}
    if dropped is None:
        dropped = stage_dropouts(seed, epoch, stage_label, [m for ly in layers for m in ly.roster])
    store.wire_ratio = compression_ratio if compressed else 1.0
    try:
        for layer in layers:
            _merge_layer(store, layer, seed, epoch, stage_label, b_min, dropped)
    finally:
        store.wire_ratio = 1.0
    slowest = 0.0
    for actor, m in store.meter.items():
        up0, down0 = before.get(actor, (0, 0))
        moved = (m.bytes_uploaded - up0) + (m.bytes_downloaded - down0)
        slowest = max(slowest, (moved * 8.0 / 1.0) / bandwidth_bps)  # transfer_duration, simkernel.py:111-115
    return slowest


def layer_from_flat(arrays: dict, device) -> dict:
    """Helper: {miner: numpy fp64 flat weights or None} -> device tensors."""
    return {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(device))
            for k, v in arrays.items()}
