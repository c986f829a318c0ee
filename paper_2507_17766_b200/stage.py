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

Deceptive miners (``deceptive=``):

* ``"reference"`` — exactly the orchestrator's corruption, ``normal(0, tamper_scale *
  rms(reduction))`` from the forked RngStream (:552-562), as a Python callable through
  the drop-in's host path (the reduction of each corrupted shard comes back to the host,
  the callable runs in the reference's call order, the copy goes back up): agreement
  entries identical to the reference's;
* ``"noise"`` (default) — GPU noise descriptors (``Corruption.noise``, amplitude
  tamper_scale x rms of the layer's synced weights x sqrt(3), the same variance): the whole
  stage stays on the device.  Merged weights, statuses, flags, meters and durations are
  the reference's — the orchestrator never injects failures into the merge (:567), so a
  shard with a deceptive assignee always has two survivors that disagree and falls back
  to the synced weights; only the agreement cosines differ.

With ``graph=True`` (default) the device merges of all of a stage's layers are recorded
into ONE CUDA graph and launched once; each layer's results are then read back and
accounted in layer order, as the reference's loop (:596-597) does.
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


def _lone_blob(store, prefix, layer, lone, merged, roster, L, P):
    """The lone qualifier publishes its serialized weights; everyone else copies them
    (orchestrator.py:528-540)."""
    d_out, d_in = layer.shape if layer.shape != (0, 0) else (1, P - 1)
    nbytes = _HEADER.size + 4 * P  # serialize_weights(...) without optimizer state (model.py:150-154)
    header = _HEADER.pack(L, d_in, d_out, 0)

    def blob(w=merged, header=header):
        return header + w.detach().cpu().numpy().astype("<f4").tobytes()

    store.objects[f"{prefix}/miner/{lone}/weights"] = bf._LazyBlob(nbytes, blob, bf._wire_part(merged, header))
    bf._meter(store, lone).bytes_uploaded += _wire(store, nbytes)
    for m in roster:
        if m.miner_id != lone:
            bf._meter(store, m.miner_id).bytes_downloaded += _wire(store, nbytes)


class _LayerMerge:
    """One layer's part of a merge stage: who qualifies (orchestrator.py:519-527), and for
    two or more qualifiers the prepared butterfly round (plan seed and corruptions drawn as
    the orchestrator draws them, :542-562)."""

    def __init__(self, layer: StageLayer, seed: int, epoch: int, stage_label: str, b_min: int, dropped: set,
                 deceptive: str):
        self.layer = layer
        self.stage_label = stage_label
        self.roster = [m for m in layer.roster if m.active]
        self.qualifying = [m for m in self.roster if m.batches_done >= b_min and m.miner_id not in dropped]
        self.L = L = layer.layer_index
        self.prefix = f"epoch/{epoch}/layer/{L}/{stage_label}"
        self.job = None
        if len(self.qualifying) < 2:
            return
        self.ids = ids = sorted(m.miner_id for m in self.qualifying)
        self.index_of = {mid: i for i, mid in enumerate(ids)}
        self.payloads = {mid: layer.weights[mid] for mid in ids}
        P = layer.synced.numel()
        plan_seed = int(RngStream(seed, "scenario").fork(f"epoch{epoch}/plan/{stage_label}/L{L}").integers(0, 2**63))
        self.plan = bf.plan_shards(bf.enumerate_pairs(len(ids)), P, bf.BYTES_PER_WEIGHT, plan_seed)
        self.corruptions = {}
        for m in self.qualifying:
            if m.kind != "deceptive":
                continue
            fork = RngStream(seed, "scenario").fork(f"epoch{epoch}/tamper/{stage_label}/L{L}/{m.miner_id}")
            if deceptive == "reference":  # the orchestrator's own callable (orchestrator.py:552-562)
                def corrupt(reduction, rng=fork, scale=m.tamper_scale):
                    rms = float(np.sqrt(np.mean(reduction ** 2))) or 1.0
                    return rng.normal(0.0, scale * rms, size=reduction.shape)

                self.corruptions[self.index_of[m.miner_id]] = corrupt
            else:
                rms = float(torch.sqrt(torch.mean(layer.synced.double() ** 2)).item()) or 1.0
                key = tuple(int(x) for x in fork.integers(0, 2**63, size=2))
                self.corruptions[self.index_of[m.miner_id]] = Corruption.noise(m.tamper_scale * rms * math.sqrt(3.0),
                                                                               key)
        self.on_device = all(isinstance(c, Corruption) for c in self.corruptions.values())
        if self.on_device:
            from .device import ButterflyMerge, DevicePlan

            self.reps = [self.payloads[mid] for mid in ids]
            dplan = DevicePlan.from_assignment(self.plan.assignment, len(ids), P, layer.synced.device)
            self.job = ButterflyMerge(self.reps, dplan, corruptions=self.corruptions, fallback=layer.synced,
                                      scatter_back=False, want_merged=True, keep_means=True)

    def settle(self, store):
        """Results into the store (reference layer order) and adoption (:575-590)."""
        layer, roster, prefix = self.layer, self.roster, self.prefix
        synced = layer.synced
        P = synced.numel()
        if not self.qualifying:
            merged = synced
        elif len(self.qualifying) == 1:
            lone = self.qualifying[0].miner_id
            merged = layer.weights[lone]
            _lone_blob(store, prefix, layer, lone, merged, roster, self.L, P)
        else:
            if self.job is not None:
                n = len(self.ids)
                res = bf._settle(store, self.plan, self.ids, self.payloads, self.reps, list(range(n)), set(), prefix,
                                 self.job, self.corruptions, {}, {}, self.job.merged)
                self.job = None
            else:
                res = bf.run_all_reduce(store, self.payloads, self.plan, failures=frozenset(),
                                        corruptions=self.corruptions, fallback=synced, key_prefix=prefix,
                                        _device_merged=True)
            merged = res.merged
            # non-participants copy the consolidated merged state (orchestrator.py:575-579)
            key = f"{prefix}/merged-weights"
            store.objects[key] = bf._LazyBlob(4 * P, lambda w=merged: w.detach().cpu().numpy().astype("<f4").tobytes(),
                                              bf._wire_part(merged))
            bf._meter(store, "orchestrator").bytes_uploaded += _wire(store, 4 * P)
            for m in roster:
                if m.miner_id not in self.index_of:
                    bf._meter(store, m.miner_id).bytes_downloaded += _wire(store, 4 * P)
        if self.stage_label.startswith("sync"):
            layer.synced = merged.clone()
            for m in layer.roster:
                layer.weights[m.miner_id] = layer.synced.clone()
                m.active = True
        else:
            for m in self.qualifying:
                layer.weights[m.miner_id] = merged.clone()
        return merged


def _run_device_merges(jobs: list, graph: bool) -> int:
    """Every layer's device round; with ``graph`` recorded into one CUDA graph and launched
    once (returns the number of launches issued: 1, or one run() per layer)."""
    if not jobs:
        return 0
    if graph:
        from . import _lib as L

        L.check(L.lib().bfly_preload())  # no lazy kernel load inside the capture
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for job in jobs:
                job.run()
        g.replay()
        return 1
    for job in jobs:
        job.run()
    return len(jobs)


def merge_stage(store, layers: list, *, seed: int, epoch: int, stage_label: str, compressed: bool, b_min: int,
                compression_ratio: float = 1.0, bandwidth_bps: float = 100e6, link_compression: float = 1.0,
                dropped: set | None = None, deceptive: str = "noise", graph: bool = True) -> float:
    """One merge stage over every layer (orchestrator.py:592-606); returns the stage
    duration in seconds: the busiest actor's moved bytes over the link,
    ``transfer_duration(moved, NetworkModel(bandwidth_bps, link_compression))``
    (simkernel.py:111-115; the orchestrator's model has compression_ratio 1.0,
    orchestrator.py:322).  ``compression_ratio`` is the store's wire_ratio during
    compressed stages (:594)."""
    if deceptive not in ("noise", "reference"):
        raise ValueError(f"deceptive must be 'noise' or 'reference', got {deceptive!r}")
    if link_compression < 1:
        raise ValueError("link_compression (NetworkModel.compression_ratio) must be >= 1")
    before = {a: (m.bytes_uploaded, m.bytes_downloaded) for a, m in store.meter.items()}
    if dropped is None:
        dropped = stage_dropouts(seed, epoch, stage_label, [m for ly in layers for m in ly.roster])
    store.wire_ratio = compression_ratio if compressed else 1.0
    try:
        parts = [_LayerMerge(layer, seed, epoch, stage_label, b_min, dropped, deceptive) for layer in layers]
        _run_device_merges([p.job for p in parts if p.job is not None], graph)
        for part in parts:
            part.settle(store)
    finally:
        store.wire_ratio = 1.0
    slowest = 0.0
    for actor, m in store.meter.items():
        up0, down0 = before.get(actor, (0, 0))
        moved = (m.bytes_uploaded - up0) + (m.bytes_downloaded - down0)
        slowest = max(slowest, (moved * 8.0 / link_compression) / bandwidth_bps)  # transfer_duration
    return slowest


def layer_from_flat(arrays: dict, device) -> dict:
    """Helper: {miner: numpy fp64 flat weights or None} -> device tensors."""
    return {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(device))
            for k, v in arrays.items()}
