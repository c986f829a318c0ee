"""Host substrate the merge path touches: the metered blob store and RngStream.

Mirrors the slice of pkg/src/iota_sim/simkernel.py the butterfly round uses:
``BlobStore`` (simkernel.py:131-200: per-actor byte meter, ``wire_ratio`` ceil
per transfer) and ``RngStream`` (simkernel.py:208-244: SHA-256-keyed Philox).
The drop-in ``run_all_reduce`` accepts either this store or the reference's —
it only needs ``meter``/``_meter_for``, ``objects`` and ``wire_ratio``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .errors import InvalidConfigError, KeyExistsError, NotFoundError


@dataclass
class TransferMeter:
    bytes_uploaded: int = 0
    bytes_downloaded: int = 0


@dataclass
class BlobStore:
    """In-memory object store with per-actor transfer metering (simkernel.py:131-200)."""

    objects: dict = field(default_factory=dict)
    meter: dict = field(default_factory=dict)
    wire_ratio: float = 1.0

    def _meter_for(self, actor: str) -> TransferMeter:
        m = self.meter.get(actor)
        if m is None:
            m = self.meter[actor] = TransferMeter()
        return m

    def _wire_bytes(self, nbytes: int) -> int:
        return nbytes if self.wire_ratio == 1.0 else math.ceil(nbytes / self.wire_ratio)

    def put(self, actor: str, key: str, data, overwrite: bool = False) -> int:
        if not key:
            raise InvalidConfigError("blob key must be non-empty")
        if key in self.objects and not overwrite:
            raise KeyExistsError(f"key already exists: {key}")
        data = bytes(data)
        self.objects[key] = data
        self._meter_for(actor).bytes_uploaded += self._wire_bytes(len(data))
        return len(data)

    def get(self, actor: str, key: str, start: int = 0, length: int | None = None) -> bytes:
        if key not in self.objects:
            raise NotFoundError(f"no such key: {key}")
        data = self.objects[key]
        chunk = data[start:] if length is None else data[start:start + length]
        self._meter_for(actor).bytes_downloaded += self._wire_bytes(len(chunk))
        return chunk

    def exists(self, key: str) -> bool:
        return key in self.objects

    def size(self, key: str) -> int:
        if key not in self.objects:
            raise NotFoundError(f"no such key: {key}")
        return len(self.objects[key])

    def total_uploaded(self) -> int:
        return sum(m.bytes_uploaded for m in self.meter.values())

    def total_downloaded(self) -> int:
        return sum(m.bytes_downloaded for m in self.meter.values())


class RngStream:
    """Forkable Philox stream keyed by SHA-256(f"{seed}\\x1f{stream_id}") (simkernel.py:203-219)."""

    def __init__(self, seed: int, stream_id: str = "root"):
        self.seed = int(seed)
        self.stream_id = stream_id
        key = np.array(L.philox_key(self.seed, stream_id), dtype=np.uint64)
        self.generator = np.random.Generator(np.random.Philox(key=key))

    def fork(self, label: str) -> "RngStream":
        return RngStream(self.seed, f"{self.stream_id}/{label}")

    def __getattr__(self, name):  # random / uniform / normal / integers / permutation / choice
        if name in ("random", "uniform", "normal", "integers", "permutation", "choice"):
            return getattr(self.generator, name)
        raise AttributeError(name)

    def __repr__(self):
        return f"RngStream(seed={self.seed}, stream_id={self.stream_id!r})"
