"""The validator's replay checks on the GPU.

Mirrors the check half of ``iota_sim.validator`` (validator.py:33-46 ``cosine_similarity``,
:116-122 ``ReplayPolicy``, :148-167 ``_check``): a validator that replays a miner's
traced passes compares every recomputed activation with the reported one by cosine
similarity, a magnitude-ratio band and a maximum relative deviation.  ``check_batch``
runs all of an epoch's comparisons in one launch of ``bfly_replay_check`` (one CTA per
pair, fixed-order reductions).  Same names, defaults, return values and ShapeError as
the reference; similarities agree with the reference's BLAS dot products to rounding
(the threshold decisions are therefore only portable away from the thresholds, as for
the merge's agreement score).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .device import _require_cuda, _stream_handle
from .errors import ShapeError

__all__ = ["ReplayPolicy", "cosine_similarity", "check", "check_batch"]


@dataclass(frozen=True)
class ReplayPolicy:
    cosine_threshold: float = 0.999
    magnitude_low: float = 0.999
    magnitude_high: float = 1.001
    max_rel_deviation: float = 1e-9
    replay_fraction: float = 1.0


def _vec(x, dev) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float64))
    return t.to(dev, torch.float64).reshape(-1) if t.dim() <= 1 else t.to(dev, torch.float64)


def _run(recomputed: list, reported: list, policy: ReplayPolicy):
    dev = _require_cuda()
    a = [_vec(x, dev) for x in recomputed]
    b = [_vec(x, dev) for x in reported]
    for x, y in zip(a, b):
        if x.shape != y.shape or x.dim() != 1 or x.numel() == 0:
            raise ShapeError(f"need equal nonzero-length vectors, got {tuple(x.shape)} and {tuple(y.shape)}")
    n = len(a)
    offsets = np.zeros(n + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([x.numel() for x in a])
    rec = torch.cat(a) if n else torch.empty(0, dtype=torch.float64, device=dev)
    rep = torch.cat(b) if n else torch.empty(0, dtype=torch.float64, device=dev)
    d_off = torch.from_numpy(offsets).to(dev)
    sim = torch.empty(n, dtype=torch.float64, device=dev)
    cos = torch.empty(n, dtype=torch.float64, device=dev)
    pol = (ctypes.c_double * 4)(policy.cosine_threshold, policy.magnitude_low, policy.magnitude_high,
                                policy.max_rel_deviation)
    with torch.cuda.device(dev):
        L.check(L.lib().bfly_replay_check(rec.data_ptr(), rep.data_ptr(), d_off.data_ptr(), n, pol,
                                          sim.data_ptr(), cos.data_ptr(), _stream_handle()))
    return sim.cpu().numpy(), cos.cpu().numpy()


def cosine_similarity(a, b) -> float:
    """a.b / (|a||b|); two zero vectors compare as 1.0 (validator.py:33-46)."""
    return float(_run([a], [b], ReplayPolicy())[1][0])


def check(recomputed, reported, policy: ReplayPolicy = ReplayPolicy()) -> float:
    """Similarity of one reported activation against its replay, 0.0 if any check
    fails (validator.py:148-167)."""
    return float(_run([recomputed], [reported], policy)[0][0])


def check_batch(recomputed: list, reported: list, policy: ReplayPolicy = ReplayPolicy()) -> np.ndarray:
    """``check`` for every pair, in one launch."""
    if len(recomputed) != len(reported):
        raise ShapeError(f"{len(recomputed)} recomputed vs {len(reported)} reported activations")
    return _run(list(recomputed), list(reported), policy)[0]
