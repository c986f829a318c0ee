"""ctypes binding of libbfly.so (the C ABI declared in include/bfly.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``).  There
is no fallback: if the shared object is missing, importing the product raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

from . import errors

_SO = Path(__file__).resolve().parent / "libbfly.so"

OK = 0
E_TOO_FEW_MINERS, E_DEGENERATE, E_SHAPE, E_INVALID_ARG, E_CUDA, E_UNSUPPORTED = 1, 2, 3, 4, 5, 6
F32, BF16, F64WIRE = 0, 1, 2
MERGED, LOST, DISAGREEMENT = 0, 1, 2
STATUS_NAMES = ("merged", "lost", "disagreement")
CORR_NONE, CORR_ADD, CORR_SCALE, CORR_NOISE, CORR_NOISE_ADD, CORR_HOST = 0, 1, 2, 3, 4, 5
PHASE_ALL, PHASE_REDUCE, PHASE_FINISH, PHASE_CHECK = 0, 1, 2, 3

# every symbol include/bfly.h declares (tests/test_capi.py checks the export table)
EXPORTS = (
    "bfly_ring_fused",
    "bfly_ring_fused_lanes",
    "bfly_ring_fused_layout",
    "bfly_ring_fused_loopback",
    "bfly_ring_fused_stat_tile",
    "bfly_version",
    "bfly_last_error",
    "bfly_n_shards",
    "bfly_philox_key",
    "bfly_plan_host",
    "bfly_permutation_host",
    "bfly_plan_device",
    "bfly_merge_scratch_bytes",
    "bfly_merge",
    "bfly_agreement",
    "bfly_apply_corruption",
    "bfly_mean_rows",
    "bfly_chain_step",
    "bfly_fanout",
    "bfly_copy_ranges",
    "bfly_fill_shards",
    "bfly_ipc_alloc",
    "bfly_ipc_open",
    "bfly_ipc_close",
    "bfly_ipc_free",
    "bfly_preload",
    "bfly_stream_create",
    "bfly_stream_destroy",
    "bfly_stream_wait_value",
    "bfly_stream_write_value",
    "bfly_upload_wire",
    "bfly_merge_host",
    "bfly_replay_check",
    "bfly_ipc_export",
    "bfly_ring_round",
    "bfly_ring_ops",
)


class Corruption(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("a", ctypes.c_double),
        ("key0", ctypes.c_uint64),
        ("key1", ctypes.c_uint64),
    ]


class MergeArgs(ctypes.Structure):
    _fields_ = [
        ("n_miners", ctypes.c_int32),
        ("redundancy", ctypes.c_int32),
        ("payload_len", ctypes.c_int64),
        ("n_shards", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("n_alive", ctypes.c_int32),
        ("d_assign", ctypes.c_void_p),
        ("d_src", ctypes.c_void_p),
        ("d_failed", ctypes.c_void_p),
        ("d_corr", ctypes.c_void_p),
        ("d_dst", ctypes.c_void_p),
        ("n_dst", ctypes.c_int32),
        ("stat_tile", ctypes.c_int32),
        ("d_fallback", ctypes.c_void_p),
        ("d_merged", ctypes.c_void_p),
        ("d_ws", ctypes.c_void_p),
        ("d_host_copies", ctypes.c_void_p),
        ("d_status", ctypes.c_void_p),
        ("d_entries", ctypes.c_void_p),
        ("d_flagged", ctypes.c_void_p),
        ("d_source", ctypes.c_void_p),
        ("d_scratch", ctypes.c_void_p),
        ("scratch_bytes", ctypes.c_size_t),
        ("tolerance", ctypes.c_double),
        ("phase", ctypes.c_int32),
        ("pad1", ctypes.c_int32),
        ("d_acc_in", ctypes.c_void_p),
        ("n_div", ctypes.c_int32),
        ("pad2", ctypes.c_int32),
        ("elem_begin", ctypes.c_int64),
        ("elem_end", ctypes.c_int64),
        ("d_fallback_src", ctypes.c_void_p),
        ("shard_begin", ctypes.c_int64),
        ("shard_end", ctypes.c_int64),
        ("d_shard_list", ctypes.c_void_p),
        ("n_shard_list", ctypes.c_int32),
        ("fallback_gone", ctypes.c_int32),
    ]


class RingDesc(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("k_chunks", ctypes.c_int32),
        ("nb", ctypes.c_int32),
        ("payload_len", ctypes.c_int64),
        ("chunk", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("esize", ctypes.c_int32),
        ("peer_base", ctypes.c_void_p),
        ("off_acc", ctypes.c_int64),
        ("off_fin", ctypes.c_int64),
        ("off_flags", ctypes.c_int64),
        ("d_src_table", ctypes.c_void_p),
        ("n_src", ctypes.c_int32),
        ("fan_n", ctypes.c_int32),
        ("fan_tables", ctypes.c_void_p),
        ("merge_args", ctypes.POINTER(MergeArgs)),
        ("reduce_tables", ctypes.c_void_p),
        ("reduce_n", ctypes.c_int32),
        ("window", ctypes.c_int32),
        ("stream_c", ctypes.c_void_p),
        ("stream_r", ctypes.c_void_p),
        ("finish_ranges", ctypes.c_void_p),
        ("stream_f", ctypes.c_void_p),
        ("reduce_events", ctypes.c_void_p),
        ("chunk_edges", ctypes.c_void_p),
    ]


class RingFusedDesc(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("lanes", ctypes.c_int32),
        ("nb", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("n_src", ctypes.c_int32),
        ("n_dst", ctypes.c_int32),
        ("n_div", ctypes.c_int32),
        ("payload_len", ctypes.c_int64),
        ("round_index", ctypes.c_uint64),
        ("peer_base", ctypes.c_void_p),
        ("d_src", ctypes.c_void_p),
        ("d_dst", ctypes.c_void_p),
        ("d_merged", ctypes.c_void_p),
        ("merge_args", ctypes.POINTER(MergeArgs)),
        ("special", ctypes.c_int32),
        ("pub_every", ctypes.c_int32),
        ("lag", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("d_profile", ctypes.c_void_p),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libbfly.so once; raise loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not _SO.exists():
        raise ImportError(f"{_SO} is missing: build the CUDA library first (`make` or __graft_entry__.build())")
    L = ctypes.CDLL(str(_SO))
    i32, i64, u64, dbl, vp, sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                                  ctypes.c_void_p, ctypes.c_size_t)
    L.bfly_version.restype = ctypes.c_char_p
    L.bfly_last_error.restype = ctypes.c_char_p
    L.bfly_n_shards.argtypes = [i32, i32]
    L.bfly_n_shards.restype = i64
    L.bfly_philox_key.argtypes = [ctypes.c_char_p, ctypes.c_char_p, vp]
    L.bfly_plan_host.argtypes = [i32, i32, i64, u64, u64, vp, vp]
    L.bfly_permutation_host.argtypes = [i64, u64, u64, vp]
    L.bfly_plan_device.argtypes = [i32, i32, i64, u64, u64, vp, vp, vp]
    L.bfly_merge_scratch_bytes.argtypes = [i32, i32, i64]
    L.bfly_merge_scratch_bytes.restype = sz
    L.bfly_merge.argtypes = [ctypes.POINTER(MergeArgs), vp]
    L.bfly_agreement.argtypes = [vp, vp, i64, dbl, vp, vp, sz, vp]
    L.bfly_apply_corruption.argtypes = [ctypes.POINTER(Corruption), vp, i64, i64, vp, vp]
    L.bfly_mean_rows.argtypes = [vp, i32, i64, vp, vp]
    L.bfly_chain_step.argtypes = [vp, i32, i32, vp, vp, i64, i64, vp]
    L.bfly_fanout.argtypes = [vp, vp, i32, i64, vp]
    u32 = ctypes.c_uint32
    L.bfly_ipc_alloc.argtypes = [sz, ctypes.POINTER(vp), vp]
    L.bfly_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
    L.bfly_ipc_close.argtypes = [vp]
    L.bfly_ipc_free.argtypes = [vp]
    L.bfly_stream_create.argtypes = [i32, ctypes.POINTER(vp)]
    L.bfly_stream_destroy.argtypes = [vp]
    L.bfly_stream_wait_value.argtypes = [vp, u32, vp]
    L.bfly_stream_write_value.argtypes = [vp, u32, vp]
    L.bfly_upload_wire.argtypes = [vp, i32, i64, vp, i32, i64, vp]
    L.bfly_ipc_export.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
    L.bfly_replay_check.argtypes = [vp, vp, vp, i32, vp, vp, vp, vp]
    L.bfly_merge_host.argtypes = [vp, i32, i64, vp, ctypes.POINTER(MergeArgs), vp, i32, i32, i64, vp]
    L.bfly_ring_round.argtypes = [ctypes.POINTER(RingDesc), u32]
    L.bfly_ring_ops.argtypes = [i32, i32, i32, i32, u32, i32, vp, i32]
    L.bfly_fill_shards.argtypes = [vp, vp, vp, vp, i32, i32, i64, i64, vp]
    L.bfly_copy_ranges.argtypes = [vp, vp, vp, i32, vp, i32, i32, i32, vp]
    L.bfly_ring_fused_lanes.argtypes = [i32]
    L.bfly_ring_fused_lanes.restype = i32
    L.bfly_ring_fused_layout.argtypes = [i32, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.bfly_ring_fused.argtypes = [ctypes.POINTER(RingFusedDesc), vp]
    L.bfly_ring_fused_loopback.argtypes = [vp, i32, vp]
    L.bfly_ring_fused_stat_tile.argtypes = [i32]
    L.bfly_ring_fused_stat_tile.restype = i32
    for name in EXPORTS:  # fail at load time if the export table is incomplete
        getattr(L, name)
    _lib = L
    return L


_ERRORS = {
    E_TOO_FEW_MINERS: errors.TooFewMinersError,
    E_DEGENERATE: errors.DegenerateShardsError,
    E_SHAPE: errors.ShapeError,
    E_INVALID_ARG: errors.InvalidArgumentError,
    E_UNSUPPORTED: NotImplementedError,
}


def check(rc: int) -> None:
    """Map a BFLY_E* status to the reference exception class (errors.py:4-45)."""
    if rc == OK:
        return
    msg = lib().bfly_last_error().decode(errors="replace")
    if rc == E_CUDA:
        raise RuntimeError(f"CUDA error in libbfly: {msg}")
    raise _ERRORS.get(rc, RuntimeError)(msg)


def philox_key(seed: int, stream_id: str) -> tuple[int, int]:
    """Key of RngStream(seed, stream_id) (simkernel.py:203-205), via the library's SHA-256."""
    out = (ctypes.c_uint64 * 2)()
    check(lib().bfly_philox_key(str(int(seed)).encode(), stream_id.encode(), out))
    return int(out[0]), int(out[1])


_STREAMS: dict = {}  # (device index, priority, role) -> stream handle, kept for the process lifetime


def own_stream(device, priority: int = 0, role=None):
    """The dedicated CUDA stream of ``role`` on ``device`` (bfly_stream_create), wrapped for
    torch.  torch.cuda.Stream() draws from a fixed pool that wraps around, so two "new"
    streams can be the same CUDA stream — fatal for streams that wait on flags other
    ranks write.  One stream per (device, priority, role), created once and never
    destroyed (torch's caching allocator remembers the stream of every block)."""
    import torch

    dev = torch.device(device)
    key = (dev.index, int(priority), role)
    h = _STREAMS.get(key)
    if h is None:
        hv = ctypes.c_void_p()
        with torch.cuda.device(dev):
            check(lib().bfly_stream_create(int(priority), ctypes.byref(hv)))
        h = _STREAMS[key] = hv.value
    return torch.cuda.ExternalStream(h, device=dev)
