"""ctypes prototypes for libnrc.so (include/nrc.h).  Marshalling only."""
from __future__ import annotations

import ctypes
import os

from . import build as _build

_lib = None


class NrcConfig(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_uint32),
        ("hidden_width", ctypes.c_uint32),
        ("n_hidden_layers", ctypes.c_uint32),
        ("reserved0", ctypes.c_uint32),
        ("max_batch", ctypes.c_uint64),
        ("aabb_min", ctypes.c_float * 3),
        ("aabb_max", ctypes.c_float * 3),
        ("learning_rate", ctypes.c_float),
        ("adam_beta1", ctypes.c_float),
        ("adam_beta2", ctypes.c_float),
        ("adam_eps", ctypes.c_float),
        ("loss_eps", ctypes.c_float),
        ("ema_alpha", ctypes.c_float),
        ("flags", ctypes.c_uint32),
        ("seed", ctypes.c_uint64),
        ("device", ctypes.c_int32),
    ]


# exported symbols, in include/nrc.h order (checked by tests/test_abi.py)
SYMBOLS = [
    "nrc_default_config", "nrc_state_bytes", "nrc_init", "nrc_destroy", "nrc_query", "nrc_train_step",
    "nrc_train_backward", "nrc_train_apply", "nrc_train_frame", "nrc_train_frame_backward", "nrc_lcg_params", "nrc_encode", "nrc_get_params",
    "nrc_set_params", "nrc_get_stats", "nrc_param_count", "nrc_status_string", "nrc_last_error",
    "nrc_frame_scratch_bytes", "nrc_frame_host", "nrc_selftest_umma", "nrc_last_launch_count",
    "nrc_assemble_targets", "nrc_query_accumulate", "nrc_train_frame_dp_peer",
    "nrc_dp_timeouts", "nrc_ipc_export", "nrc_ipc_import", "nrc_ipc_close", "nrc_train_apply_multimem",
    "nrc_peer_barrier", "nrc_multicast_alloc", "nrc_multicast_free", "nrc_train_apply_peers",
]


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libnrc.so (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("NRC_LIB_VARIANT")  # diagnostics only: an A/B build of the same sources
    if path is None:
        if build_if_missing:
            _build.build()
        path = _build.LIB
    if not os.path.exists(path):
        raise RuntimeError(f"libnrc.so not found at {path}; run paper_2106_12372_b200.build.build()")
    L = ctypes.CDLL(path)
    vp, u32, u64, st = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    sz = ctypes.c_size_t
    P = ctypes.POINTER
    L.nrc_default_config.restype = None; L.nrc_default_config.argtypes = [P(NrcConfig)]
    L.nrc_state_bytes.restype = sz; L.nrc_state_bytes.argtypes = [P(NrcConfig)]
    L.nrc_init.restype = st; L.nrc_init.argtypes = [P(NrcConfig), vp, sz, P(vp)]
    L.nrc_destroy.restype = st; L.nrc_destroy.argtypes = [vp]
    L.nrc_query.restype = st; L.nrc_query.argtypes = [vp, vp, u64, vp, vp]
    L.nrc_train_step.restype = st; L.nrc_train_step.argtypes = [vp, vp, vp, u32, vp, vp]
    L.nrc_train_backward.restype = st; L.nrc_train_backward.argtypes = [vp, vp, vp, u32, vp, vp, vp, vp]
    L.nrc_train_apply.restype = st; L.nrc_train_apply.argtypes = [vp, vp, u32, vp, vp, vp]
    L.nrc_train_frame.restype = st; L.nrc_train_frame.argtypes = [vp, vp, vp, u32, u32, u32, u64, vp, vp]
    L.nrc_train_frame_backward.restype = st
    L.nrc_train_frame_backward.argtypes = [vp, vp, vp, u32, u32, u64, u32, u32, u32, vp, vp, vp]
    L.nrc_lcg_params.restype = st; L.nrc_lcg_params.argtypes = [u64, u64, P(u64), P(u64), P(u64)]
    L.nrc_encode.restype = st; L.nrc_encode.argtypes = [vp, vp, u64, vp, vp]
    L.nrc_train_frame_dp_peer.restype = st
    L.nrc_train_frame_dp_peer.argtypes = [vp, vp, vp, u32, u32, u32, u64, u32, u32, vp, vp, vp]
    L.nrc_dp_timeouts.restype = st; L.nrc_dp_timeouts.argtypes = [vp, P(u64)]
    L.nrc_train_apply_multimem.restype = st; L.nrc_train_apply_multimem.argtypes = [vp, vp, u32, vp, vp]
    L.nrc_peer_barrier.restype = st; L.nrc_peer_barrier.argtypes = [vp, vp, u32, u32, vp]
    L.nrc_train_apply_peers.restype = st; L.nrc_train_apply_peers.argtypes = [vp, vp, u32, u32, vp, vp]
    L.nrc_multicast_alloc.restype = st; L.nrc_multicast_alloc.argtypes = [ctypes.c_int, sz, P(vp), P(vp)]
    L.nrc_multicast_free.restype = st; L.nrc_multicast_free.argtypes = [vp]
    L.nrc_ipc_export.restype = st; L.nrc_ipc_export.argtypes = [vp, vp, P(u64)]
    L.nrc_ipc_import.restype = st; L.nrc_ipc_import.argtypes = [vp, u64, P(vp)]
    L.nrc_ipc_close.restype = st; L.nrc_ipc_close.argtypes = [vp, u64]
    L.nrc_query_accumulate.restype = st
    L.nrc_query_accumulate.argtypes = [vp, vp, u64, vp, vp, vp, vp]
    L.nrc_assemble_targets.restype = st
    L.nrc_assemble_targets.argtypes = [vp, vp, vp, vp, ctypes.c_uint32, vp, vp, vp, vp]
    L.nrc_get_params.restype = st; L.nrc_get_params.argtypes = [vp, st, vp, sz]
    L.nrc_set_params.restype = st; L.nrc_set_params.argtypes = [vp, st, vp, sz]
    L.nrc_get_stats.restype = st; L.nrc_get_stats.argtypes = [vp, P(u64), P(u64), P(u64), P(u64)]
    L.nrc_param_count.restype = sz; L.nrc_param_count.argtypes = [vp]
    L.nrc_status_string.restype = ctypes.c_char_p; L.nrc_status_string.argtypes = [st]
    L.nrc_last_error.restype = ctypes.c_char_p; L.nrc_last_error.argtypes = [vp]
    L.nrc_frame_scratch_bytes.restype = sz; L.nrc_frame_scratch_bytes.argtypes = [u64, u32]
    L.nrc_frame_host.restype = st
    L.nrc_frame_host.argtypes = [vp, vp, u64, vp, vp, vp, u32, u32, u32, u64, vp, vp, sz, vp]
    L.nrc_selftest_umma.restype = st; L.nrc_selftest_umma.argtypes = [st, vp, vp, vp]
    L.nrc_last_launch_count.restype = u32; L.nrc_last_launch_count.argtypes = [vp]
    _lib = L
    return L
