"""Thin Python binding over libnrc's C ABI (include/nrc.h).

Argument marshalling only: every step of the hot path (encoding, fused MLP
query, fused forward/backward/wgrad, Adam, EMA, LCG gather) runs in the CUDA
kernels behind the C ABI.  PyTorch supplies device memory and streams; there
is no CPU fallback -- constructing a RadianceCache without a B200 raises.

Paper: Mueller et al., "Real-time Neural Radiance Caching for Path Tracing"
(arXiv 2106.12372).  API names follow the paper's problem statement: a cache
queried with records (Table 1) and trained online from
(record, target) pairs.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib

NPARAM = 5 * 64 * 64 + 3 * 64  # 20,672 (reading R1)
REC_FLOATS = 16

FACTORIZE = 1
CLAMP_QUERY = 2
EMA_PRINTED_FORM = 4
QUERY_RAW_WEIGHTS = 8
EXACT_ENCODING = 16

PARAMS_TRAIN, PARAMS_EMA, ADAM_M, ADAM_V = 0, 1, 2, 3
_PARAM_SETS = {"train": PARAMS_TRAIN, "ema": PARAMS_EMA, "adam_m": ADAM_M, "adam_v": ADAM_V}


class NRCError(RuntimeError):
    pass


@dataclass
class Config:
    """Mirror of nrc_config; defaults are the paper's constants (see nrc.h)."""
    hidden_width: int = 64
    n_hidden_layers: int = 5
    max_batch: int = 3840 * 2160
    aabb_min: Sequence[float] = (0.0, 0.0, 0.0)
    aabb_max: Sequence[float] = (1.0, 1.0, 1.0)
    learning_rate: float = 1e-2
    adam_beta1: float = 0.9
    adam_beta2: float = 0.99
    adam_eps: float = 1e-8
    loss_eps: float = 0.01
    ema_alpha: float = 0.99
    flags: int = FACTORIZE | CLAMP_QUERY
    seed: int = 1

    def to_c(self, device: int) -> _lib.NrcConfig:
        c = _lib.NrcConfig()
        _lib.load().nrc_default_config(ctypes.byref(c))
        c.hidden_width = self.hidden_width
        c.n_hidden_layers = self.n_hidden_layers
        c.max_batch = self.max_batch
        for i in range(3):
            c.aabb_min[i] = self.aabb_min[i]
            c.aabb_max[i] = self.aabb_max[i]
        c.learning_rate = self.learning_rate
        c.adam_beta1 = self.adam_beta1
        c.adam_beta2 = self.adam_beta2
        c.adam_eps = self.adam_eps
        c.loss_eps = self.loss_eps
        c.ema_alpha = self.ema_alpha
        c.flags = self.flags
        c.seed = self.seed & (2 ** 64 - 1)
        c.device = device
        return c


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


# Volume queries: "undefined parameters (surface roughness,
# normal, albedo, and specular coefficients) are simply set to default
# constants".  Reading R23: n = (0, 0, 1), r = 1, alpha = (1, 1, 1),
# beta = (0, 0, 0), so the reflectance factorisation (alpha + beta = 1) leaves
# the network output unchanged.
VOLUME_DEFAULTS = {"normal": (0.0, 0.0, 1.0), "roughness": 1.0, "albedo": (1.0, 1.0, 1.0),
                   "specular": (0.0, 0.0, 0.0)}


def volume_records(positions: torch.Tensor, directions: torch.Tensor) -> torch.Tensor:
    """Cache records [n, 16] for volume (in-medium) vertices: position and
    direction from the caller, the surface fields at VOLUME_DEFAULTS (R23).
    Data assembly only (torch ops on the caller's device)."""
    n = positions.shape[0]
    if positions.shape != (n, 3) or directions.shape != (n, 3):
        raise NRCError("positions and directions must be [n, 3]")
    rec = torch.empty((n, REC_FLOATS), dtype=torch.float32, device=positions.device)
    rec[:, 0:3] = positions
    rec[:, 3:6] = directions
    d = VOLUME_DEFAULTS
    rec[:, 6:9] = torch.tensor(d["normal"], dtype=torch.float32, device=positions.device)
    rec[:, 9] = d["roughness"]
    rec[:, 10:13] = torch.tensor(d["albedo"], dtype=torch.float32, device=positions.device)
    rec[:, 13:16] = torch.tensor(d["specular"], dtype=torch.float32, device=positions.device)
    return rec


def ipc_export(t: torch.Tensor):
    """(64-byte handle, offset) of a device tensor's allocation (CUDA IPC)."""
    L = _lib.load()
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_uint64()
    st = L.nrc_ipc_export(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off))
    if st != 0:
        raise NRCError(f"nrc_ipc_export: {L.nrc_status_string(st).decode()}")
    return bytes(h), off.value


def ipc_export_ptr(ptr: int):
    """(64-byte handle, offset) of the device allocation containing address ptr."""
    L = _lib.load()
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_uint64()
    st = L.nrc_ipc_export(ctypes.c_void_p(int(ptr)), h, ctypes.byref(off))
    if st != 0:
        raise NRCError(f"nrc_ipc_export: {L.nrc_status_string(st).decode()}")
    return bytes(h), off.value


def ipc_import(handle: bytes, offset: int) -> int:
    """Device pointer (int) to another process's allocation + offset."""
    L = _lib.load()
    hb = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    p = ctypes.c_void_p()
    st = L.nrc_ipc_import(hb, int(offset), ctypes.byref(p))
    if st != 0:
        raise NRCError(f"nrc_ipc_import: {L.nrc_status_string(st).decode()}")
    return int(p.value)


def ipc_close(ptr: int, offset: int):
    L = _lib.load()
    L.nrc_ipc_close(ctypes.c_void_p(ptr), int(offset))


def lcg_params(n: int, seed: int):
    """LCG constants (a, c, m) of reading R15, from the C ABI."""
    L = _lib.load()
    a, c, m = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    st = L.nrc_lcg_params(int(n), int(seed) & (2 ** 64 - 1), ctypes.byref(a), ctypes.byref(c), ctypes.byref(m))
    if st != 0:
        raise NRCError(f"nrc_lcg_params: {L.nrc_status_string(st).decode()}")
    return a.value, c.value, m.value


class RadianceCache:
    """The neural radiance cache on one GPU (state in a torch-owned arena)."""

    def __init__(self, config: Optional[Config] = None, device: int = 0):
        if not torch.cuda.is_available():
            raise NRCError("RadianceCache needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        self.L = _lib.load()
        self.config = config or Config()
        self.device = torch.device("cuda", device)
        self._cfg = self.config.to_c(device)
        nbytes = self.L.nrc_state_bytes(ctypes.byref(self._cfg))
        if nbytes == 0:
            raise NRCError("invalid config")
        self.state = torch.zeros(nbytes + 256, dtype=torch.uint8, device=self.device)
        off = (-self.state.data_ptr()) % 256
        self._state_ptr = self.state.data_ptr() + off
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            st = self.L.nrc_init(ctypes.byref(self._cfg), ctypes.c_void_p(self._state_ptr), nbytes, ctypes.byref(h))
        if st != 0:
            raise NRCError(f"nrc_init failed: {self.L.nrc_status_string(st).decode()}")
        self.h = h
        self.nparam = int(self.L.nrc_param_count(self.h))  # logical parameters at this hidden width

    # ------------------------------------------------------------------ helpers
    def _check(self, st: int, what: str):
        if st != 0:
            msg = self.L.nrc_last_error(self.h)
            raise NRCError(f"{what}: {self.L.nrc_status_string(st).decode()}: {msg.decode() if msg else ''}")

    def _rec(self, records: torch.Tensor) -> torch.Tensor:
        if records.device != self.device or records.dtype != torch.float32 or records.dim() != 2 \
                or records.shape[1] != REC_FLOATS or not records.is_contiguous():
            raise NRCError("records must be a contiguous float32 [n, 16] tensor on the cache's device")
        return records

    def _f32(self, t: torch.Tensor, shape, name: str) -> torch.Tensor:
        if t.device != self.device or t.dtype != torch.float32 or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
            raise NRCError(f"{name} must be a contiguous float32 {tuple(shape)} tensor on the cache's device")
        return t

    @property
    def last_launch_count(self) -> int:
        return int(self.L.nrc_last_launch_count(self.h))

    # ------------------------------------------------------------------ API
    def query(self, records: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Radiance for each record with the EMA weights."""
        records = self._rec(records)
        n = records.shape[0]
        if out is None:
            out = torch.empty((n, 3), dtype=torch.float32, device=self.device)
        self._f32(out, (n, 3), "out")
        self._check(self.L.nrc_query(self.h, _ptr(records), n, _ptr(out), _stream(stream)), "nrc_query")
        return out

    def train_step(self, records: torch.Tensor, targets: torch.Tensor, loss: Optional[torch.Tensor] = None,
                   stream=None) -> torch.Tensor:
        """One Adam + EMA step on the batch; returns the device loss."""
        records = self._rec(records)
        n = records.shape[0]
        self._f32(targets, (n, 3), "targets")
        if loss is None:
            loss = torch.zeros(1, dtype=torch.float32, device=self.device)
        self._check(self.L.nrc_train_step(self.h, _ptr(records), _ptr(targets), n, _ptr(loss), _stream(stream)),
                    "nrc_train_step")
        return loss

    def train_backward(self, records: torch.Tensor, targets: torch.Tensor, grad: Optional[torch.Tensor] = None,
                       loss_sum: Optional[torch.Tensor] = None, pred: Optional[torch.Tensor] = None, stream=None):
        """Un-normalised gradient sum (logical layout) and loss sum over the
        records; `pred` ([n, 3] fp32, optional) receives the training forward's
        factored prediction y * (alpha + beta) (a4, unclamped)."""
        records = self._rec(records)
        n = records.shape[0]
        self._f32(targets, (n, 3), "targets")
        if grad is None:
            grad = torch.empty(self.nparam, dtype=torch.float32, device=self.device)
        if loss_sum is None:
            loss_sum = torch.zeros(1, dtype=torch.float32, device=self.device)
        if pred is not None:
            self._f32(pred, (n, 3), "pred")
        self._check(self.L.nrc_train_backward(self.h, _ptr(records), _ptr(targets), n, _ptr(grad), _ptr(loss_sum),
                                              _ptr(pred), _stream(stream)), "nrc_train_backward")
        return grad, loss_sum

    def train_apply(self, grad_sum: torch.Tensor, n_global: int, loss_sum: Optional[torch.Tensor] = None,
                    loss: Optional[torch.Tensor] = None, stream=None):
        """Adam + EMA with g = grad_sum / n_global (after an all-reduce); with
        loss_sum and loss given, also loss[0] = loss_sum[0] / n_global."""
        self._f32(grad_sum, (self.nparam,), "grad_sum")
        if loss_sum is not None:
            self._f32(loss_sum, tuple(loss_sum.shape), "loss_sum")
        if loss is not None:
            self._f32(loss, tuple(loss.shape), "loss")
        self._check(self.L.nrc_train_apply(self.h, _ptr(grad_sum), int(n_global), _ptr(loss_sum), _ptr(loss),
                                           _stream(stream)), "nrc_train_apply")

    def train_frame(self, records: torch.Tensor, targets: torch.Tensor, s: int = 4, l: int = 16384,
                    shuffle_seed: int = 0, losses: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """A frame's training: LCG shuffle into s batches of l records."""
        records = self._rec(records)
        n = records.shape[0]
        self._f32(targets, (n, 3), "targets")
        if losses is None:
            losses = torch.zeros(max(int(s), 1), dtype=torch.float32, device=self.device)
        self._check(self.L.nrc_train_frame(self.h, _ptr(records), _ptr(targets), n, int(s), int(l),
                                           int(shuffle_seed) & (2 ** 64 - 1), _ptr(losses), _stream(stream)),
                    "nrc_train_frame")
        return losses

    @property
    def state_ptr(self) -> int:
        """Device address of this cache's state arena (256-byte aligned)."""
        return self._state_ptr

    def train_frame_dp_peer(self, records: torch.Tensor, targets: torch.Tensor, s: int, l: int, shuffle_seed: int,
                            rank: int, world: int, peer_states, losses: Optional[torch.Tensor] = None,
                            stream=None) -> torch.Tensor:
        """nrc_train_frame_dp_peer: data-parallel frame training with the
        gradient all-reduce fused into the optimiser over peer memory
        (peer_states: every rank's state-arena address, own included)."""
        records = self._rec(records)
        n = records.shape[0]
        self._f32(targets, (n, 3), "targets")
        if len(peer_states) != world:
            raise NRCError("one state arena per rank required")
        ps = (ctypes.c_void_p * world)(*[int(p) for p in peer_states])
        if losses is None:
            losses = torch.zeros(max(int(s), 1), dtype=torch.float32, device=self.device)
        self._check(self.L.nrc_train_frame_dp_peer(self.h, _ptr(records), _ptr(targets), n, int(s), int(l),
                                                   int(shuffle_seed) & (2 ** 64 - 1), int(rank), int(world), ps,
                                                   _ptr(losses), _stream(stream)), "nrc_train_frame_dp_peer")
        return losses

    def train_apply_multimem(self, mc_ptr: int, n_global: int, loss: Optional[torch.Tensor] = None, stream=None):
        """nrc_train_apply_multimem: Adam + EMA on the NVSwitch-reduced sum of
        every rank's [gradient | loss sum] buffer (mc_ptr: its multicast
        address), divided by n_global."""
        if loss is not None:
            self._f32(loss, tuple(loss.shape), "loss")
        self._check(self.L.nrc_train_apply_multimem(self.h, ctypes.c_void_p(int(mc_ptr)), int(n_global), _ptr(loss),
                                                    _stream(stream)), "nrc_train_apply_multimem")

    def train_apply_peers(self, buf_ptrs, n_global: int, loss: Optional[torch.Tensor] = None, stream=None):
        """nrc_train_apply_peers: Adam + EMA on the rank-order sum of every
        rank's [gradient | loss sum] buffer (buf_ptrs: device addresses, own
        included, peers' mapped over NVLink), divided by n_global."""
        if loss is not None:
            self._f32(loss, tuple(loss.shape), "loss")
        ps = (ctypes.c_void_p * len(buf_ptrs))(*[int(p) for p in buf_ptrs])
        self._check(self.L.nrc_train_apply_peers(self.h, ps, len(buf_ptrs), int(n_global), _ptr(loss), _stream(stream)),
                    "nrc_train_apply_peers")

    def peer_barrier(self, counter_ptrs, rank: int, world: int, stream=None):
        """nrc_peer_barrier: cross-rank barrier on the stream over peer-mapped
        u64 counters (counter_ptrs: every rank's counter, own included)."""
        if len(counter_ptrs) != world:
            raise NRCError("one counter per rank required")
        ps = (ctypes.c_void_p * world)(*[int(p) for p in counter_ptrs])
        self._check(self.L.nrc_peer_barrier(self.h, ps, int(rank), int(world), _stream(stream)), "nrc_peer_barrier")

    def dp_timeouts(self) -> int:
        c = ctypes.c_uint64()
        self._check(self.L.nrc_dp_timeouts(self.h, ctypes.byref(c)), "nrc_dp_timeouts")
        return int(c.value)

    def train_frame_backward(self, records: torch.Tensor, targets: torch.Tensor, l: int, shuffle_seed: int, j: int,
                             row_begin: int, row_end: int, grad: Optional[torch.Tensor] = None,
                             loss_sum: Optional[torch.Tensor] = None, stream=None):
        """Gradient/loss sums over rows [row_begin, row_end) of shuffled batch j
        (the data-parallel shard of nrc_train_frame's step j)."""
        records = self._rec(records)
        n = records.shape[0]
        self._f32(targets, (n, 3), "targets")
        if grad is None:
            grad = torch.empty(self.nparam, dtype=torch.float32, device=self.device)
        if loss_sum is None:
            loss_sum = torch.zeros(1, dtype=torch.float32, device=self.device)
        self._check(self.L.nrc_train_frame_backward(self.h, _ptr(records), _ptr(targets), n, int(l),
                                                    int(shuffle_seed) & (2 ** 64 - 1), int(j), int(row_begin),
                                                    int(row_end), _ptr(grad), _ptr(loss_sum), _stream(stream)),
                    "nrc_train_frame_backward")
        return grad, loss_sum

    def query_accumulate(self, records: torch.Tensor, pixel: torch.Tensor, throughput: torch.Tensor,
                         image: torch.Tensor, stream=None) -> torch.Tensor:
        """image[pixel[i]] += throughput[i] * radiance(records[i]),
        fused into the query epilogue (nrc_query_accumulate)."""
        records = self._rec(records)
        n = records.shape[0]
        if pixel.device != self.device or pixel.dtype != torch.int32 or tuple(pixel.shape) != (n,) \
                or not pixel.is_contiguous():
            raise NRCError(f"pixel must be a contiguous int32 [{n}] tensor on the cache's device")
        self._f32(throughput, (n, 3), "throughput")
        if image.device != self.device or image.dtype != torch.float32 or image.dim() != 2 or image.shape[1] != 3 \
                or not image.is_contiguous():
            raise NRCError("image must be a contiguous float32 [n_pixels, 3] tensor on the cache's device")
        self._check(self.L.nrc_query_accumulate(self.h, _ptr(records), n, _ptr(pixel), _ptr(throughput), _ptr(image),
                                                _stream(stream)), "nrc_query_accumulate")
        return image

    def assemble_targets(self, first: torch.Tensor, length: torch.Tensor, flags: torch.Tensor,
                         vert: torch.Tensor, tail: torch.Tensor, targets: Optional[torch.Tensor] = None,
                         stream=None) -> torch.Tensor:
        """Self-training targets: per-vertex radiance transported
        back from each training path's tail (see nrc_assemble_targets)."""
        n_paths = first.shape[0]
        for t, name in ((first, "first"), (length, "length"), (flags, "flags")):
            if t.device != self.device or t.dtype != torch.int32 or tuple(t.shape) != (n_paths,) \
                    or not t.is_contiguous():
                raise NRCError(f"{name} must be a contiguous int32 [{n_paths}] tensor on the cache's device")
        nv = vert.shape[0]
        self._f32(vert, (nv, 9), "vert")
        self._f32(tail, (n_paths, 3), "tail")
        if targets is None:
            targets = torch.empty((nv, 3), dtype=torch.float32, device=self.device)
        self._f32(targets, (nv, 3), "targets")
        self._check(self.L.nrc_assemble_targets(self.h, _ptr(first), _ptr(length), _ptr(flags), int(n_paths),
                                                _ptr(vert), _ptr(tail), _ptr(targets), _stream(stream)),
                    "nrc_assemble_targets")
        return targets

    def self_training_targets(self, first, length, flags, vert, tail_records, stream=None) -> torch.Tensor:
        """Query the cache at every path's terminal vertex (nrc_query, the
        ~1 % extra queries of P:L1030-1032), then assemble the targets."""
        tail = self.query(tail_records, stream=stream)
        return self.assemble_targets(first, length, flags, vert, tail, stream=stream)

    def encode(self, records: torch.Tensor, stream=None) -> torch.Tensor:
        """The 64-dim fp16 network input of each record (Table 1 + padding)."""
        records = self._rec(records)
        n = records.shape[0]
        out = torch.empty((n, 64), dtype=torch.float16, device=self.device)
        self._check(self.L.nrc_encode(self.h, _ptr(records), n, _ptr(out), _stream(stream)), "nrc_encode")
        return out

    def get_params(self, which: str = "train") -> np.ndarray:
        out = np.zeros(self.nparam, np.float32)
        self._check(self.L.nrc_get_params(self.h, _PARAM_SETS[which], out.ctypes.data, self.nparam),
                    "nrc_get_params")
        return out

    def set_params(self, values, which: str = "train"):
        v = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        if v.size != self.nparam:
            raise NRCError(f"expected {self.nparam} parameters")
        self._check(self.L.nrc_set_params(self.h, _PARAM_SETS[which], v.ctypes.data, self.nparam),
                    "nrc_set_params")

    def stats(self) -> dict:
        a, b, c, d = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self.L.nrc_get_stats(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)),
                    "nrc_get_stats")
        return {"step": a.value, "nonfinite_grads": b.value, "nonfinite_targets": c.value,
                "degenerate_vectors": d.value}

    def frame_host(self, query_rec: np.ndarray, rgb_out: np.ndarray, train_rec: np.ndarray, train_tgt: np.ndarray,
                   s: int, l: int, shuffle_seed: int, losses_out: np.ndarray, scratch: torch.Tensor, stream=None):
        """End-to-end frame from host buffers (pinned numpy views recommended)."""
        nq, nt = query_rec.shape[0], train_rec.shape[0]
        self._check(self.L.nrc_frame_host(self.h, query_rec.ctypes.data, nq, rgb_out.ctypes.data,
                                          train_rec.ctypes.data, train_tgt.ctypes.data, nt, int(s), int(l),
                                          int(shuffle_seed) & (2 ** 64 - 1), losses_out.ctypes.data,
                                          _ptr(scratch), scratch.numel(), _stream(stream)), "nrc_frame_host")

    def frame_scratch_bytes(self, n_query: int, n_train: int) -> int:
        return int(self.L.nrc_frame_scratch_bytes(int(n_query), int(n_train)))

    def close(self):
        if getattr(self, "h", None):
            self.L.nrc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _McOwner:
    """Releases a libnrc multicast buffer when the tensor view dies."""

    def __init__(self, L, uc):
        self.L, self.uc = L, uc

    def __del__(self):
        try:
            self.L.nrc_multicast_free(ctypes.c_void_p(self.uc))
        except Exception:
            pass


def multicast_alloc(n_floats: int, device=None):
    """nrc_multicast_alloc: a zeroed fp32 buffer of n_floats on one GPU with a
    multicast (NVLS) mapping.  Returns (tensor view of the unicast mapping,
    multicast address)."""
    L = _lib.load()
    dev = torch.device(device if device is not None else "cuda")
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
    st = L.nrc_multicast_alloc(int(idx), int(n_floats) * 4, ctypes.byref(uc), ctypes.byref(mc))
    if st != 0:
        raise RuntimeError(f"NVLS multicast is not available: nrc_multicast_alloc {L.nrc_status_string(st).decode()}")
    owner = _McOwner(L, uc.value)
    # a tensor view of the unicast mapping; the owner frees it with the tensor
    t = _tensor_from_ptr(uc.value, int(n_floats), dev, owner)
    return t, int(mc.value)


def _tensor_from_ptr(ptr: int, n: int, dev: torch.device, owner) -> torch.Tensor:
    """A float32 tensor viewing n floats of device memory at ptr (kept alive by owner)."""
    class _Cai:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                             "strides": None}
            self._owner = owner
    holder = _Cai()
    t = torch.as_tensor(holder, device=dev)
    t._nrc_owner = holder  # the tensor keeps the owner (and so the mapping) alive
    return t


def selftest_umma(mode: int, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Diagnostic tcgen05 tile product (nrc_selftest_umma) on fp16 inputs."""
    L = _lib.load()
    shape = {0: (128, 64), 1: (128, 64), 2: (64, 64), 3: (128, 16), 4: (128, 64)}[mode]
    d = torch.zeros(shape, dtype=torch.float32, device=a.device)
    a = a.contiguous()
    b = b.contiguous()
    st = L.nrc_selftest_umma(mode, _ptr(a), _ptr(b), _ptr(d))
    if st != 0:
        raise NRCError(f"nrc_selftest_umma: {L.nrc_status_string(st).decode()}")
    return d
