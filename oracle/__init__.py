"""ctypes wrapper around oracle/liboracle.so -- the fp64 CPU oracle.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_2106_12372_b200`` never imports it and
shares no code with it (see nrc_oracle.c header).  Every function here is
argument marshalling only; the arithmetic lives in nrc_oracle.c, which cites
the paper passage each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nrc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NPARAM = 5 * 64 * 64 + 3 * 64  # 20,672 logical parameters (reading R1)
MAT_OFF = [0, 4096, 8192, 12288, 16384, 20480, 20672]
MAT_ROWS = [64, 64, 64, 64, 64, 3]
FACTORIZE = 1
CLAMP_QUERY = 2

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _u64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, f, i64, u64, vp = ctypes.c_double, ctypes.c_float, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        L.orc_tri.restype = d; L.orc_tri.argtypes = [d]
        L.orc_quartic.restype = d; L.orc_quartic.argtypes = [d]
        L.orc_one_blob.restype = None; L.orc_one_blob.argtypes = [d, ctypes.c_int, vp]
        L.orc_sph.restype = ctypes.c_int; L.orc_sph.argtypes = [vp, vp]
        L.orc_freq.restype = None; L.orc_freq.argtypes = [d, vp]
        L.orc_normalize_pos.restype = f; L.orc_normalize_pos.argtypes = [f, f, f]
        L.orc_encode.restype = ctypes.c_int; L.orc_encode.argtypes = [vp, vp, vp, vp]
        L.orc_encode_batch.restype = None; L.orc_encode_batch.argtypes = [vp, i64, vp, vp, vp]
        L.orc_forward.restype = None; L.orc_forward.argtypes = [vp, vp, vp, vp]
        L.orc_query_batch.restype = None; L.orc_query_batch.argtypes = [vp, vp, i64, vp, vp, ctypes.c_uint, vp]
        L.orc_loss.restype = d; L.orc_loss.argtypes = [vp, vp, d, vp]
        L.orc_loss_frozen.restype = d; L.orc_loss_frozen.argtypes = [vp, vp, d, d]
        L.orc_backward.restype = None; L.orc_backward.argtypes = [vp, vp, vp, vp]
        L.orc_grad_batch.restype = None
        L.orc_grad_batch.argtypes = [vp, vp, vp, i64, vp, vp, d, ctypes.c_uint, vp, vp, vp]
        L.orc_grad_batch_exact.restype = None
        L.orc_grad_batch_exact.argtypes = [vp, vp, vp, i64, vp, vp, d, ctypes.c_uint, vp, vp, vp]
        L.orc_adam.restype = i64; L.orc_adam.argtypes = [vp, vp, vp, vp, i64, i64, d, d, d, d]
        L.orc_ema.restype = None; L.orc_ema.argtypes = [vp, vp, i64, i64, d, ctypes.c_int]
        L.orc_lcg_params.restype = None; L.orc_lcg_params.argtypes = [u64, u64, vp, vp, vp]
        L.orc_lcg_perm.restype = u64; L.orc_lcg_perm.argtypes = [u64, u64, u64, u64, u64]
        L.orc_lcg_permute.restype = None; L.orc_lcg_permute.argtypes = [u64, u64, u64, u64, vp]
        L.orc_init_weights.restype = None; L.orc_init_weights.argtypes = [u64, vp]
        L.orc_param_count.restype = i64; L.orc_param_count.argtypes = []
        L.orc_param_count_w.restype = i64; L.orc_param_count_w.argtypes = [ctypes.c_int]
        L.orc_forward_w.restype = None; L.orc_forward_w.argtypes = [ctypes.c_int, vp, vp, vp]
        L.orc_query_batch_w.restype = None
        L.orc_query_batch_w.argtypes = [ctypes.c_int, vp, vp, i64, vp, vp, ctypes.c_uint, vp]
        L.orc_init_weights_w.restype = None; L.orc_init_weights_w.argtypes = [ctypes.c_int, u64, vp]
        L.orc_forward_stash_w.restype = None; L.orc_forward_stash_w.argtypes = [ctypes.c_int, vp, vp, vp, vp]
        L.orc_backward_w.restype = None; L.orc_backward_w.argtypes = [ctypes.c_int, vp, vp, vp, vp]
        L.orc_grad_batch_w.restype = None
        L.orc_grad_batch_w.argtypes = [ctypes.c_int, vp, vp, vp, i64, vp, vp, d, ctypes.c_uint, vp, vp, vp]
        L.orc_train_step_w.restype = d
        L.orc_train_step_w.argtypes = [ctypes.c_int, vp, vp, vp, vp, i64, vp, vp, i64, vp, vp, d, ctypes.c_uint,
                                       d, d, d, d, d, ctypes.c_int, vp, vp, vp]
        ci = ctypes.c_int
        L.orc_param_count_d.restype = i64; L.orc_param_count_d.argtypes = [ci, ci]
        L.orc_forward_stash_d.restype = None; L.orc_forward_stash_d.argtypes = [ci, ci, vp, vp, vp, vp]
        L.orc_backward_d.restype = None; L.orc_backward_d.argtypes = [ci, ci, vp, vp, vp, vp]
        L.orc_query_batch_d.restype = None; L.orc_query_batch_d.argtypes = [ci, ci, vp, vp, i64, vp, vp, ctypes.c_uint, vp]
        L.orc_grad_batch_d.restype = None
        L.orc_grad_batch_d.argtypes = [ci, ci, vp, vp, vp, i64, vp, vp, d, ctypes.c_uint, vp, vp, vp]
        L.orc_init_weights_d.restype = None; L.orc_init_weights_d.argtypes = [ci, ci, u64, vp]
        L.orc_train_step_d.restype = d
        L.orc_train_step_d.argtypes = [ci, ci, vp, vp, vp, vp, i64, vp, vp, i64, vp, vp, d, ctypes.c_uint,
                                       d, d, d, d, d, ctypes.c_int, vp, vp, vp]
        L.orc_gauss.restype = d; L.orc_gauss.argtypes = [d]
        L.orc_freq_sin.restype = None; L.orc_freq_sin.argtypes = [d, vp]
        L.orc_one_blob_gauss.restype = None; L.orc_one_blob_gauss.argtypes = [d, ctypes.c_int, vp]
        L.orc_encode_batch_exact.restype = None; L.orc_encode_batch_exact.argtypes = [vp, i64, vp, vp, vp]
        L.orc_query_batch_exact.restype = None
        L.orc_query_batch_exact.argtypes = [vp, vp, i64, vp, vp, ctypes.c_uint, vp]
        L.orc_query_accumulate.restype = None
        L.orc_query_accumulate.argtypes = [vp, vp, i64, vp, vp, ctypes.c_uint, vp, vp, vp]
        L.orc_assemble_targets.restype = None
        L.orc_assemble_targets.argtypes = [vp, vp, vp, i64, vp, vp, vp]
        L.orc_train_step.restype = d
        L.orc_train_step.argtypes = [vp, vp, vp, vp, i64, vp, vp, i64, vp, vp, d, ctypes.c_uint,
                                     d, d, d, d, d, ctypes.c_int, vp, vp, vp]
        _lib = L
    return _lib


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- primitives
def tri(x: float) -> float:
    return lib().orc_tri(float(x))


def quartic(x: float) -> float:
    return lib().orc_quartic(float(x))


def one_blob(s: float, k: int = 4) -> np.ndarray:
    out = np.zeros(k, np.float64)
    lib().orc_one_blob(float(s), int(k), out.ctypes.data)
    return out


def sph(u) -> np.ndarray:
    u = _c(u, np.float64)
    out = np.zeros(2, np.float64)
    lib().orc_sph(u.ctypes.data, out.ctypes.data)
    return out


def freq(v: float) -> np.ndarray:
    out = np.zeros(12, np.float64)
    lib().orc_freq(float(v), out.ctypes.data)
    return out


def normalize_pos(p: float, lo: float, hi: float) -> float:
    return lib().orc_normalize_pos(p, lo, hi)


def encode(recs, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1)) -> np.ndarray:
    recs = _c(recs, np.float32).reshape(-1, 16)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    out = np.zeros((recs.shape[0], 64), np.float64)
    lib().orc_encode_batch(recs.ctypes.data, recs.shape[0], lo.ctypes.data, hi.ctypes.data, out.ctypes.data)
    return out


# ---------------------------------------------------------------- network
def forward(W, e):
    """Returns (H [6,64], y [3]) for one encoded input e [64]."""
    W = _c(W, np.float64); e = _c(e, np.float64)
    H = np.zeros((6, 64), np.float64); y = np.zeros(3, np.float64)
    lib().orc_forward(W.ctypes.data, e.ctypes.data, H.ctypes.data, y.ctypes.data)
    return H, y


def query(W, recs, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), flags=FACTORIZE | CLAMP_QUERY) -> np.ndarray:
    W = _c(W, np.float64)
    recs = _c(recs, np.float32).reshape(-1, 16)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    q = np.zeros((recs.shape[0], 3), np.float64)
    lib().orc_query_batch(W.ctypes.data, recs.ctypes.data, recs.shape[0], lo.ctypes.data, hi.ctypes.data,
                          int(flags), q.ctypes.data)
    return q


# ---------------------------------------------------------------- width ablation (C4)
def param_count_w(hw: int) -> int:
    return int(lib().orc_param_count_w(int(hw)))


def forward_w(hw, W, e):
    W = _c(W, np.float64); e = _c(e, np.float64)
    y = np.zeros(3, np.float64)
    lib().orc_forward_w(int(hw), W.ctypes.data, e.ctypes.data, y.ctypes.data)
    return y


def query_w(hw, W, recs, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), flags=FACTORIZE | CLAMP_QUERY) -> np.ndarray:
    W = _c(W, np.float64)
    assert W.size == param_count_w(hw)
    recs = _c(recs, np.float32).reshape(-1, 16)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    q = np.zeros((recs.shape[0], 3), np.float64)
    lib().orc_query_batch_w(int(hw), W.ctypes.data, recs.ctypes.data, recs.shape[0], lo.ctypes.data,
                            hi.ctypes.data, int(flags), q.ctypes.data)
    return q


def init_weights_w(hw: int, seed: int) -> np.ndarray:
    W = np.zeros(param_count_w(hw), np.float32)
    lib().orc_init_weights_w(int(hw), int(seed) & (2**64 - 1), W.ctypes.data)
    return W


def forward_stash_w(hw, W, e):
    """(H = [h0 (64) | h1..h5 (hw each)], y [3]) for one encoded input at width hw."""
    W = _c(W, np.float64); e = _c(e, np.float64)
    H = np.zeros(64 + 5 * hw, np.float64); y = np.zeros(3, np.float64)
    lib().orc_forward_stash_w(int(hw), W.ctypes.data, e.ctypes.data, H.ctypes.data, y.ctypes.data)
    return H, y


def backward_w(hw, W, H, dy):
    W = _c(W, np.float64); H = _c(H, np.float64); dy = _c(dy, np.float64)
    G = np.zeros(param_count_w(hw), np.float64)
    lib().orc_backward_w(int(hw), W.ctypes.data, H.ctypes.data, dy.ctypes.data, G.ctypes.data)
    return G


def grad_batch_w(hw, W, recs, tgts, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), eps=0.01, flags=FACTORIZE):
    """grad_batch at hidden width hw (C4): un-normalised gradient sum, loss sum, #bad targets."""
    W = _c(W, np.float64)
    assert W.size == param_count_w(hw)
    recs = _c(recs, np.float32).reshape(-1, 16)
    tgts = _c(tgts, np.float32).reshape(-1, 3)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    G = np.zeros(param_count_w(hw), np.float64)
    ls = np.zeros(1, np.float64)
    nb = np.zeros(1, np.int64)
    lib().orc_grad_batch_w(int(hw), W.ctypes.data, recs.ctypes.data, tgts.ctypes.data, recs.shape[0],
                           lo.ctypes.data, hi.ctypes.data, float(eps), int(flags), G.ctypes.data, ls.ctypes.data,
                           nb.ctypes.data)
    return G, float(ls[0]), int(nb[0])


# ---------------------------------------------------------------- depth variants (N4)
def param_count_d(hw: int, nh: int) -> int:
    return int(lib().orc_param_count_d(int(hw), int(nh)))


def forward_stash_d(hw, nh, W, e):
    W = _c(W, np.float64); e = _c(e, np.float64)
    H = np.zeros(64 + nh * hw, np.float64); y = np.zeros(3, np.float64)
    lib().orc_forward_stash_d(int(hw), int(nh), W.ctypes.data, e.ctypes.data, H.ctypes.data, y.ctypes.data)
    return H, y


def backward_d(hw, nh, W, H, dy):
    W = _c(W, np.float64); H = _c(H, np.float64); dy = _c(dy, np.float64)
    G = np.zeros(param_count_d(hw, nh), np.float64)
    lib().orc_backward_d(int(hw), int(nh), W.ctypes.data, H.ctypes.data, dy.ctypes.data, G.ctypes.data)
    return G


def query_d(hw, nh, W, recs, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), flags=FACTORIZE | CLAMP_QUERY) -> np.ndarray:
    W = _c(W, np.float64)
    assert W.size == param_count_d(hw, nh)
    recs = _c(recs, np.float32).reshape(-1, 16)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    q = np.zeros((recs.shape[0], 3), np.float64)
    lib().orc_query_batch_d(int(hw), int(nh), W.ctypes.data, recs.ctypes.data, recs.shape[0], lo.ctypes.data,
                            hi.ctypes.data, int(flags), q.ctypes.data)
    return q


def grad_batch_d(hw, nh, W, recs, tgts, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), eps=0.01, flags=FACTORIZE):
    W = _c(W, np.float64)
    assert W.size == param_count_d(hw, nh)
    recs = _c(recs, np.float32).reshape(-1, 16)
    tgts = _c(tgts, np.float32).reshape(-1, 3)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    G = np.zeros(param_count_d(hw, nh), np.float64)
    ls = np.zeros(1, np.float64)
    nb = np.zeros(1, np.int64)
    lib().orc_grad_batch_d(int(hw), int(nh), W.ctypes.data, recs.ctypes.data, tgts.ctypes.data, recs.shape[0],
                           lo.ctypes.data, hi.ctypes.data, float(eps), int(flags), G.ctypes.data, ls.ctypes.data,
                           nb.ctypes.data)
    return G, float(ls[0]), int(nb[0])


def init_weights_d(hw: int, nh: int, seed: int) -> np.ndarray:
    W = np.zeros(param_count_d(hw, nh), np.float32)
    lib().orc_init_weights_d(int(hw), int(nh), int(seed) & (2**64 - 1), W.ctypes.data)
    return W


# ---------------------------------------------------------------- exact encodings (N4)
def gauss(x: float) -> float:
    return lib().orc_gauss(float(x))


def freq_sin(v: float) -> np.ndarray:
    out = np.zeros(12, np.float64)
    lib().orc_freq_sin(float(v), out.ctypes.data)
    return out


def one_blob_gauss(s: float, k: int = 4) -> np.ndarray:
    out = np.zeros(k, np.float64)
    lib().orc_one_blob_gauss(float(s), int(k), out.ctypes.data)
    return out


def encode_exact(recs, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1)) -> np.ndarray:
    recs = _c(recs, np.float32).reshape(-1, 16)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    out = np.zeros((recs.shape[0], 64), np.float64)
    lib().orc_encode_batch_exact(recs.ctypes.data, recs.shape[0], lo.ctypes.data, hi.ctypes.data, out.ctypes.data)
    return out


def query_exact(W, recs, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), flags=FACTORIZE | CLAMP_QUERY) -> np.ndarray:
    W = _c(W, np.float64)
    recs = _c(recs, np.float32).reshape(-1, 16)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    q = np.zeros((recs.shape[0], 3), np.float64)
    lib().orc_query_batch_exact(W.ctypes.data, recs.ctypes.data, recs.shape[0], lo.ctypes.data, hi.ctypes.data,
                                int(flags), q.ctypes.data)
    return q


# ---------------------------------------------------------------- pixel reconstruction (N2)
def query_accumulate(W, recs, pix, thr, image, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1),
                     flags=FACTORIZE | CLAMP_QUERY) -> np.ndarray:
    """image [n_pixels, 3] fp64 (updated copy) += thr * query(recs) at pix."""
    W = _c(W, np.float64)
    recs = _c(recs, np.float32).reshape(-1, 16)
    pix = _c(pix, np.uint32); thr = _c(thr, np.float32).reshape(-1, 3)
    img = np.array(image, np.float64, copy=True, order="C")
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    lib().orc_query_accumulate(W.ctypes.data, recs.ctypes.data, recs.shape[0], lo.ctypes.data, hi.ctypes.data,
                               int(flags), pix.ctypes.data, thr.ctypes.data, img.ctypes.data)
    return img


# ---------------------------------------------------------------- self-training targets (N1)
def assemble_targets(first, length, flags, vert, tail) -> np.ndarray:
    """Per-vertex targets [n_vertices, 3] (fp64) of orc_assemble_targets."""
    first = _c(first, np.uint32); length = _c(length, np.uint32); flags = _c(flags, np.uint32)
    vert = _c(vert, np.float32).reshape(-1, 9); tail = _c(tail, np.float32).reshape(-1, 3)
    out = np.zeros((vert.shape[0], 3), np.float64)
    lib().orc_assemble_targets(first.ctypes.data, length.ctypes.data, flags.ctypes.data, first.size,
                               vert.ctypes.data, tail.ctypes.data, out.ctypes.data)
    return out


def loss(yhat, t, eps=0.01):
    yhat = _c(yhat, np.float64); t = _c(t, np.float64)
    d = np.zeros(3, np.float64)
    l = lib().orc_loss(yhat.ctypes.data, t.ctypes.data, float(eps), d.ctypes.data)
    return l, d


def loss_frozen(yhat, t, eps, lam):
    yhat = _c(yhat, np.float64); t = _c(t, np.float64)
    return lib().orc_loss_frozen(yhat.ctypes.data, t.ctypes.data, float(eps), float(lam))


def backward(W, H, dy):
    W = _c(W, np.float64); H = _c(H, np.float64); dy = _c(dy, np.float64)
    G = np.zeros(NPARAM, np.float64)
    lib().orc_backward(W.ctypes.data, H.ctypes.data, dy.ctypes.data, G.ctypes.data)
    return G


def grad_batch(W, recs, tgts, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), eps=0.01, flags=FACTORIZE, exact=False):
    """Un-normalised sum over records of dl/dW, the loss sum, #bad targets
    (exact=True: with the exact encoding, N4)."""
    W = _c(W, np.float64)
    recs = _c(recs, np.float32).reshape(-1, 16)
    tgts = _c(tgts, np.float32).reshape(-1, 3)
    lo, hi = _c(aabb_lo, np.float32), _c(aabb_hi, np.float32)
    G = np.zeros(NPARAM, np.float64)
    ls = np.zeros(1, np.float64)
    nb = np.zeros(1, np.int64)
    fn = lib().orc_grad_batch_exact if exact else lib().orc_grad_batch
    fn(W.ctypes.data, recs.ctypes.data, tgts.ctypes.data, recs.shape[0], lo.ctypes.data,
                         hi.ctypes.data, float(eps), int(flags), G.ctypes.data, ls.ctypes.data, nb.ctypes.data)
    return G, float(ls[0]), int(nb[0])


def adam(w, m, v, g, t, lr=1e-2, b1=0.9, b2=0.99, eps=1e-8):
    """In-place Adam on fp64 arrays; returns #non-finite gradient entries."""
    for a in (w, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = _c(g, np.float64)
    return lib().orc_adam(w.ctypes.data, m.ctypes.data, v.ctypes.data, g.ctypes.data, w.size, int(t),
                          float(lr), float(b1), float(b2), float(eps))


def ema(wbar, w, t, a=0.99, printed_form=False):
    assert wbar.dtype == np.float64 and wbar.flags.c_contiguous
    w = _c(w, np.float64)
    lib().orc_ema(wbar.ctypes.data, w.ctypes.data, wbar.size, int(t), float(a), int(bool(printed_form)))


def lcg_params(n, seed):
    a = np.zeros(1, np.uint64); c = np.zeros(1, np.uint64); m = np.zeros(1, np.uint64)
    lib().orc_lcg_params(int(n), int(seed) & (2**64 - 1), a.ctypes.data, c.ctypes.data, m.ctypes.data)
    return int(a[0]), int(c[0]), int(m[0])


def lcg_permute(n, a, c, m) -> np.ndarray:
    out = np.zeros(int(n), np.uint64)
    lib().orc_lcg_permute(int(n), int(a), int(c), int(m), out.ctypes.data)
    return out


def init_weights(seed: int) -> np.ndarray:
    W = np.zeros(NPARAM, np.float32)
    lib().orc_init_weights(int(seed) & (2**64 - 1), W.ctypes.data)
    return W


class OracleCache:
    """fp64 mirror of the cache state (W, m, v, W-bar, t) stepping with
    orc_train_step."""

    def __init__(self, W32=None, seed=1, aabb_lo=(0, 0, 0), aabb_hi=(1, 1, 1), lr=1e-2, b1=0.9, b2=0.99,
                 adam_eps=1e-8, loss_eps=0.01, ema_alpha=0.99, flags=FACTORIZE | CLAMP_QUERY,
                 ema_printed=False, hidden_width=64, hidden_layers=5):
        self.hw = int(hidden_width)
        self.nh = int(hidden_layers)
        if W32 is None:
            W32 = (init_weights_d(self.hw, self.nh, seed) if self.nh != 5 else
                   init_weights(seed) if self.hw == 64 else init_weights_w(self.hw, seed))
        W32 = np.asarray(W32, np.float32)
        self.P = param_count_d(self.hw, self.nh) if self.nh != 5 else NPARAM if self.hw == 64 else param_count_w(self.hw)
        assert W32.size == self.P
        self.w = W32.astype(np.float64)
        self.m = np.zeros(self.P); self.v = np.zeros(self.P)
        self.wbar = self.w.copy()
        self.t = 0
        self.lo = _c(aabb_lo, np.float32); self.hi = _c(aabb_hi, np.float32)
        self.lr, self.b1, self.b2, self.adam_eps = lr, b1, b2, adam_eps
        self.loss_eps, self.ema_alpha, self.flags, self.ema_printed = loss_eps, ema_alpha, flags, ema_printed
        self.bad_grads = 0
        self.bad_targets = 0

    def train_step(self, recs, tgts, return_grad=False):
        recs = _c(recs, np.float32).reshape(-1, 16)
        tgts = _c(tgts, np.float32).reshape(-1, 3)
        n = recs.shape[0]
        if n == 0:
            return 0.0
        self.t += 1
        G = np.zeros(self.P, np.float64)
        bg = np.zeros(1, np.int64); bt = np.zeros(1, np.int64)
        if self.nh != 5:
            l = lib().orc_train_step_d(self.hw, self.nh, self.w.ctypes.data, self.m.ctypes.data, self.v.ctypes.data,
                                       self.wbar.ctypes.data, self.t, recs.ctypes.data, tgts.ctypes.data, n,
                                       self.lo.ctypes.data, self.hi.ctypes.data, self.loss_eps,
                                       int(self.flags & FACTORIZE), self.lr, self.b1, self.b2, self.adam_eps,
                                       self.ema_alpha, int(self.ema_printed), G.ctypes.data, bg.ctypes.data,
                                       bt.ctypes.data)
            self.bad_grads += int(bg[0]); self.bad_targets += int(bt[0])
            return (l, G) if return_grad else l
        if self.hw != 64:
            l = lib().orc_train_step_w(self.hw, self.w.ctypes.data, self.m.ctypes.data, self.v.ctypes.data,
                                       self.wbar.ctypes.data, self.t, recs.ctypes.data, tgts.ctypes.data, n,
                                       self.lo.ctypes.data, self.hi.ctypes.data, self.loss_eps,
                                       int(self.flags & FACTORIZE), self.lr, self.b1, self.b2, self.adam_eps,
                                       self.ema_alpha, int(self.ema_printed), G.ctypes.data, bg.ctypes.data,
                                       bt.ctypes.data)
            self.bad_grads += int(bg[0]); self.bad_targets += int(bt[0])
            return (l, G) if return_grad else l
        l = lib().orc_train_step(self.w.ctypes.data, self.m.ctypes.data, self.v.ctypes.data, self.wbar.ctypes.data,
                                 self.t, recs.ctypes.data, tgts.ctypes.data, n, self.lo.ctypes.data,
                                 self.hi.ctypes.data, self.loss_eps, int(self.flags & FACTORIZE), self.lr, self.b1,
                                 self.b2, self.adam_eps, self.ema_alpha, int(self.ema_printed), G.ctypes.data,
                                 bg.ctypes.data, bt.ctypes.data)
        self.bad_grads += int(bg[0]); self.bad_targets += int(bt[0])
        return (l, G) if return_grad else l

    def query(self, recs, use_ema=True):
        W = self.wbar if (use_ema and self.ema_alpha > 0) else self.w
        if self.nh != 5:
            return query_d(self.hw, self.nh, W, recs, self.lo, self.hi, self.flags)
        if self.hw != 64:
            return query_w(self.hw, W, recs, self.lo, self.hi, self.flags)
        return query(W, recs, self.lo, self.hi, self.flags)
