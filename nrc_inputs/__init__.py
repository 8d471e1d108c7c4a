"""Seeded synthetic inputs shared (as DATA, not code) by the oracle tests, the
CUDA parity tests and bench.py.

This module holds none of the method's arithmetic: it draws cache records
shaped like the paper's workload and evaluates a fixed analytic radiance
field used as training targets.  Record layout (16 fp32 = 64 B, the shape of
a cache query, Table 1):

    pos[3] dir[3] normal[3] roughness diffuse[3] specular[3]

Distribution ("input recipe"):
  * pos ~ U[0,1)^3 (AABB = unit cube),
  * dir, normal = normalised N(0, I3), rejecting |y| < 1e-7 (avoids the
    signed-zero seam of atan2 at phi = +-pi),
  * roughness ~ Exp(mean 0.5),
  * diffuse ~ U[0,0.6)^3, specular ~ U[0,0.4)^3 (alpha + beta <= 1).

Seeds: queries 0x1080, training frame f -> 0x7EA1 + f,
convergence step j -> 0xC3 + j, weights seed 1.
"""
from __future__ import annotations

import numpy as np

REC_FLOATS = 16
SEED_QUERY = 0x1080
SEED_TRAIN = 0x7EA1
SEED_C3 = 0xC3
SEED_WEIGHTS = 1

# C2 / C5 workload sizes
N_1080P = 1920 * 1080
N_4K = 3840 * 2160
TRAIN_S = 4
TRAIN_L = 16384


def _unit_vectors(rng: np.random.Generator, n: int) -> np.ndarray:
    out = np.empty((n, 3), np.float32)
    filled = 0
    while filled < n:
        k = n - filled
        v = rng.standard_normal((k + 16, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        v = v.astype(np.float32)
        ok = (np.abs(v[:, 1]) >= 1e-7) & np.all(np.isfinite(v), axis=1)
        v = v[ok][:k]
        out[filled:filled + v.shape[0]] = v
        filled += v.shape[0]
    return out


def records(n: int, seed: int = SEED_QUERY) -> np.ndarray:
    """n synthetic cache records, float32 [n, 16]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    r = np.empty((n, REC_FLOATS), np.float32)
    r[:, 0:3] = rng.random((n, 3), dtype=np.float32)
    r[:, 3:6] = _unit_vectors(rng, n)
    r[:, 6:9] = _unit_vectors(rng, n)
    r[:, 9] = rng.exponential(0.5, n).astype(np.float32)
    r[:, 10:13] = (rng.random((n, 3)) * 0.6).astype(np.float32)
    r[:, 13:16] = (rng.random((n, 3)) * 0.4).astype(np.float32)
    return r


_F = np.array([[3.0, 1.0, 2.0], [1.0, 4.0, 2.0], [2.0, 2.0, 5.0]])


def radiance_field(recs: np.ndarray) -> np.ndarray:
    """Analytic stand-in for the scattered radiance L_s (Eq. 1):
    (alpha+beta) * (0.5 + 0.4 sin(2 pi F p + (0,1,2)) + 2 max(0, w.n)^(1/(0.05 + 1 - e^-r)) (1, .8, .6)).
    Smooth in position, glossy lobe in direction; fp64 evaluation -> fp32."""
    p = recs[:, 0:3].astype(np.float64)
    w = recs[:, 3:6].astype(np.float64)
    nrm = recs[:, 6:9].astype(np.float64)
    r = recs[:, 9].astype(np.float64)
    refl = recs[:, 10:13].astype(np.float64) + recs[:, 13:16].astype(np.float64)
    base = 0.5 + 0.4 * np.sin(2 * np.pi * p @ _F.T + np.array([0.0, 1.0, 2.0]))
    cosw = np.clip(np.sum(w * nrm, axis=1), 0.0, None)
    expo = 1.0 / (0.05 + 1.0 - np.exp(-np.maximum(r, 0.0)))
    lobe = 2.0 * cosw[:, None] ** expo[:, None] * np.array([1.0, 0.8, 0.6])
    return (refl * (base + lobe)).astype(np.float32)


def targets(recs: np.ndarray, noise: float = 0.0, seed: int = 0) -> np.ndarray:
    """Training targets: the analytic field, optionally with unbiased
    log-normal multiplicative noise exp(N(0, noise^2)) / E[.] (the noisy
    regime the relative loss targets)."""
    t = radiance_field(recs).astype(np.float64)
    if noise > 0:
        rng = np.random.Generator(np.random.PCG64(seed ^ 0x5EED))
        t *= np.exp(rng.normal(0.0, noise, t.shape) - 0.5 * noise * noise)
    return t.astype(np.float32)


def train_frame(frame: int = 0, n: int = TRAIN_S * TRAIN_L, noise: float = 0.0):
    """One frame's training records + targets (65,536 by default)."""
    rec = records(n, SEED_TRAIN + frame)
    return rec, targets(rec, noise, SEED_TRAIN + frame)


def query_batch(n: int = N_1080P, seed: int = SEED_QUERY) -> np.ndarray:
    return records(n, seed)


SEED_PATHS = 0x5E1F


def training_paths(n_vertices: int = TRAIN_S * TRAIN_L, seed: int = SEED_PATHS, u_inv: int = 16):
    """Synthetic training-path buffers for self-training target assembly
    (SURVEY 8(f) N1).  Path lengths are geometric
    (mean ~3, the paper's short suffixes plus the training extension), cut so
    the vertex count is exactly n_vertices.  Per vertex 9 floats [E N T]:
    emission E (5 % of vertices are emitters, E ~ U[0, 4)), next-event estimate
    N ~ U[0, 0.5), throughput T ~ U[0, 0.9) (energy conserving).  Every
    u_inv-th path (index % u_inv == 0) is flagged unbiased (flag bit 0,
    P:L341-343).  Returns (first, length, flags, vert [n, 9] f32, vertex
    records [n, 16] f32, tail records [n_paths, 16] f32).  Data only: no
    arithmetic of the method."""
    rng = np.random.default_rng(seed)
    lens = []
    total = 0
    while total < n_vertices:
        k = int(min(rng.geometric(1.0 / 3.0), 12, n_vertices - total))
        lens.append(k)
        total += k
    length = np.asarray(lens, np.uint32)
    first = np.concatenate([[0], np.cumsum(length)[:-1]]).astype(np.uint32)
    flags = (np.arange(length.size) % u_inv == 0).astype(np.uint32)
    vert = np.zeros((n_vertices, 9), np.float32)
    emit = rng.random(n_vertices) < 0.05
    vert[:, 0:3] = np.where(emit[:, None], rng.uniform(0, 4, (n_vertices, 3)), 0.0)
    vert[:, 3:6] = rng.uniform(0, 0.5, (n_vertices, 3))
    vert[:, 6:9] = rng.uniform(0, 0.9, (n_vertices, 3))
    vrec = records(n_vertices, seed=seed + 1)
    trec = records(length.size, seed=seed + 2)
    return first, length, flags, vert, vrec, trec


# Off-default domain (Table 1's inputs are x in R^3, omega and n arbitrary
# vectors renormalised by sph, r in R, reflectances in R):
# an offset, non-unit AABB and records inside, outside and far outside it.
DOMAIN_AABB_LO = (-3.7, 2.0, -100.0)
DOMAIN_AABB_HI = (5.1, 9.0, 250.0)


def _domain_vectors(rng: np.random.Generator, n: int) -> np.ndarray:
    """Direction-like vectors covering the encoder's edge cases: unit, non-unit
    (|u| in [1e-3, 1e3]), exact poles (0, 0, +-s), the phi seam (x < 0,
    y = +0.0 or -0.0 exactly), tiny |y| next to the seam, and zero vectors."""
    kind = rng.integers(0, 8, n)
    v = _unit_vectors(rng, n).astype(np.float64)
    mag = 10.0 ** rng.uniform(-3.0, 3.0, n)
    v[kind == 1] *= mag[kind == 1, None]
    s = mag * np.where(rng.random(n) < 0.5, 1.0, -1.0)
    pole = kind == 2
    v[pole] = 0.0
    v[pole, 2] = s[pole]
    seam = (kind == 3) | (kind == 4)
    v[seam, 0] = -np.abs(v[seam, 0]) - 1e-3
    v[seam, 1] = 0.0
    tiny = kind == 5
    v[tiny, 0] = -np.abs(v[tiny, 0]) - 1e-3
    v[tiny, 1] = rng.choice([-1.0, 1.0], tiny.sum()) * 10.0 ** rng.uniform(-30, -8, tiny.sum())
    v[kind == 6] = 0.0
    out = v.astype(np.float32)
    out[kind == 4, 1] = np.float32(-0.0)  # the other side of the seam: atan2(-0, x < 0) = -pi
    return out


def domain_records(n: int, seed: int = 0xD0, lo=DOMAIN_AABB_LO, hi=DOMAIN_AABB_HI) -> np.ndarray:
    """n records over the off-default input domain, float32 [n, 16]:
    positions inside the AABB, on its faces, outside it (up to twice its
    extent) and far outside (|p| up to ~1e3); direction / normal edge cases
    (_domain_vectors); roughness in [-2, 60] (negative reads as 0); diffuse
    and specular in [-0.5, 2) (alpha + beta > 1), with alpha = beta = 0 on
    1/16 of the records."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    ext = hi - lo
    r = np.empty((n, REC_FLOATS), np.float32)
    kind = rng.integers(0, 4, n)
    p = lo + rng.random((n, 3)) * ext                               # inside
    p[kind == 1] = lo + rng.uniform(-1.0, 2.0, ((kind == 1).sum(), 3)) * ext   # outside, near
    far = kind == 2
    p[far] = rng.uniform(-1000.0, 1000.0, (far.sum(), 3))           # far outside
    face = kind == 3
    p[face] = np.where(rng.random((face.sum(), 3)) < 0.5, lo, hi)   # faces / corners exactly
    r[:, 0:3] = p.astype(np.float32)
    r[:, 3:6] = _domain_vectors(rng, n)
    r[:, 6:9] = _domain_vectors(rng, n)
    r[:, 9] = rng.uniform(-2.0, 60.0, n).astype(np.float32)
    r[rng.random(n) < 0.1, 9] = 0.0
    r[:, 10:16] = rng.uniform(-0.5, 2.0, (n, 6)).astype(np.float32)
    r[rng.random(n) < 1.0 / 16, 10:16] = 0.0
    return r


def hdr_targets(n: int, seed: int = 0xD1, lo_exp: float = -3.0, hi_exp: float = 4.0) -> np.ndarray:
    """HDR training targets spanning 10^lo_exp .. 10^hi_exp per channel
    (log-uniform): the bright-emitter / noisy-radiance regime the relative
    loss is built for."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return (10.0 ** rng.uniform(lo_exp, hi_exp, (n, 3))).astype(np.float32)
