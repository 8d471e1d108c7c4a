"""Pins for the oracle's input encoding (Table 1 P:L499-516, P:L586-599,
fig:cheap_primitives P:L674-686).  Each expected value comes from the paper's
closed forms, SPEC's worked examples, or mathematics independent
of the oracle (inverse maps, quadrature, periodicity) -- never from oracle/."""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "encode_c0.txt")


# ---------------------------------------------------------------- tri
@pytest.mark.parametrize("x,want", [(0.0, 1.0), (1.0, -1.0), (0.5, 0.0), (-0.5, 0.0), (3.0, -1.0),
                                    (2.0, 1.0), (0.25, 0.5), (1.75, 0.5), (-1.0, -1.0)])
def test_tri_values(orc, x, want):
    # tri(x) := 2|x mod 2 - 1| - 1; S:L36-38 examples
    assert orc.tri(x) == pytest.approx(want, abs=1e-15)


def test_tri_periodic_and_bounded(orc):
    rng = np.random.default_rng(0)
    for x in rng.uniform(-50, 50, 200):
        assert orc.tri(x) == pytest.approx(orc.tri(x + 2.0), abs=1e-12)
        assert -1.0 <= orc.tri(x) <= 1.0
        # triangle wave = (2/pi) arcsin(cos(pi x)): an independent closed form of
        # the same 2-periodic wave with tri(0)=1
        assert orc.tri(x) == pytest.approx(2 / math.pi * math.asin(math.cos(math.pi * x)), abs=1e-9)


# ---------------------------------------------------------------- quartic
@pytest.mark.parametrize("x,want", [(0.0, 0.9375), (0.5, 0.52734375), (-0.5, 0.52734375), (1.0, 0.0),
                                    (-1.0, 0.0), (1.5, 0.0), (-3.0, 0.0)])
def test_quartic_values(orc, x, want):
    # quartic(x) = 15/16 (1-x^2)^2; 15/16*(3/4)^2 = 0.52734375
    assert orc.quartic(x) == want


def test_quartic_integral_and_symmetry(orc):
    # even, non-negative, compact support, integral over [-1,1] equals 1
    xs = np.linspace(-1.0, 1.0, 20001)
    ys = np.array([orc.quartic(x) for x in xs])
    h = xs[1] - xs[0]
    simpson = h / 3 * (ys[0] + ys[-1] + 4 * ys[1:-1:2].sum() + 2 * ys[2:-1:2].sum())
    assert simpson == pytest.approx(1.0, abs=1e-9)
    assert np.all(ys >= 0)
    assert all(orc.quartic(x) == orc.quartic(-x) for x in xs[::97])


# ---------------------------------------------------------------- one-blob
@pytest.mark.parametrize("s,want", [(0.125, [0.9375, 0, 0, 0]), (0.375, [0, 0.9375, 0, 0]),
                                    (0.25, [0.52734375, 0.52734375, 0, 0]), (0.0, [0.52734375, 0, 0, 0]),
                                    (1.0, [0, 0, 0, 0.52734375]), (0.875, [0, 0, 0, 0.9375]),
                                    (-0.3, [0.52734375, 0, 0, 0]), (7.0, [0, 0, 0, 0.52734375])])
def test_one_blob_values(orc, s, want):
    # S:L54-56 worked examples; centres (i+1/2)/4, width 1/4, clamp (reading R6)
    np.testing.assert_array_equal(orc.one_blob(s, 4), np.array(want, np.float64))


def test_one_blob_partition_shape(orc):
    # at most two active kernels for any s, adjacent; total mass between Q(.5)*2 and Q(0)
    for s in np.linspace(0, 1, 1001):
        ob = orc.one_blob(s, 4)
        nz = np.nonzero(ob > 0)[0]
        assert len(nz) <= 2
        if len(nz) == 2:
            assert nz[1] == nz[0] + 1
        active = int(np.clip(np.floor(4 * s), 0, 3))  # bin containing s
        assert ob[active] > 0 or s in (0.0, 1.0)


# ---------------------------------------------------------------- frequency
def test_freq_examples(orc):
    np.testing.assert_array_equal(orc.freq(0.0), np.ones(12))
    assert orc.freq(0.5)[0] == 0.0
    assert orc.freq(0.25)[1] == 0.0
    # entry d is tri(2^d v): at v = 2^-(d+1) entry d is tri(0.5) = 0
    for d in range(12):
        assert orc.freq(2.0 ** -(d + 1))[d] == 0.0


def test_freq_resolution(orc):
    # a change of 2^-11 in v changes at least one of the 12 entries
    rng = np.random.default_rng(1)
    for v in rng.uniform(0, 1 - 2 ** -11, 300):
        assert np.any(orc.freq(v) != orc.freq(v + 2 ** -11))


# ---------------------------------------------------------------- sph
@pytest.mark.parametrize("u,want", [((0, 0, 1), (0, 0.5)), ((0, 0, -1), (1, 0.5)), ((1, 0, 0), (0.5, 0.5)),
                                    ((0, 1, 0), (0.5, 0.75)), ((0, -1, 0), (0.5, 0.25)),
                                    ((0, 0, 5), (0, 0.5)), ((-1, 1e-30, 0), (0.5, 1.0))])
def test_sph_values(orc, u, want):
    # S:L72-74 + reading R7 (atan2 signed-zero semantics, non-unit renormalised)
    np.testing.assert_allclose(orc.sph(u), want, atol=1e-15)


def test_sph_inverse_map(orc):
    # independent check: spherical -> Cartesian reconstruction recovers u/|u|
    rng = np.random.default_rng(2)
    for u in rng.standard_normal((200, 3)) * rng.uniform(0.1, 10, (200, 1)):
        th, ph = orc.sph(u)
        t, p = th * math.pi, ph * 2 * math.pi - math.pi
        rec = np.array([math.sin(t) * math.cos(p), math.sin(t) * math.sin(p), math.cos(t)])
        np.testing.assert_allclose(rec, u / np.linalg.norm(u), atol=1e-12)
        assert 0 <= th <= 1 and 0 <= ph <= 1


def test_sph_zero_vector_is_z(orc):
    np.testing.assert_allclose(orc.sph([0, 0, 0]), (0, 0.5))


# ---------------------------------------------------------------- position normalisation
def test_normalize_pos_fp32(orc):
    # reading R3: v = fp32(fp32(p - lo) * fp32(1/(hi-lo)))
    p, lo, hi = np.float32(3.7), np.float32(-1.25), np.float32(6.5)
    inv = np.float32(1) / (hi - lo)
    want = np.float32((p - lo) * inv)
    assert orc.normalize_pos(float(p), float(lo), float(hi)) == float(want)
    assert orc.normalize_pos(0.3, 0.0, 1.0) == float(np.float32(0.3))


# ---------------------------------------------------------------- encode
def _golden():
    rec, vals = None, {}
    for line in open(GOLDEN):
        if line.startswith("# record:"):
            rec = np.array([float(x) for x in line.split(":")[1].split()], np.float32)
        elif line.strip() and not line.startswith("#"):
            i, v = line.split()
            vals[int(i)] = float(v)
    return rec, np.array([vals[i] for i in range(64)])


def test_encode_golden_c0(orc):
    rec, want = _golden()
    got = orc.encode(rec)[0]
    np.testing.assert_allclose(got, want, atol=1e-7, rtol=0)


def test_encode_structure(orc):
    import nrc_inputs
    recs = nrc_inputs.records(500, seed=11)
    E = orc.encode(recs)
    assert E.shape == (500, 64)
    np.testing.assert_array_equal(E[:, 62:], 1.0)
    assert np.all(np.abs(E[:, :36]) <= 1.0)
    assert np.all((E[:, 36:56] >= 0) & (E[:, 36:56] <= 15 / 16))
    np.testing.assert_array_equal(E[:, 56:59], recs[:, 10:13].astype(np.float64))
    np.testing.assert_array_equal(E[:, 59:62], recs[:, 13:16].astype(np.float64))
    # each one-blob group has at least one active kernel
    for g in range(36, 56, 4):
        assert np.all(E[:, g:g + 4].max(axis=1) > 0)


def test_encode_r0_and_alpha_locality(orc):
    import nrc_inputs
    rec = nrc_inputs.records(1, seed=5)[0].copy()
    rec[9] = 0.0
    e0 = orc.encode(rec)[0]
    np.testing.assert_array_equal(e0[52:56], orc.one_blob(0.0))
    rec2 = rec.copy()
    rec2[10:13] += np.float32(0.125)
    e2 = orc.encode(rec2)[0]
    diff = np.nonzero(e0 != e2)[0]
    assert set(diff.tolist()) == {56, 57, 58}
    rec3 = rec.copy()
    rec3[13:16] *= np.float32(0.5)
    assert set(np.nonzero(orc.encode(rec3)[0] != e0)[0].tolist()) <= {59, 60, 61}


def test_encode_aabb(orc):
    # shifting position and AABB together leaves the encoding unchanged when exact in fp32
    import nrc_inputs
    rec = nrc_inputs.records(1, seed=6)[0].copy()
    rec[0:3] = [0.25, 0.5, 0.125]
    e_unit = orc.encode(rec)[0]
    rec2 = rec.copy()
    rec2[0:3] = rec[0:3] * 4 - 2  # exact in fp32
    e_big = orc.encode(rec2, (-2, -2, -2), (2, 2, 2))[0]
    np.testing.assert_array_equal(e_unit, e_big)
