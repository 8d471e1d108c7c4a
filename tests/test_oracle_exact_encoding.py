"""Pins of the exact encodings (
readings R21, R22): sin(pi 2^d v) at dyadic and 1/6 points, the Gaussian
one-blob's closed forms, and the shared layout with orc_encode."""
import math

import numpy as np
import pytest

import nrc_inputs


def test_freq_sin_closed_forms(orc):
    f = orc.freq_sin(0.25)  # sin(pi/4 2^d): sqrt2/2, 1, 0, 0, ...
    np.testing.assert_allclose(f[:2], [math.sqrt(0.5), 1.0], rtol=1e-15)
    np.testing.assert_allclose(f[2:], 0.0, atol=1e-12)
    g = orc.freq_sin(1.0 / 6.0)  # sin(pi/6) = 1/2, sin(pi/3), sin(2pi/3), sin(4pi/3) ...
    np.testing.assert_allclose(g[:4], [0.5, math.sqrt(3) / 2, math.sqrt(3) / 2, -math.sqrt(3) / 2], rtol=1e-12)
    np.testing.assert_array_equal(orc.freq_sin(0.0), 0.0)


def test_gauss_and_one_blob(orc):
    assert orc.gauss(0.0) == 1.0 / math.sqrt(2 * math.pi)
    assert abs(orc.gauss(1.0) - math.exp(-0.5) / math.sqrt(2 * math.pi)) < 1e-16
    assert orc.gauss(0.7) == orc.gauss(-0.7)
    # s at bin centre 2: peak at bin 2, g(1) at bins 1 and 3, g(2) at bin 0
    ob = orc.one_blob_gauss(2.5 / 4.0)
    np.testing.assert_allclose(ob, [orc.gauss(2.0), orc.gauss(1.0), orc.gauss(0.0), orc.gauss(1.0)], rtol=1e-15)
    # clamping to [0, 1] as for the quartic one-blob (R6)
    np.testing.assert_array_equal(orc.one_blob_gauss(-3.0), orc.one_blob_gauss(0.0))
    # Riemann sum of g over a fine grid of blob positions integrates to ~1 per bin
    xs = np.linspace(-8, 8, 16001)
    assert abs(sum(orc.gauss(x) for x in xs) * (xs[1] - xs[0]) - 1.0) < 1e-9


def test_encode_exact_layout(orc):
    recs = nrc_inputs.records(64, seed=3)
    e = orc.encode_exact(recs)
    cheap = orc.encode(recs)
    np.testing.assert_array_equal(e[:, 56:], cheap[:, 56:])  # alpha, beta, pads identical
    for a in range(3):
        v = recs[:, a].astype(np.float64)  # unit AABB: v = p
        for d in (0, 3, 11):
            np.testing.assert_allclose(e[:, 12 * a + d], np.sin(np.pi * v * 2.0 ** d), rtol=0, atol=1e-12)
    # one-blob entries lie in (0, 1/sqrt(2 pi)]
    assert np.all(e[:, 36:56] > 0) and np.all(e[:, 36:56] <= 1 / math.sqrt(2 * math.pi))


def test_grad_batch_exact_finite_differences(orc):
    """orc_grad_batch_exact (N4 training): the un-normalised batch gradient
    through the exact encodings matches central finite differences of the
    batch loss (lambda frozen) built from the pinned encode_exact,
    forward and loss_frozen, within 1e-4 relative."""
    import nrc_inputs
    rng = np.random.default_rng(91)
    NP, OFF = 20672, [0, 4096, 8192, 12288, 16384, 20480, 20672]
    checked = 0
    for trial in range(8):
        W = rng.normal(0, 1.5 / 8, NP)
        recs = nrc_inputs.records(2, seed=600 + trial)
        tg = nrc_inputs.targets(recs, noise=0.3, seed=trial)
        G, _, _ = orc.grad_batch(W, recs, tg, exact=True)
        E = orc.encode_exact(recs)
        F = (recs[:, 10:13] + recs[:, 13:16]).astype(np.float64)
        lams, minabs = [], np.inf
        for e, f in zip(E, F):
            _, y = orc.forward(W, e)
            lams.append(0.2126 * y[0] * f[0] + 0.7152 * y[1] * f[1] + 0.0722 * y[2] * f[2])
            h = e
            for i in range(5):
                z = W[OFF[i]:OFF[i + 1]].reshape(64, 64) @ h
                minabs = min(minabs, np.abs(z).min())
                h = np.maximum(z, 0)
        if minabs < 1e-4:
            continue

        def L(Wx):
            return sum(orc.loss_frozen(orc.forward(Wx, e)[1] * f, t, 0.01, lam)
                       for e, f, t, lam in zip(E, F, tg.astype(np.float64), lams))
        for j in rng.choice(NP, 16, replace=False):
            Wp = W.copy(); Wp[j] += 1e-6
            Wm = W.copy(); Wm[j] -= 1e-6
            fd = (L(Wp) - L(Wm)) / 2e-6
            assert G[j] == pytest.approx(fd, rel=1e-4, abs=1e-8 * max(1, np.abs(G).max()))
            checked += 1
    assert checked >= 64
