"""Pins of the oracle's depth variants ("depth other than 5";
P:L694 fixes five hidden layers, the variant keeps width, input, ReLU and the
linear 3-output layer).

  * nh = 5 reproduces the separately pinned width functions bit for bit;
  * a net extended by identity hidden layers computes the same function
    (ReLU(I h) = h for h >= 0) and the same gradients on its original layers
    (the identity layers' masks equal the next layer's), which pins the
    shallower depths against the pinned five-layer oracle (a 2- or 3-layer
    net extended to 5) and the deeper ones on that subspace (a 5-layer net
    extended to 6 or 7);
  * central finite differences with general weights at nh = 2 and nh = 7 pin
    the parts the identity extension cannot see."""
import numpy as np
import pytest

import nrc_inputs


def _split(hw, nh, W):
    shapes = [(hw, 64)] + [(hw, hw)] * (nh - 1) + [(3, hw)]
    out, o = [], 0
    for r, c in shapes:
        out.append(np.asarray(W[o:o + r * c]).reshape(r, c))
        o += r * c
    assert o == W.size
    return out


def _extend(hw, nh, W, k):
    """Insert k identity hidden layers before the output layer."""
    ms = _split(hw, nh, W)
    return np.concatenate([m.reshape(-1) for m in ms[:-1]] + [np.eye(hw).reshape(-1)] * k + [ms[-1].reshape(-1)])


def _ext_mask(hw, nh, k):
    """True on the entries of the extended vector that belong to the original layers."""
    ones = np.ones(64 * hw + (nh - 1) * hw * hw + 3 * hw)
    ms = _split(hw, nh, ones)
    return np.concatenate([m.reshape(-1) for m in ms[:-1]] + [np.zeros(hw * hw)] * k + [ms[-1].reshape(-1)]) != 0


@pytest.mark.parametrize("nh", [1, 2, 3, 5, 7])
def test_param_count(orc, nh):
    assert orc.param_count_d(64, nh) == 64 * 64 + (nh - 1) * 4096 + 3 * 64
    assert orc.param_count_d(64, 5) == orc.NPARAM


@pytest.mark.parametrize("hw", [32, 64, 128])
def test_depth5_equals_width_functions(orc, hw):
    rng = np.random.default_rng(hw)
    W = rng.normal(0, 1.5 / 8, orc.param_count_w(hw))
    recs = nrc_inputs.records(200, seed=71)
    tg = nrc_inputs.targets(recs, noise=0.3, seed=72)
    np.testing.assert_array_equal(orc.query_d(hw, 5, W, recs), orc.query_w(hw, W, recs))
    Gd, ld, _ = orc.grad_batch_d(hw, 5, W, recs, tg)
    Gw, lw, _ = orc.grad_batch_w(hw, W, recs, tg)
    np.testing.assert_array_equal(Gd, Gw)
    assert ld == lw
    np.testing.assert_array_equal(orc.init_weights_d(hw, 5, 3), orc.init_weights_w(hw, 3))


@pytest.mark.parametrize("nh,k", [(2, 3), (3, 2), (4, 1), (5, 1), (5, 2)])
def test_identity_extension(orc, nh, k):
    """The nh-layer net and its (nh+k)-layer identity extension agree on the
    query and on the gradients of the original layers; the extension to five
    layers is checked against the pinned width-64 oracle."""
    rng = np.random.default_rng(10 * nh + k)
    W = rng.normal(0, 1.5 / 8, orc.param_count_d(64, nh))
    We = _extend(64, nh, W, k)
    recs = nrc_inputs.records(150, seed=73 + nh)
    tg = nrc_inputs.targets(recs, noise=0.3, seed=74)
    q = orc.query_d(64, nh, W, recs)
    np.testing.assert_array_equal(orc.query_d(64, nh + k, We, recs), q)
    G, l, _ = orc.grad_batch_d(64, nh, W, recs, tg)
    Ge, le, _ = orc.grad_batch_d(64, nh + k, We, recs, tg)
    np.testing.assert_array_equal(Ge[_ext_mask(64, nh, k)], G)
    assert le == l
    if nh + k == 5:  # the pinned five-layer oracle
        np.testing.assert_array_equal(orc.query(We, recs), q)
        G5, l5, _ = orc.grad_batch(We, recs, tg)
        np.testing.assert_array_equal(G5[_ext_mask(64, nh, k)], G)


@pytest.mark.parametrize("nh", [2, 7])
def test_backward_d_finite_differences(orc, nh):
    rng = np.random.default_rng(80 + nh)
    P = orc.param_count_d(64, nh)
    checked = 0
    for trial in range(10):
        W = rng.normal(0, 1.5 / 8, P)
        E = rng.uniform(-1, 1, (2, 64)); E[:, 62:] = 1.0
        T = rng.uniform(0, 2, (2, 3))
        F = rng.uniform(0.2, 1.0, (2, 3))
        G = np.zeros(P)
        lams = []
        for e, t, f in zip(E, T, F):
            H, y = orc.forward_stash_d(64, nh, W, e)
            _, dyhat = orc.loss(y * f, t)
            lams.append(0.2126 * y[0] * f[0] + 0.7152 * y[1] * f[1] + 0.0722 * y[2] * f[2])
            G += orc.backward_d(64, nh, W, H, dyhat * f)
        ms = _split(64, nh, W)
        minabs = np.inf
        for e in E:
            h = e
            for A in ms[:-1]:
                z = A @ h
                minabs = min(minabs, np.abs(z).min())
                h = np.maximum(z, 0)
        if minabs < 1e-4:
            continue

        def L(Wx):
            return sum(orc.loss_frozen(orc.forward_stash_d(64, nh, Wx, e)[1] * f, t, 0.01, lam)
                       for e, t, f, lam in zip(E, T, F, lams))
        offs = np.cumsum([0] + [m.size for m in ms])
        idx = np.concatenate([rng.choice(np.arange(offs[i], offs[i + 1]), 3, replace=False) for i in range(nh + 1)])
        for j in idx:
            Wp = W.copy(); Wp[j] += 1e-6
            Wm = W.copy(); Wm[j] -= 1e-6
            fd = (L(Wp) - L(Wm)) / 2e-6
            assert G[j] == pytest.approx(fd, rel=1e-4, abs=1e-8 * max(1, np.abs(G).max()))
            checked += 1
    assert checked >= 40


def test_init_weights_d_glorot(orc):
    W = orc.init_weights_d(64, 3, 9)
    ms = _split(64, 3, W)
    for i, m in enumerate(ms):
        fan_in, fan_out = m.shape[1], m.shape[0]
        b = np.sqrt(6.0 / (fan_in + fan_out))
        assert np.all(np.abs(m) <= b)
        assert abs(np.mean(m)) < 0.05 * b and abs(np.var(m) - b * b / 3) < 0.1 * b * b / 3
