"""Pins of the oracle's width-ablation TRAINING functions (BASELINE.json
configs[3] "32/64/128-neuron hidden layers at 1080p query+train").

orc_backward_w / orc_grad_batch_w / orc_train_step_w are pinned by
  * exact zero-padding embeddings against the separately pinned width-64
    functions (a width-32 net padded into width 64 and a width-64 net padded
    into width 128 have identical gradients on the embedded entries and
    exactly zero gradients on the padding: the padded units are dead, and
    ReLU'(0) = 0, reading R17), and
  * central finite differences of the batch loss (lambda frozen, fp64) at
    hw = 32 and hw = 128, so a dropped term, a wrong
    index or a transposed operand that the embedding would not see (for
    example one that only bites above column 64) fails a pin."""
import numpy as np
import pytest

import nrc_inputs

from test_oracle_width import _embed, _mats


def _embed_mask(hw_small, hw_big):
    """True on the entries of the width-hw_big vector that come from the small net."""
    return _embed(hw_small, np.ones(64 * hw_small + 4 * hw_small ** 2 + 3 * hw_small), hw_big) != 0


@pytest.mark.parametrize("small,big", [(32, 64), (64, 128)])
def test_grad_embedding_matches_pinned_width64(orc, small, big):
    rng = np.random.default_rng(11 + small)
    recs = nrc_inputs.records(200, seed=51)
    tg = nrc_inputs.targets(recs, noise=0.3, seed=52)
    Ws = rng.normal(0, 1.5 / np.sqrt(64), orc.param_count_w(small))
    Wb = _embed(small, Ws, big)
    if small == 64:
        Gs, ls, _ = orc.grad_batch(Ws, recs, tg)  # the pinned width-64 oracle
    else:
        Gs, ls, _ = orc.grad_batch_w(small, Ws, recs, tg)
    Gb, lb, _ = orc.grad_batch_w(big, Wb, recs, tg)
    mask = _embed_mask(small, big)
    np.testing.assert_array_equal(Gb[mask], Gs)
    np.testing.assert_array_equal(Gb[~mask], 0.0)
    assert lb == ls
    if big == 64:  # and the width-32 net embedded into the width-64 oracle itself
        G64, l64, _ = orc.grad_batch(Wb, recs, tg)
        np.testing.assert_array_equal(G64, Gb)
        assert l64 == lb


def _batch_loss_frozen(orc, hw, W, E, T, F, lams):
    tot = 0.0
    for e, t, f, lam in zip(E, T, F, lams):
        y = orc.forward_w(hw, W, e)
        tot += orc.loss_frozen(y * f, t, 0.01, lam)
    return tot


@pytest.mark.parametrize("hw", [32, 128])
def test_backward_w_finite_differences(orc, hw):
    """Every sampled weight gradient matches central finite differences of the
    loss with the luminance frozen within 1e-4 relative."""
    rng = np.random.default_rng(60 + hw)
    P = orc.param_count_w(hw)
    checked = 0
    for trial in range(10):
        W = rng.normal(0, 1.5 / np.sqrt(64), P)
        n = 2
        E = rng.uniform(-1, 1, (n, 64)); E[:, 62:] = 1.0
        T = rng.uniform(0, 2, (n, 3))
        F = rng.uniform(0.2, 1.0, (n, 3))
        G = np.zeros(P)
        lams = []
        for e, t, f in zip(E, T, F):
            H, y = orc.forward_stash_w(hw, W, e)
            _, dyhat = orc.loss(y * f, t)
            lams.append(0.2126 * y[0] * f[0] + 0.7152 * y[1] * f[1] + 0.0722 * y[2] * f[2])
            G += orc.backward_w(hw, W, H, dyhat * f)
        ms = _mats(hw, W)
        minabs = np.inf
        for e in E:  # skip draws where a +-h step could cross a ReLU kink
            h = e
            for i in range(5):
                z = ms[i] @ h
                minabs = min(minabs, np.abs(z).min())
                h = np.maximum(z, 0)
        step = 1e-6
        if minabs < 1e-4:
            continue
        # sample every matrix, including columns >= 64 at hw = 128
        offs = np.cumsum([0] + [m.size for m in ms])
        idx = np.concatenate([rng.choice(np.arange(offs[i], offs[i + 1]), 4, replace=False) for i in range(6)])
        for j in idx:
            Wp = W.copy(); Wp[j] += step
            Wm = W.copy(); Wm[j] -= step
            fd = (_batch_loss_frozen(orc, hw, Wp, E, T, F, lams) -
                  _batch_loss_frozen(orc, hw, Wm, E, T, F, lams)) / (2 * step)
            assert G[j] == pytest.approx(fd, rel=1e-4, abs=1e-8 * max(1, np.abs(G).max()))
            checked += 1
    assert checked >= 100


@pytest.mark.parametrize("hw", [32, 128])
def test_forward_stash_w_matches_forward_w(orc, hw):
    rng = np.random.default_rng(70 + hw)
    W = rng.normal(0, 1.5 / np.sqrt(64), orc.param_count_w(hw))
    e = rng.uniform(-1, 1, 64)
    H, y = orc.forward_stash_w(hw, W, e)
    np.testing.assert_array_equal(y, orc.forward_w(hw, W, e))
    np.testing.assert_array_equal(H[:64], e)
    ms = _mats(hw, W)
    h1 = np.maximum(ms[0] @ e, 0)
    np.testing.assert_allclose(H[64:64 + hw], h1, rtol=1e-13, atol=1e-15)


def test_train_step_w_embedding(orc):
    """Two optimisation steps (Adam + EMA) of a width-32 net equal those of the
    same net embedded into the pinned width-64 OracleCache; the padding stays 0."""
    W32 = orc.init_weights_w(32, 5)
    a = orc.OracleCache(W32=W32, hidden_width=32)
    b = orc.OracleCache(W32=_embed(32, W32.astype(np.float64), 64).astype(np.float32))
    mask = _embed_mask(32, 64)
    for f in range(2):
        recs, tg = nrc_inputs.train_frame(f, n=256, noise=0.3)
        la = a.train_step(recs, tg)
        lb = b.train_step(recs, tg)
        assert la == lb
        np.testing.assert_array_equal(b.w[mask], a.w)
        np.testing.assert_array_equal(b.w[~mask], 0.0)
        np.testing.assert_array_equal(b.wbar[mask], a.wbar)
    recs = nrc_inputs.records(64, seed=9)
    np.testing.assert_array_equal(a.query(recs), b.query(recs))
