"""Pins for the oracle's network, loss, backward, Adam, EMA, LCG and init.

Expected values come from: SPEC worked examples,
closed forms (Adam's first step, geometric EMA sums, linear-chain products),
central finite differences (the backward pass), and brute force (LCG
bijection).  Cites: architecture P:L692-698, loss Eq.(5), Adam
P:L896-902, EMA Eq.(2), LCG P:L487-491."""
import math

import numpy as np
import pytest

NP = 20672
OFF = [0, 4096, 8192, 12288, 16384, 20480, 20672]


def rand_w(rng, scale=None):
    W = np.zeros(NP)
    for i in range(6):
        rows = 64 if i < 5 else 3
        s = scale or math.sqrt(6 / (64 + rows))
        W[OFF[i]:OFF[i + 1]] = rng.uniform(-s, s, rows * 64)
    return W


def rand_e(rng, n=1):
    e = rng.uniform(-1, 1, (n, 64))
    e[:, 62:] = 1.0
    return e


# ---------------------------------------------------------------- forward
def test_forward_zero_weights(orc):
    H, y = orc.forward(np.zeros(NP), rand_e(np.random.default_rng(0))[0])
    np.testing.assert_array_equal(y, 0)


def test_forward_constant_function_via_pad(orc):
    # row 0 of W0 reads only pad entry 62; hidden layers pass channel 0
    # through with weight 1 into output channel 0 -> (1,0,0) for every input
    W = np.zeros(NP)
    W[OFF[0] + 0 * 64 + 62] = 1.0
    for i in range(1, 5):
        W[OFF[i] + 0] = 1.0
    W[OFF[5] + 0] = 1.0
    rng = np.random.default_rng(1)
    for e in rand_e(rng, 20):
        _, y = orc.forward(W, e)
        np.testing.assert_array_equal(y, [1.0, 0.0, 0.0])


def test_forward_linear_chain(orc):
    # single nonzero path -> product of the weights along it
    W = np.zeros(NP)
    w = [0.5, 1.5, 2.0, 0.25, 3.0, -0.7]
    W[OFF[0] + 7 * 64 + 13] = w[0]      # h1[7] = w0 * e[13]
    W[OFF[1] + 2 * 64 + 7] = w[1]       # h2[2] = w1 * h1[7]
    W[OFF[2] + 40 * 64 + 2] = w[2]
    W[OFF[3] + 5 * 64 + 40] = w[3]
    W[OFF[4] + 63 * 64 + 5] = w[4]
    W[OFF[5] + 1 * 64 + 63] = w[5]      # y[1] = w5 * h5[63]
    e = np.zeros(64); e[13] = 0.8; e[62:] = 1
    _, y = orc.forward(W, e)
    assert y[1] == pytest.approx(0.8 * np.prod(w), rel=1e-15)
    assert y[0] == 0 and y[2] == 0
    e[13] = -0.8  # ReLU kills the negative path
    _, y = orc.forward(W, e)
    np.testing.assert_array_equal(y, 0)


def test_forward_positive_homogeneity_and_relu(orc):
    rng = np.random.default_rng(2)
    W = rand_w(rng)
    e = rand_e(rng)[0]
    H, y = orc.forward(W, e)
    W2 = W.copy(); W2[OFF[5]:] *= 3.5
    _, y2 = orc.forward(W2, e)
    np.testing.assert_allclose(y2, 3.5 * y, rtol=1e-14)
    assert np.all(H[1:] >= 0)
    np.testing.assert_array_equal(H[0], e)


def test_forward_matches_matrix_products(orc):
    # numpy matmul chain as an independent evaluation of the same definition
    rng = np.random.default_rng(3)
    W = rand_w(rng)
    e = rand_e(rng)[0]
    h = e
    for i in range(5):
        h = np.maximum(W[OFF[i]:OFF[i + 1]].reshape(64, 64) @ h, 0)
    y_np = W[OFF[5]:].reshape(3, 64) @ h
    _, y = orc.forward(W, e)
    np.testing.assert_allclose(y, y_np, rtol=1e-12, atol=1e-14)


def test_query_factorization_and_clamp(orc):
    import nrc_inputs
    rng = np.random.default_rng(4)
    W = rand_w(rng)
    recs = nrc_inputs.records(64, seed=3)
    q = orc.query(W, recs)
    assert np.all(q >= 0)
    raw = orc.query(W, recs, flags=0)
    fac = orc.query(W, recs, flags=orc.FACTORIZE)
    np.testing.assert_allclose(fac, raw * (recs[:, 10:13].astype(np.float64) + recs[:, 13:16]), rtol=1e-14)
    np.testing.assert_array_equal(q, np.maximum(fac, 0))
    zero = recs.copy(); zero[:, 10:16] = 0
    np.testing.assert_array_equal(orc.query(W, zero), 0)
    # batch-permutation equivariance
    perm = rng.permutation(64)
    np.testing.assert_array_equal(orc.query(W, recs[perm]), q[perm])


# ---------------------------------------------------------------- loss
def test_loss_spec_values(orc):
    l, d = orc.loss([2, 2, 2], [1, 1, 1], 0.01)  # lum=2 -> 1/4.01
    assert l == pytest.approx(0.2493765586, rel=1e-9)
    np.testing.assert_allclose(d, 2 * 1 / (3 * 4.01), rtol=1e-12)  # 0.1662510
    assert d[0] == pytest.approx(0.16625104, rel=1e-7)
    l, d = orc.loss([0, 0, 0], [1, 0, 0], 0.01)  # 1/(3*0.01)
    assert l == pytest.approx(33.3333333333, rel=1e-10)
    np.testing.assert_allclose(d, [-66.6666666667, 0, 0], rtol=1e-10)
    l, d = orc.loss([1, 1, 1], [1, 1, 1])
    assert l == 0 and np.all(d == 0)


def test_loss_luminance_weights(orc):
    # per-channel normalisation by the squared luminance of the prediction
    # (P:L894), Rec.709 weights (reading R8): lum of pure R/G/B predictions
    for c, wt in enumerate([0.2126, 0.7152, 0.0722]):
        p = np.zeros(3); p[c] = 1.0
        l, _ = orc.loss(p, np.zeros(3), 0.0)
        assert l == pytest.approx(1.0 / 3.0 / wt ** 2, rel=1e-12)


def test_loss_grad_fd_frozen(orc):
    # gradient == central FD of the loss with the denominator frozen
    rng = np.random.default_rng(5)
    for _ in range(50):
        p = rng.uniform(-1, 3, 3); t = rng.uniform(0, 2, 3)
        l, d = orc.loss(p, t)
        lam = 0.2126 * p[0] + 0.7152 * p[1] + 0.0722 * p[2]
        h = 1e-6
        for c in range(3):
            pp = p.copy(); pp[c] += h
            pm = p.copy(); pm[c] -= h
            fd = (orc.loss_frozen(pp, t, 0.01, lam) - orc.loss_frozen(pm, t, 0.01, lam)) / (2 * h)
            assert d[c] == pytest.approx(fd, rel=1e-6, abs=1e-9)


# ---------------------------------------------------------------- backward
def _batch_loss_frozen(orc, W, E, T, F, lams):
    tot = 0.0
    for e, t, f, lam in zip(E, T, F, lams):
        _, y = orc.forward(W, e)
        tot += orc.loss_frozen(y * f, t, 0.01, lam)
    return tot


def test_backward_finite_differences(orc):
    """every weight gradient matches central finite
    differences of the scalar loss (lambda frozen, fp64) within 1e-4 rel."""
    rng = np.random.default_rng(6)
    checked = 0
    for trial in range(12):
        W = rand_w(rng)
        n = 2
        E = rand_e(rng, n)
        T = rng.uniform(0, 2, (n, 3))
        F = rng.uniform(0.2, 1.0, (n, 3))
        G = np.zeros(NP)
        lams = []
        Hs = []
        for e, t, f in zip(E, T, F):
            H, y = orc.forward(W, e)
            _, dyhat = orc.loss(y * f, t)
            lams.append(0.2126 * y[0] * f[0] + 0.7152 * y[1] * f[1] + 0.0722 * y[2] * f[2])
            G += orc.backward(W, H, dyhat * f)
            Hs.append(H)
        pre = []  # pre-activations, to skip draws whose step crosses a ReLU kink
        for e in E:
            h = e; z = []
            for i in range(5):
                zz = W[OFF[i]:OFF[i + 1]].reshape(64, 64) @ h
                z.append(zz); h = np.maximum(zz, 0)
            pre.append(z)
        minabs = min(np.abs(np.concatenate(p)).min() for p in pre)
        h = 1e-6
        if minabs < 1e-4:  # a +-1e-6 weight step moves pre-activations by << 1e-4
            continue
        idx = rng.choice(NP, 20, replace=False)
        for j in idx:
            Wp = W.copy(); Wp[j] += h
            Wm = W.copy(); Wm[j] -= h
            fd = (_batch_loss_frozen(orc, Wp, E, T, F, lams) - _batch_loss_frozen(orc, Wm, E, T, F, lams)) / (2 * h)
            assert G[j] == pytest.approx(fd, rel=1e-4, abs=1e-8 * max(1, np.abs(G).max()))
            checked += 1
    assert checked >= 100


def test_backward_zero_and_outer_product(orc):
    rng = np.random.default_rng(7)
    W = rand_w(rng)
    e = rand_e(rng)[0]
    H, _ = orc.forward(W, e)
    np.testing.assert_array_equal(orc.backward(W, H, np.zeros(3)), 0)
    # G5 = dy h5^T exactly (1-layer analytic outer product)
    dy = np.array([0.3, -1.2, 2.0])
    G = orc.backward(W, H, dy)
    np.testing.assert_allclose(G[OFF[5]:].reshape(3, 64), np.outer(dy, H[5]), rtol=1e-15)
    # G4 = (W5^T dy * 1[h5>0]) h4^T
    g5 = (W[OFF[5]:].reshape(3, 64).T @ dy) * (H[5] > 0)
    np.testing.assert_allclose(G[OFF[4]:OFF[5]].reshape(64, 64), np.outer(g5, H[4]), rtol=1e-12, atol=1e-15)


def test_grad_batch_masks_nonfinite_targets(orc):
    import nrc_inputs
    recs = nrc_inputs.records(16, seed=8)
    tg = nrc_inputs.targets(recs)
    W = rand_w(np.random.default_rng(8))
    G0, l0, b0 = orc.grad_batch(W, recs[:15], tg[:15])
    tg2 = tg.copy(); tg2[15] = [np.nan, 1, 1]
    G1, l1, b1 = orc.grad_batch(W, recs, tg2)
    assert b0 == 0 and b1 == 1
    np.testing.assert_allclose(G1, G0, rtol=1e-12, atol=1e-300)
    assert l1 == pytest.approx(l0, rel=1e-12)


# ---------------------------------------------------------------- Adam
def test_adam_zero_gradient(orc):
    w = np.linspace(-1, 1, 10); w0 = w.copy()
    m = np.zeros(10); v = np.zeros(10)
    orc.adam(w, m, v, np.zeros(10), 1)
    np.testing.assert_array_equal(w, w0)


def test_adam_first_step_closed_form(orc):
    # first step: m_hat = g, v_hat = g^2 -> |dw| = lr |g| / (|g| + eps)
    g = np.array([3e-5, -2.0, 1e-9, 0.5])
    w = np.zeros(4); m = np.zeros(4); v = np.zeros(4)
    orc.adam(w, m, v, g, 1, lr=1e-2, eps=1e-8)
    want = -1e-2 * g / (np.abs(g) + 1e-8)
    np.testing.assert_allclose(w, want, rtol=1e-12)
    assert abs(w[0]) == pytest.approx(0.0099966678, rel=1e-7)


def test_adam_monotone_and_nonfinite(orc):
    w = np.zeros(3); m = np.zeros(3); v = np.zeros(3)
    g = np.array([0.1, -0.2, np.inf])
    bad = orc.adam(w, m, v, g, 1)
    w1 = w.copy()
    bad += orc.adam(w, m, v, g, 2)
    assert bad == 2 and w1[2] == 0 and w[2] == 0  # non-finite zeroed and counted
    assert w[0] < w1[0] < 0 and w[1] > w1[1] > 0
    # second step closed form with identical gradients
    b1, b2 = 0.9, 0.99
    mh = ((1 - b1) * b1 * 0.1 + (1 - b1) * 0.1) / (1 - b1 ** 2)
    vh = ((1 - b2) * b2 * 0.01 + (1 - b2) * 0.01) / (1 - b2 ** 2)
    assert w[0] - w1[0] == pytest.approx(-1e-2 * mh / (math.sqrt(vh) + 1e-8), rel=1e-12)


# ---------------------------------------------------------------- EMA
def test_ema_t1_and_alpha0(orc):
    wb = np.full(5, 7.0); w = np.arange(5.0)
    orc.ema(wb, w, 1, 0.99)
    np.testing.assert_allclose(wb, w, rtol=1e-15)
    wb = np.full(5, 7.0)
    orc.ema(wb, w, 9, 0.0)
    np.testing.assert_array_equal(wb, w)


def test_ema_constant_stream(orc):
    C = np.array([1.5, -0.25, 3.0])
    wb = np.zeros(3)
    for t in range(1, 10001):
        orc.ema(wb, C, t, 0.99)
    np.testing.assert_allclose(wb, C, rtol=1e-12)


def test_ema_is_weighted_average(orc):
    # closed form: Wbar_t = sum_s (1-a) a^(t-s) W_s / (1 - a^t)
    rng = np.random.default_rng(9)
    a = 0.9
    Ws = rng.standard_normal((30, 4))
    wb = np.zeros(4)
    for t in range(1, 31):
        orc.ema(wb, Ws[t - 1], t, a)
        want = sum((1 - a) * a ** (t - s) * Ws[s - 1] for s in range(1, t + 1)) / (1 - a ** t)
        np.testing.assert_allclose(wb, want, rtol=1e-12)


def test_ema_linearity(orc):
    rng = np.random.default_rng(10)
    A = rng.standard_normal((20, 3)); B = rng.standard_normal((20, 3))
    ea, eb, ec = np.zeros(3), np.zeros(3), np.zeros(3)
    for t in range(1, 21):
        orc.ema(ea, A[t - 1], t); orc.ema(eb, B[t - 1], t); orc.ema(ec, 2 * A[t - 1] - 3 * B[t - 1], t)
    np.testing.assert_allclose(ec, 2 * ea - 3 * eb, rtol=1e-12, atol=1e-14)


def test_ema_printed_form_negative_control(orc):
    # Eq.(2) as printed does not preserve a constant: 0.5124 C at t=2
    wb = np.zeros(1); C = np.ones(1)
    orc.ema(wb, C, 1, 0.99, printed_form=True)
    orc.ema(wb, C, 2, 0.99, printed_form=True)
    # t=2: (0.01/0.0199) + 0.99*0.01*1 = 0.50251... + 0.0099 = 0.51241...
    assert wb[0] == pytest.approx(0.01 / (1 - 0.99 ** 2) + 0.99 * 0.01, rel=1e-12)
    assert wb[0] == pytest.approx(0.5124, abs=1e-4)


# ---------------------------------------------------------------- LCG
def test_lcg_spec_example(orc):
    np.testing.assert_array_equal(orc.lcg_permute(4, 5, 3, 4), [3, 0, 1, 2])
    np.testing.assert_array_equal(orc.lcg_permute(1, 1, 1, 1), [0])


@pytest.mark.parametrize("n", [1, 2, 3, 5, 1000, 16384, 65536, 65537, 2 ** 20])
def test_lcg_bijection(orc, n):
    for seed in (0, 1, 0xDEADBEEF):
        a, c, m = orc.lcg_params(n, seed)
        assert m >= n and m & (m - 1) == 0 and m < 2 * max(n, 1) + 1
        assert a % 4 == 1 and c % 2 == 1  # Hull-Dobell full period (R15)
        p = orc.lcg_permute(n, a, c, m)
        np.testing.assert_array_equal(np.sort(p), np.arange(n))


def test_lcg_power_of_two_is_affine(orc):
    # for n = 2^16 (the paper's 65,536) no cycle walking happens
    n = 65536
    a, c, m = orc.lcg_params(n, 42)
    i = np.arange(n, dtype=np.uint64)
    np.testing.assert_array_equal(orc.lcg_permute(n, a, c, m), (np.uint64(a) * i + np.uint64(c)) % np.uint64(m))


# ---------------------------------------------------------------- init
def test_init_glorot(orc):
    W = orc.init_weights(1)
    assert W.dtype == np.float32 and W.shape == (NP,)
    for i in range(6):
        rows = 64 if i < 5 else 3
        b = math.sqrt(6 / (64 + rows))
        Wi = W[OFF[i]:OFF[i + 1]].astype(np.float64)
        assert np.all(np.abs(Wi) <= b)
        # moments of U(-b, b): mean 0, variance b^2/3
        assert abs(Wi.mean()) < 4 * b / math.sqrt(3 * Wi.size)
        assert Wi.var() == pytest.approx(b * b / 3, rel=0.15 if i == 5 else 0.06)
    assert not np.array_equal(W, orc.init_weights(2))
    np.testing.assert_array_equal(W, orc.init_weights(1))
