"""Depth variants ("depth other than 5"; P:L694 fixes five
hidden layers): the query and the training with nh hidden layers at widths
32 / 64 / 128 against the depth-general fp64 oracle (oracle.query_d,
grad_batch_d, OracleCache(hidden_layers=nh)), with the parity definitions of
SURVEY 8(c) (tests/parity.py)."""
import numpy as np
import pytest
import torch

import nrc_inputs
from parity import TOL_GRAD, TOL_RADIANCE, offsets_d, per_matrix_err_d, radiance_err

pytestmark = pytest.mark.gpu

CASES = [(64, 1), (64, 2), (64, 3), (64, 7), (32, 8), (128, 3)]


@pytest.fixture(scope="module")
def nrc():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as p
    return p


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def make(nrc, hw, nh, **kw):
    return nrc.RadianceCache(nrc.Config(hidden_width=hw, n_hidden_layers=nh, **kw))


def _margin_records(orc, hw, nh, W, n, seed, tau=1e-3):
    """Records with every fp64 hidden pre-activation >= tau from the ReLU kink (R24)."""
    sizes = [(hw, 64)] + [(hw, hw)] * (nh - 1)
    mats, o = [], 0
    for r, c in sizes:
        mats.append(np.asarray(W[o:o + r * c], np.float64).reshape(r, c))
        o += r * c
    out, k = [], 0
    while sum(len(x) for x in out) < n:
        pool = nrc_inputs.records(4096, seed=seed + 7919 * k)
        h, m = orc.encode(pool), np.full(len(pool), np.inf)
        for A in mats:
            z = h @ A.T
            m = np.minimum(m, np.abs(z).min(1))
            h = np.maximum(z, 0)
        out.append(pool[m >= tau])
        k += 1
    return np.concatenate(out)[:n]


@pytest.mark.parametrize("hw,nh", CASES)
def test_depth_init_and_query(nrc, orc, hw, nh):
    c = make(nrc, hw, nh, seed=4)
    assert c.nparam == orc.param_count_d(hw, nh)
    np.testing.assert_array_equal(c.get_params("train"), orc.init_weights_d(hw, nh, 4))
    rng = np.random.default_rng(hw + nh)
    w = orc.init_weights_d(hw, nh, 11).astype(np.float64) * rng.uniform(1.0, 1.5)
    c.set_params(w.astype(np.float32), "ema")
    recs = nrc_inputs.records(3000, seed=40 + nh)
    q = c.query(dev(recs)).cpu().numpy()
    ref = orc.query_d(hw, nh, c.get_params("ema").astype(np.float64), recs)
    assert max(radiance_err(q, ref)) <= TOL_RADIANCE


@pytest.mark.parametrize("hw,nh", CASES)
@pytest.mark.parametrize("n", [129, 3000])
def test_depth_gradient_parity(nrc, orc, hw, nh, n):
    c = make(nrc, hw, nh)
    W = c.get_params("train").astype(np.float64)
    recs = _margin_records(orc, hw, nh, W, n, 700 + n) if n < 3000 else nrc_inputs.records(n, seed=700 + nh)
    tg = nrc_inputs.targets(recs, noise=0.3, seed=n)
    g, ls = c.train_backward(dev(recs), dev(tg))
    ref, l_ref, _ = orc.grad_batch_d(hw, nh, W, recs, tg)
    errs = per_matrix_err_d(g.cpu().numpy(), ref, offsets_d(hw, nh))
    assert max(errs) <= TOL_GRAD, errs
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)


@pytest.mark.parametrize("hw,nh", [(64, 2), (64, 7), (32, 8), (128, 3)])
def test_depth_train_frame_vs_oracle(nrc, orc, hw, nh):
    """Four LCG-shuffled steps of 2048 records: per-step losses within 1e-2 of
    the oracle's, the query through the trained EMA weights within 1e-2, and
    train_backward + train_apply equal to train_step bitwise."""
    n, s, l, seed = 8192, 4, 2048, 3
    recs, tg = nrc_inputs.train_frame(2, n=n, noise=0.3)
    c = make(nrc, hw, nh)
    oc = orc.OracleCache(W32=c.get_params("train"), hidden_width=hw, hidden_layers=nh)
    losses = c.train_frame(dev(recs), dev(tg), s, l, seed).cpu().numpy()
    pa, pc, pm = orc.lcg_params(n, seed)
    perm = orc.lcg_permute(n, pa, pc, pm).astype(np.int64)
    lref = [oc.train_step(recs[perm[j * l:(j + 1) * l]], tg[perm[j * l:(j + 1) * l]]) for j in range(s)]
    np.testing.assert_allclose(losses, lref, rtol=1e-2)
    # the query through the trained EMA weights (the two trajectories separate
    # slowly -- Adam's near-sign updates flip with the gradient's sign on tiny
    # entries, SURVEY 8(c) -- so the oracle evaluates the GPU's own weights)
    q = nrc_inputs.records(3000, seed=78)
    ref = orc.query_d(hw, nh, c.get_params("ema").astype(np.float64), q)
    assert max(radiance_err(c.query(dev(q)).cpu().numpy(), ref)) <= TOL_RADIANCE
    a, b = make(nrc, hw, nh), make(nrc, hw, nh)
    a.train_step(dev(recs[:5000]), dev(tg[:5000]))
    g, _ = b.train_backward(dev(recs[:5000]), dev(tg[:5000]))
    b.train_apply(g, 5000)
    np.testing.assert_array_equal(a.get_params("train"), b.get_params("train"))
    np.testing.assert_array_equal(a.get_params("ema"), b.get_params("ema"))


def test_depth5_is_the_default(nrc):
    recs, tg = nrc_inputs.train_frame(1, n=8192, noise=0.3)
    a, b = nrc.RadianceCache(), make(nrc, 64, 5)
    a.train_frame(dev(recs), dev(tg), 4, 2048, 1)
    b.train_frame(dev(recs), dev(tg), 4, 2048, 1)
    np.testing.assert_array_equal(a.get_params("train"), b.get_params("train"))


@pytest.mark.parametrize("hw,nh", [(64, 0), (64, 8), (32, 9), (128, 6)])
def test_depth_limits(nrc, hw, nh):
    with pytest.raises(nrc.NRCError):
        make(nrc, hw, nh)
