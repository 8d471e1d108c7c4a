"""Width ablation, training (BASELINE.json configs[3] "32/64/128-neuron hidden
layers at 1080p query+train"): the width-generic training kernels
(nrc_train_w.cuh) at hidden width 32, 128 and 64 (the default training path
at every width) against the width-general fp64 oracle
(oracle.grad_batch_w / OracleCache(hidden_width=hw)), with the parity
definitions of SURVEY 8(c) (tests/parity.py)."""
import numpy as np
import pytest
import torch

import nrc_inputs
from parity import TOL_GRAD, TOL_PARAM, TOL_RADIANCE, offsets_w, per_matrix_err, post_adam_err, radiance_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nrc():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as p
    return p


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def make(nrc, hw, monkeypatch=None, **kw):
    if hw == "64g":  # the default training path at width 64
        return nrc.RadianceCache(nrc.Config(hidden_width=64, **kw)), 64
    return nrc.RadianceCache(nrc.Config(hidden_width=hw, **kw)), hw


WIDTHS = [32, 128, "64g"]


def _margin_records(orc, hw, W, n, seed, tau=1e-3):
    """n records whose fp64 hidden pre-activations all lie >= tau from the ReLU
    kink (reading R24): there fp16 rounding cannot flip a ReLU decision, so a
    small batch's gradient measures the kernel's arithmetic rather than a
    rounding-triggered discontinuity (test-side selection with the oracle's
    encoding and plain fp64 matrix products)."""
    shapes = [(hw, 64)] + [(hw, hw)] * 4
    mats, o = [], 0
    for r, c in shapes:
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


@pytest.mark.parametrize("hw", WIDTHS)
@pytest.mark.parametrize("n", [1, 129, 256])
def test_width_gradient_parity_margin(nrc, orc, monkeypatch, hw, n):
    """Un-normalised gradient sums (train_backward) per matrix within 3e-2 of
    the oracle, loss sum within 1e-2, on records with a ReLU margin (R24); 1 and
    129 rows exercise the ragged tile."""
    c, w = make(nrc, hw, monkeypatch)
    W = c.get_params("train").astype(np.float64)
    recs = _margin_records(orc, w, W, n, 500 + n)
    tg = nrc_inputs.targets(recs, noise=0.3, seed=n)
    g_gpu, ls = c.train_backward(dev(recs), dev(tg))
    g_ref, l_ref, _ = orc.grad_batch_w(w, W, recs, tg)
    errs = per_matrix_err(g_gpu.cpu().numpy(), g_ref, offsets_w(w))
    assert max(errs) <= TOL_GRAD, errs
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)


@pytest.mark.parametrize("hw", WIDTHS)
@pytest.mark.parametrize("n", [3000, 16384])
def test_width_gradient_parity(nrc, orc, monkeypatch, hw, n):
    """Unselected batches of >= 3000 records (16,384 = one training batch of
    the frame): per matrix within 3e-2, loss within 1e-2."""
    c, w = make(nrc, hw, monkeypatch)
    recs = nrc_inputs.records(n, seed=500 + n)
    tg = nrc_inputs.targets(recs, noise=0.3, seed=n)
    g_gpu, ls = c.train_backward(dev(recs), dev(tg))
    g_ref, l_ref, _ = orc.grad_batch_w(w, c.get_params("train").astype(np.float64), recs, tg)
    errs = per_matrix_err(g_gpu.cpu().numpy(), g_ref, offsets_w(w))
    assert max(errs) <= TOL_GRAD, errs
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)


@pytest.mark.parametrize("hw", WIDTHS)
def test_width_train_step_parity_c1(nrc, orc, monkeypatch, hw):
    """C1 at width hw: loss, post-Adam W and W-bar (sign-agreeing entries), and
    the query through the trained EMA weights."""
    c, w = make(nrc, hw, monkeypatch)
    recs, tg = nrc_inputs.train_frame(0, n=256, noise=0.3)
    oc = orc.OracleCache(W32=c.get_params("train"), hidden_width=w)
    g_gpu, _ = c.train_backward(dev(recs), dev(tg))
    g_gpu = g_gpu.cpu().numpy() / 256.0
    loss = c.train_step(dev(recs), dev(tg)).item()
    l_ref, G_ref = oc.train_step(recs, tg, return_grad=True)
    assert loss == pytest.approx(l_ref, rel=1e-2)
    off = offsets_w(w)
    errs, flip_frac, worst = post_adam_err(c.get_params("train"), oc.w, g_gpu, G_ref, off)
    assert max(errs) <= TOL_PARAM, errs
    assert flip_frac <= 0.01 and worst <= 3e-2, (flip_frac, worst)
    e_errs, _, _ = post_adam_err(c.get_params("ema"), oc.wbar, g_gpu, G_ref, off)
    assert max(e_errs) <= TOL_PARAM
    assert c.stats()["step"] == 1
    q = nrc_inputs.records(2000, seed=77)
    out = c.query(dev(q)).cpu().numpy()
    ref = orc.query_w(w, c.get_params("ema").astype(np.float64), q)
    assert max(radiance_err(out, ref)) <= TOL_RADIANCE


@pytest.mark.parametrize("hw,n", [(32, 40_000), (128, 20_000)])
def test_width_multi_tile_ctas(nrc, orc, hw, n):
    """More tiles than CTAs (313 / 157 tiles on <= 148 CTAs): the per-CTA
    partial accumulates over its tiles (read-add-write of its own slot)."""
    c, w = make(nrc, hw)
    recs, tg = nrc_inputs.train_frame(8, n=n, noise=0.3)
    oc = orc.OracleCache(W32=c.get_params("train"), hidden_width=w)
    g_gpu, ls = c.train_backward(dev(recs), dev(tg))
    g_gpu = g_gpu.cpu().numpy()
    g_ref, l_ref, _ = orc.grad_batch_w(w, oc.w, recs, tg)
    assert max(per_matrix_err(g_gpu, g_ref, offsets_w(w))) <= TOL_GRAD
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)
    loss = c.train_step(dev(recs), dev(tg)).item()
    l1, G1 = oc.train_step(recs, tg, return_grad=True)
    assert loss == pytest.approx(l1, rel=1e-2)
    errs, flip_frac, worst = post_adam_err(c.get_params("train"), oc.w, g_gpu / n, G1, offsets_w(w))
    assert max(errs) <= TOL_PARAM, errs
    assert flip_frac <= 0.01 and worst <= 3e-2, (flip_frac, worst)


@pytest.mark.parametrize("hw", [32, 128])
def test_width_train_frame_equals_gathered_steps(nrc, orc, hw):
    """nrc_train_frame at width hw == s train steps on the LCG-gathered batches
    (bitwise: same kernels, same reduction order), losses included."""
    n, s, l, seed = 8192, 4, 2048, 11
    recs, tg = nrc_inputs.train_frame(5, n=n)
    a, _ = make(nrc, hw)
    b, _ = make(nrc, hw)
    losses = a.train_frame(dev(recs), dev(tg), s, l, seed).cpu().numpy()
    pa, pc, pm = orc.lcg_params(n, seed)
    perm = orc.lcg_permute(n, pa, pc, pm).astype(np.int64)
    lb = [b.train_step(dev(recs[perm[j * l:(j + 1) * l]]), dev(tg[perm[j * l:(j + 1) * l]])).item()
          for j in range(s)]
    np.testing.assert_array_equal(losses, np.array(lb, np.float32))
    np.testing.assert_array_equal(a.get_params("train"), b.get_params("train"))
    np.testing.assert_array_equal(a.get_params("ema"), b.get_params("ema"))
    assert a.stats()["step"] == s


@pytest.mark.parametrize("hw", [32, 128])
def test_width_train_frame_vs_oracle(nrc, orc, hw):
    """Four LCG-shuffled steps of 2048 records: per-step losses within 1e-2 of
    the oracle's on the same batches and the final query within 1e-2."""
    n, s, l, seed = 8192, 4, 2048, 3
    recs, tg = nrc_inputs.train_frame(2, n=n, noise=0.3)
    c, w = make(nrc, hw)
    oc = orc.OracleCache(W32=c.get_params("train"), hidden_width=w)
    losses = c.train_frame(dev(recs), dev(tg), s, l, seed).cpu().numpy()
    pa, pc, pm = orc.lcg_params(n, seed)
    perm = orc.lcg_permute(n, pa, pc, pm).astype(np.int64)
    lref = [oc.train_step(recs[perm[j * l:(j + 1) * l]], tg[perm[j * l:(j + 1) * l]]) for j in range(s)]
    np.testing.assert_allclose(losses, lref, rtol=1e-2)
    q = nrc_inputs.records(3000, seed=78)
    assert max(radiance_err(c.query(dev(q)).cpu().numpy(), oc.query(q))) <= TOL_RADIANCE


@pytest.mark.parametrize("hw", [32, 128])
def test_width_backward_apply_equals_step_and_determinism(nrc, hw):
    """train_backward + train_apply == train_step bitwise (the multi-GPU
    decomposition), and two identical runs agree bitwise."""
    recs, tg = nrc_inputs.train_frame(4, n=5000, noise=0.3)
    a, _ = make(nrc, hw)
    b, _ = make(nrc, hw)
    r2, _ = make(nrc, hw)
    a.train_step(dev(recs), dev(tg))
    r2.train_step(dev(recs), dev(tg))
    g, _ = b.train_backward(dev(recs), dev(tg))
    b.train_apply(g, recs.shape[0])
    np.testing.assert_array_equal(a.get_params("train"), b.get_params("train"))
    np.testing.assert_array_equal(a.get_params("ema"), b.get_params("ema"))
    np.testing.assert_array_equal(a.get_params("train"), r2.get_params("train"))


@pytest.mark.parametrize("hw", [32, 128])
def test_width_empty_and_nonfinite(nrc, hw):
    c, w = make(nrc, hw)
    recs, tg = nrc_inputs.train_frame(0, n=300)
    c.train_step(dev(recs[:0]), dev(tg[:0]))
    assert c.stats()["step"] == 0
    tg2 = tg.copy(); tg2[7] = [np.nan, 0, 0]
    c.train_step(dev(recs), dev(tg2))
    st = c.stats()
    assert st["step"] == 1 and st["nonfinite_targets"] == 1
    assert np.all(np.isfinite(c.get_params("train")))
