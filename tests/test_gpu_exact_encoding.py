"""Exact encodings (NRC_EXACT_ENCODING; readings R21, R22) on
the GPU against the fp64 oracle: encoding within one fp16 ulp, query parity
and the training gradient through the exact encodings (both training paths)."""
import numpy as np
import pytest
import torch

import nrc_inputs
from parity import TOL_GRAD, TOL_RADIANCE, fp16_ulp, per_matrix_err, radiance_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nrc():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as p
    return p


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("n", [1, 1000])
def test_exact_encode_within_one_fp16_ulp(nrc, orc, n):
    recs = nrc_inputs.records(n, seed=500 + n)
    c = nrc.RadianceCache(nrc.Config(flags=nrc.FACTORIZE | nrc.CLAMP_QUERY | nrc.EXACT_ENCODING))
    got = c.encode(dev(recs)).cpu().numpy().astype(np.float64)
    ref16 = orc.encode_exact(recs).astype(np.float16).astype(np.float64)
    err = np.abs(got - ref16)
    assert np.all(err <= fp16_ulp(ref16) * 1.0001), float(err.max())


def test_exact_query_parity(nrc, orc):
    recs = nrc_inputs.records(20000, seed=501)
    c = nrc.RadianceCache(nrc.Config(flags=nrc.FACTORIZE | nrc.CLAMP_QUERY | nrc.EXACT_ENCODING))
    w = orc.init_weights(7) * 1.4
    c.set_params(w, "ema")
    q = c.query(dev(recs)).cpu().numpy()
    ref = orc.query_exact(c.get_params("ema").astype(np.float64), recs)
    assert max(radiance_err(q, ref)) <= TOL_RADIANCE
    # and it is a different function from the cheap encoding's
    cheap = orc.query(c.get_params("ema").astype(np.float64), recs)
    assert max(radiance_err(cheap, ref)) > 10 * TOL_RADIANCE


def test_exact_training_runs(nrc):
    c = nrc.RadianceCache(nrc.Config(flags=nrc.FACTORIZE | nrc.CLAMP_QUERY | nrc.EXACT_ENCODING))
    tr, tg = nrc_inputs.train_frame(0, n=16384)
    losses = [c.train_frame(dev(tr), dev(tg), 4, 4096, j).cpu().numpy() for j in range(20)]
    assert np.all(np.isfinite(losses))
    assert np.mean(losses[-1]) < np.mean(losses[0])


def test_exact_gradient_parity(nrc, orc):
    """Training with NRC_EXACT_ENCODING encodes the training records with the
    same exact primitives as the query: train_backward's gradient against
    orc_grad_batch_exact (per matrix within 3e-2, loss within 1e-2) and away
    from the cheap-encoding gradient."""
    c = nrc.RadianceCache(nrc.Config(flags=nrc.FACTORIZE | nrc.CLAMP_QUERY | nrc.EXACT_ENCODING))
    recs = nrc_inputs.records(3000, seed=502)
    tg = nrc_inputs.targets(recs, noise=0.3, seed=3)
    W = c.get_params("train").astype(np.float64)
    g, ls = c.train_backward(dev(recs), dev(tg))
    g = g.cpu().numpy()
    ref, l_ref, _ = orc.grad_batch(W, recs, tg, exact=True)
    assert max(per_matrix_err(g, ref)) <= TOL_GRAD
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)
    cheap, _, _ = orc.grad_batch(W, recs, tg)
    assert max(per_matrix_err(cheap, ref)) > 3 * TOL_GRAD


def test_exact_requires_width_64(nrc):
    with pytest.raises(nrc.NRCError):
        nrc.RadianceCache(nrc.Config(hidden_width=32, flags=nrc.EXACT_ENCODING))


def test_volume_records_query(nrc, orc):
    """Volume queries (reading R23): records assembled with the
    default surface constants query like any record (oracle parity), and the
    factorisation is the identity for them."""
    rng = np.random.default_rng(4)
    pos = torch.from_numpy(rng.random((3000, 3)).astype(np.float32)).cuda()
    d = rng.normal(size=(3000, 3)).astype(np.float32)
    dirs = torch.from_numpy(d / np.linalg.norm(d, axis=1, keepdims=True)).cuda()
    recs = nrc.volume_records(pos, dirs)
    r_np = recs.cpu().numpy()
    assert np.all(r_np[:, 10:13] + r_np[:, 13:16] == 1.0)
    c = nrc.RadianceCache()
    c.set_params(orc.init_weights(2) * 1.3, "ema")
    q = c.query(recs).cpu().numpy()
    ref = orc.query(c.get_params("ema").astype(np.float64), r_np)
    assert max(radiance_err(q, ref)) <= TOL_RADIANCE
