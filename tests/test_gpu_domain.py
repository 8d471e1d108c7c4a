"""GPU <-> oracle parity over Table 1's whole input domain and the HDR loss
regime (VERDICT r1 "What's missing" 2, 3, 7).

Table 1 takes a position x in R^3 (normalised by the cache's
AABB, reading R3, with no clamp: the triangle waves are defined on all
reals), arbitrary direction / normal vectors renormalised by sph (R7), a
roughness r in R (r < 0 reads as 0) and reflectances in R.  These tests run
the encoder, the query and the training on an offset, non-unit AABB with
records inside / on / outside / far outside it, non-unit, zero, pole and
seam vectors, alpha + beta = 0 and > 1, and on HDR targets from 1e-3 to 1e4
(the bright-emitter regime of the relative loss), whose dL/dy
exceeds the fp16 range before the per-tile scale of reading R25."""
import numpy as np
import pytest
import torch

import nrc_inputs
from parity import (TOL_GRAD, TOL_PARAM, TOL_RADIANCE, assert_support_sets, fp16_ulp, per_matrix_err,
                    post_adam_err, radiance_err)

pytestmark = pytest.mark.gpu

LO, HI = nrc_inputs.DOMAIN_AABB_LO, nrc_inputs.DOMAIN_AABB_HI


@pytest.fixture(scope="module")
def nrc():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as p
    return p


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def domain_cache(nrc, **kw):
    return nrc.RadianceCache(nrc.Config(aabb_min=LO, aabb_max=HI, **kw))


def n_zero_vectors(recs):
    return int(np.sum(np.all(recs[:, 3:6] == 0, axis=1)) + np.sum(np.all(recs[:, 6:9] == 0, axis=1)))


@pytest.mark.parametrize("n", [1, 777, 20000])
def test_encode_domain_within_one_fp16_ulp(nrc, orc, n):
    """Every encoded feature within 1 fp16 ulp of fp16_RN(oracle), both
    one-blob support directions, pads exact; zero vectors counted."""
    recs = nrc_inputs.domain_records(n, seed=0xD0 + n)
    cache = domain_cache(nrc)
    got = cache.encode(dev(recs)).cpu().numpy().astype(np.float64)
    ref = orc.encode(recs, LO, HI)
    ref16 = ref.astype(np.float16).astype(np.float64)
    err = np.abs(got - ref16)
    bad = err > fp16_ulp(ref16) * 1.0001
    assert not bad.any(), (np.argwhere(bad)[:5], got[bad][:5], ref[bad][:5])
    assert_support_sets(got, ref)
    np.testing.assert_array_equal(got[:, 62:], 1.0)
    assert cache.stats()["degenerate_vectors"] == n_zero_vectors(recs)


def test_encode_domain_special_values(nrc, orc):
    """Hand-built edge records: AABB corners, far positions, poles, both sides
    of the phi seam (signed zeros, atan2(+-0, x<0) = +-pi), -0 components,
    zero vectors, negative roughness."""
    rows = []
    for p in ([LO[0], LO[1], LO[2]], [HI[0], HI[1], HI[2]], [999.5, -999.25, 1000.0], [-3.7, 9.0, 0.0]):
        for w in ([0, 0, 1], [0, 0, -5], [-2, 0.0, 0.5], [-2, -0.0, 0.5], [-0.0, 0.0, 3], [0, 0, 0],
                  [1e-3, 0, 0], [-1e3, 1e-20, 0]):
            rows.append(p + w + [0.3, -0.4, 0.8] + [-1.5] + [0.5, 0.25, 0.0] + [0.1, 0.1, 0.1])
    recs = np.array(rows, np.float32)
    recs[3::8, 4] = np.float32(-0.0)
    cache = domain_cache(nrc)
    got = cache.encode(dev(recs)).cpu().numpy().astype(np.float64)
    ref = orc.encode(recs, LO, HI)
    ref16 = ref.astype(np.float16).astype(np.float64)
    assert np.all(np.abs(got - ref16) <= fp16_ulp(ref16) * 1.0001)
    assert_support_sets(got, ref)
    assert cache.stats()["degenerate_vectors"] == n_zero_vectors(recs)


@pytest.mark.parametrize("n", [129, 4096 + 77, 200_000])
def test_query_domain_parity(nrc, orc, n):
    """Queries over the off-default domain against the oracle (radiance
    tolerance 1e-2), after a few training steps so the net is off init;
    alpha + beta = 0 rows give exactly 0."""
    recs = nrc_inputs.domain_records(n, seed=0xD5 + n)
    cache = domain_cache(nrc)
    tr = nrc_inputs.domain_records(8192, seed=0xD6)
    with np.errstate(over="ignore", invalid="ignore"):  # the analytic field at non-unit omega / n
        tg = nrc_inputs.targets(tr, seed=3)
    tg = np.nan_to_num(tg, nan=0.5, posinf=1.0, neginf=0.0)
    cache.train_frame(dev(tr), dev(tg), 4, 2048, 5)
    q = cache.query(dev(recs)).cpu().numpy()
    ref = orc.query(cache.get_params("ema").astype(np.float64), recs, LO, HI)
    errs = radiance_err(q, ref)
    assert max(errs) <= TOL_RADIANCE, errs
    zero = np.all(recs[:, 10:16] == 0, axis=1)
    np.testing.assert_array_equal(q[zero], 0.0)
    assert np.all(q >= 0)


@pytest.mark.parametrize("n", [3000, 16384])
def test_gradient_domain_parity(nrc, orc, n):
    """Training gradient over the off-default domain (loss, per-matrix
    gradient) against the oracle."""
    recs = nrc_inputs.domain_records(n, seed=0xD7 + n)
    tg = np.abs(nrc_inputs.targets(nrc_inputs.records(n, seed=n), seed=1))
    cache = domain_cache(nrc)
    W = cache.get_params("train").astype(np.float64)
    g, ls = cache.train_backward(dev(recs), dev(tg))
    g_ref, l_ref, _ = orc.grad_batch(W, recs, tg, LO, HI)
    errs = per_matrix_err(g.cpu().numpy(), g_ref)
    assert max(errs) <= TOL_GRAD, errs
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)
    assert cache.stats()["nonfinite_grads"] == 0


@pytest.mark.parametrize("n,hi_exp", [(3000, 4.0), (16384, 4.0), (16384, 6.0)])
def test_hdr_targets_gradient_and_adam(nrc, orc, n, hi_exp):
    """Targets from 1e-3 to 1e4 (and 1e6) from fresh weights: |dL/dy| =
    2 |y - t| (alpha + beta) / (3 (lum^2 + eps)) reaches ~1e5 .. 1e7, beyond
    fp16's 65,504; the per-tile power-of-two scale (R25) keeps the fp16
    backward finite.  Gradient, loss and post-Adam parameters match the oracle
    and no gradient entry is zeroed as non-finite."""
    recs = nrc_inputs.records(n, seed=0xAD + n)
    tg = nrc_inputs.hdr_targets(n, seed=n, hi_exp=hi_exp)
    cache = nrc.RadianceCache()
    oc = orc.OracleCache(W32=cache.get_params("train"))
    g, ls = cache.train_backward(dev(recs), dev(tg))
    g = g.cpu().numpy()
    assert np.all(np.isfinite(g))
    g_ref, l_ref, _ = orc.grad_batch(oc.w, recs, tg)
    errs = per_matrix_err(g, g_ref)
    assert max(errs) <= TOL_GRAD, errs
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)
    loss = cache.train_step(dev(recs), dev(tg)).item()
    l1, G1 = oc.train_step(recs, tg, return_grad=True)
    assert loss == pytest.approx(l1, rel=1e-2)
    assert cache.stats()["nonfinite_grads"] == 0
    errs, flip_frac, worst = post_adam_err(cache.get_params("train"), oc.w, g / n, G1)
    assert max(errs) <= TOL_PARAM, errs
    assert flip_frac <= 0.01 and worst <= 3e-2, (flip_frac, worst)


def test_hdr_training_frames_stay_finite(nrc, orc):
    """Several HDR frames in a row (LCG-shuffled, 4 x 4096): losses finite and
    within 1e-2 of the oracle's over the first frame, no non-finite gradient
    entry, finite weights."""
    n, s, l = 16384, 4, 4096
    recs = nrc_inputs.records(n, seed=0xAE)
    tg = nrc_inputs.hdr_targets(n, seed=0xAF)
    cache = nrc.RadianceCache()
    oc = orc.OracleCache(W32=cache.get_params("train"))
    losses = cache.train_frame(dev(recs), dev(tg), s, l, 3).cpu().numpy()
    a, c, m = orc.lcg_params(n, 3)
    perm = orc.lcg_permute(n, a, c, m).astype(np.int64)
    ref = [oc.train_step(recs[perm[j * l:(j + 1) * l]], tg[perm[j * l:(j + 1) * l]]) for j in range(s)]
    np.testing.assert_allclose(losses, ref, rtol=1e-2)
    for f in range(3):
        cache.train_frame(dev(recs), dev(tg), s, l, 10 + f)
    assert cache.stats()["nonfinite_grads"] == 0
    assert np.all(np.isfinite(cache.get_params("train")))


@pytest.mark.parametrize("n", [1, 300, 16384, 40_000])
def test_query_equals_training_forward_bitwise(nrc, n):
    """SURVEY 8(c) GPU self-consistency: the query kernel (a2, activations in
    TMEM) and the training forward (a4, stash in shared memory) compute the
    same factored prediction y * (alpha + beta) bit for bit on the same
    weights (query reading W_t, clamp off)."""
    recs = nrc_inputs.domain_records(n, seed=0xB0 + n)
    cfg = dict(flags=nrc.FACTORIZE | nrc.QUERY_RAW_WEIGHTS)
    cache = domain_cache(nrc, **cfg)
    tr = nrc_inputs.records(4096, seed=1)
    cache.train_frame(dev(tr), dev(nrc_inputs.targets(tr)), 2, 2048, 1)  # off init
    pred = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    tg = torch.zeros((n, 3), dtype=torch.float32, device="cuda")
    cache.train_backward(dev(recs), tg, pred=pred)
    q = cache.query(dev(recs)).cpu().numpy()
    np.testing.assert_array_equal(q, pred.cpu().numpy())
