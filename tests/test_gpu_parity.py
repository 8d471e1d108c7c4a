"""GPU <-> oracle parity through the C ABI (SURVEY 8(c) parity definitions).

Every test runs the CUDA path (libnrc.so) and compares with the fp64 oracle
on the same seeded inputs from nrc_inputs.  Tolerances are north_star's
(radiance 1e-2, gradients / post-Adam 3e-2, encoding within 1 fp16 ulp with
bit-exact integer parts)."""
import numpy as np
import pytest
import torch

import nrc_inputs
from parity import (TOL_GRAD, TOL_PARAM, TOL_RADIANCE, assert_support_sets, fp16_ulp, per_matrix_err,
                    post_adam_err, radiance_err)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nrc():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as p
    return p


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# ---------------------------------------------------------------- tcgen05 operand layouts
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
def test_selftest_umma_layouts(nrc, mode):
    g = torch.Generator().manual_seed(mode)
    a = torch.randn(128, 64, generator=g).half()
    bshape = {0: (64, 64), 1: (64, 64), 2: (128, 64), 3: (16, 64), 4: (64, 64)}[mode]
    b = torch.randn(*bshape, generator=g).half()
    d = nrc.selftest_umma(mode, a.cuda(), b.cuda()).cpu()
    A, B = a.float(), b.float()
    ref = {0: lambda: A @ B.T, 1: lambda: A @ B, 2: lambda: A.T @ B, 3: lambda: A @ B.T, 4: lambda: A @ B.T}[mode]()
    torch.testing.assert_close(d, ref, rtol=1e-4, atol=1e-3)


# ---------------------------------------------------------------- encoding
@pytest.mark.parametrize("n", [1, 127, 1000])
def test_encode_within_one_fp16_ulp(nrc, orc, n):
    recs = nrc_inputs.records(n, seed=100 + n)
    cache = nrc.RadianceCache()
    got = cache.encode(dev(recs)).cpu().numpy().astype(np.float64)
    ref = orc.encode(recs)
    ref16 = ref.astype(np.float16).astype(np.float64)
    err = np.abs(got - ref16)
    assert np.all(err <= fp16_ulp(ref16) * 1.0001), float(err.max())
    # integer parts bit-exact: the one-blob support sets (both directions) and the pads
    assert_support_sets(got, ref)
    np.testing.assert_array_equal(got[:, 62:], 1.0)


def test_encode_golden_c0(nrc):
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "encode_c0.txt")
    rec, vals = None, {}
    for line in open(path):
        if line.startswith("# record:"):
            rec = np.array([float(x) for x in line.split(":")[1].split()], np.float32)
        elif line.strip() and not line.startswith("#"):
            i, v = line.split(); vals[int(i)] = float(v)
    want = np.array([vals[i] for i in range(64)]).astype(np.float16).astype(np.float64)
    got = nrc.RadianceCache().encode(dev(rec[None])).cpu().numpy()[0].astype(np.float64)
    assert np.all(np.abs(got - want) <= fp16_ulp(want) * 1.0001)


# ---------------------------------------------------------------- query
@pytest.mark.parametrize("n", [1, 129, 1000, 4096 + 77])
def test_query_parity(nrc, orc, n):
    recs = nrc_inputs.records(n, seed=200 + n)
    cache = nrc.RadianceCache()
    q = cache.query(dev(recs)).cpu().numpy()
    W = cache.get_params("ema").astype(np.float64)
    ref = orc.query(W, recs)
    errs = radiance_err(q, ref)
    assert max(errs) <= TOL_RADIANCE, errs
    assert np.all(q >= 0)


def test_query_parity_1080p_every_record(nrc, orc):
    """C2-size query (2,073,600 records, the bench launch configuration):
    every record against the oracle (SURVEY 8(c) "Scale")."""
    n = nrc_inputs.N_1080P
    recs = nrc_inputs.records(n, seed=nrc_inputs.SEED_QUERY)
    cache = nrc.RadianceCache()
    # move the weights off init so the outputs are not trivially small
    tr, tg = nrc_inputs.train_frame(0)
    cache.train_frame(dev(tr), dev(tg), 4, 16384, 1)
    q = cache.query(dev(recs)).cpu().numpy()
    ref = orc.query(cache.get_params("ema").astype(np.float64), recs)
    errs = radiance_err(q, ref)
    assert max(errs) <= TOL_RADIANCE, errs
    assert np.all(np.isfinite(q)) and np.all(q >= 0)


def test_query_parity_4k_every_record(nrc, orc):
    """C5-size query (3840 x 2160 = 8,294,400 records, default max_batch) on
    one GPU: every record against the oracle."""
    n = nrc_inputs.N_4K
    recs = nrc_inputs.records(n, seed=nrc_inputs.SEED_QUERY + 1)
    tr, tg = nrc_inputs.train_frame(1)
    cache = nrc.RadianceCache()
    cache.train_frame(dev(tr), dev(tg), 4, 16384, 2)
    q = cache.query(dev(recs)).cpu().numpy()
    ref = orc.query(cache.get_params("ema").astype(np.float64), recs)
    errs = radiance_err(q, ref)
    assert max(errs) <= TOL_RADIANCE, errs


def test_query_raw_vs_ema_and_factorization_off(nrc, orc):
    recs = nrc_inputs.records(700, seed=7)
    tr, tg = nrc_inputs.train_frame(3, n=4096)
    for flags in (nrc.FACTORIZE | nrc.CLAMP_QUERY | nrc.QUERY_RAW_WEIGHTS, 0):
        cache = nrc.RadianceCache(nrc.Config(flags=flags))
        cache.train_step(dev(tr), dev(tg))
        q = cache.query(dev(recs)).cpu().numpy()
        which = "train" if flags & nrc.QUERY_RAW_WEIGHTS else "ema"
        ref = orc.query(cache.get_params(which).astype(np.float64), recs, flags=flags & 3)
        assert max(radiance_err(q, ref)) <= TOL_RADIANCE


def test_query_zero_reflectance_and_zero_weights(nrc):
    recs = nrc_inputs.records(300, seed=9)
    recs[:, 10:16] = 0
    cache = nrc.RadianceCache()
    np.testing.assert_array_equal(cache.query(dev(recs)).cpu().numpy(), 0)
    recs = nrc_inputs.records(300, seed=9)
    cache.set_params(np.zeros(20672, np.float32), "ema")
    np.testing.assert_array_equal(cache.query(dev(recs)).cpu().numpy(), 0)


# ---------------------------------------------------------------- training
def _grad_parity(nrc, orc, n, seed, noise=0.0):
    recs = nrc_inputs.records(n, seed=seed)
    tg = nrc_inputs.targets(recs, noise=noise, seed=seed)
    cache = nrc.RadianceCache()
    W = cache.get_params("train").astype(np.float64)
    g_gpu, ls = cache.train_backward(dev(recs), dev(tg))
    g_gpu = g_gpu.cpu().numpy()
    g_ref, l_ref, _ = orc.grad_batch(W, recs, tg)
    return g_gpu, g_ref, float(ls.item()), l_ref


@pytest.mark.parametrize("n", [256, 1, 300, 129])
def test_gradient_parity(nrc, orc, n):
    g_gpu, g_ref, l_gpu, l_ref = _grad_parity(nrc, orc, n, 300 + n, noise=0.3)
    errs = per_matrix_err(g_gpu, g_ref)
    assert max(errs) <= TOL_GRAD, errs
    assert l_gpu == pytest.approx(l_ref, rel=1e-2)


def test_gradient_parity_16384(nrc, orc):
    """One full training batch (l = 16,384) in the bench configuration."""
    g_gpu, g_ref, l_gpu, l_ref = _grad_parity(nrc, orc, 16384, 0x7EA1)
    errs = per_matrix_err(g_gpu, g_ref)
    assert max(errs) <= TOL_GRAD, errs
    assert l_gpu == pytest.approx(l_ref, rel=1e-2)


def test_train_step_parity_c1(nrc, orc):
    """C1: 256 records, one step: loss, gradient, post-Adam W and W-bar."""
    recs, tg = nrc_inputs.train_frame(0, n=256, noise=0.3)
    cache = nrc.RadianceCache()
    oc = orc.OracleCache(W32=cache.get_params("train"))
    g_gpu, _ = cache.train_backward(dev(recs), dev(tg))
    g_gpu = g_gpu.cpu().numpy() / 256.0
    loss = cache.train_step(dev(recs), dev(tg)).item()
    l_ref, G_ref = oc.train_step(recs, tg, return_grad=True)
    assert loss == pytest.approx(l_ref, rel=1e-2)
    w_gpu = cache.get_params("train")
    errs, flip_frac, worst = post_adam_err(w_gpu, oc.w, g_gpu, G_ref)
    assert max(errs) <= TOL_PARAM, errs
    assert flip_frac <= 0.01 and worst <= 3e-2, (flip_frac, worst)
    e_errs, _, _ = post_adam_err(cache.get_params("ema"), oc.wbar, g_gpu, G_ref)
    assert max(e_errs) <= TOL_PARAM
    assert cache.stats()["step"] == 1


def test_adam_kernel_alone_matches_oracle(nrc, orc):
    """Adam + EMA on the GPU's own gradient: oracle Adam on the same gradient
    agrees to 1e-6 relative (isolates the optimiser from the fp16 backward)."""
    recs, tg = nrc_inputs.train_frame(1, n=2048, noise=0.3)
    cache = nrc.RadianceCache()
    w0 = cache.get_params("train").astype(np.float64)
    g, _ = cache.train_backward(dev(recs), dev(tg))
    g_np = g.cpu().numpy().astype(np.float64)
    cache.train_apply(g, 2048)
    w = w0.copy(); m = np.zeros_like(w); v = np.zeros_like(w); wbar = w0.copy()
    orc.adam(w, m, v, g_np.astype(np.float32).astype(np.float64) / 2048.0, 1)
    orc.ema(wbar, w, 1, 0.99)
    w_gpu = cache.get_params("train").astype(np.float64)
    assert np.max(np.abs(w_gpu - w)) <= 1e-6 * np.max(np.abs(w)) + 1e-7
    np.testing.assert_allclose(cache.get_params("adam_m"), m, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(cache.get_params("adam_v"), v, rtol=1e-5, atol=1e-16)
    # step 2 with the same gradient exercises bias correction and the EMA history
    cache.train_apply(g, 2048)
    orc.adam(w, m, v, g_np.astype(np.float32).astype(np.float64) / 2048.0, 2)
    orc.ema(wbar, w, 2, 0.99)
    assert np.max(np.abs(cache.get_params("train") - w)) <= 1e-6 * np.max(np.abs(w)) + 1e-7
    assert np.max(np.abs(cache.get_params("ema") - wbar)) <= 1e-6 * np.max(np.abs(wbar)) + 1e-7


def test_train_frame_equals_gathered_steps(nrc, orc):
    """nrc_train_frame == s train steps on the LCG-gathered batches (bitwise)."""
    n, s, l, seed = 8192, 4, 2048, 11
    recs, tg = nrc_inputs.train_frame(5, n=n)
    a = nrc.RadianceCache(); b = nrc.RadianceCache()
    losses = a.train_frame(dev(recs), dev(tg), s, l, seed).cpu().numpy()
    pa, pc, pm = orc.lcg_params(n, seed)
    perm = orc.lcg_permute(n, pa, pc, pm).astype(np.int64)
    lb = []
    for j in range(s):
        idx = perm[j * l:(j + 1) * l]
        lb.append(b.train_step(dev(recs[idx]), dev(tg[idx])).item())
    np.testing.assert_array_equal(a.get_params("train"), b.get_params("train"))
    np.testing.assert_array_equal(a.get_params("ema"), b.get_params("ema"))
    np.testing.assert_array_equal(losses, np.array(lb, np.float32))
    assert a.stats()["step"] == s


def test_train_frame_shrinks_batches(nrc):
    recs, tg = nrc_inputs.train_frame(6, n=1000)
    c = nrc.RadianceCache()
    c.train_frame(dev(recs), dev(tg), 4, 16384, 3)  # l -> 1000 // 4 = 250
    assert c.stats()["step"] == 4


def test_determinism_bitwise(nrc):
    recs, tg = nrc_inputs.train_frame(7, n=16384, noise=0.3)
    q = nrc_inputs.records(5000, seed=17)
    outs = []
    for _ in range(2):
        c = nrc.RadianceCache()
        c.train_frame(dev(recs), dev(tg), 4, 4096, 5)
        outs.append((c.get_params("train"), c.query(dev(q)).cpu().numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_empty_and_nonfinite(nrc):
    c = nrc.RadianceCache()
    w0 = c.get_params("train")
    e = torch.empty((0, 16), dtype=torch.float32, device="cuda")
    c.train_step(e, torch.empty((0, 3), dtype=torch.float32, device="cuda"))
    c.query(e)
    np.testing.assert_array_equal(c.get_params("train"), w0)
    assert c.stats()["step"] == 0
    recs, tg = nrc_inputs.train_frame(8, n=512)
    tg[5] = [np.nan, 0, 0]
    tg[300] = [np.inf, 1, 1]
    c.train_step(dev(recs), dev(tg))
    st = c.stats()
    assert st["nonfinite_targets"] == 2 and st["nonfinite_grads"] == 0
    assert np.all(np.isfinite(c.get_params("train")))


def test_set_get_roundtrip(nrc):
    c = nrc.RadianceCache()
    w = np.random.default_rng(0).uniform(-0.2, 0.2, 20672).astype(np.float32)
    c.set_params(w, "train")
    np.testing.assert_array_equal(c.get_params("train"), w)
    c.set_params(w, "ema")
    np.testing.assert_array_equal(c.get_params("ema"), w)


def test_init_matches_oracle_init(nrc, orc):
    # both sides implement reading R16 (splitmix64 Glorot); identical fp32 bits
    for seed in (1, 12345):
        c = nrc.RadianceCache(nrc.Config(seed=seed))
        np.testing.assert_array_equal(c.get_params("train"), orc.init_weights(seed))
        np.testing.assert_array_equal(c.get_params("ema"), orc.init_weights(seed))


@pytest.mark.parametrize("hw,nh", [(64, 5), (128, 3), (32, 8)])
def test_frame_host_equals_device_calls(nrc, hw, nh):
    """nrc_frame_host (pinned host buffers, chunked copies overlapped with the
    query) gives the same bits as nrc_query + nrc_train_frame on device data,
    over two consecutive frames (scratch and event reuse) -- at the paper's
    network and at a width / depth variant."""
    nq, s, l = 600_001, 4, 2048
    q = nrc_inputs.records(nq, seed=61)
    tr, tg = nrc_inputs.train_frame(4, n=s * l)
    cfg = nrc.Config(hidden_width=hw, n_hidden_layers=nh)
    a, b = nrc.RadianceCache(cfg), nrc.RadianceCache(cfg)
    hq = torch.from_numpy(q).pin_memory()
    ht, htg = torch.from_numpy(tr).pin_memory(), torch.from_numpy(tg).pin_memory()
    hrgb = torch.empty((nq, 3), dtype=torch.float32).pin_memory()
    hl = torch.empty(64, dtype=torch.float32).pin_memory()
    scratch = torch.empty(a.frame_scratch_bytes(nq, s * l) + 256, dtype=torch.uint8, device="cuda")
    scratch = scratch[(-scratch.data_ptr()) % 256:]
    for frame in range(2):
        a.frame_host(hq.numpy(), hrgb.numpy(), ht.numpy(), htg.numpy(), s, l, 9 + frame, hl.numpy(), scratch)
        torch.cuda.synchronize()
        rgb_b = b.query(dev(q)).cpu().numpy()
        lb = b.train_frame(dev(tr), dev(tg), s, l, 9 + frame).cpu().numpy()
        np.testing.assert_array_equal(hrgb.numpy(), rgb_b)
        np.testing.assert_array_equal(hl.numpy()[:s], lb)
    np.testing.assert_array_equal(a.get_params("train"), b.get_params("train"))
    np.testing.assert_array_equal(a.get_params("ema"), b.get_params("ema"))


def test_multi_tile_ctas_gradient_and_step(nrc, orc):
    """Batches larger than one tile per SM (40,000 rows = 313 tiles on <= 148
    CTAs, several tiles per CTA): the partials-only path (train_backward) and
    the step (train_step) against the oracle's gradient and post-Adam
    weights."""
    n = 40_000
    recs, tg = nrc_inputs.train_frame(8, n=n, noise=0.3)
    cache = nrc.RadianceCache()
    oc = orc.OracleCache(W32=cache.get_params("train"))
    g_gpu, ls = cache.train_backward(dev(recs), dev(tg))
    g_gpu = g_gpu.cpu().numpy()
    g_ref, l_ref, _ = orc.grad_batch(oc.w, recs, tg)
    assert max(per_matrix_err(g_gpu, g_ref)) <= TOL_GRAD
    assert float(ls.item()) == pytest.approx(l_ref, rel=1e-2)
    loss = cache.train_step(dev(recs), dev(tg)).item()
    l1, G1 = oc.train_step(recs, tg, return_grad=True)
    assert loss == pytest.approx(l1, rel=1e-2)
    errs, flip_frac, worst = post_adam_err(cache.get_params("train"), oc.w, g_gpu / n, G1)
    assert max(errs) <= TOL_PARAM, errs
    assert flip_frac <= 0.01 and worst <= 3e-2, (flip_frac, worst)


def test_train_frame_eleven_steps(nrc):
    """s = 11 steps: bitwise equal to 11 single steps on the gathered
    batches, losses included."""
    n, s, l, seed = 11 * 1024, 11, 1024, 5
    recs, tg = nrc_inputs.train_frame(6, n=n)
    a, b = nrc.RadianceCache(), nrc.RadianceCache()
    la = a.train_frame(dev(recs), dev(tg), s, l, seed).cpu().numpy()
    pa, pc, pm = nrc.lcg_params(n, seed)
    import oracle
    perm = oracle.lcg_permute(n, pa, pc, pm).astype(np.int64)
    lb = [b.train_step(dev(recs[perm[j * l:(j + 1) * l]]), dev(tg[perm[j * l:(j + 1) * l]])).item()
          for j in range(s)]
    np.testing.assert_array_equal(la, np.array(lb, np.float32))
    np.testing.assert_array_equal(a.get_params("train"), b.get_params("train"))
    assert a.stats()["step"] == s
