"""Self-training target assembly on the GPU (nrc_assemble_targets, SURVEY
8(f) N1) against the fp64 oracle, alone and end to end with the
tail radiance from nrc_query."""
import numpy as np
import pytest
import torch

import nrc_inputs
from parity import TOL_RADIANCE, radiance_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nrc():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as p
    return p


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def i32(x):
    return torch.from_numpy(np.ascontiguousarray(x).astype(np.int32)).cuda()


@pytest.mark.parametrize("nv", [1, 37, 65536])
def test_assemble_targets_parity(nrc, orc, nv):
    first, length, flags, vert, _, _ = nrc_inputs.training_paths(nv, seed=nv)
    tail = np.random.default_rng(nv).uniform(0, 3, (length.size, 3)).astype(np.float32)
    c = nrc.RadianceCache()
    got = c.assemble_targets(i32(first), i32(length), i32(flags), dev(vert), dev(tail)).cpu().numpy()
    ref = orc.assemble_targets(first, length, flags, vert, tail)
    np.testing.assert_allclose(got, ref, rtol=2e-6, atol=1e-6)
    assert c.last_launch_count == 1


def test_self_training_targets_end_to_end(nrc, orc):
    first, length, flags, vert, vrec, trec = nrc_inputs.training_paths(16384, seed=77)
    c = nrc.RadianceCache()
    tr, tg = nrc_inputs.train_frame(0, n=16384)
    c.train_frame(dev(tr), dev(tg), 4, 4096, 3)  # move the cache off its init
    got = c.self_training_targets(i32(first), i32(length), i32(flags), dev(vert), dev(trec)).cpu().numpy()
    tail_ref = orc.query(c.get_params("ema").astype(np.float64), trec)
    ref = orc.assemble_targets(first, length, flags, vert, tail_ref.astype(np.float32))
    assert max(radiance_err(got, ref)) <= TOL_RADIANCE
    # the targets train the cache: one frame on the self-trained records
    losses = c.train_frame(dev(vrec), torch.from_numpy(got).cuda(), 4, 4096, 5).cpu().numpy()
    assert np.all(np.isfinite(losses))


def test_query_accumulate_parity(nrc, orc):
    """nrc_query_accumulate vs the oracle: 1080p-sized
    batch with one query per pixel in shuffled pixel order, throughputs in
    [0, 1), accumulated onto a non-zero image."""
    n = 300000
    recs = nrc_inputs.records(n, seed=91)
    rng = np.random.default_rng(2)
    pix = rng.permutation(n).astype(np.int32)
    thr = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    img0 = rng.uniform(0, 0.1, (n, 3)).astype(np.float32)
    c = nrc.RadianceCache()
    tr, tg = nrc_inputs.train_frame(0, n=16384)
    c.train_frame(dev(tr), dev(tg), 4, 4096, 3)
    image = dev(img0.copy())
    c.query_accumulate(dev(recs), dev(pix), dev(thr), image)
    got = image.cpu().numpy()
    idx = np.linspace(0, n - 1, 6000).astype(np.int64)
    ref = orc.query_accumulate(c.get_params("ema").astype(np.float64), recs[idx], pix[idx], thr[idx],
                               img0.astype(np.float64))
    # compare the touched pixels' increments against the radiance tolerance
    touched = pix[idx]
    assert max(radiance_err(got[touched] - img0[touched], ref[touched] - img0[touched])) <= TOL_RADIANCE
    # bitwise consistency with the unfused path: image + thr * query
    q = c.query(dev(recs)).cpu().numpy()
    expect = img0.copy()
    expect[pix] += thr * q
    np.testing.assert_array_equal(got, expect)
