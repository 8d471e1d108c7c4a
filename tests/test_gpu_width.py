"""Width ablation (BASELINE.json configs[3]): the query at
hidden width 32 and 128 (input 64, depth 5) against the width-general fp64
oracle (oracle.query_w), plus init parity (training at these widths: tests/test_gpu_width_train.py)."""
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


@pytest.mark.parametrize("hw", [32, 64, 128])
def test_width_init_matches_oracle(nrc, orc, hw):
    c = nrc.RadianceCache(nrc.Config(hidden_width=hw, seed=5))
    assert c.nparam == orc.param_count_w(hw)
    np.testing.assert_array_equal(c.get_params("train"), orc.init_weights_w(hw, 5))
    np.testing.assert_array_equal(c.get_params("ema"), orc.init_weights_w(hw, 5))


@pytest.mark.parametrize("hw", [32, 128])
@pytest.mark.parametrize("n", [1, 129, 5000])
def test_width_query_parity(nrc, orc, hw, n):
    rng = np.random.default_rng(hw + n)
    c = nrc.RadianceCache(nrc.Config(hidden_width=hw))
    # weights off init with a scale that keeps activations O(1) at every width
    w = orc.init_weights_w(hw, 11).astype(np.float64) * rng.uniform(0.9, 1.6)
    w += rng.normal(0, 0.02, w.size)
    c.set_params(w.astype(np.float32), "ema")
    recs = nrc_inputs.records(n, seed=300 + n)
    q = c.query(dev(recs)).cpu().numpy()
    ref = orc.query_w(hw, c.get_params("ema").astype(np.float64), recs)
    assert max(radiance_err(q, ref)) <= TOL_RADIANCE


@pytest.mark.parametrize("hw", [32, 128])
def test_width_query_1080p_sampled(nrc, orc, hw):
    n = nrc_inputs.N_1080P
    recs = nrc_inputs.records(n, seed=nrc_inputs.SEED_QUERY)
    c = nrc.RadianceCache(nrc.Config(hidden_width=hw, seed=3))
    q = c.query(dev(recs)).cpu().numpy()
    idx = np.unique(np.concatenate([np.linspace(0, n - 1, 8000).astype(np.int64), np.arange(n - 130, n)]))
    ref = orc.query_w(hw, c.get_params("ema").astype(np.float64), recs[idx])
    assert max(radiance_err(q[idx], ref)) <= TOL_RADIANCE
    assert np.all(np.isfinite(q))
