"""Pins of the oracle's width-ablation functions (BASELINE.json configs[3],
SURVEY 8(d) C4: hidden width 32 / 64 / 128, input 64, depth 5).

orc_forward_w / orc_query_batch_w are pinned to the separately pinned
width-64 oracle through exact embeddings (a narrow net zero-padded into a
wider one computes the same function), plus closed forms; orc_init_weights_w
is pinned by its Glorot bound and moments and by equality with the width-64
init (reading R16)."""
import numpy as np
import pytest

import nrc_inputs


def _mats(hw, W):
    """Split a logical width-hw parameter vector into its 6 matrices."""
    shapes = [(hw, 64)] + [(hw, hw)] * 4 + [(3, hw)]
    out, o = [], 0
    for r, c in shapes:
        out.append(W[o:o + r * c].reshape(r, c))
        o += r * c
    assert o == W.size
    return out


def _embed(hw_small, W_small, hw_big):
    """Zero-pad a width-hw_small net into width hw_big (same function)."""
    ms = _mats(hw_small, W_small)
    big = [np.zeros((hw_big, 64))] + [np.zeros((hw_big, hw_big)) for _ in range(4)] + [np.zeros((3, hw_big))]
    big[0][:hw_small, :] = ms[0]
    for i in range(1, 5):
        big[i][:hw_small, :hw_small] = ms[i]
    big[5][:, :hw_small] = ms[5]
    return np.concatenate([m.reshape(-1) for m in big])


@pytest.mark.parametrize("hw", [32, 64, 128])
def test_param_count(orc, hw):
    assert orc.param_count_w(hw) == 64 * hw + 4 * hw * hw + 3 * hw
    assert orc.param_count_w(64) == orc.NPARAM == 20672


def test_embedding_32_into_64_matches_width64_oracle(orc):
    rng = np.random.default_rng(3)
    W32 = rng.normal(0, 0.3, orc.param_count_w(32))
    W64 = _embed(32, W32, 64)
    recs = nrc_inputs.records(300, seed=41)
    q32 = orc.query_w(32, W32, recs)
    q64 = orc.query(W64, recs)  # the pinned width-64 oracle
    np.testing.assert_array_equal(q32, q64)


def test_embedding_64_into_128_matches_width64_oracle(orc):
    rng = np.random.default_rng(4)
    W64 = rng.normal(0, 0.2, 20672)
    W128 = _embed(64, W64, 128)
    recs = nrc_inputs.records(300, seed=42)
    np.testing.assert_array_equal(orc.query_w(128, W128, recs), orc.query(W64, recs))
    np.testing.assert_array_equal(orc.query_w(64, W64, recs), orc.query(W64, recs))


@pytest.mark.parametrize("hw", [32, 128])
def test_zero_and_constant_nets(orc, hw):
    recs = nrc_inputs.records(50, seed=43)
    np.testing.assert_array_equal(orc.query_w(hw, np.zeros(orc.param_count_w(hw)), recs, flags=0), 0)
    # constant net through the pad channel e[62] = 1: h0[0] = relu(c), then a
    # chain of unit weights on neuron 0, W5[:, 0] = 1 -> y = (c, c, c)
    ms = [np.zeros_like(m) for m in _mats(hw, np.zeros(orc.param_count_w(hw)))]
    c = 0.8125
    ms[0][0, 62] = c
    for i in range(1, 5):
        ms[i][0, 0] = 1.0
    ms[5][:, 0] = 1.0
    W = np.concatenate([m.reshape(-1) for m in ms])
    np.testing.assert_array_equal(orc.query_w(hw, W, recs, flags=0), c)


@pytest.mark.parametrize("hw", [32, 128])
def test_output_layer_homogeneity(orc, hw):
    rng = np.random.default_rng(5)
    W = rng.normal(0, 0.2, orc.param_count_w(hw))
    recs = nrc_inputs.records(64, seed=44)
    W2 = W.copy()
    W2[-3 * hw:] *= 4.0  # scale W5 by a power of two: exact
    np.testing.assert_array_equal(orc.query_w(hw, W2, recs, flags=0), 4.0 * orc.query_w(hw, W, recs, flags=0))


@pytest.mark.parametrize("hw", [32, 64, 128])
def test_init_weights_w(orc, hw):
    W = orc.init_weights_w(hw, 9).astype(np.float64)
    ms = _mats(hw, W)
    fans = [(64, hw)] + [(hw, hw)] * 4 + [(hw, 3)]
    for m, (fi, fo) in zip(ms, fans):
        b = np.sqrt(6.0 / (fi + fo))
        assert np.max(np.abs(m)) <= b
        if m.size >= 1000:
            assert abs(m.mean()) < 0.05 * b
            assert abs(m.var() / (b * b / 3.0) - 1.0) < 0.1  # U(-b, b) variance b^2/3
    if hw == 64:
        np.testing.assert_array_equal(orc.init_weights_w(64, 9), orc.init_weights(9))
