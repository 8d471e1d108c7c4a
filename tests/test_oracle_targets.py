"""Pins of orc_assemble_targets (self-training targets):
closed forms on one- and three-vertex paths evaluated by hand, the unbiased
flag (tail ignored), and linearity in the tail radiance."""
import numpy as np

import nrc_inputs


def _one(orc, E, N, T, tail, flag=0):
    vert = np.array([list(E) + list(N) + list(T)], np.float32)
    return orc.assemble_targets([0], [1], [flag], vert, np.array([tail], np.float32))[0]


def test_single_vertex_closed_form(orc):
    got = _one(orc, (1.0, 0.0, 0.5), (0.25, 0.5, 0.0), (0.5, 0.25, 2.0), (2.0, 4.0, 1.0))
    np.testing.assert_array_equal(got, [1.0 + 0.25 + 0.5 * 2.0, 0.0 + 0.5 + 0.25 * 4.0, 0.5 + 0.0 + 2.0 * 1.0])


def test_unbiased_flag_ignores_tail(orc):
    got = _one(orc, (1.0, 2.0, 3.0), (0.5, 0.5, 0.5), (0.9, 0.9, 0.9), (100.0, 100.0, 100.0), flag=1)
    np.testing.assert_array_equal(got, [1.5, 2.5, 3.5])


def test_three_vertex_path_by_hand(orc):
    # v0 <- v1 <- v2 <- tail, single channel values chosen to be exact in binary
    E = [0.0, 0.0, 1.0]
    N = [0.25, 0.5, 0.125]
    T = [0.5, 0.25, 0.75]
    tail = 2.0
    t2 = 1.0 + 0.125 + 0.75 * 2.0        # 2.625
    t1 = 0.0 + 0.5 + 0.25 * t2           # 1.15625
    t0 = 0.0 + 0.25 + 0.5 * t1           # 0.828125
    vert = np.array([[E[i]] * 3 + [N[i]] * 3 + [T[i]] * 3 for i in range(3)], np.float32)
    got = orc.assemble_targets([0], [3], [0], vert, np.array([[tail] * 3], np.float32))
    np.testing.assert_array_equal(got[:, 0], [t0, t1, t2])
    # the same path placed second, after a one-vertex path, in one batch
    vert2 = np.concatenate([np.ones((1, 9), np.float32), vert])
    got2 = orc.assemble_targets([0, 1], [1, 3], [1, 0], vert2, np.array([[9.0] * 3, [tail] * 3], np.float32))
    np.testing.assert_array_equal(got2[1:, 0], [t0, t1, t2])
    np.testing.assert_array_equal(got2[0], [2.0, 2.0, 2.0])  # unbiased: E + N


def test_linearity_in_tail(orc):
    first, length, flags, vert, _, _ = nrc_inputs.training_paths(3000, seed=9)
    rng = np.random.default_rng(1)
    a = rng.uniform(0, 2, (length.size, 3)).astype(np.float32)
    zero = orc.assemble_targets(first, length, flags, vert, np.zeros_like(a))
    ta = orc.assemble_targets(first, length, flags, vert, a)
    t2a = orc.assemble_targets(first, length, flags, vert, 2 * a)
    np.testing.assert_allclose(t2a - zero, 2 * (ta - zero), rtol=1e-12, atol=1e-12)
    # unbiased paths do not depend on the tail at all
    for p in np.nonzero(flags)[0][:20]:
        s = slice(int(first[p]), int(first[p] + length[p]))
        np.testing.assert_array_equal(ta[s], zero[s])


def test_query_accumulate_pins(orc):
    """orc_query_accumulate: unit throughput on distinct pixels of
    a zero image reproduces the query; a pixel permutation permutes the image;
    two records on one pixel add; a zero throughput leaves the image."""
    recs = nrc_inputs.records(200, seed=5)
    W = orc.init_weights(3).astype(np.float64) * 1.3
    q = orc.query(W, recs)
    ones = np.ones((200, 3), np.float32)
    img = orc.query_accumulate(W, recs, np.arange(200), ones, np.zeros((200, 3)))
    np.testing.assert_array_equal(img, q)
    perm = np.random.default_rng(0).permutation(200)
    img_p = orc.query_accumulate(W, recs, perm, ones, np.zeros((200, 3)))
    np.testing.assert_array_equal(img_p[perm], q)
    both = orc.query_accumulate(W, recs[:2], np.array([7, 7]), np.full((2, 3), 0.5, np.float32),
                                np.ones((10, 3)))
    np.testing.assert_allclose(both[7], 1.0 + 0.5 * q[0] + 0.5 * q[1], rtol=1e-15)
    np.testing.assert_array_equal(np.delete(both, 7, axis=0), 1.0)
    z = orc.query_accumulate(W, recs, np.arange(200), np.zeros((200, 3), np.float32), np.full((200, 3), 2.0))
    np.testing.assert_array_equal(z, 2.0)
