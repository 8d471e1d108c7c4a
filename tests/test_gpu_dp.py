"""The N > 1 data-parallel path (paper_2106_12372_b200.dp) on one GPU with a
world-size-1 NCCL group: the all-reduce is the identity, so the frame trained
through nrc_train_frame_backward + all-reduce + nrc_train_apply must agree
with the single-GPU nrc_train_frame (same gradient up to fp32 summation order) and
with the fp64 oracle on the gathered batches."""
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import nrc_inputs
from parity import TOL_RADIANCE, radiance_err

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def group():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield None
    dist.destroy_process_group()


def test_dp_frame_world1_matches_single_gpu_frame_and_oracle(group, orc):
    import paper_2106_12372_b200 as nrc
    n, s, l, seed = 8192 + 3, 4, 2048, 21
    recs, tg = nrc_inputs.train_frame(2, n=n, noise=0.3)
    d_r = torch.from_numpy(recs).cuda()
    d_t = torch.from_numpy(tg).cuda()
    fused = nrc.RadianceCache()
    lf = fused.train_frame(d_r, d_t, s, l, seed).cpu().numpy()
    cache = nrc.RadianceCache()
    frame = nrc.DataParallelFrame(cache, device=torch.device("cuda", 0))
    ld = torch.zeros(s, dtype=torch.float32, device="cuda")
    frame.train_frame(d_r, d_t, s, l, seed, ld)
    ld = ld.cpu().numpy()
    assert frame.last_launch_count == 3 * s  # train + reduce, adam per step
    np.testing.assert_allclose(ld, lf, rtol=1e-4)
    q = torch.from_numpy(nrc_inputs.records(4096, seed=3)).cuda()
    assert max(radiance_err(cache.query(q).cpu().numpy(), fused.query(q).cpu().numpy())) <= TOL_RADIANCE
    # oracle on the gathered batches: per-step losses (C3 criterion) and radiance
    pa, pc, pm = orc.lcg_params(n, seed)
    perm = orc.lcg_permute(n, pa, pc, pm).astype(np.int64)
    ref = orc.OracleCache(W32=nrc.RadianceCache().get_params("train"))
    lo = []
    for j in range(s):
        idx = perm[j * l:(j + 1) * l]
        lo.append(ref.train_step(recs[idx], tg[idx]))
    np.testing.assert_allclose(ld, lo, rtol=1e-2)
    assert max(radiance_err(cache.query(q).cpu().numpy(), ref.query(q.cpu().numpy()))) <= TOL_RADIANCE


def test_replicated_frame_world1_equals_train_frame(group):
    """N3 variant (i) through NCCL (world size 1: the all-gather is a copy):
    bitwise equal to nrc_train_frame on the same records."""
    import paper_2106_12372_b200 as nrc
    n, s, l, seed = 8192, 4, 2048, 23
    recs, tg = nrc_inputs.train_frame(3, n=n, noise=0.3)
    d_r = torch.from_numpy(recs).cuda()
    d_t = torch.from_numpy(tg).cuda()
    a, b = nrc.RadianceCache(), nrc.RadianceCache()
    la = a.train_frame(d_r, d_t, s, l, seed).cpu().numpy()
    frame = nrc.DataParallelFrame(b, device=torch.device("cuda", 0))
    lb = torch.zeros(s, dtype=torch.float32, device="cuda")
    frame.train_frame_replicated(d_r, d_t, s, l, seed, lb)
    np.testing.assert_array_equal(lb.cpu().numpy(), la)
    np.testing.assert_array_equal(b.get_params("train"), a.get_params("train"))
    np.testing.assert_array_equal(b.get_params("ema"), a.get_params("ema"))


def test_nvls_frame_world1_equals_dp_frame(group):
    """SURVEY N3 (ii), the all-reduce in the NVSwitch (multimem.ld_reduce into
    the optimiser, nrc_train_apply_multimem + nrc_peer_barrier over torch
    symmetric memory): with one rank the switch sum is the rank's own buffer,
    so the frame equals the NCCL data-parallel frame bitwise; both match the
    single-GPU frame's losses.  Skipped where the system has no multicast."""
    import paper_2106_12372_b200 as nrc
    n, s, l, seed = 8192 + 3, 4, 2048, 29
    recs, tg = nrc_inputs.train_frame(4, n=n, noise=0.3)
    d_r = torch.from_numpy(recs).cuda()
    d_t = torch.from_numpy(tg).cuda()
    a, b = nrc.RadianceCache(), nrc.RadianceCache()
    fa = nrc.DataParallelFrame(a, device=torch.device("cuda", 0))
    fb = nrc.DataParallelFrame(b, device=torch.device("cuda", 0))
    la = torch.zeros(s, dtype=torch.float32, device="cuda")
    lb = torch.zeros(s, dtype=torch.float32, device="cuda")
    try:
        fb.train_frame_allreduce_nvls(d_r, d_t, s, l, seed, lb)
    except RuntimeError as e:
        if "multicast" in str(e).lower():
            pytest.skip(str(e))
        raise
    fa.train_frame(d_r, d_t, s, l, seed, la)
    fb.train_frame_allreduce_nvls(d_r, d_t, s, l, seed + 1, lb)
    fa.train_frame(d_r, d_t, s, l, seed + 1, la)  # a second frame: the other buffer parity
    np.testing.assert_array_equal(lb.cpu().numpy(), la.cpu().numpy())
    np.testing.assert_array_equal(b.get_params("train"), a.get_params("train"))
    np.testing.assert_array_equal(b.get_params("ema"), a.get_params("ema"))
    assert b.dp_timeouts() == 0
    assert fb.last_launch_count == 4 * s  # partials + reduce, barrier, optimiser per step


def test_sym_frame_world1_equals_dp_frame(group):
    """The all-reduce folded into the optimiser over peer memory
    (nrc_train_apply_peers + nrc_peer_barrier over torch symmetric memory):
    with one rank the rank-order sum is the rank's own reduced gradient, so the
    frame equals the NCCL data-parallel frame bitwise (two frames: both buffer
    parities)."""
    import paper_2106_12372_b200 as nrc
    n, s, l, seed = 8192 + 3, 4, 2048, 31
    recs, tg = nrc_inputs.train_frame(5, n=n, noise=0.3)
    d_r = torch.from_numpy(recs).cuda()
    d_t = torch.from_numpy(tg).cuda()
    a, b = nrc.RadianceCache(), nrc.RadianceCache()
    fa = nrc.DataParallelFrame(a, device=torch.device("cuda", 0))
    fb = nrc.DataParallelFrame(b, device=torch.device("cuda", 0))
    la = torch.zeros(s, dtype=torch.float32, device="cuda")
    lb = torch.zeros(s, dtype=torch.float32, device="cuda")
    for f in range(2):
        fa.train_frame(d_r, d_t, s, l, seed + f, la)
        fb.train_frame_allreduce_sym(d_r, d_t, s, l, seed + f, lb)
    np.testing.assert_array_equal(lb.cpu().numpy(), la.cpu().numpy())
    np.testing.assert_array_equal(b.get_params("train"), a.get_params("train"))
    np.testing.assert_array_equal(b.get_params("ema"), a.get_params("ema"))
    assert b.dp_timeouts() == 0
    assert fb.last_launch_count == 4 * s  # partials + reduce, barrier, optimiser per step
