"""Data-parallel training with the gradient all-reduce fused into the
optimiser over peer memory (nrc_train_frame_dp_peer; SURVEY 8(e) mitigation
2, 8(f) N3 (ii)).  Every rank computes the per-tile partials of its share of
each batch's 128-row tiles; every rank's optimiser reduces all tiles in tile
order from the owners' arenas.  The result must be BITWISE equal to
single-GPU nrc_train_frame (same tiles, same partials, same order): checked
in-process at world 1 and with two processes sharing one GPU through real
CUDA IPC mappings and system-scope hand-off counters."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nrc_inputs

pytestmark = pytest.mark.gpu

N, FRAMES = 16384, ((4, 4096, 31), (2, 3000, 32), (1, 16384, 33))  # (s, l, seed); l = 3000 has a ragged tile


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _reference(nrc, hw=64):
    recs, tg = nrc_inputs.train_frame(4, n=N, noise=0.3)
    ref = nrc.RadianceCache(nrc.Config(hidden_width=hw))
    d_r, d_t = torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda()
    losses = [ref.train_frame(d_r, d_t, s, l, seed).cpu().numpy() for s, l, seed in FRAMES]
    return ref, losses


@pytest.mark.parametrize("hw", [64, 32])
def test_dp_peer_world1_bitwise_equals_train_frame(hw):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as nrc
    ref, ref_losses = _reference(nrc, hw)
    recs, tg = nrc_inputs.train_frame(4, n=N, noise=0.3)
    c = nrc.RadianceCache(nrc.Config(hidden_width=hw))
    d_r, d_t = torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda()
    for (s, l, seed), lr in zip(FRAMES, ref_losses):
        lz = c.train_frame_dp_peer(d_r, d_t, s, l, seed, 0, 1, [c.state_ptr]).cpu().numpy()
        np.testing.assert_array_equal(lz[:s], lr[:s])
    np.testing.assert_array_equal(c.get_params("train"), ref.get_params("train"))
    np.testing.assert_array_equal(c.get_params("ema"), ref.get_params("ema"))
    assert c.stats()["step"] == ref.stats()["step"] and c.dp_timeouts() == 0


def test_dp_peer_argument_checks():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as nrc
    c = nrc.RadianceCache()
    recs, tg = nrc_inputs.train_frame(4, n=1024)
    d_r, d_t = torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda()
    with pytest.raises(nrc.NRCError, match="INVALID"):
        c.train_frame_dp_peer(d_r, d_t, 1, 512, 1, 1, 1, [c.state_ptr])  # rank >= world
    with pytest.raises(nrc.NRCError, match="INVALID"):
        c.train_frame_dp_peer(d_r, d_t, 1, 512, 1, 0, 1, [c.state_ptr + 256])  # not this arena
    big, bt = nrc_inputs.train_frame(4, n=20000)
    with pytest.raises(nrc.NRCError, match="UNSUPPORTED"):
        c.train_frame_dp_peer(torch.from_numpy(big).cuda(), torch.from_numpy(bt).cuda(), 1, 20000, 1, 0, 1,
                              [c.state_ptr])  # 157 tiles per step


def _worker(rank, world, port, out_dir):
    import paper_2106_12372_b200 as nrc
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        recs, tg = nrc_inputs.train_frame(4, n=N, noise=0.3)
        d_r, d_t = torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda()
        cache = nrc.RadianceCache()
        frame = nrc.DataParallelFrame(cache, device=torch.device("cuda", 0))
        losses = []
        for s, l, seed in FRAMES:
            lz = torch.zeros(4, dtype=torch.float32, device="cuda")
            frame.train_frame_allreduce_peer(d_r, d_t, s, l, seed, lz)
            losses.append(lz.cpu().numpy()[:s])
        torch.cuda.synchronize()
        dist.barrier()  # peers finished reading this arena
        np.savez(os.path.join(out_dir, f"dp{rank}.npz"), w=cache.get_params("train"), e=cache.get_params("ema"),
                 losses=np.concatenate(losses), timeouts=cache.dp_timeouts())
    finally:
        dist.destroy_process_group()


def test_dp_peer_two_processes_one_gpu_bitwise(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as nrc
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ref, ref_losses = _reference(nrc)
    want = np.concatenate([lr[:s] for (s, _, _), lr in zip(FRAMES, ref_losses)])
    for r in range(world):
        res = np.load(tmp_path / f"dp{r}.npz")
        assert int(res["timeouts"]) == 0
        np.testing.assert_array_equal(res["w"], ref.get_params("train"))
        np.testing.assert_array_equal(res["e"], ref.get_params("ema"))
        np.testing.assert_array_equal(res["losses"], want)
