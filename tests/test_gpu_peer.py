"""Peer-memory frame training (nrc_train_frame_parts): two
processes on one GPU exchange CUDA IPC handles of their record buffers and
each trains the whole frame by gathering rows straight from the owner's
memory.  Both must end bitwise equal to single-process nrc_train_frame on the
concatenated records (the same kernels read the same rows in the same
order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nrc_inputs

pytestmark = pytest.mark.gpu

N_PER, S, L, SEEDS = 8192, 4, 4096, (31, 32)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import paper_2106_12372_b200 as nrc
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        recs, tg = nrc_inputs.train_frame(2, n=world * N_PER, noise=0.3)
        lo, hi = rank * N_PER, (rank + 1) * N_PER
        d_r = torch.from_numpy(recs[lo:hi].copy()).cuda()
        d_t = torch.from_numpy(tg[lo:hi].copy()).cuda()
        cache = nrc.RadianceCache()
        frame = nrc.DataParallelFrame(cache, device=torch.device("cuda", 0))
        losses = []
        for seed in SEEDS:
            lz = torch.zeros(S, dtype=torch.float32, device="cuda")
            frame.train_frame_peer(d_r, d_t, S, L, seed, lz)
            losses.append(lz.cpu().numpy())
        torch.cuda.synchronize()
        dist.barrier()  # peers finished reading before the buffers go away
        np.savez(os.path.join(out_dir, f"peer{rank}.npz"), w=cache.get_params("train"), e=cache.get_params("ema"),
                 losses=np.stack(losses))
    finally:
        dist.destroy_process_group()


def test_peer_training_two_processes_one_gpu(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as nrc
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"peer{r}.npz") for r in range(world)]
    recs, tg = nrc_inputs.train_frame(2, n=world * N_PER, noise=0.3)
    ref = nrc.RadianceCache()
    ref_losses = [ref.train_frame(torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda(), S, L, s).cpu().numpy()
                  for s in SEEDS]
    for r in res:
        np.testing.assert_array_equal(r["w"], ref.get_params("train"))
        np.testing.assert_array_equal(r["e"], ref.get_params("ema"))
        np.testing.assert_array_equal(r["losses"], np.stack(ref_losses))
