"""Dedicated multi-GPU mode: rank 0 runs each frame's
training, the other ranks query their row shards with the previous frame's
W-bar, then rank 0's query image is broadcast.  Two processes sharing one GPU
(gloo for the broadcast): rank 1's query of every frame and both ranks' final
query images must equal the single-process frame sequence bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nrc_inputs

pytestmark = pytest.mark.gpu

NQ, S, L, FRAMES = 50_000, 4, 2048, 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import paper_2106_12372_b200 as nrc
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cache = nrc.RadianceCache()
        frame = nrc.DataParallelFrame(cache, device=torch.device("cuda", 0))
        q = nrc_inputs.records(NQ, seed=81)
        q0, q1 = frame.dedicated_query_rows(NQ)
        dq = torch.from_numpy(q[q0:q1].copy()).cuda()
        outs = []
        for f in range(FRAMES):
            recs, tg = nrc_inputs.train_frame(f, n=S * L, noise=0.3)
            rgb = torch.empty((q1 - q0, 3), dtype=torch.float32, device="cuda")
            frame.frame_dedicated(dq, rgb, torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda(), S, L, 40 + f)
            outs.append(rgb.cpu().numpy())
        torch.cuda.synchronize()
        np.savez(os.path.join(out_dir, f"ded{rank}.npz"), img=cache.query_image().cpu().numpy(),
                 rgb=np.stack(outs), q0=q0, q1=q1)
    finally:
        dist.destroy_process_group()


def test_dedicated_two_processes_one_gpu(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2106_12372_b200 as nrc
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"ded{r}.npz") for r in range(world)]
    ref = nrc.RadianceCache()
    q = torch.from_numpy(nrc_inputs.records(NQ, seed=81)).cuda()
    want = []
    for f in range(FRAMES):
        want.append(ref.query(q).cpu().numpy())
        recs, tg = nrc_inputs.train_frame(f, n=S * L, noise=0.3)
        ref.train_frame(torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda(), S, L, 40 + f)
    assert int(res[1]["q0"]) == 0 and int(res[1]["q1"]) == NQ
    np.testing.assert_array_equal(res[1]["rgb"], np.stack(want))
    img = ref.query_image().cpu().numpy()
    for r in res:
        np.testing.assert_array_equal(r["img"], img)
