"""Multi-process (gloo, world_size 2, CPU) tests of the N > 1 partitioning in
paper_2106_12372_b200.dp: query row shards, per-rank rows of each LCG-shuffled
batch, one all-reduce of [gradient | loss] per step, identical Adam + EMA on
every rank.  The per-rank compute is a test-side stand-in built on the fp64
oracle (no GPU here); what is under test is the orchestration the bench runs
for N > 1, against single-process oracle training on the gathered batches
(P:L487-491 shuffle into s batches of l; Adam P:L896-902; EMA Eq. 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nrc_inputs
import oracle
from paper_2106_12372_b200 import dp


def test_shard_partition():
    for n in [0, 1, 2, 7, 1000, 16384, 2073600]:
        for world in [1, 2, 3, 4, 8]:
            spans = [dp.shard(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        dp.shard(10, 2, 2)


def test_frame_batches_shrink():
    assert dp.frame_batches(65536, 4, 16384) == (4, 16384)
    assert dp.frame_batches(65535, 4, 16384) == (4, 16383)  # batches shrink proportionally
    assert dp.frame_batches(3, 4, 16384) == (0, 0)
    assert dp.frame_batches(0, 4, 16384) == (0, 0)


class OracleShard:
    """Test stand-in for RadianceCache's data-parallel calls, on the oracle."""

    def __init__(self, seed):
        self.oc = oracle.OracleCache(seed=seed)

    def train_frame_backward(self, records, targets, l, seed, j, lo, hi, grad, loss_sum):
        recs, tg = records.numpy(), targets.numpy()
        a, c, m = oracle.lcg_params(recs.shape[0], seed)
        perm = oracle.lcg_permute(recs.shape[0], a, c, m).astype(np.int64)
        idx = perm[j * l + lo: j * l + hi]
        G, ls, _ = oracle.grad_batch(self.oc.w, recs[idx], tg[idx])
        grad.copy_(torch.from_numpy(G))
        loss_sum[0] = ls

    def train_apply(self, grad_sum, n, loss_sum=None, loss=None):
        oc = self.oc
        oc.t += 1
        oracle.adam(oc.w, oc.m, oc.v, grad_sum.numpy().astype(np.float64) / n, oc.t)
        oracle.ema(oc.wbar, oc.w, oc.t)
        if loss_sum is not None and loss is not None:  # nrc_train_apply's batch-mean loss (R10)
            loss[0] = loss_sum[0] / n

    def train_frame(self, records, targets, s, l, seed, losses=None):
        recs, tg = records.numpy(), targets.numpy()
        s, l = dp.frame_batches(recs.shape[0], s, l)
        a, c, m = oracle.lcg_params(recs.shape[0], seed)
        perm = oracle.lcg_permute(recs.shape[0], a, c, m).astype(np.int64)
        for j in range(s):
            idx = perm[j * l:(j + 1) * l]
            lj = self.oc.train_step(recs[idx], tg[idx])
            if losses is not None:
                losses[j] = lj
        return losses

    def query(self, records, out, stream=None):
        out.copy_(torch.from_numpy(self.oc.query(records.numpy())))
        return out

    def get_params(self, which="train"):
        return (self.oc.w if which == "train" else self.oc.wbar).astype(np.float32)


N_TOTAL, S, L, SEED = 3 * 1001 + 5, 3, 1001, 77


def _worker(rank, world, port, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        recs, tgts = nrc_inputs.train_frame(0, n=N_TOTAL, noise=0.3)
        shard_cache = OracleShard(seed=5)
        frame = dp.DataParallelFrame(shard_cache, dtype=torch.float64)
        losses = torch.zeros(S, dtype=torch.float64)
        frame.train_frame(torch.from_numpy(recs), torch.from_numpy(tgts), S, L, SEED, losses)
        q = nrc_inputs.records(999, seed=nrc_inputs.SEED_QUERY)
        q0, q1 = frame.query_rows(q.shape[0])
        rgb = torch.zeros((q1 - q0, 3), dtype=torch.float64)
        frame.query(torch.from_numpy(q[q0:q1].copy()), rgb)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), w=shard_cache.oc.w, wbar=shard_cache.oc.wbar,
                 losses=losses.numpy(), rgb=rgb.numpy(), q0=q0, q1=q1)
    finally:
        dist.destroy_process_group()


def _worker_replicated(rank, world, port, out_dir, n_total, pass_counts=False):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        recs, tgts = nrc_inputs.train_frame(0, n=n_total, noise=0.3)
        lo, hi = dp.shard(n_total, rank, world)  # this rank's screen region's records
        shard_cache = OracleShard(seed=5)
        frame = dp.DataParallelFrame(shard_cache, dtype=torch.float64)
        losses = torch.zeros(S, dtype=torch.float64)
        frame.verify_replicas()  # identical seeded init on every rank
        counts = [b - a for a, b in (dp.shard(n_total, r, world) for r in range(world))] if pass_counts else None
        frame.train_frame_replicated(torch.from_numpy(recs[lo:hi].copy()), torch.from_numpy(tgts[lo:hi].copy()),
                                     S, L, SEED, losses, counts=counts)
        frame.verify_replicas()  # and bitwise identical after the replicated frame
        np.savez(os.path.join(out_dir, f"rep{rank}.npz"), w=shard_cache.oc.w, losses=losses.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_data_parallel_frame_equals_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    # single process: s oracle steps on the gathered batches
    recs, tgts = nrc_inputs.train_frame(0, n=N_TOTAL, noise=0.3)
    a, c, m = oracle.lcg_params(N_TOTAL, SEED)
    perm = oracle.lcg_permute(N_TOTAL, a, c, m).astype(np.int64)
    ref = oracle.OracleCache(seed=5)
    ref_losses = []
    for j in range(S):
        idx = perm[j * L:(j + 1) * L]
        ref_losses.append(ref.train_step(recs[idx], tgts[idx]))
    for r in res:
        # identical state on every rank, equal to the single-process result up to
        # fp64 summation order of the two shard gradients
        np.testing.assert_allclose(r["w"], ref.w, rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(r["wbar"], ref.wbar, rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(r["losses"], ref_losses, rtol=1e-12)
    np.testing.assert_array_equal(res[0]["w"], res[1]["w"])
    # query shards tile the batch and match the unsharded query
    q = nrc_inputs.records(999, seed=nrc_inputs.SEED_QUERY)
    assert int(res[0]["q0"]) == 0 and int(res[0]["q1"]) == int(res[1]["q0"]) and int(res[1]["q1"]) == 999
    full = ref.query(q)
    got = np.concatenate([res[0]["rgb"], res[1]["rgb"]])
    np.testing.assert_allclose(got, full, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("world,N,pass_counts", [(2, 3 * 1000 + 6, False), (3, 3 * 1001 + 5, True),
                                                 (3, 3 * 1001 + 5, False)])
def test_replicated_frame_after_allgather(tmp_path, world, N, pass_counts):
    """N3 variant (i): one all-gather of the frame's records per frame, then
    replicated training: every rank ends bitwise identical and equal to the
    single-process training on the gathered (rank-ordered) records -- also
    when the record count does not divide by the world size (3,008 over 3
    ranks: parts padded for the collective, padding dropped), with the counts
    exchanged or passed by the caller."""
    mp.spawn(_worker_replicated, args=(world, _free_port(), str(tmp_path), N, pass_counts), nprocs=world, join=True)
    res = [np.load(tmp_path / f"rep{r}.npz") for r in range(world)]
    for r in range(1, world):
        np.testing.assert_array_equal(res[0]["w"], res[r]["w"])
    recs, tgts = nrc_inputs.train_frame(0, n=N, noise=0.3)
    ref = OracleShard(seed=5)
    ref_losses = torch.zeros(S, dtype=torch.float64)
    ref.train_frame(torch.from_numpy(recs), torch.from_numpy(tgts), S, L, SEED, ref_losses)
    np.testing.assert_array_equal(res[0]["w"], ref.oc.w)
    np.testing.assert_array_equal(res[0]["losses"], ref_losses.numpy())


class ArenaRecorder:
    """Stand-in cache for the fused peer all-reduce orchestration: records
    the arena list nrc_train_frame_dp_peer would receive."""

    def __init__(self, rank):
        self.state_ptr = 0x10000 * (rank + 1)
        self.calls = []

    def train_frame_dp_peer(self, records, targets, s, l, seed, rank, world, peer_states, losses=None):
        self.calls.append((s, l, seed, rank, world, list(peer_states)))
        return losses


def _worker_arena(rank, world, port, out_dir):
    import paper_2106_12372_b200.nrc as nrcmod
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # CUDA IPC stand-ins: a "handle" names the exporting address; an
        # imported mapping is that address + 1 (a different virtual address)
        nrcmod.ipc_export_ptr = lambda ptr: (b"%d" % ptr, 0)
        nrcmod.ipc_import = lambda handle, off: int(handle) + 1 + off
        cache = ArenaRecorder(rank)
        frame = dp.DataParallelFrame(cache)
        recs = torch.zeros((8, 16))
        for seed in (1, 2):  # the exchange happens once
            frame.train_frame_allreduce_peer(recs, torch.zeros((8, 3)), 2, 4, seed)
        np.save(os.path.join(out_dir, f"arena{rank}.npy"), np.array(cache.calls, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_allreduce_peer_arena_exchange(tmp_path):
    """train_frame_allreduce_peer: every rank passes one arena per rank in
    rank order -- its own address at its index, the peers' mapped addresses
    elsewhere -- with its rank and the world size, exchanged once."""
    world = 2
    mp.spawn(_worker_arena, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        calls = np.load(tmp_path / f"arena{r}.npy", allow_pickle=True)
        assert len(calls) == 2
        for (s, l, seed, rank, w, peers), want_seed in zip(calls, (1, 2)):
            assert (s, l, seed, rank, w) == (2, 4, want_seed, r, world)
            assert peers == [0x10000 * (k + 1) + (0 if k == r else 1) for k in range(world)]


def _worker_diverged(rank, world, port, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        frame = dp.DataParallelFrame(OracleShard(seed=5 + rank))  # different init on each rank
        try:
            frame.verify_replicas()
            raised = False
        except RuntimeError:
            raised = True
        np.save(os.path.join(out_dir, f"div{rank}.npy"), np.array([raised]))
    finally:
        dist.destroy_process_group()


def test_verify_replicas_detects_divergence(tmp_path):
    """Negative control: replicas with different initial weights are reported."""
    world = 2
    mp.spawn(_worker_diverged, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert bool(np.load(tmp_path / f"div{r}.npy")[0])
