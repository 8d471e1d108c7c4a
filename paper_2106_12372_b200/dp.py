"""Multi-GPU partitioning of the NRC frame.

One process per GPU.  Queries are independent rows: rank k of P
takes rows [k N / P, (k + 1) N / P) and nothing is exchanged.  Training is
data-parallel: every rank holds the full 20,672-parameter state, computes the
un-normalised gradient sum over its l / P rows of each LCG-shuffled batch
 with nrc_train_frame_backward, one all-reduce (SUM) of
[gradient | loss sum] per step, then identical Adam + EMA on every rank
(nrc_train_apply with n_global = l).  The result equals the single-GPU step up
to the fp32 summation order of the gradient.

This module is host orchestration only: every arithmetic step runs in the
cache's CUDA kernels (or, in the CPU tests, in a test-side stand-in).
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist

from .nrc import NPARAM


def shard(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Rows [lo, hi) of n owned by `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return rank * n // world, (rank + 1) * n // world


def frame_batches(n_total: int, s: int, l: int) -> Tuple[int, int]:
    """(s, l) actually trained on: batches shrink proportionally when the frame
    has fewer than s * l records, as nrc_train_frame does."""
    if n_total == 0 or s == 0 or l == 0:
        return 0, 0
    if s * l > n_total:
        l = n_total // s
    return (s, l) if l > 0 else (0, 0)


class DataParallelFrame:
    """The N > 1 frame: sharded query + data-parallel training.

    `cache` provides query / train_frame_backward / train_apply with the
    signatures of paper_2106_12372_b200.RadianceCache.  `group` is the
    process group (NCCL on GPUs; gloo in the CPU tests)."""

    def __init__(self, cache, group: Optional[dist.ProcessGroup] = None, device=None,
                 dtype: torch.dtype = torch.float32):
        self.cache = cache
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cpu")
        # one buffer so that gradient and loss travel in a single all-reduce
        self.buf = torch.zeros(NPARAM + 1, dtype=dtype, device=self.device)
        self.grad = self.buf[:NPARAM]
        self.loss_sum = self.buf[NPARAM:]
        self.last_launch_count = 0

    def replica_checksum(self, image_only: bool = False) -> int:
        """CRC32 of this rank's fp32 training and EMA parameters (host copy), or
        of the fp16 image the query reads (image_only: the state a query-only
        rank of the dedicated mode keeps in sync)."""
        import zlib
        if image_only:
            return zlib.crc32(self.cache.query_image().cpu().numpy().tobytes())
        w = self.cache.get_params("train")
        e = self.cache.get_params("ema")
        return zlib.crc32(w.tobytes() + e.tobytes())

    def dedicated_query_rows(self, n: int, share0: float = 0.0) -> Tuple[int, int]:
        """Dedicated mode: rank 0 trains and queries the first round(share0 n)
        rows (0 by default; a small share balances P = 2, where the single
        query rank would otherwise wait longest); ranks 1..P-1 split the rest."""
        n0 = int(round(min(max(share0, 0.0), 1.0) * n))
        if self.rank == 0:
            return 0, n0
        lo, hi = shard(n - n0, self.rank - 1, self.world - 1)
        return n0 + lo, n0 + hi

    @staticmethod
    def dedicated_share0(query_time_one_gpu: float, train_time: float, world: int) -> float:
        """Rank 0's query share that equalises t_train + f T_q (rank 0) with
        (1 - f) T_q / (P - 1) (the other ranks); 0 when the training alone is
        the longer part (P >= 3 at the paper's sizes)."""
        if world < 2 or query_time_one_gpu <= 0:
            return 0.0
        f = (query_time_one_gpu - (world - 1) * train_time) / (world * query_time_one_gpu)
        return float(min(max(f, 0.0), 0.9))

    def frame_dedicated(self, records_query_local: torch.Tensor, out: torch.Tensor, records: torch.Tensor,
                        targets: torch.Tensor, s: int, l: int, shuffle_seed: int,
                        losses: Optional[torch.Tensor] = None, stream=None):
        """One frame with the work split by function: rank 0
        runs the whole frame's training (the latency-bound part, which more
        GPUs cannot shorten), ranks 1..P-1 run the frame's query on their row
        shards with the previous frame's W-bar -- the order of the paper's frame
        (the query reads W-bar from before this frame's training) --
        and then rank 0's new query image is broadcast to every rank.  Results
        equal the single-GPU frame sequence bitwise (same kernels, same data)."""
        if self.world < 2:
            raise ValueError("the dedicated mode needs at least two ranks")
        launches = 0
        if records_query_local.shape[0] > 0:  # the previous frame's W-bar
            self.cache.query(records_query_local, out, stream=stream)
            launches += getattr(self.cache, "last_launch_count", 0)
        if self.rank == 0:
            self.cache.train_frame(records, targets, s, l, shuffle_seed, losses)
            launches += getattr(self.cache, "last_launch_count", 0)
        dist.broadcast(self.cache.query_image(), src=0, group=self.group)
        self.last_launch_count = launches
        return out

    def verify_replicas(self, image_only: bool = False) -> int:
        """every rank holds a bitwise-identical replica (same seeded
        init, identical reduced gradients or identical gathered data, the same
        deterministic kernels).  Gathers every rank's checksum and raises if
        any differs; returns the common checksum."""
        mine = self.replica_checksum(image_only)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=self.group)
        if any(c != mine for c in everyone):
            raise RuntimeError(f"replicas diverged: checksums {everyone}")
        return mine

    def query_rows(self, n: int) -> Tuple[int, int]:
        return shard(n, self.rank, self.world)

    def query(self, records_local: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
        """This rank's rows of the frame's query (no communication)."""
        return self.cache.query(records_local, out, stream=stream)

    def train_frame_replicated(self, records_local: torch.Tensor, targets_local: torch.Tensor, s: int, l: int,
                               shuffle_seed: int, losses: Optional[torch.Tensor] = None) -> Optional[torch.Tensor]:
        """SURVEY 8(f) N3 variant (i): each rank owns the training records of its
        screen region; one all-gather per frame (rank order) assembles the
        frame's records on every rank, then every rank runs the whole frame's
        training (fused nrc_train_frame) on identical data -- bitwise-identical
        replicas with no per-step collective (the kernels are deterministic).
        Every rank must pass the same number of records."""
        n_loc = int(records_local.shape[0])
        rec = torch.empty((n_loc * self.world, records_local.shape[1]), dtype=records_local.dtype,
                          device=records_local.device)
        tgt = torch.empty((n_loc * self.world, 3), dtype=targets_local.dtype, device=targets_local.device)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(rec, records_local.contiguous(), group=self.group)
            dist.all_gather_into_tensor(tgt, targets_local.contiguous(), group=self.group)
        else:  # gloo (CPU tests): list form
            dist.all_gather(list(rec.chunk(self.world)), records_local.contiguous(), group=self.group)
            dist.all_gather(list(tgt.chunk(self.world)), targets_local.contiguous(), group=self.group)
        out = self.cache.train_frame(rec, tgt, s, l, shuffle_seed, losses)
        self.last_launch_count = getattr(self.cache, "last_launch_count", 0)
        return out

    def train_frame_peer(self, records_local: torch.Tensor, targets_local: torch.Tensor, s: int, l: int,
                         shuffle_seed: int, losses: Optional[torch.Tensor] = None,
                         parts_ready: bool = False) -> Optional[torch.Tensor]:
        """SURVEY 8(f) N3, the all-gather fused into the training kernel: every
        rank exports its record / target buffers once (CUDA IPC handles over
        the process group), maps the peers', and nrc_train_frame_parts reads
        each shuffled batch row from its owner's memory (NVLink loads).  No
        collective per frame; bitwise the same result as train_frame_replicated.
        The caller keeps the local buffers alive and unchanged across the call
        on every rank (here: a barrier before the kernel, skipped with
        parts_ready=True when the caller already knows every part is final,
        e.g. buffers written once and synchronised at setup)."""
        from .nrc import ipc_export, ipc_import
        key = (records_local.data_ptr(), targets_local.data_ptr(), int(records_local.shape[0]))
        self._peer_cache = getattr(self, "_peer_cache", {})
        if key not in self._peer_cache:
            mine = (ipc_export(records_local), ipc_export(targets_local), int(records_local.shape[0]))
            everyone = [None] * self.world
            dist.all_gather_object(everyone, mine, group=self.group)
            if any(e[2] != mine[2] for e in everyone):
                raise ValueError("every rank must hold the same number of records")
            self._peer_maps = getattr(self, "_peer_maps", {})
            rec_ptrs, tgt_ptrs = [], []
            for r, (rh, th, _) in enumerate(everyone):
                if r == self.rank:
                    rec_ptrs.append(records_local.data_ptr())
                    tgt_ptrs.append(targets_local.data_ptr())
                    continue
                for hnd, lst in ((rh, rec_ptrs), (th, tgt_ptrs)):
                    if hnd not in self._peer_maps:
                        self._peer_maps[hnd] = ipc_import(*hnd)
                    lst.append(self._peer_maps[hnd])
            self._peer_cache[key] = (rec_ptrs, tgt_ptrs)
        if not parts_ready:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)  # every part is complete
        rec_ptrs, tgt_ptrs = self._peer_cache[key]
        out = self.cache.train_frame_parts(rec_ptrs, tgt_ptrs, int(records_local.shape[0]), s, l, shuffle_seed,
                                           losses)
        self.last_launch_count = getattr(self.cache, "last_launch_count", 0)
        return out

    def train_frame_allreduce_peer(self, records: torch.Tensor, targets: torch.Tensor, s: int, l: int,
                                   shuffle_seed: int, losses: Optional[torch.Tensor] = None) -> Optional[torch.Tensor]:
        """SURVEY 8(e) mitigation 2 / 8(f) N3 (ii): data-parallel training with
        the per-step gradient all-reduce fused into the optimiser kernel over
        peer memory (nrc_train_frame_dp_peer): every rank computes the partials
        of its share of each batch's 128-row tiles, then every rank's optimiser
        reads all ranks' partials in tile order (NVLink loads) -- no NCCL call,
        bitwise equal to single-GPU nrc_train_frame.  Records replicated on
        every rank (as in train_frame).  The state arenas are exchanged once
        (CUDA IPC over the process group)."""
        from .nrc import ipc_export_ptr, ipc_import
        if getattr(self, "_arena_ptrs", None) is None:
            mine = ipc_export_ptr(self.cache.state_ptr)
            everyone = [None] * self.world
            dist.all_gather_object(everyone, mine, group=self.group)
            self._arena_ptrs = [self.cache.state_ptr if r == self.rank else ipc_import(*everyone[r])
                                for r in range(self.world)]
            if torch.cuda.is_available():
                torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)  # every arena is initialised before any peer writes to it
        out = self.cache.train_frame_dp_peer(records, targets, s, l, shuffle_seed, self.rank, self.world,
                                             self._arena_ptrs, losses)
        self.last_launch_count = getattr(self.cache, "last_launch_count", 0)
        return out

    def train_frame(self, records: torch.Tensor, targets: torch.Tensor, s: int, l: int, shuffle_seed: int,
                    losses: Optional[torch.Tensor] = None) -> Optional[torch.Tensor]:
        """All s steps of the frame's training on the full (replicated) record
        set; each rank gathers only its rows of every shuffled batch."""
        n_total = int(records.shape[0])
        s, l = frame_batches(n_total, s, l)
        launches = 0
        if s == 0:
            self.last_launch_count = 0
            return losses
        lo, hi = shard(l, self.rank, self.world)
        for j in range(s):
            self.cache.train_frame_backward(records, targets, l, shuffle_seed, j, lo, hi, self.grad, self.loss_sum)
            launches += getattr(self.cache, "last_launch_count", 0)
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)
            self.cache.train_apply(self.grad, l)
            launches += getattr(self.cache, "last_launch_count", 0)
            if losses is not None:
                losses[j] = self.loss_sum[0] / l
        self.last_launch_count = launches
        return losses
