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

    def replica_checksum(self) -> int:
        """CRC32 of this rank's fp32 training and EMA parameters (host copy)."""
        import zlib
        w = self.cache.get_params("train")
        e = self.cache.get_params("ema")
        return zlib.crc32(w.tobytes() + e.tobytes())

    def verify_replicas(self) -> int:
        """every rank holds a bitwise-identical replica (same seeded
        init, identical reduced gradients or identical gathered data, the same
        deterministic kernels).  Gathers every rank's checksum and raises if
        any differs; returns the common checksum."""
        mine = self.replica_checksum()
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
                               shuffle_seed: int, losses: Optional[torch.Tensor] = None,
                               counts=None) -> Optional[torch.Tensor]:
        """SURVEY 8(f) N3 variant (i): each rank owns the training records of its
        screen region; one all-gather per frame assembles the frame's records
        in rank order on every rank, then every rank runs the whole frame's
        training (nrc_train_frame) on identical data -- bitwise-identical
        replicas with no per-step collective (the kernels are deterministic).
        Ranks may hold different record counts (e.g. 65,536 over 3 ranks): the
        counts are exchanged, every part is padded to the largest for the
        collective, and the padding is dropped before training.  `counts`
        (every rank's record count, identical on all ranks -- e.g. from the
        screen partition) skips the count exchange."""
        n_loc = int(records_local.shape[0])
        counts = self._counts(n_loc) if counts is None else [int(c) for c in counts]
        if len(counts) != self.world or counts[self.rank] != n_loc:
            raise ValueError(f"counts {counts} do not match this rank's {n_loc} records")
        nmax = max(counts)
        nrec = records_local.shape[1]
        if n_loc < nmax:  # pad to the collective's common size (dropped below)
            pad_r = torch.zeros((nmax - n_loc, nrec), dtype=records_local.dtype, device=records_local.device)
            pad_t = torch.zeros((nmax - n_loc, 3), dtype=targets_local.dtype, device=targets_local.device)
            records_local = torch.cat([records_local, pad_r])
            targets_local = torch.cat([targets_local, pad_t])
        rec = torch.empty((nmax * self.world, nrec), dtype=records_local.dtype, device=records_local.device)
        tgt = torch.empty((nmax * self.world, 3), dtype=targets_local.dtype, device=targets_local.device)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(rec, records_local.contiguous(), group=self.group)
            dist.all_gather_into_tensor(tgt, targets_local.contiguous(), group=self.group)
        else:  # gloo (CPU tests): list form
            dist.all_gather(list(rec.chunk(self.world)), records_local.contiguous(), group=self.group)
            dist.all_gather(list(tgt.chunk(self.world)), targets_local.contiguous(), group=self.group)
        if min(counts) != nmax:  # drop the padding, keep rank order
            rec = torch.cat([rec[r * nmax:r * nmax + c] for r, c in enumerate(counts)])
            tgt = torch.cat([tgt[r * nmax:r * nmax + c] for r, c in enumerate(counts)])
        out = self.cache.train_frame(rec, tgt, s, l, shuffle_seed, losses)
        self.last_launch_count = getattr(self.cache, "last_launch_count", 0)
        return out

    def _counts(self, n_loc: int):
        """Every rank's record count.  The exchange runs on every call (one
        small all-gather of Python ints), so a rank whose count changed can
        never leave the others in a different collective."""
        got = [None] * self.world
        dist.all_gather_object(got, n_loc, group=self.group)
        return [int(c) for c in got]

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

    def _sym_setup(self, multicast: bool):
        """Peer-mapped buffers for the in-kernel all-reduce modes: two [gradient |
        loss sum] buffers (step parity) + one barrier counter per rank, mapped
        on every rank -- CUDA IPC handles exchanged over the process group, or
        (multicast=True) torch symmetric memory, which also gives the buffer's
        multicast (NVLS) address."""
        self._sym_stride = (NPARAM + 1 + 63) // 64 * 64  # floats per buffer, 256-B aligned
        n = 2 * self._sym_stride + 64
        esz = 4
        mc = 0
        if not multicast:
            # peer mappings through CUDA IPC (also two ranks on one GPU, where
            # torch's symmetric memory refuses overlapping devices)
            from .nrc import ipc_export_ptr, ipc_import
            buf = torch.zeros(n, dtype=torch.float32, device=self.device)
            mine = ipc_export_ptr(buf.data_ptr())
            everyone = [None] * self.world
            dist.all_gather_object(everyone, mine, group=self.group)
            self._sym_buf = buf
            ptrs = [buf.data_ptr() if r == self.rank else ipc_import(*everyone[r]) for r in range(self.world)]
            self._sym_multicast = False
        else:
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(n, dtype=torch.float32, device=self.device)
            buf.zero_()
            gname = (self.group or dist.group.WORLD).group_name
            hdl = symm_mem.rendezvous(buf, gname)
            mc = getattr(hdl, "multicast_ptr", 0)
        if multicast and mc:
            self._sym_hdl, self._sym_buf = hdl, buf
            ptrs = [int(p) for p in hdl.buffer_ptrs]
        elif multicast and self.world == 1:
            # one rank: a single-device multicast object from libnrc (torch exports
            # multicast handles for sharing, which some systems refuse)
            from .nrc import multicast_alloc
            self._sym_buf, mc = multicast_alloc(n, self.device)
            ptrs = [self._sym_buf.data_ptr()]
        elif multicast:
            raise RuntimeError("NVLS multicast is not available on this system (symmetric memory without multicast)")
        self._sym_mc = [mc + k * self._sym_stride * esz for k in range(2)] if mc else None
        self._sym_peers = [[p + k * self._sym_stride * esz for p in ptrs] for k in range(2)]
        self._sym_ctr = [p + 2 * self._sym_stride * esz for p in ptrs]
        self._sym_seq = 0
        self._sym_multicast = bool(mc)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)  # zeroed everywhere before any rank signals

    def _train_frame_sym(self, records, targets, s, l, shuffle_seed, losses, multicast: bool):
        if getattr(self, "_sym_buf", None) is None or (multicast and not self._sym_multicast):
            self._sym_setup(multicast)
        n_total = int(records.shape[0])
        s, l = frame_batches(n_total, s, l)
        launches = 0
        if s == 0:
            self.last_launch_count = 0
            return losses
        lo, hi = shard(l, self.rank, self.world)
        for j in range(s):
            par = self._sym_seq & 1
            base = par * self._sym_stride
            grad = self._sym_buf[base:base + NPARAM]
            loss_sum = self._sym_buf[base + NPARAM:base + NPARAM + 1]
            self.cache.train_frame_backward(records, targets, l, shuffle_seed, j, lo, hi, grad, loss_sum)
            launches += getattr(self.cache, "last_launch_count", 0)
            self.cache.peer_barrier(self._sym_ctr, self.rank, self.world)
            launches += 1
            out = None if losses is None else losses[j:j + 1]
            if multicast:
                self.cache.train_apply_multimem(self._sym_mc[par], l, out)
            else:
                self.cache.train_apply_peers(self._sym_peers[par], l, out)
            launches += getattr(self.cache, "last_launch_count", 0)
            self._sym_seq += 1
        self.last_launch_count = launches
        return losses

    def train_frame_allreduce_sym(self, records: torch.Tensor, targets: torch.Tensor, s: int, l: int,
                                  shuffle_seed: int, losses: Optional[torch.Tensor] = None
                                  ) -> Optional[torch.Tensor]:
        """Data-parallel training with the per-step all-reduce folded into the
        optimiser over peer memory: this rank's rows of the shuffled batch ->
        its [gradient | loss sum] into a peer-mapped buffer (by step parity), a
        cross-rank barrier kernel, then the optimiser loads every rank's
        buffer over NVLink and sums them in rank order (nrc_train_apply_peers)
        -- no NCCL call, identical replicas, 86 KB per peer per step."""
        return self._train_frame_sym(records, targets, s, l, shuffle_seed, losses, multicast=False)

    def train_frame_allreduce_nvls(self, records: torch.Tensor, targets: torch.Tensor, s: int, l: int,
                                   shuffle_seed: int, losses: Optional[torch.Tensor] = None
                                   ) -> Optional[torch.Tensor]:
        """SURVEY 8(e) mitigation 2 / 8(f) N3 (ii): as train_frame_allreduce_sym,
        but the optimiser reads every gradient entry with multimem.ld_reduce on
        the buffer's multicast address -- the all-reduce done in the NVSwitch.
        Not bitwise equal to single-GPU training (the switch's fp32 summation
        order); every rank reads the same switch result."""
        return self._train_frame_sym(records, targets, s, l, shuffle_seed, losses, multicast=True)

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
            # Adam + EMA on grad / l; the batch-mean loss = loss sum / l is
            # computed by the library too (nrc_train_apply)
            self.cache.train_apply(self.grad, l, self.loss_sum, None if losses is None else losses[j:j + 1])
            launches += getattr(self.cache, "last_launch_count", 0)
        self.last_launch_count = launches
        return losses
