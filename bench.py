#!/usr/bin/env python
"""bench.py -- NRC frame benchmark (BASELINE.json metric).

One step = one 1080p frame of the paper's hot path (tab:timings
P:L1241-1309): a cache query of 2,073,600 records (one per pixel)
with the EMA weights, plus the frame's training -- 65,536 records LCG-
shuffled into s = 4 batches of l = 16,384, each a fused
forward / relative-L2 / backward step followed by Adam + EMA.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nrc|reference]

N > 1 (launched with torch.distributed.run, one rank per GPU, NCCL): the same
frame is split across ranks -- by function by default (--train-mode
dedicated: rank 0 trains, ranks 1..N-1 shard the query rows, then the new
query image is broadcast), or query rows sharded over all ranks with the
training replicated after one all-gather of the frame's records
(--train-mode replicated) or data-parallel (--train-mode dp:
each rank takes l/N rows of every batch, one NCCL all-reduce of the gradient
per step, identical Adam on every rank; --train-mode allreduce-peer: the same
split with the all-reduce fused into the optimiser kernel over peer memory;
--train-mode peer: the record all-gather fused into the training kernel) --
strong scaling, max-over-ranks device time.

--impl reference: the fp64 CPU oracle (oracle/, as it stands) on the host
cores, timed on a bounded sample of the same frame and scaled to the frame.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

N_QUERY = 1920 * 1080
TRAIN_S, TRAIN_L = 4, 16384
N_TRAIN = TRAIN_S * TRAIN_L
FLOP_QUERY = 2 * (64 * 64 + 4 * 64 * 64 + 64 * 3)            # 41,344
FLOP_TRAIN = FLOP_QUERY + 2 * (4 * 4096 + 192) + FLOP_QUERY  # 115,840
BYTES_QUERY = 64 + 12                                        # record in + RGB out
METRIC = "NRC frame ms (1080p: 2.07M queries + 4×16384 train); queries/s, records/s"
CONFIG_NAME = "1080p frame: 2,073,600 queries + 4x16384 train, width 64, 5 hidden layers"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None
        self._t = None

    def _reader(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                        "--format=csv,noheader,nounits", "-lms", "20"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.3)  # first sample lands before the timed region starts
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is not None:
            time.sleep(0.05)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ============================================================================ reference arm (oracle)
def oracle_frame_estimate(q_sample: int, t_sample: int, reps: int = 1):
    """Times the fp64 oracle on q_sample queries and one train step of
    t_sample records; scales to one 1080p frame.  Returns (ms_frame, detail)."""
    import nrc_inputs
    import oracle
    oracle.build()
    recs_q = nrc_inputs.records(q_sample, seed=nrc_inputs.SEED_QUERY)
    recs_t, tg = nrc_inputs.train_frame(0, n=t_sample)
    oc = oracle.OracleCache()
    tq = tt = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        oc.query(recs_q)
        t1 = time.perf_counter()
        oc.train_step(recs_t, tg)
        t2 = time.perf_counter()
        tq += t1 - t0
        tt += t2 - t1
    tq /= reps
    tt /= reps
    ms = 1e3 * (tq / q_sample * N_QUERY + tt / t_sample * N_TRAIN)
    sample = (f"{q_sample} queries + one {t_sample}-record train step per rep, scaled to 2,073,600 queries + "
              f"65,536 train records")
    return ms, sample, tq, tt


def frame_config(world: int, train_mode: str = "dp") -> dict:
    return {"workload": CONFIG_NAME, "global_batch": N_QUERY, "train_records": N_TRAIN,
            "parallelism": f"{train_mode}{world}" if world > 1 else "single",
            "l2": "flushed (256 MB write) between timed steps",
            "train_kernel": ("fused cooperative (NRC_TRAIN_FUSED=1)" if os.environ.get("NRC_TRAIN_FUSED", "0") != "0"
                             else "per step: partials + reduce/Adam/EMA, PDL-chained")}


def ncu_traffic(kernel: str):
    """dram read+write bytes per launch of `kernel` from the newest committed
    ncu --set full capture summary (profiles/rNN_traffic.json), else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    for f in reversed(files):
        try:
            with open(f) as fh:
                t = json.load(fh)
            if kernel in t:
                return float(t[kernel]["traffic_bytes"]), os.path.relpath(f, ROOT)
        except Exception:
            continue
    return None, None


def omp_threads():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_single_thread_ms():
    """The oracle on one host thread (SURVEY 8(d) oracle timing): a 4096-query
    + 512-record sample in a subprocess with OMP_NUM_THREADS=1, scaled to the
    frame; None if it fails."""
    code = ("import sys; sys.path.insert(0, %r); import bench; "
            "print(bench.oracle_frame_estimate(4096, 512)[0])" % ROOT)
    try:
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, OMP_NUM_THREADS="1"),
                             capture_output=True, text=True, timeout=300)
        return float(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # bounded samples: size each step so that warm-up + timed steps take about
    # REF_BUDGET_S of host time in total, from the oracle's measured per-record cost
    budget = float(os.environ.get("NRC_REF_BUDGET_S", "120"))
    _, _, tq, tt = oracle_frame_estimate(4096, 512)  # warm-up (build, page-in) + calibration
    per_step = budget / max(1, args.steps + args.warmup)
    per_q, per_t = tq / 4096, tt / 512
    scale = per_step / max(per_q * 32768 + per_t * 4096, 1e-9)
    q_sample = int(min(32768, max(1024, 32768 * scale)))
    t_sample = int(min(4096, max(256, 4096 * scale)))
    times = []
    for _ in range(args.warmup):
        oracle_frame_estimate(q_sample, t_sample)
    for _ in range(args.steps):
        ms, sample, _, _ = oracle_frame_estimate(q_sample, t_sample)
        times.append(ms)
    ms = float(np.mean(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (nrc_inputs seeded records)",
        "config": frame_config(args.gpus, args.train_mode),
        "queries_per_s": N_QUERY / (ms * 1e-3), "records_per_s": N_TRAIN / (ms * 1e-3),
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": omp_threads(), "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ============================================================================ CUDA arm
def run_nrc(args):
    import torch
    import torch.distributed as dist

    import nrc_inputs
    import paper_2106_12372_b200 as nrc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    # NRC_BENCH_SHARED_GPU=1 (code-path test only, timings meaningless): every rank
    # uses cuda:0 and gloo, so the N > 1 path can run on a one-GPU box
    shared = os.environ.get("NRC_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- inputs (synthetic, resident in HBM before timing)
    dedicated = world > 1 and args.train_mode == "dedicated"
    if dedicated:  # rank 0 trains, ranks 1..N-1 split the query rows (rank 0's share set after calibration)
        q0, q1 = (0, 0) if rank == 0 else nrc.shard(N_QUERY, rank - 1, world - 1)
    else:
        q0, q1 = nrc.shard(N_QUERY, rank, world)
    recs_q_all = nrc_inputs.records(N_QUERY, seed=nrc_inputs.SEED_QUERY)
    recs_q = torch.from_numpy(recs_q_all[q0:q1].copy()).to(dev)
    nq_local = q1 - q0
    frames = []
    for f in range(2):
        r, t = nrc_inputs.train_frame(f, n=N_TRAIN, noise=0.3)
        frames.append((torch.from_numpy(r).to(dev), torch.from_numpy(t).to(dev), r, t))
    rgb = torch.empty((nq_local, 3), dtype=torch.float32, device=dev)
    cache = nrc.RadianceCache(nrc.Config(max_batch=max(N_QUERY, N_TRAIN)), device=local)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    # data-parallel frame for world > 1 (query rows sharded, one all-reduce per train step)
    dpf = nrc.DataParallelFrame(cache, device=dev) if world > 1 else None

    q_start = torch.cuda.Event(enable_timing=True)
    q_end = torch.cuda.Event(enable_timing=True)

    def frame(fi, timed_query=False):
        """One 1080p frame: query (EMA weights of the previous frame) + training."""
        d_r, d_t, _, _ = frames[fi % 2]
        launches = 0
        if dedicated:
            # rank 0: the frame's training; ranks >= 1: their query rows; then the
            # new query image from rank 0 to all
            if timed_query:
                q_start.record(stream)
            if recs_q.shape[0] > 0:
                cache.query(recs_q, rgb)
                launches += cache.last_launch_count
            if timed_query:
                q_end.record(stream)
            if rank == 0:  # DataParallelFrame.frame_dedicated, with the query timed separately
                cache.train_frame(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi % 2)
                launches += cache.last_launch_count
            dist.broadcast(cache.query_image(), src=0)
            return launches
        if timed_query:
            q_start.record(stream)
        cache.query(recs_q, rgb)
        if timed_query:
            q_end.record(stream)
        launches += cache.last_launch_count
        if world == 1:
            cache.train_frame(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi % 2)
            launches += cache.last_launch_count
        elif args.train_mode == "peer":
            # N3, all-gather fused into the kernel: rows gathered from the owners' memory
            # (CUDA IPC / NVLink); the frame buffers are static and synchronised at setup
            lo, hi = nrc.shard(N_TRAIN, rank, world)
            dpf.train_frame_peer(d_r[lo:hi], d_t[lo:hi], TRAIN_S, TRAIN_L, 1000 + fi % 2, parts_ready=True)
            launches += dpf.last_launch_count
        elif args.train_mode == "allreduce-peer":
            # SURVEY 8(e) mitigation 2 / N3 (ii): each rank's tiles of every batch, the
            # gradient all-reduce fused into the optimiser over peer memory (no NCCL)
            dpf.train_frame_allreduce_peer(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi % 2)
            launches += dpf.last_launch_count
        elif args.train_mode == "replicated":
            # N3 (i): this rank's screen-region records, one all-gather, replicated training
            lo, hi = nrc.shard(N_TRAIN, rank, world)
            dpf.train_frame_replicated(d_r[lo:hi], d_t[lo:hi], TRAIN_S, TRAIN_L, 1000 + fi % 2)
            launches += dpf.last_launch_count
        else:
            # this rank's rows of every shuffled batch, gathered in-kernel
            dpf.train_frame(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi % 2)
            launches += dpf.last_launch_count
        return launches

    torch.cuda.synchronize()
    barrier()  # every rank's frame buffers are on the device (peer mode reads them remotely)
    if world > 1:
        dpf.verify_replicas(image_only=dedicated)  # the same seeded init on every rank
    for i in range(args.warmup):
        frame(i)
    torch.cuda.synchronize()
    barrier()
    if dedicated:
        # balance: rank 0's query share from the measured training time (rank 0)
        # and query time (rank 1), decided on rank 0 and broadcast
        def dev_ms(fn, reps=5):
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            for _ in range(reps):
                fn()
            b_ev.record(stream)
            torch.cuda.synchronize()
            return a_ev.elapsed_time(b_ev) / reps
        d_r0, d_t0 = frames[0][0], frames[0][1]
        mine = dev_ms(lambda: cache.train_frame(d_r0, d_t0, TRAIN_S, TRAIN_L, 999)) if rank == 0 else \
            dev_ms(lambda: cache.query(recs_q, rgb)) * (world - 1)
        got = [None] * world
        dist.all_gather_object(got, mine)
        share = [nrc.DataParallelFrame.dedicated_share0(got[1], got[0], world)]
        dist.broadcast_object_list(share, src=0)
        q0, q1 = dpf.dedicated_query_rows(N_QUERY, share[0])
        recs_q = torch.from_numpy(recs_q_all[q0:q1].copy()).to(dev)
        nq_local = q1 - q0
        rgb = torch.empty((nq_local, 3), dtype=torch.float32, device=dev)
        ded_share0 = share[0]
        for i in range(3):
            frame(i)
        torch.cuda.synchronize()
        barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    qt = []
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the timed events)
            ev[i][0].record(stream)
            launches += frame(i, timed_query=True)
            ev[i][1].record(stream)
            torch.cuda.synchronize()
            qt.append(q_start.elapsed_time(q_end))
        torch.cuda.synchronize()
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    replicas = None
    if world > 1:  # bitwise-identical replicas after the timed frames (outside the timing)
        replicas = "identical crc32 %08x" % dpf.verify_replicas(image_only=dedicated)
    ms = float(np.mean(step_ms))
    pct = [float(x) for x in np.percentile(step_ms, [10, 50, 90])]  # this rank's step distribution
    q_ms = float(np.mean(qt))
    if world > 1:
        t = torch.tensor([ms, q_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, q_ms = float(t[0]), float(t[1])

    # ---- end to end through the C ABI with host buffers (N = 1 path; for N > 1 rank-local)
    e2e = None
    if world == 1 and not args.no_e2e:
        hq = torch.from_numpy(recs_q_all).pin_memory()
        ht = torch.from_numpy(frames[0][2]).pin_memory()
        htg = torch.from_numpy(frames[0][3]).pin_memory()
        hrgb = torch.empty((N_QUERY, 3), dtype=torch.float32).pin_memory()
        hloss = torch.empty(64, dtype=torch.float32).pin_memory()
        scratch = torch.empty(cache.frame_scratch_bytes(N_QUERY, N_TRAIN) + 256, dtype=torch.uint8, device=dev)
        off = (-scratch.data_ptr()) % 256
        scratch = scratch[off:]
        hq_np, ht_np, htg_np, hrgb_np, hl_np = hq.numpy(), ht.numpy(), htg.numpy(), hrgb.numpy(), hloss.numpy()
        for _ in range(2):
            cache.frame_host(hq_np, hrgb_np, ht_np, htg_np, TRAIN_S, TRAIN_L, 7, hl_np, scratch)
        torch.cuda.synchronize()
        e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
        for i in range(args.steps):
            e_ev[i][0].record(stream)
            cache.frame_host(hq_np, hrgb_np, ht_np, htg_np, TRAIN_S, TRAIN_L, 7, hl_np, scratch)
            e_ev[i][1].record(stream)
            torch.cuda.synchronize()
        e_ms = float(np.mean([s.elapsed_time(e) for s, e in e_ev]))
        e2e = {"value": e_ms, "unit": "ms", "h2d_bytes_per_step": N_QUERY * 64 + N_TRAIN * (64 + 12),
               "d2h_bytes_per_step": N_QUERY * 12 + TRAIN_S * 4,
               "note": "nrc_frame_host: pinned host records -> device, query + 4 train steps, RGB + losses -> host"}

    peak_tf, peak_bw, peak_src = peaks()
    traffic, traffic_src = ncu_traffic("nrc_query_ts_kernel")
    nq_roof = nq_local
    if world > 1:  # the busiest query rank
        t = torch.tensor([nq_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nq_roof = int(t[0])
    q_flops = FLOP_QUERY * nq_roof
    achieved = q_flops / (q_ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f16 (fp32 accumulate, fp32 Adam/EMA)", "data": "synthetic (nrc_inputs)",
        "config": frame_config(world, args.train_mode),
        "queries_per_s": N_QUERY / (ms * 1e-3), "records_per_s": N_TRAIN / (ms * 1e-3),
        "query_ms": q_ms, "train_ms": ms - q_ms,
        "ms_p10_p50_p90": pct,
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "kernel": "nrc_query_ts_kernel", "achieved": achieved, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": traffic, "traffic_unit": "bytes/launch",
                     "traffic_source": traffic_src,
                     "algorithmic_bytes": BYTES_QUERY * nq_roof,
                     "peak_source": f"{peak_src} bf16 dense burst (fp16 same rate)",
                     "algorithmic": f"{FLOP_QUERY} FLOP/query x {nq_roof} queries",
                     # the same against the 2.25 PF dense fp16 spec, and the
                     # kernel's HBM fraction (algorithmic bytes / time / HBM peak)
                     "frac_vs_spec_2250": achieved / 2250.0,
                     "hbm_frac": BYTES_QUERY * nq_roof / (q_ms * 1e-3) / 1e9 / peak_bw},
        "clocks": clk.summary(),
    }
    if replicas:
        line["replicas"] = replicas
    if dedicated:
        line["config"]["dedicated_rank0_query_share"] = ded_share0
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and not args.no_cpu_baseline:
        cms, sample, _, _ = oracle_frame_estimate(16384, 2048)
        line["cpu_baseline"] = {"value": cms, "unit": "ms", "cores": omp_threads(), "kind": "oracle",
                                "sample": sample, "cpu_model": cpu_model(),
                                "single_thread_value": oracle_single_thread_ms()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["nrc", "reference"], default="nrc")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer (e2e) leg (profiling runs)")
    ap.add_argument("--workload", choices=["1080p", "4k"], default="1080p",
                    help="1080p: BASELINE.json configs[1] (the metric's workload); 4k: configs[4] (C5), "
                         "8,294,400 queries + 4x16384 train, for the multi-GPU scaling runs")
    ap.add_argument("--train-mode", choices=["dp", "replicated", "peer", "allreduce-peer", "dedicated"],
                    default="dedicated",
                    help="N > 1 training: split by function (dedicated, the default: rank 0 trains -- the "
                         "latency-bound step fewer rows per GPU would not shorten -- while the other ranks "
                         "query, then the new query image is broadcast), one all-gather of the frame's records "
                         "per frame and replicated training (replicated, SURVEY N3 (i)), or "
                         "data-parallel with one all-reduce per step (dp, north_star's description), or the "
                         "all-gather fused into the training kernel over peer memory (peer), or data-parallel "
                         "with the gradient all-reduce fused into the optimiser over peer memory "
                         "(allreduce-peer), or split by function: rank 0 trains while the other ranks "
                         "query, then the new query image is broadcast (dedicated)")
    args = ap.parse_args()
    if args.workload == "4k":
        global N_QUERY, METRIC, CONFIG_NAME
        N_QUERY = 3840 * 2160
        METRIC = "NRC frame ms (4K: 8.29M queries + 4\u00d716384 train); queries/s, records/s"
        CONFIG_NAME = "4K frame: 8,294,400 queries + 4x16384 train, width 64, 5 hidden layers"
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_nrc(args)


if __name__ == "__main__":
    sys.exit(main())
