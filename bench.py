#!/usr/bin/env python
"""bench.py -- NRC frame benchmark (BASELINE.json metric).

One step = one 1080p frame of the paper's hot path (tab:timings
P:L1241-1309): a cache query of 2,073,600 records (one per pixel)
with the EMA weights, plus the frame's training -- 65,536 records LCG-
shuffled into s = 4 batches of l = 16,384, each a fused
forward / relative-L2 / backward step followed by Adam + EMA.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nrc|reference]

N > 1 (launched with torch.distributed.run, one rank per GPU, NCCL):
north_star's partition -- query rows sharded over the ranks with no
communication, training data-parallel: each rank takes l/N rows of every
shuffled batch, one NCCL all-reduce of [gradient | loss sum] per step,
identical Adam on every rank (--train-mode dp, the default).  Variants
(SURVEY 8(f) N3): --train-mode replicated (one all-gather of the frame's
records, then replicated training), --train-mode allreduce-peer (the
gradient all-reduce fused into the optimiser kernel over peer memory) and
--train-mode allreduce-nvls (the all-reduce in the NVSwitch: the optimiser
reads every gradient entry with multimem.ld_reduce).
Max-over-ranks device time.

--impl reference: the fp64 CPU oracle (oracle/, as it stands) on the host
cores, timing whole frames (2,073,600 queries + 4 sequential 16,384-record
train steps).
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


def stats_ms(xs):
    """median, mean and p10/p50/p90 of a list of per-step times (ms)."""
    xs = [float(x) for x in xs]
    p10, p50, p90 = (float(v) for v in np.percentile(xs, [10, 50, 90]))
    return {"median": p50, "mean": float(np.mean(xs)), "p10": p10, "p50": p50, "p90": p90}


# ============================================================================ the oracle (reference arm, cpu_baseline)
class OracleFrame:
    """The fp64 CPU oracle on the bench's frame: query of the frame's records
    with W-bar, then s sequential train steps on the LCG-shuffled batches
    (the same generator seeds as the CUDA arm).  frac < 1 times the first
    frac of the queries and of every batch (a bounded sample) and scales the
    two phases back to the frame."""

    def __init__(self):
        import nrc_inputs
        import oracle
        oracle.build()
        self.oracle = oracle
        self.recs_q = nrc_inputs.records(N_QUERY, seed=nrc_inputs.SEED_QUERY)
        self.recs_t, self.tg = nrc_inputs.train_frame(0, n=N_TRAIN, noise=0.3)
        a, c, m = oracle.lcg_params(N_TRAIN, 1000)
        self.perm = oracle.lcg_permute(N_TRAIN, a, c, m).astype(np.int64)
        self.oc = oracle.OracleCache()

    def frame(self, frac: float = 1.0):
        nq = max(1, int(round(N_QUERY * frac)))
        lt = max(1, int(round(TRAIN_L * frac)))
        t0 = time.perf_counter()
        self.oc.query(self.recs_q[:nq])
        t1 = time.perf_counter()
        for j in range(TRAIN_S):
            idx = self.perm[j * TRAIN_L:j * TRAIN_L + lt]
            self.oc.train_step(self.recs_t[idx], self.tg[idx])
        t2 = time.perf_counter()
        tq, tt = (t1 - t0) / (nq / N_QUERY), (t2 - t1) / (lt / TRAIN_L)
        return 1e3 * (tq + tt), 1e3 * tq, 1e3 * tt


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
    """The oracle on one host thread (SURVEY 8(d) oracle timing): a 1/256
    sample of the frame (8,100 queries + 4 x 64-record steps) in a subprocess
    with OMP_NUM_THREADS=1, scaled to the frame; None if it fails."""
    code = ("import sys; sys.path.insert(0, %r); import bench; f = bench.OracleFrame(); "
            "print(f.frame(1.0 / 256)[0])" % ROOT)
    try:
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, OMP_NUM_THREADS="1"),
                             capture_output=True, text=True, timeout=600)
        return float(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None


def frame_config(world: int, train_mode: str = "dp") -> dict:
    return {"workload": CONFIG_NAME, "global_batch": N_QUERY, "train_records": N_TRAIN,
            "parallelism": f"{train_mode}{world}" if world > 1 else "single",
            "query_partition": "rows sharded over ranks, no communication" if world > 1 else "one GPU",
            "l2": "flushed (256 MB write) between timed steps",
            "train_kernel": "per step: partials + reduce/Adam/EMA, PDL-chained"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    budget = float(os.environ.get("NRC_REF_BUDGET_S", "600"))
    of = OracleFrame()
    # one whole frame first (page-in + the cost estimate); it counts as warm-up
    t0 = time.perf_counter()
    of.frame()
    est = time.perf_counter() - t0
    frac = 1.0
    if est * (args.steps + args.warmup) > budget:  # shrink to a bounded sample of every phase
        frac = max(budget / (args.steps + args.warmup) / est, 1.0 / 512)
    for _ in range(max(0, args.warmup - 1)):
        of.frame(frac)
    times, tq, tt = [], [], []
    for _ in range(args.steps):
        ms, q, t = of.frame(frac)
        times.append(ms)
        tq.append(q)
        tt.append(t)
    st = stats_ms(times)
    ms = st["median"]
    q_ms, t_ms = float(np.median(tq)), float(np.median(tt))
    sample = ("whole frames: 2,073,600 queries + 4 sequential 16,384-record train steps per step" if frac == 1.0 else
              f"{frac:.4f} of every phase per step (budget {budget:.0f} s), scaled to the frame")
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (nrc_inputs seeded records)",
        "config": frame_config(args.gpus, args.train_mode),
        "ms_mean": st["mean"], "ms_p10_p50_p90": [st["p10"], st["p50"], st["p90"]],
        "query_ms": q_ms, "train_ms": t_ms,
        "queries_per_s": N_QUERY / (q_ms * 1e-3), "records_per_s": N_TRAIN / (t_ms * 1e-3),
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": omp_threads(), "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


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
            # communicator-init log lines (rank / nranks per communicator) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    mode = args.train_mode

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- inputs (synthetic, resident in HBM before timing)
    q0, q1 = nrc.shard(N_QUERY, rank, world)
    recs_q_all = nrc_inputs.records(N_QUERY, seed=nrc_inputs.SEED_QUERY)
    recs_q = torch.from_numpy(recs_q_all[q0:q1].copy()).to(dev)
    nq_local = q1 - q0
    t_counts = [b - a for a, b in (nrc.shard(N_TRAIN, r, world) for r in range(world))]
    t0_, t1_ = nrc.shard(N_TRAIN, rank, world)
    frames = []
    for f in range(2):
        r, t = nrc_inputs.train_frame(f, n=N_TRAIN, noise=0.3)
        frames.append((torch.from_numpy(r).to(dev), torch.from_numpy(t).to(dev), r, t,
                       torch.from_numpy(r[t0_:t1_].copy()).to(dev), torch.from_numpy(t[t0_:t1_].copy()).to(dev)))
    rgb = torch.empty((nq_local, 3), dtype=torch.float32, device=dev)
    cache = nrc.RadianceCache(nrc.Config(max_batch=max(N_QUERY, N_TRAIN)), device=local)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    dpf = nrc.DataParallelFrame(cache, device=dev) if world > 1 else None

    def frame(fi, ev=None):
        """One frame: query (EMA weights of the previous frame) + training.
        ev = (start, query end, train end) events recorded on the stream."""
        d_r, d_t, _, _, d_rl, d_tl = frames[fi % 2]
        seed = 1000 + fi % 2
        if ev:
            ev[0].record(stream)
        cache.query(recs_q, rgb)
        launches = cache.last_launch_count
        if ev:
            ev[1].record(stream)
        if world == 1:
            cache.train_frame(d_r, d_t, TRAIN_S, TRAIN_L, seed)
            launches += cache.last_launch_count
        elif mode == "replicated":
            # N3 (i): this rank's screen-region records, one all-gather, replicated training
            dpf.train_frame_replicated(d_rl, d_tl, TRAIN_S, TRAIN_L, seed, counts=t_counts)
            launches += dpf.last_launch_count
        elif mode == "allreduce-sym":
            # the per-step all-reduce folded into the optimiser's loads over peer
            # memory (symmetric buffers of the reduced [gradient | loss], no NCCL call)
            dpf.train_frame_allreduce_sym(d_r, d_t, TRAIN_S, TRAIN_L, seed)
            launches += dpf.last_launch_count
        elif mode == "allreduce-nvls":
            # SURVEY 8(e) mitigation 2 / N3 (ii): the gradient all-reduce done in the
            # NVSwitch (multimem.ld_reduce read by the optimiser kernel; no NCCL call)
            dpf.train_frame_allreduce_nvls(d_r, d_t, TRAIN_S, TRAIN_L, seed)
            launches += dpf.last_launch_count
        elif mode == "allreduce-peer":
            # SURVEY 8(e) mitigation 2 / N3 (ii): the gradient all-reduce fused into
            # the optimiser over peer memory (no NCCL call)
            dpf.train_frame_allreduce_peer(d_r, d_t, TRAIN_S, TRAIN_L, seed)
            launches += dpf.last_launch_count
        else:
            # north_star: this rank's rows of every shuffled batch (gathered in-kernel,
            # P:L487-491), one NCCL all-reduce per step, identical Adam on every rank
            dpf.train_frame(d_r, d_t, TRAIN_S, TRAIN_L, seed)
            launches += dpf.last_launch_count
        if ev:
            ev[2].record(stream)
        return launches

    torch.cuda.synchronize()
    barrier()
    if world > 1:
        dpf.verify_replicas()  # the same seeded init on every rank
    for i in range(args.warmup):
        frame(i)
    torch.cuda.synchronize()
    barrier()

    evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the timed events)
            launches += frame(i, evs[i])
            torch.cuda.synchronize()
        torch.cuda.synchronize()
        barrier()
    step_ms = [a.elapsed_time(c) for a, b, c in evs]
    q_list = [a.elapsed_time(b) for a, b, c in evs]
    t_list = [b.elapsed_time(c) for a, b, c in evs]
    replicas = None
    if world > 1:  # bitwise-identical replicas after the timed frames (outside the timing)
        replicas = "identical crc32 %08x" % dpf.verify_replicas()
    # N3 comparison: the frame's training through every multi-GPU
    # partition, each on a fresh cache, device time max over ranks
    mode_ms = {}
    if world > 1 and not args.no_mode_table:
        for m in ["dp", "replicated", "allreduce-peer", "allreduce-sym", "allreduce-nvls"]:
            try:
                c2 = nrc.RadianceCache(nrc.Config(max_batch=max(N_QUERY, N_TRAIN)), device=local)
                f2 = nrc.DataParallelFrame(c2, device=dev)
                d_r, d_t, _, _, d_rl, d_tl = frames[0]

                def train(fi, m=m, c2=c2, f2=f2):
                    d_r, d_t, _, _, d_rl, d_tl = frames[fi % 2]
                    if m == "dp":
                        f2.train_frame(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi)
                    elif m == "replicated":
                        f2.train_frame_replicated(d_rl, d_tl, TRAIN_S, TRAIN_L, 1000 + fi, counts=t_counts)
                    elif m == "allreduce-peer":
                        f2.train_frame_allreduce_peer(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi)
                    elif m == "allreduce-sym":
                        f2.train_frame_allreduce_sym(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi)
                    else:
                        f2.train_frame_allreduce_nvls(d_r, d_t, TRAIN_S, TRAIN_L, 1000 + fi)
                for i in range(3):
                    train(i)
                torch.cuda.synchronize()
                barrier()
                ts = []
                for i in range(max(args.steps, 5)):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    train(i)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                t = torch.tensor([float(np.median(ts))], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                mode_ms[m] = {"train_ms": float(t[0]), "replicas": "identical crc32 %08x" % f2.verify_replicas()}
            except Exception as e:  # e.g. no NVLS multicast on this system
                mode_ms[m] = {"unavailable": str(e).splitlines()[0][:160]}
            barrier()
    st = stats_ms(step_ms)
    ms, q_ms, t_ms = st["median"], float(np.median(q_list)), float(np.median(t_list))
    pct = [st["p10"], st["p50"], st["p90"]]
    if world > 1:  # max over ranks of every reported time
        t = torch.tensor([ms, q_ms, t_ms, st["mean"]] + pct, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, q_ms, t_ms = float(t[0]), float(t[1]), float(t[2])
        st["mean"] = float(t[3])
        pct = [float(x) for x in t[4:7]]

    # ---- end to end through the C ABI with host buffers (N = 1)
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
        e_ms = float(np.median([s.elapsed_time(e) for s, e in e_ev]))
        h2d = N_QUERY * 64 + N_TRAIN * (64 + 12)
        d2h = N_QUERY * 12 + TRAIN_S * 4
        e2e = {"value": e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "pcie_gbs": (h2d + d2h) / (e_ms * 1e-3) / 1e9,
               "note": "nrc_frame_host: pinned host records -> device (chunked, overlapped with the query), "
                       "query + 4 train steps, RGB + losses -> host; bound by the PCIe copy of 137.7 MB in "
                       "+ 24.9 MB out per frame"}

    peak_tf, peak_bw, peak_src = peaks()
    traffic, traffic_src = ncu_traffic("nrc_query_ts_kernel")
    nq_roof = nq_local
    if world > 1:  # the busiest query rank
        t = torch.tensor([nq_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nq_roof = int(t[0])
    achieved = FLOP_QUERY * nq_roof / (q_ms * 1e-3) / 1e12
    t_achieved = FLOP_TRAIN * N_TRAIN / max(world, 1) / (t_ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f16 (fp32 accumulate, fp32 Adam/EMA)", "data": "synthetic (nrc_inputs)",
        "config": frame_config(world, mode),
        "ms_stat": "median over the timed frames",
        "ms_mean": st["mean"], "ms_p10_p50_p90": pct,
        "query_ms": q_ms, "train_ms": t_ms,
        # phase rates: queries over the query phase, records over the training phase
        "queries_per_s": N_QUERY / (q_ms * 1e-3), "records_per_s": N_TRAIN / (t_ms * 1e-3),
        "frame_queries_per_s": N_QUERY / (ms * 1e-3),
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "kernel": "nrc_query_ts_kernel", "achieved": achieved, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": traffic, "traffic_unit": "bytes/launch",
                     "traffic_source": traffic_src,
                     "algorithmic_bytes": BYTES_QUERY * nq_roof,
                     "peak_source": f"{peak_src} bf16 dense burst (fp16 same rate)",
                     "algorithmic": f"{FLOP_QUERY} FLOP/query x {nq_roof} queries / median query-phase time",
                     "frac_vs_spec_2250": achieved / 2250.0,
                     "hbm_frac": BYTES_QUERY * nq_roof / (q_ms * 1e-3) / 1e9 / peak_bw},
        "train_roofline": {"bound": "latency (12 dependent MMA/epilogue rounds per step)",
                           "achieved": t_achieved, "unit": "TFLOP/s", "frac": t_achieved / peak_tf,
                           "algorithmic": f"{FLOP_TRAIN} FLOP/record x {N_TRAIN // max(world, 1)} records per rank"},
        "clocks": clk.summary(),
    }
    if replicas:
        line["replicas"] = replicas
    if mode_ms:
        line["train_modes"] = mode_ms
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        of = OracleFrame()
        of.frame()  # page-in
        reps = [of.frame() for _ in range(2)]
        cms = float(np.median([r[0] for r in reps]))
        line["cpu_baseline"] = {"value": cms, "unit": "ms", "cores": omp_threads(), "kind": "oracle",
                                "sample": "whole frames (2,073,600 queries + 4 sequential 16,384-record steps), "
                                          "median of 2 after one untimed",
                                "query_ms": float(np.median([r[1] for r in reps])),
                                "train_ms": float(np.median([r[2] for r in reps])),
                                "cpu_model": cpu_model(),
                                "single_thread_value": oracle_single_thread_ms(),
                                "single_thread_sample": "1/256 of every phase, scaled to the frame"}
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
    ap.add_argument("--no-mode-table", action="store_true",
                    help="N > 1: skip the per-partition training comparison (train_modes)")
    ap.add_argument("--workload", choices=["1080p", "4k"], default="1080p",
                    help="1080p: BASELINE.json configs[1] (the metric's workload); 4k: configs[4] (C5), "
                         "8,294,400 queries + 4x16384 train, for the multi-GPU scaling runs")
    ap.add_argument("--train-mode", choices=["dp", "replicated", "allreduce-peer", "allreduce-sym", "allreduce-nvls"],
                    default="dp",
                    help="N > 1 training: data-parallel with one NCCL all-reduce per step (dp, north_star's "
                         "partition, the default), one all-gather of the frame's records then replicated "
                         "training (replicated, SURVEY N3 (i)), or data-parallel with the gradient all-reduce "
                         "fused into the optimiser over peer memory (allreduce-peer: every tile partial; "
                         "allreduce-sym: each rank's reduced gradient), or done in the NVSwitch with "
                         "multimem.ld_reduce feeding the optimiser (allreduce-nvls, N3 (ii))")
    args = ap.parse_args()
    if args.workload == "4k":
        global N_QUERY, METRIC, CONFIG_NAME
        N_QUERY = 3840 * 2160
        METRIC = "NRC frame ms (4K: 8.29M queries + 4×16384 train); queries/s, records/s"
        CONFIG_NAME = "4K frame: 8,294,400 queries + 4x16384 train, width 64, 5 hidden layers"
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_nrc(args)


if __name__ == "__main__":
    sys.exit(main())
