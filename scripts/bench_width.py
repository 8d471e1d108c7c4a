"""Width ablation (BASELINE.json configs[3]): the 1080p frame --
query of 2,073,600 records + a 4 x 16,384-record training frame -- at hidden
width 32 / 64 / 128 (input 64, depth 5): CUDA events, L2 flushed between reps,
tensor-roofline fractions of the query and of the training.  Training runs
through the per-step partials + Adam kernels at every width.
Writes one JSON line per configuration."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import nrc_inputs
import paper_2106_12372_b200 as nrc

PEAK = 1665.6
try:
    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "MEASURED_PEAKS.json")))["bf16_tflops"])
except Exception:
    pass
recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
n = recs.shape[0]
out = torch.empty((n, 3), device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
n_train = tr.shape[0]


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for hw in (32, 64, 128):
    c = nrc.RadianceCache(nrc.Config(hidden_width=hw))
    q_ms = timeit(lambda: c.query(recs, out))
    t_ms = timeit(lambda: c.train_frame(tr, tg, 4, 16384, 1), reps=30)
    fq = 2 * (64 * hw + 4 * hw * hw + 3 * hw)          # query FLOP per record
    ft = 2 * fq + 2 * (4 * hw * hw + 3 * hw)            # + dgrad (no layer 0) + wgrad per record
    q_tf = fq * n / (q_ms * 1e-3) / 1e12
    t_tf = ft * n_train / (t_ms * 1e-3) / 1e12
    print(json.dumps({"config": "C4 width ablation, 1080p frame (query + 4x16384 train)", "hidden_width": hw,
                      "train_kernel": "partials + adam (PDL)",
                      "query_ms": q_ms, "train_ms": t_ms, "frame_ms": q_ms + t_ms,
                      "queries_per_s": n / (q_ms * 1e-3), "records_per_s": n_train / (t_ms * 1e-3),
                      "flop_per_query": fq, "flop_per_train_record": ft,
                      "query_tflops": q_tf, "query_tensor_frac": q_tf / PEAK,
                      "train_tflops": t_tf, "train_tensor_frac": t_tf / PEAK,
                      "frame_tensor_frac": (fq * n + ft * n_train) / ((q_ms + t_ms) * 1e-3) / 1e12 / PEAK,
                      "peak_tflops": PEAK}), flush=True)
