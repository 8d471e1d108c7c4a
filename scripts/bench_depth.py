"""Depth variants: the 1080p frame -- 2,073,600 queries + a
4 x 16,384-record training frame -- at width 64 with 1 / 2 / 3 / 5 / 7
hidden layers: CUDA events, L2 flushed between reps, tensor-roofline fraction
of the query.  One JSON line per depth."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import nrc_inputs
import paper_2106_12372_b200 as nrc

PEAK = 1590.0
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


for nh in (1, 2, 3, 5, 7):
    c = nrc.RadianceCache(nrc.Config(hidden_width=64, n_hidden_layers=nh))
    q_ms = timeit(lambda: c.query(recs, out))
    t_ms = timeit(lambda: c.train_frame(tr, tg, 4, 16384, 1), reps=30)
    fq = 2 * (64 * 64 + (nh - 1) * 64 * 64 + 3 * 64)
    print(json.dumps({"config": "N4 depth variants, 1080p frame (query + 4x16384 train), width 64",
                      "hidden_layers": nh, "query_ms": q_ms, "train_ms": t_ms, "frame_ms": q_ms + t_ms,
                      "flop_per_query": fq, "query_tflops": fq * n / (q_ms * 1e-3) / 1e12,
                      "query_tensor_frac": fq * n / (q_ms * 1e-3) / 1e12 / PEAK, "peak_tflops": PEAK}), flush=True)
