"""Width ablation (BASELINE.json configs[3]): 1080p query time and
tensor-roofline fraction at hidden width 32 / 64 / 128 (input 64, depth 5),
CUDA events, L2 flushed between reps.  Training is built for W = 64 only, so
the frame column adds the W = 64 training time to every width.
Writes one JSON line per width."""
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
c64 = nrc.RadianceCache()


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


t_train = timeit(lambda: c64.train_frame(tr, tg, 4, 16384, 1))
for hw in (32, 64, 128):
    c = nrc.RadianceCache(nrc.Config(hidden_width=hw))
    ms = timeit(lambda: c.query(recs, out))
    flop = 2 * (64 * hw + 4 * hw * hw + 3 * hw)
    tf = flop * n / (ms * 1e-3) / 1e12
    print(json.dumps({"config": "C4 width ablation, 1080p query", "hidden_width": hw, "query_ms": ms,
                      "queries_per_s": n / (ms * 1e-3), "flop_per_query": flop, "achieved_tflops": tf,
                      "tensor_frac": tf / PEAK, "train_frame_ms_w64": t_train, "frame_ms": ms + t_train}))
