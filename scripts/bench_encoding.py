"""N4: 1080p query with the cheap encoding primitives (tri / quartic, the
default) vs the exact ones (sin / Gaussian, NRC_EXACT_ENCODING) -- the
paper's fig:cheap_primitives ablation (0.25 ms per frame on an RTX 3090,
P:L680-683).  CUDA events, L2 flushed, median of 50."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import nrc_inputs
import paper_2106_12372_b200 as nrc

recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
out = torch.empty((recs.shape[0], 3), device="cuda")
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


res = {}
for name, flags in (("cheap", nrc.FACTORIZE | nrc.CLAMP_QUERY),
                    ("exact", nrc.FACTORIZE | nrc.CLAMP_QUERY | nrc.EXACT_ENCODING)):
    c = nrc.RadianceCache(nrc.Config(flags=flags))
    res[name] = {"query_ms": timeit(lambda: c.query(recs, out)),
                 "train_frame_ms": timeit(lambda: c.train_frame(tr, tg, 4, 16384, 1))}
res["frame_delta_ms"] = (res["exact"]["query_ms"] + res["exact"]["train_frame_ms"]
                         - res["cheap"]["query_ms"] - res["cheap"]["train_frame_ms"])
print(json.dumps({"config": "N4 encoding primitives, 1080p query + 4x16384 train", **res}))
