"""Quick device timing of nrc_query (1080p) and nrc_train_frame (4x16384) for
the query configuration selected by NRC_QUERY_CFG (tuning aid, not the bench)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import nrc_inputs
import paper_2106_12372_b200 as nrc

recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
c = nrc.RadianceCache()
out = torch.empty((recs.shape[0], 3), device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(5):
    c.query(recs, out); c.train_frame(tr, tg, 4, 16384, 1)
torch.cuda.synchronize()
def timeit(fn, reps=30):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3
tq = timeit(lambda: c.query(recs, out))
tt = timeit(lambda: c.train_frame(tr, tg, 4, 16384, 1))
ref = out.clone()
print(json.dumps({"cfg": os.environ.get("NRC_QUERY_CFG", "0"), "query_us": tq, "train_frame_us": tt,
                  "checksum": float(ref.double().sum())}))
