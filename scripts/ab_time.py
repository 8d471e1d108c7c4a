"""A/B timing of the 1080p frame phases for the loaded libnrc build
(NRC_LIB_VARIANT selects a variant .so): median over reps of the query
(2,073,600 records) and of a 4 x 16,384 training frame, L2 flushed between
reps, CUDA events.  Prints one JSON line tagged with argv[1]."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs
import paper_2106_12372_b200 as nrc

tag = sys.argv[1] if len(sys.argv) > 1 else "base"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
out = torch.empty((recs.shape[0], 3), device="cuda")
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
c = nrc.RadianceCache()
for _ in range(5):
    c.query(recs, out=out); c.train_frame(tr, tg, 4, 16384, 1)
tq, tt = [], []
for i in range(reps):
    flush.fill_(float(i))
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(); c.query(recs, out=out); e1.record(); c.train_frame(tr, tg, 4, 16384, 1 + i); e2.record()
    torch.cuda.synchronize()
    tq.append(e0.elapsed_time(e1)); tt.append(e1.elapsed_time(e2))
print(json.dumps({"tag": tag, "query_us": round(1e3 * float(np.median(tq)), 2), "train_us": round(1e3 * float(np.median(tt)), 2),
                  "query_p10_p90": [round(1e3 * float(np.percentile(tq, p)), 2) for p in (10, 90)],
                  "train_p10_p90": [round(1e3 * float(np.percentile(tt, p)), 2) for p in (10, 90)]}))
