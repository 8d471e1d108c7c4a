"""A/B timing of whole 1080p frames (query + 4 x 16,384 training, no event
between the two phases) for the loaded libnrc build (NRC_LIB_VARIANT selects
a variant .so): median over reps, L2 flushed between reps, CUDA events.
Prints one JSON line tagged with argv[1]."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs
import paper_2106_12372_b200 as nrc

tag = sys.argv[1] if len(sys.argv) > 1 else "base"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
out = torch.empty((recs.shape[0], 3), device="cuda")
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
c = nrc.RadianceCache()
for _ in range(5):
    c.query(recs, out=out); c.train_frame(tr, tg, 4, 16384, 1)
tf = []
for i in range(reps):
    flush.fill_(float(i))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.query(recs, out=out); c.train_frame(tr, tg, 4, 16384, 1 + i); e1.record()
    torch.cuda.synchronize()
    tf.append(e0.elapsed_time(e1))
print(json.dumps({"tag": tag, "graph": os.environ.get("NRC_TRAIN_GRAPH", "1"), "frame_us": round(1e3 * float(np.median(tf)), 2),
                  "frame_p10_p90": [round(1e3 * float(np.percentile(tf, p)), 2) for p in (10, 90)]}))
