"""Probe: query and frame training on two streams at once, with the query
grid capped (NRC_QUERY_CTAS) so the training kernel (NRC_TRAIN_CTAS CTAs)
finds free SMs.  Timing only (no EMA double buffering here)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs, paper_2106_12372_b200 as nrc
recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
c = nrc.RadianceCache()
out = torch.empty((recs.shape[0], 3), device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def seq():
    c.query(recs, out); c.train_frame(tr, tg, 4, 16384, 1)
def par():
    ev = torch.cuda.Event(); ev.record()
    s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s2):
        c.train_frame(tr, tg, 4, 16384, 1, stream=s2)
    with torch.cuda.stream(s1):
        c.query(recs, out, stream=s1)
    e1 = torch.cuda.Event(); e2 = torch.cuda.Event()
    e1.record(s1); e2.record(s2)
    torch.cuda.current_stream().wait_event(e1); torch.cuda.current_stream().wait_event(e2)
def timeit(fn, reps=30):
    for _ in range(5): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))
print(json.dumps({"q": os.environ.get("NRC_QUERY_CTAS"), "t": os.environ.get("NRC_TRAIN_CTAS"),
                  "query_us": timeit(lambda: c.query(recs, out)),
                  "train_us": timeit(lambda: c.train_frame(tr, tg, 4, 16384, 1)),
                  "seq_us": timeit(seq), "par_us": timeit(par)}))
