"""Probe: device time of one 4-step training frame launched normally vs as a
captured CUDA graph (same kernels and PDL edges; the graph's arguments are
frozen, so this is a timing probe only)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs, paper_2106_12372_b200 as nrc
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
c = nrc.RadianceCache()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        c.train_frame(tr, tg, 4, 16384, 1, stream=s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    c.train_frame(tr, tg, 4, 16384, 1, stream=s)
torch.cuda.synchronize()
def t(fn, reps=30):
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(2_000_000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))
print(json.dumps({"stream_us": t(lambda: c.train_frame(tr, tg, 4, 16384, 1)), "graph_us": t(lambda: g.replay())}))
