"""Probe: device time of the optimiser kernel alone (nrc_train_apply: logical
gradient in, no partials) and of partials kernel + reduce (train_backward),
back to back on the stream, per call."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import nrc_inputs, paper_2106_12372_b200 as nrc
c = nrc.RadianceCache()
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr[:16384]).cuda(), torch.from_numpy(tg[:16384]).cuda()
g, _ = c.train_backward(tr, tg)
for name, fn in [("apply", lambda: c.train_apply(g, 16384)), ("backward", lambda: c.train_backward(tr, tg, grad=g)),
                 ("step", lambda: c.train_step(tr, tg))]:
    for _ in range(10): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, "us per call", round(1e3 * e0.elapsed_time(e1) / 200, 2))
