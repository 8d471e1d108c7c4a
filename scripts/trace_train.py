"""Phase trace of the train kernel (CTA 0) via nrc_debug_set_trace (32 slots
per fused step), plus event timing of one training frame."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs, paper_2106_12372_b200 as nrc
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
c = nrc.RadianceCache()
buf = torch.zeros(256 + 8 * 256, dtype=torch.int64, device="cuda")
c.L.nrc_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
c.L.nrc_debug_set_trace(c.h, ctypes.c_void_p(buf.data_ptr()))
for _ in range(5):
    c.train_frame(tr, tg, 4, 16384, 1)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); c.train_frame(tr, tg, 4, 16384, 1); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(f"train_frame median {np.median(ts):.1f} us (single call: includes host submission)")
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    c.train_frame(tr, tg, 4, 16384, 1)
b.record(); torch.cuda.synchronize()
print(f"train_frame back-to-back {a.elapsed_time(b) * 1e3 / 20:.1f} us/frame")
d = buf.cpu().numpy(); t0 = d[0]
names = {0: "start", 1: "setup done", 2: "records gathered", 3: "weights resident", 4: "encoded",
         10: "loss", 11: "bwd layer 5", 16: "bwd final", 30: "partials stored", 17: "grid sync 1",
         18: "partials summed", 19: "adam done", 20: "grid sync 2", 21: "weights reloaded"}
for step in range(4):
    print(f"--- step {step}")
    for i in [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 30, 17, 18, 19, 20, 21]:
        if step == 0 or i != 3:
            v = d[32 * step + i]
            nm = names.get(i, f"fwd L{i-5}" if i < 10 else f"bwd round i={16-i}")
            print(f"{nm:24s} {int(v - t0):8d}")
print(f"{'end':24s} {int(d[3 * 32 + 31] - t0):8d}")

# per-CTA global-timer marks of step 1 (ns): 6 step start, 0 tiles done, 1 partials
# written, 2 after barrier 1, 3 optimiser done, 4 after barrier 2, 5 weights reloaded
g = d[256:].reshape(-1, 8)
g = g[g[:, 6] != 0]
base = g[:, 6].min()
print(f"CTAs traced: {len(g)}")
for k, nm in [(6, "step start"), (0, "tiles done"), (1, "partials written"), (2, "after barrier 1"),
              (3, "optimiser done"), (4, "after barrier 2"), (5, "weights reloaded")]:
    col = g[:, k] - base
    print(f"{nm:20s} min {col.min():6d} med {int(np.median(col)):6d} max {col.max():6d} ns  argmax cta {int(np.argmax(col))}")
