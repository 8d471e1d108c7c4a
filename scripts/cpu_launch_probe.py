"""Is the training frame CPU-submission-bound?  CPU wall time of one
train_frame call (enqueue only) and its device time when the queue is
pre-filled with a sleep kernel (the GPU cannot overtake the CPU)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs, paper_2106_12372_b200 as nrc
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
c = nrc.RadianceCache()
for _ in range(10):
    c.train_frame(tr, tg, 4, 16384, 1)
torch.cuda.synchronize()
cpu, dev_free, dev_pref = [], [], []
for _ in range(30):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); t0 = time.perf_counter(); c.train_frame(tr, tg, 4, 16384, 1); t1 = time.perf_counter(); b.record()
    torch.cuda.synchronize(); cpu.append((t1 - t0) * 1e6); dev_free.append(a.elapsed_time(b) * 1e3)
    torch.cuda._sleep(2_000_000)  # ~1 ms of GPU work queued first
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); c.train_frame(tr, tg, 4, 16384, 1); b.record()
    torch.cuda.synchronize(); dev_pref.append(a.elapsed_time(b) * 1e3)
print(json.dumps({"cpu_enqueue_us": float(np.median(cpu)), "device_us_alone": float(np.median(dev_free)),
                  "device_us_prefilled_queue": float(np.median(dev_pref)), "launches": c.last_launch_count}))
