"""Global-timer phase trace of the default training path (nrc_train_w_kernel
+ nrc_adam_w_kernel, PDL-chained) over one 4-step frame, via
nrc_debug_set_trace: per step, per-CTA marks 0 start, 1 encoded (before
griddepcontrol.wait), 2 after the wait, 3 forward + loss done, 4 backward
rounds 5..1 done, 5 tile done (G0 drained), 6 loss written, 8+L forward layer
L's MMA done, 14+2(5-j) / 15+2(5-j) backward round j before / after its MMA
wait; Adam blocks 0 and last: start (after wait) / end.  argv[1]: hidden
width (64)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import nrc_inputs
import paper_2106_12372_b200 as nrc

hw = int(sys.argv[1]) if len(sys.argv) > 1 else 64
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
c = nrc.RadianceCache(nrc.Config(hidden_width=hw))
for _ in range(5):
    c.train_frame(tr, tg, 4, 16384, 1)
buf = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")  # adam SM ids at 32768 + 4096 step + block
c.L.nrc_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
c.L.nrc_debug_set_trace(c.h, ctypes.c_void_p(buf.data_ptr()))
torch.cuda.synchronize()
c.train_frame(tr, tg, 4, 16384, 1)
torch.cuda.synchronize()
dall = buf.cpu().numpy()
d = dall[:4 * 4096].reshape(4, 4096)
step0 = c.stats()["step"] - 4
t0 = None
names = {0: "start", 1: "encoded", 2: "after wait", 8: "fwd L0 mma", 9: "fwd L1 mma", 10: "fwd L2 mma",
         11: "fwd L3 mma", 12: "fwd L4 mma", 13: "fwd L5 mma", 3: "fwd+loss"}
for j in range(5, 0, -1):
    names[14 + 2 * (5 - j)] = f"bwd {j} issued"
    names[15 + 2 * (5 - j)] = f"bwd {j} mma"
for j in range(5, 1, -1):
    names[24 + (5 - j)] = f"bwd {j} mask done"
    names[28 + (5 - j)] = f"bwd {j} synced"
names.update({4: "bwd 5..1", 5: "tile done", 6: "loss written"})
order = [0, 1, 2, 8, 9, 10, 11, 12, 13, 3]
for j in range(5, 0, -1):
    order += [14 + 2 * (5 - j), 15 + 2 * (5 - j)] + ([24 + (5 - j), 28 + (5 - j)] if j >= 2 else [])
order += [4, 5, 6]
names = {k: names[k] for k in order}
for k in range(4):
    blk = d[(step0 + k) % 4]
    g = blk[:32 * 127].reshape(127, 32)
    g = g[g[:, 8] != 0]  # (the frame kernel writes mark 0 at its start only)
    if t0 is None:
        t0 = g[:, 0].min() if g[:, 0].min() > 0 else g[:, 8].min()
    print(f"--- step {k} ({len(g)} CTAs), ns from the frame's first CTA start")
    for i, nm in names.items():
        col = g[:, i] - t0
        print(f"  {nm:14s} min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d}")
    st = g[:, 0] - t0
    late = np.nonzero(st > np.median(st) + 1000)[0]
    if len(late) and g[:, 7].max() > 0:  # CTAs starting > 1 us after the median: block index, SM, start
        print("  late CTAs (block, sm, start):", [(int(b), int(g[b, 7]), int(st[b])) for b in late])
        prev = dall[32768 + 4096 * ((step0 + k - 1) % 4):32768 + 4096 * ((step0 + k - 1) % 4) + 4096]
        nblk = int((prev != 0).sum()) + 1
        ad = np.bincount(prev[:nblk], minlength=160)
        early = [int(ad[int(g[b, 7])]) for b in range(len(g)) if b not in set(late)]
        lat = [int(ad[int(g[b, 7])]) for b in late]
        print(f"  previous optimiser blocks on the SM of each early CTA: {np.bincount(early).tolist()}, late CTA: {np.bincount(lat).tolist()}")
        print(f"  optimiser blocks per SM histogram: {np.bincount(ad[:148]).tolist()}")
        res = dall[49152 + 4096 * ((step0 + k - 1) % 4):49152 + 4096 * ((step0 + k - 1) % 4) + nblk] - t0
        print(f"  previous optimiser blocks resident at (ns): min {res.min()} p25 {int(np.percentile(res, 25))} med {int(np.median(res))} p75 {int(np.percentile(res, 75))} max {res.max()}")
    fl = dall[16384 + 4096 * ((step0 + k) % 4):16384 + 4096 * ((step0 + k) % 4) + 32 * 127].reshape(127, 32)
    if fl[:, 8:13].any():  # frame kernel: exchange marks of thread 0
        for m, nm in enumerate(["exchange entry", "barrier A passed", "slice loads done", "adam done", "barrier B passed"]):
            col = fl[:, 8 + m]
            col = col[col != 0] - t0
            if len(col):
                print(f"  {nm:16s} min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d}")
    if fl[:, :8].any():  # NRC_TRACE_FLUSH builds: wgrad_j completion seen by the flush warps
        for j in range(5, -1, -1):
            col = fl[:, j] - t0
            print(f"  wgrad {j} done     min {col.min():7d} med {int(np.median(col)):7d} max {col.max():7d}")
    print(f"  adam blk0 {blk[4088] - t0:7d} -> w0 loads {blk[4086] - t0:7d} -> sum {blk[4084] - t0:7d} -> math "
          f"{blk[4092] - t0:7d} -> {blk[4089] - t0:7d}   last blk {blk[4090] - t0:7d} -> w0 loads {blk[4087] - t0:7d} -> sum "
          f"{blk[4085] - t0:7d} -> math {blk[4093] - t0:7d} -> {blk[4091] - t0:7d}")
c.L.nrc_debug_set_trace(c.h, None)
