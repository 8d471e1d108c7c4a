"""Per-round clock64 trace of the TS query kernel (build with NRC_NVCC_DEFINES=NRC_TRACE_QUERY;
CTA 0, group 0, 4 warps):
fields 0 before MMA wait, 1 MMA done, 2 epilogue done, 3 after group barrier,
4 slot*16+layer, 5 encode start, 6 encode done, 7 after encode barrier."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs, paper_2106_12372_b200 as nrc
recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
c = nrc.RadianceCache()
out = torch.empty((recs.shape[0], 3), device="cuda")
buf = torch.zeros(4096 + 3072 + 2 * 96, dtype=torch.int64, device="cuda")
c.L.nrc_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
for _ in range(3):
    c.query(recs, out)
c.L.nrc_debug_set_trace(c.h, ctypes.c_void_p(buf.data_ptr()))
c.query(recs, out)
torch.cuda.synchronize()
bb = buf.cpu().numpy()
d = bb[4096:4096 + 8 * 4 * 96].reshape(96, 4, 8)
iss = bb[4096 + 8 * 4 * 96:].reshape(96, 2)
t0 = d[0, :, 0].min()
print("k  w slot lay | wait0  mmadone  epi_done  bar_done | enc_start enc_done enc_bar   (cycles rel. to first wait)")
for k in range(60):
    for w in range(4):
        f = d[k, w]
        rel = lambda x: int(x - t0) if x else -1
        print(f"{k:2d} {w} {int(f[4]) // 16:2d} {int(f[4]) % 16:3d} | {rel(f[0]):7d} {rel(f[1]):8d} {rel(f[2]):8d} {rel(f[3]):8d} | "
              f"{rel(f[5]):8d} {rel(f[6]):8d} {rel(f[7]):8d}" + (f"  issue {rel(iss[k,0])} -> {rel(iss[k,1])}" if w == 0 else ""))
# summary: per round, MMA wait (f1-f0), epilogue (f2-f1), barrier wait (f3-f2) averaged over warps
mw = d[:60, :, 1] - d[:60, :, 0]
ep = d[:60, :, 2] - d[:60, :, 1]
print("mean MMA-wait per warp-round", float(mw.mean()), " mean epilogue", float(ep.mean()))
