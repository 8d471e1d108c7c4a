"""Diagnostic: post-Adam parity statistics at C1 (fraction of exact-zero and
near-zero gradient entries, flips, per-matrix errors with / without the
near-zero exclusion)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import nrc_inputs
import oracle as orc
import paper_2106_12372_b200 as nrc

recs, tg = nrc_inputs.train_frame(0, n=256, noise=0.3)
cache = nrc.RadianceCache()
oc = orc.OracleCache(W32=cache.get_params("train"))
g_gpu, _ = cache.train_backward(torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda())
g_gpu = g_gpu.cpu().numpy().astype(np.float64) / 256.0
cache.train_step(torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda())
l_ref, G = oc.train_step(recs, tg, return_grad=True)
w = cache.get_params("train").astype(np.float64)
print("zero ref", np.mean(G == 0), "zero gpu", np.mean(g_gpu == 0), "both zero", np.mean((G == 0) & (g_gpu == 0)))
near = (np.abs(G) <= 1e-7) & (G != 0)
print("near-zero nonzero ref", near.mean())
print("ref zero & gpu nonzero", np.mean((G == 0) & (g_gpu != 0)), "max |g_gpu| there", np.max(np.abs(g_gpu[(G == 0)])) if (G == 0).any() else 0)
dw = np.abs(w - oc.w)
for name, m in [("all", np.ones_like(G, bool)), ("near", near), ("zero", G == 0)]:
    if m.any():
        print(name, "max |dw|", dw[m].max(), "max|w|", np.abs(oc.w).max())
from parity import OFF
for i in range(6):
    s = slice(OFF[i], OFF[i + 1])
    print(i, "zero", np.mean(G[s] == 0), "near", near[s].mean(), "maxdw", dw[s].max() / np.abs(oc.w[s]).max())
