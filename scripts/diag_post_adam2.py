"""Diagnostic: post-Adam conditioning at W=128, n=20,000 (the multi-tile
width test): per threshold tau on |g_ref| (batch-mean gradient), the fraction
of entries below it and the worst post-Adam error over sign-agreeing entries
above it; plus the worst entry's values."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import nrc_inputs
import oracle as orc
import paper_2106_12372_b200 as nrc
from parity import offsets_w

for hw, n, seed in [(128, 20000, 8), (64, 40000, 8), (32, 40000, 8), (64, 256, 0)]:
    c = nrc.RadianceCache(nrc.Config(hidden_width=hw))
    recs, tg = nrc_inputs.train_frame(seed, n=n, noise=0.3)
    oc = orc.OracleCache(W32=c.get_params("train"), hidden_width=hw)
    d_r, d_t = torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda()
    g, _ = c.train_backward(d_r, d_t)
    g = g.cpu().numpy().astype(np.float64) / n
    c.train_step(d_r, d_t)
    _, G = oc.train_step(recs, tg, return_grad=True)
    w = c.get_params("train").astype(np.float64)
    off = offsets_w(hw)
    print(f"== W={hw} n={n}")
    for tau in [0, 1e-7, 3e-7, 1e-6, 3e-6, 1e-5]:
        ill = (np.abs(G) <= tau) & ~((G == 0) & (g == 0))
        errs = []
        for i in range(len(off) - 1):
            s = slice(off[i], off[i + 1])
            agree = (np.sign(g[s]) == np.sign(G[s])) & ~ill[s]
            d = np.abs(w[s] - oc.w[s])[agree]
            errs.append(d.max() / np.abs(oc.w[s]).max() if d.size else 0)
        print(f"tau {tau:.0e}: ill frac {ill.mean():.4f}  max err {max(errs):.4f}  per matrix {np.round(errs, 4)}")
    agree = (np.sign(g) == np.sign(G))
    d = np.where(agree, np.abs(w - oc.w), 0)
    k = int(np.argmax(d))
    print("worst entry", k, "g_ref", G[k], "g_gpu", g[k], "dw", d[k])
