"""C3 (BASELINE.json configs[2]): 1000 Adam steps of 16,384
fresh records each, fitting the synthetic analytic radiance field, on the GPU
and with the fp64 oracle from the same initial weights.  Writes the two loss
curves and their 50-step windowed ratio as JSON (default
profiles/r01_c3_convergence.json).  The oracle leg is the slow part
(minutes on the host cores).

  python scripts/c3_convergence.py [--steps 1000] [--batch 16384] [--noise 0.3] [--out FILE]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import nrc_inputs
import oracle
import paper_2106_12372_b200 as nrc

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1000)
ap.add_argument("--batch", type=int, default=16384)
ap.add_argument("--noise", type=float, default=0.3)
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_c3_convergence.json"))
args = ap.parse_args()

c = nrc.RadianceCache()
oc = oracle.OracleCache(W32=c.get_params("train"))
lg, lo = [], []
t_gpu = t_orc = 0.0
for j in range(args.steps):
    recs = nrc_inputs.records(args.batch, seed=nrc_inputs.SEED_C3 + j)
    tg = nrc_inputs.targets(recs, noise=args.noise, seed=j)
    d_r, d_t = torch.from_numpy(recs).cuda(), torch.from_numpy(tg).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lg.append(c.train_step(d_r, d_t).item())
    t1 = time.perf_counter()
    lo.append(oc.train_step(recs, tg))
    t2 = time.perf_counter()
    t_gpu += t1 - t0
    t_orc += t2 - t1
lg, lo = np.array(lg), np.array(lo)
win = 50
ratios = [float(lg[w:w + win].mean() / lo[w:w + win].mean()) for w in range(0, args.steps, win)]
q = torch.from_numpy(nrc_inputs.records(8192, seed=12345)).cuda()
qg = c.query(q).cpu().numpy()
qo = oc.query(q.cpu().numpy())
rad = [float(np.max(np.abs(qg[:, k] - qo[:, k])) / max(np.max(np.abs(qo[:, k])), 1e-30)) for k in range(3)]
res = {"config": "C3: 1000 Adam steps x 16384 fresh records, analytic radiance field",
       "steps": args.steps, "batch": args.batch, "noise": args.noise,
       "loss_gpu_first10": lg[:10].tolist(), "loss_oracle_first10": lo[:10].tolist(),
       "first10_max_rel_diff": float(np.max(np.abs(lg[:10] / lo[:10] - 1.0))),
       "windowed_ratio_gpu_over_oracle": ratios, "window": win,
       "loss_gpu_last50": float(lg[-50:].mean()), "loss_oracle_last50": float(lo[-50:].mean()),
       "loss_gpu_first5": float(lg[:5].mean()),
       "final_query_radiance_rel_err_vs_oracle": rad,
       "host_wall_s": {"gpu_steps_incl_copies": t_gpu, "oracle_steps": t_orc},
       "loss_gpu": lg.tolist(), "loss_oracle": lo.tolist()}
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    json.dump(res, f)
print(json.dumps({k: v for k, v in res.items() if k not in ("loss_gpu", "loss_oracle")}))
