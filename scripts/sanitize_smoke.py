"""Small end-to-end workload for compute-sanitizer runs: query, train_step,
train_frame, train_backward/apply, encode, assemble_targets, query_accumulate
on small sizes at hidden width 64 (default training path), training at width
32 and 128.  NRC_SANITIZE_MIN=1: query + one train step only (memcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nrc_inputs, paper_2106_12372_b200 as nrc
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
c = nrc.RadianceCache()
recs = nrc_inputs.records(1000, seed=1)
q = c.query(dev(recs))
tr, tg = nrc_inputs.train_frame(0, n=4096)
c.train_step(dev(tr[:300]), dev(tg[:300]))
if os.environ.get("NRC_SANITIZE_MIN", "0") == "1":
    torch.cuda.synchronize()
    print("sanitize workload (min) ok", float(q.sum()))
    sys.exit(0)
c.train_frame(dev(tr), dev(tg), 4, 1024, 3)
g, l = c.train_backward(dev(tr[:300]), dev(tg[:300]))
c.train_apply(g, 300)
e = c.encode(dev(recs))
first, length, flags, vert, vrec, trec = nrc_inputs.training_paths(2000, seed=3)
i32 = lambda x: torch.from_numpy(x.astype(np.int32)).cuda()
t = c.self_training_targets(i32(first), i32(length), i32(flags), dev(vert), dev(trec))
img = torch.zeros((1000, 3), device="cuda")
c.query_accumulate(dev(recs), i32(np.arange(1000)), dev(np.ones((1000, 3), np.float32)), img)
for hw, nh in ((32, 5), (128, 5), (64, 2), (32, 8)):  # width / depth variants (streamed weights at 128)
    cw = nrc.RadianceCache(nrc.Config(hidden_width=hw, n_hidden_layers=nh))
    cw.train_frame(dev(tr), dev(tg), 2, 300, 5)
    cw.query(dev(recs))
big = nrc_inputs.train_frame(1, n=40000)  # > 148 tiles: the single-schedule partials kernel
c.train_step(dev(big[0]), dev(big[1]))
cd = nrc.RadianceCache()  # fused peer all-reduce path at world 1 (hand-off kernel, table-driven optimiser)
cd.train_frame_dp_peer(dev(tr), dev(tg), 2, 1024, 7, 0, 1, [cd.state_ptr])
torch.cuda.synchronize()
print("sanitize workload ok", float(q.sum()), float(t.sum()), float(img.sum()))
