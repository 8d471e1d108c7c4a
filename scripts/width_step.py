"""One 1080p frame (query + 4 x 16,384 train) at hidden width argv[1] after
warm-up; for ncu (scripts/ncu_width.sh).  argv[2] == 'f': W = 64 through the
fused cooperative training kernel (NRC_TRAIN_FUSED=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import nrc_inputs
import paper_2106_12372_b200 as nrc

hw = int(sys.argv[1])
if len(sys.argv) > 2 and sys.argv[2] == "f":
    os.environ["NRC_TRAIN_FUSED"] = "1"
c = nrc.RadianceCache(nrc.Config(hidden_width=hw))
recs = torch.from_numpy(nrc_inputs.records(nrc_inputs.N_1080P)).cuda()
tr, tg = nrc_inputs.train_frame(0, noise=0.3)
tr, tg = torch.from_numpy(tr).cuda(), torch.from_numpy(tg).cuda()
for _ in range(3):
    c.query(recs)
    c.train_frame(tr, tg, 4, 16384, 1)
torch.cuda.synchronize()
