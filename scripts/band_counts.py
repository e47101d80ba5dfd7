import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1706_02740_b200 as d
from dsft_synth import planted
N, s = 2**26, 1000
pl = planted(N, s, cfg=2, trial=0)
f = torch.from_numpy(pl.f).cuda()
plan = d.Plan(N, s)
fr = torch.empty(s, dtype=torch.int64, device="cuda"); co = torch.empty(s, dtype=torch.complex128, device="cuda")
plan.dsft_execute(f, fr, co)
torch.cuda.synchronize()
bn = torch.empty(256, dtype=torch.int32, device="cuda")
plan.dsft_debug_copy(1, bn)
torch.cuda.synchronize()
print("band_n", bn.cpu().numpy()[:plan.info.J].tolist())
