import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np, digen, paper_1204_6255_b200 as di
n = digen.CONFIGS["c5"].n
s, d, _ = digen.make_range_gpu("c5", 0, n)
indeg = torch.bincount(d.long(), minlength=n)
top = int(indeg.max()); L = d.numel()
print("top", top, "L", L, "share", top / L, flush=True)
for w in (0, -1):
    di.set_option("warm", w)
    g = di.Graph(s, d, n)
    o = g.test_perm()
    o = o.cpu().numpy() if hasattr(o, "cpu") else np.asarray(o)
    print("warm", w, "old_of[60:70]", o[60:70], "indeg of old_of[64..]", indeg[torch.from_numpy(o[64:72].astype(np.int64)).cuda()].tolist(), flush=True)
    g.free()
