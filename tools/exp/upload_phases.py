"""Upload (DI_HOST_PTRS: H2D + build) of C4 from pinned host memory, per builder, with the
build_trace option's phase timestamps on stderr: python tools/exp/upload_phases.py [config]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
sp, dp = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
for rs in (1, 0, 1, 0):
    di.set_option("row_sort", rs)
    for k in range(4):
        di.set_option("build_trace", 1 if k == 3 else 0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        g = di.Graph(sp, dp, n)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        print(f"row_sort={rs} upload {ms:.1f} ms", flush=True)
        g.free()
