"""Scene creation of a config, timed (development aid): total wall time and
the local-expansion octree's build (gwn_fmm.cu)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2408_04466_b200 as G  # noqa: E402
from paper_2408_04466_b200 import scenes  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s = scenes.make(cfg, 8)
torch.cuda.init()
G.Scene(scenes.make(1, 8).ctrl)
for _ in range(2):
    t = time.perf_counter()
    sc = G.Scene(s.ctrl)
    torch.cuda.synchronize()
    print(f"scene create {time.perf_counter() - t:.3f} s  {sc.local_expansions}", flush=True)
