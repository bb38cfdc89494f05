"""Which batch sizes change one query's far-field result (development aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s = scenes.make(3, 1 << 14)
sc = G.Scene(s.ctrl)
q = torch.from_numpy(s.queries).cuda()
w2, _ = G.winding_numbers(sc, q)
w2 = w2.cpu().numpy()
i = int(sys.argv[1]) if len(sys.argv) > 1 else 161
for k in (1, 2, 31, 32, 33, 64, 127, 128, 129, 256, 1000, 4096):
    for off in (0, 1, 5):
        a = max(0, i - off)
        w, _ = G.winding_numbers(sc, q[a:a + k], index_base=a)
        print(k, off, repr(w.cpu().numpy()[i - a]) if i - a < k else None, repr(w2[i]))
