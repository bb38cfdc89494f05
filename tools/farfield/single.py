"""One open patch (one boundary cycle), queries at R/rho = 15..60 (development aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s = scenes.make(1, 16)
sc = G.Scene(s.ctrl)
print("far cycles", sc.n_far_cycles)
rng = np.random.default_rng(0)
c = s.ctrl.reshape(-1, 3).mean(0)
out = []
for R in (8, 12, 20, 40):
    u = rng.normal(size=(256, 3)); u /= np.linalg.norm(u, axis=1)[:, None]
    out.append(c + R * u)
q = np.concatenate(out)
w, st = G.winding_numbers(sc, torch.from_numpy(q).cuda())
np.save(sys.argv[1], np.stack([w.cpu().numpy(), st.cpu().numpy()]))
print(sc.stats()["far_pairs"])
