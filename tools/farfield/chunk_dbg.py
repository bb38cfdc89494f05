"""Chunked vs unchunked eval with the far field (development aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s = scenes.make(3, 1 << 14)
sc = G.Scene(s.ctrl)
w2, st2 = G.winding_numbers(sc, s.queries)
r2 = sc.stats()["retried"]
for cq in (1000, 4096):
    sc2 = G.Scene(s.ctrl, chunk_queries=cq)
    w3, st3 = G.winding_numbers(sc2, s.queries)
    d = np.abs(w3 - w2)
    idx = np.nonzero(d > 0)[0]
    print(cq, "ndiff", len(idx), "max", d.max(), "retried", r2, sc2.stats()["retried"], "first", idx[:8])
# single-query evals of the differing ones
for i in idx[:4]:
    w1, _ = G.winding_numbers(sc, s.queries[i:i+1], index_base=int(i))
    print(i, repr(w2[i]), repr(w3[i]), repr(w1[0]))
