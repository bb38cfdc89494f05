import sys
sys.path.insert(0,'.')
import torch, os
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s = scenes.make(5, 8388608)
sc = G.Scene(s.ctrl)
q = torch.from_numpy(s.queries).cuda()
for _ in range(2):
    w, st = G.winding_numbers(sc, q)
torch.cuda.synchronize()
