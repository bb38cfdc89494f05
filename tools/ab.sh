timeout 900 python -m pytest tests/test_gpu_farfield.py -x -q 2>&1 | tail -3
python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s=scenes.make(5, 1<<23); sc=G.Scene(s.ctrl); q=torch.from_numpy(s.queries).cuda()
G.winding_numbers(sc,q); torch.cuda.synchronize()
sc.set_timing(True); G.winding_numbers(sc,q); st=sc.stats()
print({k: st[k] for k in ['near_pairs','far_pairs','shadow_pairs','far_terms','boundary_segments','ms_k4_far','ms_k4_exact','ms_boundary']})
"
