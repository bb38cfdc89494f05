"""Far-field K4 vs exact K4 (development aid): python check.py <cfg> <nq> <out.npz>;
run twice, with GWN_FARFIELD=0 and without, then compare."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
cfg, nq, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
t0 = time.perf_counter()
s = scenes.make(cfg, nq)
sc = G.Scene(s.ctrl)
t1 = time.perf_counter()
q = torch.from_numpy(s.queries).cuda()
w, st = G.winding_numbers(sc, q)
torch.cuda.synchronize()
sc.set_timing(True)
w, st = G.winding_numbers(sc, q)
stt = sc.stats()

print(f"cfg{cfg} nq={nq} scene {t1-t0:.2f}s far_cycles={getattr(sc, 'n_far_cycles', '?')} "
      f"boundary {stt['ms_boundary']:.3f} ms segs={stt['boundary_segments']} far_pairs={stt.get('far_pairs')}",
      flush=True)
np.savez(out, w=w.cpu().numpy(), st=st.cpu().numpy())
