# far-field vs exact K4 on configs (development aid): cmp.sh nq cfg...
nq=$1; shift
for c in "$@"; do
  GWN_FARFIELD=0 timeout 600 python tools/farfield/check.py $c $nq gpurun_out/ex$c.npz
  timeout 600 python tools/farfield/check.py $c $nq gpurun_out/ff$c.npz
  python - <<PY
import numpy as np
a=np.load("gpurun_out/ex$c.npz"); b=np.load("gpurun_out/ff$c.npz")
ok=(a["st"]==0)&(b["st"]==0)
print("cfg$c max|dw|", np.abs(a["w"]-b["w"])[ok].max(), "status equal", (a["st"]==b["st"]).all(), "bitwise", np.array_equal(a["w"],b["w"]))
PY
done
