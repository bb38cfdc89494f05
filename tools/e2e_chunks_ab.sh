#!/bin/bash
# e2e (pinned host buffers) vs pipeline chunking (development aid):
# e2e_chunks_ab.sh "CHUNKS:TAIL:AHEAD" ...
cd ${GRAFT_REPO_ROOT:-.}
for ct in "$@"; do
  IFS=: read c t a <<< "$ct"
  for i in 1 2; do
    GWN_PIPE_CHUNKS=$c GWN_PIPE_TAIL=$t GWN_PIPE_AHEAD=$a python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ray-reuse --no-far-field 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $c tail $t ahead $a e2e %.3f G/s  dev %.3f' % (d['e2e']['value']/1e9, d['value']/1e9))"
  done
done
