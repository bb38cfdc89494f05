#!/bin/bash
# ms/step of the C2 bench, repeated (development aid): quick_bench.sh [runs] [extra bench args]
n=${1:-3}; shift
for i in $(seq $n); do
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-ray-reuse --no-far-field "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.4f  %s' % (d['ms_per_step'], {k: round(v*1e3,1) for k,v in d['stage_ms'].items()}))"
done
