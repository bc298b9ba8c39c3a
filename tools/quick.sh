#!/bin/bash
# usage: tools/quick.sh [configs...] -> device-only bench lines (phases) per config, for iteration
mkdir -p gpurun_out
for c in "${@:-C4 C5}"; do
  python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 2>gpurun_out/quick_$c.err | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('$c', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['phases_ms'].items()}, 'frac', round(d['roofline']['frac'],4))" || tail -5 gpurun_out/quick_$c.err
done
