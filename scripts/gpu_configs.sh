#!/bin/bash
# bench.py on every BASELINE config (fp64 + mixed sub-line), lines under gpurun_out/configs_TAG/
set -u
TAG=${1:-r02}
O=gpurun_out/configs_$TAG; mkdir -p $O
for c in 1 2 3 5a 5b; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
  python -c "
import json;d=json.loads(open('$O/bench_cfg$c.json').read().strip().splitlines()[-1]);print('$c', d['config']['atoms'], round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['mixed']['value']/1e6,2) if d.get('mixed') else None, d['counters'].get('timed_rebuilds'))"
done
