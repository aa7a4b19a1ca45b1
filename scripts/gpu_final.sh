#!/bin/bash
# Round-end set on the GPU box: GPU tests, smoke, the default bench line and the reference arm,
# the ncu set (scripts/gpu_final_profiles.sh) and the other BASELINE configs; results under gpurun_out/.
set -u
TAG=${1:-r02}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gt_full.log 2>&1; tail -3 $O/gt_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; tail -c 300 $O/bench_$TAG.json
timeout 900 python bench.py --impl reference > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err; tail -c 300 $O/bench_ref_$TAG.json
bash scripts/gpu_final_profiles.sh $TAG
bash scripts/gpu_configs.sh $TAG
