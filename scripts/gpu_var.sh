#!/bin/bash
# parity file(s) then bench.py (cfg4, 100 steps, fp64) for the main build and the given variants
set -u
O=gpurun_out; mkdir -p $O
T=${TESTS:-tests/test_gpu_parity.py}
if [ "$T" != none ]; then timeout 900 python -m pytest $T -x -q > $O/tv.log 2>&1; tail -3 $O/tv.log; fi
bash scripts/bench_variants.sh "$@"
