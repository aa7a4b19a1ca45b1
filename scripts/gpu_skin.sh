#!/bin/bash
# parity file, cfg4 bench, then the cfg4 skin sweep (diag_skin.py)
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/tv.log 2>&1; tail -2 $O/tv.log
bash scripts/bench_variants.sh
timeout 900 python scripts/diag_skin.py 4 fp64 ${SKINS:-0.8,1.0,1.3,1.6,2.0} 2>&1 | tail -8
