#!/bin/bash
# ncu capture of selected kernels of a short cfg4 bench run, post-processed on the GPU box into text
# (the .ncu-rep stays in /tmp: gpurun returns at most 64 MiB).  usage: bash scripts/gpu_prof.sh TAG KREGEX SKIP COUNT [bench args]
set -u
TAG=$1; K=$2; S=$3; C=$4; shift 4
O=gpurun_out; mkdir -p $O
RUN="python bench.py --steps 3 --warmup 3 --no-mixed --no-e2e --no-cpu-baseline $*"
timeout 300 $RUN > $O/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -5 $O/plain_$TAG.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_$TAG.csv $RUN > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s $S -c $C -o /tmp/prof_$TAG $RUN > $O/ncu_$TAG.log 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > $O/details_$TAG.csv 2>&1
for k in $(echo $K | tr '|' ' '); do
  python scripts/ncu_lines.py /tmp/prof_$TAG.ncu-rep "$k" 45 > $O/lines_${k}_$TAG.txt 2>&1
done
ls -la $O | grep $TAG
