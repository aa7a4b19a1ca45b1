#!/bin/bash
# On the GPU box: the round's ncu set (scripts/collect_profiles.sh TAG all) turned into the committed
# summaries (scripts/make_profile_summary.py) on the box; the summaries and the per-line hotspot
# tables come back under gpurun_out/prof_TAG/ (the .ncu-rep captures stay on the box: > 64 MiB).
set -u
TAG=${1:-r02}
O=gpurun_out
bash scripts/collect_profiles.sh $TAG all > $O/collect_$TAG.log 2>&1 || { tail -5 $O/collect_$TAG.log; exit 1; }
python scripts/make_profile_summary.py $O/launches_$TAG.csv $O/prof_full_${TAG}_lj.ncu-rep,$O/prof_full_${TAG}_bond.ncu-rep $TAG \
  $O/flops_fp64_$TAG.csv $O/flops_mixed_$TAG.csv > $O/summary_$TAG.log 2>&1
mkdir -p $O/prof_$TAG
cp profiles/*_$TAG.* $O/prof_$TAG/ 2>/dev/null
for k in k_lj_far k_lj_near; do python scripts/ncu_lines.py $O/prof_full_${TAG}_lj.ncu-rep $k 45 > $O/prof_$TAG/ncu_lines_${k}_$TAG.txt 2>&1; done
for k in k_rebo k_bstar_lite k_short; do python scripts/ncu_lines.py $O/prof_full_${TAG}_bond.ncu-rep $k 30 > $O/prof_$TAG/ncu_lines_${k}_$TAG.txt 2>&1; done
mkdir -p /tmp/reps && mv $O/*.ncu-rep /tmp/reps/
ls -la $O/prof_$TAG
