#!/bin/bash
# Round-end ncu set, run on the GPU box from the repo root (bash scripts/collect_profiles.sh TAG):
# the launch list of a short bench.py run (gpu__time_duration, --clock-control none: cold-cache,
# serialised; compare shares) of the default bench workload (cfg4, 1,008,000-atom PE), one `--set full` capture of each hot kernel and the FP64 / FP32
# instruction-count passes (fp64 and mixed) that scripts/make_profile_summary.py turns into
# profiles/ncu_summary_TAG.json.  Every ncu pass profiles a command that first exits 0 without ncu.
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
RUN="python bench.py --steps 3 --warmup 3 --no-mixed --no-e2e --no-cpu-baseline"
K='regex:k_lj_near|k_lj_far|k_bstar|k_rebo|k_short'
FL=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,gpu__time_duration.sum
$RUN > $O/plain_$TAG.json 2> $O/plain_$TAG.err || { echo "plain run failed"; exit 1; }
$RUN --precision mixed > $O/plain_mixed_$TAG.json 2> $O/plain_mixed_$TAG.err || { echo "plain mixed run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_$TAG.csv $RUN > $O/ncu_ll_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k "$K" -s 20 -c 6 -o $O/prof_full_$TAG $RUN > $O/ncu_full_$TAG.log 2>&1
ncu --metrics $FL --clock-control none -k "$K" -s 40 -c 12 --csv --log-file $O/flops_fp64_$TAG.csv $RUN > $O/ncu_f64_$TAG.log 2>&1
ncu --metrics $FL --clock-control none -k "$K" -s 40 -c 12 --csv --log-file $O/flops_mixed_$TAG.csv $RUN --precision mixed > $O/ncu_f32_$TAG.log 2>&1
ls -la $O | grep $TAG
