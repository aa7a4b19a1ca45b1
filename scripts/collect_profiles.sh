#!/bin/bash
# Round-end ncu set, run on the GPU box from the repo root (bash scripts/collect_profiles.sh TAG PART):
# the launch list of a short bench.py run of the default bench workload (cfg4, 1,008,000-atom PE;
# gpu__time_duration, --clock-control none: cold-cache, serialised -- compare shares), the FP64 /
# FP32 instruction-count passes (fp64 and mixed) and `--set full` captures of the hot kernels that
# scripts/make_profile_summary.py turns into profiles/ncu_summary_TAG.json.  A gpurun call returns
# at most 64 MiB, so the --set full captures come in two parts: PART = base (launch list + flop
# passes), lj (near / far LJ), bond (short list, REBO batches, b* plateau batch), or all.  Every
# ncu pass profiles a command that first exits 0 without ncu.
set -u
TAG=${1:-r02}
PART=${2:-all}
O=gpurun_out
mkdir -p $O
RUN="python bench.py --steps 3 --warmup 3 --no-mixed --no-e2e --no-cpu-baseline"
K='regex:k_lj_near|k_lj_far|k_bstar_lite|k_rebo|k_short'
FL=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,gpu__time_duration.sum
$RUN > $O/plain_$TAG.json 2> $O/plain_$TAG.err || { echo "plain run failed"; exit 1; }
if [ $PART = all ] || [ $PART = base ]; then
  $RUN --precision mixed > $O/plain_mixed_$TAG.json 2> $O/plain_mixed_$TAG.err || { echo "plain mixed run failed"; exit 1; }
  ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_$TAG.csv $RUN > $O/ncu_ll_$TAG.log 2>&1
  ncu --metrics $FL --clock-control none -k "$K" -s 40 -c 12 --csv --log-file $O/flops_fp64_$TAG.csv $RUN > $O/ncu_f64_$TAG.log 2>&1
  ncu --metrics $FL --clock-control none -k "$K" -s 40 -c 12 --csv --log-file $O/flops_mixed_$TAG.csv $RUN --precision mixed > $O/ncu_f32_$TAG.log 2>&1
fi
if [ $PART = all ] || [ $PART = lj ]; then
  ncu --set full --import-source on --clock-control none -k 'regex:k_lj_near|k_lj_far' -s 2 -c 2 -o $O/prof_full_${TAG}_lj $RUN > $O/ncu_full_${TAG}_lj.log 2>&1
fi
if [ $PART = all ] || [ $PART = bond ]; then
  ncu --set full --import-source on --clock-control none -k 'regex:k_bstar_lite|k_rebo|k_short' -s 12 -c 6 -o $O/prof_full_${TAG}_bond $RUN > $O/ncu_full_${TAG}_bond.log 2>&1
fi
ls -la $O | grep $TAG
