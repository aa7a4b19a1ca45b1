set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/t2.log 2>&1; tail -3 $O/t2.log
RUN="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 400 $RUN > $O/b2.log 2>&1; head -c 300 $O/b2.log; echo; python - <<'P'
import json;d=json.loads(open('gpurun_out/b2.log').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['phase_ms_per_step']);print(d['mixed']['value'], d['mixed']['roofline']['phase_ms_per_step'])
P
R2="python bench.py --steps 3 --warmup 3 --no-mixed --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_lj_near|k_lj_far|k_build_lj' -s 1 -c 3 -o $O/prof_r2a $R2 > $O/ncu_r2a.log 2>&1; tail -3 $O/ncu_r2a.log
