for v in main "$@"; do
  if [ $v = main ]; then unset AIREBO_B200_LIB; else export AIREBO_B200_LIB=build_variants/$v/libairebo_b200.so; fi
  timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-mixed > gpurun_out/bench_var_$v.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/bench_var_$v.json').read().strip().splitlines()[-1]);ph=d['roofline']['phase_ms_per_step'];print('$v', round(d['value']/1e6,2), round(d['ms_per_step'],4), {k:round(v,4) for k,v in ph.items()})"
done
