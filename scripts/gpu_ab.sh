# A/B of engine variants on cfg4: AB_REBO_G4 off / on (in-tree lib) and extra libs given as args
set -u
O=gpurun_out; mkdir -p $O
RUN="python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline"
summ() { python - "$1" <<'P'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);ph=d['roofline']['phase_ms_per_step']
print(sys.argv[1], round(d['value']/1e6,2), round(d['ms_per_step'],4), {k:round(v,4) for k,v in ph.items()}, 'mixed', round(d['mixed']['value']/1e6,2), round(d['mixed']['roofline']['phase_ms_per_step']['rebo'],4))
P
}
AB_REBO_G4=0 timeout 400 $RUN > $O/ab_g0.log 2>&1; summ $O/ab_g0.log
timeout 400 $RUN > $O/ab_g1.log 2>&1; summ $O/ab_g1.log
for L in "$@"; do n=$(basename $L .so); AIREBO_B200_LIB=$L timeout 400 $RUN > $O/ab_$n.log 2>&1; summ $O/ab_$n.log; done
