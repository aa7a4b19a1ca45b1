# alternating A/B of N engine libraries (fp64 cfg4, 100 steps): bash scripts/gpu_abn.sh REPS lib1.so lib2.so ...
set -u
O=gpurun_out; mkdir -p $O
REPS=$1; shift
RUN="python bench.py --steps 100 --warmup 5 --no-mixed --no-e2e --no-cpu-baseline"
for rep in $(seq 1 $REPS); do for L in "$@"; do n=$(basename $(dirname $L))
AIREBO_B200_LIB=$L timeout 400 $RUN > $O/abn_${n}_${rep}.log 2>&1
python -c "import json;d=json.loads(open('$O/abn_${n}_${rep}.log').read().strip().splitlines()[-1]);ph=d['roofline']['phase_ms_per_step'];print('$n', round(d['value']/1e6,2), round(d['ms_per_step'],4), 'far',round(ph['lj_far'],4),'near',round(ph['lj_near'],4),'rebo',round(ph['rebo'],4),'rebuild',round(ph['rebuild'],4),'short',round(ph['short'],4),'bstar',round(ph['bstar'],4))"
done; done
