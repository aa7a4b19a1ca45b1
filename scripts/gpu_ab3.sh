# alternating A/B of two engine libraries (fp64 cfg4, 100 steps, 3 pairs)
set -u
O=gpurun_out; mkdir -p $O
RUN="python bench.py --steps 100 --warmup 5 --no-mixed --no-e2e --no-cpu-baseline"
A=${1:-var/lib_old.so}; B=${2:-paper_1810_07026_b200/libairebo_b200.so}
for rep in 1 2 3; do for L in $A $B; do n=$(basename $L .so)
AIREBO_B200_LIB=$L timeout 400 $RUN > $O/ab3_${n}_${rep}.log 2>&1
python -c "import json;d=json.loads(open('$O/ab3_${n}_${rep}.log').read().strip().splitlines()[-1]);ph=d['roofline']['phase_ms_per_step'];print('$n', round(d['value']/1e6,2), round(d['ms_per_step'],4), 'far',round(ph['lj_far'],4),'near',round(ph['lj_near'],4),'rebo',round(ph['rebo'],4))"
done; done
