# alternating A/B of AB_REBO_G4 (3 pairs, 100 steps each, fp64 only), then ncu of k_build_lj
set -u
O=gpurun_out; mkdir -p $O
RUN="python bench.py --steps 100 --warmup 5 --no-mixed --no-e2e --no-cpu-baseline"
for rep in 1 2 3; do for g in 0 1; do
AB_REBO_G4=$g timeout 400 $RUN > $O/ab2_${g}_${rep}.log 2>&1
python -c "import json;d=json.loads(open('$O/ab2_${g}_${rep}.log').read().strip().splitlines()[-1]);print('g4=$g', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['phase_ms_per_step']['rebo'],4))"
done; done
R2="python bench.py --steps 3 --warmup 3 --no-mixed --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_build_lj -c 1 -o /tmp/prof_bl $R2 > $O/ncu_bl.log 2>&1; tail -2 $O/ncu_bl.log
ncu -i /tmp/prof_bl.ncu-rep --page details --csv > $O/prof_bl.csv 2>/dev/null; python scripts/ncu_lines.py /tmp/prof_bl.ncu-rep k_build_lj 40 > $O/lines_bl.txt 2>&1
