set -u
O=gpurun_out; mkdir -p $O
R2="python bench.py --steps 3 --warmup 3 --no-mixed --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rebo_g4 -s 4 -c 1 -o /tmp/prof_g4 $R2 > $O/ncu_g4.log 2>&1; tail -2 $O/ncu_g4.log
AB_REBO_G4=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rebo -s 16 -c 1 -o /tmp/prof_g0 $R2 > $O/ncu_g0.log 2>&1; tail -2 $O/ncu_g0.log
for f in g4 g0; do ncu -i /tmp/prof_$f.ncu-rep --page details --csv > $O/prof_$f.csv 2>/dev/null; python scripts/ncu_lines.py /tmp/prof_$f.ncu-rep k_rebo 40 > $O/lines_$f.txt 2>&1; done
ls -la $O
