set -u
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gt_full.log 2>&1; tail -5 $O/gt_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > $O/b_head.log 2>&1; tail -c 600 $O/b_head.log
