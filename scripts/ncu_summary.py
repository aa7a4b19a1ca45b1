"""Summarise an ncu report: key metrics per kernel + hottest SASS regions (stall samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy', 'Compute (SM) Throughput',
        'Memory Throughput', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Executed Ipc Active',
        'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp', 'Executed Instructions',
        'Branch Efficiency']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
idx = {n: i for i, n in enumerate(hdr)}
seen = set()
for r in rows[1:]:
    k = r[idx['Kernel Name']][:30]
    m = r[idx['Metric Name']]
    if m in want and (k, m) not in seen:
        seen.add((k, m))
        print(f'{k:30s} {m:38s} {r[idx["Metric Value"]]:>14s} {r[idx["Metric Unit"]]}')
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
for key in ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__average_warp_latency_issue_stalled',
            'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
            'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum', 'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum',
            'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum']:
    for j, n in enumerate(h):
        if n == key:
            for r in rr[2:]:
                print(f'{r[4][:30]:30s} {key:60s} {r[j]} {rr[1][j]}')
# stall reasons
for j, n in enumerate(h):
    if n.startswith('smsp__pcsamp_warps_issue_stalled_') and not n.endswith('not_issued'):
        vals = [r[j] for r in rr[2:]]
        try:
            if max(float(v.replace(',', '')) for v in vals) > 0:
                print(f'stall {n[34:]:40s} {vals}')
        except ValueError:
            pass
