"""Per-CUDA-source-line aggregation of an ncu --import-source report (stall samples, instructions)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
# optional 5th argument: launch index among the matching kernels (--launch-skip N --launch-count 1)
extra = ['--launch-skip', sys.argv[5], '--launch-count', '1'] if len(sys.argv) > 5 else []
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass', '-k', 'regex:' + kern] + extra,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
fname = '?'
cur = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != '':
        cur = (fname, int(r[0]), r[1][:90])
        continue
    try:
        s = int(r[4] or 0)
        ie = int(r[7] or 0)
        te = int(r[8] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0, 0])
    a[0] += s
    a[1] += ie
    a[2] += te
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print('samples', tot, 'warp-inst', toti)
key = 1 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 0
for k, v in sorted(agg.items(), key=lambda x: -x[1][key])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{100*v[0]/tot:5.1f}% smp {100*v[1]/toti:5.1f}% inst  act={v[2]/max(v[1],1):4.1f}  {k[0]}:{k[1]}  {k[2]}")
