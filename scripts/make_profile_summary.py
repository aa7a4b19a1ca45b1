"""Turn ncu outputs from gpurun_out/ into the committed summaries under profiles/.

usage: python scripts/make_profile_summary.py <launch_list.csv> <full.ncu-rep> <round tag>
                                             [<fp64 flops.csv> <mixed flops.csv>]
Writes profiles/launches_<tag>.csv (copy), profiles/launch_shares_<tag>.txt,
profiles/ncu_full_<tag>.txt and profiles/ncu_summary_<tag>.json (per-kernel DRAM bytes per
launch, read by bench.py as roofline.traffic; with the optional metric-pass CSVs also the
hardware FP64 / FP32 flop counts per launch, 2 DFMA + DMUL + DADD (FFMA ...) thread
instructions, read by bench.py as roofline.hw -- SURVEY §8(d) fraction (i)).
"""
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
launch_csv, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)
shutil.copy(launch_csv, os.path.join(prof, f"launches_{tag}.csv"))

rows = list(csv.reader(open(launch_csv)))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
idx = {n: i for i, n in enumerate(rows[h])}
tot = {}
for r in rows[h + 1:]:
    if len(r) < len(rows[h]):
        continue
    name = re.sub(r"\(.*", "", r[idx["Kernel Name"]]).replace("void ", "").strip()
    v = float(r[idx["Metric Value"]].replace(",", ""))
    unit = r[idx["Metric Unit"]]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    if "k_fma_peak" in name:  # the FMA-peak microbenchmark bench.py runs once, not part of a step
        continue
    t = tot.setdefault(name, [0.0, 0])
    t[0] += v
    t[1] += 1
all_us = sum(v[0] for v in tot.values())
with open(os.path.join(prof, f"launch_shares_{tag}.txt"), "w") as f:
    f.write(f"# ncu launch list ({os.path.basename(launch_csv)}): gpu__time_duration.sum per kernel, "
            f"--clock-control none, cold-cache serialised launches; compare SHARES, not absolutes\n")
    f.write(f"{'kernel':60s} {'total_us':>12s} {'launches':>9s} {'avg_us':>9s} {'share':>7s}\n")
    for k, (us, n) in sorted(tot.items(), key=lambda x: -x[1][0]):
        f.write(f"{k[:60]:60s} {us:12.1f} {n:9d} {us / n:9.2f} {100 * us / all_us:6.2f}%\n")

reps = rep.split(",")  # several --set full captures (a gpurun call returns <= 64 MiB)
out = "".join(subprocess.run(["python", os.path.join(ROOT, "scripts", "ncu_summary.py"), r], capture_output=True,
                             text=True).stdout for r in reps)
open(os.path.join(prof, f"ncu_full_{tag}.txt"), "w").write(
    f"# ncu --set full --clock-control none --import-source on (scripts/collect_profiles.sh: short bench.py run, cfg4 (1,008,000-atom PE), fp64)\n" + out)

summ = {"fp64": {}}
for rep1 in reps:
  raw = subprocess.run(["ncu", "-i", rep1, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
  rr = list(csv.reader(raw.splitlines()))
  hdr = rr[0]
  col = {n: i for i, n in enumerate(hdr)}
  for r in rr[2:]:
      kname = re.sub(r"<.*|\(.*", "", r[col["Kernel Name"]]).replace("void ", "").replace("ab::", "").strip()
      d = {}
      for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
          if key in col:
              unit = rr[1][col[key]]
              v = float(r[col[key]].replace(",", ""))
              scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
                       "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
              d[key] = v * scale
      e = summ["fp64"].setdefault(kname, {"launches": 0, "dram_bytes": 0.0, "duration_us": 0.0})
      e["launches"] += 1
      e["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
      e["duration_us"] += d.get("gpu__time_duration.sum", 0)
for e in summ["fp64"].values():
    e["dram_bytes_per_launch"] = e["dram_bytes"] / max(e["launches"], 1)
summ["_note"] = ("ncu --set full capture (cache flushed between replays, i.e. cold-cache DRAM traffic per "
                 "launch) of a short bench.py run on cfg4 (1,008,000-atom PE), fp64 (scripts/collect_profiles.sh)")


def flops_pass(path, prec):
    """per kernel: hardware flops per launch from a --metrics pass CSV (long format)"""
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    idx = {n: i for i, n in enumerate(rows[h])}
    per = {}
    for r in rows[h + 1:]:
        if len(r) < len(rows[h]):
            continue
        kname = re.sub(r"<.*|\(.*", "", r[idx["Kernel Name"]]).replace("void ", "").replace("ab::", "").strip()
        launch = (kname, r[idx["ID"]])
        v = float(r[idx["Metric Value"]].replace(",", ""))
        per.setdefault(launch, {})[r[idx["Metric Name"]]] = v
    out = {}
    for (kname, _), m in per.items():
        if prec == "fp64":
            fl = 2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
        else:
            fl = 2 * m.get("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", 0) + \
                m.get("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", 0)
        e = out.setdefault(kname, {"launches": 0, "hw_flops": 0.0})
        e["launches"] += 1
        e["hw_flops"] += fl
    for e in out.values():
        e["hw_flops_per_launch"] = e["hw_flops"] / max(e["launches"], 1)
    return out


if len(sys.argv) > 5:
    for prec, path in (("fp64", sys.argv[4]), ("mixed", sys.argv[5])):
        for k, v in flops_pass(path, prec).items():
            summ.setdefault(prec, {}).setdefault(k, {}).update(v)
    summ["_note_hw"] = ("hw_flops_per_launch: ncu --metrics pass (smsp__sass_thread_inst_executed_op_{d,f}{fma,mul,add}"
                        "_pred_on.sum; 2 per FMA) of a short bench.py run on cfg4 in each precision (scripts/collect_profiles.sh)")
json.dump(summ, open(os.path.join(prof, f"ncu_summary_{tag}.json"), "w"), indent=1)
print(open(os.path.join(prof, f"launch_shares_{tag}.txt")).read())
print(json.dumps(summ, indent=1))
