"""Precision study (the paper's section 5.2 experiment): total-energy
drift of long NVE runs in fp64, mixed, single (AB_SINGLE: fp32 accumulation) and reduced precision
(AB_REDUCED: binary32 accumulation and binary32 positions / velocities, reading A35) on the
all-carbon nanotube (the paper's CNT workload) and on polyethylene.  argv: steps, dt_fs,
systems (all | cnt | pe | cfg2), precisions (comma list).  Prints one JSON line per (system, precision): the maximal
|E_tot(t) - E_tot(0)| per atom and the slope of a linear fit (eV/atom/ps)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
dt = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
every = max(1, steps // 200)
systems = [I.nanotube(10, 10, 12, jitter=0.01, seed_x=41, seed_v=42, T=300.0, name="cnt-10-10-x12"),
           I.polyethylene((2, 2, 6), 0.02, 43, 44, name="pe-2x2x6")]
which = sys.argv[3] if len(sys.argv) > 3 else "all"
precs = sys.argv[4].split(",") if len(sys.argv) > 4 else ["fp64", "mixed", "single"]
if which == "cfg2":  # the headline workload (BASELINE configs[1], 32,256 atoms)
    systems = [I.config(2)]
systems = [s for s in systems if which in ("all", "cfg2") or s.name.startswith(which)]
for s in systems:
    for prec in precs:
        e = E.make(s, prec)
        th = e.run_nve(steps, dt, every=every)
        t_ps = th[:, 0] * dt * 1e-3
        de = (th[:, 3] - th[0, 3]) / s.n
        slope = float(np.polyfit(t_ps, de, 1)[0])
        print(json.dumps({"system": s.name, "atoms": int(s.n), "precision": prec, "steps": steps, "dt_fs": dt,
                          "max_abs_dE_per_atom_eV": float(np.abs(de).max()), "drift_eV_per_atom_per_ps": slope,
                          "E0_per_atom": float(th[0, 3] / s.n)}), flush=True)
