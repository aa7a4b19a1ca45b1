"""Diagnostic: NVE step time of cfg2 against the neighbour-list skin (the param file's
neigh.skin replaced in memory; results are skin-independent, tests/test_oracle.py).  Prints
device us/step over 200 back-to-back steps (rebuilds included) and the rebuild count."""
import os
import re
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
s = I.config(int(cfg) if cfg.isdigit() else cfg)
base = open(E.PARAMS, "rb").read().decode()
for skin in [float(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1.0", "0.8", "0.6", "0.5", "0.4"])]:
    txt = re.sub(r"^neigh\.skin .*$", f"neigh.skin {skin}", base, flags=re.M).encode()
    eng = E.Engine(prec, 0, params=txt)
    eng.set_box(s.box)
    eng.set_atoms(s.types, s.x)
    eng.set_velocities(s.v)
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)
    eng.run_nve(20, s.dt)
    torch.cuda.synchronize()
    nb0 = eng.stats()["n_rebuilds"]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    eng.run_nve(200, s.dt)
    b.record(st)
    torch.cuda.synchronize()
    st2 = eng.stats()
    print(f"{s.name} {prec} skin {skin}: {a.elapsed_time(b) / 200 * 1e3:.1f} us/step, rebuilds {st2['n_rebuilds'] - nb0} "
          f"in 200 steps, E {eng.compute()['E']:.9f}", flush=True)
    eng.close()
