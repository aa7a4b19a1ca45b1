"""Short NVE run of a BASELINE config for profiling (ncu launch lists / --set full captures)."""
import argparse
import sys

sys.path.insert(0, ".")
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--precision", default="fp64")
a = ap.parse_args()
cfg = int(a.config) if a.config.isdigit() else a.config
s = I.config(cfg)
e = E.make(s, a.precision)
e.run_nve(a.steps, s.dt)
print("ok", s.name, e.stats()["n_rebuilds"])
