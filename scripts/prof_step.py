"""Short NVE run of a BASELINE config for profiling (ncu launch lists / --set full captures);
prints the engine's counters (list sizes, pair counts) of the last evaluation."""
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
st = e.stats()
print("ok", s.name, {k: st[k] for k in ("n_rebuilds", "n_lj", "n_lj_entries", "n_lj_far", "n_lj_taper", "lj_capacity",
                                        "n_C0", "n_bstar", "max_reach", "n_overflow_retries", "n_ghosts")})
print("slots per atom (both directions)", st["n_lj_entries"] / s.n, "useful full pairs per atom", 2 * st["n_lj"] / s.n)
