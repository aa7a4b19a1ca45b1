"""Diagnostic: max_reach (distinct images within 3 bonds) and reach-table overflows per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3"]):
    s = I.config(int(cfg) if cfg.isdigit() else cfg)
    e = E.make(s, "fp64")
    e.compute()
    st = e.stats()
    print(cfg, s.n, "max_reach", st["max_reach"], "overflows", st["n_overflow_retries"], "n_lj", st["n_lj"], "n_C0", st["n_C0"])
