"""Diagnostic: one long NVE run of a config with host-side timing breakdown (AB_HOST_TIMING)
and the rebuild count."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
s = I.config(int(cfg) if cfg.isdigit() else cfg)
eng = E.make(s, "fp64")
eng.run_nve(10, s.dt)
torch.cuda.synchronize()
nb = eng.stats()["n_rebuilds"]
t0 = time.perf_counter()
th = eng.run_nve(K, s.dt, every=K)
torch.cuda.synchronize()
t = (time.perf_counter() - t0) / K * 1e3
st = eng.stats()
print(f"{s.name}: {t:.3f} ms/step, {st['n_rebuilds'] - nb} rebuilds in {K} steps, stats {st}")
eng.close()
