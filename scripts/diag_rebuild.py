"""Diagnostic: cost of a skin-triggered list rebuild inside the NVE loop (cfg2, fp64): host time
of the run_nve(1) calls that rebuilt vs those that did not, and the device time of the rebuild
phase (CUDA events)."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
s = I.config(int(cfg) if cfg.isdigit() else cfg)
eng = E.make(s, "fp64")
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
torch.cuda.set_stream(st)
eng.run_nve(5, s.dt)
torch.cuda.synchronize()
eng.L.ab_set_profiling(eng.h, 1)
ms = (C.c_double * 8)()
cnt = (C.c_int64 * 8)()
nb0 = eng.stats()["n_rebuilds"]
reb, norm = [], []
for k in range(120):
    t0 = time.perf_counter()
    eng.run_nve(1, s.dt)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) * 1e3
    nb = eng.stats()["n_rebuilds"]
    (reb if nb != nb0 else norm).append(t)
    nb0 = nb
eng.L.ab_get_phase_ms(eng.h, ms, cnt)
print(f"{s.name}: steps without rebuild: {len(norm)}, median host {sorted(norm)[len(norm) // 2]:.3f} ms")
print(f"steps with rebuild: {len(reb)}, host ms {[round(x, 2) for x in reb]}")
print(f"rebuild phase device ms total {ms[5]:.3f} over {cnt[5]} rebuilds; phases {[round(ms[q], 3) for q in range(8)]}")
