"""Per-kernel device times (serial DAG, CUDA events) and the concurrent long-run step time of the
library given by AIREBO_B200_LIB (cfg2 fp64 unless argv[1] gives a config)."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
s = I.config(int(cfg) if cfg.isdigit() else cfg)
res = {}
for serial in ("1", "0"):
    os.environ["AB_SERIAL_KERNELS"] = serial
    eng = E.make(s, prec)
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)
    eng.run_nve(30, s.dt)
    torch.cuda.synchronize()
    if serial == "1":
        eng.L.ab_set_profiling(eng.h, 1)
        eng.run_nve(50, s.dt)
        ms = (C.c_double * 8)()
        cnt = (C.c_int64 * 8)()
        eng.L.ab_get_phase_ms(eng.h, ms, cnt)
        eng.L.ab_set_profiling(eng.h, 0)
        res["kernels_us"] = {n: round(1e3 * ms[q] / max(cnt[q], 1), 1)
                             for q, n in enumerate(["short", "rebo", "near", "bstar", "integ", "rebuild", "far"])}
    K = 200
    t0 = time.perf_counter()
    eng.run_nve(K, s.dt)
    torch.cuda.synchronize()
    res["step_ms_" + ("serial" if serial == "1" else "conc")] = round((time.perf_counter() - t0) / K * 1e3, 4)
    eng.close()
print(os.environ.get("AIREBO_B200_LIB", "default"), res)
