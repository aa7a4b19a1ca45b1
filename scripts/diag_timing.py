"""Diagnostic: step time of the NVE loop measured several ways on cfg2, fp64 (device events per
step with / without an L2 flush before each step, with / without phase profiling; host time
inside the call; host wall clock over a long batch)."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

s = I.config(2)
eng = E.make(s, "fp64")
st = torch.cuda.current_stream()
eng.set_stream(st.cuda_stream)
eng.run_nve(5, s.dt)
torch.cuda.synchronize()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def loop(tag, do_flush, prof, n=40):
    eng.L.ab_set_profiling(eng.h, int(prof))
    dev, host = [], []
    for _ in range(n):
        if do_flush:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        t0 = time.perf_counter()
        eng.run_nve(1, s.dt)
        host.append((time.perf_counter() - t0) * 1e3)
        b.record(st)
        b.synchronize()
        dev.append(a.elapsed_time(b))
    ms = (C.c_double * 8)()
    cnt = (C.c_int64 * 8)()
    eng.L.ab_get_phase_ms(eng.h, ms, cnt)
    eng.L.ab_set_profiling(eng.h, 0)
    dev.sort()
    host.sort()
    print(f"{tag:28s} device median {dev[n // 2]:.4f} ms (min {dev[0]:.4f})  host-in-call median {host[n // 2]:.4f} ms"
          + (f"  phases {[round(ms[q] / n, 4) for q in range(8)]}" if prof else ""))


for rep in range(2):
    loop("flush, no prof", True, False)
    loop("flush, prof", True, True)
    loop("no flush, no prof", False, False)
    loop("no flush, prof", False, True)
for K in (200,):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.run_nve(K, s.dt)
    torch.cuda.synchronize()
    print(f"wall run_nve({K}): {(time.perf_counter() - t0) / K * 1e3:.4f} ms/step  stats {eng.stats()['n_rebuilds']}")
