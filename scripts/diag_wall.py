"""Diagnostic: NVE throughput of cfg2 fp64 measured (1) as one long run_nve(K) call (device events
around it + host wall clock) and (2) per step with an L2 flush in between (bench.py's method),
for the concurrent and the serial (AB_SERIAL_KERNELS=1) kernel DAG."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

s = I.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for serial in ("0", "1", "0", "1"):
    os.environ["AB_SERIAL_KERNELS"] = serial
    eng = E.make(s, "fp64")
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)
    torch.cuda.set_stream(st)
    eng.run_nve(30, s.dt)
    torch.cuda.synchronize()
    K = 200
    nb = eng.stats()["n_rebuilds"]
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(st)
    eng.run_nve(K, s.dt)
    b.record(st)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / K * 1e3
    dev = a.elapsed_time(b) / K
    nb1 = eng.stats()["n_rebuilds"] - nb
    ts = []
    nb = eng.stats()["n_rebuilds"]
    for _ in range(100):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.run_nve(1, s.dt)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    nb2 = eng.stats()["n_rebuilds"] - nb
    ts.sort()
    import ctypes as C
    eng.L.ab_set_profiling(eng.h, 1)
    eng.run_nve(50, s.dt)
    ms = (C.c_double * 8)()
    cnt = (C.c_int64 * 8)()
    eng.L.ab_get_phase_ms(eng.h, ms, cnt)
    eng.L.ab_set_profiling(eng.h, 0)
    ph = {n: round(ms[q] / max(cnt[q], 1), 4) for q, n in enumerate(["short", "rebo", "near", "bstar", "integ", "rebuild", "far"])}
    print(ph)
    print(f"serial={serial}: long run {K} steps ({nb1} rebuilds): device {dev:.4f} ms/step, wall {wall:.4f} | "
          f"per-step flushed 100 steps ({nb2} rebuilds): mean {sum(ts) / len(ts):.4f} median {ts[50]:.4f} max {ts[-1]:.3f}")
    eng.close()
