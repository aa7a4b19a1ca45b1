"""Diagnostic: host time of each C-ABI call of bench.py's end-to-end step (cfg2, fp64)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

s = I.config(2)
eng = E.make(s, "fp64")
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
eng.run_nve(10, s.dt)
vh = torch.from_numpy(eng.get_velocities()).pin_memory()
xh = torch.empty((s.n, 3), dtype=torch.float64).pin_memory()
th = np.zeros((2, 4))
dp = C.POINTER(C.c_double)
vptr, xptr, thp = C.cast(vh.data_ptr(), dp), C.cast(xh.data_ptr(), dp), th.ctypes.data_as(dp)
torch.cuda.synchronize()
T = np.zeros(4)
K = 50
for k in range(K):
    t0 = time.perf_counter()
    eng._ck(eng.L.ab_set_velocities(eng.h, vptr))
    t1 = time.perf_counter()
    eng._ck(eng.L.ab_run_nve(eng.h, 1, s.dt, 1, thp))
    t2 = time.perf_counter()
    eng._ck(eng.L.ab_get_positions(eng.h, xptr))
    t3 = time.perf_counter()
    T += [t1 - t0, t2 - t1, t3 - t2, t3 - t0]
print("ms per call: set_velocities %.4f run_nve(1, thermo) %.4f get_positions %.4f total %.4f" % tuple(T / K * 1e3))
T[:] = 0
for k in range(K):
    t0 = time.perf_counter()
    eng._ck(eng.L.ab_run_nve(eng.h, 1, s.dt, 0, None))
    t1 = time.perf_counter()
    eng._ck(eng.L.ab_get_positions(eng.h, xptr))
    t2 = time.perf_counter()
    T[:2] += [t1 - t0, t2 - t1]
print("no thermo: run_nve(1) %.4f get_positions %.4f" % tuple(T[:2] / K * 1e3))
