"""Diagnostic: spread of the cfg4 step time between calls of one process and between processes
(repeated ab_run_nve(100) calls on one engine, CUDA events on the engine stream)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

s = I.config(4)
eng = E.make(s, "fp64")
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
eng.run_nve(5, s.dt)
torch.cuda.synchronize()
out = []
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    nb0 = eng.stats()["n_rebuilds"]
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        eng.run_nve(100, s.dt, every=10)
        b.record(st)
    st.synchronize()
    out.append((round(a.elapsed_time(b) / 100, 4), eng.stats()["n_rebuilds"] - nb0))
print(os.getpid(), out, flush=True)
eng.close()
