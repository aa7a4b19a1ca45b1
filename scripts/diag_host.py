"""Diagnostic: host-side time per NVE step (AB_HOST_TIMING=1, printed at close) next to the
device time per step, for a plain (unprofiled) NVE run: shows whether the host enqueue keeps
ahead of the GPU."""
import os
import sys

os.environ["AB_HOST_TIMING"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
s = I.config(int(cfg) if cfg.isdigit() else cfg)
if len(sys.argv) > 3:  # time step override (e.g. 1e-9 fs: frozen atoms, for AB_SKIP ablations)
    s.dt = float(sys.argv[3])
eng = E.make(s, prec)
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
eng.run_nve(20, s.dt)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time  # noqa: E402
for n in (1, 10, 100):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record(st)
    eng.run_nve(n, s.dt)
    b.record(st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{s.name} {prec} n={n}: device {a.elapsed_time(b) / n * 1e3:.1f} us/step, host enqueue "
          f"{(t1 - t0) / n * 1e6:.1f} us/step, wall {(t2 - t0) / n * 1e6:.1f} us/step", flush=True)
eng.close()
