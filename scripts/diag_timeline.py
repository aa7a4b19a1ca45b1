"""Diagnostic: the concurrent kernel DAG's timeline (AB_TIMELINE=1): mean start / end offset of
each force phase from the start of the evaluation, with the DAG concurrent, printed at close."""
import os
import sys

os.environ["AB_TIMELINE"] = "1"
os.environ.setdefault("AB_SERIAL_KERNELS", "0")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
s = I.config(int(cfg) if cfg.isdigit() else cfg)
eng = E.make(s, prec)
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
eng.run_nve(20, s.dt)
eng.L.ab_set_profiling(eng.h, 1)
eng.run_nve(50, s.dt)
torch.cuda.synchronize()
eng.L.ab_set_profiling(eng.h, 0)
print(s.name, prec, flush=True)
eng.close()
