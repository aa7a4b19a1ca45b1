"""Two NCCL ranks as threads of one process on one GPU, with the test-only fake NCCL library
(tests/fake_nccl/fake_nccl.cpp, selected through AB_NCCL_LIB before the engine first touches
NCCL).  Exercises ab_create_dist and every NCCL branch of the engine (halo and force exchange,
flag / result / caller-order all-reduces, set_positions redistribution, thermo rows) against the
whole-box engine.  Prints one JSON line with the measured differences; the pytest wrapper
(tests/test_gpu_nccl_path.py) applies the tolerances."""
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
assert os.environ.get("AB_NCCL_LIB"), "set AB_NCCL_LIB to the fake library"
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "3"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s = I.config(int(name)) if name.isdigit() else I.random_cluster(160, 5, box_len=40.0, spread=14.0, dmin=0.95)
if s.v is None:
    s.v = np.zeros_like(s.x)
steps, dt = 12, s.dt

ref = E.make(s, "fp64")
g0 = ref.compute()
th_ref = ref.run_nve(steps, dt, every=4)
x_ref, v_ref = ref.get_positions(), ref.get_velocities()
g1 = ref.compute()

uid = E.nccl_unique_id()
out = [None] * nr
err = [None] * nr


def rank_main(r):
    try:
        e = E.Engine("fp64", 0, ranks=("nccl", r, nr, uid))
        e.set_box(s.box)
        e.set_atoms(s.types, s.x)
        e.set_velocities(s.v)
        a = e.compute()
        st = e.stats()
        th = e.run_nve(steps, dt, every=4)
        x, v = e.get_positions(), e.get_velocities()
        b = e.compute()
        # new positions that move every atom to another slab: ownership recomputed
        x2 = I.wrap(x_ref + np.array([0.37 * s.box[0], 0.0, 0.0]), s.box)  # same frame as the reference
        e.set_positions(x2)
        c = e.compute()
        out[r] = dict(a=a, b=b, c=c, th=th, x=x, v=v, st=st, lst=e.get_list(2))
        e.close()
    except Exception as ex:  # reported by the main thread
        err[r] = repr(ex)


ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(nr)]
for t in ts:
    t.start()
for t in ts:
    t.join()
if any(err):
    print(json.dumps({"error": err}))
    sys.exit(1)
ref.set_positions(I.wrap(x_ref + np.array([0.37 * s.box[0], 0.0, 0.0]), s.box))
g2 = ref.compute()
res = {"n": int(s.n)}
for r in range(nr):
    o = out[r]
    res[f"r{r}"] = {
        "dF0": float(np.abs(o["a"]["F"] - g0["F"]).max()), "dE0": abs(o["a"]["E"] - g0["E"]) / abs(g0["E"]),
        "dW0": float(np.abs(o["a"]["W"] - g0["W"]).max()),
        "dx": float(np.abs(o["x"] - x_ref).max()), "dv": float(np.abs(o["v"] - v_ref).max()),
        "dth": float(np.abs(o["th"] - th_ref).max()),
        "dF1": float(np.abs(o["b"]["F"] - g1["F"]).max()),
        "dF2": float(np.abs(o["c"]["F"] - g2["F"]).max()), "dE2": abs(o["c"]["E"] - g2["E"]) / abs(g2["E"]),
        "n_atoms": o["st"]["n_atoms"], "n_lj_equal": o["st"]["n_lj"] == ref.stats()["n_lj"] or None,
        "list_rows": int(len(o["lst"]))}
print(json.dumps(res))
