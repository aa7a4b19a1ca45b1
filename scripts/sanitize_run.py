"""Small whole-path workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
cfg1 (multi-image PE) and cfg2 (32 k PE) whole-box engines, fp64 and mixed, and the virtual
slab engine (3 slabs) on a reactive cluster and on cfg2: one force evaluation with stage
recording, list queries and a few NVE steps each (rebuilds included).  Exits 0 when every call
succeeded; the sanitizer's own summary decides about errors."""
import sys

sys.path.insert(0, ".")
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
jobs = [(I.config(1), "fp64", None), (I.config(1), "mixed", None), (I.config(2), "fp64", None),
        (I.random_cluster(60, 11, spread=7.0, dmin=0.95, frac_c=0.4), "fp64", ("virtual", 3)),
        (I.config(2), "mixed", ("virtual", 3))]
for s, prec, ranks in jobs:
    e = E.make(s, prec, ranks=ranks)
    e.record_stages(True)
    r = e.compute()
    e.record_stages(False)
    for w in (0, 1, 2):
        e.list_digest(w)
    if s.v is not None:
        e.run_nve(steps, s.dt, every=2)
    e.compute()
    print("ok", s.name, prec, ranks, round(r["E"], 6), e.stats()["n_rebuilds"], flush=True)
    e.close()
