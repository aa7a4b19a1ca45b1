"""GPU: the all-carbon nanotube workload (the paper's CNT) -- parity
with the oracle in fp64 and mixed precision, bit-exact lists, and the precision study of the
paper's section 5.2 in short form: the total-energy drift of an NVE run in mixed precision stays
within a small factor of fp64's (scripts/energy_drift.py runs the 20 000-step version:
profiles/energy_drift_r01.jsonl)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng_mod():
    from paper_1810_07026_b200 import build, engine
    build.build()
    return engine


@pytest.mark.parametrize("nm", [(10, 10, 4), (12, 0, 3), (8, 4, 1)])
def test_cnt_parity(eng_mod, nm):
    n, m, r = nm
    s = I.nanotube(n, m, r, jitter=0.03, seed_x=n + m)
    o = O.compute(s.types, s.x, s.box)
    e = eng_mod.make(s, "fp64")
    g = e.compute()
    assert abs(g["E"] - o["E"]) <= 1e-11 * abs(o["E"])
    assert np.abs(g["F"] - o["F"]).max() <= 1e-9
    for which in (0, 1, 2):
        assert np.array_equal(e.get_list(which), O.get_list(s.types, s.x, s.box, which))
    st = e.stats()
    for k in ("n_bonds", "n_quads", "n_lj", "n_C0", "n_bstar", "max_reach"):
        assert st[k] == o["counters"][k], k
    gm = eng_mod.make(s, "mixed").compute()
    rel = np.sqrt(((gm["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-4 and abs(gm["E"] - o["E"]) <= 1e-6 * abs(o["E"])


def test_cnt_energy_drift_mixed_vs_fp64(eng_mod):
    s = I.nanotube(10, 10, 12, jitter=0.01, seed_x=41, seed_v=42, T=300.0)
    drift = {}
    for prec in ("fp64", "mixed"):
        th = eng_mod.make(s, prec).run_nve(2000, 0.5, every=20)
        drift[prec] = np.abs(th[:, 3] - th[0, 3]).max() / s.n
    assert drift["fp64"] <= 1e-4, drift
    assert drift["mixed"] <= 3 * drift["fp64"] + 1e-6, drift
