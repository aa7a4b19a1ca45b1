"""GPU parity of the potential variants (param key `potential`): REBO (bond
terms only: no LJ kernels, no LJ lists, no torsion) and AIREBO-M (Morse radial form in the near,
far and b* kernels, every gate kept) against the oracle, at the fp64 / mixed tolerances of
BASELINE.json north_star, with exact integer counters and bit-exact lists."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I

pytestmark = pytest.mark.gpu
COUNTERS = ["n_short", "n_bonds", "n_quads", "n_lj", "n_C0", "n_bstar", "n_sb_trans", "max_short", "max_reach",
            "n_badarg"]


@pytest.fixture(scope="module")
def eng_mod():
    from paper_1810_07026_b200 import build, engine
    build.build()
    return engine


def variant(text, name):
    return text.replace(b"potential airebo\n", b"potential " + name.encode() + b"\n")


def make(E, s, precision, params, ranks=None):
    e = E.Engine(precision, 0, params=params, ranks=ranks)
    e.set_box(s.box)
    e.set_atoms(s.types, s.x)
    if s.v is not None:
        e.set_velocities(s.v)
    return e


SYSTEMS = {"cfg1": lambda: I.config(1), "cluster": lambda: I.random_cluster(60, 11, spread=7.0, dmin=0.95, frac_c=0.4),
           "diamond": lambda: I.diamond((2, 2, 2), 0.04, 21), "cfg2": lambda: I.config(2)}


@pytest.mark.parametrize("name", ["rebo", "airebo-m"])
@pytest.mark.parametrize("sysname", list(SYSTEMS))
def test_variant_fp64_parity(eng_mod, params_text, name, sysname):
    p = variant(params_text, name)
    s = SYSTEMS[sysname]()
    o = O.compute(s.types, s.x, s.box, params=p)
    e = make(eng_mod, s, "fp64", p)
    g = e.compute()
    assert abs(g["E"] - o["E"]) <= 1e-11 * abs(o["E"]) + 1e-13, (g["E"], o["E"])
    for t in range(3):
        assert abs(g["terms"][t] - o["terms"][t]) <= 1e-11 * max(abs(o["E"]), 1.0), t
    assert np.abs(g["F"] - o["F"]).max() <= 1e-9
    assert np.abs(g["W"] - o["W"]).max() <= 1e-10 * max(np.abs(o["W"]).max(), 1.0)
    st = e.stats()
    for k in COUNTERS:
        assert st[k] == o["counters"][k], (k, st[k], o["counters"][k])
    for which in (0, 1, 2):
        assert np.array_equal(e.get_list(which), O.get_list(s.types, s.x, s.box, which, params=p)), which
    if name == "rebo":
        assert g["terms"][1] == 0.0 and g["terms"][2] == 0.0 and st["n_lj"] == 0


@pytest.mark.parametrize("name", ["rebo", "airebo-m"])
def test_variant_mixed_and_slabs(eng_mod, params_text, name):
    p = variant(params_text, name)
    s = I.config(2)
    o = O.compute(s.types, s.x, s.box, params=p)
    g = make(eng_mod, s, "mixed", p).compute()
    rel = np.sqrt(((g["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-4 and abs(g["E"] - o["E"]) <= 1e-6 * abs(o["E"])
    g3 = make(eng_mod, s, "fp64", p, ranks=("virtual", 3)).compute()
    assert np.abs(g3["F"] - o["F"]).max() <= 1e-9 and abs(g3["E"] - o["E"]) <= 1e-11 * abs(o["E"])


def test_airebo_m_nve_replay(eng_mod, params_text):
    p = variant(params_text, "airebo-m")
    s = I.config(1)
    e = make(eng_mod, s, "fp64", p)
    th = e.run_nve(40, 0.5, every=10)
    x = e.get_positions()
    F = e.compute()["F"]
    o = O.compute(s.types, x, s.box, params=p)
    assert np.abs(F - o["F"]).max() <= 1e-9
    assert np.abs(th[:, 3] - th[0, 3]).max() <= 1e-3 * abs(th[0, 1])
