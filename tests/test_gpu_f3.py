"""GPU parity of the SURVEY §8(f) F3 functional details (params/toy_ch_f3.param: distance-dependent
lambda_jik of H centres, reading A33 -- the fictitious distance rho of b* now matters, P:488-494;
coordination-dependent g_C, reading A34) against the oracle at BASELINE.json's fp64 / mixed
tolerances, with exact counters, bit-exact lists and stage-wise b_ij / b* parity."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COUNTERS = ["n_short", "n_bonds", "n_quads", "n_lj", "n_C0", "n_bstar", "n_sb_trans", "max_short", "max_reach",
            "n_badarg"]


@pytest.fixture(scope="module")
def eng_mod():
    from paper_1810_07026_b200 import build, engine
    build.build()
    return engine


@pytest.fixture(scope="module")
def f3():
    return open(os.path.join(ROOT, "params", "toy_ch_f3.param"), "rb").read()


def make(E, s, precision, params):
    e = E.Engine(precision, 0, params=params)
    e.set_box(s.box)
    e.set_atoms(s.types, s.x)
    if s.v is not None:
        e.set_velocities(s.v)
    return e


SYSTEMS = {"cfg1": lambda: I.config(1), "cluster0": lambda: I.random_cluster(30, 0, spread=4.6, dmin=1.0),
           "cluster3": lambda: I.random_cluster(30, 3, spread=4.6, dmin=1.0),
           "cluster-big": lambda: I.random_cluster(60, 11, spread=7.0, dmin=0.95, frac_c=0.4),
           "diamond": lambda: I.diamond((2, 2, 2), 0.04, 21), "cfg3": lambda: I.config(3)}


@pytest.mark.parametrize("sysname", list(SYSTEMS))
def test_f3_fp64_parity(eng_mod, f3, sysname):
    s = SYSTEMS[sysname]()
    o = O.compute(s.types, s.x, s.box, params=f3)
    e = make(eng_mod, s, "fp64", f3)
    g = e.compute()
    assert abs(g["E"] - o["E"]) <= 1e-11 * abs(o["E"]) + 1e-13, (g["E"], o["E"])
    for t in range(3):
        assert abs(g["terms"][t] - o["terms"][t]) <= 1e-11 * max(abs(o["E"]), 1.0), t
    dF = np.abs(g["F"] - o["F"]).max()
    assert dF <= 1e-9, dF
    assert np.abs(g["W"] - o["W"]).max() <= 1e-10 * max(np.abs(o["W"]).max(), 1.0)
    st = e.stats()
    for k in COUNTERS:
        assert st[k] == o["counters"][k], (k, st[k], o["counters"][k])
    if s.n < 5000:
        for which in (0, 1, 2):
            assert np.array_equal(e.get_list(which), O.get_list(s.types, s.x, s.box, which, params=f3))


@pytest.mark.parametrize("sysname", ["cluster-big", "cfg3"])
def test_f3_mixed_parity(eng_mod, f3, sysname):
    s = SYSTEMS[sysname]()
    o = O.compute(s.types, s.x, s.box, params=f3)
    g = make(eng_mod, s, "mixed", f3).compute()
    rel = np.sqrt(((g["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-4, rel
    assert abs(g["E"] - o["E"]) <= 1e-6 * abs(o["E"])


def test_f3_stage_parity_bond_order_and_bstar(eng_mod, f3):
    """b_ij (with its p, pi^rc, pi^dh parts, N_ij, N_ji, N^conj) per bond and b* per LJ pair: the
    b* of H-centred pairs uses rho for r_ij inside lambda."""
    for s in (I.random_cluster(40, 3, spread=6.0, dmin=1.0), I.random_cluster(30, 0, spread=4.6, dmin=1.0)):
        e = make(eng_mod, s, "fp64", f3)
        e.record_stages(True)
        e.compute()
        B_o, L_o = O.stages(s.types, s.x, s.box, params=f3)
        rb = O.get_list(s.types, s.x, s.box, 1, params=f3)
        rl = O.get_list(s.types, s.x, s.box, 2, params=f3)
        key0 = {tuple(int(v) for v in r[:5]): r[5:] for r in e.get_stage(0)}
        for row, ref in zip(rb, B_o):
            assert np.allclose(key0[tuple(int(v) for v in row)], ref, rtol=1e-12, atol=1e-13), row
        key1 = {tuple(int(v) for v in r[:5]): r[5:] for r in e.get_stage(1)}
        nb = 0
        for row, ref in zip(rl, L_o):
            got = key1[tuple(int(v) for v in row)]
            assert abs(got[0] - ref[0]) <= 1e-13 and abs(got[1] - ref[1]) <= 1e-12, (row, got, ref)
            nb += ref[1] != 0.0
        assert nb > 0


def test_f3_changes_results_and_nve_replay(eng_mod, f3, params_text):
    """The F3 file changes energies and forces of a reactive cluster (the terms are live), and an
    NVE run with it stays on the oracle's forces at the GPU's frames (dump / rerun)."""
    s = I.random_cluster(60, 11, spread=7.0, dmin=0.95, frac_c=0.4)
    a = make(eng_mod, s, "fp64", params_text).compute()
    b = make(eng_mod, s, "fp64", f3).compute()
    assert abs(a["E"] - b["E"]) > 1e-4 and np.abs(a["F"] - b["F"]).max() > 1e-3
    c = I.config(1)
    e = make(eng_mod, c, "fp64", f3)
    for _ in range(3):
        e.run_nve(10, 0.5)
        x = e.get_positions()
        F = e.compute()["F"]
        assert np.abs(F - O.compute(c.types, x, c.box, params=f3)["F"]).max() <= 1e-9
