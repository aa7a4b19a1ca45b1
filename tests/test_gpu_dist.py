"""GPU parity of the slab decomposition through the C-ABI.

n slab domains on one GPU (ab_create_virtual: the decomposition code of the distributed engine,
halo exchanged by device copies instead of ncclSend/ncclRecv) must reproduce the oracle within
the fp64 / mixed tolerances of BASELINE.json north_star, give bit-exact lists and exact integer
counters (every term computed once globally), and follow the whole-box engine's trajectory
through rebuilds with atoms migrating between slabs.
"""
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


def system(name):
    if name == "pe-4x2x4":
        return I.polyethylene((4, 2, 4), 0.03, 7, 8, name=name)  # L_x = 29.7 A: 2 slabs of 14.8 A
    if name == "diamond-7x2x2":
        return I.diamond((7, 2, 2), 0.04, 21, 22, name=name)  # 24.97 A; y, z multi-image
    if name == "cluster-40":
        # reactive cluster centred on the x = 20 A slab face of 2 / 3 slabs: fractional w, C paths,
        # S_b transitions across the boundary
        return I.random_cluster(160, 5, box_len=40.0, spread=14.0, dmin=0.95, frac_c=0.5, name=name)
    return I.config(int(name))


def check_fp64(g, o, name):
    assert abs(g["E"] - o["E"]) <= 1e-11 * abs(o["E"]) + 1e-13, (name, g["E"], o["E"])
    for t in range(3):
        assert abs(g["terms"][t] - o["terms"][t]) <= 1e-11 * max(abs(o["E"]), 1.0), (name, t)
    dF = np.abs(g["F"] - o["F"]).max()
    assert dF <= 1e-9, (name, dF)
    dW = np.abs(g["W"] - o["W"]).max()
    assert dW <= 1e-10 * max(np.abs(o["W"]).max(), 1.0), (name, dW)


CASES = [("pe-4x2x4", 2), ("diamond-7x2x2", 2), ("cluster-40", 2), ("cluster-40", 3), ("2", 2), ("2", 3), ("2", 7),
         ("3", 2), ("3", 5)]


@pytest.mark.parametrize("name,n", CASES)
def test_virtual_slabs_fp64_vs_oracle(eng_mod, name, n):
    s = system(name)
    o = O.compute(s.types, s.x, s.box)
    e = eng_mod.make(s, "fp64", ranks=("virtual", n))
    g = e.compute()
    check_fp64(g, o, (name, n))
    st = e.stats()
    for k in COUNTERS:
        assert st[k] == o["counters"][k], (name, n, k, st[k], o["counters"][k])
    assert st["n_atoms"] == s.n
    for which in (0, 1, 2):
        a = e.get_list(which)
        b = O.get_list(s.types, s.x, s.box, which)
        assert a.shape == b.shape and np.array_equal(a, b), (name, n, which)


def test_virtual_slabs_mixed(eng_mod):
    s = I.config(2)
    o = O.compute(s.types, s.x, s.box)
    g = eng_mod.make(s, "mixed", ranks=("virtual", 4)).compute()
    rel = np.sqrt(((g["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-4, rel
    assert abs(g["E"] - o["E"]) <= 1e-6 * abs(o["E"])


def test_slab_narrower_than_halo_is_rejected(eng_mod):
    s = I.config(2)  # L_x = 89.04 A, halo 11.2 A: 8 slabs of 11.13 A are too narrow
    e = eng_mod.Engine("fp64", ranks=("virtual", 8))
    with pytest.raises(eng_mod.ABError) as ei:
        e.set_box(s.box)
    assert ei.value.status == -3 and "halo" in str(ei.value)


def test_virtual_nve_migration_matches_whole_box(eng_mod):
    """Reactive a-CH2 at 1500 K: skin-triggered rebuilds with atoms crossing slab faces.  Over a
    few steps the slab run follows the whole-box run to roundoff; over 40 steps (rebuilds,
    migrations) the chaotic 1500 K dynamics amplifies the summation-order roundoff, so the
    physics checks are the oracle's forces at the slab run's final frame and the conservation of
    the total energy."""
    s = I.config(3)
    dt = 0.25
    e1 = eng_mod.make(s, "fp64")
    e3 = eng_mod.make(s, "fp64", ranks=("virtual", 3))
    e1.run_nve(6, dt)
    e3.run_nve(6, dt)
    assert np.abs(e1.get_positions() - e3.get_positions()).max() <= 1e-10
    assert np.abs(e1.get_velocities() - e3.get_velocities()).max() <= 1e-10
    th1 = e1.run_nve(34, dt, every=10)
    th3 = e3.run_nve(34, dt, every=10)
    x3 = e3.get_positions()
    assert np.abs(e1.get_positions() - x3).max() <= 1e-3
    drift1 = np.abs(th1[:, 3] - th1[0, 3]).max()
    drift3 = np.abs(th3[:, 3] - th3[0, 3]).max()
    assert drift3 <= 2 * drift1 + 1e-6 * abs(th1[0, 3]), (drift1, drift3)
    st = e3.stats()
    assert st["n_rebuilds"] >= 2, st
    own0 = np.array([eng_mod.slab_of(x, s.box[0], 3) for x in s.x[:, 0]])
    own1 = np.array([eng_mod.slab_of(x, s.box[0], 3) for x in x3[:, 0]])
    assert (own0 != own1).sum() > 0  # atoms migrated between slabs
    F3 = e3.compute()["F"]
    smp = np.concatenate([np.nonzero(own0 != own1)[0][:12], np.arange(0, s.n, 4001)])
    Fs = O.forces_sampled(s.types, x3, s.box, smp)
    assert np.abs(F3[smp] - Fs).max() <= 1e-9


def test_virtual_set_positions_redistributes(eng_mod):
    """New positions may move every atom to another slab: ownership is recomputed."""
    s = system("pe-4x2x4")
    e = eng_mod.make(s, "fp64", ranks=("virtual", 2))
    e.compute()
    x2 = s.x.copy()
    x2[:, 0] += 0.37 * s.box[0]
    e.set_positions(x2)
    g = e.compute()
    o = O.compute(s.types, I.wrap(x2, s.box), s.box)  # the oracle takes wrapped positions
    check_fp64(g, o, "shifted")
    assert np.abs(e.get_velocities() - s.v).max() == 0.0


def test_virtual_stage_rows(eng_mod):
    s = system("cluster-40")
    e = eng_mod.make(s, "fp64", ranks=("virtual", 2))
    e.record_stages(True)
    e.compute()
    rb = O.get_list(s.types, s.x, s.box, 1)
    B_o, _ = O.stages(s.types, s.x, s.box)
    st0 = e.get_stage(0)
    key0 = {tuple(int(v) for v in r[:5]): r[5:] for r in st0}
    assert len(key0) == len(rb)
    for row, ref in zip(rb, B_o):
        assert np.allclose(key0[tuple(int(v) for v in row)], ref, rtol=1e-12, atol=1e-13)


def test_empty_slab_domain(eng_mod):
    """A small cluster in a 40 A box cut into 3 slabs leaves a slab without atoms (and a neighbour
    whose halo is empty): every kernel of the empty domain must launch cleanly and the result
    still equal the oracle's."""
    s = I.random_cluster(40, 8, box_len=40.0, spread=6.0, dmin=1.0, name="small-cluster")
    owners = {eng_mod.slab_of(x, s.box[0], 3) for x in s.x[:, 0]}
    assert len(owners) < 3
    o = O.compute(s.types, s.x, s.box)
    e = eng_mod.make(s, "fp64", ranks=("virtual", 3))
    g = e.compute()
    check_fp64(g, o, "empty-slab")
    e.set_velocities(np.zeros_like(s.x))
    e.run_nve(5, 0.25)
    x = e.get_positions()
    assert np.abs(e.compute()["F"] - O.compute(s.types, x, s.box)["F"]).max() <= 1e-9


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_virtual_nve_halo_overlap(eng_mod, monkeypatch, precision):
    """Slab NVE steps launch the far-LJ pairs of the interior atoms (LJ stencil inside the slab)
    beside the halo exchange; the boundary atoms follow the exchange.  The
    trajectory equals the non-overlapped one (AB_NO_OVERLAP=1) and the whole-box one to summation
    roundoff, and the overlapped schedule really ran (two more launches per step: the locals'
    image refresh and the interior far-LJ kernel)."""
    s = I.config(2)  # L_x = 89 A: 2 slabs of 44.5 A with an interior
    runs = {}
    for tag in ("overlap", "plain", "whole"):
        if tag == "plain":
            monkeypatch.setenv("AB_NO_OVERLAP", "1")
        else:
            monkeypatch.delenv("AB_NO_OVERLAP", raising=False)
        e = eng_mod.make(s, precision, ranks=None if tag == "whole" else ("virtual", 2))
        l0 = e.device_info()["kernel_launches"]
        th = e.run_nve(12, s.dt, every=6)
        runs[tag] = (e.get_positions(), e.get_velocities(), th, e.device_info()["kernel_launches"] - l0)
    xo, vo, tho, lo = runs["overlap"]
    xp, vp, thp, lp = runs["plain"]
    xw, vw, thw, lw = runs["whole"]
    assert lo >= lp + 2 * 12 - 4, (lo, lp)  # (a rebuild step takes the plain path)
    tol = 1e-10 if precision == "fp64" else 1e-8
    assert np.abs(xo - xp).max() <= tol and np.abs(vo - vp).max() <= tol
    # whole box vs slabs: fp32 terms in mixed mode make the evaluations differ beyond fp64 roundoff
    assert np.abs(xo - xw).max() <= (tol if precision == "fp64" else 1e-6)
    assert np.allclose(tho[:, 1:], thw[:, 1:], rtol=1e-10 if precision == "fp64" else 1e-6)
