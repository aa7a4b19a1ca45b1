"""GPU parity: the CUDA path (through the C-ABI) against the fp64 CPU oracle on the same seeded
inputs.  Tolerances (BASELINE.json north_star, SURVEY reading A25):
  fp64 : max |F_gpu - F_orc| <= 1e-9 eV/A per component;  |E_gpu - E_orc| <= 1e-11 |E_orc|
  mixed: ||F_gpu - F_orc||_2 / ||F_orc||_2 <= 1e-4 (RMS over atoms);  |dE| <= 1e-6 |E|
  lists: bit-exact as sorted (i, j, sx, sy, sz) sets; integer counters equal (fp64).
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


def run_gpu(engine, s, precision="fp64"):
    e = engine.make(s, precision)
    res = e.compute()
    res["stats"] = e.stats()
    res["eng"] = e
    return res


def systems_small():
    out = [I.config(1), I.diamond((2, 2, 2), 0.04, 21, name="diamond-2x2x2"),
           I.diamond((1, 1, 1), 0.05, 9, name="diamond-1x1x1-multi-image"),
           I.polyethylene((1, 1, 1), 0.03, 5, None, name="pe-cell-multi-image")]
    for seed in range(4):
        out.append(I.random_cluster(30, seed, spread=5.0, dmin=1.0, name=f"cluster{seed}"))
    out.append(I.random_cluster(60, 11, spread=7.0, dmin=0.95, frac_c=0.4, name="cluster-big"))
    return out


def check_fp64(s, g, o):
    E_o = o["E"]
    assert abs(g["E"] - E_o) <= 1e-11 * abs(E_o) + 1e-13, (s.name, g["E"], E_o)
    for t in range(3):
        assert abs(g["terms"][t] - o["terms"][t]) <= 1e-11 * max(abs(E_o), 1.0), (s.name, t)
    dF = np.abs(g["F"] - o["F"]).max()
    assert dF <= 1e-9, (s.name, dF)
    dW = np.abs(g["W"] - o["W"]).max()
    assert dW <= 1e-10 * max(np.abs(o["W"]).max(), 1.0), (s.name, dW)


@pytest.mark.parametrize("idx", range(9))
def test_fp64_parity_small(eng_mod, idx):
    s = systems_small()[idx]
    o = O.compute(s.types, s.x, s.box)
    g = run_gpu(eng_mod, s)
    check_fp64(s, g, o)
    for k in COUNTERS:
        assert g["stats"][k] == o["counters"][k], (s.name, k, g["stats"][k], o["counters"][k])


@pytest.mark.parametrize("idx", range(9))
def test_lists_bit_exact(eng_mod, idx):
    s = systems_small()[idx]
    e = eng_mod.make(s)
    for which in (0, 1, 2):
        a = e.get_list(which)
        b = O.get_list(s.types, s.x, s.box, which)
        assert a.shape == b.shape and np.array_equal(a, b), (s.name, which)


@pytest.mark.parametrize("cfg", [2, 3])
def test_fp64_parity_configs(eng_mod, cfg):
    s = I.config(cfg)
    o = O.compute(s.types, s.x, s.box)
    g = run_gpu(eng_mod, s)
    check_fp64(s, g, o)
    for k in COUNTERS:
        assert g["stats"][k] == o["counters"][k], (s.name, k)
    for which in (0, 1, 2):
        a = g["eng"].get_list(which)
        b = O.get_list(s.types, s.x, s.box, which)
        assert np.array_equal(a, b), (s.name, which)


@pytest.mark.parametrize("cfg", [1, 2, 3, "diamond"])
def test_mixed_parity(eng_mod, cfg):
    s = I.diamond((4, 4, 4), 0.03, 105) if cfg == "diamond" else I.config(cfg)
    o = O.compute(s.types, s.x, s.box)
    g = run_gpu(eng_mod, s, "mixed")
    rel = np.sqrt(((g["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-4, rel
    assert abs(g["E"] - o["E"]) <= 1e-6 * abs(o["E"])
    assert np.array_equal(g["eng"].get_list(2), O.get_list(s.types, s.x, s.box, 2))


def test_stage_parity_bond_orders_and_cij(eng_mod):
    """Stage-wise parity: b_ij and its parts per bond, C_ij and b* per LJ pair."""
    for s in (I.config(1), I.random_cluster(40, 3, spread=6.0, dmin=1.0)):
        e = eng_mod.make(s)
        e.record_stages(True)
        e.compute()
        B_o, L_o = O.stages(s.types, s.x, s.box)
        rb = O.get_list(s.types, s.x, s.box, 1)
        rl = O.get_list(s.types, s.x, s.box, 2)
        st0 = e.get_stage(0)
        st1 = e.get_stage(1)
        key0 = {tuple(int(v) for v in r[:5]): r[5:] for r in st0}
        assert len(key0) == len(rb)
        for row, ref in zip(rb, B_o):
            got = key0[tuple(int(v) for v in row)]
            assert np.allclose(got, ref, rtol=1e-12, atol=1e-13), (row, got, ref)
        key1 = {tuple(int(v) for v in r[:5]): r[5:] for r in st1}
        assert len(key1) == len(rl)
        for row, ref in zip(rl, L_o):
            got = key1[tuple(int(v) for v in row)]
            assert abs(got[0] - ref[0]) <= 1e-13
            assert abs(got[1] - ref[1]) <= 1e-12


def test_edge_cases(eng_mod):
    box = np.array([30.0, 30.0, 30.0])
    # single atom: no terms
    e = eng_mod.Engine("fp64")
    e.set_box(box)
    e.set_atoms([0], [[1.0, 2.0, 3.0]])
    r = e.compute()
    assert r["E"] == 0.0 and np.all(r["F"] == 0.0)
    # pair exactly at r_max (closed boundary, w = 0) and exactly at r_c
    for x in ([[10.0, 10, 10], [12.0, 10, 10]], [[5.0, 5, 5], [15.2, 5, 5]]):
        x = np.array(x)
        o = O.compute([0, 0], x, box)
        e.set_atoms([0, 0], x)
        g = e.compute()
        assert abs(g["E"] - o["E"]) <= 1e-15 and np.abs(g["F"] - o["F"]).max() <= 1e-12
        assert np.array_equal(e.get_list(0), O.get_list([0, 0], x, box, 0))
        assert np.array_equal(e.get_list(2), O.get_list([0, 0], x, box, 2))
    # tiny box: an atom interacting with its own images (box < r_c)
    s = I.diamond((1, 1, 1), 0.0)
    o = O.compute(s.types, s.x, s.box)
    g = run_gpu(eng_mod, s)
    check_fp64(s, g, o)
    # bad arguments fail loudly
    with pytest.raises(eng_mod.ABError):
        e.set_box([0.0, 1.0, 1.0])
    with pytest.raises(eng_mod.ABError):
        e.set_atoms([2], [[0.0, 0, 0]])


def test_caller_order_and_permutation(eng_mod):
    s = I.config(1)
    rng = np.random.default_rng(4)
    p = rng.permutation(s.n)
    g1 = run_gpu(eng_mod, s)
    s2 = I.System("perm", s.types[p], s.x[p], s.box)
    g2 = run_gpu(eng_mod, s2)
    assert np.abs(g2["F"] - g1["F"][p]).max() <= 1e-12
    assert abs(g2["E"] - g1["E"]) <= 1e-12 * abs(g1["E"])


def test_nve_replay_parity_and_conservation(eng_mod):
    """NVE on the GPU; the oracle re-evaluates forces at the GPU's own frames (dump/rerun)."""
    s = I.config(1)
    e = eng_mod.make(s)
    frames = []
    th_all = []
    for k in range(10):
        th = e.run_nve(10, 0.5, every=10)
        th_all.append(th)
        x = e.get_positions()
        F = e.compute()["F"]
        frames.append((x, F))
    for x, F in frames[::3]:
        o = O.compute(s.types, x, s.box)
        assert np.abs(F - o["F"]).max() <= 1e-9
    # compare the free-running oracle trajectory (report-only quantity: must stay tiny for 100 steps)
    xo, vo, tho = O.nve(s.types, s.x, s.v, s.box, 100, 0.5, every=10)
    dx = frames[-1][0] - xo
    dx -= s.box * np.round(dx / s.box)
    assert np.abs(dx).max() < 1e-6
    # energy conservation: dt^2 scaling of the max drift
    d = []
    for dt, n in ((0.5, 100), (0.25, 200)):
        e2 = eng_mod.make(s)
        th = e2.run_nve(n, dt, every=1)
        d.append(np.abs(th[:, 3] - th[0, 3]).max())
    assert 3.0 <= d[0] / d[1] <= 5.0, d


def test_nve_rebuild_path_matches_fresh_lists(eng_mod):
    """After many steps with skin-triggered rebuilds, the lists equal a from-scratch build."""
    s = I.config(3)
    e = eng_mod.make(s)
    e.run_nve(30, 0.25)
    x = e.get_positions()
    F = e.compute()["F"]
    smp = np.arange(0, s.n, 997)
    Fs = O.forces_sampled(s.types, x, s.box, smp)
    assert np.abs(F[smp] - Fs).max() <= 1e-9


@pytest.mark.parametrize("cfg", [4, "5a", "5b"])
def test_full_size_parity(eng_mod, cfg):
    """BASELINE full sizes (cfg4 1,008,000-atom PE, cfg5a 2,000,376-atom diamond, cfg5b
    2,016,000-atom PE), whole-system parity against ONE full oracle evaluation (P:557-576 compares
    whole stages): fp64 E (1e-11 rel), every force component (1e-9 eV/A), W, all ten counters
    exact, the short list, the REBO half bonds and the LJ half pairs bit-exact (row digests of
    ab_get_list_digest, up to ~7e8 rows); mixed: RMS force error over ALL atoms <= 1e-4, E <= 1e-6."""
    s = I.config(cfg)
    o = O.compute_digest(s.types, s.x, s.box)
    g = run_gpu(eng_mod, s)
    check_fp64(s, g, o)
    for k in COUNTERS:
        assert g["stats"][k] == o["counters"][k], (s.name, k, g["stats"][k], o["counters"][k])
    for which in (0, 1, 2):
        assert g["eng"].list_digest(which) == o["digest"][which], (s.name, which)
    g["eng"].close()
    gm = run_gpu(eng_mod, s, "mixed")
    rel = np.sqrt(((gm["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-4, rel
    assert abs(gm["E"] - o["E"]) <= 1e-6 * abs(o["E"])
    assert gm["stats"]["n_lj"] == o["counters"]["n_lj"]


def test_list_digest_matches_rows(eng_mod):
    """ab_get_list_digest equals the numpy digest of ab_get_list's rows (pins the device-side
    digest used by the full-size list parity above)."""
    from tests.digest import digest
    for s in (I.config(1), I.random_cluster(30, 2, spread=5.0, dmin=1.0)):
        e = eng_mod.make(s)
        for which in (0, 1, 2):
            assert e.list_digest(which) == digest(e.get_list(which)), (s.name, which)


def test_two_engines_interleaved_different_boxes(eng_mod):
    """Several engines in one process share the __constant__ banks (box, cutoffs, table
    pointers); interleaved NVE calls without host synchronisation must each see their own."""
    a = I.config(1)
    b = I.diamond((2, 2, 2), 0.04, 21, seed_v=5)
    ea, eb = eng_mod.make(a), eng_mod.make(b)
    ra, rb = eng_mod.make(a), eng_mod.make(b)
    for _ in range(4):
        ea.run_nve(3, 0.5)
        eb.run_nve(3, 0.5)
    ra.run_nve(12, 0.5)
    rb.run_nve(12, 0.5)
    assert np.abs(ea.get_positions() - ra.get_positions()).max() <= 1e-10
    assert np.abs(eb.get_positions() - rb.get_positions()).max() <= 1e-10


def test_set_positions_rejects_nonfinite(eng_mod):
    s = I.config(1)
    e = eng_mod.make(s)
    x = s.x.copy()
    x[17, 1] = np.nan
    with pytest.raises(eng_mod.ABError) as ei:
        e.set_positions(x)
    assert ei.value.status == -8
    g = e.compute()  # state unchanged
    o = O.compute(s.types, s.x, s.box)
    assert np.abs(g["F"] - o["F"]).max() <= 1e-9


def test_nve_last_step_energies_and_counters(eng_mod):
    """Inside the NVE loop the partial-row reduction runs only on thermo steps; the call's last
    step is reduced when energies / counters are read.  Both must equal the oracle at the
    frames the GPU produced (thermo PE at the thermo step, counters of the last evaluation)."""
    s = I.config(1)
    e = eng_mod.make(s)
    th = e.run_nve(7, 0.5, every=7)  # thermo row at step 7 (reduced with the second half-kick)
    x7 = e.get_positions()
    o7 = O.compute(s.types, x7, s.box)
    assert abs(th[-1, 1] - o7["E"]) <= 1e-11 * abs(o7["E"])
    e.run_nve(5, 0.5)  # no thermo row: the last step's rows stay unreduced until read
    st = e.stats()
    x12 = e.get_positions()
    o12 = O.compute(s.types, x12, s.box)
    for k in COUNTERS:
        assert st[k] == o12["counters"][k], (k, st[k], o12["counters"][k])
    g = e.compute()  # a fresh evaluation at the same frame: same energy as the oracle's
    assert abs(g["E"] - o12["E"]) <= 1e-11 * abs(o12["E"])
    # several calls of one step, each read back: every one is the oracle's at its frame
    for _ in range(3):
        th = e.run_nve(1, 0.5, every=1)
        o = O.compute(s.types, e.get_positions(), s.box)
        assert abs(th[-1, 1] - o["E"]) <= 1e-11 * abs(o["E"])
        assert e.stats()["n_lj"] == o["counters"]["n_lj"]


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_nve_deferred_half_kick_paths_agree(eng_mod, precision):
    """The second half-kick of a step without a thermo row is deferred into the next drift kernel
    (or applied when v / F are read or replaced).  Every call pattern integrates the same
    trajectory: thermo every step (no deferral), one call, one-step calls, and calls split by a
    velocity read; up to fp64 atomic-order noise in F."""
    s = I.config(1)

    def run(pattern):
        e = eng_mod.make(s, precision)
        for n, every, read_v in pattern:
            e.run_nve(n, 0.5, every=every)
            if read_v:
                e.get_velocities()
        return e.get_positions(), e.get_velocities(), e

    ref_x, ref_v, _ = run([(10, 1, False)])
    for pattern in ([(10, 0, False)], [(1, 0, False)] * 10, [(3, 0, True), (4, 0, False), (3, 0, True)],
                    [(5, 0, False), (5, 5, False)]):
        x, v, e = run(pattern)
        assert np.abs(x - ref_x).max() <= 1e-10, pattern
        assert np.abs(v - ref_v).max() <= 1e-12, pattern
    # compute() after a deferred step: forces / energy at the current frame equal the oracle's,
    # and the pending kick used the forces of that frame (velocities unchanged by compute)
    x, v, e = run([(4, 0, False)])
    g = e.compute()
    o = O.compute(s.types, x, s.box)
    if precision == "fp64":
        assert np.abs(g["F"] - o["F"]).max() <= 1e-9
    else:
        assert np.linalg.norm(g["F"] - o["F"]) <= 1e-4 * np.linalg.norm(o["F"])
    assert np.array_equal(e.get_velocities(), v)


def test_inputs_copied_from_pinned_caller_buffers(eng_mod):
    """The library copies every input array (header): a page-locked caller buffer may be reused as
    soon as ab_set_velocities / ab_set_positions return."""
    import ctypes as C
    import torch
    s = I.config(2)
    e = eng_mod.make(s)
    e.run_nve(2, s.dt)  # work queued on the stream ahead of the copies
    v0 = np.ascontiguousarray(s.v * 0.5)
    vh = torch.from_numpy(v0.copy()).pin_memory()
    dp = C.POINTER(C.c_double)
    e.run_nve(3, s.dt)
    e._ck(e.L.ab_set_velocities(e.h, C.cast(vh.data_ptr(), dp)))
    vh.fill_(123.0)  # the caller reuses its buffer at once
    assert np.array_equal(e.get_velocities(), v0)
    x0 = e.get_positions()
    xh = torch.from_numpy(np.ascontiguousarray(x0)).pin_memory()
    e.run_nve(3, s.dt)
    e._ck(e.L.ab_set_positions(e.h, C.cast(xh.data_ptr(), dp)))
    xh.fill_(-7.0)
    assert np.array_equal(e.get_positions(), x0)


@pytest.mark.parametrize("which", ["small", 2, 3])
def test_cluster_lj_path_parity(eng_mod, which, monkeypatch):
    """The opt-in j-cluster LJ kernel (AB_LJ_CLUSTER=1, k_ljc.cuh): same fp64 tolerances, counters
    and LJ half list as the default near / far kernels and the oracle."""
    monkeypatch.setenv("AB_LJ_CLUSTER", "1")
    systems = systems_small()[:6] if which == "small" else [I.config(which)]
    for s in systems:
        o = O.compute(s.types, s.x, s.box)
        g = run_gpu(eng_mod, s)
        check_fp64(s, g, o)
        for k in COUNTERS:
            assert g["stats"][k] == o["counters"][k], (s.name, k, g["stats"][k], o["counters"][k])
        assert np.array_equal(g["eng"].get_list(2), O.get_list(s.types, s.x, s.box, 2)), s.name
        gm = run_gpu(eng_mod, s, "mixed")
        rel = np.sqrt(((gm["F"] - o["F"]) ** 2).sum()) / max(np.sqrt((o["F"] ** 2).sum()), 1e-300)
        assert rel <= 1e-4, (s.name, rel)


def fcc_carbon(rep=3, nn=1.6, jitter=0.04, seed=3):
    """Over-coordinated test solid: fcc carbon with a 1.6 A nearest-neighbour distance (12 short
    neighbours, second shell beyond r_max), jittered: 146 atom images within 3 bonds of an atom,
    more than the 64-slot reach table of the near-LJ kernel holds."""
    a = nn * np.sqrt(2)
    fcc = np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0]])
    g = np.stack(np.meshgrid(*[np.arange(rep)] * 3, indexing="ij"), -1).reshape(-1, 3)
    x = ((g[:, None, :] + fcc[None]) * a).reshape(-1, 3)
    x = x + np.random.default_rng(seed).uniform(-jitter, jitter, x.shape)
    box = np.full(3, rep * a)
    return I.System("fcc-carbon-overcoordinated", np.zeros(len(x), dtype=np.int32), I.wrap(x, box), box)


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_reach_table_overflow_fallback(eng_mod, precision):
    """Reach sets larger than the shared-memory table ("sequential fallback"): the near-LJ
    kernel falls back to the nested path search for those atoms; results stay at the
    parity tolerances and the overflow is counted (n_overflow_retries > 0)."""
    s = fcc_carbon()
    o = O.compute(s.types, s.x, s.box)
    assert o["counters"]["max_reach"] > 64
    g = run_gpu(eng_mod, s, precision)
    assert g["stats"]["n_overflow_retries"] > 0
    if precision == "fp64":
        check_fp64(s, g, o)
        for k in COUNTERS:
            if k != "max_reach":  # the GPU reports the table fill, capped by its size
                assert g["stats"][k] == o["counters"][k], (k, g["stats"][k], o["counters"][k])
    else:
        rel = np.sqrt(((g["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
        assert rel <= 1e-4 and abs(g["E"] - o["E"]) <= 1e-6 * abs(o["E"])


def test_skinned_lj_list_at_build_positions(eng_mod, params_text):
    """AB_LIST_LJ_SKIN: right after the build, the skinned LJ half list is the set of
    half pairs with r <= r_c + skin -- the oracle's LJ list for a parameter text whose r_c are
    r_c + skin (the same doubles), bit-exact; it contains AB_LIST_LJ."""
    import re
    skin = float(re.search(rb"neigh.skin ([0-9.eE+-]+)", params_text).group(1))
    txt = params_text
    for pair in (b"CC", b"CH", b"HH"):
        m = re.search(rb"lj\." + pair + rb"\.rc ([0-9.eE+-]+)", txt)
        txt = txt.replace(m.group(0), b"lj." + pair + b".rc " + repr(float(m.group(1)) + skin).encode())
    for s in (I.config(1), I.random_cluster(40, 3, spread=6.0, dmin=1.0), I.diamond((2, 2, 2), 0.04, 21)):
        e = eng_mod.make(s)
        sk = e.get_list(3)
        ref = O.get_list(s.types, s.x, s.box, 2, params=txt)
        assert sk.shape == ref.shape and np.array_equal(sk, ref), s.name
        lj = {tuple(r) for r in e.get_list(2)}
        assert lj <= {tuple(r) for r in sk}


def test_adaptive_reach_table_after_rebuild(eng_mod, monkeypatch):
    """After a list build that saw only small reach sets (PE: <= 16 images) the NVE near-pair kernel
    switches to the 32-slot reach table; its trajectory equals the 64-slot one and the forces at
    the end frame equal the oracle's."""
    s = I.config(1)
    out = []
    for fixed in (False, True):
        if fixed:
            monkeypatch.setenv("AB_NEAR_SLOTS_FIXED", "64")
        e = eng_mod.make(s)
        e.run_nve(2, 0.5)
        e.set_box(s.box)  # forces a list build, which reads the max reach of the steps before
        e.run_nve(40, 0.5, every=10)
        out.append(e.get_positions())
        if fixed:
            monkeypatch.delenv("AB_NEAR_SLOTS_FIXED")
        else:
            x = out[0]
            F = e.compute()["F"]
            o = O.compute(s.types, x, s.box)
            assert np.abs(F - o["F"]).max() <= 1e-9
    d = out[0] - out[1]
    d -= s.box * np.round(d / s.box)
    assert np.abs(d).max() <= 1e-9


def _engine_with_skin(eng_mod, s, skin):
    import re
    txt = open(eng_mod.PARAMS, "rb").read().decode()
    txt = re.sub(r"^neigh\.skin .*$", f"neigh.skin {skin}", txt, flags=re.M).encode()
    e = eng_mod.Engine("fp64", 0, params=txt)
    e.set_box(s.box)
    e.set_atoms(s.types, s.x)
    return e


@pytest.mark.parametrize("skin", [1.0, 2.5])
def test_far_bins_under_displacement(eng_mod, skin):
    """Far-row bins settled by the displacement bound (k_lists.cuh FB_*): after the list
    build every atom is moved by up to 0.49 skin (no rebuild), so pairs cross the window radius,
    r_lo and r_c relative to their build distances; forces, energy and counters must still equal
    the oracle at the new positions.  skin 2.5 A breaks a_p + 2 skin <= r_lo (H-H): the unbinned
    fallback, every far entry fully tested."""
    s = I.config(2)
    e = _engine_with_skin(eng_mod, s, skin)
    e.compute()  # builds the lists at s.x
    rng = np.random.default_rng(7)
    d = rng.normal(size=s.x.shape)
    d *= (0.49 * skin * rng.uniform(0.2, 1.0, size=(s.n, 1))) / np.linalg.norm(d, axis=1, keepdims=True)
    out = np.any((s.x + d < 0.0) | (s.x + d >= s.box), axis=1)
    d[out] = 0.0  # no atom crosses a face (a wrap would count as a box-length displacement)
    x = s.x + d
    nb0 = e.stats()["n_rebuilds"]
    e.set_positions(x)
    g = e.compute()
    assert e.stats()["n_rebuilds"] == nb0  # evaluated on the lists of the first build
    o = O.compute(s.types, x, s.box)
    check_fp64(s, g, o)
    st = e.stats()
    for k in COUNTERS:
        assert st[k] == o["counters"][k], (skin, k, st[k], o["counters"][k])
    # the LJ half pairs within r_c at the displaced positions, from the build-time rows
    a = e.get_list(2)
    b = O.get_list(s.types, x, s.box, 2)
    assert a.shape == b.shape and np.array_equal(a, b)
