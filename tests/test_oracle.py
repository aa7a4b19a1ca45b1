"""Pins of the fp64 CPU oracle against things other than itself (closed forms, brute force,
invariants, finite differences, library routines).  CPU only (-m "not gpu")."""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I
from tests import closed_forms as CF

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "survey_worked_examples.json")))


def big_box(x, L=60.0):
    x = np.asarray(x, dtype=np.float64)
    return x - x.mean(0) + L / 2, np.array([L, L, L])


# ------------------------------------------------------------------------ parameters
def test_params_parse_and_errors(params_text):
    ok, _ = O.parse_ok(params_text)
    assert ok
    bad = params_text.replace(b"pair.CC.rmin 1.7", b"pair.CC.rmin 2.5")
    ok, msg = O.parse_ok(bad)
    assert not ok and "pair.CC.rmin" in msg and "rmax" in msg
    bad = params_text.replace(b"lambda.HCH 0.0\n", b"")
    ok, msg = O.parse_ok(bad)
    assert not ok and "lambda.HCH" in msg
    bad = b"12.0 3.0\n" + params_text
    ok, msg = O.parse_ok(bad)
    assert not ok and "line 1" in msg


# ------------------------------------------------------------------------ switch / splines
def test_switch_closed_form_and_fd():
    lo, hi = 1.7, 2.0
    assert O.switch(lo, lo, hi)[0] == 1.0
    assert O.switch(hi, lo, hi)[0] == 0.0
    assert abs(O.switch(0.5 * (lo + hi), lo, hi)[0] - 0.5) < 1e-15
    xs = np.linspace(lo - 0.1, hi + 0.1, 64)
    vals = np.array([O.switch(x, lo, hi) for x in xs])
    assert np.all(np.diff(vals[:, 0]) <= 1e-15)  # monotone non-increasing
    h = 1e-6
    for x in xs[(xs > lo + 1e-3) & (xs < hi - 1e-3)]:
        fd = (O.switch(x + h, lo, hi)[0] - O.switch(x - h, lo, hi)[0]) / (2 * h)
        d = O.switch(x, lo, hi)[1]
        assert abs(fd - d) <= 1e-7 * max(1.0, abs(d))
        assert abs(d - (-0.5 * math.pi * math.sin(math.pi * (x - lo) / (hi - lo)) / (hi - lo))) < 1e-12


def test_g_spline_matches_scipy_hermite():
    for sp, k in (("C", 0), ("H", 1)):
        ref = CF.g_spline(sp)
        dref = ref.derivative()
        for c in np.linspace(-1.2, 1.2, 97):
            o = O.spline(0, k, c)
            cc = min(1.0, max(-1.0, c))
            assert abs(o[0] - float(ref(cc))) < 1e-13
            if -1 < c < 1:
                assert abs(o[1] - float(dref(c))) < 1e-11
            else:
                assert o[1] == 0.0  # clamped: zero derivative


def test_grid_splines_knots_bilinear_and_c1():
    kv = CF.KV
    # exact at knots
    for x in range(5):
        for y in range(5):
            assert O.spline(1, 0, x, y)[0] == kv["P.CC"][x * 5 + y]
            for z in range(1, 10):
                assert O.spline(2, 1, x, y, z)[0] == pytest.approx(kv["R.CH"][(x * 5 + y) * 9 + z - 1], abs=1e-17)
                assert O.spline(3, 0, x, y, z)[0] == pytest.approx(kv["T.CC"][(x * 5 + y) * 9 + z - 1], abs=1e-17)
    # P_CC is bilinear in (a, b) on the grid (a*b term) -> reproduced exactly in interior cells
    for a in (1.3, 2.5, 2.9):
        for b in (1.1, 2.7):
            exact = -0.02 * a - 0.01 * b + 0.003 * a * b
            assert abs(O.spline(1, 0, a, b)[0] - exact) < 1e-15
    # C1 continuity across cell boundaries and gradient vs FD
    rng = np.random.default_rng(7)
    h = 1e-7
    for _ in range(40):
        x, y = rng.uniform(0, 4, 2)
        z = rng.uniform(1, 9)
        o = O.spline(2, 0, x, y, z)
        for ax in range(3):
            p = [x, y, z]
            m = [x, y, z]
            p[ax] += h
            m[ax] -= h
            fd = (O.spline(2, 0, *p)[0] - O.spline(2, 0, *m)[0]) / (2 * h)
            assert abs(fd - o[1 + ax]) < 1e-7
    for knot in (1.0, 2.0, 3.0):
        e = 1e-9
        lo, hi = O.spline(3, 0, knot - e, 2.5, 4.5), O.spline(3, 0, knot + e, 2.5, 4.5)
        assert abs(lo[0] - hi[0]) < 1e-11 and abs(lo[1] - hi[1]) < 1e-7
    # clamped outside the grid with zero derivative
    o = O.spline(2, 0, -1.0, 6.0, 12.0)
    assert o[0] == CF.KV["R.CC"][(0 * 5 + 4) * 9 + 8] and o[1] == o[2] == o[3] == 0.0


# ------------------------------------------------------------------------ lists
@pytest.mark.parametrize("which", [0, 1, 2])
def test_lists_cell_vs_bruteforce(which):
    systems = [I.config(1), I.polyethylene((1, 1, 1), 0.03, 5, None), I.diamond((1, 1, 1), 0.03, 9),
               I.random_cluster(25, 3)]
    for s in systems:
        a = O.get_list(s.types, s.x, s.box, which)
        b = O.get_list(s.types, s.x, s.box, which, brute=True)
        assert a.shape == b.shape and np.array_equal(a, b)


def test_short_list_symmetric_and_exact():
    s = I.config(1)
    rows = O.get_list(s.types, s.x, s.box, 0)
    fwd = {tuple(r) for r in rows}
    for i, j, sx, sy, sz in rows:
        assert (j, i, -sx, -sy, -sz) in fwd
    # independent min-image check (box > 2 r_max in every direction here)
    X, L = s.x, s.box
    rm = {(0, 0): 2.0, (0, 1): 1.8, (1, 0): 1.8, (1, 1): 1.5}
    d = X[None, :, :] - X[:, None, :]
    d -= L * np.round(d / L)
    r = np.sqrt((d ** 2).sum(-1))
    cnt = sum(1 for i in range(s.n) for j in range(s.n) if i != j and r[i, j] <= rm[(s.types[i], s.types[j])])
    assert cnt == len(rows)


# ------------------------------------------------------------------------ closed forms
def test_dimer_closed_form():
    x0 = np.array([[20.0, 20.0, 20.0]])
    box = np.array([40.0, 40.0, 40.0])
    R00 = CF.tab_RT("R", "CC", 0, 0, 1)
    for r, Eg in zip(GOLD["dimer_cc_rebo"]["r"], GOLD["dimer_cc_rebo"]["E"]):
        x = np.concatenate([x0, x0 + [r, 0, 0]])
        res = O.compute([0, 0], x, box)
        b = 0.5 * (1 + 1) + R00  # isolated dimer: p = (1 + P_CC(0,0))^-1/2 = 1, N^conj = 1
        closed = CF.fR(r) + b * CF.fA(r)
        assert abs(res["terms"][0] - closed) < 1e-12 * abs(closed)
        assert abs(res["terms"][0] - Eg) < 2e-12
        assert res["terms"][1] == 0.0 and res["terms"][2] == 0.0
        assert abs(res["F"].sum(0)).max() < 1e-12
    for r, Eg in zip(GOLD["dimer_cc_lj"]["r"], GOLD["dimer_cc_lj"]["E"]):
        x = np.concatenate([x0, x0 + [r, 0, 0]])
        res = O.compute([0, 0], x, box)
        sig = CF.p1("lj.CC.sigma")
        P = CF.S(r, sig, sig * 1.122462048309373)
        closed = (1 - P) * CF.V_lj(r)  # b* = 1.02 > b_max -> S_b = 0 -> Q = 1 - S_r
        assert abs(res["terms"][2] - closed) < 1e-15 + 1e-12 * abs(closed)
        assert abs(res["terms"][2] - Eg) < 1e-14


def test_trimer_closed_form():
    for th in (95.0, 112.0, 125.0, 150.0):
        t = math.radians(th)
        x = np.array([[0, 0, 0], [1.4, 0, 0], [1.4 * math.cos(t), 1.4 * math.sin(t), 0]])
        x, box = big_box(x)
        res = O.compute([0, 0, 0], x, box)
        ref = CF.trimer_energy(th)
        assert abs(res["E"] - ref) < 1e-12 * abs(ref)


def test_perfect_diamond_worked_example():
    g = GOLD["perfect_diamond"]
    cf = CF.diamond_energy_per_atom(g["a"])
    assert cf["n_far"] == g["lj_partners_C1_per_atom"]
    assert abs(cf["p"] - g["p"]) < 1e-12 and abs(cf["b"] - g["b"]) < 1e-12
    s = I.diamond((3, 3, 3))
    res = O.compute(s.types, s.x, s.box)
    n = s.n
    assert abs(res["terms"][0] / n - cf["rebo"]) < 1e-12
    assert abs(res["terms"][1] / n) < 1e-14  # torsion cancels exactly for uniform eps (SURVEY c-4)
    assert abs(res["terms"][2] / n - cf["lj"]) < 1e-13
    assert abs(res["E"] / n - g["E_per_atom"]) < 1e-11
    assert np.abs(res["F"]).max() < 1e-12
    assert res["counters"]["max_reach"] == g["reach_set_size"]
    assert res["counters"]["n_quads"] == 18 * n  # 9 per bond, 2 bonds per atom
    # virial: W_xx = W_yy = W_zz = -(a/3) dE/da, off-diagonals 0
    h = 1e-5
    dEda = (CF.diamond_energy_per_atom(g["a"] + h)["E"] - CF.diamond_energy_per_atom(g["a"] - h)["E"]) / (2 * h)
    W = res["W"] / n
    assert np.allclose(W[:3], -(g["a"] / 3) * dEda, rtol=1e-7, atol=0)
    assert abs(W[0] - g["W_diag_per_atom"]) < 1e-6
    assert np.abs(W[3:]).max() < 1e-13


def test_diamond_bstar_shell4():
    """b* of the 4-bond shell (3.567 A): cos theta in {+-1/sqrt 3}, N^C_ij = 4, N^conj = 1,
    sum (1 - cos^2 w) = 8 (SURVEY c-4 'b* / S_b')."""
    s = I.diamond((3, 3, 3))
    rows = O.get_list(s.types, s.x, s.box, 2)
    B, Lj = O.stages(s.types, s.x, s.box)
    g = CF.g_spline("C")
    c = 1 / math.sqrt(3)
    ref = (1 + 2 * float(g(c)) + 2 * float(g(-c)) + CF.tab_P("CC", 4, 0)) ** -0.5 \
        + CF.tab_RT("R", "CC", 4, 4, 1) + 8 * CF.tab_RT("T", "CC", 4, 4, 1)
    d = s.x[rows[:, 1]] + rows[:, 2:5] * s.box - s.x[rows[:, 0]]
    r = np.linalg.norm(d, axis=1)
    sh4 = np.abs(r - 3.567) < 1e-9
    assert sh4.sum() == 3 * s.n  # 6 per atom, half pairs
    assert np.all(np.abs(Lj[sh4, 1] - ref) < 1e-13)
    assert np.all(Lj[sh4, 0] == 1.0)
    assert np.all(np.abs(B[:, 0] - GOLD["perfect_diamond"]["b"]) < 1e-12)


def test_torsion_bruteforce_pe():
    """All-quadruple brute-force torsion on jittered PE (min image valid: r_max < L/2)."""
    s = I.config(1)
    X, L, t = s.x, s.box, s.types
    kv = CF.KV
    rmax = {(0, 0): 2.0, (0, 1): 1.8, (1, 0): 1.8, (1, 1): 1.5}
    pk = {(0, 0): "CC", (0, 1): "CH", (1, 0): "CH", (1, 1): "HH"}
    d = X[None, :, :] - X[:, None, :]
    d -= L * np.round(d / L)
    r = np.sqrt((d ** 2).sum(-1))
    nb = [[j for j in range(s.n) if j != i and r[i, j] <= rmax[(t[i], t[j])]] for i in range(s.n)]
    S_ = lambda q: "CH"[q]

    def w(a, b):
        p = pk[(t[a], t[b])]
        return CF.S(r[a, b], kv[f"pair.{p}.rmin"][0], kv[f"pair.{p}.rmax"][0])

    def G(c):
        return 1 - CF.S(1 - c * c, kv["dihedral.sin2_lo"][0], kv["dihedral.sin2_hi"][0])

    E = 0.0
    nq = 0
    for i in range(s.n):
        for j in nb[i]:
            if not i < j:
                continue
            for k in nb[i]:
                if k == j:
                    continue
                for l in nb[j]:
                    if l in (i, k):
                        continue
                    nq += 1
                    a, b, e = d[i, k], d[i, j], d[j, l]
                    cjik = a @ b / (np.linalg.norm(a) * np.linalg.norm(b))
                    cijl = (-b) @ e / (np.linalg.norm(b) * np.linalg.norm(e))
                    n1, n2 = np.cross(a, b), np.cross(-b, e)
                    cw = n1 @ n2 / (np.linalg.norm(n1) * np.linalg.norm(n2))
                    V = (256 / 405) * ((1 + cw) / 2) ** 5 - 0.1
                    eps = kv[f"tors.{S_(t[k])}{S_(t[i])}{S_(t[j])}{S_(t[l])}"][0]
                    E += eps * w(i, k) * w(i, j) * w(j, l) * G(cjik) * G(cijl) * V
    res = O.compute(s.types, s.x, s.box, lj=False)
    assert res["counters"]["n_quads"] == nq == 360
    assert abs(res["terms"][1] - E) < 1e-12 * max(1.0, abs(E))


def test_cij_bruteforce_maxproduct():
    """C_ij of every LJ pair of random clusters vs a brute-force max-product path search."""
    for seed in (0, 1, 4):
        s = I.random_cluster(30, seed, spread=5.0, dmin=1.0)
        X, t = s.x, s.types
        rmin = np.array([[1.7, 1.3], [1.3, 1.1]])
        rmax = np.array([[2.0, 1.8], [1.8, 1.5]])
        D = np.linalg.norm(X[:, None] - X[None], axis=-1)
        W = np.zeros_like(D)
        for a in range(s.n):
            for b in range(s.n):
                if a != b and D[a, b] <= rmax[t[a], t[b]]:
                    W[a, b] = CF.S(D[a, b], rmin[t[a], t[b]], rmax[t[a], t[b]])
        M = CF.maxprod_paths(W)
        rows = O.get_list(s.types, s.x, s.box, 2)
        _, Lj = O.stages(s.types, s.x, s.box)
        for (i, j, *_), c in zip(rows, Lj[:, 0]):
            assert abs(c - (1 - M[i, j])) < 1e-15


# ------------------------------------------------------------------------ forces and invariants
def fd_check(s, atoms, h=1e-4, tol=1e-6):
    res = O.compute(s.types, s.x, s.box)
    F = res["F"]
    worst = 0.0
    for a in atoms:
        for c in range(3):
            e = []
            for k in (-2, -1, 1, 2):
                xp = s.x.copy()
                xp[a, c] += k * h
                e.append(O.compute(s.types, xp, s.box, forces=False)["E"])
            g = -(8 * (e[2] - e[1]) - (e[3] - e[0])) / (12 * h)
            err = abs(g - F[a, c]) / max(abs(F[a, c]), 1.0)
            worst = max(worst, err)
    assert worst <= tol, worst
    return res


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_fd_random_clusters_switching_regions(seed):
    s = I.random_cluster(30, seed, spread=5.0, dmin=1.0)
    res = fd_check(s, range(s.n))
    c = res["counters"]
    assert c["n_badarg"] == 0
    # these clusters exercise fractional weights, C-path and S_b transition derivatives
    assert c["n_sb_trans"] > 0 and c["n_C0"] < c["n_lj"]
    assert np.abs(res["F"].sum(0)).max() < 1e-10


def test_fd_periodic_pe_and_diamond():
    fd_check(I.config(1), range(0, 120, 11))
    fd_check(I.diamond((1, 1, 1), 0.05, 11), range(8))


def test_invariances_cluster():
    s = I.random_cluster(30, 5, spread=5.0, dmin=1.0)
    base = O.compute(s.types, s.x, s.box)
    c0 = s.x.mean(0)
    # zero net force and torque
    assert np.abs(base["F"].sum(0)).max() < 1e-10
    assert np.abs(np.cross(s.x - c0, base["F"]).sum(0)).max() < 1e-8
    # translation
    xt = s.x + np.array([0.31, -0.72, 1.13])
    assert abs(O.compute(s.types, xt, s.box, forces=False)["E"] - base["E"]) < 1e-10
    # rotation
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    xr = (s.x - c0) @ q.T + c0
    rr = O.compute(s.types, xr, s.box)
    assert abs(rr["E"] - base["E"]) < 1e-9
    assert np.abs(rr["F"] - base["F"] @ q.T).max() < 1e-9
    # permutation
    p = rng.permutation(s.n)
    rp = O.compute(s.types[p], s.x[p], s.box)
    assert abs(rp["E"] - base["E"]) < 1e-10 * abs(base["E"])
    assert np.abs(rp["F"] - base["F"][p]).max() < 1e-10


def test_separability():
    a = I.random_cluster(20, 1, spread=4.0, dmin=1.0)
    b = I.random_cluster(20, 2, spread=4.0, dmin=1.0)
    xa = a.x - a.x.mean(0) + [15.0, 30, 30]
    xb = b.x - b.x.mean(0) + [45.0, 30, 30]  # > r_c apart, box 60
    box = np.array([60.0, 60, 60])
    ea = O.compute(a.types, xa, box, forces=False)["E"]
    eb = O.compute(b.types, xb, box, forces=False)["E"]
    eab = O.compute(np.concatenate([a.types, b.types]), np.concatenate([xa, xb]), box, forces=False)["E"]
    assert abs(eab - (ea + eb)) < 1e-10 * abs(eab)


def test_periodic_translation_and_axis_permutation():
    s = I.diamond((2, 2, 2), 0.04, 21)
    base = O.compute(s.types, s.x, s.box)
    xt = I.wrap(s.x + np.array([1.234, -0.567, 2.891]), s.box)
    assert abs(O.compute(s.types, xt, s.box, forces=False)["E"] - base["E"]) < 1e-10
    xp = s.x[:, [1, 2, 0]]
    rp = O.compute(s.types, xp, s.box)
    assert abs(rp["E"] - base["E"]) < 1e-10
    assert np.abs(rp["F"] - base["F"][:, [1, 2, 0]]).max() < 1e-10


def test_replication_invariance_multi_image():
    """PE cell 1x1x1 (c = 2.54 A < 2 r_max: an atom meets its own images) vs 1x1x10 vs 2x2x1."""
    out = []
    for reps in ((1, 1, 1), (1, 1, 10), (2, 2, 1)):
        s = I.polyethylene(reps, 0.0, 1, None)
        r = O.compute(s.types, s.x, s.box)
        out.append((r["E"] / s.n, r["terms"] / s.n, r["W"] / s.n))
    for o in out[1:]:
        assert abs(o[0] - out[0][0]) < 1e-12 * abs(out[0][0])
        assert np.allclose(o[1], out[0][1], rtol=1e-11, atol=1e-14)
        assert np.allclose(o[2], out[0][2], rtol=1e-9, atol=1e-12)


def test_virial_vs_strain_fd():
    # periodic, diagonal: scale x_a and L_a by (1 + eps)
    s = I.config(1)
    W = O.compute(s.types, s.x, s.box)["W"]
    eps = 1e-6
    for ax in range(3):
        f = np.ones(3)
        f[ax] = 1 + eps
        ep = O.compute(s.types, s.x * f, s.box * f, forces=False)["E"]
        f[ax] = 1 - eps
        em = O.compute(s.types, s.x * f, s.box * f, forces=False)["E"]
        fd = -(ep - em) / (2 * eps)
        assert abs(W[ax] - fd) <= 1e-6 * max(1.0, abs(fd))
    # cluster, full tensor: x_b -> x_b + eps x_a gives dE/deps = -W_ab
    c = I.random_cluster(25, 8, spread=5.0, dmin=1.0)
    Wc = O.compute(c.types, c.x, c.box)["W"]
    idx = {(0, 0): 0, (1, 1): 1, (2, 2): 2, (0, 1): 3, (0, 2): 4, (1, 2): 5}
    x0 = c.x - c.x.mean(0)
    for (a, b), k in idx.items():
        def E(e):
            x = x0.copy()
            x[:, b] += e * x0[:, a]
            return O.compute(c.types, x + c.x.mean(0), c.box, forces=False)["E"]
        fd = -(E(eps) - E(-eps)) / (2 * eps)
        assert abs(Wc[k] - fd) <= 1e-6 * max(1.0, abs(fd)), (a, b)


def test_sampled_forces_equal_full():
    s = I.config(1)
    full = O.compute(s.types, s.x, s.box)["F"]
    smp = np.array([0, 7, 33, 61, 119])
    Fs = O.forces_sampled(s.types, s.x, s.box, smp)
    assert np.abs(Fs - full[smp]).max() < 1e-12


def test_gate_statistics_pe_orders_of_magnitude():
    """Paper: C = 0 in 3.2 % of LJ pairs, b* needed in 2.2 %, S_b' != 0 in 0.0 %."""
    s = I.polyethylene((4, 4, 6), 0.02, 102, None)
    c = O.compute(s.types, s.x, s.box, forces=False)["counters"]
    assert 0.005 < c["n_C0"] / c["n_lj"] < 0.1
    assert 0.005 < c["n_bstar"] / c["n_lj"] < 0.1
    assert c["n_sb_trans"] == 0
    assert c["n_bonds"] == s.n and c["n_quads"] == 3 * s.n  # 9 quads per C-C bond, n/3 C-C bonds


# ------------------------------------------------------------------------ NVE
def test_nve_free_flight_and_reversibility():
    # two atoms far apart (> r_c): zero force -> free flight
    x = np.array([[5.0, 5, 5], [25.0, 25, 25]])
    v = np.array([[0.01, -0.02, 0.005], [-0.003, 0.0, 0.002]])
    box = np.array([40.0, 40, 40])
    x1, v1, _ = O.nve([0, 1], x, v, box, 10, 0.5, every=0)
    assert np.allclose(x1, x + 10 * 0.5 * v, atol=1e-12) and np.array_equal(v1, v)
    # reversibility
    s = I.config(1)
    xa, va, _ = O.nve(s.types, s.x, s.v, s.box, 20, 0.5, every=0)
    xb, vb, _ = O.nve(s.types, xa, -va, s.box, 20, 0.5, every=0)
    dx = xb - s.x
    dx -= s.box * np.round(dx / s.box)
    assert np.abs(dx).max() < 1e-8


@pytest.mark.slow
def test_nve_energy_drift_dt2_scaling():
    s = I.config(1)
    _, _, th1 = O.nve(s.types, s.x, s.v, s.box, 100, 0.5, every=1)
    _, _, th2 = O.nve(s.types, s.x, s.v, s.box, 200, 0.25, every=1)
    d1 = np.abs(th1[:, 3] - th1[0, 3]).max()
    d2 = np.abs(th2[:, 3] - th2[0, 3]).max()
    assert 3.0 <= d1 / d2 <= 5.0, (d1, d2)


@pytest.mark.parametrize("nm", [(10, 10), (12, 0), (8, 4), (6, 1)])
def test_nanotube_generator(nm):
    """The CNT generator (no method arithmetic) against graphene geometry: every atom has exactly
    three neighbours within r_max, nearest-neighbour distances are the C-C bond shortened only by
    the curvature, the radius is a sqrt(n^2 + nm + m^2) / (2 pi), and the atom count per
    translational cell is 4 (n^2 + nm + m^2) / gcd(2m + n, 2n + m)."""
    n, m = nm
    s = I.nanotube(n, m, 2, vacuum=10.0)
    rows = O.get_list(s.types, s.x, s.box, 0)
    assert np.all(np.bincount(rows[:, 0], minlength=s.n) == 3)
    d = s.x[rows[:, 1]] + rows[:, 2:] * s.box - s.x[rows[:, 0]]
    r = np.sqrt((d ** 2).sum(1))
    assert r.max() <= 1.42 + 1e-9 and r.min() >= 1.42 * 0.97
    a = 1.42 * math.sqrt(3.0)
    R = a * math.sqrt(n * n + n * m + m * m) / (2 * math.pi)
    rad = np.sqrt((s.x[:, 0] - s.box[0] / 2) ** 2 + (s.x[:, 1] - s.box[1] / 2) ** 2)
    assert np.abs(rad - R).max() <= 1e-9
    assert s.n == 2 * 4 * (n * n + n * m + m * m) // math.gcd(2 * m + n, 2 * n + m)
