"""Pins of the oracle's SURVEY §8(f) F3 functional details (params/toy_ch_f3.param; readings
A33 / A34 of DESIGN.md), CPU only:

  A33  lambda_jik = lambda.JIK + kappa delta(t_i, H) [(rho_{t_k H} - r_ik) - (rho_{t_j H} - r_ij)]
       (P:505-506 prints e^{lambda_jik}; "every occurrence of r_ij is replaced by a
       constant" in b*, which with this lambda makes the fictitious distance rho matter;
       P:650-651 names the Kronecker-delta factors and the r_ij construction of b* as bug sources)
  A34  g_C(cos, N) = g_C2(cos) + S(N; nlo, nhi) (g_C(cos) - g_C2(cos)), N = N_i - w_ij

Closed forms: an H-bridged C-H-C trimer and an H-C-H fragment (REBO energies written out from the
definitions with scipy splines and the table values), the b* of an H-centred LJ pair (lambda at
r_ij = rho), p_ij of a carbon with fractional coordination in the blend window; invariants
(coordination below / above the window reduces to g_C / g_C2); FD forces on switching-region
clusters.  Nothing here is imported by oracle/ or the CUDA package.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I
from tests import closed_forms as CF
from tests.test_oracle_pins_r2 import hermite_1d, tensor_2d, tensor_3d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F3 = os.path.join(ROOT, "params", "toy_ch_f3.param")
KV3 = CF.read_params(F3)


@pytest.fixture(scope="module")
def f3_text():
    return open(F3, "rb").read()


def p1(k):
    return KV3[k][0]


def gH(c):
    return hermite_1d(KV3["angle.H.knots"], KV3["angle.H.values"], c)


def gC(c, N):
    g1 = hermite_1d(KV3["angle.C.knots"], KV3["angle.C.values"], c)
    g2 = hermite_1d(KV3["angle.C2.knots"], KV3["angle.C2.values"], c)
    return g2 + CF.S(N, p1("angle.C.nlo"), p1("angle.C.nhi")) * (g1 - g2)


def R3(pair, x, y, z):
    return tensor_3d(KV3[f"R.{pair}"], x, y, z)


def P2(pair, a, b):
    return tensor_2d(KV3[f"P.{pair}"], a, b)


def put(*pts):
    x = np.array(pts, dtype=float)
    return x - x.mean(0) + 20.0, np.array([40.0, 40.0, 40.0])


def test_f3_file_is_base_plus_keys(params_text, f3_text):
    assert f3_text.startswith(params_text.rstrip(b"\n"))
    assert p1("lambda.kappa") == 4.0 and len(KV3["angle.C2.values"]) == len(KV3["angle.C.knots"])


def test_h_bridge_trimer_lambda_of_r(f3_text):
    """C(j) - H(i) - C(k), both C-H bonds on the plateau, j-k beyond r_max: per bond
    b = 1/2 (p_ij + p_ji) + R_CH(0, 1, 2), p_ij = (1 + g_H(cos) e^{lambda})^{-1/2},
    lambda_jik = lambda.CHC + kappa (r_ij - r_ik) (rho_CH cancels), p_ji = (1 + P_CH(0, 0))^{-1/2};
    C_jk = 0 through the bridge, no dihedrals, no torsion."""
    kap, lam0 = p1("lambda.kappa"), p1("lambda.CHC")
    for r1, r2, th in ((1.12, 1.2, 150.0), (1.05, 1.27, 140.0), (1.18, 1.1, 165.0)):
        t = math.radians(th)
        x, box = put([0, 0, 0], [r1, 0, 0], [r2 * math.cos(t), r2 * math.sin(t), 0])
        c = math.cos(t)
        pji = (1 + P2("CH", 0, 0)) ** -0.5
        E = 0.0
        for ra, rb in ((r1, r2), (r2, r1)):  # bond i-a with the other C (b) as k
            pij = (1 + gH(c) * math.exp(lam0 + kap * (ra - rb))) ** -0.5
            b = 0.5 * (pij + pji) + R3("CH", 0, 1, 2)
            E += CF.fR(ra, "CH") + b * CF.fA(ra, "CH")
        o = O.compute([1, 0, 0], x, box, params=f3_text)
        assert abs(o["terms"][0] - E) < 1e-12 * abs(E), (r1, r2, th, o["terms"][0], E)
        assert o["terms"][1] == 0.0 and abs(o["terms"][2]) < 1e-300


def test_h_c_h_fragment_carbon_centre_lambda_constant(f3_text):
    """H(j) - C(i) - H(k): the C-centred lambda stays the constant lambda.HCH (delta(t_i, H) = 0)
    whatever the bond lengths; the H centres have no other neighbour (no lambda at all)."""
    for r1, r2, th in ((1.09, 1.2, 109.0), (1.15, 1.05, 120.0)):
        t = math.radians(th)
        x, box = put([0, 0, 0], [r1, 0, 0], [r2 * math.cos(t), r2 * math.sin(t), 0])
        c = math.cos(t)
        E = 0.0
        for ra in (r1, r2):
            pij = (1 + gC(c, 1.0) * math.exp(p1("lambda.HCH")) + P2("CH", 0, 1)) ** -0.5
            b = 0.5 * (pij + 1.0) + R3("CH", 1, 0, 1)
            E += CF.fR(ra, "CH") + b * CF.fA(ra, "CH")
        o = O.compute([0, 1, 1], x, box, params=f3_text)
        assert abs(o["terms"][0] - E) < 1e-12 * abs(E), (r1, r2, th)


def test_bstar_h_centre_uses_rho_for_r_ij(f3_text):
    """LJ pair H(i) ... C(j) inside the S_r window, H bonded to C(k): b*_ij with d_ij -> rho d_hat
    (P:491): lambda*_jik = lambda.CHC + kappa (rho_CH - r_ik) -- the r_ij of lambda is rho too."""
    kap, lam0, rho = p1("lambda.kappa"), p1("lambda.CHC"), p1("lj.CH.rho")
    rik, rij, th = 1.15, 3.2, 100.0
    t = math.radians(th)
    x, box = put([0, 0, 0], [rij, 0, 0], [rik * math.cos(t), rik * math.sin(t), 0])
    rows = O.get_list([1, 0, 0], x, box, 2, params=f3_text)
    _, Lj = O.stages([1, 0, 0], x, box, params=f3_text)
    q = next(n for n, r in enumerate(rows) if (r[0], r[1]) == (0, 1))
    pij = (1 + gH(math.cos(t)) * math.exp(lam0 + kap * (rho - rik))) ** -0.5
    pji = (1 + P2("CH", 0, 0)) ** -0.5
    ref = 0.5 * (pij + pji) + R3("CH", 0, 1, 2)
    assert Lj[q, 0] == 1.0 and Lj[q, 1] != 0.0
    assert abs(Lj[q, 1] - ref) < 1e-13, (Lj[q, 1], ref)
    # the actual distance in lambda would give a different b*
    bad = 0.5 * ((1 + gH(math.cos(t)) * math.exp(lam0 + kap * ((rho - rik) - (rho - rij)))) ** -0.5 + pji) \
        + R3("CH", 0, 1, 2)
    assert abs(bad - ref) > 1e-3


def blend_carbon(w_frac_r):
    """C(i) with C(j), three plateau C neighbours and an H in the C-H switching window."""
    rng = np.random.default_rng(5)
    dirs = [np.array([1.0, 0, 0])]
    while len(dirs) < 5:
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        if all(np.dot(v, u) < math.cos(math.radians(62)) for u in dirs):
            dirs.append(v)
    x = [np.zeros(3)] + [1.45 * d for d in dirs[:4]] + [w_frac_r * dirs[4]]
    return np.array([0, 0, 0, 0, 0, 1], dtype=np.int32), x, dirs


def test_gC_coordination_blend_p_ij(f3_text):
    """p_ij of the C-C bond (i, j) of a carbon with N_ij = 3 + w(H) in the blend window:
    p_ij = (1 + sum_k w_k g_C(cos_k, N_ij) e^{lambda.CC t_k} + P_CC(3, w))^{-1/2} (reading A34)."""
    for r_h in (1.55, 1.6, 1.45):
        types, x, dirs = blend_carbon(r_h)
        xx, box = put(*x)
        rows = O.get_list(types, xx, box, 1, params=f3_text)
        B, _ = O.stages(types, xx, box, params=f3_text)
        q = next(n for n, r in enumerate(rows) if (r[0], r[1]) == (0, 1))
        w_h = CF.S(r_h, p1("pair.CH.rmin"), p1("pair.CH.rmax"))
        N = 3.0 + w_h
        s = sum(gC(float(np.dot(dirs[0], d)), N) * math.exp(p1("lambda.CCC")) for d in dirs[1:4])
        s += w_h * gC(float(np.dot(dirs[0], dirs[4])), N) * math.exp(p1("lambda.CCH"))
        ref = (1 + s + P2("CC", 3.0, w_h)) ** -0.5
        assert abs(B[q, 1] - ref) < 1e-13, (r_h, B[q, 1], ref)
        assert abs(B[q, 5] - N) < 1e-14


def test_gC_outside_window_reduces_to_single_spline(params_text, f3_text):
    """N_ij <= nlo everywhere (PE, diamond: N_ij <= 3): g_C2 never contributes -- with kappa = 0 the
    F3 file gives bitwise the base energies.  N_ij >= nhi (a 5-coordinated carbon on the plateau):
    the F3 file equals a base file whose angle.C table is replaced by angle.C2."""
    no_kappa = f3_text.replace(b"lambda.kappa 4.0", b"lambda.kappa 0.0")
    for s in (I.polyethylene((1, 1, 2), 0.03, 3, None), I.diamond((1, 1, 1), 0.03, 4)):
        a = O.compute(s.types, s.x, s.box, params=params_text)
        b = O.compute(s.types, s.x, s.box, params=no_kappa)
        assert a["E"] == b["E"] and np.array_equal(a["F"], b["F"])
    types, x, _ = blend_carbon(1.2)  # H on the plateau: N_ij = 4 for every C-C bond of the centre
    types = np.array([0, 0, 0, 0, 0, 0], dtype=np.int32)
    x = [x[0]] + [v * 1.45 / np.linalg.norm(v) for v in x[1:]]
    xx, box = put(*x)
    swapped = params_text.replace(
        ("angle.C.values " + " ".join(str(v) for v in KV3["angle.C.values"])).encode(),
        ("angle.C.values " + " ".join(str(v) for v in KV3["angle.C2.values"])).encode())
    assert swapped != params_text
    rows = O.get_list(types, xx, box, 1, params=f3_text)
    B3, _ = O.stages(types, xx, box, params=no_kappa)
    Bs, _ = O.stages(types, xx, box, params=swapped)
    for n, r in enumerate(rows):
        if r[0] == 0:  # bonds of the 5-coordinated centre: its p_ij uses g_C2 only
            assert B3[n, 5] >= p1("angle.C.nhi")
            assert abs(B3[n, 1] - Bs[n, 1]) < 1e-15


@pytest.mark.parametrize("seed", [0, 3])
def test_f3_forces_fd(f3_text, seed):
    """Central FD of the F3 energy on switching-region clusters (fractional w, H centres, carbons
    in the g_C blend window): the lambda(r) and g_C(N) derivatives."""
    s = I.random_cluster(30, seed, spread=4.6, dmin=1.0)
    res = O.compute(s.types, s.x, s.box, params=f3_text)
    F = res["F"]
    h = 1e-4
    worst = 0.0
    for a in range(0, s.n, 2):
        for c in range(3):
            e = []
            for k in (-2, -1, 1, 2):
                xp = s.x.copy()
                xp[a, c] += k * h
                e.append(O.compute(s.types, xp, s.box, params=f3_text, forces=False)["E"])
            g = -(8 * (e[2] - e[1]) - (e[3] - e[0])) / (12 * h)
            worst = max(worst, abs(g - F[a, c]) / max(abs(F[a, c]), 1.0))
    assert worst <= 1e-6, worst
    assert np.abs(F.sum(0)).max() < 1e-10
    base = O.compute(s.types, s.x, s.box)
    assert abs(base["E"] - res["E"]) > 1e-6  # the F3 terms are active on this cluster
