"""CPU pins of the oracle's potential variants (param key `potential`):
REBO (the REBO bond terms only) and AIREBO-M (the LJ radial form replaced by Morse, SPEC S:71,
every gate / switch / taper kept, reading A31).  Each pin is a property the variant must have,
not a retyped formula: the Morse well depth and zero force at r_e, the curvature the toy rule
shares with the LJ well, the asymptotic decay rate, finite differences of the oracle's own
energy, the identity of the REBO bond energy with AIREBO's, and invariants."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I


def variant(text, name):
    out = text.replace(b"potential airebo\n", b"potential " + name.encode() + b"\n")
    assert out != text or name == "airebo"
    return out


def pval(text, key):
    for line in text.decode().splitlines():
        w = line.split("#")[0].split()
        if w and w[0] == key:
            return float(w[1])
    raise KeyError(key)


def dimer(r, L=40.0):
    x0 = np.array([[L / 2, L / 2, L / 2]])
    return np.concatenate([x0, x0 + [r, 0, 0]]), np.array([L, L, L])


def test_variant_parse_errors(params_text):
    with pytest.raises(RuntimeError) as ei:
        O.compute([0, 0], *dimer(4.0), params=variant(params_text, "lennard"))
    assert "potential" in str(ei.value)
    bad = variant(params_text, "airebo-m").replace(b"morse.CH.re", b"morse.CH.rx")
    with pytest.raises(RuntimeError) as ei:
        O.compute([0, 0], *dimer(4.0), params=bad)
    assert "morse.CH.re" in str(ei.value)


def test_morse_well_depth_zero_force_and_curvature(params_text):
    """Unbonded C-C dimer (r > r_max, no paths: C = 1), at r = r_e: S_r = 0 at the window's upper
    end 2^(1/6) sigma = r_e and the taper is 1, so E = V_M(r_e) = -eps_m and F = 0.  The toy rule
    gives the Morse well the LJ well's curvature, so the oracle's AIREBO-M and AIREBO energies
    must share E''(r_e) (one branch pins the other)."""
    pm = variant(params_text, "airebo-m")
    eps, re = pval(pm, "morse.CC.eps"), pval(pm, "morse.CC.re")
    x, box = dimer(re)
    res = O.compute([0, 0], x, box, params=pm)
    assert abs(res["E"] + eps) <= 1e-15
    assert np.abs(res["F"]).max() <= 1e-13
    h = 1e-3

    def curv(p):
        e = [O.compute([0, 0], *dimer(re + k * h), params=p, forces=False)["E"] for k in (-1, 0, 1)]
        return (e[0] - 2 * e[1] + e[2]) / h ** 2

    k_m, k_lj = curv(pm), curv(params_text)
    assert abs(k_m - k_lj) <= 1e-4 * abs(k_lj), (k_m, k_lj)


def test_morse_asymptotic_decay(params_text):
    """Far outside the well (and inside r_lo) V_M -> -2 eps_m e^{-a (r - r_e)}: successive
    energies at spacing 1 A decay by e^{-a} up to the e^{-a (r - r_e)} correction."""
    pm = variant(params_text, "airebo-m")
    a, re = pval(pm, "morse.CC.alpha"), pval(pm, "morse.CC.re")
    r1, r2 = 7.5, 8.5
    e1 = O.compute([0, 0], *dimer(r1), params=pm, forces=False)["E"]
    e2 = O.compute([0, 0], *dimer(r2), params=pm, forces=False)["E"]
    corr = math.exp(-a * (r1 - re))
    assert abs(e2 / e1 - math.exp(-a)) <= 2 * corr * math.exp(-a)


def fd_check(s, params, atoms, h=1e-4, tol=1e-6):
    res = O.compute(s.types, s.x, s.box, params=params)
    worst = 0.0
    for a in atoms:
        for c in range(3):
            e = []
            for k in (-2, -1, 1, 2):
                xp = s.x.copy()
                xp[a, c] += k * h
                e.append(O.compute(s.types, xp, s.box, params=params, forces=False)["E"])
            g = -(8 * (e[2] - e[1]) - (e[3] - e[0])) / (12 * h)
            worst = max(worst, abs(g - res["F"][a, c]) / max(abs(res["F"][a, c]), 1.0))
    assert worst <= tol, worst
    return res


@pytest.mark.parametrize("name", ["rebo", "airebo-m"])
def test_variant_forces_fd_and_invariants(params_text, name):
    p = variant(params_text, name)
    s = I.random_cluster(30, 1, spread=5.0, dmin=1.0)
    res = fd_check(s, p, range(s.n))
    assert np.abs(res["F"].sum(0)).max() < 1e-10
    rng = np.random.default_rng(3)
    perm = rng.permutation(s.n)
    r2 = O.compute(s.types[perm], s.x[perm], s.box, params=p)
    assert abs(r2["E"] - res["E"]) <= 1e-12 * abs(res["E"])
    assert np.abs(r2["F"] - res["F"][perm]).max() <= 1e-10
    fd_check(I.config(1), p, range(0, 120, 17))


def test_rebo_is_the_bond_part_of_airebo(params_text):
    """REBO = the REBO bond terms alone: E_TORS = E_LJ = 0, no LJ pairs, and the bond energy,
    the bond/dihedral counters equal AIREBO's on the same system."""
    pr = variant(params_text, "rebo")
    for s in (I.config(1), I.random_cluster(30, 2, spread=5.0, dmin=1.0)):
        a = O.compute(s.types, s.x, s.box)
        r = O.compute(s.types, s.x, s.box, params=pr)
        assert r["terms"][1] == 0.0 and r["terms"][2] == 0.0
        assert r["terms"][0] == a["terms"][0]
        for k in ("n_bonds", "n_quads", "n_short"):
            assert r["counters"][k] == a["counters"][k]
        assert r["counters"]["n_lj"] == 0 and r["counters"]["max_reach"] == 0
        assert len(O.get_list(s.types, s.x, s.box, 2, params=pr)) == 0


def test_airebo_m_keeps_gates(params_text):
    """AIREBO-M changes only V: the gate statistics (C_ij == 0 pairs, b* pairs) are those of
    AIREBO on the same configuration."""
    pm = variant(params_text, "airebo-m")
    s = I.random_cluster(40, 3, spread=6.0, dmin=1.0)
    a = O.compute(s.types, s.x, s.box, forces=False)
    m = O.compute(s.types, s.x, s.box, params=pm, forces=False)
    for k in ("n_lj", "n_C0", "n_bstar", "n_sb_trans"):
        assert m["counters"][k] == a["counters"][k], k
    assert m["terms"][0] == a["terms"][0] and m["terms"][1] == a["terms"][1]
    assert m["terms"][2] != a["terms"][2]
