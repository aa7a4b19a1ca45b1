"""Round-2 pins of the two oracle parts round 1 left pinned only where a mutation could hide:

* the knot-slope rule of the 2-D / 3-D Hermite splines P, pi^rc and T:
  central-difference slopes at interior knots and m = 0 at both end knots.  Pinned by
  (a) per-axis quadratic reproduction in cells whose two knots are interior (central
      differences are exact for quadratics; a forward / backward difference rule is not), and
  (b) every cell, boundary cells [0,1], [3,4], [8,9] included, against an independent tensor
      product of scipy ``CubicHermiteSpline`` 1-D interpolants (end slopes 0; a one-sided end
      slope fails here);
* N^C_ij, N^H_ij, N_ij and N^conj_ij with the N_k - w_ik exclusion (O4 and O5 step 4, S:246-254,
  P:500-501) re-summed independently in numpy from an all-pairs x all-images short list, on
  geometries where F(N_k - w_ik) and F(N_k) differ (a C neighbour with exactly two other
  neighbours: F(2) = 1, F(3) = 0; fractional weights in the switching region).

CPU only (-m "not gpu").  Nothing here is imported by oracle/ or the CUDA package.
"""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest
from scipy.interpolate import CubicHermiteSpline

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I
from tests import closed_forms as CF


# ------------------------------------------------------------------ parameter-text helpers
def set_table(text: bytes, key: str, values, per_line: int) -> bytes:
    """Replace the numeric block that follows the line `key` in a parameter text."""
    lines = text.decode().split("\n")
    k = next(q for q, ln in enumerate(lines) if ln.strip() == key)
    e = k + 1
    while e < len(lines) and lines[e].strip() and lines[e].split()[0][0] in "-0123456789.":
        e += 1
    vals = [repr(float(v)) for v in values]
    rows = ["  " + " ".join(vals[q:q + per_line]) for q in range(0, len(vals), per_line)]
    return "\n".join(lines[:k + 1] + rows + lines[e:]).encode()


def hermite_1d(knots, y, x):
    """SURVEY A7 1-D rule through scipy: slopes (y_{i+1} - y_{i-1}) / (x_{i+1} - x_{i-1}) inside,
    0 at both end knots, argument clamped to [x_0, x_n].  Value only."""
    knots = np.asarray(knots, float)
    y = np.asarray(y, float)
    m = np.zeros_like(y)
    m[1:-1] = (y[2:] - y[:-2]) / (knots[2:] - knots[:-2])
    xc = min(max(x, knots[0]), knots[-1])
    return float(CubicHermiteSpline(knots, y, m)(xc))


def tensor_2d(tab, x, y, n=(5, 5), lo=(0, 0)):
    kx = np.arange(n[0]) + lo[0]
    ky = np.arange(n[1]) + lo[1]
    T = np.asarray(tab, float).reshape(n)
    gy = [hermite_1d(kx, T[:, b], x) for b in range(n[1])]  # interpolate along x for each y knot
    return hermite_1d(ky, gy, y)


def tensor_3d(tab, x, y, z, n=(5, 5, 9), lo=(0, 0, 1)):
    kz = np.arange(n[2]) + lo[2]
    T = np.asarray(tab, float).reshape(n)
    gz = [tensor_2d(T[:, :, c].ravel(), x, y, n[:2], lo[:2]) for c in range(n[2])]
    return hermite_1d(kz, gz, z)


# ------------------------------------------------------------------ (a) quadratic reproduction
def q1(a):
    return 0.3 - 0.7 * a + 0.45 * a * a


def q2(b):
    return -1.1 + 0.2 * b - 0.35 * b * b


def q3(c):
    return 0.5 + 0.13 * c + 0.021 * c * c


def test_quadratic_reproduction_interior_cells(params_text):
    """Tables sampled from products of per-axis quadratics are reproduced EXACTLY (to rounding) in
    cells whose two knots are both interior: P on [1,3]^2, pi^rc / T on [1,3]^2 x [2,8]
    (central differences are exact for quadratics).  A forward-difference slope rule
    or a wrong end slope is caught, because the cells [1,2] and [2,3] read the slopes at 1 and 3,
    whose central differences reach the end knots 0 and 4."""
    P = [q1(a) * q2(b) for a in range(5) for b in range(5)]
    RT = [q1(a) * q2(b) * q3(c) for a in range(5) for b in range(5) for c in range(1, 10)]
    txt = set_table(params_text, "P.CC", P, 5)
    txt = set_table(txt, "R.CH", RT, 9)
    txt = set_table(txt, "T.HH", RT, 9)
    rng = np.random.default_rng(11)
    for _ in range(60):
        a, b = rng.uniform(1.0, 3.0, 2)
        c = rng.uniform(2.0, 8.0)
        exact2 = q1(a) * q2(b)
        o = O.spline(1, 0, a, b, params=txt)  # P_CC
        assert abs(o[0] - exact2) < 1e-13, (a, b, o[0], exact2)
        # the gradient of the reproduced polynomial is exact too
        assert abs(o[1] - (-0.7 + 0.9 * a) * q2(b)) < 1e-12
        assert abs(o[2] - q1(a) * (0.2 - 0.7 * b)) < 1e-12
        exact3 = exact2 * q3(c)
        for which, pair in ((2, 1), (3, 2)):  # R.CH, T.HH
            o = O.spline(which, pair, a, b, c, params=txt)
            assert abs(o[0] - exact3) < 1e-13, (which, a, b, c)
            assert abs(o[3] - exact2 * (0.13 + 0.042 * c)) < 1e-12


def test_quadratic_not_reproduced_in_boundary_cells(params_text):
    """Sanity of the pin above: with m = 0 at the end knots a quadratic with non-zero end slope is
    NOT reproduced in the boundary cells, so the interior-cell pin really tests the slope rule."""
    P = [q1(a) * q2(b) for a in range(5) for b in range(5)]
    txt = set_table(params_text, "P.CC", P, 5)
    assert abs(O.spline(1, 0, 0.5, 2.0, params=txt)[0] - q1(0.5) * q2(2.0)) > 1e-3


# ------------------------------------------------------------------ (b) every cell vs scipy
@pytest.mark.parametrize("seed", [0, 1])
def test_tensor_splines_all_cells_vs_scipy(params_text, seed):
    """Random tables; points in every cell including the boundary cells [0,1], [3,4] (P, N) and
    [1,2], [8,9] (N^conj), plus clamped points outside the grid, against the independent scipy
    tensor product.  Values at 1e-13; gradients against FD of the scipy tensor product."""
    rng = np.random.default_rng(100 + seed)
    P = rng.normal(size=25)
    R = rng.normal(size=225)
    T = rng.normal(size=225)
    txt = set_table(params_text, "P.CH", P, 5)
    txt = set_table(txt, "R.CC", R, 9)
    txt = set_table(txt, "T.CH", T, 9)
    pts2 = [(ia + rng.uniform(0.05, 0.95), ib + rng.uniform(0.05, 0.95)) for ia in range(4) for ib in range(4)]
    pts2 += [(-0.4, 2.3), (4.6, 0.2), (1.7, 5.5)]
    for a, b in pts2:
        o = O.spline(1, 1, a, b, params=txt)  # P_CH (centre C, t_j = H)
        ref = tensor_2d(P, a, b)
        assert abs(o[0] - ref) < 1e-13, (a, b)
        h = 1e-6
        if 0 < a < 4 and 0 < b < 4:
            fdx = (tensor_2d(P, a + h, b) - tensor_2d(P, a - h, b)) / (2 * h)
            fdy = (tensor_2d(P, a, b + h) - tensor_2d(P, a, b - h)) / (2 * h)
            assert abs(o[1] - fdx) < 1e-7 and abs(o[2] - fdy) < 1e-7
    cells_z = [1, 2, 5, 8]  # z cells [1,2], [2,3], [5,6], [8,9]
    for ia, ib, iz in itertools.product(range(4), range(4), cells_z):
        a, b = ia + rng.uniform(0.05, 0.95), ib + rng.uniform(0.05, 0.95)
        c = iz + rng.uniform(0.05, 0.95)
        for which, tab in ((2, R), (3, T)):
            pair = 0 if which == 2 else 1
            o = O.spline(which, pair, a, b, c, params=txt)
            ref = tensor_3d(tab, a, b, c)
            assert abs(o[0] - ref) < 1e-13, (which, a, b, c)
    # gradients in the corner cells (end-knot slopes matter most there)
    h = 1e-6
    for a, b, c in ((0.3, 0.6, 1.4), (3.7, 3.2, 8.8), (0.2, 3.9, 8.1)):
        o = O.spline(2, 0, a, b, c, params=txt)
        for ax in range(3):
            p, m = [a, b, c], [a, b, c]
            p[ax] += h
            m[ax] -= h
            fd = (tensor_3d(R, *p) - tensor_3d(R, *m)) / (2 * h)
            assert abs(o[1 + ax] - fd) < 1e-7, (a, b, c, ax)
    # outside the grid: clamped value, zero derivative along the clamped axis
    o = O.spline(2, 0, -0.5, 2.5, 9.7, params=txt)
    assert abs(o[0] - tensor_3d(R, 0.0, 2.5, 9.0)) < 1e-13 and o[1] == 0.0 and o[3] == 0.0


# ------------------------------------------------------------------ N^C, N^H, N^conj re-summation
PAIR = {(0, 0): "CC", (0, 1): "CH", (1, 0): "CH", (1, 1): "HH"}


def short_list_bruteforce(types, x, box):
    """All (i, j, s) with r <= r_max(t_i, t_j), all pairs x all images (|s| <= 1 suffices for the
    boxes used here, checked), with the switch weight w = S(r; r_min, r_max)."""
    n = len(types)
    nb = [[] for _ in range(n)]
    rng = range(-1, 2)
    for i in range(n):
        for j in range(n):
            for s in itertools.product(rng, rng, rng):
                if i == j and s == (0, 0, 0):
                    continue
                d = x[j] + np.array(s) * box - x[i]
                r = math.sqrt(float(d @ d))
                p = PAIR[(types[i], types[j])]
                rmin, rmax = CF.p1(f"pair.{p}.rmin"), CF.p1(f"pair.{p}.rmax")
                if r <= rmax:
                    assert r < min(box) - rmax  # one image layer is enough
                    nb[i].append((j, s, CF.S(r, rmin, rmax)))
    return nb


def resum(types, x, box):
    """Per half bond (i, j, s) -> (N_ij, N_ji, N^conj_ij), summed from the definitions."""
    nb = short_list_bruteforce(types, x, box)
    NC = np.array([sum(w for k, _, w in nb[i] if types[k] == 0) for i in range(len(types))])
    NH = np.array([sum(w for k, _, w in nb[i] if types[k] == 1) for i in range(len(types))])
    Ntot = NC + NH
    lo, hi = CF.p1("conj.lo"), CF.p1("conj.hi")
    out = {}
    for i in range(len(types)):
        for j, s, wij in nb[i]:
            if not (i < j or (i == j and s > (0, 0, 0))):
                continue
            neg = tuple(-q for q in s)
            # N^C_ij = N^C_i - [t_j = C] w_ij ; N^H_ij likewise (O4)
            nij = (NC[i] - (wij if types[j] == 0 else 0.0)) + (NH[i] - (wij if types[j] == 1 else 0.0))
            nji = (NC[j] - (wij if types[i] == 0 else 0.0)) + (NH[j] - (wij if types[i] == 1 else 0.0))
            # N^conj (O5 step 4): C neighbours of i other than (j, s), and of j other than (i, -s)
            si = sum(w * CF.S(Ntot[k] - w, lo, hi) for k, sk, w in nb[i] if types[k] == 0 and (k, sk) != (j, s))
            sj = sum(w * CF.S(Ntot[l] - w, lo, hi) for l, sl, w in nb[j] if types[l] == 0 and (l, sl) != (i, neg))
            out[(i, j) + tuple(s)] = (nij, nji, 1.0 + si * si + sj * sj)
    return out


def branched_carbon():
    """j - i - k with k carrying two more carbons (a, b): N_k = 3 on the plateau, so the
    N^conj term of bond (i, j) needs F(N_k - w_ik) = F(2) = 1, not F(N_k) = F(3) = 0.  Another
    carbon m hangs off a at a fractional weight (r in the C-C switching window)."""
    t = math.radians(112.0)
    d = 1.52
    x = [[0.0, 0.0, 0.0],  # i
         [-d, 0.0, 0.0],  # j
         [d * -math.cos(t), d * math.sin(t), 0.0]]  # k
    k = np.array(x[2])
    x.append((k + [1.45, 0.35, 0.3]).tolist())  # a
    x.append((k + [-0.4, 0.9, 1.1]).tolist())  # b
    a = np.array(x[3])
    x.append((a + [0.9, 1.4, -0.6]).tolist())  # m: |d| ~ 1.77 -> fractional w_am
    x.append([-d - 0.6, -0.9, 0.4])  # H on j
    x = np.array(x)
    return np.array([0, 0, 0, 0, 0, 0, 1], dtype=np.int32), x - x.mean(0) + 20.0, np.array([40.0, 40.0, 40.0])


def check_resum(types, x, box):
    rows = O.get_list(types, x, box, 1)
    B, _ = O.stages(types, x, box, lj=False)
    ref = resum(types, x, box)
    assert len(ref) == len(rows) > 0
    for r, b in zip(rows, B):
        nij, nji, nconj = ref[tuple(int(v) for v in r)]
        assert abs(b[5] - nij) < 1e-12 and abs(b[6] - nji) < 1e-12 and abs(b[7] - nconj) < 1e-12, (r, b[5:8])
    return rows, B, ref


def test_nconj_branched_carbon_separates_exclusion():
    types, x, box = branched_carbon()
    rows, B, ref = check_resum(types, x, box)
    # bond (0, 1): F(N_k - w_ik) = F(2) = 1 for k = 2, so N^conj >= 2; without the exclusion it
    # would be F(3) = 0 and N^conj = 1 (+ j's side)
    q = next(n for n, r in enumerate(rows) if (r[0], r[1]) == (0, 1))
    assert B[q, 7] > 1.9
    # and the fractional m makes at least one N^conj non-integer
    assert any(abs(v[2] - round(v[2])) > 1e-3 for v in ref.values())


@pytest.mark.parametrize("seed", [0, 2, 5])
def test_nconj_resummation_random_clusters(seed):
    s = I.random_cluster(30, seed, spread=5.0, dmin=1.0)
    _, B, ref = check_resum(s.types, s.x, s.box)
    # fractional coordinations present: the F(N - w) arguments sit inside the (2, 3) window
    assert any(abs(v[0] - round(v[0])) > 1e-3 for v in ref.values())


def test_nconj_resummation_periodic_multi_image():
    """cfg1-type PE cell 1x1x2 with jitter: a chain meets its own periodic image along c."""
    s = I.polyethylene((1, 1, 2), 0.05, 7, None)
    check_resum(s.types, s.x, s.box)


# ------------------------------------------------------------------ list digests (full-size list parity)
def test_oracle_list_digest_matches_rows():
    """oracle.compute_digest's three digests equal the numpy digest of oracle.get_list's rows, and
    its forces / energies / counters are those of oracle.compute (same list build)."""
    from tests.digest import digest
    for s in (I.config(1), I.random_cluster(30, 1, spread=5.0, dmin=1.0), I.diamond((1, 1, 1), 0.05, 9)):
        d = O.compute_digest(s.types, s.x, s.box)
        for which in range(3):
            assert d["digest"][which] == digest(O.get_list(s.types, s.x, s.box, which)), (s.name, which)
        o = O.compute(s.types, s.x, s.box)
        assert d["E"] == o["E"] and np.array_equal(d["F"], o["F"]) and d["counters"] == o["counters"]
    # the digest separates sets that differ in one image shift or one index
    r = O.get_list(I.config(1).types, I.config(1).x, I.config(1).box, 2)
    r2 = r.copy()
    r2[5, 4] += 1
    r3 = r.copy()
    r3[7, 1] += 1
    assert digest(r) != digest(r2) and digest(r) != digest(r3)
