"""Independent closed forms and brute-force references used to PIN the oracle (not the oracle).

Nothing here is imported by oracle/ or by the CUDA package.  Each function evaluates a special
case of the paper's definitions that reduces to something checkable by eye (a dimer, a trimer,
the perfect diamond lattice with its knot-valued splines), or a brute-force enumeration on a
tiny input (max-product path search for C_ij, all-quadruple torsion sum).
"""
from __future__ import annotations

import math
import os

import numpy as np
from scipy.interpolate import CubicHermiteSpline

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_params(path=os.path.join(ROOT, "params", "toy_ch.param")):
    """Minimal third parser (tests only): key -> list of floats (or strings)."""
    kv, last = {}, None
    for line in open(path):
        line = line.split("#", 1)[0].split()
        if not line:
            continue
        try:
            float(line[0])
            kv[last] += [float(v) for v in line]
            continue
        except ValueError:
            pass
        last = line[0]
        vals = []
        for v in line[1:]:
            try:
                vals.append(float(v))
            except ValueError:
                vals.append(v)
        kv[last] = vals
    return kv


KV = read_params()


def p1(key):
    return KV[key][0]


def S(x, lo, hi):
    """Half-cosine switch."""
    t = (x - lo) / (hi - lo)
    if t <= 0:
        return 1.0
    if t >= 1:
        return 0.0
    return 0.5 * (1 + math.cos(math.pi * t))


def g_spline(species: str):
    """g_i as a scipy CubicHermiteSpline with the knot-slope rule of SURVEY A7."""
    x = np.array(KV[f"angle.{species}.knots"])
    y = np.array(KV[f"angle.{species}.values"])
    m = np.zeros_like(y)
    m[1:-1] = (y[2:] - y[:-2]) / (x[2:] - x[:-2])
    return CubicHermiteSpline(x, y, m)


def fR(r, pair="CC"):
    w = S(r, p1(f"pair.{pair}.rmin"), p1(f"pair.{pair}.rmax"))
    return w * (1 + p1(f"pair.{pair}.Q") / r) * p1(f"pair.{pair}.A") * math.exp(-p1(f"pair.{pair}.alpha") * r)


def fA(r, pair="CC"):
    w = S(r, p1(f"pair.{pair}.rmin"), p1(f"pair.{pair}.rmax"))
    B, be = KV[f"pair.{pair}.B"], KV[f"pair.{pair}.beta"]
    return -w * sum(b * math.exp(-q * r) for b, q in zip(B, be))


def tab_P(pair, a, b):
    return KV[f"P.{pair}"][a * 5 + b]


def tab_RT(which, pair, x, y, z):
    return KV[f"{which}.{pair}"][(x * 5 + y) * 9 + (z - 1)]


def V_lj(r, pair="CC"):
    eps, sig = p1(f"lj.{pair}.eps"), p1(f"lj.{pair}.sigma")
    return 4 * eps * ((sig / r) ** 12 - (sig / r) ** 6) * S(r, p1(f"lj.{pair}.rlo"), p1(f"lj.{pair}.rc"))


def diamond_sites(a, rmax):
    """Lattice sites of perfect diamond within rmax of the origin atom (origin excluded)."""
    fcc = np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0]])
    basis = np.concatenate([fcc, fcc + 0.25])
    n = int(math.ceil(rmax / a)) + 1
    rng = np.arange(-n, n + 1)
    cells = np.stack(np.meshgrid(rng, rng, rng, indexing="ij"), -1).reshape(-1, 3)
    pts = (cells[:, None, :] + basis[None, :, :]).reshape(-1, 3) * a
    r = np.linalg.norm(pts, axis=1)
    keep = (r > 1e-9) & (r <= rmax)
    return pts[keep], r[keep]


def diamond_hops(a, pts, maxhops=3):
    """Bond-graph distance (BFS over nearest-neighbour bonds) from the origin, capped at maxhops+1."""
    d_nn = math.sqrt(3) * a / 4
    allp = np.concatenate([np.zeros((1, 3)), pts])
    D = np.linalg.norm(allp[:, None, :] - allp[None, :, :], axis=-1)
    adj = np.abs(D - d_nn) < 1e-6
    hops = np.full(len(allp), maxhops + 1)
    hops[0] = 0
    frontier = [0]
    for h in range(1, maxhops + 1):
        nxt = []
        for u in frontier:
            for v in np.nonzero(adj[u])[0]:
                if hops[v] > h:
                    hops[v] = h
                    nxt.append(v)
        frontier = nxt
    return hops[1:]


def diamond_energy_per_atom(a=3.567):
    """Closed form for the perfect diamond (SURVEY c-4): every bond on the w=1 plateau, all
    cos(theta) = -1/3 (a g_C knot), N_ij = 3, N^conj = 1 (F(3) = 0), sum_kl (1 - cos^2 w) = 4.5,
    E_TORS = 0, LJ only to sites more than 3 bonds away (C = 1), b* < b_min so Q = 1."""
    d = math.sqrt(3) * a / 4
    p = (1 + 3 * 0.1 + tab_P("CC", 3, 0)) ** -0.5
    b = p + tab_RT("R", "CC", 3, 3, 1) + 4.5 * tab_RT("T", "CC", 3, 3, 1)
    e_rebo = 2 * (fR(d) + b * fA(d))
    pts, r = diamond_sites(a, p1("lj.CC.rc"))
    hops = diamond_hops(a, pts)
    far = hops > 3
    e_lj = 0.5 * sum(V_lj(x) for x in r[far])
    return dict(p=p, b=b, rebo=e_rebo, lj=e_lj, E=e_rebo + e_lj, n_far=int(far.sum()))


def trimer_energy(theta_deg, r=1.4):
    """C3 'V' trimer i-j, i-k (plateau bonds, j-k unbonded): per bond b = 1/2(p_ij + 1) + R_CC(1,0,2)
    with p_ij = (1 + g_C(cos theta) + P_CC(1,0))^-1/2, N^conj = 1 + F(0)^2 = 2, pi^dh = 0."""
    c = math.cos(math.radians(theta_deg))
    g = float(g_spline("C")(c))
    pij = (1 + g + tab_P("CC", 1, 0)) ** -0.5
    b = 0.5 * (pij + 1.0) + tab_RT("R", "CC", 1, 0, 2)
    return 2 * (fR(r) + b * fA(r))


def maxprod_paths(W):
    """M_ij = max(W_ij, max_k W_ik W_kj, max_kl W_ik W_kl W_lj) by brute force (max-times products)."""
    M1 = W
    M2 = np.max(W[:, :, None] * W[None, :, :], axis=1)
    M3 = np.max(M2[:, :, None] * W[None, :, :], axis=1)
    return np.maximum(np.maximum(M1, M2), M3)
