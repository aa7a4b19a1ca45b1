"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no AIREBO terms, no forces): it only builds
geometries, species, wrapped coordinates and Maxwell velocities, exactly as SURVEY.md
§8(d) / Appendix B specify.  Both sides (oracle/ and the CUDA engine) receive the same bits.

Readings:
  * PE unit cell: SURVEY A21 / Appendix B (a=7.42, b=4.95, c=2.54 A, 12 atoms, chains at (0,0)
    and (a/2,b/2), setting angles +45/-45 deg, C-C 1.53, C-H 1.09, H-C-H 109.47 deg).
  * cfg 1 = cell x (1,1,10) = 120 atoms.
  * Maxwell velocities: SURVEY A23 (seeded PCG64, COM removed, rescaled to exactly T, 3N-3 dof).
  * wrap: y = x - L floor(x/L); y >= L -> y -= L; y < 0 -> y += L.
  * cfg 3 amorphous: random sequential insertion (d_min = 1.0 A); the 200-step relaxation
    of BASELINE cfg 3 is NOT applied (reading A22' in DESIGN.md).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import hashlib
import os

import numpy as np

# unit constants, same values as params/toy_ch.param; used only to draw velocities
KB = 8.617333262e-5  # eV/K
MVV2E = 103.6426965  # eV per amu A^2/fs^2
MASS = np.array([12.011, 1.008])  # C, H (amu)

C, H = 0, 1


@dataclass
class System:
    name: str
    types: np.ndarray  # int32 [N], 0 = C, 1 = H
    x: np.ndarray  # float64 [N,3], wrapped into [0, L)
    box: np.ndarray  # float64 [3]
    v: np.ndarray | None = None  # float64 [N,3], A/fs
    dt: float = 0.5  # fs
    steps: int = 100

    @property
    def n(self) -> int:
        return int(self.types.shape[0])


def wrap(x: np.ndarray, box: np.ndarray) -> np.ndarray:
    """SURVEY O1 wrap, elementwise, float64."""
    x = np.asarray(x, dtype=np.float64)
    L = np.asarray(box, dtype=np.float64)
    y = x - L * np.floor(x / L)
    y = np.where(y >= L, y - L, y)
    y = np.where(y < 0.0, y + L, y)
    return y


# ---------------------------------------------------------------- polyethylene
PE_A, PE_B, PE_C = 7.42, 4.95, 2.54


def pe_cell() -> tuple[np.ndarray, np.ndarray]:
    """12-atom orthorhombic PE cell. Returns (types[12], xyz[12,3])."""
    half_ang = math.radians(109.47 / 2.0)  # H-C-H half angle (54.735 deg)
    dc = 0.42661  # carbon offset from the chain axis along the zigzag direction
    types, pos = [], []
    for (x0, y0), psi in (((0.0, 0.0), math.radians(45.0)), ((PE_A / 2, PE_B / 2), math.radians(-45.0))):
        u = np.array([math.cos(psi), math.sin(psi), 0.0])
        v = np.array([-math.sin(psi), math.cos(psi), 0.0])  # ab-plane, perpendicular to u
        for z, s in ((0.0, 1.0), (PE_C / 2, -1.0)):
            c = np.array([x0, y0, z]) + s * dc * u
            types.append(C)
            pos.append(c)
            for sign in (1.0, -1.0):
                types.append(H)
                pos.append(c + 1.09 * (s * u * math.cos(half_ang) + sign * v * math.sin(half_ang)))
    return np.array(types, dtype=np.int32), np.array(pos, dtype=np.float64)


def replicate(types, xyz, cell, reps):
    """Cell-major replication: ix slowest, then iy, iz, then basis index."""
    nx, ny, nz = reps
    ii = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    shifts = ii.astype(np.float64) * np.asarray(cell, dtype=np.float64)
    allx = (shifts[:, None, :] + xyz[None, :, :]).reshape(-1, 3)
    allt = np.tile(types, ii.shape[0])
    box = np.asarray(cell, dtype=np.float64) * np.array(reps, dtype=np.float64)
    return allt.astype(np.int32), allx, box


def maxwell(types: np.ndarray, T: float, seed: int) -> np.ndarray:
    """v = sqrt(kB T/(m mvv2e)) N(0,1); remove mass-weighted COM; rescale to T exactly."""
    rng = np.random.default_rng(seed)
    n = types.shape[0]
    m = MASS[types]
    v = rng.standard_normal((n, 3)) * np.sqrt(KB * T / (m * MVV2E))[:, None]
    p = (m[:, None] * v).sum(0) / m.sum()
    v = v - p[None, :]
    if n > 1 and T > 0:
        ke = 0.5 * (m[:, None] * v * v).sum() * MVV2E
        t_now = 2.0 * ke / ((3 * n - 3) * KB)
        v = v * math.sqrt(T / t_now)
    return v


def polyethylene(reps, jitter, seed_x, seed_v, T=300.0, name="pe") -> System:
    t, x = pe_cell()
    types, xyz, box = replicate(t, x, (PE_A, PE_B, PE_C), reps)
    rng = np.random.default_rng(seed_x)
    xyz = xyz + rng.uniform(-jitter, jitter, xyz.shape)
    xyz = wrap(xyz, box)
    v = maxwell(types, T, seed_v) if seed_v is not None else None
    return System(name, types, xyz, box, v)


# ---------------------------------------------------------------- diamond
DIAMOND_A = 3.567


def diamond(reps, jitter=0.0, seed_x=None, seed_v=None, T=1000.0, a=DIAMOND_A, name="diamond") -> System:
    fcc = np.array([[0, 0, 0], [0, 0.5, 0.5], [0.5, 0, 0.5], [0.5, 0.5, 0]], dtype=np.float64)
    basis = np.concatenate([fcc, fcc + 0.25]) * a
    types, xyz, box = replicate(np.zeros(8, dtype=np.int32), basis, (a, a, a), reps)
    if jitter > 0:
        rng = np.random.default_rng(seed_x)
        xyz = xyz + rng.uniform(-jitter, jitter, xyz.shape)
    xyz = wrap(xyz, box)
    v = maxwell(types, T, seed_v) if seed_v is not None else None
    return System(name, types, xyz, box, v)


# ---------------------------------------------------------------- carbon nanotube
def nanotube(n, m, reps, bond=1.42, vacuum=12.0, jitter=0.0, seed_x=None, seed_v=None, T=300.0,
             name=None) -> System:
    """All-carbon (n, m) single-wall nanotube along z, periodic in z (reps translational unit
    cells), isolated in x/y by `vacuum` A of empty space.  The paper's second workload is a custom
    CNT ("contains no hydrogen, and stresses all the dihedral terms"; its geometry is
    not in the container), so it is generated here: the graphene sheet (C-C distance `bond`) is
    rolled along the chiral vector C_h = n a1 + m a2 with the translation vector
    T = ((2m+n) a1 - (2n+m) a2) / gcd(2m+n, 2n+m).  Geometry only; no method arithmetic."""
    if n < 1 or m < 0 or m > n:
        raise ValueError("need n >= 1, 0 <= m <= n")
    a = bond * math.sqrt(3.0)
    a1 = np.array([a, 0.0])
    a2 = np.array([a / 2.0, a * math.sqrt(3.0) / 2.0])
    ch = n * a1 + m * a2
    dr = math.gcd(2 * m + n, 2 * n + m)
    t1, t2 = (2 * m + n) // dr, -(2 * n + m) // dr
    tv = t1 * a1 + t2 * a2
    lc, lt = float(np.linalg.norm(ch)), float(np.linalg.norm(tv))
    nhex = 2 * (n * n + n * m + m * m) // dr  # hexagons (2 atoms each) per translational cell
    basis = [np.zeros(2), (a1 + a2) / 3.0]  # the two graphene sublattices
    pts = []
    rng_i = range(-abs(t1) - n - abs(t2) - m - 2, abs(t1) + n + abs(t2) + m + 3)
    for i in rng_i:
        for j in rng_i:
            for b in basis:
                p = i * a1 + j * a2 + b
                u, w = float(p @ ch) / lc ** 2, float(p @ tv) / lt ** 2  # fractional coordinates
                if -1e-9 <= u < 1 - 1e-9 and -1e-9 <= w < 1 - 1e-9:
                    pts.append((u, w))
    if len(pts) != 2 * nhex:
        raise RuntimeError(f"nanotube({n},{m}): {len(pts)} sites, expected {2 * nhex}")
    radius = lc / (2.0 * math.pi)
    side = 2.0 * radius + 2.0 * vacuum
    box = np.array([side, side, lt * reps])
    xyz = []
    for k in range(reps):
        for u, w in pts:
            ph = 2.0 * math.pi * u
            xyz.append((side / 2 + radius * math.cos(ph), side / 2 + radius * math.sin(ph), (w + k) * lt))
    xyz = np.array(xyz)
    types = np.zeros(len(xyz), dtype=np.int32)
    if jitter > 0:
        xyz = xyz + np.random.default_rng(seed_x).uniform(-jitter, jitter, xyz.shape)
    xyz = wrap(xyz, box)
    v = maxwell(types, T, seed_v) if seed_v is not None else None
    return System(name or f"cnt-{n}-{m}-x{reps}", types, xyz, box, v)


# ---------------------------------------------------------------- amorphous CH2
def random_insertion(n, box, dmin, seed):
    """Random sequential insertion, uniform in the periodic box, reject if any distance < dmin."""
    rng = np.random.default_rng(seed)
    box = np.asarray(box, dtype=np.float64)
    ncell = np.maximum(1, np.floor(box / dmin).astype(int))
    csize = box / ncell
    cells: dict[tuple, list] = {}
    pts = np.empty((n, 3))
    k = 0
    d2 = dmin * dmin
    while k < n:
        p = rng.random(3) * box
        c = tuple((p // csize).astype(int) % ncell)
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    cc = ((c[0] + dx) % ncell[0], (c[1] + dy) % ncell[1], (c[2] + dz) % ncell[2])
                    for q in cells.get(cc, ()):
                        d = pts[q] - p
                        d -= box * np.round(d / box)
                        if d @ d < d2:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if not ok:
                break
        if ok:
            pts[k] = p
            cells.setdefault(c, []).append(k)
            k += 1
    return pts


RELAXED_CFG3 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "cfg3_relaxed.npz")


def amorphous(n_c=21334, n_h=42668, L=82.038, dmin=1.0, seed_x=103, seed_t=303, seed_v=203, T=1500.0,
              name="a-CH2", relaxed=False) -> System:
    """Random sequential insertion (SURVEY §8(d) cfg 3).  relaxed=True: positions from the frozen
    file written by scripts/relax_cfg3.py (200 capped steepest-descent iterations with oracle
    forces, SURVEY reading A22), checked against its SHA-256."""
    n = n_c + n_h
    box = np.array([L, L, L])
    types = np.full(n, H, dtype=np.int32)
    types[np.random.default_rng(seed_t).permutation(n)[:n_c]] = C
    if relaxed:
        f = np.load(RELAXED_CFG3)
        xyz = np.ascontiguousarray(f["x"], dtype=np.float64)
        if hashlib.sha256(xyz.tobytes()).hexdigest() != str(f["sha256"]) or not np.array_equal(f["types"], types):
            raise RuntimeError(f"{RELAXED_CFG3}: checksum / species mismatch")
    else:
        xyz = wrap(random_insertion(n, box, dmin, seed_x), box)
    v = maxwell(types, T, seed_v) if seed_v is not None else None
    return System(name, types, xyz, box, v, dt=0.25)


def random_cluster(n, seed, box_len=40.0, spread=6.0, dmin=0.9, frac_c=0.5, name="cluster") -> System:
    """Small random C/H cluster near the centre of a large box (non-periodic in effect)."""
    box = np.array([box_len] * 3)
    rng = np.random.default_rng(seed)
    pts = []
    while len(pts) < n:
        p = rng.uniform(-spread / 2, spread / 2, 3) + box / 2
        if all(np.linalg.norm(p - q) >= dmin for q in pts):
            pts.append(p)
    types = (rng.random(n) >= frac_c).astype(np.int32)
    return System(name, types, wrap(np.array(pts), box), box)


# ---------------------------------------------------------------- BASELINE.json configs
def config(idx: int, n_rep: int = 1) -> System:
    """BASELINE.json configs: 1 tiny PE, 2 PE 32k, 3 a-CH2 64k, 4 PE 1M,
    '5a' diamond 2M x n_rep, '5b' PE 2M x n_rep."""
    if idx == 1:
        s = polyethylene((1, 1, 10), 0.05, 101, 201, name="cfg1-pe-120")
    elif idx == 2:
        s = polyethylene((12, 16, 14), 0.02, 102, 202, name="cfg2-pe-32k")
    elif idx == 3:
        s = amorphous(name="cfg3-aCH2-64k", relaxed=True)  # SURVEY reading A22 (scripts/relax_cfg3.py)
        s.steps = 100
        return s
    elif idx == 4:
        s = polyethylene((40, 50, 42), 0.02, 104, 204, name="cfg4-pe-1M")
    elif idx == "5a":
        s = diamond((63 * n_rep, 63, 63), 0.03, 105, 205, name=f"cfg5a-diamond-{n_rep}x2M")
        s.steps = 50
    elif idx == "5b":
        s = polyethylene((40 * n_rep, 50, 84), 0.02, 106, 206, name=f"cfg5b-pe-{n_rep}x2M")
        s.steps = 50
    else:
        raise ValueError(idx)
    return s
