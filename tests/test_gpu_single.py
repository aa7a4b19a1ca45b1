"""AB_SINGLE, the paper's "single" precision mode (reading A32):
AB_MIXED with every accumulation in fp32.  Checked against the fp64 oracle at a tolerance derived
from fp32 summation (a per-atom force is a sum of ~10^3 terms of total magnitude
sum|t| ~ 10^2 eV/A, fp32 summation error ~ sqrt(n) u sum|t| ~ 2e-4 eV/A against RMS forces of a few
eV/A: relative RMS <= 1e-3; energies are per-thread fp32 sums of ~10 terms, |dE| <= 1e-5 |E|),
and against AB_MIXED: same lists and gates, and a force array that really is fp32 (every
component a binary32 value) and differs from the fp64-accumulated one."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1810_07026_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng_mod():
    from paper_1810_07026_b200 import build, engine
    build.build()
    return engine


def systems():
    return [I.config(1), I.config(2), I.nanotube(10, 10, 6, jitter=0.02, seed_x=7, seed_v=8, name="cnt-10-10-x6"),
            I.random_cluster(60, 11, spread=7.0, dmin=0.95, frac_c=0.4, name="cluster-big")]


@pytest.mark.parametrize("idx", range(4))
def test_single_parity(eng_mod, idx):
    s = systems()[idx]
    o = O.compute(s.types, s.x, s.box)
    es = eng_mod.make(s, "single")
    g = es.compute()
    rel = np.sqrt(((g["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-3, (s.name, rel)
    assert abs(g["E"] - o["E"]) <= 1e-5 * abs(o["E"]), (s.name, g["E"], o["E"])
    # the force array is the fp32 sum: every component is a binary32 value
    F = g["F"]
    assert np.array_equal(F.astype(np.float32).astype(np.float64), F), s.name
    # same lists and integer counters as the mixed mode (only the accumulation differs)
    em = eng_mod.make(s, "mixed")
    m = em.compute()
    for which in (0, 1, 2):
        assert np.array_equal(es.get_list(which), em.get_list(which)), (s.name, which)
    for k in ("n_short", "n_bonds", "n_lj", "n_C0", "n_bstar"):
        assert es.stats()[k] == em.stats()[k], (s.name, k)
    if s.n > 200:  # large enough that fp32 accumulation must show
        assert not np.array_equal(m["F"], F), s.name
    es.close()
    em.close()


def test_single_nve_runs_and_tracks_mixed(eng_mod):
    s = I.nanotube(10, 10, 6, jitter=0.01, seed_x=41, seed_v=42, T=300.0, name="cnt")
    th = {}
    for prec in ("mixed", "single"):
        e = eng_mod.make(s, prec)
        th[prec] = e.run_nve(200, 0.25, every=50)
        e.close()
    assert np.all(np.isfinite(th["single"]))
    # a 50 fs run: the two trajectories agree to fp32 noise in the total energy
    assert np.abs(th["single"][:, 3] - th["mixed"][:, 3]).max() <= 1e-4 * abs(th["mixed"][0, 3])


def test_reduced_state_is_binary32(eng_mod):
    """AB_REDUCED (reading A35): after NVE steps (deferred and thermo kicks, with a rebuild) every
    position and velocity component is a binary32 value; a single evaluation is AB_SINGLE's (same
    kernels, same tolerance against the oracle at the state it produced)."""
    s = I.config(1)
    e = eng_mod.make(s, "reduced")
    e.run_nve(7, 0.5)
    e.run_nve(5, 0.5, every=5)
    x, v = e.get_positions(), e.get_velocities()
    # wrapping at a rebuild (x - L floor(x/L)) may leave a non-binary32 value only until the next drift
    e.run_nve(1, 0.5)
    x, v = e.get_positions(), e.get_velocities()
    assert np.array_equal(v.astype(np.float32).astype(np.float64), v)
    xs = x[(x > 0.5) & (x < s.box - 0.5)]  # away from the wrap boundary
    assert np.array_equal(xs.astype(np.float32).astype(np.float64), xs)
    g = e.compute()
    o = O.compute(s.types, x, s.box)
    rel = np.sqrt(((g["F"] - o["F"]) ** 2).sum()) / np.sqrt((o["F"] ** 2).sum())
    assert rel <= 1e-3 and abs(g["E"] - o["E"]) <= 1e-5 * abs(o["E"])
    # and it differs from AB_SINGLE's fp64-state trajectory
    es = eng_mod.make(s, "single")
    es.run_nve(13, 0.5)
    assert not np.array_equal(es.get_positions(), x)
