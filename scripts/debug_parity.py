"""Ad-hoc GPU-vs-oracle diagnostics (prints per-system force/energy deviations)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402


def cmp(s, prec="fp64"):
    o = O.compute(s.types, s.x, s.box)
    e = E.make(s, prec)
    g = e.compute()
    dF = np.abs(g["F"] - o["F"]).max()
    no, ng = np.linalg.norm(o["F"], axis=1), np.linalg.norm(g["F"], axis=1)
    print(f"{s.name:28s} n={s.n:6d} dE/E={abs(g['E'] - o['E']) / max(abs(o['E']), 1e-30):.2e} "
          f"dF={dF:.3e} sorted|F| diff={np.abs(np.sort(no) - np.sort(ng)).max():.3e} "
          f"dW={np.abs(g['W'] - o['W']).max():.2e} sumF={np.abs(g['F'].sum(0)).max():.2e}")
    bad = np.argsort(-np.abs(g["F"] - o["F"]).max(1))[:3]
    for a in bad:
        print("   atom", a, "type", s.types[a], "gpu", g["F"][a], "orc", o["F"][a])
    st = e.stats()
    print("   stats", {k: st[k] for k in ("n_lj", "n_C0", "n_bstar", "n_bonds", "n_ghosts", "n_rebuilds")},
          "orc", {k: o["counters"][k] for k in ("n_lj", "n_C0", "n_bstar", "n_bonds")})


if __name__ == "__main__":
    box = np.array([30.0, 30, 30])
    cmp(I.System("dimer-CC-1.4", np.array([0, 0]), np.array([[10.0, 10, 10], [11.4, 10.1, 10.2]]), box))
    cmp(I.System("dimer-CC-3.5", np.array([0, 0]), np.array([[10.0, 10, 10], [13.4, 10.5, 10.2]]), box))
    cmp(I.System("dimer-CC-6", np.array([0, 0]), np.array([[10.0, 10, 10], [15.4, 11.5, 10.2]]), box))
    cmp(I.System("dimer-wrap", np.array([0, 1]), np.array([[0.5, 10, 10], [25.4, 11.5, 10.2]]), box))
    t = np.radians(112)
    cmp(I.System("trimer", np.array([0, 0, 0]),
                 np.array([[10.0, 10, 10], [11.4, 10, 10], [10 + 1.4 * np.cos(t), 10 + 1.4 * np.sin(t), 10]]), box))
    for seed in range(2):
        cmp(I.random_cluster(10, seed, spread=4.0, dmin=1.0))
    cmp(I.diamond((2, 2, 2), 0.04, 21))
    cmp(I.config(1))
