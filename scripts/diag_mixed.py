"""Diagnostic: where does the mixed-precision force error of a config concentrate?  Compares
mixed vs fp64 GPU forces per atom and prints the worst atoms with their short-list neighbours."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_07026_b200 import engine as E  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

s = I.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
g = E.make(s, "fp64").compute()
m = E.make(s, "mixed").compute()
d = np.sqrt(((m["F"] - g["F"]) ** 2).sum(1))
rel = np.sqrt((d ** 2).sum()) / np.sqrt((g["F"] ** 2).sum())
print("rel RMS", rel, "E rel", abs(m["E"] - g["E"]) / abs(g["E"]), "terms", g["terms"], m["terms"])
short = E.make(s, "fp64").get_list(0)
order = np.argsort(-d)[:12]
for a in order:
    nb = short[short[:, 0] == a]
    dist = [np.linalg.norm(s.x[j] + np.array(sh) * s.box - s.x[a]) for j, *sh in nb[:, 1:]]
    print(a, "type", s.types[a], "|dF|", d[a], "|F|", np.linalg.norm(g["F"][a]), "nbrs", list(zip(nb[:, 1].tolist(), np.round(dist, 4).tolist())))
# pair-type breakdown: fp64 vs mixed with LJ / REBO only via potential variants
pt = open(E.PARAMS, "rb").read()
for name in ("rebo",):
    p = pt.replace(b"potential airebo\n", b"potential rebo\n")
    gg = E.Engine("fp64", params=p); gg.set_box(s.box); gg.set_atoms(s.types, s.x); a = gg.compute()
    mm = E.Engine("mixed", params=p); mm.set_box(s.box); mm.set_atoms(s.types, s.x); b = mm.compute()
    print(name, "rel RMS", np.sqrt(((a["F"] - b["F"]) ** 2).sum()) / np.sqrt((a["F"] ** 2).sum()))
