"""Input preparation for BASELINE cfg 3 ("relaxed for 200 steps"), SURVEY reading A22: 200
iterations of capped steepest descent, x <- x + delta F / max_a |F_a| with delta = 0.05 A, on the
seeded random-insertion a-CH2 system, with forces from the fp64 ORACLE only (this script calls
oracle/ and the method-free input generator, nothing of the CUDA path).  The relaxed positions
are frozen in paper_1810_07026_b200/data/cfg3_relaxed.npz with their SHA-256; both the oracle
and the GPU then start from the file (inputs.config(3)).  Not under test: input preparation."""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1810_07026_b200 import inputs as I  # noqa: E402

OUT = os.path.join(ROOT, "paper_1810_07026_b200", "data", "cfg3_relaxed.npz")


def main(iters=200, delta=0.05, threads=os.cpu_count()):
    s = I.amorphous(relaxed=False)
    x = s.x.copy()
    t0 = time.time()
    for it in range(iters):
        r = O.compute(s.types, x, s.box, threads=threads)
        fn = np.sqrt((r["F"] ** 2).sum(1))
        x = I.wrap(x + delta * r["F"] / fn.max(), s.box)
        if it % 10 == 0 or it == iters - 1:
            print(f"iter {it:4d}  E {r['E']:.6f} eV  max|F| {fn.max():.4f} eV/A  ({time.time() - t0:.0f} s)", flush=True)
    sha = hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()
    np.savez_compressed(OUT, x=x, types=s.types, box=s.box, sha256=np.array(sha), iters=np.array(iters),
                        delta=np.array(delta))
    print("wrote", OUT, sha)


if __name__ == "__main__":
    main()
