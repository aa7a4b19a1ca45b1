"""Build kernel variants of libairebo_b200.so with extra -D flags (A/B experiments; not shipped):
python scripts/build_variants.py name=-DFOO=1,-DBAR=2 other=-DFOO=0 ...  ->  build_variants/<name>/"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1810_07026_b200 import build as B  # noqa: E402


def one(spec):
    name, flags = spec.split("=", 1)
    out = os.path.join(ROOT, "build_variants", name)
    os.makedirs(out, exist_ok=True)
    cmd = ["/usr/local/cuda/bin/nvcc"] + B.NVCC_FLAGS + [f for f in flags.split(",") if f] + \
        [os.path.join(B.CSRC, s) for s in B.SOURCES] + ["-o", os.path.join(out, "libairebo_b200.so")]
    r = subprocess.run(cmd, cwd=B.CSRC, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-2000:]


with ThreadPoolExecutor(max_workers=7) as ex:
    for name, rc, err in ex.map(one, sys.argv[1:]):
        print(name, "ok" if rc == 0 else "FAILED\n" + err)
