"""GPU: the NCCL branch of the engine (ab_create_dist) with two and three ranks as threads of one
process on one GPU, through the test-only fake NCCL library (tests/fake_nccl/fake_nccl.cpp: host
rendezvous + device copies; no kernel waits on another rank).  Forces, energies, virial, the NVE
trajectory with thermo rows and the set_positions redistribution must match the whole-box engine
(fp64 tolerances of BASELINE.json north_star; the trajectory differs only by summation order)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.join(ROOT, "tests", "fake_nccl")


@pytest.fixture(scope="module")
def fake_lib():
    from paper_1810_07026_b200 import build
    build.build()
    lib = os.path.join(HERE, "libfake_nccl.so")
    subprocess.run(["g++", "-std=c++17", "-O1", "-shared", "-fPIC", os.path.join(HERE, "fake_nccl.cpp"),
                    "-I/usr/local/cuda/include", "-L/usr/local/cuda/lib64/stubs", "-lcuda", "-o", lib], check=True)
    return lib


@pytest.mark.parametrize("name,nr", [("cluster", 2), ("3", 2), ("3", 3)])
def test_nccl_branch_matches_whole_box(fake_lib, name, nr):
    env = dict(os.environ, AB_NCCL_LIB=fake_lib)
    p = subprocess.run([sys.executable, os.path.join(HERE, "run_dist.py"), name, str(nr)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    for r in range(nr):
        o = res[f"r{r}"]
        assert o["dF0"] <= 1e-9 and o["dE0"] <= 1e-11, o
        # dF1 compares frames that differ by the trajectories' roundoff (chaotic at 1500 K):
        # reported only; dF2 is at identical positions (after ab_set_positions on both)
        assert o["dF2"] <= 1e-9 and o["dE2"] <= 1e-11, o
        assert o["dx"] <= 1e-9 and o["dv"] <= 1e-9 and o["dth"] <= 1e-7, o
        assert o["n_atoms"] == res["n"]
