"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports every symbol
that include/airebo_b200.h declares (no compute calls: there is no GPU here)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "airebo_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ab_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1810_07026_b200 import build, engine
    build.build()
    return engine.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_1810_07026_b200 import engine
    funcs = header_functions()
    assert len(funcs) >= 18
    missing = [f for f in funcs if not hasattr(lib, f)]
    assert not missing, missing
    assert set(funcs) == set(engine.EXPORTS)


def test_sass_is_sm100a(lib):
    from paper_1810_07026_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_create_fails_loudly(lib):
    """Without a Blackwell GPU the engine must refuse to run (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1810_07026_b200 import engine
    with pytest.raises(engine.ABError) as ei:
        engine.Engine("fp64")
    assert ei.value.status == -6


def test_param_errors_reported_by_library(lib, params_text):
    """ab_create parses the parameter text before touching the GPU: errors name key or line."""
    import ctypes as C
    h = C.c_void_p()
    bad = params_text.replace(b"pair.CH.rmin 1.3", b"pair.CH.rmin 1.9")
    rc = lib.ab_create(bad, len(bad), 0, 0, C.byref(h))
    assert rc == -2
    assert b"pair.CH.rmin" in lib.ab_last_error(None)
    bad = params_text.replace(b"tors.HCCH 0.12\n", b"")
    rc = lib.ab_create(bad, len(bad), 0, 0, C.byref(h))
    assert rc == -2 and b"tors.HCCH" in lib.ab_last_error(None)
    bad = b"1.0 2.0\n" + params_text
    rc = lib.ab_create(bad, len(bad), 0, 0, C.byref(h))
    assert rc == -2 and b"line 1" in lib.ab_last_error(None)


def test_slab_geometry_host_calls(lib):
    """ab_slab_info / ab_slab_of need no GPU: slabs tile [0, L_x), the owner of x is the slab that
    contains wrap(x), and a slab narrower than the halo is reported (AB_E_BOX)."""
    from paper_1810_07026_b200 import engine
    L = [89.04, 79.2, 35.56]
    for n in (1, 2, 3, 7):
        b = [engine.slab_info(L, 11.2, n, r) for r in range(n)]
        assert b[0][0] == 0.0 and b[-1][1] == L[0] and all(ok for _, _, ok in b)
        for r in range(n - 1):
            assert b[r][1] == b[r + 1][0]
        for x in np.linspace(-L[0], 2 * L[0], 301):
            r = engine.slab_of(x, L[0], n)
            xw = x - L[0] * np.floor(x / L[0])
            assert b[r][0] <= xw < b[r][1] or (xw == L[0] and r == 0)
    assert not engine.slab_info(L, 11.2, 8, 0)[2]  # 11.13 A < 11.2 A


def test_nccl_resolves_at_run_time(lib):
    """The distributed mode dlopens libnccl.so.2 and creates the 128-byte unique id that the
    ranks share (no GPU needed for the id)."""
    from paper_1810_07026_b200 import engine
    a, b = engine.nccl_unique_id(), engine.nccl_unique_id()
    assert len(a) == 128 and a != b
