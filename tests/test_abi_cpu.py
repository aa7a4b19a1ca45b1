"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports every symbol
that include/airebo_b200.h declares (no compute calls: there is no GPU here)."""
import os
import re
import subprocess

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
