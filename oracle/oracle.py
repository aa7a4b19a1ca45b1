"""ctypes wrapper around oracle/liboracle.so (the fp64 CPU oracle).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module.  It never imports the CUDA package and the CUDA
package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = [os.path.join(HERE, f) for f in ("airebo.cpp", "ad.hpp", "params.hpp")]
PARAMS = os.path.join(os.path.dirname(HERE), "params", "toy_ch.param")

COUNTERS = ["n_short", "n_bonds", "n_quads", "n_lj", "n_C0", "n_bstar", "n_sb_trans", "max_short", "max_reach",
            "n_badarg"]

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -ffp-contract=off -fopenmp)."""
    newest = max(os.path.getmtime(s) for s in SRC)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fopenmp", "-std=c++17", "-shared", "-fPIC", "-o", LIB,
               os.path.join(HERE, "airebo.cpp")]
        subprocess.run(cmd, check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        dp, ip, lp = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_longlong)
        L.oracle_compute.argtypes = [C.c_char_p, C.c_int, ip, dp, dp, dp, dp, dp, lp, C.c_int, C.c_int]
        L.oracle_compute_digest.argtypes = [C.c_char_p, C.c_int, ip, dp, dp, dp, dp, dp, lp, C.c_int,
                                            C.POINTER(C.c_ulonglong)]
        L.oracle_forces_sampled.argtypes = [C.c_char_p, C.c_int, ip, dp, dp, C.c_int, ip, dp, C.c_int]
        L.oracle_list.argtypes = [C.c_char_p, C.c_int, ip, dp, dp, C.c_int, lp, lp, C.c_int]
        L.oracle_stages.argtypes = [C.c_char_p, C.c_int, ip, dp, dp, dp, dp]
        L.oracle_nve.argtypes = [C.c_char_p, C.c_int, ip, dp, dp, dp, C.c_int, C.c_double, C.c_int, dp, C.c_int]
        L.oracle_switch.argtypes = [C.c_double, C.c_double, C.c_double, dp]
        L.oracle_spline.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, dp]
        L.oracle_parse.argtypes = [C.c_char_p]
        L.oracle_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def params_text(path: str = PARAMS) -> bytes:
    with open(path, "rb") as f:
        return f.read()


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def _prep(types, x, box):
    t = np.ascontiguousarray(types, dtype=np.int32)
    xx = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
    b = np.ascontiguousarray(box, dtype=np.float64)
    return t, xx, b


def _check(rc):
    if rc != 0:
        raise RuntimeError("oracle: " + lib().oracle_last_error().decode())


def compute(types, x, box, params=None, forces=True, brute=False, lj=True, rebo=True, threads=None):
    """Returns dict(E=total, terms=[E_REBO, E_TORS, E_LJ], F=[n,3] or None, W=[6], counters={...})."""
    t, xx, b = _prep(types, x, box)
    n = t.shape[0]
    F = np.zeros((n, 3)) if forces else None
    W = np.zeros(6)
    E3 = np.zeros(3)
    cnt = np.zeros(len(COUNTERS), dtype=np.int64)
    flags = (1 if brute else 0) | (0 if lj else 2) | (0 if rebo else 4)
    nt = threads or os.cpu_count() or 1
    _check(lib().oracle_compute(params or params_text(), n, _p(t, C.c_int), _p(xx, C.c_double), _p(b, C.c_double),
                                _p(F, C.c_double), _p(E3, C.c_double), _p(W, C.c_double) if forces else None,
                                _p(cnt, C.c_longlong), nt, flags))
    return dict(E=float(E3.sum()), terms=E3, F=F, W=W if forces else None,
                counters={k: int(v) for k, v in zip(COUNTERS, cnt)})


def compute_digest(types, x, box, params=None, threads=None):
    """compute() (forces, energy terms, virial, counters) plus the order-independent digests
    {count, sum h, xor h} of the short list, the REBO half bonds and the LJ half pairs from one
    list build (ab_get_list_digest's definition; full-size list parity)."""
    t, xx, b = _prep(types, x, box)
    n = t.shape[0]
    F = np.zeros((n, 3))
    W = np.zeros(6)
    E3 = np.zeros(3)
    cnt = np.zeros(len(COUNTERS), dtype=np.int64)
    dig = np.zeros(9, dtype=np.uint64)
    nt = threads or os.cpu_count() or 1
    _check(lib().oracle_compute_digest(params or params_text(), n, _p(t, C.c_int), _p(xx, C.c_double),
                                       _p(b, C.c_double), _p(F, C.c_double), _p(E3, C.c_double), _p(W, C.c_double),
                                       _p(cnt, C.c_longlong), nt, _p(dig, C.c_ulonglong)))
    return dict(E=float(E3.sum()), terms=E3, F=F, W=W, counters={k: int(v) for k, v in zip(COUNTERS, cnt)},
                digest=[tuple(int(v) for v in dig[3 * w:3 * w + 3]) for w in range(3)])


def forces_sampled(types, x, box, sample, params=None, threads=None):
    t, xx, b = _prep(types, x, box)
    s = np.ascontiguousarray(sample, dtype=np.int32)
    Fs = np.zeros((s.shape[0], 3))
    nt = threads or os.cpu_count() or 1
    _check(lib().oracle_forces_sampled(params or params_text(), t.shape[0], _p(t, C.c_int), _p(xx, C.c_double),
                                       _p(b, C.c_double), s.shape[0], _p(s, C.c_int), _p(Fs, C.c_double), nt))
    return Fs


def get_list(types, x, box, which, params=None, brute=False):
    """which: 0 short (full), 1 REBO half bonds, 2 LJ half pairs.  Rows (i, j, sx, sy, sz), sorted."""
    t, xx, b = _prep(types, x, box)
    cnt = C.c_longlong(0)
    args = (params or params_text(), t.shape[0], _p(t, C.c_int), _p(xx, C.c_double), _p(b, C.c_double), which)
    _check(lib().oracle_list(*args, C.byref(cnt), None, int(brute)))
    rows = np.zeros((cnt.value, 5), dtype=np.int64)
    _check(lib().oracle_list(*args, C.byref(cnt), _p(rows, C.c_longlong), int(brute)))
    return rows


def stages(types, x, box, params=None, lj=True):
    """Per-bond [b, p_ij, p_ji, pi_rc, pi_dh, N_ij, N_ji, N_conj] and per-LJ-pair [C, b*, Q, E]."""
    nb = get_list(types, x, box, 1, params).shape[0]
    nl = get_list(types, x, box, 2, params).shape[0] if lj else 0
    t, xx, b = _prep(types, x, box)
    B = np.zeros((nb, 8))
    Lj = np.zeros((nl, 4)) if lj else None
    _check(lib().oracle_stages(params or params_text(), t.shape[0], _p(t, C.c_int), _p(xx, C.c_double),
                               _p(b, C.c_double), _p(B, C.c_double), _p(Lj, C.c_double)))
    return B, Lj


def nve(types, x, v, box, nsteps, dt, every=10, params=None, threads=None):
    t, xx, b = _prep(types, x, box)
    xx = xx.copy()
    vv = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3).copy()
    nrow = nsteps // every + 1 if every > 0 else 0
    th = np.zeros((max(nrow, 1), 4))
    nt = threads or os.cpu_count() or 1
    _check(lib().oracle_nve(params or params_text(), t.shape[0], _p(t, C.c_int), _p(xx, C.c_double),
                            _p(vv, C.c_double), _p(b, C.c_double), nsteps, dt, every, _p(th, C.c_double), nt))
    return xx, vv, th[:nrow]


def switch(x, lo, hi):
    out = np.zeros(2)
    lib().oracle_switch(x, lo, hi, _p(out, C.c_double))
    return out


def spline(which, a, x, y=0.0, z=0.0, params=None):
    """which 0 = g (a = species), 1 = P (a = t_j), 2 = R (a = pair 0 CC / 1 CH / 2 HH), 3 = T."""
    out = np.zeros(4)
    _check(lib().oracle_spline(params or params_text(), which, a, x, y, z, _p(out, C.c_double)))
    return out


def parse_ok(text: bytes) -> tuple[bool, str]:
    rc = lib().oracle_parse(text)
    return rc == 0, lib().oracle_last_error().decode()
