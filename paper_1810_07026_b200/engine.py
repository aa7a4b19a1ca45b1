"""Thin ctypes binding of libairebo_b200.so (include/airebo_b200.h): argument marshalling only.

Every step of the force / NVE path runs in the CUDA kernels of the library.  There is no CPU
fallback: if the library cannot be loaded or no sm_100 GPU is present, the calls raise.
Function names mirror the C-ABI (ab_create, ab_set_box, ...); `Engine` bundles them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AIREBO_B200_LIB", os.path.join(HERE, "libairebo_b200.so"))
PARAMS = os.path.join(os.path.dirname(HERE), "params", "toy_ch.param")

AB_FP64, AB_MIXED, AB_SINGLE, AB_REDUCED = 0, 1, 2, 3
AB_LIST_SHORT, AB_LIST_BONDS, AB_LIST_LJ, AB_LIST_LJ_SKIN = 0, 1, 2, 3
STATUS = {0: "AB_OK", -1: "AB_E_ARG", -2: "AB_E_PARAM", -3: "AB_E_BOX", -4: "AB_E_STATE", -5: "AB_E_OOM",
          -6: "AB_E_CUDA", -7: "AB_E_NCCL", -8: "AB_E_NONFINITE"}


class ABError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ABStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "n_short", "n_bonds", "n_quads", "n_lj", "n_C0", "n_bstar", "n_sb_trans", "max_short", "max_reach",
        "n_badarg", "n_atoms", "n_ghosts", "n_rebuilds", "n_steps", "n_overflow_retries", "lj_capacity",
        "inter_capacity", "n_lj_entries", "n_angles", "n_lj_far", "n_lj_entries_far", "n_lj_taper")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


EXPORTS = ["ab_create", "ab_destroy", "ab_last_error", "ab_set_stream", "ab_set_box", "ab_set_atoms",
           "ab_set_positions", "ab_set_velocities", "ab_compute", "ab_run_nve", "ab_get_positions",
           "ab_get_velocities", "ab_get_forces", "ab_get_list", "ab_get_stats", "ab_record_stages", "ab_get_stage",
           "ab_set_profiling", "ab_get_phase_ms", "ab_peak_flops", "ab_device_info", "ab_nccl_unique_id",
           "ab_create_dist", "ab_create_virtual", "ab_slab_info", "ab_slab_of", "ab_set_concurrency",
           "ab_get_list_digest"]

_lib = None


def load(path: str = LIB_PATH):
    """dlopen the in-tree library and declare the C signatures (no compute, works without a GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ABError(-6, f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(path)
    vp, dp, i64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)
    L.ab_create.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.POINTER(vp)]
    L.ab_destroy.argtypes = [vp]
    L.ab_destroy.restype = None
    L.ab_last_error.argtypes = [vp]
    L.ab_last_error.restype = C.c_char_p
    L.ab_set_stream.argtypes = [vp, vp]
    L.ab_set_box.argtypes = [vp, dp]
    L.ab_set_atoms.argtypes = [vp, C.c_int64, C.POINTER(C.c_int32), dp]
    L.ab_set_positions.argtypes = [vp, dp]
    L.ab_set_velocities.argtypes = [vp, dp]
    L.ab_compute.argtypes = [vp, dp, dp, dp, dp]
    L.ab_run_nve.argtypes = [vp, C.c_int64, C.c_double, C.c_int64, dp]
    L.ab_get_positions.argtypes = [vp, dp]
    L.ab_get_velocities.argtypes = [vp, dp]
    L.ab_get_forces.argtypes = [vp, dp]
    L.ab_get_list.argtypes = [vp, C.c_int, i64p, i64p]
    L.ab_get_list_digest.argtypes = [vp, C.c_int, C.POINTER(C.c_uint64)]
    L.ab_get_stats.argtypes = [vp, C.POINTER(ABStats)]
    L.ab_record_stages.argtypes = [vp, C.c_int]
    L.ab_get_stage.argtypes = [vp, C.c_int, i64p, dp]
    L.ab_device_info.argtypes = [vp, C.POINTER(C.c_int), C.c_char_p, C.c_size_t, i64p]
    L.ab_set_profiling.argtypes = [vp, C.c_int]
    L.ab_get_phase_ms.argtypes = [vp, dp, i64p]
    L.ab_peak_flops.argtypes = [vp, C.c_int, dp]
    L.ab_nccl_unique_id.argtypes = [C.c_char_p]
    L.ab_create_dist.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]
    L.ab_create_virtual.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
    L.ab_slab_info.argtypes = [dp, C.c_double, C.c_int, C.c_int, dp, dp]
    L.ab_slab_of.argtypes = [C.c_double, C.c_double, C.c_int]
    L.ab_slab_of.restype = C.c_int
    L.ab_set_concurrency.argtypes = [vp, C.c_int]
    _lib = L
    return L


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for ab_create_dist (create on one rank, broadcast to all)."""
    L = load()
    buf = C.create_string_buffer(128)
    rc = L.ab_nccl_unique_id(buf)
    if rc != 0:
        raise ABError(rc, L.ab_last_error(None).decode())
    return buf.raw


def slab_info(box, halo, nranks, rank):
    """(xlo, xhi, ok) of slab `rank` (host-only library call, no GPU)."""
    L = load()
    b = np.ascontiguousarray(box, dtype=np.float64)
    lo, hi = C.c_double(), C.c_double()
    rc = L.ab_slab_info(_dp(b), halo, nranks, rank, C.byref(lo), C.byref(hi))
    if rc not in (0, -3):
        raise ABError(rc, "ab_slab_info")
    return lo.value, hi.value, rc == 0


def slab_of(x, Lx, nranks):
    return load().ab_slab_of(float(x), float(Lx), int(nranks))


class Engine:
    """One engine handle (one precision).  Arrays in and out are in the caller's atom order.

    ranks=None: one GPU, whole box.  ranks=("virtual", n): n slab domains on this GPU exchanging
    their halo by device copies.  ranks=("nccl", rank, n, uid): slab `rank` of an n-process job
    (collective calls; uid from nccl_unique_id() on one rank, a fresh one per engine: single-use)."""

    def __init__(self, precision: str = "fp64", device: int = 0, params: bytes | None = None, ranks=None):
        self.L = load()
        if params is None:
            with open(PARAMS, "rb") as f:
                params = f.read()
        h = C.c_void_p()
        prec = {"fp64": AB_FP64, "mixed": AB_MIXED, "single": AB_SINGLE, "reduced": AB_REDUCED}[precision]
        if ranks is None:
            rc = self.L.ab_create(params, len(params), prec, device, C.byref(h))
        elif ranks[0] == "virtual":
            rc = self.L.ab_create_virtual(params, len(params), prec, device, int(ranks[1]), C.byref(h))
        elif ranks[0] == "nccl":
            _, rank, n, uid = ranks
            rc = self.L.ab_create_dist(params, len(params), prec, device, int(rank), int(n), uid, C.byref(h))
        else:
            raise ValueError(ranks)
        if rc != 0:
            raise ABError(rc, self.L.ab_last_error(None).decode())
        self.h = h
        self.n = 0
        self.precision = precision

    def _ck(self, rc):
        if rc != 0:
            raise ABError(rc, self.L.ab_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.ab_destroy(self.h)
            self.h = None

    __del__ = close

    def set_stream(self, stream_ptr: int | None):
        """Run on a caller's cudaStream_t (e.g. torch.cuda.Stream().cuda_stream).  None: the
        engine's own stream.  0 (torch's legacy default stream) maps to cudaStreamLegacy, so the
        engine's work is ordered with work on that stream."""
        if stream_ptr is None:
            ptr = 0
        else:
            ptr = 1 if stream_ptr == 0 else stream_ptr
        self._ck(self.L.ab_set_stream(self.h, C.c_void_p(ptr)))

    def set_concurrency(self, on: bool):
        self._ck(self.L.ab_set_concurrency(self.h, int(on)))

    def set_box(self, L):
        b = np.ascontiguousarray(L, dtype=np.float64)
        self._ck(self.L.ab_set_box(self.h, _dp(b)))

    def set_atoms(self, types, xyz):
        t = np.ascontiguousarray(types, dtype=np.int32)
        x = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        self._ck(self.L.ab_set_atoms(self.h, t.shape[0], t.ctypes.data_as(C.POINTER(C.c_int32)), _dp(x)))
        self.n = t.shape[0]

    def set_positions(self, xyz):
        x = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        self._ck(self.L.ab_set_positions(self.h, _dp(x)))

    def set_velocities(self, v):
        x = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3)
        self._ck(self.L.ab_set_velocities(self.h, _dp(x)))

    def compute(self, forces=True):
        F = np.zeros((self.n, 3)) if forces else None
        E = C.c_double()
        W = np.zeros(6)
        T = np.zeros(3)
        self._ck(self.L.ab_compute(self.h, _dp(F), C.byref(E), _dp(W), _dp(T)))
        return dict(E=E.value, terms=T, F=F, W=W)

    def run_nve(self, nsteps, dt, every=0):
        th = np.zeros((nsteps // every + 1, 4)) if every > 0 else None
        self._ck(self.L.ab_run_nve(self.h, nsteps, dt, every, _dp(th)))
        return th

    def get_positions(self):
        x = np.zeros((self.n, 3))
        self._ck(self.L.ab_get_positions(self.h, _dp(x)))
        return x

    def get_velocities(self):
        v = np.zeros((self.n, 3))
        self._ck(self.L.ab_get_velocities(self.h, _dp(v)))
        return v

    def get_forces(self):
        f = np.zeros((self.n, 3))
        self._ck(self.L.ab_get_forces(self.h, _dp(f)))
        return f

    def get_list(self, which):
        cnt = C.c_int64()
        self._ck(self.L.ab_get_list(self.h, which, C.byref(cnt), None))
        rows = np.zeros((cnt.value, 5), dtype=np.int64)
        self._ck(self.L.ab_get_list(self.h, which, C.byref(cnt), rows.ctypes.data_as(C.POINTER(C.c_int64))))
        return rows

    def list_digest(self, which):
        """(count, sum h, xor h) of the list's rows (ab_get_list_digest)."""
        d = (C.c_uint64 * 3)()
        self._ck(self.L.ab_get_list_digest(self.h, which, d))
        return tuple(int(v) for v in d)

    def stats(self):
        s = ABStats()
        self._ck(self.L.ab_get_stats(self.h, C.byref(s)))
        return s.as_dict()

    def record_stages(self, on=True):
        self._ck(self.L.ab_record_stages(self.h, int(on)))

    def get_stage(self, stage):
        cnt = C.c_int64()
        self._ck(self.L.ab_get_stage(self.h, stage, C.byref(cnt), None))
        w = 13 if stage == 0 else 7
        out = np.zeros((cnt.value, w))
        self._ck(self.L.ab_get_stage(self.h, stage, C.byref(cnt), _dp(out)))
        return out

    def device_info(self):
        dev = C.c_int()
        name = C.create_string_buffer(256)
        n = C.c_int64()
        self._ck(self.L.ab_device_info(self.h, C.byref(dev), name, 256, C.byref(n)))
        return dict(device=dev.value, name=name.value.decode(), kernel_launches=n.value)


def make(system, precision="fp64", device=0, ranks=None):
    """Engine loaded with an inputs.System (box, types, positions, velocities)."""
    e = Engine(precision, device, ranks=ranks)
    e.set_box(system.box)
    e.set_atoms(system.types, system.x)
    if system.v is not None:
        e.set_velocities(system.v)
    return e
