#!/usr/bin/env python
"""bench.py -- AIREBO NVE throughput (atom-steps/s) of the B200 engine on BASELINE.json's metric config.

Contract (driver): python bench.py --gpus N --steps K --warmup W [--impl reference]
  * one JSON line on rank 0; value = whole-job atom-steps/s (all ranks' atoms x K / max-over-ranks
    device time), CUDA events on the engine's stream; inputs resident in HBM before the timed region.
  * workload (N=1): BASELINE configs[3] = cfg4, the polyethylene crystal 40x50x42 cells
    (1,008,000 atoms), +-0.02 A jitter, 300 K, dt = 0.5 fs, NVE (velocity Verlet, skin 1 A, lists
    rebuilt on demand) -- the configuration BASELINE's metric ("atom-steps/s (fp64 and mixed) at
    1/2/4/8 B200") is quoted on, which fits one B200.  fp64 headline + a mixed sub-line.
  * timed region = ONE ab_run_nve(K, dt, thermo_every=10) call (the loop includes
    forces, integration, skin-triggered rebuilds and thermo output every 10 steps).  The working
    set (LJ lists ~1 GB, positions, short lists) is far larger than the 126 MB L2, so no flush.
  * e2e: the same metric through the C-ABI with HOST buffers, the host holding the state: per step
    ab_set_velocities (H2D from pinned memory) + ab_run_nve(1 step, thermo row D2H) +
    ab_get_positions + ab_get_velocities (D2H), wall clock.
  * cpu_baseline / --impl reference: the fp64 CPU oracle (oracle/) on the host cores (see
    cpu_oracle_baseline / run_reference for the bounded samples).
Multi-GPU (N > 1, torchrun, one process per GPU): slab decomposition along x with
  the engine's own NCCL communicator (ab_create_dist): halo positions and ghost forces travel by
  ncclSend/ncclRecv between slab neighbours every step.  Default: cfg4 strong scaling (the
  1,008,000-atom system split over N slabs, BASELINE configs[3]); --config 5a / 5b: weak scaling,
  the 2 M-atom diamond / PE block per GPU replicated along x (BASELINE configs[4]).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AIREBO atom-steps/s (fp64 and mixed) at 1/2/4/8 B200; % of FP64/FP32 peak"
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary_r02.json")


# ------------------------------------------------------------------ helpers
def reduce_max(x, ws, device=None):
    """Max of a host scalar over all ranks (torch.distributed; identity for one rank)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload(config, ws, scaling):
    """The bench system: BASELINE config `config` at N = 1; at N > 1 strong scaling keeps it,
    weak scaling replicates the per-GPU block along x (cfg5a / 5b: n_rep = N, same seeds)."""
    from paper_1810_07026_b200 import inputs as I
    if ws > 1 and scaling == "weak":
        if config in ("5a", "5b"):
            return I.config(config, n_rep=ws)
        if config == 2:
            return I.polyethylene((12 * ws, 16, 14), 0.02, 102, 202, name=f"cfg2-pe-32k-x{ws}")
    return I.config(config)


def default_scaling(config):
    return "weak" if config in ("5a", "5b", 2) else "strong"


CFG_TEXT = {1: "BASELINE configs[0]: tiny PE 1x1x10 cells, 120 atoms, 300 K, dt 0.5 fs",
            2: "BASELINE configs[1]: PE 12x16x14 cells, 32,256 atoms, 300 K, dt 0.5 fs",
            3: "BASELINE configs[2]: relaxed amorphous CH2, 64,002 atoms, 1500 K, dt 0.25 fs",
            4: "BASELINE configs[3]: PE 40x50x42 cells, 1,008,000 atoms, 300 K, dt 0.5 fs, NVE, LJ cutoff 3 sigma, "
               "torsion on (the metric's 1/2/4/8-GPU configuration)",
            "5a": "BASELINE configs[4]: diamond 63n x 63 x 63 cells, 2,000,376 atoms per GPU, 1000 K, dt 0.5 fs",
            "5b": "BASELINE configs[4]: PE 40n x 50 x 84 cells, 2,016,000 atoms per GPU, 300 K, dt 0.5 fs"}


def config_dict(s, args, ws):
    """The `config` object of the JSON line (shared by both arms, so they carry the same dict)."""
    return {"workload": f"{s.name} ({CFG_TEXT.get(args.config, args.config)})", "atoms": s.n, "dt_fs": s.dt,
            "precision": args.precision, "potential": args.potential,
            "parallelism": "single GPU" if ws == 1 else f"slab{ws} (x slabs, NCCL halo send/recv)",
            "scaling": "weak" if ws == 1 else args.scaling,
            "l2": "not flushed: inputs larger than L2 (LJ lists ~1 GB + positions / short lists vs 126 MB L2)"
                  if s.n >= 500000 else "L2 flushed (256 MiB write) before the timed region",
            "timed_step": f"ab_run_nve(K, dt, thermo_every={args.thermo}): integrate, rebuild check / list rebuild, "
                          "forces, integrate, thermo row every 10 steps"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clock and clock-event (throttle) reasons DURING the timed region (B200_PROFILING recipe):
    NVML polled every 2 ms from a thread (a 100-step cfg2 region lasts ~40 ms, too short for
    nvidia-smi's 200 ms loop); nvidia-smi is the fallback when NVML is unavailable."""

    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.nvml = None

    def _poll(self):
        N = self.nvml
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while True:
            try:
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            except AttributeError:
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.samples.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), mx, r))
            if self.stop.wait(0.002):
                break

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
            self._smi()
        return self

    def _smi(self):
        try:
            q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
            f = [x.strip() for x in out.split(",")]
            self.samples.append((float(f[0]), float(f[1]), int(f[2], 16)))
        except Exception:
            pass

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=5)
        else:
            self._smi()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = sorted({n for _, _, r in self.samples for n, b in self.BITS.items() if r & b})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml (2 ms poll)" if self.nvml else "nvidia-smi"}


def algorithmic_flops(stats):
    """Per-phase algorithmic flop counts per launch (SURVEY §8(d) op weights).
    LJ: 31 flops per half pair inside r_c + 25 more per half pair in the taper band, split between
    the near-pair kernel (k_lj_near: pairs that may need C_ij / b*) and the far-pair kernel
    (k_lj_far, n_lj_far pairs, every taper pair); REBO: 700 per bond (pair terms, P, pi^rc, T) + 65
    per angle term + 260 per dihedral quad (pi^dh + torsion, forward and reverse); b*: 1500 per
    evaluated pair; short list: 15 per entry.  Skin entries are overhead, not algorithmic work."""
    rebo = 700 * stats["n_bonds"] + 65 * stats["n_angles"] + 260 * stats["n_quads"]
    far = stats["n_lj_far"]
    return {"short": 15 * stats["n_short"], "rebo": rebo, "lj_near": 31 * (stats["n_lj"] - far),
            "bstar": 1500 * stats["n_bstar"], "lj_far": 31 * far + 25 * stats["n_lj_taper"]}


PHASES = ["short", "rebo", "lj_near", "bstar", "integrate", "rebuild", "lj_far", "comm"]  # ab_get_phase_ms slots
KERNEL_OF = {"short": "k_short", "rebo": "k_rebo", "lj_near": "k_lj_near", "bstar": "k_bstar_lite", "lj_far": "k_lj_far"}


def fp64_peak_tflops(sm_mhz, nsm=148):
    """148 SMs x 64 FP64 FMA/clk x 2 flop x f_SM (B200_PROFILING / SURVEY §8(d) unit counts)."""
    return nsm * 64 * 2 * sm_mhz * 1e6 / 1e12


def fp32_peak_tflops(sm_mhz, nsm=148):
    return nsm * 128 * 2 * sm_mhz * 1e6 / 1e12


# ------------------------------------------------------------------ our arm
def run_ours(args, ws, rank, local):
    import torch
    from paper_1810_07026_b200 import build as B
    from paper_1810_07026_b200 import engine as E
    from paper_1810_07026_b200 import inputs as I

    if rank == 0:
        B.build()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()

    def fresh_uid():
        """A new NCCL unique id for each distributed engine (an id is single-use: NCCL's bootstrap
        root serves one communicator); collective over the ranks."""
        import torch.distributed as dist
        obj = [E.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    s = workload(args.config, ws, args.scaling)
    # a dedicated stream: the engine's kernels, the L2 flush and the timing events are all ordered
    # on it (torch's legacy default stream would leave the engine on its own stream)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if s.n < 500000 else None

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        return reduce_max(x, ws, dev)

    params = open(E.PARAMS, "rb").read()
    if args.potential != "airebo":  # the paper's REBO / AIREBO-M variants
        params = params.replace(b"potential airebo\n", b"potential " + args.potential.encode() + b"\n")

    def make_engine(precision):
        ranks = ("nccl", rank, ws, fresh_uid()) if ws > 1 else None
        e = E.Engine(precision, local, params=params, ranks=ranks)
        e.set_box(s.box)
        e.set_atoms(s.types, s.x)
        if s.v is not None:
            e.set_velocities(s.v)
        return e

    def timed_steps(eng, K, L2flush=False):
        """ONE ab_run_nve(K, dt, thermo_every) call bracketed by CUDA events on the engine's
        stream (the flush, if any, before the start event).  Returns the device time (ms)."""
        with torch.cuda.stream(stream):
            if L2flush:
                flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.run_nve(K, s.dt, every=args.thermo)
            b.record(stream)
        stream.synchronize()
        return a.elapsed_time(b)

    def leg(precision):
        import ctypes as C
        eng = make_engine(precision)
        eng.set_stream(stream.cuda_stream)
        eng.run_nve(args.warmup, s.dt)  # warm-up (untimed): builds lists
        torch.cuda.synchronize()
        nb0 = eng.stats()["n_rebuilds"]
        l0 = eng.device_info()["kernel_launches"]
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            t_ms = timed_steps(eng, args.steps, L2flush=s.n < 500000)
        torch.cuda.synchronize()
        barrier()
        launches = eng.device_info()["kernel_launches"] - l0
        nb1 = eng.stats()["n_rebuilds"]
        eng.compute()  # outside the timed region: the ab_compute kernels also count taper-band pairs
        st = eng.stats()
        st["n_rebuilds"] = nb1
        st["timed_rebuilds"] = nb1 - nb0
        total_ms = max_over_ranks(t_ms)
        # profiled replay: the next K steps with the kernels one at a time (each has the GPU to
        # itself) and per-phase CUDA events on the engine stream -> per-kernel launch durations
        # for the roofline (the events cost ~10 % of a step and the concurrent DAG overlaps the
        # kernels, so the headline above is taken without them)
        eng.set_concurrency(False)
        eng.L.ab_set_profiling(eng.h, 1)
        ptime = timed_steps(eng, args.steps)
        ms = (C.c_double * 8)()
        n = (C.c_int64 * 8)()
        eng.L.ab_get_phase_ms(eng.h, ms, n)
        eng.L.ab_set_profiling(eng.h, 0)
        eng.set_concurrency(True)
        out = dict(eng=eng, total_ms=total_ms, clocks=clk.summary(), launches=launches,
                   phase={p: (ms[q], int(n[q])) for q, p in enumerate(PHASES)}, stats=st,
                   prof_total_ms=ptime)
        return out

    res = {}
    for prec in ([args.precision] + (["mixed"] if args.precision == "fp64" and not args.no_mixed else [])):
        res[prec] = leg(prec)

    main = res[args.precision]
    eng = main["eng"]
    st = main["stats"]
    n_atoms = s.n
    K = args.steps
    value = n_atoms * K / (main["total_ms"] * 1e-3)  # all ranks' atoms / max-over-ranks time
    ms_per_step = main["total_ms"] / K

    def roofline(r, precision):
        flops = algorithmic_flops(r["stats"])
        dom = max(("short", "rebo", "lj_near", "bstar", "lj_far"), key=lambda p: r["phase"][p][0])
        tot_ms, cnt = r["phase"][dom]
        avg_s = tot_ms / max(cnt, 1) * 1e-3
        achieved = flops[dom] / avg_s / 1e12 if avg_s > 0 else 0.0
        clk = r["clocks"]["sm_mhz"] or 1965.0
        peak = fp64_peak_tflops(clk) if precision == "fp64" else fp32_peak_tflops(clk)
        traffic, hw = None, None
        if os.path.exists(PROFILE_SUMMARY):
            try:
                summ = json.load(open(PROFILE_SUMMARY))
                ks = summ.get(precision, {}).get(KERNEL_OF[dom], {})
                traffic = summ.get("fp64", {}).get(KERNEL_OF[dom], {}).get("dram_bytes_per_launch") \
                    if precision == "fp64" else ks.get("dram_bytes_per_launch")
                if ks.get("hw_flops_per_launch") and avg_s > 0:
                    # SURVEY §8(d) fraction (i): executed FP64 (FP32) flops of the kernel, counted by ncu
                    # (2 DFMA + DMUL + DADD thread instructions per launch), over the live duration
                    hw_tf = ks["hw_flops_per_launch"] / avg_s / 1e12
                    hw = {"flops_per_launch": ks["hw_flops_per_launch"], "tflops": round(hw_tf, 4),
                          "frac": round(hw_tf / peak, 5), "source": os.path.basename(PROFILE_SUMMARY)}
            except (ValueError, OSError):
                traffic = None
        step_flops = sum(flops.values())
        step_s = r["total_ms"] / K * 1e-3
        # DRAM bytes of one evaluation (ncu cold-cache bytes per launch x launches per
        # NVE step: short 1, REBO 2, near 1, far 1, b* 3) against the measured HBM bandwidth
        dram = None
        try:
            summ = json.load(open(PROFILE_SUMMARY)).get(precision, {})
            per = {"k_short": 1, "k_rebo": 2, "k_lj_near": 1, "k_lj_far": 1, "k_bstar_lite": 1}
            if all(k in summ and summ[k].get("dram_bytes_per_launch") for k in per):
                byts = sum(summ[k]["dram_bytes_per_launch"] * n for k, n in per.items())
                hbm = None
                mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
                if os.path.exists(mp):
                    hbm = json.load(open(mp)).get("hbm_gbs")
                gbs = byts / step_s / 1e9
                dram = {"bytes_per_step": byts, "gbs_at_step_time": round(gbs, 1), "hbm_gbs": hbm,
                        "frac": round(gbs / hbm, 4) if hbm else None,
                        "source": os.path.basename(PROFILE_SUMMARY) + " (cold-cache per-launch bytes)"}
        except (ValueError, OSError):
            dram = None
        return {"bound": "alu", "kernel": KERNEL_OF[dom], "achieved": round(achieved, 4), "peak": round(peak, 3),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 5), "traffic": traffic, "hw": hw,
                "peak_basis": f"{'FP64' if precision == 'fp64' else 'FP32'} FMA units x 2 x median SM clock "
                              f"{clk:.0f} MHz under load (no FP64 entry in MEASURED_PEAKS.json)",
                "algorithmic_flops_per_launch": flops[dom], "avg_launch_ms": round(avg_s * 1e3, 5),
                "kernel_share_of_step": round(tot_ms / max(r["prof_total_ms"], 1e-9), 4),
                "measured_in": "profiled replay of K further timed steps with the kernels serialised "
                               "(ab_set_concurrency(0)), CUDA events on the engine stream; the headline "
                               "value runs the concurrent DAG",
                "whole_step_tflops": round(step_flops / step_s / 1e12, 4),
                "whole_step_frac": round(step_flops / step_s / 1e12 / peak, 5),
                "phase_ms_per_step": {p: round(v[0] / K, 5) for p, v in r["phase"].items()},
                "comm_ms_per_step": round(r["phase"]["comm"][0] / K, 5) if ws > 1 else None,
                "dram_per_step": dram}

    peak_meas = {}
    for p, code in (("fp64", E.AB_FP64), ("fp32", E.AB_MIXED)):
        import ctypes as C
        tf = C.c_double()
        if eng.L.ab_peak_flops(eng.h, code, C.byref(tf)) == 0:
            peak_meas[p] = round(tf.value, 2)

    # ---- e2e through the C-ABI with host buffers (pinned): the host holds the dynamical state.
    # Every step: velocities H2D (the host's copy, as a host-side thermostat or analysis would
    # hand them back), one NVE step with its thermo row D2H, positions and velocities D2H.
    e2e = None
    if not args.no_e2e:
        import torch
        eng2 = make_engine(args.precision)
        eng2.set_stream(stream.cuda_stream)
        eng2.run_nve(args.warmup, s.dt)
        vh = torch.from_numpy(eng2.get_velocities()).pin_memory()
        xh = torch.empty((n_atoms, 3), dtype=torch.float64).pin_memory()
        th = np.zeros((2, 4))
        import ctypes as C
        dp = C.POINTER(C.c_double)
        vptr = C.cast(vh.data_ptr(), dp)
        xptr = C.cast(xh.data_ptr(), dp)
        thp = th.ctypes.data_as(dp)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            eng2._ck(eng2.L.ab_set_velocities(eng2.h, vptr))
            eng2._ck(eng2.L.ab_run_nve(eng2.h, 1, s.dt, 1, thp))
            eng2._ck(eng2.L.ab_get_positions(eng2.h, xptr))
            eng2._ck(eng2.L.ab_get_velocities(eng2.h, vptr))
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": n_atoms * K / t_e2e, "unit": "atom-steps/s", "h2d_bytes_per_step": 24 * n_atoms,
               "d2h_bytes_per_step": 48 * n_atoms + 64,
               "step": "ab_set_velocities (H2D, pinned) + ab_run_nve(1, thermo row) + ab_get_positions + "
                       "ab_get_velocities (D2H, pinned)"}
        eng2.close()

    # ---- CPU baseline: the oracle as it stands, on this host's cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(s, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "atom-steps/s", "n_gpus": ws, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if (ws > 1 and args.scaling == "strong") else "weak",
            "vs_baseline": None,
            "dtype": {"fp64": "f64", "mixed": "f32+f64acc", "single": "f32"}[args.precision],
            "data": "synthetic (seeded generator, paper_1810_07026_b200/inputs.py)",
            "config": config_dict(s, args, ws),
            "roofline": roofline(main, args.precision),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": main["clocks"],
            "gpu_launches": main["launches"],
            "peak_measured_fma_tflops": peak_meas,
            "counters": {k: st[k] for k in ("n_lj", "n_C0", "n_bstar", "n_sb_trans", "n_bonds", "n_quads",
                                            "n_rebuilds", "timed_rebuilds", "n_ghosts")},
            "thermo_rows_per_call": args.steps // args.thermo + 1,
        }
        if "mixed" in res and args.precision == "fp64":
            r = res["mixed"]
            line["mixed"] = {"value": n_atoms * K / (r["total_ms"] * 1e-3), "ms_per_step": r["total_ms"] / K,
                             "roofline": roofline(r, "mixed"), "clocks": r["clocks"]}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def sample_block(config):
    """A bounded CPU sample of the workload: the same crystal / chemistry in a periodic block the
    oracle steps in well under a second per step on the host's cores (per-atom work of a periodic
    crystal does not depend on the block size).  cfg 1-3: the config itself."""
    from paper_1810_07026_b200 import inputs as I
    if config in (4, "5b"):
        return I.polyethylene((12, 16, 14), 0.02, 104, 204, name="pe-12x16x14-sample")  # 32,256 atoms
    if config == "5a":
        return I.diamond((16, 16, 16), 0.03, 105, 205, name="diamond-16^3-sample")  # 32,768 atoms
    return I.config(config)


def cpu_oracle_baseline(s, args):
    """The oracle as it stands: (i) all host cores on the FULL workload, one force
    evaluation timed and extrapolated to atom-steps/s (cfgs 4-5 rule: the oracle rebuilds its lists
    and AD forces every evaluation, the integration is negligible); (ii) one thread, ONE
    velocity-Verlet NVE call of a few steps on the bounded sample block (K steps = K + 1
    evaluations, all counted against K steps)."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    O.compute(s.types, s.x, s.box, threads=cores)
    t_all = time.perf_counter() - t0
    b = sample_block(args.config)
    k1 = 2
    t0 = time.perf_counter()
    O.nve(b.types, b.x, b.v, b.box, k1, b.dt, every=0, threads=1)
    t_one = time.perf_counter() - t0
    return {"value": s.n / t_all, "unit": "atom-steps/s", "cores": cores, "kind": "oracle",
            "sample": f"one full force evaluation (lists + energy + AD forces + virial) of the {s.n}-atom {s.name} "
                      f"on {cores} threads, {t_all:.1f} s wall, extrapolated as 1 evaluation per step",
            "single_thread": {"value": b.n * k1 / t_one, "unit": "atom-steps/s", "cores": 1,
                              "sample": f"one oracle NVE call of {k1} steps ({k1 + 1} evaluations) of {b.name} "
                                        f"({b.n} atoms), {t_one:.1f} s wall"},
            "host": host_info()}


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model}


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args, ws, rank, local):
    """The oracle as it stands on the host cores, rank 0 only.  Each step is a bounded sample of the
    workload: one oracle NVE call of K steps (after W warm-up steps) on sample_block(config), the
    same crystal in a ~32 k-atom periodic block, value = sample atoms x K / wall seconds."""
    if rank != 0:
        return
    from oracle import oracle as O
    s = workload(args.config, ws, args.scaling)
    b = sample_block(args.config)
    cores = os.cpu_count() or 1
    x, v = b.x.copy(), b.v.copy()
    x, v, _ = O.nve(b.types, x, v, b.box, args.warmup, b.dt, every=0, threads=cores)
    t0 = time.perf_counter()
    x, v, _ = O.nve(b.types, x, v, b.box, args.steps, b.dt, every=0, threads=cores)
    t = time.perf_counter() - t0
    val = b.n * args.steps / t
    sample = (f"one oracle NVE call of {args.steps} steps ({args.steps + 1} evaluations) of {b.name} ({b.n} atoms), "
              f"a periodic block of the workload's crystal, after {args.warmup} warm-up steps; {t:.1f} s wall")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "atom-steps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak" if ws == 1 else args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(s, args, ws),
            "cpu_baseline": {"value": val, "unit": "atom-steps/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "host": host_info()},
            "e2e": {"value": val, "unit": "atom-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed", "single"])
    ap.add_argument("--config", default=4, type=lambda v: int(v) if v.isdigit() else v)
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"])
    ap.add_argument("--thermo", type=int, default=10, help="thermo row every THERMO steps (SURVEY §8(d): 10)")
    ap.add_argument("--potential", default="airebo", choices=["airebo", "rebo", "airebo-m"])
    ap.add_argument("--no-mixed", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.scaling is None:
        args.scaling = default_scaling(args.config)
    args.warmup = max(3, args.warmup)
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
