/* airebo_b200.h -- C-ABI of the B200-native AIREBO force/energy engine (libairebo_b200.so).
 *
 * The calls follow the paper's statement of the problem: set atom types,
 * positions and a periodic box; compute per-atom forces, total energy and virial; advance
 * velocity-Verlet NVE steps.  PAPER.md P:212-222 (MD step: "calculates the forces that act on
 * each atom, and updates the positions and velocities"), P:231-238 (F_i = -grad_{x_i} V),
 * P:415-417 / P:467 / P:496-506 (the AIREBO terms), P:281-291 (neighbour lists with skin).
 *
 * Conventions (all calls):
 *   - Every call returns ab_status: AB_OK (0) or a negative error code; ab_last_error() gives text.
 *   - Units: Angstrom, eV, amu, fs (metal style; constants come from the parameter file).
 *   - Host pointers only.  The library COPIES every input array and never retains a caller
 *     pointer; output arrays are caller-allocated.  All device memory, streams and kernels are
 *     owned by the engine and released by ab_destroy.
 *   - Per-atom arrays are in the CALLER's atom order (the engine sorts atoms by cell internally
 *     and permutes back).  xyz arrays are n*3 doubles, AoS (x0 y0 z0 x1 ...).
 *   - One engine per host thread; a handle is not thread-safe.  After AB_E_CUDA the engine is
 *     unusable (destroy it).
 *   - There is no CPU fallback: if no sm_100 device is present ab_create fails with AB_E_CUDA.
 */
#ifndef AIREBO_B200_H
#define AIREBO_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ab_engine ab_engine;

typedef enum {
  AB_OK = 0,
  AB_E_ARG = -1,       /* bad argument (NULL pointer, n < 0, unknown enum) */
  AB_E_PARAM = -2,     /* parameter text: parse error (names line or key) or invariant violation */
  AB_E_BOX = -3,       /* box edge <= 0 or not finite; slab narrower than the halo */
  AB_E_STATE = -4,     /* call order (e.g. compute before set_atoms) or capacity beyond a hard limit */
  AB_E_OOM = -5,       /* device allocation failed */
  AB_E_CUDA = -6,      /* CUDA error or no sm_100 device; engine unusable */
  AB_E_NCCL = -7,      /* NCCL library missing or a collective failed (distributed mode) */
  AB_E_NONFINITE = -8  /* non-finite input coordinate or non-finite energy */
} ab_status;

typedef enum {
  AB_FP64 = 0,  /* IEEE binary64 throughout */
  AB_MIXED = 1, /* fp64 positions/displacements/list decisions/accumulators; fp32 term arithmetic
                   after the displacement vector (SURVEY reading A14) */
  AB_SINGLE = 2, /* the paper's "single" mode for the precision study (SURVEY
                   8(f) F2): AB_MIXED with every accumulation in fp32 -- per-thread force / energy
                   / virial sums, the warp reductions and the per-atom force array (fp32 atomics)
                   -- so the accumulator precision is the only difference to AB_MIXED (reading
                   A32).  Positions, velocities and the integrator stay fp64. */
  AB_REDUCED = 3 /* "binary32 throughout" (the x86 single precision of P:886-888 that
                    packs positions in fp32): AB_SINGLE plus a binary32 dynamical state -- every
                    half-kick v + dtf F and drift x + dt v is two binary32 operations (no FMA), so
                    positions and velocities stay binary32 values between steps (reading A35).
                    List / gate decisions are still exact fp64 tests of those positions. */
} ab_precision;

typedef enum {
  AB_LIST_SHORT = 0, /* full REBO short list: r <= r_max(t_i,t_j), both directions */
  AB_LIST_BONDS = 1, /* REBO half bonds: short-list entries with i < j (image tie-break s >_lex 0) */
  AB_LIST_LJ = 2,    /* LJ half pairs with r <= r_c(t_i,t_j) (half convention P:275-278) */
  AB_LIST_LJ_SKIN = 3 /* the skinned LJ half list of the last rebuild: half pairs with
                         r <= r_c + skin at the build positions (rows of the current instances) */
} ab_list;

/* Integer counters of the last force evaluation (must equal the oracle's exactly in fp64) and
 * bookkeeping of the engine.  Gate statistics mirror P:482-483. */
typedef struct ab_stats {
  int64_t n_short;     /* full short-list entries over owned atoms */
  int64_t n_bonds;     /* REBO half bonds */
  int64_t n_quads;     /* (bond, k, l) dihedral quadruples enumerated, l != k */
  int64_t n_lj;        /* LJ half pairs with r <= r_c */
  int64_t n_C0;        /* ... of which C_ij == 0 (skipped, Alg. 3) */
  int64_t n_bstar;     /* ... with C_ij != 0 and S_r != 0 (b* evaluated) */
  int64_t n_sb_trans;  /* ... of which b* strictly inside (b_min, b_max) */
  int64_t max_short;   /* max |N(i)| */
  int64_t max_reach;   /* max number of distinct atom images within 3 bonds of an atom (capped at the
                          64-slot reach table when it overflows; overflows: n_overflow_retries) */
  int64_t n_badarg;    /* p^{sigma pi} arguments <= 0 (must be 0) */
  int64_t n_atoms, n_ghosts, n_rebuilds, n_steps, n_overflow_retries;
  int64_t lj_capacity, inter_capacity;
  int64_t n_lj_entries; /* LJ atom slots streamed (both directions): cluster slots (4 per listed
                           cluster) with AB_LJ_CLUSTER=1, else skinned list entries */
  int64_t n_angles;     /* bond-order angle terms (k in N(i)\j plus l in N(j)\i, per half bond) */
  int64_t n_lj_far;     /* ... of n_lj, pairs of the far-pair kernel (AB_LJ_CLUSTER=1: pairs with r > 3 r_max) */
  int64_t n_lj_entries_far;
  int64_t n_lj_taper;   /* ... of n_lj, pairs in the taper band r_lo < r <= r_c (reading A10); counted by
                           ab_compute evaluations only (0 after ab_run_nve steps) */
} ab_stats;

/* Create an engine on CUDA device `cuda_device` from parameter-file text (params/toy_ch.param
 * grammar).  `len` = bytes of param_text (need not be NUL-terminated).  *out receives the handle.
 * Errors: AB_E_ARG, AB_E_PARAM (message names the line or key), AB_E_CUDA (no sm_100 device). */
ab_status ab_create(const char* param_text, size_t len, ab_precision prec, int cuda_device, ab_engine** out);

/* ---- Spatial slab decomposition (the paper's MPI domains of LAMMPS).
 * The box is cut into nranks equal slabs along x; slab r owns the atoms whose wrapped x lies in
 * [r L_x / n, (r+1) L_x / n).  Each slab keeps a halo of ghost atom instances within
 * h = r_c,max + skin of its faces (LJ partners, C_ij paths, b* neighbourhoods and complete ghost
 * short lists all lie inside it); halo positions are exchanged every step and the forces the
 * slab puts on ghosts are returned to their owners and added there.  Each pair / bond /
 * dihedral term is computed once globally by the owner of its lower (gid, image) instance.
 * Requirement: slab width L_x / n >= h, else ab_set_box fails with AB_E_BOX.
 * In both modes every rank passes the same GLOBAL arrays to ab_set_atoms / ab_set_positions /
 * ab_set_velocities and receives complete global arrays from ab_get_* (gathered over ranks);
 * energies, virial and counters are sums over all ranks.
 *
 * ab_create_dist: one process per GPU.  All ranks call it collectively with the same 128-byte
 * NCCL unique id (from ab_nccl_unique_id on one rank, broadcast by the caller); an id is
 * single-use (NCCL's bootstrap root serves one communicator), so each engine needs a fresh one.  The halo and
 * force exchanges are ncclSend / ncclRecv between slab neighbours on the engine's stream, the
 * rebuild decision and results are NCCL all-reduces; libnccl.so.2 is loaded at run time.
 * Every call on a distributed engine is collective (all ranks, same order).  ab_get_list
 * returns the rows of this rank's owned atoms only.  Errors: AB_E_NCCL (library or comm).
 *
 * ab_create_virtual: nranks slab domains driven by one handle on one GPU, exchanging the halo by
 * device-to-device copies (the same decomposition code; only the transport differs).  Used to
 * check the decomposition against the whole-box engine and the oracle on a single GPU. */
ab_status ab_nccl_unique_id(void* id128 /* out: 128 bytes */);
ab_status ab_create_dist(const char* param_text, size_t len, ab_precision prec, int cuda_device, int rank,
                         int nranks, const void* id128, ab_engine** out);
ab_status ab_create_virtual(const char* param_text, size_t len, ab_precision prec, int cuda_device, int nranks,
                            ab_engine** out);
/* Host-only slab geometry (no GPU needed): bounds [xlo, xhi) of slab `rank`, and AB_E_BOX if the
 * slab width L[0]/nranks is below `halo`; ab_slab_of: owning slab of coordinate x (wrapped into
 * [0, Lx) first), -1 on bad arguments. */
ab_status ab_slab_info(const double L[3], double halo, int nranks, int rank, double* xlo, double* xhi);
int ab_slab_of(double x, double Lx, int nranks);

void ab_destroy(ab_engine* e);
/* Text of the last error on this engine (or of the last failed ab_create if e == NULL). */
const char* ab_last_error(const ab_engine* e);

/* Use an external CUDA stream (cudaStream_t passed as void*; NULL = the engine's own stream,
 * which is non-blocking: pass cudaStreamLegacy ((void*)1) to order with the legacy default
 * stream) for every subsequent kernel and copy.  The caller keeps ownership of the stream.
 * Independent force kernels fork onto two engine-owned streams and join back before the call's
 * last operation on this stream, so events recorded on it bracket all of the engine's work. */
ab_status ab_set_stream(ab_engine* e, void* cuda_stream);

/* Orthorhombic periodic box, edge lengths L[3] in Angstrom (periodic in x, y, z).  Any edge
 * length > 0 is allowed (images are explicit).  AB_E_BOX if an edge <= 0. */
ab_status ab_set_box(ab_engine* e, const double L[3]);

/* Atoms: n >= 1, type[n] (0 = C, 1 = H), xyz[n*3].  Positions should lie in [0, L); they are
 * wrapped with x - L floor(x/L) otherwise.  Velocities are reset to zero.  Triggers a list build
 * at the next compute. */
ab_status ab_set_atoms(ab_engine* e, int64_t n, const int32_t* type, const double* xyz);
/* New positions for the same n atoms (caller order).  Lists are rebuilt only if some atom moved
 * more than skin/2 since the last build.  A non-finite coordinate fails with
 * AB_E_NONFINITE before anything is copied (engine state unchanged). */
ab_status ab_set_positions(ab_engine* e, const double* xyz);
ab_status ab_set_velocities(ab_engine* e, const double* v /* n*3, Angstrom/fs */);

/* One force evaluation at the current positions.  Outputs (each may be NULL):
 *   f[n*3]     forces, eV/Angstrom, caller order
 *   energy     total potential energy E_REBO + E_TORS + E_LJ, eV
 *   virial[6]  W = sum x (x) F over all terms: xx yy zz xy xz yz, eV (= -dE/d strain)
 *   terms[3]   E_REBO, E_TORS, E_LJ, eV */
ab_status ab_compute(ab_engine* e, double* f, double* energy, double virial[6], double terms[3]);

/* Advance nsteps velocity-Verlet NVE steps of dt_fs: v += dt/2 F/m; x += dt v;
 * (rebuild lists if any atom moved > skin/2); F = F(x); v += dt/2 F/m.  If thermo != NULL and
 * thermo_every > 0 it receives rows (step, PE, KE, Etot) for steps 0, every, 2 every, ... <= nsteps
 * (nsteps/thermo_every + 1 rows, 4 doubles each).  The call returns once the last step is
 * enqueued on the engine's stream (it synchronises once per step on the rebuild decision only);
 * every call that returns data orders after it.  Internally the last step's second half-kick
 * and its energy / counter reduction may be left pending (applied by the next step's drift
 * kernel, or by the next call that reads or replaces velocities, positions, forces, energies or
 * counters); no call can observe the difference. */
ab_status ab_run_nve(ab_engine* e, int64_t nsteps, double dt_fs, int64_t thermo_every, double* thermo);

ab_status ab_get_positions(ab_engine* e, double* xyz);  /* caller order; not re-wrapped between rebuilds */
ab_status ab_get_velocities(ab_engine* e, double* v);
ab_status ab_get_forces(ab_engine* e, double* f);       /* forces of the last evaluation */

/* Lists of the current positions as rows (i, j, sx, sy, sz), i and j caller indices, s the image
 * of j (position x_j + s L), sorted lexicographically.  rows == NULL: *count = number of rows. */
ab_status ab_get_list(ab_engine* e, ab_list which, int64_t* count, int64_t* rows);

/* Order-independent digest of the same row set, for lists too large to return as rows (the LJ
 * half list of a 2 M-atom system has ~7e8 rows; the bit-exact list comparison of BASELINE's
 * north star at full size, SURVEY reading A26).  With mix(z) = splitmix64's finaliser
 *   z += 0x9e3779b97f4a7c15; z = (z ^ z>>30) * 0xbf58476d1ce4e5b9; z = (z ^ z>>27) * 0x94d049bb133111eb;
 *   mix = z ^ z>>31
 * each row hashes to h = mix(((u64)(u32)i << 32 | (u32)j) ^ mix((sx+128) << 16 | (sy+128) << 8 | (sz+128))),
 * and digest = {number of rows, sum of h mod 2^64, xor of h}.  Output: digest[3] (caller-owned).
 * Errors as ab_get_list. */
ab_status ab_get_list_digest(ab_engine* e, ab_list which, uint64_t digest[3]);

ab_status ab_get_stats(ab_engine* e, ab_stats* s);

/* Stage outputs of the last evaluation for stage-wise parity.  Rows in no particular
 * order, each starting with (i, j, sx, sy, sz) as doubles (caller indices, image of j):
 *   stage 0: per REBO half bond: + b, p_ij, p_ji, pi_rc, pi_dh, N_ij, N_ji, N_conj  (13 doubles)
 *   stage 1: per LJ half pair with r <= r_c: + C_ij, b* (0 if not evaluated)          (7 doubles)
 * Stage recording costs extra memory traffic; it is enabled by ab_record_stages(e, 1).
 * out == NULL: *count = number of rows. */
ab_status ab_record_stages(ab_engine* e, int on);
ab_status ab_get_stage(ab_engine* e, int stage, int64_t* count, double* out);

/* Per-phase device timing with CUDA events on the engine's stream (the paper's profile labels,
 * P:359-360): phase 0 short list + N_i, 1 REBO + bond order + torsion, 2 LJ pairs +
 * C_ij reach sets (the near pairs; every pair with AB_LJ_CLUSTER=1), 3 b* batch,
 * 4 integrator, 5 list rebuild, 6 LJ far pairs (none with AB_LJ_CLUSTER=1), 7 slab transfers
 * (halo positions, ghost forces, migration; multi-domain engines only).
 * ab_get_phase_ms returns accumulated milliseconds ms[AB_NPHASE] and launch counts n[AB_NPHASE]
 * since profiling was switched on (on != 0 resets them). */
#define AB_NPHASE 8
ab_status ab_set_profiling(ab_engine* e, int on);
ab_status ab_get_phase_ms(ab_engine* e, double ms[AB_NPHASE], int64_t n[AB_NPHASE]);

/* Kernel concurrency inside one force evaluation (default on): the far-LJ kernel and the REBO
 * kernel run on two engine-owned streams beside the near-LJ -> b* chain.  on = 0 runs the whole
 * evaluation on the engine stream, one kernel at a time (isolated per-kernel timing; the
 * environment variable AB_SERIAL_KERNELS=1 sets the default at ab_create).  Results are the same
 * up to the order of fp64 atomic additions. */
ab_status ab_set_concurrency(ab_engine* e, int on);

/* FP64 (prec = AB_FP64) or FP32 (AB_MIXED) FMA-throughput microbenchmark on the engine's GPU:
 * all SMs, 8 independent FMA chains per thread; returns the achieved TFLOP/s (2 flops per FMA).
 * Used as the measured ALU roofline denominator by bench.py. */
ab_status ab_peak_flops(ab_engine* e, ab_precision prec, double* tflops);

/* Device id / name of the engine's GPU; launches of the engine's own kernels since creation. */
ab_status ab_device_info(ab_engine* e, int* device, char* name, size_t name_len, int64_t* kernel_launches);

#ifdef __cplusplus
}
#endif
#endif /* AIREBO_B200_H */
