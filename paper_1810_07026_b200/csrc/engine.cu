// engine.cu -- the C-ABI (include/airebo_b200.h) and host orchestration of the B200 AIREBO engine.
//
// One translation unit (unity build) so the __constant__ parameter tables are visible to every
// kernel.  Per force evaluation, on one stream: exact short list + N_i (k_short) -> REBO + bond
// order + torsion per bond (k_rebo) -> C_ij reach set + LJ per atom (k_lj) -> deferred b* batch
// (k_bstar).  List rebuilds (binning, ghosts, skinned lists) happen when an atom moved more than
// skin/2.  No CPU fallback: every step of the path is a kernel below.
//
// Domains.  An engine handle drives one or more spatial domains:
//   * single GPU, whole box (nranks == 1): the handle is the domain; ghosts are periodic images;
//   * NCCL rank r of n (ab_create_dist): the handle is slab r; the halo travels with ncclSend /
//     ncclRecv on the engine stream, ghost forces come back the same way;
//   * n virtual slabs on one GPU (ab_create_virtual): the handle owns n domain engines (subs) and
//     the halo travels by device-to-device copies on the shared stream.  Every phase is enqueued
//     for all domains by the host in order, so no kernel ever waits on another domain's kernel.
// Only the transfer (xfer) differs between the last two; the slab logic is the same code.
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is dlopen'ed by the distributed mode

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <map>

#include "../../include/airebo_b200.h"
#include "dev_common.cuh"
#include "k_bond.cuh"
#include "k_dist.cuh"
#include "k_lists.cuh"
#include "k_lj.cuh"
#include "k_ljc.cuh"
#include "k_misc.cuh"
#include "k_scan.cuh"
#include "params.h"

using namespace ab;

namespace {

std::string g_create_error;

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  // allocates with 25 % slack: atom / ghost / list counts drift between list rebuilds, and a
  // reallocation inside the NVE loop (cudaFree synchronises the device, large cudaMalloc maps
  // pages) costs tens of milliseconds -- measured 77 ms for the first in-loop rebuild of cfg2
  cudaError_t ensure(size_t cnt) {
    if (cnt <= n && p) return cudaSuccess;
    size_t c = std::max<size_t>(cnt + cnt / 4, 1);
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, c * sizeof(T));
    if (e == cudaSuccess) n = c;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// at least one block: every kernel bounds-checks, and an empty domain must still launch cleanly
inline int nblk(long long n, int t) { return (int)std::max<long long>(1, (n + t - 1) / t); }

constexpr size_t SCRATCH_BYTES = 1024, SCRATCH_CT = 128, SCRATCH_SMALL = 512, SCRATCH_ZERO_BYTES = 512 + 96;
constexpr size_t SCRATCH_TICKET = 1016;
// bits of the max displacement^2 of any local atom since the last build (atomicMax by the drift /
// displacement kernels, zeroed at every build; never in the zeroed region): the far-LJ kernel's bins
constexpr size_t SCRATCH_DBOUND = 1000;
// max reach-set size seen by k_lj_near since the last build (atomicMax; read + zeroed at each build)
constexpr size_t SCRATCH_MAXREACH = 992;
#ifndef AB_INT_BLOCK
#define AB_INT_BLOCK 128  // k_integrate1_img block (measured cfg2: 128 beats 256; 64 / 32 equal)
#endif  // k_integrate1_img's last-block ticket (never memset after init)

// ---- NCCL, resolved at run time (only the distributed mode needs it)
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl(std::string& err) {
  static NcclApi api;
  static bool tried = false;
  static std::string why;
  if (!tried) {
    tried = true;
    const char* env = std::getenv("AB_NCCL_LIB");
    void* h = nullptr;
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = std::string("cannot load libnccl.so.2: ") + dlerror();
    } else {
      bool all = true;
      auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        if (!fp) all = false;
      };
      sym(api.getUniqueId, "ncclGetUniqueId");
      sym(api.commInitRank, "ncclCommInitRank");
      sym(api.commDestroy, "ncclCommDestroy");
      sym(api.groupStart, "ncclGroupStart");
      sym(api.groupEnd, "ncclGroupEnd");
      sym(api.send, "ncclSend");
      sym(api.recv, "ncclRecv");
      sym(api.allReduce, "ncclAllReduce");
      sym(api.errStr, "ncclGetErrorString");
      api.ok = all;
      if (!all) why = "libnccl.so.2 lacks a required symbol";
    }
  }
  if (!api.ok) err = why;
  return api;
}

}  // namespace

struct ab_engine {
  std::string err;
  HostParams hp;
  Tab<double> td;
  Tab<float> tf;
  ab_precision prec = AB_FP64;
  int dev = 0;
  char devname[256] = {0};
  int nsm = 148;
  cudaStream_t own = nullptr, st = nullptr;
  cudaStream_t aux[2] = {nullptr, nullptr};     // concurrent force kernels (REBO, LJ far)
  cudaStream_t chain = nullptr;                  // AB_PRIO 3rd value: the short -> near -> b* chain's own stream
  cudaEvent_t ev_chain[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork[2] = {nullptr, nullptr}, ev_join[2] = {nullptr, nullptr};
  bool serial = false;  // AB_SERIAL_KERNELS=1: the whole DAG on one stream (isolated kernel timing)
  bool have_box = false, have_atoms = false, lists_valid = false, forces_valid = false;
  bool record = false;
  double L[3] = {0, 0, 0};
  int N = 0, NT = 0, G = 0;
  int NX = 0;  // locals + x-ghosts (== N on a whole-box domain); image ghosts follow
  double halo = 0, rcmax = 0, rmaxmax = 0;
  Grid grid{};
  int ncell = 0, nrLJ = 1, nrI = 1;
  int capI = 0, capS = 0, capQ = 0;
  int far_at = 0;
  bool pdl = false;  // AB_PDL=1: programmatic dependent launch of the b* kernels
  bool rebo_g4 = false;  // AB_REBO_G4=1: the sp3 C-C batch 4 lanes per bond (k_rebo_g4; measured slower)
  int skip = 0;  // AB_SKIP bit mask (timing ablations only, results wrong): 1 REBO, 2 far, 4 near, 8 b*  // enqueue_forces: fork point of the far-LJ kernel (AB_FAR_AT)
  // NVE steps: the reduction of the partial rows is fused into the second half-kick (k_post)
  bool defer_reduce = false, post_pending = false;
  // the last NVE step's partial rows, reduced only if energies / counters are read before the
  // next evaluation overwrites them (collect); NVE steps without a thermo row skip the reduction
  bool reduce_lazy = false;
  // whole-box NVE: the second half-kick of a step without a thermo row is deferred and applied by
  // the next step's drift kernel (v += dtf_prev F; v += dtf F, the two roundings of the separate
  // kernels), or by flush_kick before anything reads / replaces v or F (ab_get_velocities, ...)
  bool kick_pending = false;
  double kick_dtf[2] = {0, 0};
  RedRows lazy_rr{};
  int lazy_rows = 0;
  // set by k_integrate1_img (whole-box NVE): the image ghosts are current and F is zero
  bool ghosts_fresh = false, f_zeroed = false, scratch_zeroed = false;
  RedRows post_rr{};
  int post_rows = 0;
  int qcap[3] = {0, 0, 0}, qoff[3] = {0, 0, 0};  // b* candidate queue regions (build-time bounds)
  // slab domains, halo / interior overlap: the cell-sorted locals [far_i0, far_i1)
  // whose LJ stencil lies inside the slab (no x-ghost partner until the next rebuild), the
  // images of locals [NX, NX + G_loc) (the rest are images of x-ghosts); far_early: this step's
  // far-LJ kernel for the interior atoms was launched beside the halo exchange
  int far_i0 = 0, far_i1 = 0, G_loc = 0;
  bool far_early = false;
  long long launches = 0, rebuilds = 0, steps = 0, retries = 0;
  // device state
  DBuf<double4> pos, pos_tmp, xref, spos;  // spos: positions in the cell-sorted order (list builds)
  DBuf<double> vel, vel_tmp, F, io;
  DBuf<float> Ff;  // AB_SINGLE: fp32 force accumulation array of an evaluation
  DBuf<int> gid, gid_tmp, owner, key, val, val2, cell_start, gcnt, goff;
  DBuf<char4> shift, rshift;
  DBuf<signed char> typ;
  DBuf<int> ljc[3], ljn[3], in_cnt, in_nbr;  // LJ near / far / (unused) lists, intermediate list
  DBuf<unsigned short> ljboff;               // far-row bin ends (k_lists.cuh FB_*)
  DBuf<int> smq;                             // k_lj_far per-SM queue counters (AB_FAR_SMQ)
  int capL[3] = {0, 0, 0};
  // j-cluster LJ path (k_cluster.cuh, k_ljc.cuh), AB_LJ_CLUSTER=1; default: per-atom near / far lists
  bool cl_path = false;
  ClGrid clg{};
  int nrun = 0, NCL = 0, capC = 0;
  DBuf<int> cl_k, cl_v, cl_v2, run_start, run_cl, cl_atom, clc, cln;
  DBuf<double4> cpos, cbb;
  bool want_virial = true;
  int near_slots = 64;      // k_lj_near reach-table size (32 while the reach sets stay <= 20 images)
  bool want_energy = true;  // false: an NVE step whose energies / counters nobody reads (far LJ forces only)
  DBuf<int> s_cnt, s_nbr;
  DBuf<unsigned char> s_dr, s_w, s_N;  // typed by precision at use
  DBuf<double> s_wd;                   // fp64 switch weights of the short list (C_ij gate)
  DBuf<int2> bonds;
  DBuf<int4> q_item;
  DBuf<int> ovf_bond, ovf_q, ovf_q2;  // overflow (large side / full b*) index lists
  DBuf<int> ovf_mid;                  // CH / HH bonds with two non-empty sides (general REBO kernel)
  DBuf<int> ovf_und;                  // b* candidates the plateau batch hands to the forward-pass kernel
  DBuf<double> q_M;
  // one small device scratch block, zeroed with a single memset per evaluation:
  //   acc (ACC_N doubles) at 0, ct (CT_N + 1 u64; [CT_N] = max displacement^2) at 128,
  //   small_i (16 ints: nbonds, qcount, list maxima x4, stage counts x2, overflow counts x2,
  //   b* queue counts x3 at 13..15) at 512
  DBuf<unsigned char> scratch;
  DBuf<int> small_i;
  DBuf<double> acc;
  DBuf<unsigned long long> ct;
  bool host_stale = false;  // acc / ct of the last evaluation not yet copied to the host
  cudaEvent_t ev_disp = nullptr;
  DBuf<double> stage0, stage1, red_d;
  DBuf<unsigned long long> red_u;
  DBuf<int> sc_bsum, sc_cur, sc_off;  // scan / counting-sort scratch (k_scan.cuh)
  // pinned host mirror for small readbacks
  unsigned long long* h_ct = nullptr;
  unsigned long long* h_ct_dev = nullptr;  // h_ct as seen by kernels (mapped pinned memory)
  double* h_acc = nullptr;
  int* h_small = nullptr;
  // results of the last evaluation (whole system: summed over domains / ranks)
  double E3[3] = {0, 0, 0}, W6[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long last_ct[CT_N] = {0};
  // per-phase CUDA-event profiling (ab_set_profiling)
  bool prof = false;
  // AB_TIMELINE=1 (with profiling on): per-phase start / end offsets from the start of each
  // evaluation, averaged and printed at close (the concurrent DAG's timeline)
  bool timeline = false;
  cudaEvent_t tl_ref = nullptr;      // start of the current evaluation
  std::vector<cudaEvent_t> tl_refs;  // the pending evaluations' start events (back to the pool)
  double tl_sum[10][2] = {};  // 0..7 = phases, 8 = first half-kick + drift, 9 = k_post
  long long tl_n[10] = {};
  int tl_sub = -1;            // timeline slot of the next prof_begin (-1: the phase's own)
  double tl_period = 0;       // sum of start-to-start times of consecutive evaluations
  long long tl_np = 0;
  double phase_ms[AB_NPHASE] = {0};
  long long phase_n[AB_NPHASE] = {0};
  struct Pend {
    int phase;
    cudaEvent_t a, b, ref;  // ref: the evaluation's start (AB_TIMELINE), not owned
    int tl;                 // timeline slot
  };
  std::vector<Pend> pending;
  std::vector<cudaEvent_t> pool;
  int open_phase = -1;
  cudaEvent_t open_ev = nullptr;
  // ---- slab decomposition; nranks == 1: whole box
  int rank = 0, nranks = 1;
  int Nglob = 0;                     // atoms of the whole system (caller arrays)
  double xlo = 0, xhi = 0;           // owned slab [xlo, xhi) along x
  std::vector<ab_engine*> subs;      // virtual mode: the domains driven by this handle
  ab_engine* root = nullptr;         // a sub's handle
  ncclComm_t comm = nullptr;         // NCCL mode
  int ns[2] = {0, 0}, nr[2] = {0, 0};  // halo atoms sent to / ghosts received from (left, right)
  DBuf<int> sendl[2];                // local indices of the halo atoms per channel
  DBuf<unsigned char> sb[2], rb[2];  // transfer buffers per channel
  size_t xs[2] = {0, 0}, xr[2] = {0, 0};  // bytes of the next transfer
  DBuf<int> fl[3], idx[3];           // selection scratch (flags, selected indices)
  DBuf<int> cnt_d;                   // selection counts (device)
  DBuf<unsigned char> redx;          // all-reduce staging
  DBuf<double> gio;                  // caller-order global array (3 Nglob) of a handle
  DBuf<unsigned char> gtab;          // global copies of the spline tables (Tab::gRT / gP / gG)
  // CUDA graph of one NVE force evaluation (ghost refresh + the kernel DAG), captured after a list
  // build and replayed every step until the next one (single-domain engines)
  cudaGraphExec_t gexec = nullptr;
  long long graph_launches = 0;  // kernel launches per replay
  long long graph_epoch = -1;    // layout version the graph was captured at
  long long layout = 0;          // bumped whenever buffers / capacities / kernel choices change
  double disp1 = -1.0, disp2 = -1.0;  // max displacement since the last build at the last two steps
  unsigned long long* h_flag = nullptr;  // pinned: the D2H of the reduced flags must not block the host
  double* h_th = nullptr;  // pinned staging of thermo rows
  size_t h_th_cap = 0;
  // host-side time breakdown of the NVE loop (AB_HOST_TIMING=1: printed by ab_destroy)
  double host_ms[6] = {0, 0, 0, 0, 0, 0};  // integrate1+flags, speculative enqueue, wait, rebuild path, integrate2
  long long host_steps = 0;
  double rb_ms[4] = {0, 0, 0, 0};  // rebuild: sort, image count (sync), image fill + binning, lists (sync)
  long long rb_n = 0;
};

namespace {

const ab_engine* g_const_owner = nullptr;  // whose box / tables the __constant__ banks hold

std::vector<ab_engine*> doms(ab_engine* e) {
  if (e->subs.empty()) return {e};
  return e->subs;
}
inline bool slabbed(const ab_engine* e) { return e->nranks > 1; }

cudaEvent_t ev_get(ab_engine* e) {
  if (!e->pool.empty()) {
    cudaEvent_t x = e->pool.back();
    e->pool.pop_back();
    return x;
  }
  cudaEvent_t x;
  cudaEventCreate(&x);
  return x;
}
// phase timing with events on the stream the phase runs on (phases may overlap on different
// streams); prof_start returns nullptr when profiling is off
cudaEvent_t prof_start(ab_engine* e, cudaStream_t s) {
  if (!e->prof) return nullptr;
  cudaEvent_t a = ev_get(e);
  cudaEventRecord(a, s);
  return a;
}
void prof_stop(ab_engine* e, int phase, cudaStream_t s, cudaEvent_t a) {
  if (!a) return;
  cudaEvent_t b = ev_get(e);
  cudaEventRecord(b, s);
  e->pending.push_back({phase, a, b, e->tl_ref, e->tl_sub >= 0 ? e->tl_sub : phase});
  e->tl_sub = -1;
}
void prof_begin(ab_engine* e, int phase) {
  e->open_phase = phase;
  e->open_ev = prof_start(e, e->st);
}
void prof_end(ab_engine* e) {
  prof_stop(e, e->open_phase, e->st, e->open_ev);
  e->open_ev = nullptr;
}
// call after a stream synchronisation
void prof_collect(ab_engine* e) {
  for (auto& p : e->pending) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      e->phase_ms[p.phase] += ms;
      e->phase_n[p.phase] += 1;
    }
    float t0 = 0, t1 = 0;
    if (e->timeline && p.ref && cudaEventElapsedTime(&t0, p.ref, p.a) == cudaSuccess &&
        cudaEventElapsedTime(&t1, p.ref, p.b) == cudaSuccess && t0 >= 0) {
      e->tl_sum[p.tl][0] += t0, e->tl_sum[p.tl][1] += t1, e->tl_n[p.tl] += 1;
    }
    e->pool.push_back(p.a);
    e->pool.push_back(p.b);
  }
  for (size_t q = 1; q < e->tl_refs.size(); ++q) {
    float dt = 0;
    if (cudaEventElapsedTime(&dt, e->tl_refs[q - 1], e->tl_refs[q]) == cudaSuccess) e->tl_period += dt, ++e->tl_np;
  }
  for (cudaEvent_t r : e->tl_refs) e->pool.push_back(r);
  e->tl_refs.clear();
  e->pending.clear();
}

template <typename T>
__global__ void k_fma_peak(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = (T)(threadIdx.x + c) * (T)1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == (T)12345.678) out[threadIdx.x] = s;  // keeps the chains alive
}
}  // namespace

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      e->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call;       \
      return e_ == cudaErrorMemoryAllocation ? AB_E_OOM : AB_E_CUDA;                      \
    }                                                                                     \
  } while (0)
// AB_DEBUG_SYNC=1 (diagnostics only): synchronise after every launch and name the source line
static bool debug_sync() {
  static int v = -1;
  if (v < 0) v = std::getenv("AB_DEBUG_SYNC") && std::getenv("AB_DEBUG_SYNC")[0] == '1';
  return v == 1;
}
#define CKL()                                                                             \
  do {                                                                                    \
    ++e->launches;                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ == cudaSuccess && debug_sync()) e_ = cudaDeviceSynchronize();                  \
    if (e_ != cudaSuccess) {                                                              \
      e->err = std::string("CUDA launch error: ") + cudaGetErrorString(e_) + " (engine.cu:" + std::to_string(__LINE__) + ")"; \
      return AB_E_CUDA;                                                                   \
    }                                                                                     \
  } while (0)
#define TRY(x)                   \
  do {                           \
    ab_status s_ = (x);          \
    if (s_ != AB_OK) return s_;  \
  } while (0)
// per-domain call from a handle-level function: the domain's error text moves to the handle
#define TRYD(d, x)                         \
  do {                                     \
    ab_status s_ = (x);                    \
    if (s_ != AB_OK) {                     \
      if ((d) != e) e->err = (d)->err;     \
      return s_;                           \
    }                                      \
  } while (0)
#define CKN(call)                                                                         \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess) {                                                              \
      e->err = std::string("NCCL error: ") + NC.errStr(r_) + " at " #call;                \
      return AB_E_NCCL;                                                                   \
    }                                                                                     \
  } while (0)

namespace {

template <typename R>
void fill_tab(const HostParams& hp, Tab<R>& t) {
  for (int p = 0; p < 3; ++p) {
    const PairSet& s = hp.pr[p];
    t.rmin[p] = (R)s.rmin, t.rmax[p] = (R)s.rmax, t.Q[p] = (R)s.Q, t.alpha[p] = (R)s.alpha, t.A[p] = (R)s.A;
    for (int n = 0; n < 3; ++n) t.B[p][n] = (R)s.B[n], t.beta[p][n] = (R)s.beta[n];
    t.eps[p] = (R)s.eps, t.sigma[p] = (R)s.sigma, t.sigma2[p] = (R)(s.sigma * s.sigma), t.rc[p] = (R)s.rc;
    t.rlo[p] = (R)s.rlo, t.bmin[p] = (R)s.bmin, t.bmax[p] = (R)s.bmax, t.rho[p] = (R)s.rho;
    t.srhi[p] = (R)(s.sigma * 1.122462048309373);  // 2^(1/6) sigma (reading A11)
    t.inv_taper[p] = (R)(1.0 / (s.rc - s.rlo));
    t.lj_e4[p] = (R)(4.0 * s.eps), t.lj_c12[p] = (R)(48.0 * s.eps), t.lj_c6[p] = (R)(24.0 * s.eps);
  }
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i)
      for (int k = 0; k < 2; ++k) t.explam[j][i][k] = (R)std::exp(hp.lam[j][i][k]);
  for (int c = 0; c < 3; ++c) {  // g_C, g_H, g_C2 (slot 2 = g_C when angle.C2 is absent)
    const std::vector<double>& kn = c < 2 ? hp.gknot[c] : (hp.gknot2.empty() ? hp.gknot[0] : hp.gknot2);
    const std::vector<double>& va = c < 2 ? hp.gval[c] : (hp.gknot2.empty() ? hp.gval[0] : hp.gval2);
    int n = (int)kn.size();
    t.gn[c] = n;
    for (int q = 0; q < 16; ++q) t.gx[c][q] = t.gy[c][q] = t.gm[c][q] = 0;
    for (int q = 0; q < n; ++q) {
      t.gx[c][q] = (R)kn[q];
      t.gy[c][q] = (R)va[q];
      double m = (q == 0 || q == n - 1) ? 0.0 : (va[q + 1] - va[q - 1]) / (kn[q + 1] - kn[q - 1]);
      t.gm[c][q] = (R)m;
    }
  }
  t.kappa = (R)hp.kappa;
  t.rhoH[0] = (R)hp.pr[1].rho, t.rhoH[1] = (R)hp.pr[2].rho;  // rho_{CH}, rho_{HH}
  t.g2on = hp.gknot2.empty() ? 0 : 1;
  t.gnlo = (R)hp.gnlo, t.gnhi = (R)hp.gnhi;
  // f = sum_abc phi_a phi_b phi_c F_abc with sum phi = 1 and sum |phi| <= (1 + 8/27)^3 per point
  // (1-D Hermite weights: h00 + h01 = 1, |h10|, |h11| <= 4/27), so f lies within [min F - k dF,
  // max F + k dF], k = ((35/27)^3 - 1) / 2, dF = max F - min F
  const double ko = (std::pow(35.0 / 27.0, 3) - 1.0) / 2.0;
  for (int p = 0; p < 3; ++p)
    for (int w = 0; w < 2; ++w) {
      const std::vector<double>& tab = w == 0 ? hp.Rtab[p] : hp.Ttab[p];
      const double mn = *std::min_element(tab.begin(), tab.end()), mx = *std::max_element(tab.begin(), tab.end());
      const double lo = mn - ko * (mx - mn), hi = mx + ko * (mx - mn);
      (w == 0 ? t.bRlo : t.bTlo)[p] = (R)lo, (w == 0 ? t.bRhi : t.bThi)[p] = (R)hi;
    }
  for (int a = 0; a < 2; ++a)
    for (int q = 0; q < 25; ++q) t.P[a][q] = (R)hp.Ptab[a][q];
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 225; ++q) t.Rt[p][q] = (R)hp.Rtab[p][q], t.Tt[p][q] = (R)hp.Ttab[p][q];
  t.conj_lo = (R)hp.conj_lo, t.conj_hi = (R)hp.conj_hi, t.s2lo = (R)hp.sin2_lo, t.s2hi = (R)hp.sin2_hi;
  for (int k = 0; k < 2; ++k)
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int l = 0; l < 2; ++l)  // REBO has no torsion term
          t.tors[k][i][j][l] = hp.potential == kREBO ? R(0) : (R)hp.tors[k][i][j][l];
  for (int p = 0; p < 3; ++p)
    t.meps[p] = (R)hp.pr[p].meps, t.malpha[p] = (R)hp.pr[p].malpha, t.mre[p] = (R)hp.pr[p].mre;
}

// host-side geometry of the engine (cutoffs, halo); no device work
void geo_fields(ab_engine* e) {
  double rmm = 0, rcm = 0;
  for (int p = 0; p < 3; ++p) rmm = std::max(rmm, e->hp.pr[p].rmax), rcm = std::max(rcm, e->hp.pr[p].rc);
  e->rmaxmax = rmm;
  e->rcmax = rcm;
  e->halo = rcm + e->hp.skin;  // LJ cutoff + skin covers every REBO/torsion/C_ij/b* reach
}

// The __constant__ banks (box, cutoffs, parameter tables) are per process: (re)load them when a
// different handle than the last one launches kernels (several engines may live in one process).
ab_status bind_consts(ab_engine* e) {
  const ab_engine* owner = e->root ? e->root : e;
  if (g_const_owner == owner) return AB_OK;
  Geo g;
  const HostParams& hp = e->hp;
  double rmm = 0;
  for (int p = 0; p < 3; ++p) {
    const PairSet& s = hp.pr[p];
    g.rmax2[p] = s.rmax * s.rmax;
    g.rc2[p] = s.rc * s.rc;
    g.rmax_s2[p] = (s.rmax + hp.skin) * (s.rmax + hp.skin);
    g.rc_s2[p] = (s.rc + hp.skin) * (s.rc + hp.skin);
    g.rlo2[p] = s.rlo * s.rlo;
    g.tv2[p] = g.rlo2[p] * (1.0 - 1e-9);
    double srhi = s.sigma * 1.122462048309373;
    g.srhi2_hi[p] = srhi * srhi * (1.0 + 1e-9);
    rmm = std::max(rmm, s.rmax);
  }
  g.reach2 = (3 * rmm) * (3 * rmm);
  for (int c = 0; c < 3; ++c) g.L[c] = e->L[c];
  g.mass[0] = hp.mass[0], g.mass[1] = hp.mass[1], g.ftm2v = hp.ftm2v, g.mvv2e = hp.mvv2e;
  g.potential = hp.potential;
  // the banks are process-wide: kernels of the previous owner (or of this engine, after a box
  // change) may still be in flight on other streams -- rewrite them only when the device is idle
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyToSymbolAsync(c_geo, &g, sizeof(Geo), 0, cudaMemcpyHostToDevice, e->st));
  CK(cudaMemcpyToSymbolAsync(c_tabd, &e->td, sizeof(e->td), 0, cudaMemcpyHostToDevice, e->st));
  CK(cudaMemcpyToSymbolAsync(c_tabf, &e->tf, sizeof(e->tf), 0, cudaMemcpyHostToDevice, e->st));
  g_const_owner = owner;
  return AB_OK;
}

template <typename R>
ShortList<R> short_view(ab_engine* e) {
  ShortList<R> S;
  S.capS = e->capS;
  S.cnt = e->s_cnt.p;
  S.nbr = e->s_nbr.p;
  S.dr = reinterpret_cast<decltype(S.dr)>(e->s_dr.p);
  S.w = reinterpret_cast<decltype(S.w)>(e->s_w.p);
  S.wd = e->s_wd.p;
  R* base = reinterpret_cast<R*>(e->s_N.p);
  S.Ntot = base;
  S.NC = base + e->NT;
  S.NH = base + 2 * (size_t)e->NT;
  return S;
}

size_t real_size(const ab_engine* e) { return e->prec == AB_FP64 ? 8 : 4; }

ab_status ensure_short(ab_engine* e) {
  size_t rs = real_size(e);
  size_t ent = (size_t)e->NT * e->capS;
  CK(e->s_cnt.ensure(e->NT));
  CK(e->s_nbr.ensure(ent));
  CK(e->s_dr.ensure(ent * 4 * rs));
  CK(e->s_w.ensure(ent * 2 * rs));
  CK(e->s_wd.ensure(ent));
  CK(e->s_N.ensure((size_t)e->NT * 3 * rs));
  CK(e->bonds.ensure(3 * ((size_t)e->N * e->capS + 1)));
  return AB_OK;
}

// grow a position / index array to cap entries keeping the first keep entries
template <class T>
ab_status grow_keep(ab_engine* e, DBuf<T>& b, size_t cap, size_t keep) {
  if (b.n >= cap && b.p) return AB_OK;
  DBuf<T> nb;
  CK(nb.ensure(cap + cap / 8));
  keep = b.p ? std::min(keep, b.n) : 0;
  if (keep) CK(cudaMemcpyAsync(nb.p, b.p, sizeof(T) * keep, cudaMemcpyDeviceToDevice, e->st));
  CK(cudaStreamSynchronize(e->st));
  b.release();
  b = nb;
  return AB_OK;
}

// exclusive scan of in[0..n) (FLAG: of in[q] != 0) into out[0..n], out[n] = total (k_scan.cuh)
template <bool FLAG>
ab_status scan_ex(ab_engine* e, const int* in, int n, int* out) {
  const int nb = std::max(1, (n + SCAN_E - 1) / SCAN_E);
  CK(e->sc_bsum.ensure(nb + 1));
  k_scan_blocks<FLAG><<<nb, SCAN_T, 0, e->st>>>(in, n, out, e->sc_bsum.p);
  CKL();
  k_scan_carry<<<1, SCAN_T, 0, e->st>>>(nb, e->sc_bsum.p);
  CKL();
  k_scan_add<<<nblk(n + 1, 256), 256, 0, e->st>>>(n, nb, e->sc_bsum.p, out);
  CKL();
  return AB_OK;
}

// stable index selection: out = indices q < n with flag[q] != 0 (in order), count at *num
ab_status select_flagged(ab_engine* e, int n, const int* flags, int* out, int* num) {
  CK(e->sc_off.ensure((size_t)n + 1));
  TRY(scan_ex<true>(e, flags, n, e->sc_off.p));
  k_select_scatter<<<nblk(n, 256), 256, 0, e->st>>>(n, flags, e->sc_off.p, out, num);
  CKL();
  return AB_OK;
}

// stable counting sort of [0, n) by key[a] in [0, nkey): perm = indices ordered by (key, sec[a] if
// sec != nullptr, a); start[0..nkey] = first position of each key (k_scan.cuh)
ab_status key_sort(ab_engine* e, int n, const int* key, int nkey, const int* sec, int* perm, int* start) {
  CK(e->sc_cur.ensure((size_t)nkey + 1));
  CK(cudaMemsetAsync(e->sc_cur.p, 0, sizeof(int) * (size_t)nkey, e->st));
  k_cell_hist<<<nblk(n, 256), 256, 0, e->st>>>(n, key, e->sc_cur.p);
  CKL();
  TRY(scan_ex<false>(e, e->sc_cur.p, nkey, start));
  CK(cudaMemcpyAsync(e->sc_cur.p, start, sizeof(int) * (size_t)nkey, cudaMemcpyDeviceToDevice, e->st));
  k_cell_scatter<<<nblk(n, 256), 256, 0, e->st>>>(n, key, e->sc_cur.p, perm);
  CKL();
  k_cell_order<<<nblk(nkey, 128), 128, 0, e->st>>>(nkey, start, sec, perm);
  CKL();
  return AB_OK;
}

// ---------------------------------------------------------------- transfer between domains
// Channel 0 goes to / comes from the left neighbour (rank - 1), channel 1 the right one (rank + 1),
// periodic.  Each domain sends sb[c] (xs[c] bytes) and receives rb[c] (xr[c] bytes); what the
// left neighbour sends on its channel 1 arrives in my rb[0] and vice versa.  NCCL order per
// rank: send(left) recv(right) send(right) recv(left) -- with two ranks (left == right) the pairs
// match in issue order: my first send lands in the peer's first receive (its rb[1]).
ab_status xfer_impl(ab_engine* e);
// every transfer is timed as phase 7 (halo exchange / reverse communication, SURVEY §8(d):
// "communication time per step") when profiling is on
ab_status xfer(ab_engine* e) {
  if (!slabbed(e)) return AB_OK;
  cudaEvent_t t = prof_start(e, e->st);
  ab_status s = xfer_impl(e);
  prof_stop(e, 7, e->st, t);
  return s;
}
ab_status xfer_impl(ab_engine* e) {
  if (!e->subs.empty()) {
    const int n = (int)e->subs.size();
    for (int r = 0; r < n; ++r) {
      ab_engine* d = e->subs[r];
      ab_engine* left = e->subs[(r + n - 1) % n];
      ab_engine* right = e->subs[(r + 1) % n];
      if (d->xr[0] != left->xs[1] || d->xr[1] != right->xs[0]) {
        e->err = "internal: halo transfer sizes disagree between domains";
        return AB_E_STATE;
      }
      if (d->xr[0]) CK(cudaMemcpyAsync(d->rb[0].p, left->sb[1].p, d->xr[0], cudaMemcpyDeviceToDevice, e->st));
      if (d->xr[1]) CK(cudaMemcpyAsync(d->rb[1].p, right->sb[0].p, d->xr[1], cudaMemcpyDeviceToDevice, e->st));
    }
    return AB_OK;
  }
  NcclApi& NC = nccl(e->err);
  if (!NC.ok || !e->comm) return AB_E_NCCL;
  const int left = (e->rank + e->nranks - 1) % e->nranks, right = (e->rank + 1) % e->nranks;
  CKN(NC.groupStart());
  if (e->xs[0]) CKN(NC.send(e->sb[0].p, e->xs[0], ncclUint8, left, e->comm, e->st));
  if (e->xr[1]) CKN(NC.recv(e->rb[1].p, e->xr[1], ncclUint8, right, e->comm, e->st));
  if (e->xs[1]) CKN(NC.send(e->sb[1].p, e->xs[1], ncclUint8, right, e->comm, e->st));
  if (e->xr[0]) CKN(NC.recv(e->rb[0].p, e->xr[0], ncclUint8, left, e->comm, e->st));
  CKN(NC.groupEnd());
  return AB_OK;
}

ab_status ensure_xbufs(ab_engine* e, size_t s0, size_t s1, size_t r0, size_t r1) {
  CK(e->sb[0].ensure(s0 + 16));
  CK(e->sb[1].ensure(s1 + 16));
  CK(e->rb[0].ensure(r0 + 16));
  CK(e->rb[1].ensure(r1 + 16));
  e->xs[0] = s0, e->xs[1] = s1, e->xr[0] = r0, e->xr[1] = r1;
  return AB_OK;
}

// image shift of the ghosts received on a channel (periodic wrap across x = 0 / x = L)
inline int chan_sx(const ab_engine* d, int c) {
  if (c == 0) return d->rank == 0 ? -1 : 0;
  return d->rank == d->nranks - 1 ? 1 : 0;
}

// ---------------------------------------------------------------- list build
void setup_grid(ab_engine* e) {
  const double h = e->halo;
  // cell grid over the padded region: edge >= (r_c,max + skin)/3 >= r_max + skin
  double cs_t = std::max((e->rcmax + e->hp.skin) / 3.0, e->rmaxmax + e->hp.skin);
  double csmin = 1e300;
  for (int c = 0; c < 3; ++c) {
    double lo = -h, span = e->L[c] + 2 * h;
    if (c == 0 && slabbed(e)) lo = e->xlo - h, span = (e->xhi - e->xlo) + 2 * h;
    e->grid.nc[c] = std::max(1, (int)std::floor(span / cs_t));
    e->grid.cs[c] = span / e->grid.nc[c];
    e->grid.lo[c] = lo;
    csmin = std::min(csmin, e->grid.cs[c]);
  }
  e->ncell = e->grid.nc[0] * e->grid.nc[1] * e->grid.nc[2];
  e->nrLJ = (int)std::ceil((e->rcmax + e->hp.skin) / csmin);
  e->nrI = (int)std::ceil((e->rmaxmax + e->hp.skin) / csmin);
}

// wrap + spatial sort of the local atoms (pos, vel, gid permuted together)
ab_status sort_locals(ab_engine* e) {
  const int N = e->N;
  cudaStream_t st = e->st;
  CK(e->key.ensure(N));
  CK(e->val.ensure(N));
  CK(e->val2.ensure(N));
  CK(e->cell_start.ensure((size_t)e->ncell + 1));
  CK(e->pos_tmp.ensure(N));
  CK(e->vel_tmp.ensure(3 * (size_t)N));
  CK(e->gid_tmp.ensure(N));
  k_wrap_and_key<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->grid, e->key.p, e->val.p);
  CKL();
  TRY(key_sort(e, N, e->key.p, e->ncell, nullptr, e->val2.p, e->cell_start.p));  // stable by (cell, index)
  e->far_i0 = e->far_i1 = 0;
  if (slabbed(e) && N) {  // interior x-columns: cells whose +-nrLJ x-stencil lies inside [xlo, xhi)
    const Grid& g = e->grid;
    int c0 = 0, c1 = g.nc[0] - 1;
    while (c0 < g.nc[0] && g.lo[0] + c0 * g.cs[0] < e->xlo) ++c0;
    while (c1 >= 0 && g.lo[0] + (c1 + 1) * g.cs[0] > e->xhi) --c1;
    const int a = c0 + e->nrLJ, b = c1 - e->nrLJ;  // cell x-range of the interior atoms
    if (a <= b) {
      const int plane = g.nc[1] * g.nc[2];  // keys are x-major: an x-range is a contiguous range
      int ab[2];
      CK(cudaMemcpyAsync(&ab[0], e->cell_start.p + (size_t)a * plane, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&ab[1], e->cell_start.p + (size_t)(b + 1) * plane, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      e->far_i0 = ab[0], e->far_i1 = ab[1];
    }
  }
  k_permute<<<nblk(N, 256), 256, 0, st>>>(N, e->val2.p, e->pos.p, e->pos_tmp.p, e->vel.p, e->vel_tmp.p, e->gid.p,
                                          e->gid_tmp.p);
  CKL();
  if (N) {
    CK(cudaMemcpyAsync(e->pos.p, e->pos_tmp.p, sizeof(double4) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(e->vel.p, e->vel_tmp.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(e->gid.p, e->gid_tmp.p, sizeof(int) * N, cudaMemcpyDeviceToDevice, st));
  }
  return AB_OK;
}

// j-clusters of all atoms (locals + ghosts) for the LJ pair loop (k_cluster.cuh): columns of
// ~2.5 A over the padded region, runs by (column, species), z-sorted, chopped into groups of 4
ab_status build_clusters(ab_engine* e) {
  const int NT = e->NT;
  cudaStream_t st = e->st;
  ClGrid& g = e->clg;
  double span[3];
  for (int c = 0; c < 3; ++c) g.lo[c] = e->grid.lo[c], span[c] = e->grid.nc[c] * e->grid.cs[c];
  double cw = 2.5;
  if (const char* v = std::getenv("AB_CL_COL")) cw = std::max(1.0, std::atof(v));
  const double Rm = e->rcmax + e->hp.skin;
  auto nside = [&](double w) { return 2 * ((int)std::ceil(Rm / w) + 1) + 1; };
  while (std::floor(span[0] / cw) * std::floor(span[1] / cw) * 2 > CL_RUNS_MAX ||
         2 * nside(cw) * nside(cw) > CL_MAXRUN)
    cw *= 1.05;
  g.ncx = std::max(1, (int)std::floor(span[0] / cw));
  g.ncy = std::max(1, (int)std::floor(span[1] / cw));
  g.cw[0] = span[0] / g.ncx, g.cw[1] = span[1] / g.ncy;
  g.zspan = span[2];
  e->nrun = g.ncx * g.ncy * 2;
  CK(e->cl_k.ensure(NT));
  CK(e->cl_v.ensure(NT));
  CK(e->cl_v2.ensure(NT));
  CK(e->run_start.ensure(e->nrun + 1));
  CK(e->run_cl.ensure(e->nrun + 1));
  k_cl_keys<<<nblk(NT, 256), 256, 0, st>>>(NT, e->pos.p, g, e->cl_k.p, e->cl_v.p);  // run, quantised z
  CKL();
  TRY(key_sort(e, NT, e->cl_k.p, e->nrun, e->cl_v.p, e->cl_v2.p, e->run_start.p));  // by (run, z, index)
  k_cl_run_scan<<<1, 1024, 0, st>>>(e->nrun, e->run_start.p, e->run_cl.p);
  CKL();
  int ncl = 0;
  CK(cudaMemcpyAsync(&ncl, e->run_cl.p + e->nrun, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  e->NCL = ncl;
  CK(e->cl_atom.ensure((size_t)CL_SIZE * ncl + 1));
  CK(e->cpos.ensure((size_t)CL_SIZE * ncl + 1));
  CK(e->cbb.ensure(2 * (size_t)ncl + 1));
  CK(cudaMemsetAsync(e->cl_atom.p, 0xff, sizeof(int) * CL_SIZE * (size_t)ncl, st));
  k_cl_fill<<<nblk(NT, 256), 256, 0, st>>>(NT, e->cl_k.p, e->cl_v2.p, e->run_start.p, e->run_cl.p, e->cl_atom.p);
  CKL();
  k_cl_bbox<<<nblk(ncl, 128), 128, 0, st>>>(ncl, e->cl_atom.p, e->pos.p, e->cbb.p, e->cpos.p);
  CKL();
  return AB_OK;
}

// images of the base atoms [0, NX) + binning of all atoms + skinned lists.  On entry: locals
// sorted at [0, N), x-ghosts (slab domains) at [N, NX) with their bookkeeping set.
ab_status images_and_lists(ab_engine* e) {
  const int N = e->N, NB = e->NX;
  cudaStream_t st = e->st;
  const double h = e->halo;
  // 2. periodic images (ghosts) within the halo: all three directions on a whole-box domain, y/z
  // only on a slab domain (its x halo came from the neighbours)
  int3 smax = make_int3((int)std::ceil(h / e->L[0]), (int)std::ceil(h / e->L[1]), (int)std::ceil(h / e->L[2]));
  double3 lo = make_double3(-h, -h, -h), hi = make_double3(e->L[0] + h, e->L[1] + h, e->L[2] + h);
  if (slabbed(e)) smax.x = 0, lo.x = e->xlo - h, hi.x = e->xhi + h;
  CK(e->gcnt.ensure(NB));
  CK(e->goff.ensure((size_t)NB + 1));
  k_image_count<<<nblk(NB, 256), 256, 0, st>>>(NB, e->pos.p, smax, lo, hi, e->gcnt.p);
  CKL();
  TRY(scan_ex<false>(e, e->gcnt.p, NB, e->goff.p));
  e->G_loc = 0;
  if (slabbed(e) && N < NB) {  // images of the locals come first (k_image_fill order)
    CK(cudaMemcpyAsync(&e->G_loc, e->goff.p + N, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  int tail[2] = {0, 0};
  if (NB) {
    CK(cudaMemcpyAsync(&tail[0], e->goff.p + NB - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&tail[1], e->gcnt.p + NB - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  }
  auto tq = std::chrono::steady_clock::now();
  CK(cudaStreamSynchronize(st));
  auto tms = [](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  e->rb_ms[1] += tms(tq);
  tq = std::chrono::steady_clock::now();
  e->NT = NB + tail[0] + tail[1];
  e->G = e->NT - N;
  if (!(N < NB)) e->G_loc = e->NT - NB;
  const int NT = e->NT;
  TRY(grow_keep(e, e->pos, NT, NB));
  TRY(grow_keep(e, e->gid, NT, NB));
  TRY(grow_keep(e, e->owner, NT, NB));
  TRY(grow_keep(e, e->shift, NT, NB));
  TRY(grow_keep(e, e->rshift, NT, NB));
  CK(e->typ.ensure(NT));
  CK(e->F.ensure(3 * (size_t)NT));
  k_image_fill<<<nblk(NB, 256), 256, 0, st>>>(NB, N, NB, e->pos.p, smax, lo, hi, e->goff.p, e->owner.p, e->gid.p,
                                             e->shift.p, e->rshift.p);
  CKL();
  k_types<<<nblk(NT, 256), 256, 0, st>>>(NT, e->pos.p, e->typ.p);
  CKL();
  // 3. bin all atoms (locals + ghosts)
  CK(e->key.ensure(NT));
  CK(e->val.ensure(NT));
  CK(e->val2.ensure(NT));
  CK(e->cell_start.ensure((size_t)e->ncell + 1));
  k_cell_keys<<<nblk(NT, 256), 256, 0, st>>>(NT, e->pos.p, e->grid, e->key.p, e->val.p);
  CKL();
  TRY(key_sort(e, NT, e->key.p, e->ncell, nullptr, e->val2.p, e->cell_start.p));  // cell list
  CK(e->spos.ensure(NT));
  k_sorted_pos<<<nblk(NT, 256), 256, 0, st>>>(NT, e->val2.p, e->pos.p, e->spos.p);
  CKL();
  const bool clp = e->cl_path && e->hp.potential != kREBO;
  if (clp) TRY(build_clusters(e));
  e->rb_ms[2] += tms(tq);
  tq = std::chrono::steady_clock::now();
  // 4. skinned lists: LJ (local atoms, full) and intermediate REBO (all atoms)
  // cell edge >= (r_c,max + skin)/3 and >= r_max + skin (setup_grid): nrLJ <= 3, nrI <= 1
  if ((2 * e->nrLJ + 1) * (2 * e->nrLJ + 1) > STENCIL_MAXCOL || (2 * e->nrI + 1) * (2 * e->nrI + 1) > STENCIL_MAXCOL)
    return AB_E_STATE;
  CK(e->small_i.ensure(8));
  for (int c = 0; c < 3; ++c) CK(e->ljc[c].ensure(N));
  CK(e->in_cnt.ensure(NT));
  const double skin = e->hp.skin;
  // a_p: radius of the S_r window pre-filter (r^2 < a_p^2 = (2^(1/6) sigma)^2 (1 + 1e-9), c_geo.srhi2_hi)
  double fa[3], amax = 0;
  for (int p = 0; p < 3; ++p) {
    const double srhi = e->hp.pr[p].sigma * 1.122462048309373;
    fa[p] = std::sqrt(srhi * srhi * (1.0 + 1e-9));
    amax = std::max(amax, fa[p]);
  }
  if (e->capL[0] == 0 && e->hp.potential == kREBO) e->capL[0] = e->capL[1] = e->capL[2] = 1;
  if (e->capL[0] == 0) {  // first build: capacities from the mean density (grown on overflow)
    double vol = e->L[0] * e->L[1] * e->L[2];
    if (slabbed(e)) vol = (e->xhi - e->xlo) * e->L[1] * e->L[2];
    double rho = std::max(N, 1) / vol, fpi = 4.18879020478639;
    const double rn = amax + skin, r2 = e->rcmax + skin, r1 = std::max(amax - skin, 0.0);
    e->capL[0] = 32 + (int)(1.3 * rho * fpi * rn * rn * rn);
    e->capL[1] = 32 + (int)(1.3 * rho * fpi * (r2 * r2 * r2 - r1 * r1 * r1));
    e->capL[2] = 1;
  }
  if (e->capI == 0) e->capI = 16;
  if (clp && e->capC == 0) {  // clusters within r_c,max + skin + a cluster extent, 4 slots each
    double vol = e->L[0] * e->L[1] * e->L[2];
    if (slabbed(e)) vol = (e->xhi - e->xlo) * e->L[1] * e->L[2];
    const double rho = std::max(N, 1) / vol, R = e->rcmax + skin + 2.5;
    e->capC = 32 + (int)(1.4 * rho * 4.18879020478639 * R * R * R / CL_SIZE / 0.8);
  }
  LJLists Lg;
  for (int p = 0; p < 3; ++p) {
    // rounding margins (1e-7 A) on the safe side: every pair that can be inside / outside the
    // window before the next build is in the near / far list
    const double lo = fa[p] - skin - 1e-7, hi = fa[p] + skin + 1e-7;
    Lg.flo2[p] = lo > 0 ? lo * lo : 0.0;
    Lg.bq2[p] = hi * hi;
    Lg.fa[p] = fa[p];
    Lg.rlo[p] = e->hp.pr[p].rlo, Lg.rc[p] = e->hp.pr[p].rc, Lg.rc2[p] = Lg.rc[p] * Lg.rc[p];
  }
  Lg.skin = skin;
  Lg.ih2 = skin > 0 ? 4.0 / skin : 0.0, Lg.ih8 = skin > 0 ? 8.0 / skin : 0.0;
  Lg.bqcnt = e->small_i.p + 6;
  Lg.reach = (e->rcmax + skin) * (1.0 + 1e-9) + 1e-9;
  for (int t = 0; t < 2; ++t)  // per species of the atom: its largest LJ cutoff (C: CC / CH, H: CH / HH) + skin
    Lg.reach_t[t] = (std::max(e->hp.pr[t].rc, e->hp.pr[t + 1].rc) + skin) * (1.0 + 1e-9) + 1e-9;
  for (int attempt = 0; attempt < 4; ++attempt) {
    for (int c = 0; c < 3; ++c) {
      if (!clp) CK(e->ljn[c].ensure((size_t)N * e->capL[c]));
      Lg.cap[c] = e->capL[c];
      Lg.cnt[c] = e->ljc[c].p;
      Lg.nbr[c] = e->ljn[c].p;
    }
    if (!clp) CK(e->ljboff.ensure((size_t)N * FB_STRIDE));
    Lg.boff = e->ljboff.p;
    Lg.fcap_smem = e->capL[1];
    CK(e->in_nbr.ensure((size_t)NT * e->capI));
    CK(cudaMemsetAsync(e->small_i.p + 2, 0, 7 * sizeof(int), st));
    const bool dbg = std::getenv("AB_HOST_TIMING") && std::getenv("AB_HOST_TIMING")[0] == '2';
    cudaEvent_t dbg_ev[3] = {nullptr, nullptr, nullptr};
    if (dbg)
      for (auto& x : dbg_ev) cudaEventCreate(&x), cudaEventRecord(x, st);
    double t_pre = tms(tq);
    if (clp) {
      CK(e->clc.ensure(N));
      CK(e->cln.ensure((size_t)N * e->capC));
      ClLists CLs;
      CLs.cap = e->capC, CLs.cnt = e->clc.p, CLs.nbr = e->cln.p, CLs.bqcnt = Lg.bqcnt;
      for (int p = 0; p < 3; ++p) CLs.rcs[p] = (e->hp.pr[p].rc + skin) * (1.0 + 1e-9) + 1e-9, CLs.bq2[p] = Lg.bq2[p];
      k_build_cl<<<nblk((long long)N * 32, 128), 128, 0, st>>>(N, e->pos.p, e->clg, e->run_cl.p, e->cbb.p,
                                                                e->cl_atom.p, CLs, e->small_i.p + 2);
      CKL();
    } else if (e->hp.potential != kREBO) {  // REBO has no inter-molecular term: no LJ lists
      // far entries staged in shared memory: 4 warps per block, 1 if the rows are very long
      const size_t per_warp = (size_t)((e->capL[1] + 3) / 4) * 5 * sizeof(int);
      const int wpb = per_warp * 4 <= 200 * 1024 ? 4 : 1;
      if (per_warp * wpb > 200 * 1024) {
        e->err = "LJ far list longer than the shared-memory staging of the list build supports";
        return AB_E_STATE;
      }
      const size_t dyn = per_warp * wpb;
      if (dyn > 48 * 1024) CK(cudaFuncSetAttribute(k_build_lj, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
      k_build_lj<<<nblk((long long)N * 32, 32 * wpb), 32 * wpb, dyn, st>>>(N, e->pos.p, e->spos.p, e->grid,
                                                                            e->cell_start.p, e->val2.p, e->nrLJ, Lg,
                                                                            e->small_i.p + 2);
      CKL();
    } else {
      for (int c = 0; c < 3; ++c)
        if (N) CK(cudaMemsetAsync(e->ljc[c].p, 0, sizeof(int) * N, st));
    }
    k_build_inter<<<nblk((long long)NT * 32, 128), 128, 0, st>>>(NT, e->pos.p, e->spos.p, e->grid, e->cell_start.p, e->val2.p,
                                                                  e->nrI, (e->rmaxmax + skin) * (1.0 + 1e-9) + 1e-9,
                                                                  e->capI, e->in_cnt.p, e->in_nbr.p,
                                                                  e->small_i.p + 5);
    CKL();
    if (dbg) cudaEventRecord(dbg_ev[2], st);
    int mx[7];
    CK(cudaMemcpyAsync(mx, e->small_i.p + 2, 7 * sizeof(int), cudaMemcpyDeviceToHost, st));
    unsigned long long mreach = 0;
    if (attempt == 0) {
      CK(cudaMemcpyAsync(&mreach, e->scratch.p + SCRATCH_MAXREACH, sizeof(mreach), cudaMemcpyDeviceToHost, st));
      CK(cudaMemsetAsync(e->scratch.p + SCRATCH_MAXREACH, 0, sizeof(mreach), st));
    }
    auto tw = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(st));
    // the next interval's reach-table size (AB_NEAR_SLOTS_FIXED=64: always 64, diagnostics / tests)
    const bool fixed64 = std::getenv("AB_NEAR_SLOTS_FIXED") && std::atoi(std::getenv("AB_NEAR_SLOTS_FIXED")) == 64;
    if (mreach && !fixed64) e->near_slots = mreach <= 20 ? 32 : 64;
    if (dbg) {
      float k1 = 0;
      cudaEventElapsedTime(&k1, dbg_ev[1], dbg_ev[2]);
      std::fprintf(stderr, "[airebo_b200] rebuild lists: host before kernels %.3f ms, build kernels %.3f ms, sync wait %.3f ms\n",
                   t_pre, k1, tms(tw));
      for (auto& x : dbg_ev) cudaEventDestroy(x);
    }
    bool ok = true;
    if (clp) {
      if (mx[0] > e->capC) e->capC = mx[0] + mx[0] / 8 + 32, ok = false;
    } else {
      for (int c = 0; c < 3; ++c)
        if (mx[c] > e->capL[c]) e->capL[c] = mx[c] + mx[c] / 8 + 32, ok = false;
    }
    if (mx[3] > e->capI) e->capI = mx[3] + 4, ok = false;
    if (ok) {
      int off = 0;
      for (int t = 0; t < 3; ++t) e->qcap[t] = mx[4 + t] + 64, e->qoff[t] = off, off += e->qcap[t];
      e->capQ = off;
      CK(e->q_item.ensure(e->capQ));
      CK(e->q_M.ensure(e->capQ));
      break;
    }
    ++e->retries;
  }
  e->capS = std::min(e->capI, 32);
  auto te = std::chrono::steady_clock::now();
  TRY(ensure_short(e));
  if (std::getenv("AB_HOST_TIMING") && std::getenv("AB_HOST_TIMING")[0] == '2')
    std::fprintf(stderr, "[airebo_b200] rebuild ensure_short %.3f ms\n", tms(te));
  e->rb_ms[3] += tms(tq);
  CK(e->xref.ensure(N));
  k_copy_xref<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->xref.p);
  CKL();
  CK(cudaMemsetAsync(e->scratch.p + SCRATCH_DBOUND, 0, sizeof(unsigned long long), st));
  e->lists_valid = true;
  ++e->rebuilds;
  return AB_OK;
}

// ---- slab rebuild phases (per domain; the handle transfers between them)
// M1: wrap, classify, select stayers / leavers; leaver counts into sb[c]
ab_status mig_select(ab_engine* e) {
  const int N = e->N;
  cudaStream_t st = e->st;
  for (int c = 0; c < 3; ++c) {
    CK(e->fl[c].ensure(N));
    CK(e->idx[c].ensure(N));
  }
  CK(e->cnt_d.ensure(8));
  TRY(ensure_xbufs(e, 4, 4, 4, 4));
  CK(cudaMemsetAsync(e->cnt_d.p, 0, 8 * sizeof(int), st));
  k_wrap<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p);
  CKL();
  k_mig_flags<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->nranks, e->rank, e->fl[0].p, e->fl[1].p, e->fl[2].p,
                                            reinterpret_cast<unsigned long long*>(e->cnt_d.p + 4));
  CKL();
  TRY(select_flagged(e, N, e->fl[0].p, e->idx[0].p, e->cnt_d.p));
  TRY(select_flagged(e, N, e->fl[1].p, e->idx[1].p, reinterpret_cast<int*>(e->sb[0].p)));
  TRY(select_flagged(e, N, e->fl[2].p, e->idx[2].p, reinterpret_cast<int*>(e->sb[1].p)));
  return AB_OK;
}

// M2 (after the count transfer): pack the migrants' records into sb[c]
ab_status mig_pack(ab_engine* e) {
  cudaStream_t st = e->st;
  int h[8];
  int rin[2];
  CK(cudaMemcpyAsync(h, e->cnt_d.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
  int sent[2];
  CK(cudaMemcpyAsync(&sent[0], e->sb[0].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&sent[1], e->sb[1].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&rin[0], e->rb[0].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&rin[1], e->rb[1].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  unsigned long long bad;
  std::memcpy(&bad, &h[4], sizeof(bad));
  if (bad) {
    e->err = "an atom crossed more than one slab between two list builds (rank " + std::to_string(e->rank) + ")";
    return AB_E_STATE;
  }
  e->ns[0] = sent[0], e->ns[1] = sent[1];  // reused as migrant counts until the halo selection
  e->nr[0] = rin[0], e->nr[1] = rin[1];
  e->NX = h[0];                            // stayers
  const size_t rec = 8 * sizeof(double);
  TRY(ensure_xbufs(e, rec * sent[0], rec * sent[1], rec * rin[0], rec * rin[1]));
  for (int c = 0; c < 2; ++c) {
    k_mig_pack<<<nblk(sent[c], 128), 128, 0, st>>>(sent[c], e->idx[1 + c].p, e->pos.p, e->vel.p, e->gid.p,
                                                   reinterpret_cast<double*>(e->sb[c].p));
    CKL();
  }
  return AB_OK;
}

// M3 (after the payload transfer): new local set = stayers + arrivals
ab_status mig_assemble(ab_engine* e) {
  cudaStream_t st = e->st;
  const int nstay = e->NX, n0 = e->nr[0], n1 = e->nr[1];
  const int Nn = nstay + n0 + n1;
  CK(e->pos_tmp.ensure((size_t)Nn + 64));
  CK(e->vel_tmp.ensure(3 * (size_t)Nn + 3));
  CK(e->gid_tmp.ensure((size_t)Nn + 64));
  k_mig_assemble<<<nblk(Nn, 256), 256, 0, st>>>(nstay, e->idx[0].p, e->pos.p, e->vel.p, e->gid.p, n0,
                                                reinterpret_cast<const double*>(e->rb[0].p), n1,
                                                reinterpret_cast<const double*>(e->rb[1].p), e->pos_tmp.p,
                                                e->vel_tmp.p, e->gid_tmp.p);
  CKL();
  // the assembled arrays become the state (no buffer is freed under a pending kernel)
  std::swap(e->pos, e->pos_tmp);
  std::swap(e->vel, e->vel_tmp);
  std::swap(e->gid, e->gid_tmp);
  e->N = Nn;
  CK(e->F.ensure(3 * (size_t)Nn + 3));
  return AB_OK;
}

// H1 (locals sorted): halo send lists, counts into sb[c]
ab_status halo_select(ab_engine* e) {
  const int N = e->N;
  cudaStream_t st = e->st;
  for (int c = 0; c < 2; ++c) {
    CK(e->fl[c].ensure(N));
    CK(e->sendl[c].ensure(N));
  }
  TRY(ensure_xbufs(e, 4, 4, 4, 4));
  k_halo_flags<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->xlo, e->xhi, e->halo, e->fl[0].p, e->fl[1].p);
  CKL();
  for (int c = 0; c < 2; ++c)
    TRY(select_flagged(e, N, e->fl[c].p, e->sendl[c].p, reinterpret_cast<int*>(e->sb[c].p)));
  return AB_OK;
}

// per step (and H2): positions of the halo atoms into sb[c]
ab_status halo_pack(ab_engine* e) {
  TRY(ensure_xbufs(e, 32 * (size_t)e->ns[0], 32 * (size_t)e->ns[1], 32 * (size_t)e->nr[0], 32 * (size_t)e->nr[1]));
  k_halo_pack<<<nblk(e->ns[0] + e->ns[1], 128), 128, 0, e->st>>>(
      e->ns[0], e->sendl[0].p, e->ns[1], e->sendl[1].p, e->pos.p, reinterpret_cast<double4*>(e->sb[0].p),
      reinterpret_cast<double4*>(e->sb[1].p));
  CKL();
  return AB_OK;
}

// H2 (after the count transfer): read the halo sizes, size the ghost slots, pack positions
ab_status halo_size(ab_engine* e) {
  cudaStream_t st = e->st;
  int v[4];
  CK(cudaMemcpyAsync(&v[0], e->sb[0].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&v[1], e->sb[1].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&v[2], e->rb[0].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&v[3], e->rb[1].p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  e->ns[0] = v[0], e->ns[1] = v[1], e->nr[0] = v[2], e->nr[1] = v[3];
  e->NX = e->N + v[2] + v[3];
  return halo_pack(e);
}

// per step: received halo positions into the x-ghost slots
ab_status halo_unpack(ab_engine* e) {
  k_halo_unpack<<<nblk(e->nr[0] + e->nr[1], 128), 128, 0, e->st>>>(
      e->N, e->nr[0], reinterpret_cast<const double4*>(e->rb[0].p), chan_sx(e, 0), e->nr[1],
      reinterpret_cast<const double4*>(e->rb[1].p), chan_sx(e, 1), e->pos.p);
  CKL();
  return AB_OK;
}

// H3 (after the payload transfer): x-ghosts in place, then images, binning and lists
ab_status halo_finish(ab_engine* e) {
  const int NX = e->NX;
  TRY(grow_keep(e, e->pos, (size_t)NX + 64, e->N));
  TRY(grow_keep(e, e->gid, (size_t)NX + 64, e->N));
  TRY(grow_keep(e, e->owner, (size_t)NX + 64, 0));
  TRY(grow_keep(e, e->shift, (size_t)NX + 64, 0));
  TRY(grow_keep(e, e->rshift, (size_t)NX + 64, 0));
  TRY(halo_unpack(e));
  k_xghost_meta<<<nblk(e->nr[0] + e->nr[1], 128), 128, 0, e->st>>>(e->N, e->nr[0], chan_sx(e, 0), e->nr[1],
                                                                   chan_sx(e, 1), e->pos.p, e->owner.p, e->gid.p,
                                                                   e->shift.p, e->rshift.p);
  CKL();
  return images_and_lists(e);
}

ab_status rebuild_all(ab_engine* e) {
  prof_begin(e, 5);
  auto D = doms(e);
  // the rebuild regenerates the images and may reallocate F (F.ensure keeps no contents)
  for (ab_engine* d : D) d->ghosts_fresh = d->scratch_zeroed = d->f_zeroed = false;
  if (!slabbed(e)) {
    auto t0 = std::chrono::steady_clock::now();
    setup_grid(e);
    TRY(sort_locals(e));
    e->rb_ms[0] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    e->NX = e->N;
    TRY(images_and_lists(e));
    ++e->rb_n;
  } else {
    for (ab_engine* d : D) setup_grid(d);
    for (ab_engine* d : D) TRYD(d, mig_select(d));
    TRY(xfer(e));  // migrant counts
    for (ab_engine* d : D) TRYD(d, mig_pack(d));
    TRY(xfer(e));  // migrant records
    for (ab_engine* d : D) TRYD(d, mig_assemble(d));
    for (ab_engine* d : D) TRYD(d, sort_locals(d));
    for (ab_engine* d : D) TRYD(d, halo_select(d));
    TRY(xfer(e));  // halo counts
    for (ab_engine* d : D) TRYD(d, halo_size(d));
    TRY(xfer(e));  // halo positions
    for (ab_engine* d : D) TRYD(d, halo_finish(d));
    if (e != D[0]) ++e->rebuilds;
  }
  e->lists_valid = true;
  ++e->layout;
  prof_end(e);
  return AB_OK;
}

void graph_drop(ab_engine* e) {
  if (e->gexec) cudaGraphExecDestroy(e->gexec);
  e->gexec = nullptr;
  e->graph_epoch = -1;
}

// grid sizes of one force evaluation and the partial-row layout of its reduction:
// short | REBO (CC sp3, one-empty-side, hand-over, NBMAX) | near LJ | far LJ | b* (lite, fast,
// NBMAX, full) | [far LJ of the slab interior, launched beside the halo exchange]
#ifndef AB_LITE_GRID
#define AB_LITE_GRID 6  // blocks per SM of the b* plateau batch (grid-stride; measured 6: 0.33 ms vs 4: 0.43 on cfg4)
#endif
struct Grids {
  int g_short, g_rebo, g_near, g_far, g_bstar, g_lite, g_slow, base;
};
// far-LJ / near-LJ kernel arguments (lists of the last build, displacement bound of the far bins)
LJArgs lj_args(ab_engine* e) {
  LJArgs A;
  A.N = e->N;
  A.pos = e->pos.p;
  A.r0b = 0, A.r0e = e->N, A.r1b = A.r1e = 0;
  for (int c = 0; c < 3; ++c) A.cap[c] = e->capL[c], A.cnt[c] = e->ljc[c].p, A.nbr[c] = e->ljn[c].p;
  A.boff = e->ljboff.p;
  A.xref = e->xref.p;
  // slab domains: halo atoms are displaced by other ranks' steps -- the rebuild invariant (every
  // atom moved <= skin/2) bounds them; whole box: the device-side bound of this engine
  A.dbound = slabbed(e) ? nullptr : reinterpret_cast<const unsigned long long*>(e->scratch.p + SCRATCH_DBOUND);
  A.skin = e->hp.skin;
  A.i2 = e->hp.skin > 0 ? 4.0 / e->hp.skin : 0.0, A.i8 = e->hp.skin > 0 ? 8.0 / e->hp.skin : 0.0;
  bool binned = e->hp.skin > 0.0;
  for (int p = 0; p < 3; ++p) {
    const PairSet& s = e->hp.pr[p];
    const double a = std::sqrt(s.sigma * 1.122462048309373 * s.sigma * 1.122462048309373 * (1.0 + 1e-9));
    binned = binned && a + 2.0 * e->hp.skin + 1e-6 <= s.rlo && s.rlo < s.rc;
  }
  A.binned = binned ? 1 : 0;
  A.maxreach = reinterpret_cast<unsigned long long*>(e->scratch.p + SCRATCH_MAXREACH);
  A.smq = nullptr, A.nq = 0, A.qper = 0;
  return A;
}

Grids grids_of(const ab_engine* e) {
  Grids G;
  const int N = e->N;
  const bool clp = e->cl_path && e->hp.potential != kREBO;
  G.g_short = nblk(e->NT, 128), G.g_rebo = e->nsm * 4;
  G.g_near = clp ? std::min(nblk((long long)N * 32, 128), e->nsm * AB_LJC_MINBLOCKS) : nblk(N, NEAR_ATOMS);
#ifndef AB_FAR_GRID
#define AB_FAR_GRID 32  // blocks per SM of the far-LJ grid (contiguous ranges of ~N / (32 nsm) atoms)
#endif
#if AB_FAR_SMQ
#ifndef AB_FAR_SMQ_BLOCKS
#define AB_FAR_SMQ_BLOCKS AB_FAR_MINBLOCKS
#endif
  // per-SM queues: one resident wave (slab mode keeps the static ranges and their finer grid)
  G.g_far = clp ? 0 : std::min(nblk((long long)N * 32, 128), e->nsm * ((slabbed(e) || AB_FAR_SMQ == 2) ? AB_FAR_GRID : AB_FAR_SMQ_BLOCKS));
#else
  G.g_far = clp ? 0 : std::min(nblk((long long)N * 32, 128), e->nsm * AB_FAR_GRID);
#endif
  G.g_bstar = e->nsm * 4, G.g_lite = e->nsm * AB_LITE_GRID, G.g_slow = e->nsm * 2;
  G.base = G.g_short + 2 * G.g_rebo + 2 * G.g_slow + G.g_near + G.g_far + G.g_lite + G.g_bstar + 2 * G.g_slow;
  return G;
}

// Slab domain, NVE step: the far-LJ pairs of the interior atoms [far_i0, far_i1) need no x-ghost
// (their stencil lies inside the slab) -- launched on aux stream 1 as soon as the images of the
// locals are current, so they run while the halo positions travel (SURVEY §8(e) "overlap
// interior compute with the exchange").  F is zeroed here; enqueue_forces takes the remaining
// atoms.  Off for stage recording, the fp32-accumulation modes, the cluster path and serial runs.
template <typename R>
ab_status launch_far_early_t(ab_engine* e) {
  ab_engine* const d = e;  // (CK reports into e->err)
  const Grids G = grids_of(d);
  const int nrows = G.base + G.g_far;
  CK(d->red_d.ensure((size_t)ACC_N * nrows));
  CK(d->red_u.ensure((size_t)CT_N * nrows));
  if (!d->f_zeroed) CK(cudaMemsetAsync(d->F.p, 0, sizeof(double) * 3 * d->NX, d->st));
  d->f_zeroed = true;  // enqueue_forces must not zero F again
  CK(cudaEventRecord(d->ev_fork[1], d->st));
  CK(cudaStreamWaitEvent(d->aux[1], d->ev_fork[1], 0));
  LJArgs A = lj_args(d);
  A.r0b = d->far_i0, A.r0e = d->far_i1, A.r1b = A.r1e = 0;
  RedRows RR{d->red_d.p, d->red_u.p, nrows, G.base};
  StageBuf sb{nullptr, nullptr, 0};
  auto far = [&](auto kern) {
    kern<<<G.g_far, 128, 0, d->aux[1]>>>(A, d->gid.p, d->shift.p, d->F.p, d->acc.p, d->ct.p, sb, RR);
  };
  const bool morse = d->hp.potential == kAIREBOM;
  if (d->want_virial) morse ? far(k_lj_far<R, true, true, false, true>) : far(k_lj_far<R, true, false, false, true>);
  else if (d->want_energy) morse ? far(k_lj_far<R, false, true, false, true>) : far(k_lj_far<R, false, false, false, true>);
  else morse ? far(k_lj_far<R, false, true, false, true, false>) : far(k_lj_far<R, false, false, false, true, false>);
  ++d->launches;
  CK(cudaGetLastError());
  d->far_early = true;
  return AB_OK;
}
ab_status launch_far_early(ab_engine* d) {
  d->far_early = false;
  const bool ok = d->hp.potential != kREBO && !d->cl_path && !d->record && !d->serial && !(d->skip & 2) &&
                  (d->prec == AB_FP64 || d->prec == AB_MIXED) && d->far_i1 > d->far_i0;
  if (!ok) return AB_OK;
  return d->prec == AB_FP64 ? launch_far_early_t<double>(d) : launch_far_early_t<float>(d);
}

// ghosts follow the owned atoms (every step without a rebuild); early: NVE step of slab domains,
// the interior far-LJ pairs start beside the halo exchange (launch_far_early)
ab_status refresh_ghosts_all(ab_engine* e, bool early = false) {
  auto D = doms(e);
  early = early && slabbed(e) && std::getenv("AB_NO_OVERLAP") == nullptr;
  if (early) {
    for (ab_engine* d : D) {
      if (d->G_loc > 0 && !d->ghosts_fresh) {  // images of the locals first: they need no halo
        k_image_update<<<nblk(d->G_loc, 256), 256, 0, d->st>>>(d->NX, d->NX + d->G_loc, d->pos.p, d->owner.p,
                                                                d->rshift.p);
        ++d->launches;
        CK(cudaGetLastError());
      }
      TRYD(d, launch_far_early(d));
    }
  }
  if (slabbed(e)) {
    for (ab_engine* d : D) TRYD(d, halo_pack(d));
    TRY(xfer(e));
    for (ab_engine* d : D) TRYD(d, halo_unpack(d));
  }
  for (ab_engine* d : D)
    if (d->ghosts_fresh) {
      d->ghosts_fresh = false;
    } else if (d->NT > d->NX) {
      const int first = d->NX + (early ? d->G_loc : 0);  // (early: the locals' images are done)
      if (d->NT > first)
        k_image_update<<<nblk(d->NT - first, 256), 256, 0, d->st>>>(first, d->NT, d->pos.p, d->owner.p, d->rshift.p);
      ++d->launches;
      cudaError_t ce = cudaGetLastError();
      if (ce != cudaSuccess) {
        e->err = std::string("CUDA launch error: ") + cudaGetErrorString(ce);
        return AB_E_CUDA;
      }
    }
  return AB_OK;
}

// ---------------------------------------------------------------- force evaluation
// SG: AB_SINGLE (fp32 accumulation: fp32 force array, fp32 running sums), only with R = float
template <typename R, bool SG = false>
ab_status enqueue_forces(ab_engine* e) {
  const int N = e->N, NT = e->NT;
  cudaStream_t st = e->st;
  if (e->chain && !e->serial) {  // AB_PRIO experiment: the DAG's main branch on its own stream
    CK(cudaEventRecord(e->ev_chain[0], e->st));
    CK(cudaStreamWaitEvent(e->chain, e->ev_chain[0], 0));
    st = e->chain;
  }
  StageBuf sb0{nullptr, nullptr, 0}, sb1{nullptr, nullptr, 0};
  const bool clp = e->cl_path && e->hp.potential != kREBO;
  if (e->record) {
    size_t n0 = (size_t)N * e->capS + 16;
    size_t n1 = (clp ? (size_t)N * e->capC * CL_SIZE : (size_t)N * (e->capL[0] + e->capL[1] + e->capL[2] + NEAR_SLOTS)) + 16;
    CK(e->stage0.ensure(n0 * 13));
    CK(e->stage1.ensure(n1 * 7));
    sb0 = StageBuf{e->stage0.p, e->small_i.p + 6, (int)n0};
    sb1 = StageBuf{e->stage1.p, e->small_i.p + 7, (int)n1};
  }
  if (e->f_zeroed) e->f_zeroed = false;  // zeroed by k_integrate1_img
  else CK(cudaMemsetAsync(e->F.p, 0, sizeof(double) * 3 * e->NX, st));
  // AB_SINGLE: the kernels sum forces into an fp32 array (atomic_add3), widened into F below
  if (e->prof && e->timeline) {
    e->tl_ref = ev_get(e);
    e->tl_refs.push_back(e->tl_ref);
    CK(cudaEventRecord(e->tl_ref, st));
  }
  if (SG) {
    CK(e->Ff.ensure(3 * (size_t)e->NX + 3));
    CK(cudaMemsetAsync(e->Ff.p, 0, sizeof(float) * 3 * e->NX, st));
  }
  double* const Fk = SG ? reinterpret_cast<double*>(e->Ff.p) : e->F.p;
  e->reduce_lazy = false;  // a new evaluation: the previous one's rows are overwritten
  if (e->scratch_zeroed) e->scratch_zeroed = false;  // zeroed by k_integrate1_img's last block
  else CK(cudaMemsetAsync(e->scratch.p, 0, SCRATCH_ZERO_BYTES, st));  // acc, counters, small ints
  ShortList<R> S = short_view<R>(e);
  // grids and the per-block partial rows of the energy / virial / counter reduction
  const Grids GR = grids_of(e);
  const int g_short = GR.g_short, g_rebo = GR.g_rebo, g_near = GR.g_near, g_far = GR.g_far, g_bstar = GR.g_bstar;
  const int g_slow = GR.g_slow;
  // REBO: general NB_FAST kernel on the CC region, one-empty-side kernel on CH / HH, general kernel
  // on the bonds the latter hands over, NBMAX kernel on the large-side overflow
  const int g_rebo_rows = 2 * g_rebo + 2 * g_slow;
  const int nrows = GR.base + (e->far_early ? g_far : 0);  // (+ the early interior far-LJ rows)
  CK(e->ovf_bond.ensure((size_t)N * e->capS + 1));
  CK(e->ovf_mid.ensure((size_t)N * e->capS + 1));
  CK(e->ovf_und.ensure(e->capQ));
  CK(e->ovf_q.ensure(e->capQ));
  CK(e->ovf_q2.ensure(e->capQ));
  CK(e->red_d.ensure((size_t)ACC_N * nrows));
  CK(e->red_u.ensure((size_t)CT_N * nrows));
  RedRows RR{e->red_d.p, e->red_u.p, nrows, 0};
  // Kernel DAG of one evaluation (the 32k-atom kernels each fill only part of the GPU, so the
  // independent ones run concurrently): the far LJ pairs need only the skinned lists and start
  // at once on aux[1]; REBO + torsion (aux[0]) and the near LJ pairs -> b* batch (main stream)
  // need the short list.  Partial rows of the reduction are disjoint per kernel; F takes fp64
  // atomics from all of them.
  const bool serial = e->serial;
  const bool lj = e->hp.potential != kREBO, morse = e->hp.potential == kAIREBOM;
  const int nrows_used = lj ? nrows : g_short + g_rebo_rows;  // REBO: short + bond kernels only
  const cudaStream_t s_rebo = serial ? st : e->aux[0], s_far = serial ? st : e->aux[1];
  const int row_far = g_short + g_rebo_rows + g_near;
  BstarQueue Qu;
  Qu.item = e->q_item.p, Qu.M = e->q_M.p, Qu.count = e->small_i.p + 13;
  for (int t = 0; t < 3; ++t) Qu.cap[t] = e->qcap[t], Qu.off[t] = e->qoff[t];
  const BondList BL{e->bonds.p, e->small_i.p + 10, e->N * e->capS + 1};
  LJArgs A = lj_args(e);
  const bool far_split = e->far_early;  // the interior atoms' far pairs are already running
  if (far_split) A.r0b = 0, A.r0e = e->far_i0, A.r1b = e->far_i1, A.r1e = N;  // the rest of the atoms
  else A.r0b = 0, A.r0e = N, A.r1b = A.r1e = 0;
  e->far_early = false;
  // the far kernel forks from the engine stream at e->far_at: 0 = at once, 1 = after the short
  // list, 2 = after the near kernel (it then fills the GPU beside the b* batch)
  auto launch_far = [&]() -> ab_status {
    if (!lj || clp) return AB_OK;
    CK(cudaEventRecord(e->ev_fork[1], st));
    CK(cudaStreamWaitEvent(s_far, e->ev_fork[1], 0));
    cudaEvent_t t = prof_start(e, s_far);
    RedRows R6 = RR;
    R6.row0 = row_far;
    auto far = [&](auto kern) {
      if (!(e->skip & 2)) kern<<<g_far, 128, 0, s_far>>>(A, e->gid.p, e->shift.p, Fk, e->acc.p, e->ct.p, sb1, R6);
    };
#if AB_FAR_SMQ
    if (!far_split && !slabbed(e) && !(e->skip & 2)) {
      CK(e->smq.ensure((size_t)e->nsm));
      CK(cudaMemsetAsync(e->smq.p, 0, sizeof(int) * e->nsm, s_far));
      A.smq = e->smq.p, A.nq = e->nsm, A.qper = (N + e->nsm - 1) / e->nsm;
    }
#endif
    if (far_split) {
      if (e->want_virial) morse ? far(k_lj_far<R, true, true, SG, true>) : far(k_lj_far<R, true, false, SG, true>);
      else if (e->want_energy) morse ? far(k_lj_far<R, false, true, SG, true>) : far(k_lj_far<R, false, false, SG, true>);
      else morse ? far(k_lj_far<R, false, true, SG, true, false>) : far(k_lj_far<R, false, false, SG, true, false>);
    } else if (e->want_virial) {
      morse ? far(k_lj_far<R, true, true, SG>) : far(k_lj_far<R, true, false, SG>);
    } else {
      if (e->want_energy) morse ? far(k_lj_far<R, false, true, SG>) : far(k_lj_far<R, false, false, SG>);
      else morse ? far(k_lj_far<R, false, true, SG, false, false>) : far(k_lj_far<R, false, false, SG, false, false>);
    }
    CKL();
    prof_stop(e, 6, s_far, t);
    CK(cudaEventRecord(e->ev_join[1], s_far));
    return AB_OK;
  };
  if (e->far_at == 0) TRY(launch_far());
  if (clp) {  // current positions of the cluster slots (locals and ghost images)
    k_cpos<<<nblk((long long)CL_SIZE * e->NCL, 256), 256, 0, st>>>(CL_SIZE * e->NCL, e->cl_atom.p, e->pos.p,
                                                                   e->cpos.p);
    CKL();
  }
  {
    cudaEvent_t t = prof_start(e, st);
    k_short<R><<<g_short, 128, 0, st>>>(N, NT, e->pos.p, e->in_cnt.p, e->in_nbr.p, e->capI, S, e->gid.p,
                                        e->shift.p, BL, e->ct.p, RR);
    CKL();
    prof_stop(e, 0, st, t);
  }
  if (e->far_at == 1) TRY(launch_far());
  CK(cudaEventRecord(e->ev_fork[0], st));
  CK(cudaStreamWaitEvent(s_rebo, e->ev_fork[0], 0));
  {
    cudaEvent_t t = prof_start(e, s_rebo);
    RedRows R1 = RR;
    R1.row0 = g_short;
    int* const nbig = e->small_i.p + 8;  // large-side overflow (NBMAX kernel)
    int* const nmid = e->small_i.p + 0;  // CH / HH bonds with two non-empty sides
    auto rebo = [&](auto three, auto grp, auto fast, auto one, auto slow) {
      if (e->skip & 1) return;
      // CC region: sides of <= 3 neighbours (sp3 carbon) in the 4-lanes-per-bond kernel (or the
      // NB = 3 thread-per-bond kernel), larger ones go on to the general NB_FAST kernel through
      // the same hand-over list as the CH / HH bonds
      if (e->rebo_g4)
        grp<<<g_rebo, 128, 0, s_rebo>>>(BL, 0, e->ovf_mid.p, nmid, S, e->typ.p, e->owner.p, e->gid.p, e->shift.p, Fk,
                                        sb0, R1);
      else
        three<<<g_rebo, 128, 0, s_rebo>>>(BL, nullptr, nullptr, 0, 1, e->ovf_mid.p, nmid, S, e->typ.p, e->owner.p,
                                          e->gid.p, e->shift.p, Fk, sb0, R1);
      R1.row0 += g_rebo;
      one<<<g_rebo, 128, 0, s_rebo>>>(BL, nullptr, nullptr, 1, 3, e->ovf_mid.p, nmid, S, e->typ.p, e->owner.p,
                                      e->gid.p, e->shift.p, Fk, sb0, R1);
      R1.row0 += g_rebo;
      fast<<<g_slow, 128, 0, s_rebo>>>(BL, e->ovf_mid.p, nmid, 0, 0, e->ovf_bond.p, nbig, S, e->typ.p, e->owner.p,
                                       e->gid.p, e->shift.p, Fk, sb0, R1);
      R1.row0 += g_slow;
      slow<<<g_slow, 128, 0, s_rebo>>>(BL, e->ovf_bond.p, nbig, 0, 0, nullptr, nullptr, S, e->typ.p, e->owner.p,
                                       e->gid.p, e->shift.p, Fk, sb0, R1);
    };
    if (e->want_virial)
      rebo(k_rebo<R, 3, true, SG>, k_rebo_g4<R, true, SG>, k_rebo<R, NB_FAST, true, SG>,
           k_rebo<R, NB_FAST, true, SG, 0>, k_rebo<R, NBMAX, true, SG>);
    else
      rebo(k_rebo<R, 3, false, SG>, k_rebo_g4<R, false, SG>, k_rebo<R, NB_FAST, false, SG>,
           k_rebo<R, NB_FAST, false, SG, 0>, k_rebo<R, NBMAX, false, SG>);
    e->launches += 3;  // + the CKL below: four launches
    CKL();
    prof_stop(e, 1, s_rebo, t);
  }
  if (!lj) CK(cudaEventRecord(e->ev_join[0], s_rebo));
  RR.row0 = g_short + g_rebo_rows;
  if (lj) {
    cudaEvent_t t = prof_start(e, st);
    auto near = [&](auto kern) {
      if (!(e->skip & 4)) kern<<<g_near, NEAR_GROUP * NEAR_ATOMS, 0, st>>>(A, S, e->owner.p, e->gid.p, e->shift.p, Fk, e->acc.p,
                                                       e->ct.p, Qu, sb1, RR);
    };
    auto ljc = [&](auto kern) {
      LjcArgs CA;
      CA.N = N, CA.pos = e->pos.p, CA.cpos = e->cpos.p, CA.cl_atom = e->cl_atom.p;
      CA.cap = e->capC, CA.cnt = e->clc.p, CA.nbr = e->cln.p;
      if (!(e->skip & 4))
        kern<<<g_near, 128, 0, st>>>(CA, S, e->owner.p, e->gid.p, e->shift.p, Fk, e->ct.p, Qu, sb1, RR);
    };
    if (clp) {
      if (e->want_virial) morse ? ljc(k_ljc<R, true, true, SG>) : ljc(k_ljc<R, true, false, SG>);
      else morse ? ljc(k_ljc<R, false, true, SG>) : ljc(k_ljc<R, false, false, SG>);
    } else if (e->want_virial) {
      morse ? near(k_lj_near<R, true, true, SG>) : near(k_lj_near<R, true, false, SG>);
    } else {
      if (e->near_slots == 32) morse ? near(k_lj_near<R, false, true, SG, 32>) : near(k_lj_near<R, false, false, SG, 32>);
      else morse ? near(k_lj_near<R, false, true, SG>) : near(k_lj_near<R, false, false, SG>);
    }
    CKL();
    prof_stop(e, 2, st, t);
  }
  if (e->far_at == 2) TRY(launch_far());
  RR.row0 = row_far + g_far;
  if (lj) {
    cudaEvent_t t = prof_start(e, st);
    // forward-only fast path; pairs needing the reverse pass / path forces -> ovf_q (NB_FAST
    // sides, count small_i[9]), pairs with a large side -> ovf_q2 (NBMAX, count small_i[1])
    int* const nund = e->small_i.p + 16;  // plateau batch -> forward-pass kernel
    auto bstar = [&](auto lite, auto fast, auto full, auto big) -> ab_status {
      if (e->skip & 8) return AB_OK;
      lite<<<GR.g_lite, 128, 0, st>>>(Qu, e->ovf_und.p, nund, e->pos.p, S, e->typ.p, e->owner.p, Fk,
                                      sb1.rows != nullptr, RR);
      RR.row0 += GR.g_lite;
      // AB_PDL=1: the fast and full b* kernels are launched as programmatic dependents of the
      // kernel before them on the stream (their CTAs launch while it drains and wait in
      // griddepcontrol.wait); the NBMAX batch then forks after the full kernel
      cudaLaunchAttribute pdl[1];
      pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      pdl[0].val.programmaticStreamSerializationAllowed = 1;
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(g_bstar), lc.blockDim = dim3(128), lc.dynamicSmemBytes = 0, lc.stream = st;
      cudaLaunchConfig_t lf = lc;  // the reverse-pass batch (usually empty): one wave of 2 CTAs / SM
      lf.gridDim = dim3(g_slow);
      lc.attrs = pdl, lc.numAttrs = e->pdl ? 1 : 0;
      CK(cudaLaunchKernelEx(&lc, fast, Qu, (const int*)e->ovf_und.p, (const int*)nund, e->ovf_q.p, e->small_i.p + 9, e->ovf_q2.p,
                            e->small_i.p + 1, (const double4*)e->pos.p, S, (const signed char*)e->typ.p,
                            (const int*)e->owner.p, (const int*)e->gid.p, (const char4*)e->shift.p, Fk, sb1, RR));
      // the two deferred batches are independent: the NBMAX one (few pairs, long threads) runs
      // on aux stream 0 (REBO is done or finishing there) beside the NB_FAST reverse-pass batch
      RedRows Rb = RR;
      Rb.row0 += g_bstar + g_slow;
      auto fork_big = [&]() -> ab_status {
        if (!serial) {
          CK(cudaEventRecord(e->ev_fork[0], st));
          CK(cudaStreamWaitEvent(s_rebo, e->ev_fork[0], 0));
        }
        big<<<g_slow, 128, 0, s_rebo>>>(Qu, e->ovf_q2.p, e->small_i.p + 1, nullptr, nullptr, nullptr, nullptr, e->pos.p, S,
                                        e->typ.p, e->owner.p, e->gid.p, e->shift.p, Fk, sb1, Rb);
        return AB_OK;
      };
      if (!e->pdl) TRY(fork_big());
      RR.row0 += g_bstar;
      CK(cudaLaunchKernelEx(&lf, full, Qu, (const int*)e->ovf_q.p, (const int*)(e->small_i.p + 9), (int*)nullptr,
                            (int*)nullptr, (int*)nullptr,
                            (int*)nullptr, (const double4*)e->pos.p, S, (const signed char*)e->typ.p,
                            (const int*)e->owner.p, (const int*)e->gid.p, (const char4*)e->shift.p, Fk, sb1, RR));
      if (e->pdl) TRY(fork_big());
      return AB_OK;
    };
    if (e->want_virial)
      TRY(bstar(k_bstar_lite<R, true, SG>, k_bstar<R, NB_FAST, false, true, SG>, k_bstar<R, NB_FAST, true, true, SG>,
                k_bstar<R, NBMAX, true, true, SG>));
    else
      TRY(bstar(k_bstar_lite<R, false, SG>, k_bstar<R, NB_FAST, false, false, SG>,
                k_bstar<R, NB_FAST, true, false, SG>, k_bstar<R, NBMAX, true, false, SG>));
    e->launches += 3;  // + the CKL below: four launches
    CKL();
    CK(cudaEventRecord(e->ev_join[0], s_rebo));
    prof_stop(e, 3, st, t);
  }
  CK(cudaStreamWaitEvent(st, e->ev_join[0], 0));
  if (lj && !clp) CK(cudaStreamWaitEvent(st, e->ev_join[1], 0));
  RR.row0 = 0;
  if (e->defer_reduce) {  // NVE step: reduced by k_post together with the second half-kick
    e->post_rr = RR, e->post_rows = nrows_used, e->post_pending = true;
  } else {
    k_reduce<<<ACC_N + CT_N, 256, 0, st>>>(RR, nrows_used, e->acc.p, e->ct.p);
    CKL();
  }
  if (SG) {
    k_widen<<<nblk(3LL * e->NX, 256), 256, 0, st>>>(3 * e->NX, e->Ff.p, e->F.p);
    CKL();
  }
  if (st != e->st) {
    CK(cudaEventRecord(e->ev_chain[1], st));
    CK(cudaStreamWaitEvent(e->st, e->ev_chain[1], 0));
  }
  return AB_OK;
}

ab_status enqueue_forces_any(ab_engine* e) {
  if (e->prec == AB_FP64) return enqueue_forces<double>(e);
  if (e->prec == AB_SINGLE || e->prec == AB_REDUCED) return enqueue_forces<float, true>(e);
  return enqueue_forces<float>(e);
}

// reverse communication: forces on x-ghosts go home and are added to the owned atoms
ab_status force_pack(ab_engine* e) {
  TRY(ensure_xbufs(e, 32 * (size_t)e->nr[0], 32 * (size_t)e->nr[1], 32 * (size_t)e->ns[0], 32 * (size_t)e->ns[1]));
  k_force_pack<<<nblk(e->nr[0] + e->nr[1], 128), 128, 0, e->st>>>(e->N, e->nr[0], e->nr[1], e->F.p,
                                                                  reinterpret_cast<double4*>(e->sb[0].p),
                                                                  reinterpret_cast<double4*>(e->sb[1].p));
  CKL();
  return AB_OK;
}
ab_status force_unpack(ab_engine* e) {
  for (int c = 0; c < 2; ++c) {
    k_force_unpack<<<nblk(e->ns[c], 128), 128, 0, e->st>>>(e->ns[c], e->sendl[c].p,
                                                           reinterpret_cast<const double4*>(e->rb[c].p), e->F.p);
    CKL();
  }
  return AB_OK;
}

ab_status nonfinite_or_ovf(ab_engine* e) {
  if (e->last_ct[CT_OVF_SHORT]) {
    e->err = "an atom has more than 16 REBO short-list neighbours (NBMAX); unsupported geometry";
    return AB_E_STATE;
  }
  if (!std::isfinite(e->E3[0] + e->E3[1] + e->E3[2])) {
    e->err = "non-finite energy";
    return AB_E_NONFINITE;
  }
  return AB_OK;
}

inline bool ct_max_col(int c) { return c == CT_MAXSHORT || c == CT_MAXREACH; }

// energies / virial / counters of the last evaluation, summed over all domains and ranks
// reduce the partial rows an NVE call left unreduced (its last step), before acc / ct are read
ab_status flush_lazy(ab_engine* e) {
  for (ab_engine* d : doms(e))
    if (d->reduce_lazy) {
      k_reduce<<<ACC_N + CT_N, 256, 0, e->st>>>(d->lazy_rr, d->lazy_rows, d->acc.p, d->ct.p);
      CKL();
      d->reduce_lazy = false;
    }
  return AB_OK;
}

// apply a deferred second half-kick (v += dtf F with the forces it belongs to)
ab_status flush_kick(ab_engine* e) {
  for (ab_engine* d : doms(e))
    if (d->kick_pending) {
      d->kick_pending = false;
      k_integrate2<<<nblk(d->N, 256), 256, 0, e->st>>>(d->N, d->pos.p, d->vel.p, d->F.p, d->kick_dtf[0], d->kick_dtf[1],
                                                     d->prec == AB_REDUCED);
      CKL();
    }
  return AB_OK;
}
void drop_kick(ab_engine* e) {  // v is about to be replaced
  for (ab_engine* d : doms(e)) d->kick_pending = false;
}

ab_status collect(ab_engine* e) {
  auto D = doms(e);
  TRY(flush_lazy(e));
  double acc[ACC_N] = {0};
  unsigned long long ct[CT_N] = {0};
  if (e->comm) {
    NcclApi& NC = nccl(e->err);
    if (!NC.ok) return AB_E_NCCL;
    const size_t bd = sizeof(double) * ACC_N, bu = sizeof(unsigned long long) * CT_N;
    CK(e->redx.ensure(bd + 2 * bu));
    unsigned char* x = e->redx.p;
    CK(cudaMemcpyAsync(x, e->acc.p, bd, cudaMemcpyDeviceToDevice, e->st));
    CK(cudaMemcpyAsync(x + bd, e->ct.p, bu, cudaMemcpyDeviceToDevice, e->st));
    CK(cudaMemcpyAsync(x + bd + bu, e->ct.p, bu, cudaMemcpyDeviceToDevice, e->st));
    CKN(NC.groupStart());
    CKN(NC.allReduce(x, x, ACC_N, ncclFloat64, ncclSum, e->comm, e->st));
    CKN(NC.allReduce(x + bd, x + bd, CT_N, ncclUint64, ncclSum, e->comm, e->st));
    CKN(NC.allReduce(x + bd + bu, x + bd + bu, CT_N, ncclUint64, ncclMax, e->comm, e->st));
    CKN(NC.groupEnd());
    unsigned long long mx[CT_N];
    CK(cudaMemcpyAsync(acc, x, bd, cudaMemcpyDeviceToHost, e->st));
    CK(cudaMemcpyAsync(ct, x + bd, bu, cudaMemcpyDeviceToHost, e->st));
    CK(cudaMemcpyAsync(mx, x + bd + bu, bu, cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    for (int c = 0; c < CT_N; ++c)
      if (ct_max_col(c)) ct[c] = mx[c];
  } else {
    for (ab_engine* d : D) {
      CK(cudaMemcpyAsync(d->h_ct, d->ct.p, sizeof(unsigned long long) * CT_N, cudaMemcpyDeviceToHost, e->st));
      CK(cudaMemcpyAsync(d->h_acc, d->acc.p, sizeof(double) * ACC_N, cudaMemcpyDeviceToHost, e->st));
    }
    CK(cudaStreamSynchronize(e->st));
    for (ab_engine* d : D) {  // fixed domain order: deterministic sums
      for (int c = 0; c < ACC_N; ++c) acc[c] += d->h_acc[c];
      for (int c = 0; c < CT_N; ++c) ct[c] = ct_max_col(c) ? std::max(ct[c], d->h_ct[c]) : ct[c] + d->h_ct[c];
    }
  }
  for (ab_engine* d : D) prof_collect(d);
  if (e != D[0]) prof_collect(e);
  std::memcpy(e->last_ct, ct, sizeof(ct));
  for (int c = 0; c < 3; ++c) e->E3[c] = acc[ACC_EREBO + c];
  for (int c = 0; c < 6; ++c) e->W6[c] = acc[ACC_W + c];
  e->host_stale = false;
  return AB_OK;
}

ab_status forces_all(ab_engine* e, bool sync_host = true) {
  auto D = doms(e);
  for (int attempt = 0; attempt < 3; ++attempt) {
    for (ab_engine* d : D) TRYD(d, enqueue_forces_any(d));
    if (slabbed(e)) {
      for (ab_engine* d : D) TRYD(d, force_pack(d));
      TRY(xfer(e));
      for (ab_engine* d : D) TRYD(d, force_unpack(d));
    }
    e->forces_valid = true;
    if (!sync_host) {  // NVE steps: results stay on the device until somebody needs them
      e->host_stale = true;
      return AB_OK;
    }
    TRY(collect(e));
    if (e->last_ct[CT_OVF_QUEUE] && !e->last_ct[CT_OVF_SHORT]) {  // (bound violated) grow the b* queue, redo
      for (ab_engine* d : D) {
        int off = 0;
        for (int t = 0; t < 3; ++t) d->qcap[t] = 2 * d->qcap[t] + 1024, d->qoff[t] = off, off += d->qcap[t];
        d->capQ = off;
        TRYD(d, d->q_item.ensure(d->capQ) == cudaSuccess && d->q_M.ensure(d->capQ) == cudaSuccess ? AB_OK : AB_E_OOM);
        ++d->retries;
      }
      ++e->layout;
      continue;
    }
    break;
  }
  return nonfinite_or_ovf(e);
}

// bring energies / virial / counters of the last (asynchronous) evaluation to the host
ab_status pull_results(ab_engine* e) {
  if (!e->host_stale) return AB_OK;
  TRY(collect(e));
  return nonfinite_or_ovf(e);
}

// max displacement^2 since the last build over all domains / ranks (d2 slot ct[CT_N]) plus the
// short-list overflow flag: enqueue the read-back into e->h_flag (valid after a sync)
ab_status enqueue_flags(ab_engine* e) {
  auto D = doms(e);
  if (e->comm) {
    NcclApi& NC = nccl(e->err);
    if (!NC.ok) return AB_E_NCCL;
    CK(e->redx.ensure(64));
    unsigned long long* f = reinterpret_cast<unsigned long long*>(e->redx.p);
    k_flags2<<<1, 1, 0, e->st>>>(e->ct.p, CT_OVF_SHORT, CT_N, f);
    CKL();
    CKN(NC.allReduce(f, f, 2, ncclUint64, ncclMax, e->comm, e->st));
    CK(cudaMemcpyAsync(e->h_flag, f, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->st));
    return AB_OK;
  }
  for (ab_engine* d : D)
    CK(cudaMemcpyAsync(d->h_ct, d->ct.p, sizeof(unsigned long long) * (CT_N + 1), cudaMemcpyDeviceToHost, e->st));
  return AB_OK;
}
// after the sync: combine into h_flag
void read_flags(ab_engine* e) {
  if (e->comm) return;
  e->h_flag[0] = e->h_flag[1] = 0;
  for (ab_engine* d : doms(e)) {
    e->h_flag[0] = std::max(e->h_flag[0], d->h_ct[CT_N]);
    e->h_flag[1] = std::max(e->h_flag[1], d->h_ct[CT_OVF_SHORT]);
  }
}
double flag_d2(const ab_engine* e) {
  double d2;
  std::memcpy(&d2, &e->h_flag[0], sizeof(d2));
  return d2;
}

// make lists valid for the current positions (rebuild if needed, else move the ghosts)
ab_status prepare_all(ab_engine* e, bool check_disp) {
  if (!e->lists_valid) return rebuild_all(e);
  if (check_disp) {
    for (ab_engine* d : doms(e)) {
      CK(cudaMemsetAsync(d->ct.p + CT_N, 0, sizeof(unsigned long long), e->st));
      k_maxdisp<<<nblk(d->N, 256), 256, 0, e->st>>>(d->N, d->pos.p, d->xref.p, d->ct.p + CT_N,
                                                     reinterpret_cast<unsigned long long*>(d->scratch.p + SCRATCH_DBOUND));
      CKL();
    }
    TRY(enqueue_flags(e));
    CK(cudaStreamSynchronize(e->st));
    read_flags(e);
    double half = 0.5 * e->hp.skin;
    if (flag_d2(e) > half * half) return rebuild_all(e);
  }
  return refresh_ghosts_all(e);
}

bool bad_ptr(ab_engine* e, const void* p, const char* what) {
  if (p) return false;
  e->err = std::string("NULL pointer: ") + what;
  return true;
}

// ---- engine construction (shared by the three modes)
ab_status init_engine(ab_engine* e, const char* text, size_t len, ab_precision prec, int device) {
  std::string perr = parse_host_params(text, len, e->hp);
  if (!perr.empty()) {
    e->err = perr;
    return AB_E_PARAM;
  }
  e->prec = prec;
  e->dev = device;
  cudaDeviceProp prop;
  if (cudaSetDevice(device) != cudaSuccess || cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    e->err = "no CUDA device " + std::to_string(device);
    cudaGetLastError();
    return AB_E_CUDA;
  }
  if (prop.major != 10) {
    e->err = std::string("device is not sm_100 (Blackwell): ") + prop.name;
    return AB_E_CUDA;
  }
  std::snprintf(e->devname, sizeof(e->devname), "%s", prop.name);
  e->nsm = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking) != cudaSuccess) {
    e->err = "cudaStreamCreate failed";
    return AB_E_CUDA;
  }
  e->st = e->own;
  e->serial = std::getenv("AB_SERIAL_KERNELS") && std::getenv("AB_SERIAL_KERNELS")[0] == '1';
  e->timeline = std::getenv("AB_TIMELINE") && std::getenv("AB_TIMELINE")[0] == '1';
  // AB_LJ_CLUSTER=1: the j-cluster LJ kernel (k_ljc.cuh; parity-green, measured 2.3x slower than
  // the per-atom near / far kernels on cfg4) instead of k_lj_near + k_lj_far
  e->cl_path = std::getenv("AB_LJ_CLUSTER") && std::getenv("AB_LJ_CLUSTER")[0] == '1';
  if (const char* fa = std::getenv("AB_FAR_AT")) e->far_at = std::max(0, std::min(2, std::atoi(fa)));
  if (const char* sk = std::getenv("AB_SKIP")) e->skip = std::atoi(sk);
  e->pdl = std::getenv("AB_PDL") && std::getenv("AB_PDL")[0] == '1';
  if (const char* rg = std::getenv("AB_REBO_G4")) e->rebo_g4 = rg[0] != '0';
  // AB_PRIO=<rebo>,<far>: stream priorities of the REBO and far-LJ branches (scheduling
  // experiments; lower = higher priority, clamped to the device range; default 0 = the engine
  // stream's)
  int prio[3] = {0, 0, 1};
  if (const char* pe = std::getenv("AB_PRIO")) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const int nv = std::sscanf(pe, "%d,%d,%d", &prio[0], &prio[1], &prio[2]);
    for (int& q : prio) q = std::max(hi, std::min(lo, q));
    if (nv == 3 &&
        (cudaStreamCreateWithPriority(&e->chain, cudaStreamNonBlocking, prio[2]) != cudaSuccess ||
         cudaEventCreateWithFlags(&e->ev_chain[0], cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&e->ev_chain[1], cudaEventDisableTiming) != cudaSuccess)) {
      e->err = "cudaStreamCreate / cudaEventCreate failed";
      return AB_E_CUDA;
    }
  }
  for (int c = 0; c < 2; ++c)
    if (cudaStreamCreateWithPriority(&e->aux[c], cudaStreamNonBlocking, prio[c]) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_fork[c], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_join[c], cudaEventDisableTiming) != cudaSuccess) {
      e->err = "cudaStreamCreate / cudaEventCreate failed";
      return AB_E_CUDA;
    }
  fill_tab(e->hp, e->td);
  fill_tab(e->hp, e->tf);
  geo_fields(e);
  {  // global-memory spline tables (read through L1 with divergent knot indices)
    const size_t nrt = 2 * 3 * 225, np = 2 * 25, ng = 3 * 3 * 16, nall = nrt + np + ng;
    std::vector<double> hd(nall);
    std::vector<float> hf(nall);
    for (int w = 0; w < 2; ++w)
      for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 225; ++q) hd[(w * 3 + p) * 225 + q] = w == 0 ? e->td.Rt[p][q] : e->td.Tt[p][q];
    for (int a = 0; a < 2; ++a)
      for (int q = 0; q < 25; ++q) hd[nrt + a * 25 + q] = e->td.P[a][q];
    for (int c = 0; c < 3; ++c)
      for (int q = 0; q < 16; ++q) {
        hd[nrt + np + c * 16 + q] = e->td.gx[c][q];
        hd[nrt + np + 48 + c * 16 + q] = e->td.gy[c][q];
        hd[nrt + np + 96 + c * 16 + q] = e->td.gm[c][q];
      }
    for (size_t q = 0; q < nall; ++q) hf[q] = (float)hd[q];
    if (e->gtab.ensure(nall * (sizeof(double) + sizeof(float))) != cudaSuccess ||
        cudaMemcpy(e->gtab.p, hd.data(), nall * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(e->gtab.p + nall * sizeof(double), hf.data(), nall * sizeof(float), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
      e->err = "spline table upload failed";
      return AB_E_CUDA;
    }
    const double* dd = reinterpret_cast<const double*>(e->gtab.p);
    const float* ff = reinterpret_cast<const float*>(e->gtab.p + nall * sizeof(double));
    e->td.gRT = dd, e->td.gP = dd + nrt, e->td.gG = dd + nrt + np;
    e->tf.gRT = ff, e->tf.gP = ff + nrt, e->tf.gG = ff + nrt + np;
  }
  bool ok = e->scratch.ensure(SCRATCH_BYTES) == cudaSuccess &&
            cudaMemset(e->scratch.p, 0, SCRATCH_BYTES) == cudaSuccess &&
            cudaMallocHost(&e->h_ct, sizeof(unsigned long long) * (CT_N + 1)) == cudaSuccess &&
            cudaMallocHost(&e->h_acc, sizeof(double) * ACC_N) == cudaSuccess &&
            cudaMallocHost(&e->h_small, sizeof(int) * 8) == cudaSuccess &&
            cudaMallocHost(&e->h_flag, sizeof(unsigned long long) * 2) == cudaSuccess;
  if (ok) e->h_flag[0] = e->h_flag[1] = 0;
  static_assert(sizeof(double) * ACC_N <= SCRATCH_CT, "scratch layout");
  static_assert(SCRATCH_CT + sizeof(unsigned long long) * (CT_N + 1) <= SCRATCH_SMALL, "scratch layout");
  ok = ok && cudaHostGetDevicePointer((void**)&e->h_ct_dev, e->h_ct, 0) == cudaSuccess;
  if (ok) {  // views into the scratch block (not separately allocated)
    e->acc.p = reinterpret_cast<double*>(e->scratch.p), e->acc.n = ACC_N;
    e->ct.p = reinterpret_cast<unsigned long long*>(e->scratch.p + SCRATCH_CT), e->ct.n = CT_N + 1;
    e->small_i.p = reinterpret_cast<int*>(e->scratch.p + SCRATCH_SMALL), e->small_i.n = 24;
  }
  if (!ok) {
    e->err = std::string("CUDA init failed: ") + cudaGetErrorString(cudaGetLastError());
    return AB_E_CUDA;
  }
  return AB_OK;
}

void free_engine(ab_engine* e) {
  if (!e) return;
  if (e->host_steps && std::getenv("AB_HOST_TIMING"))
    std::fprintf(stderr,
                 "[airebo_b200] host ms/step over %lld NVE steps: integrate1+flags %.4f, speculative enqueue %.4f, "
                 "wait %.4f, rebuild path %.4f, integrate2 %.4f\n",
                 e->host_steps, e->host_ms[0] / e->host_steps, e->host_ms[1] / e->host_steps,
                 e->host_ms[2] / e->host_steps, e->host_ms[3] / e->host_steps, e->host_ms[4] / e->host_steps);
  if (e->timeline) {
    const char* nm[10] = {"short", "rebo", "near", "bstar", "integ", "rebuild", "far", "comm", "integ1", "post"};
    if (e->tl_np)
      std::fprintf(stderr, "[airebo_b200] timeline period %8.1f us between evaluation starts (n %lld)\n",
                   1e3 * e->tl_period / e->tl_np, e->tl_np);
    for (int q = 0; q < 10; ++q)
      if (e->tl_n[q])
        std::fprintf(stderr, "[airebo_b200] timeline %-6s start %8.1f us  end %8.1f us  (n %lld)\n", nm[q],
                     1e3 * e->tl_sum[q][0] / e->tl_n[q], 1e3 * e->tl_sum[q][1] / e->tl_n[q], e->tl_n[q]);
  }
  if (e->rb_n && std::getenv("AB_HOST_TIMING"))
    std::fprintf(stderr, "[airebo_b200] host ms/rebuild over %lld: sort %.3f, image count+sync %.3f, fill+bin %.3f, lists %.3f (retries %lld)\n",
                 e->rb_n, e->rb_ms[0] / e->rb_n, e->rb_ms[1] / e->rb_n, e->rb_ms[2] / e->rb_n, e->rb_ms[3] / e->rb_n,
                 e->retries);
  cudaSetDevice(e->dev);
  if (e->st) cudaStreamSynchronize(e->st);
  for (int c = 0; c < 2; ++c)
    if (e->aux[c]) cudaStreamSynchronize(e->aux[c]);
  for (ab_engine* s : e->subs) free_engine(s);
  e->subs.clear();
  if (g_const_owner == e) g_const_owner = nullptr;
  if (e->gexec) cudaGraphExecDestroy(e->gexec);
  if (e->comm) {
    std::string tmp;
    NcclApi& NC = nccl(tmp);
    if (NC.ok) NC.commDestroy(e->comm);
    e->comm = nullptr;
  }
  DBuf<double4>* b4[] = {&e->pos, &e->pos_tmp, &e->xref, &e->spos, &e->cpos, &e->cbb};
  for (auto* b : b4) b->release();
  e->acc.p = nullptr, e->ct.p = nullptr, e->small_i.p = nullptr;  // views into scratch
  e->scratch.release();
  DBuf<double>* bd[] = {&e->vel, &e->vel_tmp, &e->F, &e->io, &e->q_M, &e->stage0, &e->stage1, &e->gio, &e->s_wd};
  for (auto* b : bd) b->release();
  DBuf<int>* bi[] = {&e->gid, &e->gid_tmp, &e->owner, &e->key, &e->val, &e->val2, &e->cell_start,
                     &e->gcnt, &e->goff, &e->ljc[0], &e->ljc[1], &e->ljc[2], &e->ljn[0], &e->ljn[1],
                     &e->ljn[2], &e->in_cnt, &e->in_nbr, &e->s_cnt, &e->s_nbr, &e->ovf_bond, &e->ovf_mid, &e->ovf_und, &e->ovf_q, &e->ovf_q2,
                     &e->sendl[0], &e->sendl[1], &e->fl[0], &e->fl[1], &e->fl[2], &e->idx[0], &e->idx[1],
                     &e->idx[2], &e->cnt_d, &e->cl_k, &e->cl_v, &e->cl_v2, &e->run_start, &e->sc_bsum, &e->sc_cur, &e->sc_off, &e->run_cl,
                     &e->cl_atom, &e->clc, &e->cln};
  for (auto* b : bi) b->release();
  DBuf<unsigned char>* bu[] = {&e->s_dr, &e->s_w, &e->s_N, &e->gtab, &e->sb[0], &e->sb[1], &e->rb[0], &e->rb[1],
                               &e->redx};
  for (auto* b : bu) b->release();
  e->Ff.release();
  e->ljboff.release();
  e->smq.release();
  e->shift.release();
  e->rshift.release();
  e->typ.release();
  e->bonds.release();
  e->q_item.release();
  e->red_d.release();
  e->red_u.release();
  if (e->h_ct) cudaFreeHost(e->h_ct);
  if (e->h_acc) cudaFreeHost(e->h_acc);
  if (e->h_small) cudaFreeHost(e->h_small);
  if (e->h_flag) cudaFreeHost(e->h_flag);
  if (e->h_th) cudaFreeHost(e->h_th);
  if (e->ev_disp) cudaEventDestroy(e->ev_disp);
  for (auto& p : e->pending) cudaEventDestroy(p.a), cudaEventDestroy(p.b);
  for (auto& x : e->pool) cudaEventDestroy(x);
  for (int c = 0; c < 2; ++c) {
    if (e->aux[c]) cudaStreamDestroy(e->aux[c]);
    if (e->ev_fork[c]) cudaEventDestroy(e->ev_fork[c]);
    if (e->ev_join[c]) cudaEventDestroy(e->ev_join[c]);
  }
  if (e->chain) cudaStreamSynchronize(e->chain), cudaStreamDestroy(e->chain);
  for (cudaEvent_t x : e->ev_chain)
    if (x) cudaEventDestroy(x);
  if (e->own) cudaStreamDestroy(e->own);
  delete e;
}

// host copy of the device wrap (same IEEE operations; host code is built with -ffp-contract=off)
double wrap_host(double x, double L) {
  double y = x - L * std::floor(x / L);
  if (y >= L) y = y - L;
  if (y < 0.0) y = y + L;
  return y;
}

// load one domain with the atoms `sel` of the caller arrays (velocities zero)
ab_status load_domain(ab_engine* e, const std::vector<int64_t>& sel, const int32_t* type, const double* xyz,
                      int64_t nglob) {
  const int64_t n = (int64_t)sel.size();
  std::vector<double4> p(n);
  std::vector<int> g(n);
  for (int64_t q = 0; q < n; ++q) {
    int64_t i = sel[q];
    long long key = make_key((int)i, 0, 0, 0, type[i]);
    double kd;
    std::memcpy(&kd, &key, sizeof(kd));
    p[q] = make_double4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], kd);
    g[q] = (int)i;
  }
  e->N = (int)n;
  e->NT = e->NX = (int)n;
  e->Nglob = (int)nglob;
  CK(e->pos.ensure((size_t)n + n / 4 + 64));
  CK(e->gid.ensure((size_t)n + n / 4 + 64));
  CK(e->vel.ensure(3 * (size_t)n + 3));
  CK(e->F.ensure(3 * (size_t)n + 3));
  if (!e->root) CK(e->io.ensure(3 * (size_t)nglob));  // virtual domains use the handle's array
  if (n) {
    CK(cudaMemcpyAsync(e->pos.p, p.data(), sizeof(double4) * n, cudaMemcpyHostToDevice, e->st));
    CK(cudaMemcpyAsync(e->gid.p, g.data(), sizeof(int) * n, cudaMemcpyHostToDevice, e->st));
    CK(cudaMemsetAsync(e->vel.p, 0, sizeof(double) * 3 * n, e->st));
  }
  CK(cudaStreamSynchronize(e->st));
  e->have_atoms = true;
  e->lists_valid = false;
  e->forces_valid = false;
  e->capL[0] = e->capL[1] = e->capL[2] = e->capI = 0;
  return AB_OK;
}

// caller-order global array <-> domains.  to_caller: which = 0 positions, 1 velocities, 2 forces.
ab_status to_caller(ab_engine* e, int which, double* host) {
  auto D = doms(e);
  const size_t bytes = sizeof(double) * 3 * (size_t)e->Nglob;
  double* buf = nullptr;
  if (!slabbed(e)) {
    buf = e->io.p;
  } else {
    CK(e->gio.ensure(3 * (size_t)e->Nglob));
    buf = e->gio.p;
    if (e->comm) CK(cudaMemsetAsync(buf, 0, bytes, e->st));
  }
  for (ab_engine* d : D) {
    if (which == 0)
      k_scatter_caller_pos<<<nblk(d->N, 256), 256, 0, e->st>>>(d->N, d->gid.p, d->pos.p, buf);
    else
      k_to_caller_vec<<<nblk(d->N, 256), 256, 0, e->st>>>(d->N, d->gid.p, which == 1 ? d->vel.p : d->F.p, buf);
    ++d->launches;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) {
      e->err = std::string("CUDA launch error: ") + cudaGetErrorString(ce);
      return AB_E_CUDA;
    }
  }
  if (e->comm) {  // each entry has exactly one non-zero contributor: the sum is exact
    NcclApi& NC = nccl(e->err);
    if (!NC.ok) return AB_E_NCCL;
    CKN(NC.allReduce(buf, buf, 3 * (size_t)e->Nglob, ncclFloat64, ncclSum, e->comm, e->st));
  }
  CK(cudaMemcpyAsync(host, buf, bytes, cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  return AB_OK;
}

// A host-to-device copy straight from caller memory: from pageable memory cudaMemcpyAsync returns
// once the data is staged, but from page-locked memory the DMA reads the caller's buffer later;
// then wait for the copy, so the caller may reuse the buffer when the call returns (header: the
// library copies every input array and never retains a caller pointer).
static bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  // page-locked and managed memory are both read by the DMA after cudaMemcpyAsync returns
  return a.type != cudaMemoryTypeUnregistered;
}

ab_status from_caller_vel(ab_engine* e, const double* host) {
  auto D = doms(e);
  double* buf = e->io.p;
  if (!e->subs.empty()) {
    CK(e->gio.ensure(3 * (size_t)e->Nglob));
    buf = e->gio.p;
  }
  CK(cudaMemcpyAsync(buf, host, sizeof(double) * 3 * (size_t)e->Nglob, cudaMemcpyHostToDevice, e->st));
  for (ab_engine* d : D) {
    k_from_caller_vec<<<nblk(d->N, 256), 256, 0, e->st>>>(d->N, d->gid.p, buf, d->vel.p);
    ++d->launches;
  }
  CK(cudaGetLastError());
  if (host_pinned(host)) CK(cudaStreamSynchronize(e->st));
  return AB_OK;
}

ab_status set_atoms_impl(ab_engine* e, int64_t n, const int32_t* type, const double* xyz) {
  if (!slabbed(e)) {
    std::vector<int64_t> sel(n);
    for (int64_t i = 0; i < n; ++i) sel[i] = i;
    TRY(load_domain(e, sel, type, xyz, n));
  } else {
    auto D = doms(e);
    std::vector<std::vector<int64_t>> sel(e->nranks);
    for (int64_t i = 0; i < n; ++i) sel[slab_of(wrap_host(xyz[3 * i], e->L[0]), e->nranks, e->L[0])].push_back(i);
    for (ab_engine* d : D) TRYD(d, load_domain(d, sel[d->rank], type, xyz, n));
  }
  e->Nglob = (int)n;
  e->N = slabbed(e) && !e->subs.empty() ? (int)n : e->N;
  e->have_atoms = true;
  e->lists_valid = false;
  e->forces_valid = false;
  if (!e->subs.empty()) e->rebuilds = 0;
  return AB_OK;
}

ab_status check_slab_box(ab_engine* e) {
  if (!slabbed(e)) return AB_OK;
  double w = e->L[0] / e->nranks;
  if (w < e->halo) {
    char b[256];
    std::snprintf(b, sizeof(b), "slab width L_x/n = %.4f A is below the halo width %.4f A (r_c,max + skin) for %d ranks",
                  w, e->halo, e->nranks);
    e->err = b;
    return AB_E_BOX;
  }
  return AB_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

ab_status ab_create(const char* text, size_t len, ab_precision prec, int device, ab_engine** out) {
  if (!text || !out || (prec != AB_FP64 && prec != AB_MIXED && prec != AB_SINGLE && prec != AB_REDUCED)) {
    g_create_error = "ab_create: bad argument";
    return AB_E_ARG;
  }
  *out = nullptr;
  ab_engine* e = new ab_engine();
  ab_status s = init_engine(e, text, len, prec, device);
  if (s != AB_OK) {
    g_create_error = e->err;
    free_engine(e);
    return s;
  }
  *out = e;
  return AB_OK;
}

ab_status ab_create_virtual(const char* text, size_t len, ab_precision prec, int device, int nranks,
                            ab_engine** out) {
  if (!out || nranks < 1 || nranks > 64) {
    g_create_error = "ab_create_virtual: bad argument (nranks in [1, 64])";
    return AB_E_ARG;
  }
  TRY(ab_create(text, len, prec, device, out));
  ab_engine* e = *out;
  if (nranks == 1) return AB_OK;
  e->nranks = nranks;
  for (int r = 0; r < nranks; ++r) {
    ab_engine* d = nullptr;
    ab_status s = ab_create(text, len, prec, device, &d);
    if (s != AB_OK) {
      free_engine(e);
      *out = nullptr;
      return s;
    }
    d->root = e;
    d->rank = r;
    d->nranks = nranks;
    d->st = e->st;
    e->subs.push_back(d);
  }
  return AB_OK;
}

ab_status ab_nccl_unique_id(void* id128) {
  if (!id128) return AB_E_ARG;
  NcclApi& NC = nccl(g_create_error);
  if (!NC.ok) return AB_E_NCCL;
  ncclUniqueId id;
  ncclResult_t r = NC.getUniqueId(&id);
  if (r != ncclSuccess) {
    g_create_error = std::string("ncclGetUniqueId: ") + NC.errStr(r);
    return AB_E_NCCL;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  std::memcpy(id128, &id, 128);
  return AB_OK;
}

ab_status ab_create_dist(const char* text, size_t len, ab_precision prec, int device, int rank, int nranks,
                         const void* id128, ab_engine** out) {
  if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) {
    g_create_error = "ab_create_dist: bad argument";
    return AB_E_ARG;
  }
  TRY(ab_create(text, len, prec, device, out));
  ab_engine* e = *out;
  e->rank = rank;
  e->nranks = nranks;
  if (nranks == 1) return AB_OK;
  NcclApi& NC = nccl(e->err);
  if (!NC.ok) {
    g_create_error = e->err;
    free_engine(e);
    *out = nullptr;
    return AB_E_NCCL;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  ncclResult_t r = NC.commInitRank(&e->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    g_create_error = std::string("ncclCommInitRank: ") + NC.errStr(r);
    e->comm = nullptr;
    free_engine(e);
    *out = nullptr;
    return AB_E_NCCL;
  }
  return AB_OK;
}

ab_status ab_slab_info(const double L[3], double halo, int nranks, int rank, double* xlo, double* xhi) {
  if (!L || nranks < 1 || rank < 0 || rank >= nranks || !(L[0] > 0)) return AB_E_ARG;
  if (xlo) *xlo = slab_lo(rank, nranks, L[0]);
  if (xhi) *xhi = slab_lo(rank + 1, nranks, L[0]);
  if (nranks > 1 && L[0] / nranks < halo) return AB_E_BOX;
  return AB_OK;
}

int ab_slab_of(double x, double Lx, int nranks) {
  if (!(Lx > 0) || nranks < 1) return -1;
  return slab_of(wrap_host(x, Lx), nranks, Lx);
}

void ab_destroy(ab_engine* e) { free_engine(e); }

const char* ab_last_error(const ab_engine* e) { return e ? e->err.c_str() : g_create_error.c_str(); }

ab_status ab_set_stream(ab_engine* e, void* stream) {
  if (!e) return AB_E_ARG;
  cudaSetDevice(e->dev);
  TRY(flush_kick(e));
  CK(cudaStreamSynchronize(e->st));
  e->st = stream ? (cudaStream_t)stream : e->own;
  for (ab_engine* d : e->subs) d->st = e->st;
  return AB_OK;
}

ab_status ab_set_box(ab_engine* e, const double L[3]) {
  if (!e) return AB_E_ARG;
  if (bad_ptr(e, L, "L")) return AB_E_ARG;
  cudaSetDevice(e->dev);
  TRY(flush_kick(e));
  for (int c = 0; c < 3; ++c)
    if (!(L[c] > 0.0) || !std::isfinite(L[c])) {
      e->err = "box edge " + std::to_string(c) + " must be finite and > 0";
      return AB_E_BOX;
    }
  cudaSetDevice(e->dev);
  for (ab_engine* d : doms(e)) {
    for (int c = 0; c < 3; ++c) d->L[c] = L[c];
    d->xlo = slab_lo(d->rank, d->nranks, L[0]);
    d->xhi = slab_lo(d->rank + 1, d->nranks, L[0]);
    d->have_box = true;
    d->lists_valid = d->forces_valid = false;
  }
  for (int c = 0; c < 3; ++c) e->L[c] = L[c];
  e->have_box = true;
  e->lists_valid = e->forces_valid = false;
  TRY(check_slab_box(e));
  if (g_const_owner == e) g_const_owner = nullptr;
  graph_drop(e);  // box changed: the captured graph is stale; reload the constants
  return bind_consts(e);
}

ab_status ab_set_atoms(ab_engine* e, int64_t n, const int32_t* type, const double* xyz) {
  if (!e) return AB_E_ARG;
  drop_kick(e);
  if (n < 1 || n > (1ll << 30)) {
    e->err = "n must be in [1, 2^30]";
    return AB_E_ARG;
  }
  if (bad_ptr(e, type, "type") || bad_ptr(e, xyz, "xyz")) return AB_E_ARG;
  if (!e->have_box) {
    e->err = "ab_set_box must precede ab_set_atoms";
    return AB_E_STATE;
  }
  cudaSetDevice(e->dev);
  for (int64_t i = 0; i < n; ++i) {
    if (type[i] != 0 && type[i] != 1) {
      e->err = "type[" + std::to_string(i) + "] must be 0 (C) or 1 (H)";
      return AB_E_ARG;
    }
    for (int c = 0; c < 3; ++c)
      if (!std::isfinite(xyz[3 * i + c])) {
        e->err = "non-finite coordinate of atom " + std::to_string(i);
        return AB_E_NONFINITE;
      }
  }
  TRY(bind_consts(e));
  return set_atoms_impl(e, n, type, xyz);
}

static ab_status need_atoms(ab_engine* e) {
  if (!e) return AB_E_ARG;
  if (!e->have_atoms) {
    e->err = "ab_set_atoms has not been called";
    return AB_E_STATE;
  }
  cudaSetDevice(e->dev);
  return bind_consts(e);
}

ab_status ab_set_positions(ab_engine* e, const double* xyz) {
  TRY(need_atoms(e));
  if (bad_ptr(e, xyz, "xyz")) return AB_E_ARG;
  {
    const int64_t n = slabbed(e) ? e->Nglob : e->N;
    for (int64_t i = 0; i < 3 * n; ++i)
      if (!std::isfinite(xyz[i])) {
        e->err = "non-finite coordinate of atom " + std::to_string(i / 3);
        return AB_E_NONFINITE;
      }
  }
  TRY(flush_kick(e));
  if (!slabbed(e)) {
    CK(cudaMemcpyAsync(e->io.p, xyz, sizeof(double) * 3 * e->N, cudaMemcpyHostToDevice, e->st));
    k_from_caller_pos<<<nblk(e->N, 256), 256, 0, e->st>>>(e->N, e->gid.p, e->io.p, e->pos.p);
    CKL();
    e->forces_valid = false;
    if (host_pinned(xyz)) CK(cudaStreamSynchronize(e->st));
    return AB_OK;
  }
  // slab domains: atoms may change owner arbitrarily -> redistribute (velocities kept)
  const int64_t n = e->Nglob;
  std::vector<double> v(3 * n);
  std::vector<int32_t> t(n);
  TRY(to_caller(e, 1, v.data()));
  {  // species from the instance keys of the owned atoms
    std::vector<double> buf(3 * n, 0.0);
    for (ab_engine* d : doms(e)) {
      std::vector<double4> p(d->N);
      std::vector<int> g(d->N);
      if (d->N) {
        CK(cudaMemcpy(p.data(), d->pos.p, sizeof(double4) * d->N, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(g.data(), d->gid.p, sizeof(int) * d->N, cudaMemcpyDeviceToHost));
      }
      for (int q = 0; q < d->N; ++q) {
        long long k;
        std::memcpy(&k, &p[q].w, sizeof(k));
        buf[g[q]] = (double)(k & 3) + 1.0;
      }
    }
    if (e->comm) {
      NcclApi& NC = nccl(e->err);
      if (!NC.ok) return AB_E_NCCL;
      CK(e->gio.ensure(3 * (size_t)n));
      CK(cudaMemcpyAsync(e->gio.p, buf.data(), sizeof(double) * n, cudaMemcpyHostToDevice, e->st));
      CKN(NC.allReduce(e->gio.p, e->gio.p, n, ncclFloat64, ncclSum, e->comm, e->st));
      CK(cudaMemcpyAsync(buf.data(), e->gio.p, sizeof(double) * n, cudaMemcpyDeviceToHost, e->st));
      CK(cudaStreamSynchronize(e->st));
    }
    for (int64_t i = 0; i < n; ++i) t[i] = (int32_t)buf[i] - 1;
  }
  TRY(set_atoms_impl(e, n, t.data(), xyz));
  return from_caller_vel(e, v.data());
}

ab_status ab_set_velocities(ab_engine* e, const double* v) {
  TRY(need_atoms(e));
  if (bad_ptr(e, v, "v")) return AB_E_ARG;
  drop_kick(e);
  return from_caller_vel(e, v);
}

ab_status ab_get_forces(ab_engine* e, double* f);

ab_status ab_compute(ab_engine* e, double* f, double* energy, double virial[6], double terms[3]) {
  TRY(need_atoms(e));
  TRY(flush_kick(e));  // with the forces it belongs to, before they are recomputed
  TRY(prepare_all(e, true));
  TRY(forces_all(e));
  if (energy) *energy = e->E3[0] + e->E3[1] + e->E3[2];
  if (terms)
    for (int c = 0; c < 3; ++c) terms[c] = e->E3[c];
  if (virial)
    for (int c = 0; c < 6; ++c) virial[c] = e->W6[c];
  if (f) return ab_get_forces(e, f);
  return AB_OK;
}

static ab_status run_nve_impl(ab_engine* e, int64_t nsteps, double dt, int64_t every, double* thermo);

// The NVE loop needs forces and energies but no virial: the per-pair virial accumulation is
// compiled out of the LJ kernel for these steps (ab_compute always evaluates it).
ab_status ab_run_nve(ab_engine* e, int64_t nsteps, double dt, int64_t every, double* thermo) {
  TRY(need_atoms(e));
  // the analysis instantiations (virial, stage rows) run only when stage recording is on
  for (ab_engine* d : doms(e)) d->want_virial = e->record;
  ab_status s = run_nve_impl(e, nsteps, dt, every, thermo);
  for (ab_engine* d : doms(e)) d->want_virial = true;
  return s;
}

// One force evaluation on the current lists inside the NVE loop.  Opt-in (AB_GRAPH=1): a
// single-domain engine without phase profiling captures ghost refresh + the kernel DAG (three
// streams, fork/join events) into a CUDA graph after each list build and replays it every step;
// any rebuild / capacity / concurrency / recording change drops the graph.  Measured on cfg2:
// serialised DAG 0.425 -> 0.412 ms/step, but the concurrent DAG 0.361 -> 0.393 ms/step (the
// graph's branch scheduling overlaps the REBO / far-LJ branches worse than the three streams),
// so the stream path is the default.
static ab_status step_forces(ab_engine* e) {
  const bool graphable = e->subs.empty() && !slabbed(e) && !e->prof && std::getenv("AB_GRAPH") != nullptr &&
                         std::getenv("AB_GRAPH")[0] == '1';
  if (!graphable) {
    graph_drop(e);
    TRY(refresh_ghosts_all(e, true));
    return forces_all(e, false);
  }
  e->want_energy = true;  // one captured graph serves every step
  if (!e->gexec || e->graph_epoch != e->layout) {
    graph_drop(e);
    cudaGraph_t g = nullptr;
    const long long l0 = e->launches;
    CK(cudaStreamBeginCapture(e->st, cudaStreamCaptureModeRelaxed));
    ab_status st = refresh_ghosts_all(e);
    if (st == AB_OK) st = forces_all(e, false);
    cudaError_t ce = cudaStreamEndCapture(e->st, &g);
    if (st != AB_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    CK(ce);
    ce = cudaGraphInstantiate(&e->gexec, g, 0);
    cudaGraphDestroy(g);
    CK(ce);
    e->graph_launches = e->launches - l0;
    e->launches = l0;
    e->graph_epoch = e->layout;
  }
  CK(cudaGraphLaunch(e->gexec, e->st));
  if (e->defer_reduce) e->post_pending = true;  // the captured evaluation left its rows (post_rr)
  e->launches += e->graph_launches;
  e->forces_valid = true;
  e->host_stale = true;
  return AB_OK;
}

static ab_status run_nve_impl(ab_engine* e, int64_t nsteps, double dt, int64_t every, double* thermo) {
  if (nsteps < 0 || !(dt > 0)) {
    e->err = "nsteps must be >= 0 and dt > 0";
    return AB_E_ARG;
  }
  cudaStream_t st = e->st;
  auto D = doms(e);
  if (!e->forces_valid) {
    TRY(flush_kick(e));  // with the forces it belongs to, before they are recomputed
    TRY(prepare_all(e, true));
    TRY(forces_all(e));
  }
  const HostParams& hp = e->hp;
  double dtf0 = 0.5 * dt * hp.ftm2v / hp.mass[0], dtf1 = 0.5 * dt * hp.ftm2v / hp.mass[1];
  // Thermo rows are staged on the device stream (energies of the evaluation + KE after the
  // second half-kick, copied into pinned host memory) and assembled after one synchronisation at
  // the end of the call: thermo steps add no host round trip.
  const int nrows = (thermo && every > 0) ? (int)(nsteps / every) + 1 : 0;
  const int nd = e->comm ? 1 : (int)D.size();
  if (nrows) {
    size_t need = (size_t)nrows * nd * 4;
    if (e->h_th_cap < need) {
      if (e->h_th) cudaFreeHost(e->h_th);
      e->h_th = nullptr;
      e->h_th_cap = 0;
      CK(cudaMallocHost(&e->h_th, sizeof(double) * (need + need / 2 + 64)));
      e->h_th_cap = need + need / 2 + 64;
    }
  }
  int row = 0;
  auto stage_row = [&]() -> ab_status {
    for (ab_engine* d : D) {
      CK(cudaMemsetAsync(d->acc.p + ACC_KE, 0, sizeof(double), st));
      k_ke<<<nblk(d->N, 256), 256, 0, st>>>(d->N, d->pos.p, d->vel.p, hp.mass[0], hp.mass[1], d->acc.p);
      CKL();
    }
    double* h = e->h_th + (size_t)row * nd * 4;
    if (e->comm) {
      NcclApi& NC = nccl(e->err);
      if (!NC.ok) return AB_E_NCCL;
      CK(e->redx.ensure(64));
      double* x = reinterpret_cast<double*>(e->redx.p);
      CK(cudaMemcpyAsync(x, e->acc.p + ACC_EREBO, 3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(x + 3, e->acc.p + ACC_KE, sizeof(double), cudaMemcpyDeviceToDevice, st));
      CKN(NC.allReduce(x, x, 4, ncclFloat64, ncclSum, e->comm, st));
      CK(cudaMemcpyAsync(h, x, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    } else {
      for (int q = 0; q < nd; ++q) {
        CK(cudaMemcpyAsync(h + 4 * q, D[q]->acc.p + ACC_EREBO, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(h + 4 * q + 3, D[q]->acc.p + ACC_KE, sizeof(double), cudaMemcpyDeviceToHost, st));
      }
    }
    ++row;
    return AB_OK;
  };
  TRY(flush_lazy(e));  // the first thermo row reads the previous evaluation's energies
  if (nrows) {
    TRY(flush_kick(e));  // the first row's KE reads v
    TRY(stage_row());
  }
  // The rebuild decision (max displacement) is the only per-step host round trip and
  // it is hidden: after the drift the force kernels are enqueued speculatively on the current
  // lists (they only write F, the scratch block and the b* queue), the host then waits for the
  // displacement read-back alone and, if a rebuild is needed (rare), rebuilds and re-enqueues
  // the forces before the second half-kick.  Energies and counters stay on the device except on
  // thermo steps; the b* queue is sized so it cannot overflow, and the short-list overflow flag
  // of step s is read at step s+1.  Slab domains: the displacement and overflow flags are
  // max-reduced over all ranks first, so every rank takes the same rebuild decision.
  if (!e->ev_disp) CK(cudaEventCreateWithFlags(&e->ev_disp, cudaEventDisableTiming));
  // the step's evaluations leave their partial rows to k_post (reduction + second half-kick)
  struct DeferGuard {
    std::vector<ab_engine*> ds;
    ~DeferGuard() {
      for (ab_engine* d : ds)
        d->defer_reduce = false, d->post_pending = false, d->ghosts_fresh = d->f_zeroed = d->scratch_zeroed = false,
        d->want_energy = true;
    }
  } defer_guard{D};
  for (ab_engine* d : D) d->defer_reduce = true;
  // whole-box engines refresh their image ghosts and zero F inside the drift kernel (not with
  // slab domains, whose x-ghosts arrive by exchange after the drift, nor under CUDA graphs)
  const bool fuse_img = !slabbed(e) && e->subs.empty() && !(std::getenv("AB_GRAPH") && std::getenv("AB_GRAPH")[0] == '1');
  using clk = std::chrono::steady_clock;
  auto ms_since = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  for (int64_t s = 1; s <= nsteps; ++s) {
    const bool th = thermo && every > 0 && s % every == 0;
    // energies / counters of this step are read only on thermo steps and after the call's last step
    for (ab_engine* d : D) d->want_energy = th || s == nsteps;
    auto t0 = clk::now();
    e->tl_sub = 8;
    prof_begin(e, 4);
    bool flags_published = false;
    for (ab_engine* d : D) {
      d->reduce_lazy = false;  // the drift starts a new evaluation (and may zero the scratch)
      const bool fused = fuse_img && d->lists_valid && d->NX == d->N;
      if (!fused && d->kick_pending) TRY(flush_kick(d));
      const bool pre = fused && d->kick_pending;  // the previous step's second half-kick, fused
      const double pd0 = pre ? d->kick_dtf[0] : 0.0, pd1 = pre ? d->kick_dtf[1] : 0.0;
      d->kick_pending = false;
      // the fused kernel's last block leaves the displacement slot zero for the next step, and every
      // other writer of the slot (k_maxdisp, k_integrate1) is followed by an evaluation that zeroes
      // the scratch block; a stale value could only be larger (a max), i.e. cause an early rebuild
      if (!fused) CK(cudaMemsetAsync(d->ct.p + CT_N, 0, sizeof(unsigned long long), st));
      if (fused) {
        FlagOut fo{d->h_ct_dev, reinterpret_cast<unsigned int*>(d->scratch.p + SCRATCH_TICKET),
                   reinterpret_cast<unsigned long long*>(d->scratch.p), (int)(SCRATCH_ZERO_BYTES / 8), CT_OVF_SHORT,
                   d->ct.p};
        k_integrate1_img<<<nblk(d->N, AB_INT_BLOCK), AB_INT_BLOCK, 0, st>>>(d->N, d->pos.p, d->vel.p, d->F.p, pre, pd0, pd1, dtf0, dtf1, dt,
                                                          d->xref.p, d->ct.p + CT_N,
                                                          reinterpret_cast<unsigned long long*>(d->scratch.p + SCRATCH_DBOUND),
                                                          d->NX, d->goff.p, d->gcnt.p,
                                                          d->rshift.p, fo, d->prec == AB_REDUCED);
        d->ghosts_fresh = d->f_zeroed = d->scratch_zeroed = true;
        flags_published = true;
      } else {
        k_integrate1<<<nblk(d->N, 256), 256, 0, st>>>(d->N, d->pos.p, d->vel.p, d->F.p, dtf0, dtf1, dt, d->xref.p,
                                                      d->ct.p + CT_N,
                                                      reinterpret_cast<unsigned long long*>(d->scratch.p + SCRATCH_DBOUND),
                                                      d->prec == AB_REDUCED);
      }
      CKL();
    }
    prof_end(e);
    if (!flags_published) TRY(enqueue_flags(e));  // else written by k_integrate1_img into h_ct
    CK(cudaEventRecord(e->ev_disp, st));
    e->host_ms[0] += ms_since(t0);
    t0 = clk::now();
    // Speculate unless the displacement trend predicts a rebuild at this step (linear
    // extrapolation of the max displacement since the last build): in hot systems that rebuild
    // every few steps a wasted speculative evaluation would sit in front of the rebuild.
    bool speculated = false;
    const double half_skin = 0.5 * hp.skin;
    const bool predict_rebuild = e->disp1 >= 0.0 && e->disp2 >= 0.0 && 2.0 * e->disp1 - e->disp2 > half_skin;
    if (e->lists_valid && !predict_rebuild) {
      TRY(step_forces(e));
      speculated = true;
    }
    e->host_ms[1] += ms_since(t0);
    t0 = clk::now();
    CK(cudaEventSynchronize(e->ev_disp));
    e->host_ms[2] += ms_since(t0);
    t0 = clk::now();
    read_flags(e);
    if (e->h_flag[1]) {
      e->err = "an atom has more than 16 REBO short-list neighbours (NBMAX); unsupported geometry";
      return AB_E_STATE;
    }
    double half = 0.5 * hp.skin;
    const double dnow = std::sqrt(std::max(flag_d2(e), 0.0));
    if (flag_d2(e) > half * half) e->lists_valid = false, speculated = false;
    if (e->lists_valid) e->disp2 = e->disp1, e->disp1 = dnow;
    else e->disp1 = 0.0, e->disp2 = -1.0;  // a rebuild: displacement 0 at the new build
    if (!speculated) {
      TRY(prepare_all(e, false));
      TRY(forces_all(e, false));
    }
    e->host_ms[3] += ms_since(t0);
    t0 = clk::now();
    e->tl_sub = 9;
    prof_begin(e, 4);
    for (ab_engine* d : D) {
      if (d->post_pending && th) {  // the thermo row needs the energies now
        k_post<<<ACC_N + CT_N + nblk(d->N, 256), 256, 0, st>>>(d->post_rr, d->post_rows, d->acc.p, d->ct.p, d->N,
                                                               d->pos.p, d->vel.p, d->F.p, dtf0, dtf1,
                                                               d->prec == AB_REDUCED);
        d->post_pending = false;
      } else {
        if (d->post_pending && s == nsteps) d->reduce_lazy = true, d->lazy_rr = d->post_rr, d->lazy_rows = d->post_rows;
        d->post_pending = false;
        if (fuse_img && !th) {  // deferred to the next drift kernel (or flush_kick)
          d->kick_pending = true, d->kick_dtf[0] = dtf0, d->kick_dtf[1] = dtf1;
          continue;
        }
        k_integrate2<<<nblk(d->N, 256), 256, 0, st>>>(d->N, d->pos.p, d->vel.p, d->F.p, dtf0, dtf1,
                                                      d->prec == AB_REDUCED);
      }
      CKL();
    }
    prof_end(e);
    e->host_ms[4] += ms_since(t0);
    ++e->host_steps;
    ++e->steps;
    if (th) TRY(stage_row());
  }
  if (nrows) {  // the one synchronisation of a thermo call
    CK(cudaStreamSynchronize(st));
    for (int r = 0; r < nrows; ++r) {
      double ee = 0, ke = 0;
      for (int q = 0; q < nd; ++q) {
        const double* h = e->h_th + ((size_t)r * nd + q) * 4;
        ee += h[0] + h[1] + h[2];
        ke += h[3];
      }
      ke *= hp.mvv2e;
      double* t = thermo + 4 * r;
      t[0] = (double)(r * every), t[1] = ee, t[2] = ke, t[3] = ee + ke;
    }
  }
  // no final synchronisation: the last step's kernels may still run; every call that returns
  // data (or the stream itself) orders after them
  CK(cudaGetLastError());
  return AB_OK;
}

ab_status ab_get_positions(ab_engine* e, double* xyz) {
  TRY(need_atoms(e));
  if (bad_ptr(e, xyz, "xyz")) return AB_E_ARG;
  return to_caller(e, 0, xyz);
}

ab_status ab_get_velocities(ab_engine* e, double* v) {
  TRY(need_atoms(e));
  if (bad_ptr(e, v, "v")) return AB_E_ARG;
  TRY(flush_kick(e));
  return to_caller(e, 1, v);
}

ab_status ab_get_forces(ab_engine* e, double* f) {
  TRY(need_atoms(e));
  if (bad_ptr(e, f, "f")) return AB_E_ARG;
  if (!e->forces_valid) {
    e->err = "no force evaluation at the current positions";
    return AB_E_STATE;
  }
  return to_caller(e, 2, f);
}

extern "C++" {
// rows of one domain's list (canonical rows only for bonds / LJ), handed to visit(i, j, sx, sy, sz)
template <class Visit>
static ab_status list_visit(ab_engine* e, ab_engine* d, ab_list which, Visit&& visit) {
  const int N = d->N, NT = d->NT;
  std::vector<int> gid(NT);
  std::vector<char4> sh(NT);
  std::vector<double4> pos(NT);
  if (NT) {
    CK(cudaMemcpyAsync(gid.data(), d->gid.p, sizeof(int) * NT, cudaMemcpyDeviceToHost, e->st));
    CK(cudaMemcpyAsync(sh.data(), d->shift.p, sizeof(char4) * NT, cudaMemcpyDeviceToHost, e->st));
    CK(cudaMemcpyAsync(pos.data(), d->pos.p, sizeof(double4) * NT, cudaMemcpyDeviceToHost, e->st));
  }
  auto type_h = [&](int a) {
    long long k;
    std::memcpy(&k, &pos[a].w, sizeof(k));
    return (int)(k & 3);
  };
  auto canon_of = [&](int i, int J) {
    char4 s = sh[J];
    return gid[i] != gid[J] ? gid[i] < gid[J] : (s.x > 0 || (s.x == 0 && (s.y > 0 || (s.y == 0 && s.z > 0))));
  };
  auto in_rc = [&](int i, int J) {  // exact (un-fused) r^2 <= r_c^2 as on the device
    volatile double dx = pos[J].x - pos[i].x, dy = pos[J].y - pos[i].y, dz = pos[J].z - pos[i].z;
    volatile double a = dx * dx, b = dy * dy, cc = dz * dz;
    volatile double ab = a + b;
    double r2 = ab + cc;
    double rc = d->hp.pr[type_h(i) + type_h(J)].rc;
    return r2 <= rc * rc;
  };
  const bool skinned = which == AB_LIST_LJ_SKIN;
  if (skinned) which = AB_LIST_LJ;  // the same rows without the r <= r_c filter
  if (which == AB_LIST_LJ && d->cl_path) {  // cluster lists: expand the slots of every listed cluster
    if (d->hp.potential == kREBO) return AB_OK;
    std::vector<int> cnt(N), nbr((size_t)N * d->capC), cla((size_t)CL_SIZE * d->NCL);
    if (N) {
      CK(cudaMemcpyAsync(cnt.data(), d->clc.p, sizeof(int) * N, cudaMemcpyDeviceToHost, e->st));
      CK(cudaMemcpyAsync(nbr.data(), d->cln.p, sizeof(int) * N * (size_t)d->capC, cudaMemcpyDeviceToHost, e->st));
      CK(cudaMemcpyAsync(cla.data(), d->cl_atom.p, sizeof(int) * cla.size(), cudaMemcpyDeviceToHost, e->st));
    }
    CK(cudaStreamSynchronize(e->st));
    for (int i = 0; i < N; ++i)
      for (int q = 0; q < cnt[i]; ++q) {
        const int c = nbr[(size_t)i * d->capC + q];
        for (int s = 0; s < CL_SIZE; ++s) {
          const int J = cla[(size_t)CL_SIZE * c + s];
          if (J < 0 || J == i || !canon_of(i, J) || (!skinned && !in_rc(i, J))) continue;
          visit(gid[i], gid[J], sh[J].x, sh[J].y, sh[J].z);
        }
      }
    return AB_OK;
  }
  // (count, neighbour) tables of the requested list(s).  LJ: the near list and the far list
  // without its L bins (the overlap shell, k_lists.cuh: those pairs are near-list members too)
  int nl = which == AB_LIST_LJ ? 2 : 1;
  std::vector<unsigned short> boff;
  if (which == AB_LIST_LJ && N && d->capL[1] > 1) {
    boff.resize((size_t)N * FB_STRIDE);
    CK(cudaMemcpyAsync(boff.data(), d->ljboff.p, sizeof(unsigned short) * boff.size(), cudaMemcpyDeviceToHost, e->st));
  }
  std::vector<int> cnt[3], nbr[3];
  int cap[3];
  for (int c = 0; c < nl; ++c) {
    cap[c] = which == AB_LIST_LJ ? d->capL[c] : d->capS;
    const int* dc = which == AB_LIST_LJ ? d->ljc[c].p : d->s_cnt.p;
    const int* dn = which == AB_LIST_LJ ? d->ljn[c].p : d->s_nbr.p;
    cnt[c].resize(N);
    nbr[c].resize((size_t)N * cap[c]);
    if (N) {
      CK(cudaMemcpyAsync(cnt[c].data(), dc, sizeof(int) * N, cudaMemcpyDeviceToHost, e->st));
      CK(cudaMemcpyAsync(nbr[c].data(), dn, sizeof(int) * N * (size_t)cap[c], cudaMemcpyDeviceToHost, e->st));
    }
  }
  CK(cudaStreamSynchronize(e->st));
  for (int c = 0; c < nl; ++c)
    for (int i = 0; i < N; ++i)
      for (int q = (c == 1 && !boff.empty()) ? (int)boff[(size_t)i * FB_STRIDE + FB_P - 1] : 0; q < cnt[c][i]; ++q) {
        int J = nbr[c][(size_t)i * cap[c] + q];
        char4 s = sh[J];
        bool canon = gid[i] != gid[J] ? gid[i] < gid[J]
                                      : (s.x > 0 || (s.x == 0 && (s.y > 0 || (s.y == 0 && s.z > 0))));
        if (which != AB_LIST_SHORT && !canon) continue;
        if (which == AB_LIST_LJ && !skinned) {  // exact (un-fused) r^2 <= r_c^2 as on the device
          volatile double dx = pos[J].x - pos[i].x, dy = pos[J].y - pos[i].y, dz = pos[J].z - pos[i].z;
          volatile double a = dx * dx, b = dy * dy, cc = dz * dz;
          volatile double ab = a + b;
          double r2 = ab + cc;
          double rc = d->hp.pr[type_h(i) + type_h(J)].rc;
          if (!(r2 <= rc * rc)) continue;
        }
        visit(gid[i], gid[J], s.x, s.y, s.z);
      }
  return AB_OK;
}
static ab_status list_rows(ab_engine* e, ab_engine* d, ab_list which, std::vector<std::array<int64_t, 5>>& out) {
  return list_visit(e, d, which, [&](int i, int j, int sx, int sy, int sz) { out.push_back({i, j, sx, sy, sz}); });
}

// order-independent row digest (header: ab_get_list_digest)
static inline uint64_t dig_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
}  // extern "C++"

ab_status ab_get_list(ab_engine* e, ab_list which, int64_t* count, int64_t* rows) {
  TRY(need_atoms(e));
  if (bad_ptr(e, count, "count")) return AB_E_ARG;
  if (which != AB_LIST_SHORT && which != AB_LIST_BONDS && which != AB_LIST_LJ && which != AB_LIST_LJ_SKIN) {
    e->err = "unknown list";
    return AB_E_ARG;
  }
  if (!e->forces_valid) {
    TRY(prepare_all(e, true));
    TRY(forces_all(e));
  }
  std::vector<std::array<int64_t, 5>> out;
  for (ab_engine* d : doms(e)) TRY(list_rows(e, d, which, out));
  std::sort(out.begin(), out.end());
  *count = (int64_t)out.size();
  if (rows)
    for (size_t r = 0; r < out.size(); ++r)
      for (int c = 0; c < 5; ++c) rows[5 * r + c] = out[r][c];
  return AB_OK;
}

ab_status ab_get_list_digest(ab_engine* e, ab_list which, uint64_t digest[3]) {
  TRY(need_atoms(e));
  if (bad_ptr(e, digest, "digest")) return AB_E_ARG;
  if (which != AB_LIST_SHORT && which != AB_LIST_BONDS && which != AB_LIST_LJ && which != AB_LIST_LJ_SKIN) {
    e->err = "unknown list";
    return AB_E_ARG;
  }
  if (!e->forces_valid) {
    TRY(prepare_all(e, true));
    TRY(forces_all(e));
  }
  uint64_t c = 0, sum = 0, x = 0;
  for (ab_engine* d : doms(e))
    TRY(list_visit(e, d, which, [&](int i, int j, int sx, int sy, int sz) {
      uint64_t a = ((uint64_t)(uint32_t)i << 32) | (uint32_t)j;
      uint64_t b = ((uint64_t)(sx + 128) << 16) | ((uint64_t)(sy + 128) << 8) | (uint64_t)(sz + 128);
      uint64_t h = dig_mix(a ^ dig_mix(b));
      ++c, sum += h, x ^= h;
    }));
  digest[0] = c, digest[1] = sum, digest[2] = x;
  return AB_OK;
}

ab_status ab_get_stats(ab_engine* e, ab_stats* s) {
  if (!e || !s) return AB_E_ARG;
  cudaSetDevice(e->dev);
  TRY(pull_results(e));
  const unsigned long long* c = e->last_ct;
  s->n_short = c[CT_SHORT], s->n_bonds = c[CT_BONDS], s->n_quads = c[CT_QUADS], s->n_lj = c[CT_LJ];
  s->n_C0 = c[CT_C0], s->n_bstar = c[CT_BSTAR], s->n_sb_trans = c[CT_SBTRANS], s->max_short = c[CT_MAXSHORT];
  s->max_reach = c[CT_MAXREACH], s->n_badarg = c[CT_BADARG];
  s->n_atoms = slabbed(e) ? e->Nglob : e->N;
  s->n_ghosts = 0, s->n_rebuilds = e->rebuilds, s->n_steps = e->steps;
  s->n_overflow_retries = c[CT_OVF_REACH];
  s->lj_capacity = 0, s->inter_capacity = 0;
  for (ab_engine* d : doms(e)) {
    s->n_ghosts += d->G;
    s->n_overflow_retries += d->retries;
    s->lj_capacity = std::max<int64_t>(s->lj_capacity, d->cl_path ? (int64_t)d->capC * CL_SIZE
                                                                  : d->capL[0] + d->capL[1] + d->capL[2]);
    s->inter_capacity = std::max<int64_t>(s->inter_capacity, d->capI);
  }
  if (!e->subs.empty()) s->n_rebuilds = e->rebuilds;
  s->n_lj_entries = c[CT_LJENT], s->n_angles = c[CT_ANGLES];
  s->n_lj_far = c[CT_LJFAR], s->n_lj_entries_far = c[CT_LJENTFAR];
  s->n_lj_taper = c[CT_LJTAPER];
  return AB_OK;
}

ab_status ab_record_stages(ab_engine* e, int on) {
  if (!e) return AB_E_ARG;
  cudaSetDevice(e->dev);
  TRY(flush_kick(e));
  for (ab_engine* d : doms(e)) d->record = on != 0;
  e->record = on != 0;
  e->forces_valid = false;
  ++e->layout;
  return AB_OK;
}

ab_status ab_get_stage(ab_engine* e, int stage, int64_t* count, double* out) {
  TRY(need_atoms(e));
  if (bad_ptr(e, count, "count")) return AB_E_ARG;
  if ((stage != 0 && stage != 1) || !e->record || !e->forces_valid) {
    e->err = "stage must be 0 or 1, recording on (ab_record_stages) and forces evaluated";
    return AB_E_STATE;
  }
  const int width = stage == 0 ? 13 : 7;
  std::vector<double> all;
  for (ab_engine* d : doms(e)) {
    int n[2];
    CK(cudaMemcpyAsync(n, d->small_i.p + 6, 2 * sizeof(int), cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    const int rows = n[stage];
    const size_t at = all.size();
    all.resize(at + (size_t)width * rows);
    if (rows)
      CK(cudaMemcpy(all.data() + at, stage == 0 ? d->stage0.p : d->stage1.p, sizeof(double) * width * rows,
                    cudaMemcpyDeviceToHost));
  }
  int64_t total = (int64_t)(all.size() / width);
  if (stage == 1) {
    // a far-zone pair of the reach set has two rows: k_lj_far's (C = 1) and k_lj_near's correction
    // (C = 1 - M < 1); the pair's C_ij is the smaller one
    std::map<std::array<double, 5>, size_t> best;
    for (int64_t r = 0; r < total; ++r) {
      const double* row = all.data() + (size_t)r * width;
      std::array<double, 5> k{row[0], row[1], row[2], row[3], row[4]};
      auto it = best.find(k);
      if (it == best.end()) best.emplace(k, (size_t)r);
      else if (row[5] < all[it->second * width + 5]) it->second = (size_t)r;
    }
    std::vector<double> ded;
    ded.reserve(best.size() * width);
    for (auto& kv : best) ded.insert(ded.end(), all.begin() + kv.second * width, all.begin() + (kv.second + 1) * width);
    all.swap(ded);
    total = (int64_t)best.size();
  }
  if (out && total) std::memcpy(out, all.data(), sizeof(double) * width * total);
  *count = total;
  return AB_OK;
}

ab_status ab_set_profiling(ab_engine* e, int on) {
  if (!e) return AB_E_ARG;
  cudaSetDevice(e->dev);
  CK(cudaStreamSynchronize(e->st));
  for (ab_engine* d : doms(e)) {
    prof_collect(d);
    d->prof = on != 0;
    for (int q = 0; q < AB_NPHASE; ++q) d->phase_ms[q] = 0, d->phase_n[q] = 0;
  }
  prof_collect(e);
  e->prof = on != 0;
  for (int q = 0; q < AB_NPHASE; ++q) e->phase_ms[q] = 0, e->phase_n[q] = 0;
  return AB_OK;
}

ab_status ab_set_concurrency(ab_engine* e, int on) {
  if (!e) return AB_E_ARG;
  cudaSetDevice(e->dev);
  CK(cudaStreamSynchronize(e->st));
  e->serial = on == 0;
  for (ab_engine* d : doms(e)) d->serial = on == 0;
  ++e->layout;
  return AB_OK;
}

ab_status ab_get_phase_ms(ab_engine* e, double ms[AB_NPHASE], int64_t n[AB_NPHASE]) {
  if (!e || !ms || !n) return AB_E_ARG;
  cudaSetDevice(e->dev);
  CK(cudaStreamSynchronize(e->st));
  for (int q = 0; q < AB_NPHASE; ++q) ms[q] = 0, n[q] = 0;
  auto D = doms(e);
  if (D[0] != e) D.push_back(e);
  for (ab_engine* d : D) {
    prof_collect(d);
    for (int q = 0; q < AB_NPHASE; ++q) ms[q] += d->phase_ms[q], n[q] += d->phase_n[q];
  }
  return AB_OK;
}

ab_status ab_peak_flops(ab_engine* e, ab_precision prec, double* tflops) {
  if (!e || !tflops) return AB_E_ARG;
  cudaSetDevice(e->dev);
  const int iters = 1 << 16, threads = 256, blocks = e->nsm * 8;
  DBuf<double> out;
  CK(out.ensure(threads));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaEventRecord(a, e->st));
    if (prec == AB_FP64)
      k_fma_peak<double><<<blocks, threads, 0, e->st>>>(out.p, iters, 0.999999, 1e-7);
    else
      k_fma_peak<float><<<blocks, threads, 0, e->st>>>((float*)out.p, iters, 0.999999f, 1e-7f);
    CKL();
    CK(cudaEventRecord(b, e->st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (rep > 0) best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  out.release();
  double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  return AB_OK;
}

ab_status ab_device_info(ab_engine* e, int* device, char* name, size_t name_len, int64_t* launches) {
  if (!e) return AB_E_ARG;
  if (device) *device = e->dev;
  if (name && name_len) std::snprintf(name, name_len, "%s", e->devname);
  if (launches) {
    int64_t n = e->launches;
    for (ab_engine* d : e->subs) n += d->launches;
    *launches = n;
  }
  return AB_OK;
}

}  // extern "C"
