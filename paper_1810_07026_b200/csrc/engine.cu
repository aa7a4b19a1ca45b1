// engine.cu -- the C-ABI (include/airebo_b200.h) and host orchestration of the B200 AIREBO engine.
//
// One translation unit (unity build) so the __constant__ parameter tables are visible to every
// kernel.  Per force evaluation, on one stream: exact short list + N_i (k_short) -> REBO + bond
// order + torsion per bond (k_rebo) -> C_ij reach set + LJ per atom (k_lj) -> deferred b* batch
// (k_bstar).  List rebuilds (binning, ghosts, skinned lists) happen when an atom moved more than
// skin/2.  No CPU fallback: every step of the path is a kernel below.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/airebo_b200.h"
#include "dev_common.cuh"
#include "k_bond.cuh"
#include "k_lists.cuh"
#include "k_lj.cuh"
#include "k_misc.cuh"
#include "params.h"

using namespace ab;

namespace {

std::string g_create_error;

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t cnt) {
    if (cnt <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t c = std::max<size_t>(cnt, 1);
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

inline int nblk(long long n, int t) { return (int)((n + t - 1) / t); }

constexpr size_t SCRATCH_BYTES = 1024, SCRATCH_CT = 128, SCRATCH_SMALL = 512, SCRATCH_ZERO_BYTES = 512 + 64;

}  // namespace

struct ab_engine {
  std::string err;
  HostParams hp;
  ab_precision prec = AB_FP64;
  int dev = 0;
  char devname[256] = {0};
  int nsm = 148;
  cudaStream_t own = nullptr, st = nullptr;
  bool have_box = false, have_atoms = false, lists_valid = false, forces_valid = false;
  bool record = false;
  double L[3] = {0, 0, 0};
  int N = 0, NT = 0, G = 0;
  double halo = 0, rcmax = 0, rmaxmax = 0;
  Grid grid{};
  int ncell = 0, nrLJ = 1, nrI = 1;
  int capI = 0, capS = 0, capQ = 0;
  long long launches = 0, rebuilds = 0, steps = 0, retries = 0;
  // device state
  DBuf<double4> pos, pos_tmp, xref;
  DBuf<double> vel, vel_tmp, F, io;
  DBuf<int> gid, gid_tmp, owner, key, key2, val, val2, cell_start, gcnt, goff;
  DBuf<char4> shift;
  DBuf<signed char> typ;
  DBuf<int> ljc[3], ljn[3], in_cnt, in_nbr;  // LJ near / pure / band lists, intermediate list
  int capL[3] = {0, 0, 0};
  bool want_virial = true;
  DBuf<int> s_cnt, s_nbr;
  DBuf<unsigned char> s_dr, s_w, s_N;  // typed by precision at use
  DBuf<int2> bonds;
  DBuf<int4> q_item;
  DBuf<int> ovf_bond, ovf_q;  // overflow (large side / full b*) index lists
  DBuf<double> q_M;
  // one small device scratch block, zeroed with a single memset per evaluation:
  //   acc (ACC_N doubles) at 0, ct (CT_N + 1 u64; [CT_N] = max displacement^2) at 128,
  //   small_i (16 ints: nbonds, qcount, list maxima x4, stage counts x2, overflow counts x2) at 512
  DBuf<unsigned char> scratch;
  DBuf<int> small_i;
  DBuf<double> acc;
  DBuf<unsigned long long> ct;
  bool host_stale = false;  // acc / ct of the last evaluation not yet copied to the host
  cudaEvent_t ev_disp = nullptr;
  DBuf<double> stage0, stage1, red_d;
  DBuf<unsigned long long> red_u;
  DBuf<unsigned char> cub_tmp;
  // pinned host mirror for small readbacks
  unsigned long long* h_ct = nullptr;
  double* h_acc = nullptr;
  int* h_small = nullptr;
  // results of the last evaluation
  double E3[3] = {0, 0, 0}, W6[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long last_ct[CT_N] = {0};
  // per-phase CUDA-event profiling (ab_set_profiling)
  bool prof = false;
  double phase_ms[AB_NPHASE] = {0};
  long long phase_n[AB_NPHASE] = {0};
  struct Pend {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Pend> pending;
  std::vector<cudaEvent_t> pool;
  int open_phase = -1;
  cudaEvent_t open_ev = nullptr;
};

namespace {
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
void prof_begin(ab_engine* e, int phase) {
  if (!e->prof) return;
  e->open_phase = phase;
  e->open_ev = ev_get(e);
  cudaEventRecord(e->open_ev, e->st);
}
void prof_end(ab_engine* e) {
  if (!e->prof || e->open_phase < 0) return;
  cudaEvent_t b = ev_get(e);
  cudaEventRecord(b, e->st);
  e->pending.push_back({e->open_phase, e->open_ev, b});
  e->open_phase = -1;
}
// call after a stream synchronisation
void prof_collect(ab_engine* e) {
  for (auto& p : e->pending) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      e->phase_ms[p.phase] += ms;
      e->phase_n[p.phase] += 1;
    }
    e->pool.push_back(p.a);
    e->pool.push_back(p.b);
  }
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
#define CKL()                                                                             \
  do {                                                                                    \
    ++e->launches;                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess) {                                                              \
      e->err = std::string("CUDA launch error: ") + cudaGetErrorString(e_);               \
      return AB_E_CUDA;                                                                   \
    }                                                                                     \
  } while (0)
#define TRY(x)                   \
  do {                           \
    ab_status s_ = (x);          \
    if (s_ != AB_OK) return s_;  \
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
  }
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i)
      for (int k = 0; k < 2; ++k) t.explam[j][i][k] = (R)std::exp(hp.lam[j][i][k]);
  for (int c = 0; c < 2; ++c) {
    int n = (int)hp.gknot[c].size();
    t.gn[c] = n;
    for (int q = 0; q < 16; ++q) t.gx[c][q] = t.gy[c][q] = t.gm[c][q] = 0;
    for (int q = 0; q < n; ++q) {
      t.gx[c][q] = (R)hp.gknot[c][q];
      t.gy[c][q] = (R)hp.gval[c][q];
      double m = (q == 0 || q == n - 1)
                     ? 0.0
                     : (hp.gval[c][q + 1] - hp.gval[c][q - 1]) / (hp.gknot[c][q + 1] - hp.gknot[c][q - 1]);
      t.gm[c][q] = (R)m;
    }
  }
  for (int a = 0; a < 2; ++a)
    for (int q = 0; q < 25; ++q) t.P[a][q] = (R)hp.Ptab[a][q];
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 225; ++q) t.Rt[p][q] = (R)hp.Rtab[p][q], t.Tt[p][q] = (R)hp.Ttab[p][q];
  t.conj_lo = (R)hp.conj_lo, t.conj_hi = (R)hp.conj_hi, t.s2lo = (R)hp.sin2_lo, t.s2hi = (R)hp.sin2_hi;
  for (int k = 0; k < 2; ++k)
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int l = 0; l < 2; ++l) t.tors[k][i][j][l] = (R)hp.tors[k][i][j][l];
}

ab_status upload_geo(ab_engine* e) {
  Geo g;
  const HostParams& hp = e->hp;
  double rmm = 0, rcm = 0;
  for (int p = 0; p < 3; ++p) {
    const PairSet& s = hp.pr[p];
    g.rmax2[p] = s.rmax * s.rmax;
    g.rc2[p] = s.rc * s.rc;
    g.rmax_s2[p] = (s.rmax + hp.skin) * (s.rmax + hp.skin);
    g.rc_s2[p] = (s.rc + hp.skin) * (s.rc + hp.skin);
    g.rlo2[p] = s.rlo * s.rlo;
    double srhi = s.sigma * 1.122462048309373;
    g.srhi2_hi[p] = srhi * srhi * (1.0 + 1e-9);
    rmm = std::max(rmm, s.rmax);
    rcm = std::max(rcm, s.rc);
  }
  g.reach2 = (3 * rmm) * (3 * rmm);
  for (int c = 0; c < 3; ++c) g.L[c] = e->L[c];
  g.mass[0] = hp.mass[0], g.mass[1] = hp.mass[1], g.ftm2v = hp.ftm2v, g.mvv2e = hp.mvv2e;
  e->rmaxmax = rmm;
  e->rcmax = rcm;
  e->halo = rcm + hp.skin;  // LJ cutoff + skin covers every REBO/torsion/C_ij/b* reach
  CK(cudaMemcpyToSymbolAsync(c_geo, &g, sizeof(Geo), 0, cudaMemcpyHostToDevice, e->st));
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
  CK(e->s_N.ensure((size_t)e->NT * 3 * rs));
  CK(e->bonds.ensure((size_t)e->N * e->capS + 1));
  return AB_OK;
}

// ---------------------------------------------------------------- list build
ab_status rebuild_impl(ab_engine* e) {
  const int N = e->N;
  cudaStream_t st = e->st;
  const double h = e->halo;
  // cell grid over the padded region [-h, L+h): edge >= (r_c,max + skin)/3 >= r_max + skin
  double cs_t = std::max((e->rcmax + e->hp.skin) / 3.0, e->rmaxmax + e->hp.skin);
  double csmin = 1e300;
  for (int c = 0; c < 3; ++c) {
    double span = e->L[c] + 2 * h;
    e->grid.nc[c] = std::max(1, (int)std::floor(span / cs_t));
    e->grid.cs[c] = span / e->grid.nc[c];
    e->grid.lo[c] = -h;
    csmin = std::min(csmin, e->grid.cs[c]);
  }
  e->ncell = e->grid.nc[0] * e->grid.nc[1] * e->grid.nc[2];
  e->nrLJ = (int)std::ceil((e->rcmax + e->hp.skin) / csmin);
  e->nrI = (int)std::ceil((e->rmaxmax + e->hp.skin) / csmin);
  // 1. wrap + spatial sort of the local atoms
  CK(e->key.ensure(N));
  CK(e->val.ensure(N));
  CK(e->key2.ensure(N));
  CK(e->val2.ensure(N));
  CK(e->pos_tmp.ensure(N));
  CK(e->vel_tmp.ensure(3 * (size_t)N));
  CK(e->gid_tmp.ensure(N));
  k_wrap_and_key<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->grid, e->key.p, e->val.p);
  CKL();
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, e->key.p, e->key2.p, e->val.p, e->val2.p, N, 0, 31, st);
  CK(e->cub_tmp.ensure(need));
  size_t have = e->cub_tmp.n;
  CK(cub::DeviceRadixSort::SortPairs(e->cub_tmp.p, have, e->key.p, e->key2.p, e->val.p, e->val2.p, N, 0, 31, st));
  ++e->launches;
  k_permute<<<nblk(N, 256), 256, 0, st>>>(N, e->val2.p, e->pos.p, e->pos_tmp.p, e->vel.p, e->vel_tmp.p, e->gid.p,
                                          e->gid_tmp.p);
  CKL();
  CK(cudaMemcpyAsync(e->pos.p, e->pos_tmp.p, sizeof(double4) * N, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(e->vel.p, e->vel_tmp.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(e->gid.p, e->gid_tmp.p, sizeof(int) * N, cudaMemcpyDeviceToDevice, st));
  // 2. periodic images (ghosts) within the halo
  int3 smax = make_int3((int)std::ceil(h / e->L[0]), (int)std::ceil(h / e->L[1]), (int)std::ceil(h / e->L[2]));
  CK(e->gcnt.ensure(N));
  CK(e->goff.ensure(N));
  k_ghost_count<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, smax, h, e->gcnt.p);
  CKL();
  need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, e->gcnt.p, e->goff.p, N, st);
  CK(e->cub_tmp.ensure(need));
  have = e->cub_tmp.n;
  CK(cub::DeviceScan::ExclusiveSum(e->cub_tmp.p, have, e->gcnt.p, e->goff.p, N, st));
  ++e->launches;
  int tail[2];
  CK(cudaMemcpyAsync(&tail[0], e->goff.p + N - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&tail[1], e->gcnt.p + N - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  e->G = tail[0] + tail[1];
  e->NT = N + e->G;
  const int NT = e->NT;
  if (e->pos.n < (size_t)NT) {  // grow, keeping the local part
    DBuf<double4> np;
    CK(np.ensure((size_t)NT + NT / 8));
    CK(cudaMemcpyAsync(np.p, e->pos.p, sizeof(double4) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    e->pos.release();
    e->pos = np;
  }
  if (e->gid.n < (size_t)NT) {
    DBuf<int> ng;
    CK(ng.ensure((size_t)NT + NT / 8));
    CK(cudaMemcpyAsync(ng.p, e->gid.p, sizeof(int) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    e->gid.release();
    e->gid = ng;
  }
  CK(e->owner.ensure(NT));
  CK(e->shift.ensure(NT));
  CK(e->typ.ensure(NT));
  k_ghost_fill<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, smax, h, e->goff.p, e->owner.p, e->gid.p, e->shift.p);
  CKL();
  k_types<<<nblk(NT, 256), 256, 0, st>>>(NT, e->pos.p, e->typ.p);
  CKL();
  // 3. bin all atoms (locals + ghosts)
  CK(e->key.ensure(NT));
  CK(e->val.ensure(NT));
  CK(e->key2.ensure(NT));
  CK(e->val2.ensure(NT));
  CK(e->cell_start.ensure((size_t)e->ncell + 1));
  k_cell_keys<<<nblk(NT, 256), 256, 0, st>>>(NT, e->pos.p, e->grid, e->key.p, e->val.p);
  CKL();
  need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, e->key.p, e->key2.p, e->val.p, e->val2.p, NT, 0, 31, st);
  CK(e->cub_tmp.ensure(need));
  have = e->cub_tmp.n;
  CK(cub::DeviceRadixSort::SortPairs(e->cub_tmp.p, have, e->key.p, e->key2.p, e->val.p, e->val2.p, NT, 0, 31, st));
  ++e->launches;
  k_cell_bounds<<<nblk(NT + 1, 256), 256, 0, st>>>(NT, e->ncell, e->key2.p, e->cell_start.p);
  CKL();
  // 4. skinned lists: LJ (local atoms, full) and intermediate REBO (all atoms)
  CK(e->small_i.ensure(8));
  for (int c = 0; c < 3; ++c) CK(e->ljc[c].ensure(N));
  CK(e->in_cnt.ensure(NT));
  const double skin = e->hp.skin;
  const double rnear = 3 * e->rmaxmax + skin;
  if (e->capL[0] == 0) {  // first build: capacities from the mean density (grown on overflow)
    double rho = N / (e->L[0] * e->L[1] * e->L[2]), fpi = 4.18879020478639;
    double rlo_max = 0;
    for (int p = 0; p < 3; ++p) rlo_max = std::max(rlo_max, e->hp.pr[p].rlo);
    double r1 = std::max(rnear, rlo_max - skin), r2 = e->rcmax + skin;
    e->capL[0] = 32 + (int)(1.3 * rho * fpi * rnear * rnear * rnear);
    e->capL[1] = 32 + (int)(1.3 * rho * fpi * (r1 * r1 * r1 - rnear * rnear * rnear));
    e->capL[2] = 32 + (int)(1.3 * rho * fpi * (r2 * r2 * r2 - std::min(r1, rnear) * std::min(r1, rnear) * std::min(r1, rnear)));
  }
  if (e->capI == 0) e->capI = 16;
  LJLists Lg;
  Lg.near2 = rnear * rnear;
  for (int p = 0; p < 3; ++p) {
    double b = e->hp.pr[p].rlo - skin;
    Lg.pure2[p] = b > rnear ? b * b : -1.0;
  }
  for (int attempt = 0; attempt < 4; ++attempt) {
    for (int c = 0; c < 3; ++c) {
      CK(e->ljn[c].ensure((size_t)N * e->capL[c]));
      Lg.cap[c] = e->capL[c];
      Lg.cnt[c] = e->ljc[c].p;
      Lg.nbr[c] = e->ljn[c].p;
    }
    CK(e->in_nbr.ensure((size_t)NT * e->capI));
    CK(cudaMemsetAsync(e->small_i.p + 2, 0, 4 * sizeof(int), st));
    k_build_lj<<<nblk((long long)N * 32, 128), 128, 0, st>>>(N, e->pos.p, e->grid, e->cell_start.p, e->val2.p,
                                                              e->nrLJ, Lg, e->small_i.p + 2);
    CKL();
    k_build_inter<<<nblk((long long)NT * 32, 128), 128, 0, st>>>(NT, e->pos.p, e->grid, e->cell_start.p, e->val2.p,
                                                                  e->nrI, e->capI, e->in_cnt.p, e->in_nbr.p,
                                                                  e->small_i.p + 5);
    CKL();
    int mx[4];
    CK(cudaMemcpyAsync(mx, e->small_i.p + 2, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bool ok = true;
    for (int c = 0; c < 3; ++c)
      if (mx[c] > e->capL[c]) e->capL[c] = mx[c] + mx[c] / 8 + 32, ok = false;
    if (mx[3] > e->capI) e->capI = mx[3] + 4, ok = false;
    if (ok) break;
    ++e->retries;
  }
  e->capS = std::min(e->capI, 32);
  TRY(ensure_short(e));
  CK(e->xref.ensure(N));
  k_copy_xref<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->xref.p);
  CKL();
  e->lists_valid = true;
  ++e->rebuilds;
  return AB_OK;
}

ab_status rebuild(ab_engine* e) {
  prof_begin(e, 5);
  ab_status s = rebuild_impl(e);
  prof_end(e);
  return s;
}

template <typename R>
ab_status forces_impl(ab_engine* e, bool sync_host) {
  const int N = e->N, NT = e->NT;
  cudaStream_t st = e->st;
  StageBuf sb0{nullptr, nullptr, 0}, sb1{nullptr, nullptr, 0};
  if (e->record) {
    size_t n0 = (size_t)N * e->capS + 16, n1 = (size_t)N * (e->capL[0] + e->capL[1] + e->capL[2]) + 16;
    CK(e->stage0.ensure(n0 * 13));
    CK(e->stage1.ensure(n1 * 7));
    sb0 = StageBuf{e->stage0.p, e->small_i.p + 6, (int)n0};
    sb1 = StageBuf{e->stage1.p, e->small_i.p + 7, (int)n1};
  }
  // b* queue: the canonical near-list pairs bound the queue, so it cannot overflow
  {
    long long qb = (long long)N * e->capL[0] / 2 + 1024;
    if (e->capQ < qb) {
      e->capQ = (int)std::min<long long>(qb, 1ll << 30);
      CK(e->q_item.ensure(e->capQ));
      CK(e->q_M.ensure(e->capQ));
    }
  }
  for (int attempt = 0; attempt < 3; ++attempt) {
    CK(cudaMemsetAsync(e->F.p, 0, sizeof(double) * 3 * N, st));
    CK(cudaMemsetAsync(e->scratch.p, 0, SCRATCH_ZERO_BYTES, st));  // acc, counters, small ints
    ShortList<R> S = short_view<R>(e);
    // grids and the per-block partial rows of the energy / virial / counter reduction
    const int g_short = nblk(NT, 128), g_rebo = e->nsm * 4, g_near = nblk(N, NEAR_ATOMS);
    const int g_far = std::min(nblk((long long)N * 32, 128), e->nsm * 8), g_bstar = e->nsm * 4, g_slow = e->nsm;
    const int nrows = g_short + g_rebo + g_near + g_far + g_bstar + 2 * g_slow;
    CK(e->ovf_bond.ensure((size_t)N * e->capS + 1));
    CK(e->ovf_q.ensure(e->capQ));
    CK(e->red_d.ensure((size_t)ACC_N * nrows));
    CK(e->red_u.ensure((size_t)CT_N * nrows));
    RedRows RR{e->red_d.p, e->red_u.p, nrows, 0};
    prof_begin(e, 0);
    k_short<R><<<g_short, 128, 0, st>>>(N, NT, e->pos.p, e->in_cnt.p, e->in_nbr.p, e->capI, S, e->gid.p,
                                        e->shift.p, e->bonds.p, e->small_i.p, e->ct.p, RR);
    CKL();
    prof_end(e);
    RR.row0 += g_short;
    prof_begin(e, 1);
    k_rebo<R, NB_FAST><<<g_rebo, 128, 0, st>>>(e->bonds.p, e->small_i.p, nullptr, e->ovf_bond.p, e->small_i.p + 8,
                                               S, e->typ.p, e->owner.p, e->gid.p, e->shift.p, e->F.p, sb0, RR);
    CKL();
    RR.row0 += g_rebo;
    k_rebo<R, NBMAX><<<g_slow, 128, 0, st>>>(e->bonds.p, e->small_i.p, e->ovf_bond.p, nullptr, e->small_i.p + 8, S,
                                             e->typ.p, e->owner.p, e->gid.p, e->shift.p, e->F.p, sb0, RR);
    CKL();
    RR.row0 += g_slow;
    prof_end(e);
    BstarQueue Qu{e->q_item.p, e->q_M.p, e->small_i.p + 1, e->capQ};
    LJArgs A;
    A.N = N;
    A.pos = e->pos.p;
    for (int c = 0; c < 3; ++c) A.cap[c] = e->capL[c], A.cnt[c] = e->ljc[c].p, A.nbr[c] = e->ljn[c].p;
    prof_begin(e, 2);
    if (e->want_virial)
      k_lj_near<R, true><<<g_near, NEAR_GROUP * NEAR_ATOMS, 0, st>>>(A, S, e->owner.p, e->gid.p, e->shift.p, e->F.p,
                                                                     e->acc.p, e->ct.p, Qu, sb1, RR);
    else
      k_lj_near<R, false><<<g_near, NEAR_GROUP * NEAR_ATOMS, 0, st>>>(A, S, e->owner.p, e->gid.p, e->shift.p, e->F.p,
                                                                      e->acc.p, e->ct.p, Qu, sb1, RR);
    CKL();
    prof_end(e);
    RR.row0 += g_near;
    prof_begin(e, 6);
    if (e->want_virial)
      k_lj_far<R, true><<<g_far, 128, 0, st>>>(A, e->gid.p, e->shift.p, e->F.p, e->acc.p, e->ct.p, sb1, RR);
    else
      k_lj_far<R, false><<<g_far, 128, 0, st>>>(A, e->gid.p, e->shift.p, e->F.p, e->acc.p, e->ct.p, sb1, RR);
    CKL();
    prof_end(e);
    RR.row0 += g_far;
    prof_begin(e, 3);
    k_bstar<R, NB_FAST, false><<<g_bstar, 128, 0, st>>>(Qu, nullptr, e->ovf_q.p, e->small_i.p + 9, e->pos.p, S,
                                                        e->typ.p, e->owner.p, e->gid.p, e->shift.p, e->F.p, sb1, RR);
    CKL();
    RR.row0 += g_bstar;
    k_bstar<R, NBMAX, true><<<g_slow, 128, 0, st>>>(Qu, e->ovf_q.p, nullptr, e->small_i.p + 9, e->pos.p, S, e->typ.p,
                                                    e->owner.p, e->gid.p, e->shift.p, e->F.p, sb1, RR);
    CKL();
    prof_end(e);
    RR.row0 = 0;
    k_reduce<<<ACC_N + CT_N, 256, 0, st>>>(RR, nrows, e->acc.p, e->ct.p);
    CKL();
    if (!sync_host) {  // NVE steps: results stay on the device until somebody needs them
      e->host_stale = true;
      e->forces_valid = true;
      return AB_OK;
    }
    CK(cudaMemcpyAsync(e->h_ct, e->ct.p, sizeof(unsigned long long) * CT_N, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(e->h_acc, e->acc.p, sizeof(double) * ACC_N, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    prof_collect(e);
    if (e->h_ct[CT_OVF_SHORT]) {
      e->err = "an atom has more than 16 REBO short-list neighbours (NBMAX); unsupported geometry";
      return AB_E_STATE;
    }
    if (e->h_ct[CT_OVF_QUEUE]) {  // grow the b* queue and redo the evaluation
      int need = (int)(e->h_ct[CT_BSTAR] + e->h_ct[CT_OVF_QUEUE]);
      e->capQ = std::max(2 * e->capQ, need + need / 4 + 1024);
      CK(e->q_item.ensure(e->capQ));
      CK(e->q_M.ensure(e->capQ));
      ++e->retries;
      continue;
    }
    break;
  }
  std::memcpy(e->last_ct, e->h_ct, sizeof(e->last_ct));
  for (int c = 0; c < 3; ++c) e->E3[c] = e->h_acc[ACC_EREBO + c];
  for (int c = 0; c < 6; ++c) e->W6[c] = e->h_acc[ACC_W + c];
  if (!std::isfinite(e->E3[0] + e->E3[1] + e->E3[2])) {
    e->err = "non-finite energy";
    return AB_E_NONFINITE;
  }
  e->forces_valid = true;
  e->host_stale = false;
  return AB_OK;
}

ab_status forces(ab_engine* e, bool sync_host = true) {
  return e->prec == AB_FP64 ? forces_impl<double>(e, sync_host) : forces_impl<float>(e, sync_host);
}

// bring energies / virial / counters of the last (asynchronous) evaluation to the host
ab_status pull_results(ab_engine* e) {
  if (!e->host_stale) return AB_OK;
  CK(cudaMemcpyAsync(e->h_ct, e->ct.p, sizeof(unsigned long long) * CT_N, cudaMemcpyDeviceToHost, e->st));
  CK(cudaMemcpyAsync(e->h_acc, e->acc.p, sizeof(double) * ACC_N, cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  prof_collect(e);
  e->host_stale = false;
  if (e->h_ct[CT_OVF_SHORT]) {
    e->err = "an atom has more than 16 REBO short-list neighbours (NBMAX); unsupported geometry";
    return AB_E_STATE;
  }
  std::memcpy(e->last_ct, e->h_ct, sizeof(e->last_ct));
  for (int c = 0; c < 3; ++c) e->E3[c] = e->h_acc[ACC_EREBO + c];
  for (int c = 0; c < 6; ++c) e->W6[c] = e->h_acc[ACC_W + c];
  if (!std::isfinite(e->E3[0] + e->E3[1] + e->E3[2])) {
    e->err = "non-finite energy";
    return AB_E_NONFINITE;
  }
  return AB_OK;
}

// make lists valid for the current positions (rebuild if needed, else move the ghosts)
ab_status prepare(ab_engine* e, bool check_disp) {
  if (!e->lists_valid) return rebuild(e);
  if (check_disp) {
    CK(cudaMemsetAsync(e->ct.p + CT_N, 0, sizeof(unsigned long long), e->st));
    k_maxdisp<<<nblk(e->N, 256), 256, 0, e->st>>>(e->N, e->pos.p, e->xref.p, e->ct.p + CT_N);
    CKL();
    unsigned long long bits;
    CK(cudaMemcpyAsync(&bits, e->ct.p + CT_N, sizeof(bits), cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    double d2;
    std::memcpy(&d2, &bits, sizeof(d2));
    double half = 0.5 * e->hp.skin;
    if (d2 > half * half) return rebuild(e);
  }
  if (e->NT > e->N) {
    k_ghost_update<<<nblk(e->NT - e->N, 256), 256, 0, e->st>>>(e->N, e->NT, e->pos.p, e->owner.p, e->shift.p);
    CKL();
  }
  return AB_OK;
}

bool bad_ptr(ab_engine* e, const void* p, const char* what) {
  if (p) return false;
  e->err = std::string("NULL pointer: ") + what;
  return true;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

ab_status ab_create(const char* text, size_t len, ab_precision prec, int device, ab_engine** out) {
  if (!text || !out || (prec != AB_FP64 && prec != AB_MIXED)) {
    g_create_error = "ab_create: bad argument";
    return AB_E_ARG;
  }
  *out = nullptr;
  ab_engine* e = new ab_engine();
  std::string perr = parse_host_params(text, len, e->hp);
  if (!perr.empty()) {
    g_create_error = perr;
    delete e;
    return AB_E_PARAM;
  }
  e->prec = prec;
  e->dev = device;
  cudaDeviceProp prop;
  if (cudaSetDevice(device) != cudaSuccess || cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    g_create_error = "no CUDA device " + std::to_string(device);
    cudaGetLastError();
    delete e;
    return AB_E_CUDA;
  }
  if (prop.major != 10) {
    g_create_error = std::string("device is not sm_100 (Blackwell): ") + prop.name;
    delete e;
    return AB_E_CUDA;
  }
  std::snprintf(e->devname, sizeof(e->devname), "%s", prop.name);
  e->nsm = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking) != cudaSuccess) {
    g_create_error = "cudaStreamCreate failed";
    delete e;
    return AB_E_CUDA;
  }
  e->st = e->own;
  Tab<double> td;
  Tab<float> tf;
  fill_tab(e->hp, td);
  fill_tab(e->hp, tf);
  bool ok = cudaMemcpyToSymbol(c_tabd, &td, sizeof(td)) == cudaSuccess &&
            cudaMemcpyToSymbol(c_tabf, &tf, sizeof(tf)) == cudaSuccess &&
            e->scratch.ensure(SCRATCH_BYTES) == cudaSuccess &&
            cudaMemset(e->scratch.p, 0, SCRATCH_BYTES) == cudaSuccess &&
            cudaMallocHost(&e->h_ct, sizeof(unsigned long long) * (CT_N + 1)) == cudaSuccess &&
            cudaMallocHost(&e->h_acc, sizeof(double) * ACC_N) == cudaSuccess &&
            cudaMallocHost(&e->h_small, sizeof(int) * 8) == cudaSuccess;
  static_assert(sizeof(double) * ACC_N <= SCRATCH_CT, "scratch layout");
  static_assert(SCRATCH_CT + sizeof(unsigned long long) * (CT_N + 1) <= SCRATCH_SMALL, "scratch layout");
  if (ok) {  // views into the scratch block (not separately allocated)
    e->acc.p = reinterpret_cast<double*>(e->scratch.p), e->acc.n = ACC_N;
    e->ct.p = reinterpret_cast<unsigned long long*>(e->scratch.p + SCRATCH_CT), e->ct.n = CT_N + 1;
    e->small_i.p = reinterpret_cast<int*>(e->scratch.p + SCRATCH_SMALL), e->small_i.n = 16;
  }
  if (!ok) {
    g_create_error = std::string("CUDA init failed: ") + cudaGetErrorString(cudaGetLastError());
    ab_destroy(e);
    return AB_E_CUDA;
  }
  *out = e;
  return AB_OK;
}

void ab_destroy(ab_engine* e) {
  if (!e) return;
  cudaSetDevice(e->dev);
  if (e->st) cudaStreamSynchronize(e->st);
  DBuf<double4>* b4[] = {&e->pos, &e->pos_tmp, &e->xref};
  for (auto* b : b4) b->release();
  e->acc.p = nullptr, e->ct.p = nullptr, e->small_i.p = nullptr;  // views into scratch
  e->scratch.release();
  DBuf<double>* bd[] = {&e->vel, &e->vel_tmp, &e->F, &e->io, &e->q_M, &e->stage0, &e->stage1};
  for (auto* b : bd) b->release();
  DBuf<int>* bi[] = {&e->gid, &e->gid_tmp, &e->owner, &e->key, &e->key2, &e->val, &e->val2, &e->cell_start,
                     &e->gcnt, &e->goff, &e->ljc[0], &e->ljc[1], &e->ljc[2], &e->ljn[0], &e->ljn[1],
                     &e->ljn[2], &e->in_cnt, &e->in_nbr, &e->s_cnt, &e->s_nbr,
                     &e->small_i, &e->ovf_bond, &e->ovf_q};
  for (auto* b : bi) b->release();
  e->shift.release();
  e->typ.release();
  e->s_dr.release();
  e->s_w.release();
  e->s_N.release();
  e->bonds.release();
  e->q_item.release();
  e->ct.release();
  e->red_d.release();
  e->red_u.release();
  e->cub_tmp.release();
  if (e->h_ct) cudaFreeHost(e->h_ct);
  if (e->h_acc) cudaFreeHost(e->h_acc);
  if (e->h_small) cudaFreeHost(e->h_small);
  if (e->ev_disp) cudaEventDestroy(e->ev_disp);
  for (auto& p : e->pending) cudaEventDestroy(p.a), cudaEventDestroy(p.b);
  for (auto& x : e->pool) cudaEventDestroy(x);
  if (e->own) cudaStreamDestroy(e->own);
  delete e;
}

const char* ab_last_error(const ab_engine* e) { return e ? e->err.c_str() : g_create_error.c_str(); }

ab_status ab_set_stream(ab_engine* e, void* stream) {
  if (!e) return AB_E_ARG;
  cudaSetDevice(e->dev);
  CK(cudaStreamSynchronize(e->st));
  e->st = stream ? (cudaStream_t)stream : e->own;
  return AB_OK;
}

ab_status ab_set_box(ab_engine* e, const double L[3]) {
  if (!e) return AB_E_ARG;
  if (bad_ptr(e, L, "L")) return AB_E_ARG;
  for (int c = 0; c < 3; ++c)
    if (!(L[c] > 0.0) || !std::isfinite(L[c])) {
      e->err = "box edge " + std::to_string(c) + " must be finite and > 0";
      return AB_E_BOX;
    }
  cudaSetDevice(e->dev);
  for (int c = 0; c < 3; ++c) e->L[c] = L[c];
  e->have_box = true;
  e->lists_valid = false;
  e->forces_valid = false;
  return upload_geo(e);
}

ab_status ab_set_atoms(ab_engine* e, int64_t n, const int32_t* type, const double* xyz) {
  if (!e) return AB_E_ARG;
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
  std::vector<double4> p(n);
  std::vector<int> g(n);
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
    long long key = make_key((int)i, 0, 0, 0, type[i]);
    double kd;
    std::memcpy(&kd, &key, sizeof(kd));
    p[i] = make_double4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], kd);
    g[i] = (int)i;
  }
  e->N = (int)n;
  e->NT = (int)n;
  CK(e->pos.ensure((size_t)n + n / 4 + 64));
  CK(e->gid.ensure((size_t)n + n / 4 + 64));
  CK(e->vel.ensure(3 * (size_t)n));
  CK(e->F.ensure(3 * (size_t)n));
  CK(e->io.ensure(3 * (size_t)n));
  CK(cudaMemcpyAsync(e->pos.p, p.data(), sizeof(double4) * n, cudaMemcpyHostToDevice, e->st));
  CK(cudaMemcpyAsync(e->gid.p, g.data(), sizeof(int) * n, cudaMemcpyHostToDevice, e->st));
  CK(cudaMemsetAsync(e->vel.p, 0, sizeof(double) * 3 * n, e->st));
  CK(cudaStreamSynchronize(e->st));
  e->have_atoms = true;
  e->lists_valid = false;
  e->forces_valid = false;
  e->capL[0] = e->capL[1] = e->capL[2] = e->capI = 0;
  return AB_OK;
}

static ab_status need_atoms(ab_engine* e) {
  if (!e) return AB_E_ARG;
  if (!e->have_atoms) {
    e->err = "ab_set_atoms has not been called";
    return AB_E_STATE;
  }
  cudaSetDevice(e->dev);
  return AB_OK;
}

ab_status ab_set_positions(ab_engine* e, const double* xyz) {
  TRY(need_atoms(e));
  if (bad_ptr(e, xyz, "xyz")) return AB_E_ARG;
  CK(cudaMemcpyAsync(e->io.p, xyz, sizeof(double) * 3 * e->N, cudaMemcpyHostToDevice, e->st));
  k_from_caller_pos<<<nblk(e->N, 256), 256, 0, e->st>>>(e->N, e->gid.p, e->io.p, e->pos.p);
  CKL();
  e->forces_valid = false;
  return AB_OK;
}

ab_status ab_set_velocities(ab_engine* e, const double* v) {
  TRY(need_atoms(e));
  if (bad_ptr(e, v, "v")) return AB_E_ARG;
  CK(cudaMemcpyAsync(e->io.p, v, sizeof(double) * 3 * e->N, cudaMemcpyHostToDevice, e->st));
  k_from_caller_vec<<<nblk(e->N, 256), 256, 0, e->st>>>(e->N, e->gid.p, e->io.p, e->vel.p);
  CKL();
  return AB_OK;
}

ab_status ab_compute(ab_engine* e, double* f, double* energy, double virial[6], double terms[3]) {
  TRY(need_atoms(e));
  TRY(prepare(e, true));
  TRY(forces(e));
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
  e->want_virial = false;
  ab_status s = run_nve_impl(e, nsteps, dt, every, thermo);
  e->want_virial = true;
  return s;
}

static ab_status run_nve_impl(ab_engine* e, int64_t nsteps, double dt, int64_t every, double* thermo) {
  if (nsteps < 0 || !(dt > 0)) {
    e->err = "nsteps must be >= 0 and dt > 0";
    return AB_E_ARG;
  }
  cudaStream_t st = e->st;
  const int N = e->N;
  if (!e->forces_valid) {
    TRY(prepare(e, true));
    TRY(forces(e));
  }
  const HostParams& hp = e->hp;
  double dtf0 = 0.5 * dt * hp.ftm2v / hp.mass[0], dtf1 = 0.5 * dt * hp.ftm2v / hp.mass[1];
  int row = 0;
  auto record = [&](int64_t step) -> ab_status {
    CK(cudaMemsetAsync(e->acc.p + ACC_KE, 0, sizeof(double), st));
    k_ke<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->vel.p, hp.mass[0], hp.mass[1], e->acc.p);
    CKL();
    double ke;
    CK(cudaMemcpyAsync(&ke, e->acc.p + ACC_KE, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ke *= hp.mvv2e;
    double pe = e->E3[0] + e->E3[1] + e->E3[2];
    double* t = thermo + 4 * row++;
    t[0] = (double)step, t[1] = pe, t[2] = ke, t[3] = pe + ke;
    return AB_OK;
  };
  if (thermo && every > 0) TRY(record(0));
  // The rebuild decision (max displacement) is the only per-step host round trip and
  // it is hidden: after the drift the force kernels are enqueued speculatively on the current
  // lists (they only write F, the scratch block and the b* queue), the host then waits for the
  // displacement read-back alone and, if a rebuild is needed (rare), rebuilds and re-enqueues
  // the forces before the second half-kick.  Energies and counters stay on the device except on
  // thermo steps; the b* queue is sized so it cannot overflow, and the short-list overflow flag
  // of step s is read at step s+1.
  if (!e->ev_disp) CK(cudaEventCreateWithFlags(&e->ev_disp, cudaEventDisableTiming));
  for (int64_t s = 1; s <= nsteps; ++s) {
    const bool th = thermo && every > 0 && s % every == 0;
    CK(cudaMemsetAsync(e->ct.p + CT_N, 0, sizeof(unsigned long long), st));
    prof_begin(e, 4);
    k_integrate1<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->vel.p, e->F.p, dtf0, dtf1, dt, e->xref.p,
                                                e->ct.p + CT_N);
    CKL();
    prof_end(e);
    CK(cudaMemcpyAsync(e->h_ct, e->ct.p, sizeof(unsigned long long) * (CT_N + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e->ev_disp, st));
    bool speculated = false;
    if (e->lists_valid && !th) {
      TRY(prepare(e, false));
      TRY(forces(e, false));
      speculated = true;
    }
    CK(cudaEventSynchronize(e->ev_disp));
    if (e->h_ct[CT_OVF_SHORT]) {
      e->err = "an atom has more than 16 REBO short-list neighbours (NBMAX); unsupported geometry";
      return AB_E_STATE;
    }
    double d2;
    std::memcpy(&d2, &e->h_ct[CT_N], sizeof(d2));
    double half = 0.5 * hp.skin;
    if (d2 > half * half) e->lists_valid = false, speculated = false;
    if (!speculated) {
      TRY(prepare(e, false));
      TRY(forces(e, th));
    }
    prof_begin(e, 4);
    k_integrate2<<<nblk(N, 256), 256, 0, st>>>(N, e->pos.p, e->vel.p, e->F.p, dtf0, dtf1);
    CKL();
    prof_end(e);
    ++e->steps;
    if (th) TRY(record(s));
  }
  // no final synchronisation: the last step's kernels may still run; every call that returns
  // data (or the stream itself) orders after them
  CK(cudaGetLastError());
  return AB_OK;
}

ab_status ab_get_positions(ab_engine* e, double* xyz) {
  TRY(need_atoms(e));
  if (bad_ptr(e, xyz, "xyz")) return AB_E_ARG;
  k_to_caller_pos<<<nblk(e->N, 256), 256, 0, e->st>>>(e->N, e->gid.p, e->pos.p, e->io.p);
  CKL();
  CK(cudaMemcpyAsync(xyz, e->io.p, sizeof(double) * 3 * e->N, cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  return AB_OK;
}

ab_status ab_get_velocities(ab_engine* e, double* v) {
  TRY(need_atoms(e));
  if (bad_ptr(e, v, "v")) return AB_E_ARG;
  k_to_caller_vec<<<nblk(e->N, 256), 256, 0, e->st>>>(e->N, e->gid.p, e->vel.p, e->io.p);
  CKL();
  CK(cudaMemcpyAsync(v, e->io.p, sizeof(double) * 3 * e->N, cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  return AB_OK;
}

ab_status ab_get_forces(ab_engine* e, double* f) {
  TRY(need_atoms(e));
  if (bad_ptr(e, f, "f")) return AB_E_ARG;
  if (!e->forces_valid) {
    e->err = "no force evaluation at the current positions";
    return AB_E_STATE;
  }
  k_to_caller_vec<<<nblk(e->N, 256), 256, 0, e->st>>>(e->N, e->gid.p, e->F.p, e->io.p);
  CKL();
  CK(cudaMemcpyAsync(f, e->io.p, sizeof(double) * 3 * e->N, cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  return AB_OK;
}

ab_status ab_get_list(ab_engine* e, ab_list which, int64_t* count, int64_t* rows) {
  TRY(need_atoms(e));
  if (bad_ptr(e, count, "count")) return AB_E_ARG;
  if (which != AB_LIST_SHORT && which != AB_LIST_BONDS && which != AB_LIST_LJ) {
    e->err = "unknown list";
    return AB_E_ARG;
  }
  if (!e->forces_valid) {
    TRY(prepare(e, true));
    TRY(forces(e));
  }
  const int N = e->N, NT = e->NT;
  std::vector<int> gid(NT);
  std::vector<char4> sh(NT);
  std::vector<double4> pos(NT);
  CK(cudaMemcpyAsync(gid.data(), e->gid.p, sizeof(int) * NT, cudaMemcpyDeviceToHost, e->st));
  CK(cudaMemcpyAsync(sh.data(), e->shift.p, sizeof(char4) * NT, cudaMemcpyDeviceToHost, e->st));
  CK(cudaMemcpyAsync(pos.data(), e->pos.p, sizeof(double4) * NT, cudaMemcpyDeviceToHost, e->st));
  // (count, neighbour) tables of the requested list(s)
  int nl = which == AB_LIST_LJ ? 3 : 1;
  std::vector<int> cnt[3], nbr[3];
  int cap[3];
  for (int c = 0; c < nl; ++c) {
    cap[c] = which == AB_LIST_LJ ? e->capL[c] : e->capS;
    const int* dc = which == AB_LIST_LJ ? e->ljc[c].p : e->s_cnt.p;
    const int* dn = which == AB_LIST_LJ ? e->ljn[c].p : e->s_nbr.p;
    cnt[c].resize(N);
    nbr[c].resize((size_t)N * cap[c]);
    CK(cudaMemcpyAsync(cnt[c].data(), dc, sizeof(int) * N, cudaMemcpyDeviceToHost, e->st));
    CK(cudaMemcpyAsync(nbr[c].data(), dn, sizeof(int) * N * (size_t)cap[c], cudaMemcpyDeviceToHost, e->st));
  }
  CK(cudaStreamSynchronize(e->st));
  auto type_h = [&](int a) {
    long long k;
    std::memcpy(&k, &pos[a].w, sizeof(k));
    return (int)(k & 3);
  };
  std::vector<std::array<int64_t, 5>> out;
  for (int c = 0; c < nl; ++c)
    for (int i = 0; i < N; ++i)
      for (int q = 0; q < cnt[c][i]; ++q) {
        int J = nbr[c][(size_t)i * cap[c] + q];
        char4 s = sh[J];
        bool canon = gid[i] != gid[J] ? gid[i] < gid[J]
                                      : (s.x > 0 || (s.x == 0 && (s.y > 0 || (s.y == 0 && s.z > 0))));
        if (which != AB_LIST_SHORT && !canon) continue;
        if (which == AB_LIST_LJ) {  // exact (un-fused) r^2 <= r_c^2 as on the device
          volatile double dx = pos[J].x - pos[i].x, dy = pos[J].y - pos[i].y, dz = pos[J].z - pos[i].z;
          volatile double a = dx * dx, b = dy * dy, cc = dz * dz;
          volatile double ab = a + b;
          double r2 = ab + cc;
          double rc = e->hp.pr[type_h(i) + type_h(J)].rc;
          if (!(r2 <= rc * rc)) continue;
        }
        out.push_back({gid[i], gid[J], s.x, s.y, s.z});
      }
  std::sort(out.begin(), out.end());
  *count = (int64_t)out.size();
  if (rows)
    for (size_t r = 0; r < out.size(); ++r)
      for (int c = 0; c < 5; ++c) rows[5 * r + c] = out[r][c];
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
  s->n_atoms = e->N, s->n_ghosts = e->G, s->n_rebuilds = e->rebuilds, s->n_steps = e->steps;
  s->n_overflow_retries = e->retries + c[CT_OVF_REACH];
  s->lj_capacity = e->capL[0] + e->capL[1] + e->capL[2], s->inter_capacity = e->capI;
  s->n_lj_entries = c[CT_LJENT], s->n_angles = c[CT_ANGLES];
  s->n_lj_far = c[CT_LJFAR], s->n_lj_entries_far = c[CT_LJENTFAR];
  return AB_OK;
}

ab_status ab_record_stages(ab_engine* e, int on) {
  if (!e) return AB_E_ARG;
  e->record = on != 0;
  e->forces_valid = false;
  return AB_OK;
}

ab_status ab_get_stage(ab_engine* e, int stage, int64_t* count, double* out) {
  TRY(need_atoms(e));
  if (bad_ptr(e, count, "count")) return AB_E_ARG;
  if ((stage != 0 && stage != 1) || !e->record || !e->forces_valid) {
    e->err = "stage must be 0 or 1, recording on (ab_record_stages) and forces evaluated";
    return AB_E_STATE;
  }
  int n[2];
  CK(cudaMemcpyAsync(n, e->small_i.p + 6, 2 * sizeof(int), cudaMemcpyDeviceToHost, e->st));
  CK(cudaStreamSynchronize(e->st));
  int width = stage == 0 ? 13 : 7;
  int rows = n[stage];
  *count = rows;
  if (out && rows)
    CK(cudaMemcpy(out, stage == 0 ? e->stage0.p : e->stage1.p, sizeof(double) * width * rows,
                  cudaMemcpyDeviceToHost));
  return AB_OK;
}

ab_status ab_set_profiling(ab_engine* e, int on) {
  if (!e) return AB_E_ARG;
  cudaSetDevice(e->dev);
  CK(cudaStreamSynchronize(e->st));
  prof_collect(e);
  e->prof = on != 0;
  for (int q = 0; q < AB_NPHASE; ++q) e->phase_ms[q] = 0, e->phase_n[q] = 0;
  return AB_OK;
}

ab_status ab_get_phase_ms(ab_engine* e, double ms[AB_NPHASE], int64_t n[AB_NPHASE]) {
  if (!e || !ms || !n) return AB_E_ARG;
  cudaSetDevice(e->dev);
  CK(cudaStreamSynchronize(e->st));
  prof_collect(e);
  for (int q = 0; q < AB_NPHASE; ++q) ms[q] = e->phase_ms[q], n[q] = e->phase_n[q];
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
  if (launches) *launches = e->launches;
  return AB_OK;
}

}  // extern "C"
