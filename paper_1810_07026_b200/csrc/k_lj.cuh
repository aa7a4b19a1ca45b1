// k_lj.cuh -- the LJ term gated by C_ij (Alg. 3; E = Q C V) with the
// per-atom reach set of the C_ij connectivity switch.
//
// GPU mapping: one warp per local atom i, streaming i's FULL skinned LJ lists (both directions,
// so no force scatter onto j: every pair is evaluated from both ends and F_i is a gather).
//   near list (r_b <= 3 r_max + skin): the warp first maps out every atom image reachable from i
//     in 1, 2 or 3 bonds with the maximum path-weight product M (the paper's "map out all the
//     atoms j connected to atom i once") into an open-addressing table in shared memory
//     (keys = image index, value = M via atomicMax on its bit pattern, M >= 0).  Overflow
//     -> the direct nested search of P:844-853 for that atom ("sequential fallback").
//     Per pair: cutoff, C = 1 - M (lookup within 3 r_max), skip if C == 0 (gate order of
//     P:824-830), pairs inside the S_r window are deferred to the b* batch (canonical direction
//     only), others give E/2 = C V/2 and the pair force on i.
//   pure list: C = Q = S_taper = 1 guaranteed by the build: branch-free 12-6 LJ.
//   band list: C = Q = 1; cutoff and taper per pair.
// Forces from dC (0 < C < 1, reactive systems only) are applied once, by the canonical direction.
// Counters count canonical directions only (key_i < key_J), so they equal the oracle's half sums.
#pragma once
#include "dev_common.cuh"
#include "k_bond.cuh"

namespace ab {

constexpr int LJ_WARPS = 4;
constexpr int TWOHOP_CAP = NBMAX * NBMAX;

struct ReachSmem {
  int keys[REACH_SLOTS];
  unsigned long long mbits[REACH_SLOTS];
  int two_l[TWOHOP_CAP];
  double two_w[TWOHOP_CAP];
  int ntwo, nins, ovf;
};

__device__ __forceinline__ unsigned reach_hash(int key) { return ((unsigned)key * 2654435761u) >> 24; }

__device__ __forceinline__ void reach_insert(ReachSmem& s, int key, double M) {
  unsigned h = reach_hash(key) & (REACH_SLOTS - 1);
  for (int probe = 0; probe < REACH_SLOTS; ++probe) {
    int old = atomicCAS(&s.keys[h], REACH_EMPTY, key);
    if (old == REACH_EMPTY || old == key) {
      if (old == REACH_EMPTY) atomicAdd(&s.nins, 1);
      atomicMax(&s.mbits[h], (unsigned long long)__double_as_longlong(M));
      return;
    }
    h = (h + 1) & (REACH_SLOTS - 1);
  }
  s.ovf = 1;
}

__device__ __forceinline__ double reach_lookup(const ReachSmem& s, int key) {
  unsigned h = reach_hash(key) & (REACH_SLOTS - 1);
  for (int probe = 0; probe < REACH_SLOTS; ++probe) {
    int k = s.keys[h];
    if (k == key) return __longlong_as_double((long long)s.mbits[h]);
    if (k == REACH_EMPTY) return 0.0;
    h = (h + 1) & (REACH_SLOTS - 1);
  }
  return 0.0;
}

// plain 12-6 part: V0 = 4 eps (sr^12 - sr^6) and (dV0/dr)/r, with sr^2 = sigma^2 / r^2
template <typename R>
__device__ __forceinline__ R lj_plain(R e4, R sig2, R inv_r2, R& dVr) {
  R sr2 = sig2 * inv_r2;
  R sr6 = sr2 * sr2 * sr2;
  dVr = e4 * (R(6) * sr6 - R(12) * sr6 * sr6) * inv_r2;
  return e4 * (sr6 * sr6 - sr6);
}

struct LJArgs {
  int N;
  const double4* pos;
  int cap[3];
  const int* cnt[3];
  const int* nbr[3];
};

template <typename R>
__device__ __forceinline__ R to_r(double x) {
  return (R)x;
}

template <typename R, bool VIRIAL>
__global__ void __launch_bounds__(32 * LJ_WARPS) k_lj(LJArgs A, ShortList<R> S, const int* owner, const int* gid,
                                                     const char4* shift, double* F, double* acc,
                                                     unsigned long long* ct, BstarQueue Qu, StageBuf stage) {
  __shared__ ReachSmem sm_all[LJ_WARPS];
  const Tab<R>& T = tab<R>();
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ReachSmem& s = sm_all[warp];
  int i = blockIdx.x * LJ_WARPS + warp;
  if (i >= A.N) return;  // whole warp exits together

  const double4 pi = A.pos[i];
  const int ti = type_of(pi);
  const long long ki = key_of(pi);
  double fx = 0, fy = 0, fz = 0, en = 0;
  double W[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long nlj = 0, nc0 = 0;

  // ------------------------------------------------------------ near list
  const int cntN = A.cnt[0][i];
  if (cntN > 0) {
    // 1. reach set of i (1-, 2-, 3-bond paths)
    for (int q = lane; q < REACH_SLOTS; q += 32) {
      s.keys[q] = REACH_EMPTY;
      s.mbits[q] = 0ull;
    }
    if (lane == 0) s.ntwo = 0, s.nins = 0, s.ovf = 0;
    __syncwarp();
    size_t bi = (size_t)i * S.capS;
    int ni = S.cnt[i];
    if (lane < ni) {
      int k = S.nbr[bi + lane];
      R w1 = S.w[bi + lane].x;
      reach_insert(s, k, (double)w1);
      size_t bk = (size_t)k * S.capS;
      int nk = S.cnt[k];
      for (int b = 0; b < nk; ++b) {
        int l = S.nbr[bk + b];
        if (l == i) continue;
        R w12 = w1 * S.w[bk + b].x;
        reach_insert(s, l, (double)w12);
        int slot = atomicAdd(&s.ntwo, 1);
        s.two_l[slot] = l;
        s.two_w[slot] = (double)w12;
      }
    }
    __syncwarp();
    int ntwo = s.ntwo;
    for (int t = lane; t < ntwo; t += 32) {
      int l = s.two_l[t];
      R w12 = (R)s.two_w[t];
      size_t bl = (size_t)l * S.capS;
      int nl = S.cnt[l];
      for (int c = 0; c < nl; ++c) {
        int m = S.nbr[bl + c];
        if (m == i) continue;
        reach_insert(s, m, (double)(w12 * S.w[bl + c].x));
      }
    }
    __syncwarp();
    const bool ovf = s.ovf != 0;
    // 2. pairs
    const int* row = A.nbr[0] + (size_t)i * A.cap[0];
    for (int q = lane; q < cntN; q += 32) {
      int J = row[q];
      double4 pj = A.pos[J];
      double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
      double r2 = r2_exact(dx, dy, dz);
      int p = ti + type_of(pj);
      if (r2 > c_geo.rc2[p]) continue;
      bool canon = ki < key_of(pj);
      nlj += canon;
      double Md = 0.0;
      if (r2 <= c_geo.reach2) Md = ovf ? (double)path_search(S, i, J).M : reach_lookup(s, J);
      if (Md == 1.0) {  // C_ij == 0 (Alg. 3 "continue")
        nc0 += canon;
        if (canon && stage.rows) {
          double* rw = stage_row(stage, 7);
          if (rw) {
            char4 sh = shift[J];
            rw[0] = gid[i], rw[1] = gid[J], rw[2] = sh.x, rw[3] = sh.y, rw[4] = sh.z, rw[5] = 0.0, rw[6] = 0.0;
          }
        }
        continue;
      }
      double rd = sqrt(r2);
      // S_r(r) != 0 decided in fp64 in both precision modes (gates on r are fp64, reading A14)
      double tP = (rd - c_tabd.sigma[p]) / (c_tabd.srhi[p] - c_tabd.sigma[p]);
      if (tP < 1.0) {  // deferred b* batch, whole pair evaluated once by the canonical direction
        if (canon) {
          int k = atomicAdd(Qu.count, 1);
          if (k < Qu.cap) {
            Qu.item[k] = make_int4(i, J, 0, 0);
            Qu.M[k] = Md;
          } else {
            atomicAdd(ct + CT_OVF_QUEUE, 1ull);
          }
        }
        continue;
      }
      R dVr;
      R V = lj_plain<R>(R(4) * T.eps[p], T.sigma2[p], R(1) / (R)r2, dVr);
      if (r2 > c_geo.rlo2[p]) {  // taper S(r; r_lo, r_c) (reading A10)
        R r = (R)rd, dsw;
        R sv = sw<R>(r, T.rlo[p], T.rc[p], dsw);
        dVr = dVr * sv + V * dsw / r;
        V = V * sv;
      }
      R C = R(1) - (R)Md;
      R fr = C * dVr;  // F_i += fr d  (E(d), d = x_j - x_i)
      fx += (double)(fr * (R)dx);
      fy += (double)(fr * (R)dy);
      fz += (double)(fr * (R)dz);
      en += (double)(C * V);
      if (VIRIAL) {
        V3<R> dd = mk3<R>((R)dx, (R)dy, (R)dz);
        vir_add(W, dd, (R(0.5) * fr) * dd);
      }
      if (canon && Md > 0.0) {  // 0 < C < 1: dC/dx along the maximising path, once per pair
        PathRes<R> pr = path_search(S, i, J);
        double Wp[6] = {0, 0, 0, 0, 0, 0};
        path_forces(S, owner, pr, -V, F, Wp);
        if (VIRIAL)
          for (int c = 0; c < 6; ++c) W[c] += Wp[c];
      }
      if (canon && stage.rows) {
        double* rw = stage_row(stage, 7);
        if (rw) {
          char4 sh = shift[J];
          rw[0] = gid[i], rw[1] = gid[J], rw[2] = sh.x, rw[3] = sh.y, rw[4] = sh.z, rw[5] = (double)C, rw[6] = 0.0;
        }
      }
    }
    if (lane == 0) {
      atomicMax(ct + CT_MAXREACH, (unsigned long long)s.nins);
      if (ovf) atomicAdd(ct + CT_OVF_REACH, 1ull);
    }
  }

  // ------------------------------------------------------------ pure list: plain 12-6 LJ
  {
    const int cnt = A.cnt[1][i];
    const int* row = A.nbr[1] + (size_t)i * A.cap[1];
    for (int q = lane; q < cnt; q += 32) {
      int J = row[q];
      double4 pj = A.pos[J];
      double dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
      int p = ti + type_of(pj);
      nlj += ki < key_of(pj);
      R rx = (R)dx, ry = (R)dy, rz = (R)dz;
      R dVr;
      R V = lj_plain<R>(R(4) * T.eps[p], T.sigma2[p], R(1) / (rx * rx + ry * ry + rz * rz), dVr);
      fx += (double)(dVr * rx);
      fy += (double)(dVr * ry);
      fz += (double)(dVr * rz);
      en += (double)V;
      if (VIRIAL) {
        V3<R> dd = mk3<R>(rx, ry, rz);
        vir_add(W, dd, (R(0.5) * dVr) * dd);
      }
      if (stage.rows && ki < key_of(pj)) {
        double* rw = stage_row(stage, 7);
        if (rw) {
          char4 sh = shift[J];
          rw[0] = gid[i], rw[1] = gid[J], rw[2] = sh.x, rw[3] = sh.y, rw[4] = sh.z, rw[5] = 1.0, rw[6] = 0.0;
        }
      }
    }
  }

  // ------------------------------------------------------------ band list: cutoff + taper
  {
    const int cnt = A.cnt[2][i];
    const int* row = A.nbr[2] + (size_t)i * A.cap[2];
    for (int q = lane; q < cnt; q += 32) {
      int J = row[q];
      double4 pj = A.pos[J];
      double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
      double r2 = r2_exact(dx, dy, dz);
      int p = ti + type_of(pj);
      if (r2 > c_geo.rc2[p]) continue;
      bool canon = ki < key_of(pj);
      nlj += canon;
      R dVr;
      R V = lj_plain<R>(R(4) * T.eps[p], T.sigma2[p], R(1) / (R)r2, dVr);
      if (r2 > c_geo.rlo2[p]) {
        R r = (R)sqrt(r2), dsw;
        R sv = sw<R>(r, T.rlo[p], T.rc[p], dsw);
        dVr = dVr * sv + V * dsw / r;
        V = V * sv;
      }
      fx += (double)(dVr * (R)dx);
      fy += (double)(dVr * (R)dy);
      fz += (double)(dVr * (R)dz);
      en += (double)V;
      if (VIRIAL) {
        V3<R> dd = mk3<R>((R)dx, (R)dy, (R)dz);
        vir_add(W, dd, (R(0.5) * dVr) * dd);
      }
      if (canon && stage.rows) {
        double* rw = stage_row(stage, 7);
        if (rw) {
          char4 sh = shift[J];
          rw[0] = gid[i], rw[1] = gid[J], rw[2] = sh.x, rw[3] = sh.y, rw[4] = sh.z, rw[5] = 1.0, rw[6] = 0.0;
        }
      }
    }
  }

  // ------------------------------------------------------------ reductions
  fx = warp_sum(fx);
  fy = warp_sum(fy);
  fz = warp_sum(fz);
  if (lane == 0) atomic_add3(F, i, fx, fy, fz);
  double e1[1] = {0.5 * en};
  warp_acc(e1, acc + ACC_ELJ);
  if (VIRIAL) warp_acc(W, acc + ACC_W);
  unsigned long long s1 = warp_sum_u(nlj), s2 = warp_sum_u(nc0);
  if (lane == 0) {
    if (s1) atomicAdd(ct + CT_LJ, s1);
    if (s2) atomicAdd(ct + CT_C0, s2);
    atomicAdd(ct + CT_LJENT, (unsigned long long)(A.cnt[0][i] + A.cnt[1][i] + A.cnt[2][i]));
  }
}

}  // namespace ab
