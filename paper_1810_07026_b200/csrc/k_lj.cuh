// k_lj.cuh -- the LJ term gated by C_ij (Alg. 3; E = Q C V) with the
// per-atom reach set of the C_ij connectivity switch.
//
// GPU mapping: one warp per local atom i.
//   1. The warp maps out every atom image reachable from i in 1, 2 or 3 bonds with the maximum
//      path-weight product M (the paper's "map out all the atoms j connected to atom i once",
//      P:862) into an open-addressing table in shared memory (256 slots per warp, keys =
//      image index, value = M with atomicMax on its bit pattern, M >= 0).  Overflow -> the direct
//      nested search of P:844-853 is used for that atom (the paper's "sequential fallback").
//   2. Lanes stream i's FULL skinned LJ list (both directions, no force scatter to j): distance
//      gate r <= r_c, C = 1 - M by table lookup (only within 3 r_max), skip if C == 0 (gate order
//      of P:824-830), pairs inside the S_r window are deferred to the b* batch (canonical
//      direction only), all others give E/2 = C V/2 and the pair force on i.
//   3. Warp-reduce F_i, E and the virial; one fp64 atomic per component per atom.
// Forces from dC (0 < C < 1, reactive systems only) are applied once, by the canonical direction.
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

template <typename R>
__global__ void __launch_bounds__(32 * LJ_WARPS) k_lj(int N, const double4* pos, const int* lj_cnt,
                                                     const int* lj_nbr, int capLJ, ShortList<R> S,
                                                     const signed char* typ, const int* owner, const int* gid,
                                                     const char4* shift, double* F, double* acc,
                                                     unsigned long long* ct, BstarQueue Qu, StageBuf stage) {
  __shared__ ReachSmem sm_all[LJ_WARPS];
  const Tab<R>& T = tab<R>();
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ReachSmem& s = sm_all[warp];
  int i = blockIdx.x * LJ_WARPS + warp;
  if (i >= N) return;  // whole warp exits together

  // ---- 1. reach set of i
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
    double w1 = (double)S.w[bi + lane].x;
    reach_insert(s, k, w1);
    size_t bk = (size_t)k * S.capS;
    int nk = S.cnt[k];
    for (int b = 0; b < nk; ++b) {
      int l = S.nbr[bk + b];
      if (l == i) continue;
      R w12 = (R)w1 * S.w[bk + b].x;
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

  // ---- 2. pair loop over the full skinned LJ list
  double4 pi = pos[i];
  int ti = typ[i];
  int gi = gid[i];
  double fx = 0, fy = 0, fz = 0;
  double e[1 + 6] = {0, 0, 0, 0, 0, 0, 0};
  double Wpath[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long nlj = 0, nc0 = 0;
  int cnt = lj_cnt[i];
  const int* row = lj_nbr + (size_t)i * capLJ;
  for (int q = lane; q < cnt; q += 32) {
    int J = row[q];
    double4 pj = pos[J];
    double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
    double r2 = r2_exact(dx, dy, dz);
    int tj = typ[J];
    int p = ti + tj;
    if (r2 > c_geo.rc2[p]) continue;
    bool canon = canonical_pair(gi, gid[J], shift[J]);
    nlj += canon;
    double Md = 0.0;
    if (r2 <= c_geo.reach2) {
      if (!ovf) Md = reach_lookup(s, J);
      else Md = (double)path_search(S, i, J).M;
    }
    if (Md == 1.0) {  // C_ij == 0 (Alg. 3 "continue")
      nc0 += canon;
      if (canon && stage.rows) {
        double* rw = stage_row(stage, 7);
        if (rw) {
          char4 sh = shift[J];
          rw[0] = gi, rw[1] = gid[J], rw[2] = sh.x, rw[3] = sh.y, rw[4] = sh.z, rw[5] = 0.0, rw[6] = 0.0;
        }
      }
      continue;
    }
    double rd = sqrt(r2);
    // S_r(r) != 0 decided in fp64 in both precision modes (gates on r are fp64, reading A14)
    double tP = (rd - c_tabd.sigma[p]) / (c_tabd.srhi[p] - c_tabd.sigma[p]);
    if (tP < 1.0) {  // deferred b* batch
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
    R V = lj_v<R>(p, (R)r2, r2, dVr);
    R C = R(1) - (R)Md;
    R fr = C * dVr;  // F_i += fr d  (E(d), d = x_j - x_i)
    fx += (double)(fr * (R)dx);
    fy += (double)(fr * (R)dy);
    fz += (double)(fr * (R)dz);
    e[0] += 0.5 * (double)(C * V);
    V3<R> dd = mk3<R>((R)dx, (R)dy, (R)dz);
    V3<R> gg = (R(0.5) * fr) * dd;
    vir_add(e + 1, dd, gg);
    if (canon && Md > 0.0) {  // 0 < C < 1: dC/dx along the maximising path, once per pair
      PathRes<R> pr = path_search(S, i, J);
      path_forces(S, owner, pr, -V, F, Wpath);
    }
    if (canon && stage.rows) {
      double* rw = stage_row(stage, 7);
      if (rw) {
        char4 sh = shift[J];
        rw[0] = gi, rw[1] = gid[J], rw[2] = sh.x, rw[3] = sh.y, rw[4] = sh.z, rw[5] = (double)C, rw[6] = 0.0;
      }
    }
  }
  // ---- 3. reductions
  fx = warp_sum(fx);
  fy = warp_sum(fy);
  fz = warp_sum(fz);
  if (lane == 0) atomic_add3(F, i, fx, fy, fz);
  for (int c = 0; c < 6; ++c) e[1 + c] += Wpath[c];
  double e1[1] = {e[0]};
  warp_acc(e1, acc + ACC_ELJ);
  double w6[6] = {e[1], e[2], e[3], e[4], e[5], e[6]};
  warp_acc(w6, acc + ACC_W);
  unsigned long long s1 = warp_sum_u(nlj), s2 = warp_sum_u(nc0);
  if (lane == 0) {
    if (s1) atomicAdd(ct + CT_LJ, s1);
    if (s2) atomicAdd(ct + CT_C0, s2);
    atomicMax(ct + CT_MAXREACH, (unsigned long long)s.nins);
    atomicAdd(ct + CT_LJENT, (unsigned long long)cnt);
    if (ovf) atomicAdd(ct + CT_OVF_REACH, 1ull);
  }
}

}  // namespace ab
