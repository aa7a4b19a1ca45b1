// k_ljc.cuh -- the LJ term gated by C_ij (Alg. 3; E = Q C V) over j-clusters,
// with the per-atom C_ij reach set.  One kernel for every LJ pair.
//
// One warp per local atom i (grid-stride):
//   1. reach set of i: every atom image reachable in 1, 2 or 3 bonds with its maximal path
//      product M ("map out all the atoms j connected to atom i once") in a 64-slot
//      shared-memory hash table behind a 512-bit Bloom filter.  The walk is spread over
//      the warp: lane k takes the k-th short-list neighbour, the (k, l) pairs are spread over all
//      lanes, each lane walks its own l's neighbours m.  Products keep the association
//      (w_ik w_kl) w_lm of the nested enumeration.  Overflow -> the direct nested search
//       per pair (the paper's "sequential fallback").
//   2. filter: the warp streams i's cluster list 8 clusters (32 atom slots) at a time -- the 4
//      slots of a cluster are one 128-byte line of cpos -- and computes the exact (un-fused)
//      r^2 of each slot.  Pairs inside r_c(t_i, t_j) are compacted (warp ballot) into one of
//      three per-warp shared-memory ring queues:
//        near  r <= 3 r_max,max: may have C < 1 (reach lookup) or need b* (S_r window)
//        pure  3 r_max < r <= r_lo: C = Q = S_taper = 1, plain 12-6 (or Morse) pair
//        band  r_lo < r <= r_c:     C = Q = 1, tapered (reading A10)
//      Slots outside r_c (skin, empty slots, i itself) never reach the arithmetic.
//   3. evaluate: whenever a queue holds 32 pairs the warp evaluates them, one pair per lane, all
//      lanes doing the same kind of work (no masked taper / lookup code in the common batches).
//      E/2 = C V/2 per direction (each pair is met from both ends), the pair force on i only.
//      Near pairs: C = 1 - M (fp64 gate, reading A14); C = 0 skipped (Alg. 3 "continue"); pairs
//      that may lie in the S_r window (r^2 < (2^(1/6) sigma)^2 (1 + 1e-9)) are queued for the b*
//      batch by the canonical side and skipped here; forces from dC (0 < C < 1) are
//      applied once, by the canonical side, along the maximising path.
// Counters count canonical directions only (key_i < key_J): they equal the oracle's half sums.
#pragma once
#include <type_traits>
#include "dev_common.cuh"
#include "k_bond.cuh"
#include "k_cluster.cuh"
#include "k_lj.cuh"

namespace ab {

constexpr int LJC_Q = 64;  // ring capacity per queue (<= 31 left over + 32 appended)
template <typename R>
struct LjcQueue {
  double dx[LJC_Q], dy[LJC_Q], dz[LJC_Q], r2[LJC_Q];
  int J[LJC_Q];
  int pc[LJC_Q];  // species pair | canonical << 2
};
template <typename R>
struct LjcPar {  // the two species pairs a warp-uniform centre species can form (index h = t_j)
  R e4[2], s2[2], re[2], rlo[2], rc[2], iv[2];
  double rlo2[2], rc2[2], win2[2];
};
template <typename R>
struct LjcWarp {
  ReachSmem<NEAR_SLOTS> s;
  LjcQueue<R> q[3];
  LjcPar<R> P;  // per-warp copy (shared memory: keeps the registers for the pair arithmetic)
};

struct LjcArgs {
  int N;
  const double4* pos;
  const double4* cpos;
  const int* cl_atom;
  int cap;
  const int* cnt;
  const int* nbr;
};

// reach set of atom i over the short list, one warp (see header)
template <typename R>
__device__ __forceinline__ void reach_build_warp(ReachSmem<NEAR_SLOTS>& s, const ShortList<R>& S, int i) {
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < NEAR_SLOTS; q += 32) s.keys[q] = REACH_EMPTY, s.mbits[q] = 0ull;
#if AB_NEAR_BLOOM
  for (int q = lane; q < AB_NEAR_BLOOM; q += 32) s.bloom[q] = 0u;
#endif
  if (lane == 0) s.nins = 0, s.ovf = 0;
  __syncwarp();
  const size_t bi = (size_t)i * S.capS;
  const int ni = S.cnt[i];
  int k1 = -1, n1 = 0;
  double w1 = 0.0;
  if (lane < ni) {
    k1 = S.nbr[bi + lane];
    w1 = S.wd[bi + lane];
    n1 = S.cnt[k1];
    reach_insert(s, k1, w1);
  }
  int incl = n1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const int excl = incl - n1;
  const int T2 = __shfl_sync(0xffffffffu, incl, 31);
  for (int base = 0; base < T2; base += 32) {
    const int e = base + lane;
    // owner lane t of entry e: the last lane with excl_t <= e (5-step search over the warp)
    int t = 0;
#pragma unroll
    for (int b = 16; b > 0; b >>= 1) {
      const int ex = __shfl_sync(0xffffffffu, excl, t + b);
      if (t + b < 32 && ex <= e) t += b;
    }
    const int k = __shfl_sync(0xffffffffu, k1, t);
    const double wk = __shfl_sync(0xffffffffu, w1, t);
    const int off = e - __shfl_sync(0xffffffffu, excl, t);
    if (e < T2) {
      const size_t ek = (size_t)k * S.capS + off;
      const int l = S.nbr[ek];
      if (l != i) {
        const double w12 = wk * S.wd[ek];
        reach_insert(s, l, w12);
        const size_t bl = (size_t)l * S.capS;
        const int nl = S.cnt[l];
        for (int c = 0; c < nl; ++c) {
          const int m = S.nbr[bl + c];
          if (m == i) continue;
          reach_insert(s, m, w12 * S.wd[bl + c]);
        }
      }
    }
  }
  __syncwarp();
}

template <class T>
__device__ __forceinline__ T pick(const T (&a)[2], int h) {
  return a[h];
}

// rare paths out of line (their register demand would otherwise be the whole kernel's)
template <typename R>
__device__ __noinline__ double ljc_path_M(const ShortList<R>& S, int i, int J) {
  return path_search(S, i, J).M;
}
// Wsh: the block's shared virial row (nullptr: no virial)
template <typename R, bool SG>
__device__ __noinline__ void ljc_path_forces(const ShortList<R>& S, const int* owner, int i, int J, R V, double* F,
                                             double* Wsh) {
  PathRes<R> pr = path_search(S, i, J);
  double Wp[6] = {0, 0, 0, 0, 0, 0};
  path_forces<R, SG>(S, owner, pr, -V, F, Wp);
  if (Wsh)
    for (int c = 0; c < 6; ++c) atomicAdd(Wsh + c, Wp[c]);
}

// pair energy and (dV/dr)/r: 12-6 (or Morse) x taper (band only)
template <typename R, bool MORSE, bool BAND>
__device__ __forceinline__ R ljc_pair(const LjcPar<R>& P, int h, R rr2, R& dVr) {
  R y = (BAND || MORSE) ? rsqrt_fast(rr2) : R(0);  // 1/r (taper / Morse only)
  R V = MORSE ? morse_plain<R>(pick(P.e4, h), pick(P.s2, h), pick(P.re, h), rr2 * y, y, dVr)
              : lj_plain<R>(pick(P.e4, h), pick(P.s2, h), BAND ? y * y : rcp_fast(rr2), dVr);
  if (BAND) {  // taper S(r; r_lo, r_c) (reading A10); every band pair has r > r_lo
    R r = rr2 * y;
    R tt = (r - pick(P.rlo, h)) * pick(P.iv, h);
    R sv, ds;
    halfcos_poly(tt < R(0) ? R(0) : (tt > R(1) ? R(1) : tt), sv, ds);
    ds *= pick(P.iv, h);
    dVr = dVr * sv + V * ds * y;
    V = V * sv;
  }
  return V;
}

template <typename R, bool VIRIAL, bool SG>
__device__ __forceinline__ void ljc_acc(R fr, double dx, double dy, double dz, R V, double& fx, double& fy,
                                        double& fz, double& en, double (&W)[6]) {
  const R rx = (R)dx, ry = (R)dy, rz = (R)dz;
  fx = acc_round<SG>(fx + (double)(fr * rx));
  fy = acc_round<SG>(fy + (double)(fr * ry));
  fz = acc_round<SG>(fz + (double)(fr * rz));
  en = acc_round<SG>(en + (double)V);
  if (VIRIAL) {
    V3<R> dd = mk3<R>(rx, ry, rz);
    vir_add(W, dd, (R(0.5) * fr) * dd);
  }
}

template <typename R, bool VIRIAL, bool MORSE, bool SG = false>
#ifndef AB_LJC_MINBLOCKS
#define AB_LJC_MINBLOCKS 4
#endif
__global__ void __launch_bounds__(128, AB_LJC_MINBLOCKS) k_ljc(LjcArgs A, ShortList<R> S, const int* owner,
                                                               const int* gid, const char4* shift, double* F,
                                                               unsigned long long* ct, BstarQueue Qu,
                                                               StageBuf stage, RedRows RR) {
  __shared__ LjcWarp<R> wsm[4];
  __shared__ RedSmem rs;
  red_init(rs);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  LjcWarp<R>& ws = wsm[wid];
  const unsigned lt = (1u << lane) - 1u;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const Tab<R>& T = tab<R>();
  double en = 0;
  double W[6] = {0, 0, 0, 0, 0, 0};
  unsigned nlj = 0, nc0 = 0, nslot = 0, nfar = 0, nband = 0, nins_max = 0, novf = 0;  // per lane / warp
  const double reach2 = c_geo.reach2;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < A.N; i += nwarps) {
    reach_build_warp<R>(ws.s, S, i);
    const bool ovf = ws.s.ovf != 0;
    nins_max = max(nins_max, (unsigned)ws.s.nins);
    novf += ovf ? 1u : 0u;
    const double4 pi = A.pos[i];
    const int ti = type_of(pi);
    const long long ki = key_of(pi);
    LjcPar<R>& P = ws.P;
    if (lane < 2) {
      const int h = lane, p = ti + h;
      P.e4[h] = MORSE ? T.meps[p] : R(4) * T.eps[p];
      P.s2[h] = MORSE ? T.malpha[p] : T.sigma2[p];
      P.re[h] = MORSE ? T.mre[p] : R(0);
      P.rlo[h] = T.rlo[p], P.rc[h] = T.rc[p], P.iv[h] = T.inv_taper[p];
      P.rlo2[h] = c_geo.rlo2[p], P.rc2[h] = c_geo.rc2[p], P.win2[h] = c_geo.srhi2_hi[p];
    }
    __syncwarp();
    double fx = 0, fy = 0, fz = 0;
    int head[3] = {0, 0, 0}, tail[3] = {0, 0, 0};

    // ---- evaluation of 32 queued pairs of queue Q (n <= 32 valid lanes)
    auto eval = [&](auto QC, int n) {
      constexpr int Qn = decltype(QC)::value;
      LjcQueue<R>& q = ws.q[Qn];
      const int e = (head[Qn] + lane) & (LJC_Q - 1);
      const bool valid = lane < n;
      const double dx = valid ? q.dx[e] : 0.0, dy = valid ? q.dy[e] : 0.0, dz = valid ? q.dz[e] : 0.0;
      const double r2 = valid ? q.r2[e] : 1.0;
      const int J = valid ? q.J[e] : i;
      const int pc = valid ? q.pc[e] : ti;
      const int h = (pc & 3) - ti;  // 0: t_J = C side of the pair table, 1: H
      const bool canon = (pc >> 2) & 1;
      head[Qn] += n;
      if constexpr (Qn == 0) {  // near: C_ij gate, b* window
        double Md = 0.0;
        if (valid) Md = ovf ? ljc_path_M<R>(S, i, J) : reach_lookup_fast(ws.s, J);
        const bool c0 = valid && Md == 1.0;
        const bool cand = valid && !c0 && r2 < pick(P.win2, h);
        const bool norm = valid && !c0 && !cand;
        nc0 += (c0 && canon) ? 1u : 0u;
        R rr2 = norm ? (R)r2 : R(1);
        R dVr;
        R V = ljc_pair<R, MORSE, false>(P, h, rr2, dVr);
        if (norm && r2 > pick(P.rlo2, h)) {  // taper inside 3 r_max: not for the toy parameters
          R y = rsqrt_fast(rr2), dsw;
          R sv = sw<R>(rr2 * y, pick(P.rlo, h), pick(P.rc, h), dsw);
          dVr = dVr * sv + V * dsw * y;
          V = V * sv;
        }
        const R C = norm ? (R)(1.0 - Md) : R(0);  // 1 - M in fp64 (gate, reading A14)
        ljc_acc<R, VIRIAL, SG>(C * dVr, dx, dy, dz, C * V, fx, fy, fz, en, W);
        if (cand && canon) {  // the whole pair, once, in the b* batch
          const int p = pc & 3;
          const unsigned am = __activemask();
          const unsigned grp = __match_any_sync(am, p);
          const int leader = __ffs(grp) - 1;
          int b = 0;
          if (lane == leader) b = atomicAdd(Qu.count + p, __popc(grp));
          b = __shfl_sync(grp, b, leader) + __popc(grp & lt);
          if (b < Qu.cap[p]) {
            Qu.item[Qu.off[p] + b] = make_int4(i, J, 0, 0);
            Qu.M[Qu.off[p] + b] = Md;
          } else {
            atomicAdd(ct + CT_OVF_QUEUE, 1ull);
          }
        }
        if (norm && canon && Md > 0.0) {  // 0 < C < 1: dC/dx along the maximising path
          ljc_path_forces<R, SG>(S, owner, i, J, V, F, VIRIAL ? rs.d + ACC_W : nullptr);
        }
        if (VIRIAL && stage.rows && canon && (norm || c0))
          stage_lj_row(stage, gid[i], gid[J], shift[J], norm ? (double)C : 0.0, 0.0);
      } else {
        R rr2 = valid ? (R)r2 : R(1);
        R dVr;
        R V = ljc_pair<R, MORSE, Qn == 2>(P, h, rr2, dVr);
        const R wgt = valid ? R(1) : R(0);
        ljc_acc<R, VIRIAL, SG>(wgt * dVr, dx, dy, dz, wgt * V, fx, fy, fz, en, W);
        if (VIRIAL && stage.rows && valid && canon) stage_lj_row(stage, gid[i], gid[J], shift[J], 1.0, 0.0);
      }
    };

    // ---- filter: stream the cluster list, 8 clusters per round
    const int nc = A.cnt[i];
    const int* row = A.nbr + (size_t)i * A.cap;
    nslot += (unsigned)nc * CL_SIZE;
    int cn = (lane >> 2) < nc ? row[lane >> 2] : -1;
    for (int base = 0; base < nc; base += 8) {
      const int c = cn;
      const int qn = base + 8 + (lane >> 2);
      cn = qn < nc ? row[qn] : -1;  // next round's cluster index in flight
      const int s = CL_SIZE * (c >= 0 ? c : 0) + (lane & 3);
      const int J = c >= 0 ? A.cl_atom[s] : -1;
      const double4 pj = A.cpos[s];
      const double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
      const double r2 = r2_exact(dx, dy, dz);
      const int h = type_of(pj);
      const bool in = c >= 0 && J >= 0 && J != i && r2 <= pick(P.rc2, h);
      const bool canon = in && ki < key_of(pj);
      const int cls = !in ? -1 : (r2 <= reach2 ? 0 : (r2 <= pick(P.rlo2, h) ? 1 : 2));
      nlj += canon ? 1u : 0u;
      nfar += (canon && cls > 0) ? 1u : 0u;
      nband += (canon && cls == 2) ? 1u : 0u;
#pragma unroll
      for (int Qn = 0; Qn < 3; ++Qn) {
        const unsigned m = __ballot_sync(0xffffffffu, cls == Qn);
        if (cls == Qn) {
          LjcQueue<R>& q = ws.q[Qn];
          const int e = (tail[Qn] + __popc(m & lt)) & (LJC_Q - 1);
          q.dx[e] = dx, q.dy[e] = dy, q.dz[e] = dz, q.r2[e] = r2;
          q.J[e] = J;
          q.pc[e] = (ti + h) | (canon ? 4 : 0);
        }
        tail[Qn] += __popc(m);
      }
      __syncwarp();
      if (tail[0] - head[0] >= 32) eval(std::integral_constant<int, 0>{}, 32), __syncwarp();
      if (tail[1] - head[1] >= 32) eval(std::integral_constant<int, 1>{}, 32), __syncwarp();
      if (tail[2] - head[2] >= 32) eval(std::integral_constant<int, 2>{}, 32), __syncwarp();
    }
    if (tail[0] > head[0]) eval(std::integral_constant<int, 0>{}, tail[0] - head[0]), __syncwarp();
    if (tail[1] > head[1]) eval(std::integral_constant<int, 1>{}, tail[1] - head[1]), __syncwarp();
    if (tail[2] > head[2]) eval(std::integral_constant<int, 2>{}, tail[2] - head[2]), __syncwarp();
    fx = warp_sum<SG>(fx);
    fy = warp_sum<SG>(fy);
    fz = warp_sum<SG>(fz);
    if (lane == 0) atomic_add3<SG>(F, i, fx, fy, fz);
    __syncwarp();
  }
  red_add_d(rs, ACC_ELJ, 0.5 * en);
  if (VIRIAL)
    for (int c = 0; c < 6; ++c) red_add_d(rs, ACC_W + c, W[c]);
  red_add_u(rs, CT_LJ, nlj);
  red_add_u(rs, CT_C0, nc0);
  red_add_u(rs, CT_LJFAR, nfar);
  red_add_u(rs, CT_LJTAPER, nband);
  red_add_u(rs, CT_LJENT, lane == 0 ? nslot : 0u);
  red_max_u(rs, CT_MAXREACH, lane == 0 ? nins_max : 0u);
  red_add_u(rs, CT_OVF_REACH, lane == 0 ? novf : 0u);
  red_flush(rs, RR);
}

}  // namespace ab
