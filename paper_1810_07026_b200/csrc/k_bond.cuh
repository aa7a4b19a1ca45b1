// k_bond.cuh -- bond order b_ij (forward + hand-derived reverse pass), REBO + torsion per bond,
// and the deferred b* batch of the LJ term.
//
// Paper: E^REBO_ij = f_R(r) + b_ij f_A(r) (Alg. 1); b_ij = 1/2(p_ij + p_ji)
// + pi^rc + pi^dh (reading A1: sum); p_ij = [1 + sum_k w_ik g_i(cos th_jik) e^{lam}
// + P_ij]^{-1/2}; pi^rc spline in N_ij, N_ji, N^conj; pi^dh =
// T_ij sum_k sum_l (1 - cos^2 w) w_ik w_jl G G; torsion (Alg. 2)
// merged with REBO as in P:789; b* at the fictitious distance (reading A8) in batches
// "calculated in the same manner as short-ranged forces".
// Forward/reverse two-pass chain rule of P:242-253: the forward pass forms the sums, the reverse
// pass turns dE/db into gradients on every relative vector (d_ij, d_ik, d_jl, d_km, d_ln) which
// are scattered as forces with fp64 atomics (force on b -= g, on a += g for v = x_b - x_a) and
// folded into the virial W -= v (x) g.
// GPU mapping: one thread per REBO half bond / per queued b* pair (interaction-wise).
// Register residency: a side (neighbours of i or of j, partner excluded) is held in fully
// unrolled fixed-size arrays of NB = NB_FAST = 4 entries; bonds with a larger side are appended
// to an overflow list processed by an NB = NBMAX instantiation (rolled loops).  The b* batch is
// split the same way: the fast kernel does the forward pass only (S_b on a plateau, C = 0 or 1)
// and defers transition / fractional-C / large-side pairs to the full kernel.
#pragma once
#include "dev_common.cuh"
#include "k_lists.cuh"

namespace ab {

constexpr int NB_FAST = 4;

// Unrolling the side loops keeps the side arrays in registers but multiplies the code size:
// measured (bench, cfg2): it wins for the forward-only b* kernel and loses for the REBO kernel
// (instruction-cache stalls), so each caller chooses.
template <int NB, bool U>
struct Unr {
  static constexpr int v = (U && NB <= NB_FAST && NB > 0) ? NB : 1;
};
template <int NB>
struct Cap {  // array extent for a side of NB entries (NB = 0: the side is empty)
  static constexpr int v = NB > 0 ? NB : 1;
};

// NB: capacity of the i side, NBJ: of the J side (NBJ = 0: specialised for an empty J side, e.g.
// the H end of a C-H bond of a saturated hydrocarbon)
template <typename R, int NB, int NBJ = NB>
struct BoState {
  int i, J, ti, tj;
  V3<R> d, u;  // the bond vector used for angles (d_ij or rho d_hat) and its unit vector
  R r;
  int nI, nJ;
  int pq, pl;     // slot of the partner in N(i) / of i in N(J), -1 if absent
  bool overflow;  // a side has more than NB neighbours: use the NB = NBMAX instantiation
  R cl[Cap<NBJ>::v], Gl[Cap<NBJ>::v], dGl[Cap<NBJ>::v];
  R Si, Sj, PxI, PyI, PxJ, PyJ;
  R pij, pji, Nij, Nji, Nconj;
  R QI, dQI, QJ, dQJ;  // F3 g_C(cos, N) blend weight S(N) per side and dS/dN (sum_1 - sum_2)
  R Rv, Rx, Ry, Rz, Tv, Tx, Ty, Tz;  // derivatives w.r.t. (N_ij, N_ji, N^conj)
  R D, Tsum;
  int nquads;
  bool bad;
};

// slot in the short list of the a-th side neighbour (the partner's slot is skipped)
__device__ __forceinline__ int side_slot(int a, int partner_slot) {
  return (partner_slot >= 0 && a >= partner_slot) ? a + 1 : a;
}

template <typename R>
__device__ __forceinline__ R clamp_cos(R c) {
  return c > R(1) ? R(1) : (c < R(-1) ? R(-1) : c);
}

// collinearity guard G(c) = 1 - S(1 - c^2; s2lo, s2hi) (reading A9) and dG/dc
template <typename R>
__device__ __forceinline__ R guardG(R c, R& dG) {
  const Tab<R>& T = tab<R>();
  R ds;
  R s = sw<R>(R(1) - c * c, T.s2lo, T.s2hi, ds);
  dG = R(2) * c * ds;
  return R(1) - s;
}

// V_tors(c) = (256/405) ((1+c)/2)^5 - 1/10 and its derivative
template <typename R>
__device__ __forceinline__ R vtors(R c, R& dv) {
  R h = R(0.5) * (R(1) + c);
  R h2 = h * h, h4 = h2 * h2;
  dv = R(128.0 / 81.0) * h4;
  return R(256.0 / 405.0) * h4 * h - R(0.1);
}

template <typename R>
__device__ __forceinline__ R F_conj(R x, R& dF) {
  const Tab<R>& T = tab<R>();
  return sw<R>(x, T.conj_lo, T.conj_hi, dF);
}

// F3 (reading A33): e^{lambda_jik} for centre t_c with partner t_p at distance r
// (the fictitious rho in b*) and neighbour t_k at r_k; lambda depends on the distances for H
// centres only: lambda.JIK + kappa [(rho_{t_k H} - r_k) - (rho_{t_p H} - r)]
template <typename R>
__device__ __forceinline__ R explam_r(int tp, int tc, int tk, R r, R rk) {
  const Tab<R>& T = tab<R>();
  R e = T.explam[tp][tc][tk];
  if (tc == 1 && T.kappa != R(0)) e *= ex(T.kappa * ((T.rhoH[tk] - rk) - (T.rhoH[tp] - r)));
  return e;
}

// F3 (reading A34): g of centre species tc, blended with g_C2 by the side's coordination weight Q
template <typename R>
__device__ __forceinline__ R gblend(int tc, R c, R Q, R& dg) {
  R g = gspline<R>(tc, c, dg);
  if (tc == 0 && tab<R>().g2on) {
    R dg2;
    R g2 = gspline<R>(2, c, dg2);
    g = g2 + Q * (g - g2);
    dg = dg2 + Q * (dg - dg2);
  }
  return g;
}

// ---------------------------------------------------------------- forward pass
template <typename R, bool TORS, int NB, bool UNROLL = false, int NBJ = NB>
__device__ __forceinline__ void bo_forward(const ShortList<R>& S, const signed char* typ, int i, int J, V3<R> d, R r,
                           BoState<R, NB, NBJ>& st) {
  const Tab<R>& T = tab<R>();
  st.i = i, st.J = J, st.ti = typ[i], st.tj = typ[J], st.d = d, st.r = r;
  const int ti = st.ti, tj = st.tj;
  const size_t bi = (size_t)i * S.capS, bj = (size_t)J * S.capS;
  const int ni = S.cnt[i], nj = S.cnt[J];
  int pq = -1, pl = -1;
  for (int q = 0; q < ni; ++q)
    if (S.nbr[bi + q] == J) pq = q;
  for (int q = 0; q < nj; ++q)
    if (S.nbr[bj + q] == i) pl = q;
  const int nI = ni - (pq >= 0), nJ = nj - (pl >= 0);
  st.pq = pq, st.pl = pl, st.nI = nI, st.nJ = nJ;
  st.overflow = nI > NB || nJ > NBJ;
  st.bad = false;
  if (st.overflow) return;
  R ir = R(1) / r;
  st.u = ir * d;
  // ---- i side: k in N(i) \ {J}
  const bool blendI = ti == 0 && T.g2on;  // F3: sum with g_C and with g_C2, blended by S(N_ij)
  R sumI = 0, sumI2 = 0, NCi = 0, NHi = 0, Si = 0;
#pragma unroll(Unr<NB, UNROLL>::v)
  for (int a = 0; a < NB; ++a) {
    if (a >= nI) continue;
    int q = side_slot(a, pq);
    int k = S.nbr[bi + q];
    R rk;
    V3<R> dk = sl_d(S, i, q, rk);
    R wk = S.w[bi + q].x;
    int tk = typ[k];
    R c = clamp_cos(dot3(d, dk) * ir / rk);
    R dg;
    R g = gspline<R>(ti, c, dg);
    const R ek = explam_r<R>(tj, ti, tk, r, rk);
    sumI += wk * g * ek;
    if (blendI) sumI2 += wk * gspline<R>(2, c, dg) * ek;
    if (tk == 0) {
      NCi += wk;
      R dF;
      Si += wk * F_conj<R>(S.Ntot[k] - wk, dF);
    } else {
      NHi += wk;
    }
  }
  // ---- J side: l in N(J) \ {i}
  const bool blendJ = tj == 0 && T.g2on;
  R sumJ = 0, sumJ2 = 0, NCj = 0, NHj = 0, Sj = 0;
  const V3<R> md = mk3(-d.x, -d.y, -d.z);
#pragma unroll(Unr<NBJ, UNROLL>::v)
  for (int c = 0; c < NBJ; ++c) {
    if (c >= nJ) continue;
    int q = side_slot(c, pl);
    int l = S.nbr[bj + q];
    R rl;
    V3<R> dl = sl_d(S, J, q, rl);
    R wl = S.w[bj + q].x;
    int tl = typ[l];
    R cc = clamp_cos(dot3(md, dl) * ir / rl);
    R dg;
    R g = gspline<R>(tj, cc, dg);
    const R el = explam_r<R>(ti, tj, tl, r, rl);
    sumJ += wl * g * el;
    if (blendJ) sumJ2 += wl * gspline<R>(2, cc, dg) * el;
    if (tl == 0) {
      NCj += wl;
      R dF;
      Sj += wl * F_conj<R>(S.Ntot[l] - wl, dF);
    } else {
      NHj += wl;
    }
    st.cl[c] = cc;
    R dG;
    st.Gl[c] = guardG<R>(cc, dG);
    st.dGl[c] = dG;
  }
  st.QI = st.QJ = R(1), st.dQI = st.dQJ = R(0);
  if (blendI) {  // g_C(cos, N_ij) = g_C2 + S(N_ij) (g_C - g_C2): sum = sum_2 + S (sum_1 - sum_2)
    R dQ;
    const R Q = sw<R>(NCi + NHi, T.gnlo, T.gnhi, dQ);
    st.QI = Q, st.dQI = dQ * (sumI - sumI2);
    sumI = sumI2 + Q * (sumI - sumI2);
  }
  if (blendJ) {
    R dQ;
    const R Q = sw<R>(NCj + NHj, T.gnlo, T.gnhi, dQ);
    st.QJ = Q, st.dQJ = dQ * (sumJ - sumJ2);
    sumJ = sumJ2 + Q * (sumJ - sumJ2);
  }
  R PI = 0, PJ = 0;
  st.PxI = st.PyI = st.PxJ = st.PyJ = 0;
  if (ti == 0) PI = pspline<R>(tj, NCi, NHi, st.PxI, st.PyI);
  if (tj == 0) PJ = pspline<R>(ti, NCj, NHj, st.PxJ, st.PyJ);
  R argI = R(1) + sumI + PI, argJ = R(1) + sumJ + PJ;
  st.bad = !(argI > R(0)) || !(argJ > R(0));
  st.pij = rsq(argI);
  st.pji = rsq(argJ);
  st.Si = Si, st.Sj = Sj;
  st.Nij = NCi + NHi;
  st.Nji = NCj + NHj;
  st.Nconj = R(1) + Si * Si + Sj * Sj;
  int p = ti + tj;
  if (ti == 1 && tj == 0) {  // CH tables take the carbon-side N first
    st.Rv = rtspline<R>(0, p, st.Nji, st.Nij, st.Nconj, st.Ry, st.Rx, st.Rz);
    st.Tv = rtspline<R>(1, p, st.Nji, st.Nij, st.Nconj, st.Ty, st.Tx, st.Tz);
  } else {
    st.Rv = rtspline<R>(0, p, st.Nij, st.Nji, st.Nconj, st.Rx, st.Ry, st.Rz);
    st.Tv = rtspline<R>(1, p, st.Nij, st.Nji, st.Nconj, st.Tx, st.Ty, st.Tz);
  }
  // ---- dihedral sum (and torsion sum): k in N(i)\J, l in N(J)\{i, k}
  R D = 0, Ts = 0;
  int nq = 0;
#pragma unroll(Unr<NB, UNROLL>::v)
  for (int a = 0; a < NB; ++a) {
    if (a >= nI) continue;
    int q = side_slot(a, pq);
    int k = S.nbr[bi + q];
    R rk;
    V3<R> dk = sl_d(S, i, q, rk);
    R wk = S.w[bi + q].x;
    R ck = clamp_cos(dot3(d, dk) * ir / rk);
    R dGk;
    R Gk = guardG<R>(ck, dGk);
    V3<R> n1 = cross3(dk, d);
    R n1s = dot3(n1, n1);
#pragma unroll(Unr<NBJ, UNROLL>::v)
    for (int c = 0; c < NBJ; ++c) {
      if (c >= nJ) continue;
      int ql = side_slot(c, pl);
      int l = S.nbr[bj + ql];
      if (l == k) continue;
      ++nq;
      if (Gk == R(0) || st.Gl[c] == R(0)) continue;
      R rl;
      V3<R> dl = sl_d(S, J, ql, rl);
      R wl = S.w[bj + ql].x;
      V3<R> n2 = cross3(md, dl);
      R cw = dot3(n1, n2) * rsq(n1s * dot3(n2, n2));
      R base = wk * wl * Gk * st.Gl[c];
      D += (R(1) - cw * cw) * base;
      if (TORS) {
        R dv;
        Ts += T.tors[typ[k]][ti][tj][typ[l]] * base * vtors<R>(cw, dv);
      }
    }
  }
  st.D = D;
  st.Tsum = Ts;
  st.nquads = nq;
}

template <typename R, int NB, int NBJ>
__device__ __forceinline__ R bo_value(const BoState<R, NB, NBJ>& st) {
  return R(0.5) * (st.pij + st.pji) + st.Rv + st.Tv * st.D;
}

template <typename R, bool SG = false>
__device__ __forceinline__ void scatter_vec(double* F, const int* owner, int a_to, int a_from, V3<R> g) {
  // vector v = x_to - x_from with gradient g: F_to -= g, F_from += g
  atomic_add3<SG>(F, owner[a_to], -(double)g.x, -(double)g.y, -(double)g.z);
  atomic_add3<SG>(F, owner[a_from], (double)g.x, (double)g.y, (double)g.z);
}

// N^conj chain: N_c = sum_m w_cm (m != excluded) -> forces on every m with dw != 0
template <typename R, bool SG = false>
__device__ __forceinline__ void conj_chain(const ShortList<R>& S, const int* owner, int c, int excl, R chain,
                                           double* F, double W[6]) {
  size_t bc = (size_t)c * S.capS;
  int nc = S.cnt[c];
  for (int q2 = 0; q2 < nc; ++q2) {
    int m = S.nbr[bc + q2];
    if (m == excl) continue;
    R dw = S.w[bc + q2].y;
    if (dw == R(0)) continue;
    R rcm;
    V3<R> dcm = sl_d(S, c, q2, rcm);
    V3<R> g = (chain * dw / rcm) * dcm;
    scatter_vec<R, SG>(F, owner, m, c, g);
    vir_add(W, dcm, g);
  }
}

// ---------------------------------------------------------------- reverse pass
// cb = dE/db.  wij: weight of the bond for the merged torsion term (TORS only).
// Output gd = dE/d(d) through the bond-order (and torsion) terms; fi / fj = force contributions
// on i / J from the k and l vectors (the forces on k, l, m, n are scattered here).
template <typename R, bool TORS, int NB, bool UNROLL = false, bool SG = false, int NBJ = NB>
__device__ __forceinline__ void bo_reverse(const ShortList<R>& S, const signed char* typ, const int* owner, const BoState<R, NB, NBJ>& st,
                           R cb, R wij, double* F, double W[6], V3<R>& gd, V3<R>& fi, V3<R>& fj) {
  const Tab<R>& T = tab<R>();
  const int i = st.i, J = st.J, ti = st.ti, tj = st.tj, nI = st.nI, nJ = st.nJ;
  const V3<R> d = st.d, u = st.u;
  const V3<R> md = mk3(-d.x, -d.y, -d.z);
  const R r = st.r, ir = R(1) / r;
  const R cI = R(-0.25) * cb * st.pij * st.pij * st.pij;
  const R cJ = R(-0.25) * cb * st.pji * st.pji * st.pji;
  const R dNij = cb * (st.Rx + st.Tx * st.D);
  const R dNji = cb * (st.Ry + st.Ty * st.D);
  const R dNc = cb * (st.Rz + st.Tz * st.D);
  const R cD = cb * st.Tv;
  const size_t bi = (size_t)i * S.capS, bj = (size_t)J * S.capS;
  gd = mk3<R>(0, 0, 0);
  fi = mk3<R>(0, 0, 0);
  fj = mk3<R>(0, 0, 0);
  R Wl[Cap<NBJ>::v], Cl[Cap<NBJ>::v], Ll[Cap<NBJ>::v];
  V3<R> gl[Cap<NBJ>::v];
  const bool lamI = ti == 1 && T.kappa != R(0), lamJ = tj == 1 && T.kappa != R(0);  // F3 lambda(r)
#pragma unroll(Unr<NBJ, UNROLL>::v)
  for (int c = 0; c < NBJ; ++c) {
    if (c >= nJ) continue;
    int q = side_slot(c, st.pl);
    int l = S.nbr[bj + q];
    int tl = typ[l];
    R wl = S.w[bj + q].x;
    R dg;
    R g = gblend<R>(tj, st.cl[c], st.QJ, dg);
    R el = T.explam[ti][tj][tl];
    if (lamJ) el = explam_r<R>(ti, tj, tl, r, S.dr[bj + q].w);
    R Pd = tl == 0 ? st.PxJ : st.PyJ;
    Wl[c] = cJ * (g * el + Pd + st.dQJ) + dNji;
    Ll[c] = lamJ ? cJ * wl * g * el * T.kappa : R(0);  // dE/dlambda_ijl (x kappa)
    if (tl == 0) {
      R dF;
      R Fl = F_conj<R>(S.Ntot[l] - wl, dF);
      Wl[c] += dNc * R(2) * st.Sj * Fl;
    }
    Cl[c] = cJ * wl * dg * el;
    gl[c] = mk3<R>(0, 0, 0);
  }
#pragma unroll(Unr<NB, UNROLL>::v)
  for (int a = 0; a < NB; ++a) {
    if (a >= nI) continue;
    int q = side_slot(a, st.pq);
    int k = S.nbr[bi + q];
    int tk = typ[k];
    R rk;
    V3<R> dk = sl_d(S, i, q, rk);
    R wk = S.w[bi + q].x, dwk = S.w[bi + q].y;
    R irk = R(1) / rk;
    V3<R> uk = irk * dk;
    R ck = clamp_cos(dot3(u, uk));
    R dg;
    R g = gblend<R>(ti, ck, st.QI, dg);
    R ek = lamI ? explam_r<R>(tj, ti, tk, r, rk) : T.explam[tj][ti][tk];
    R Wk = cI * (g * ek + (tk == 0 ? st.PxI : st.PyI) + st.dQI) + dNij;
    R Ck = cI * wk * dg * ek;
    // lambda_jik(r_ij, r_ik) of an H centre (F3): d lambda/d r_ik = -kappa, d lambda/d r_ij = +kappa
    const R Lk = lamI ? cI * wk * g * ek * T.kappa : R(0);
    if (lamI) addto(gd, Lk * u);
    R chain = 0;
    if (tk == 0) {
      R dF;
      R Fk = F_conj<R>(S.Ntot[k] - wk, dF);
      Wk += dNc * R(2) * st.Si * Fk;
      chain = dNc * R(2) * st.Si * wk * dF;
    }
    V3<R> gk = mk3<R>(0, 0, 0);
    R dGk;
    R Gk = guardG<R>(ck, dGk);
    if (Gk != R(0)) {
      V3<R> n1 = cross3(dk, d);
      R inv1 = rsq(dot3(n1, n1));
#pragma unroll(Unr<NBJ, UNROLL>::v)
      for (int c = 0; c < NBJ; ++c) {
        if (c >= nJ) continue;
        int ql = side_slot(c, st.pl);
        int l = S.nbr[bj + ql];
        if (l == k || st.Gl[c] == R(0)) continue;
        R rl;
        V3<R> dl = sl_d(S, J, ql, rl);
        R wl = S.w[bj + ql].x;
        V3<R> n2 = cross3(md, dl);
        R inv2 = rsq(dot3(n2, n2));
        R cw = dot3(n1, n2) * inv1 * inv2;
        R Gl = st.Gl[c];
        R coef = cD * (R(1) - cw * cw);
        R dcoef = cD * (R(-2) * cw);
        if (TORS) {
          R eps = T.tors[tk][ti][tj][typ[l]] * wij;
          R dv;
          R v = vtors<R>(cw, dv);
          coef += eps * v;
          dcoef += eps * dv;
        }
        R wG = wk * wl;
        R GG = Gk * Gl;
        R dEdcw = dcoef * wG * GG;
        Wk += coef * wl * GG;
        Wl[c] += coef * wk * GG;
        Ck += coef * wG * Gl * dGk;
        Cl[c] += coef * wG * Gk * st.dGl[c];
        // d cos w / d a = b x g1, / d e = b x g2, / d b = g1 x a + g2 x e  (a = d_ik, b = d, e = d_jl)
        V3<R> g1 = inv1 * (inv2 * n2 - (cw * inv1) * n1);
        V3<R> g2 = inv2 * (inv1 * n1 - (cw * inv2) * n2);
        addto(gk, dEdcw * cross3(d, g1));
        addto(gl[c], dEdcw * cross3(d, g2));
        addto(gd, dEdcw * (cross3(g1, dk) + cross3(g2, dl)));
      }
    }
    // w_ik(r_ik) and cos(theta_jik) derivatives
    addto(gk, (Wk * dwk - Lk) * uk);
    addto(gk, (Ck * irk) * (u - ck * uk));
    addto(gd, (Ck * ir) * (uk - ck * u));
    // force on k now; the +gk on i is accumulated in fi (one atomic per bond for i)
    atomic_add3<SG>(F, owner[k], -(double)gk.x, -(double)gk.y, -(double)gk.z);
    addto(fi, gk);
    vir_add(W, dk, gk);
    if (chain != R(0)) conj_chain<R, SG>(S, owner, k, i, chain, F, W);
  }
#pragma unroll(Unr<NBJ, UNROLL>::v)
  for (int c = 0; c < NBJ; ++c) {
    if (c >= nJ) continue;
    int q = side_slot(c, st.pl);
    int l = S.nbr[bj + q];
    int tl = typ[l];
    R rl;
    V3<R> dl = sl_d(S, J, q, rl);
    R wl = S.w[bj + q].x, dwl = S.w[bj + q].y;
    R irl = R(1) / rl;
    V3<R> ul = irl * dl;
    R cl = st.cl[c];
    V3<R> g = gl[c];
    addto(g, (Wl[c] * dwl - Ll[c]) * ul);
    if (lamJ) addto(gd, Ll[c] * u);
    addto(g, (Cl[c] * irl) * (mk3(-u.x, -u.y, -u.z) - cl * ul));
    addto(gd, (-Cl[c] * ir) * (ul + cl * u));
    atomic_add3<SG>(F, owner[l], -(double)g.x, -(double)g.y, -(double)g.z);
    addto(fj, g);
    vir_add(W, dl, g);
    if (tl == 0) {
      R dF;
      F_conj<R>(S.Ntot[l] - wl, dF);
      R chain = dNc * R(2) * st.Sj * wl * dF;
      if (chain != R(0)) conj_chain<R, SG>(S, owner, l, J, chain, F, W);
    }
  }
}

struct StageBuf {
  double* rows;
  int* count;
  int cap;
};

__device__ __forceinline__ double* stage_row(StageBuf sb, int width) {
  int k = atomicAdd(sb.count, 1);
  if (k >= sb.cap) return nullptr;
  return sb.rows + (size_t)k * width;
}

// warp-aggregated append of v to list (count at *cnt); lanes outside `take` do nothing
__device__ __forceinline__ void list_append(int* list, int* cnt, int cap, int v) {
  unsigned am = __activemask();
  int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(cnt, __popc(am));
  base = __shfl_sync(am, base, leader);
  int k = base + __popc(am & ((1u << lane) - 1u));
  if (k < cap) list[k] = v;
}

// ---------------------------------------------------------------- REBO + torsion, one thread per bond
// list = (i, slot) pairs; NB = NB_FAST: bonds with a larger side are appended to ovf (indices into
// list) for the NB = NBMAX instantiation, which runs over ovf (list_idx != nullptr).
#ifndef AB_REBO_MINBLOCKS
#define AB_REBO_MINBLOCKS 1
#endif
#ifndef AB_REBO_UNROLL  // which REBO instantiations unroll their side loops (registers vs i-cache)
#define AB_REBO_UNROLL(nb) ((nb) <= 3)
#endif
#ifndef AB_REBO3_MINBLOCKS
#define AB_REBO3_MINBLOCKS 2  // the sp3 C-C batch (sides of <= 3)
#endif
#ifndef AB_REBO1_MINBLOCKS
#define AB_REBO1_MINBLOCKS 4  // the one-empty-side batch (no J-side arrays, no dihedral loop; measured 4 beats 3)
#endif
#ifndef AB_BSTAR_MINBLOCKS
#define AB_BSTAR_MINBLOCKS 3  // measured (cfg2): 3 blocks (170 regs) 56 us vs 64 us at 2 blocks
#endif
// VIR = false (NVE steps): no virial accumulation and no stage rows (compiled out)
// Work: the bonds of the species regions [reg0, reg1) (list_idx == nullptr) or the *nlist bond
// indices of list_idx.  Bonds this instantiation cannot take are appended to ovf (count *novf).
// NBJ = 0 (the "one empty side" batch of the CH / HH regions): a bond whose i side is empty is
// evaluated with its ends swapped (b_ij, the pair terms and the forces are symmetric in i, j);
// a bond with two non-empty sides goes to ovf for the general NB_FAST kernel.
template <typename R, int NB, bool VIR, bool SG = false, int NBJ = NB>
__global__ void __launch_bounds__(128, NBJ == 0 ? AB_REBO1_MINBLOCKS
                                                  : (NB == 3 ? AB_REBO3_MINBLOCKS : (NB <= NB_FAST ? AB_REBO_MINBLOCKS : 1)))
    k_rebo(BondList BL, const int* list_idx, const int* nlist, int reg0, int reg1, int* ovf, int* novf,
           ShortList<R> S, const signed char* typ, const int* owner, const int* gid, const char4* shift, double* F,
           StageBuf stage, RedRows RR) {
  __shared__ RedSmem rs;
  int nr[3] = {0, 0, 0};
  for (int g = reg0; g < reg1; ++g) nr[g] = BL.cnt[g];
  const int nb = list_idx ? *nlist : nr[0] + nr[1] + nr[2];
  if (red_idle_block(nb, RR)) return;
  red_init(rs);
  const Tab<R>& T = tab<R>();
  double e[3 + 6] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long nq = 0, nbad = 0, ncount = 0, nang = 0;
  int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += stride) {
    int bidx;
    if (list_idx) {
      bidx = list_idx[t];
    } else {
      int g = 0, u = t;
      while (u >= nr[g]) u -= nr[g++];
      bidx = g * BL.cap + u;
    }
    int2 bd = BL.b[bidx];
    int i = bd.x, q = bd.y;
    size_t e0 = (size_t)i * S.capS + q;
    int J = S.nbr[e0];
    R r;
    V3<R> d = sl_d(S, i, q, r);
    bool swapped = false;
    if (NBJ == 0) {  // the partner occupies one slot of each list: the sides are cnt - 1
      const int nI0 = S.cnt[i] - 1, nJ0 = S.cnt[J] - 1;
      if (nJ0 != 0) {
        if (nI0 != 0) {  // two non-empty sides: the general kernel
          list_append(ovf, novf, 1 << 30, bidx);
          continue;
        }
        swapped = true;
        const int tmp = i;
        i = J, J = tmp;
        d = mk3(-d.x, -d.y, -d.z);
      }
    }
    BoState<R, NB, NBJ> st;
    bo_forward<R, true, NB, AB_REBO_UNROLL(NB), NBJ>(S, typ, i, J, d, r, st);
    if (st.overflow) {  // only possible for NB = NB_FAST
      list_append(ovf, novf, 1 << 30, bidx);
      continue;
    }
    R w = S.w[e0].x, dw = S.w[e0].y;
    int ti = typ[i], tj = typ[J], p = ti + tj;
    // pair terms f_R = w (1 + Q/r) A e^{-alpha r},  f_A = -w sum_n B_n e^{-beta_n r}
    R ir = R(1) / r;
    R ea = ex(-T.alpha[p] * r);
    R qr = R(1) + T.Q[p] * ir;
    R VR = w * qr * T.A[p] * ea;
    R dVR = dw * qr * T.A[p] * ea + w * T.A[p] * ea * (-T.Q[p] * ir * ir - T.alpha[p] * qr);
    R sb = 0, sbb = 0;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      R eb = T.B[p][n] * ex(-T.beta[p][n] * r);
      sb += eb;
      sbb += T.beta[p][n] * eb;
    }
    R VA = -w * sb;
    R dVA = -dw * sb + w * sbb;
    R b = bo_value(st);
    V3<R> gd, fi, fj;
    bo_reverse<R, true, NB, AB_REBO_UNROLL(NB), SG, NBJ>(S, typ, owner, st, VA, w, F, VIR ? e + 3 : nullptr, gd, fi,
                                                          fj);
    R dEdr = dVR + b * dVA + dw * st.Tsum;
    addto(gd, (dEdr * ir) * d);
    atomic_add3<SG>(F, owner[i], (double)(gd.x + fi.x), (double)(gd.y + fi.y), (double)(gd.z + fi.z));
    atomic_add3<SG>(F, owner[J], (double)(fj.x - gd.x), (double)(fj.y - gd.y), (double)(fj.z - gd.z));
    vir_add(VIR ? e + 3 : nullptr, d, gd);
    e[0] = acc_round<SG>(e[0] + (double)(VR + b * VA));
    e[1] = acc_round<SG>(e[1] + (double)(w * st.Tsum));
    nq += st.nquads;
    nbad += st.bad;
    ncount += 1;
    nang += st.nI + st.nJ;
    if (VIR && stage.rows) {
      double* row = stage_row(stage, 13);
      if (row) {  // in the canonical orientation of the bond list
        const int a = swapped ? J : i, c = swapped ? i : J;
        char4 s = shift[c];
        row[0] = gid[a], row[1] = gid[c], row[2] = s.x, row[3] = s.y, row[4] = s.z;
        row[5] = b, row[6] = swapped ? st.pji : st.pij, row[7] = swapped ? st.pij : st.pji, row[8] = st.Rv;
        row[9] = st.Tv * st.D;
        row[10] = swapped ? st.Nji : st.Nij, row[11] = swapped ? st.Nij : st.Nji, row[12] = st.Nconj;
      }
    }
  }
  red_add_d(rs, ACC_EREBO, e[0]);
  red_add_d(rs, ACC_ETORS, e[1]);
  for (int c = 0; c < 6; ++c) red_add_d(rs, ACC_W + c, e[3 + c]);
  red_add_u(rs, CT_ANGLES, nang);
  red_add_u(rs, CT_QUADS, nq);
  red_add_u(rs, CT_BADARG, nbad);
  red_add_u(rs, CT_BONDS, ncount);
  red_flush(rs, RR);
}

// ---------------------------------------------------------------- REBO + torsion, 4 lanes per bond
// The sp3 C-C batch (both sides <= 3 neighbours; P:496-506 for b_ij, Alg. 2 P:390-407 for the
// torsion) with a lane group per bond instead of one thread: lane s of the group takes side
// neighbour s of i (k_s) and of J (l_s).  The side sums of the forward pass are reduced over the
// group; the P splines (lanes 0 / 1) and the pi^rc / T splines (lanes 2 / 3) are evaluated once
// per group and broadcast; the dihedral / torsion double sum runs as one fused loop over l (each
// lane its own k): the forward sums D, T and the reverse-pass terms of the same (k, l) pair
// together (their coefficients need only dE/db = V_A, p_ij / p_ji and T_ij, all known before the
// loop; the D-dependent parts dN/dN_ij ... are added after it).  The l-side accumulators are
// reduced to their owning lane; every lane scatters the forces of its own k and l (and their
// N^conj chains), lane 0 those of i and J.  Per term the arithmetic is that of bo_forward /
// bo_reverse; only the summation order differs.
constexpr int RG = 4;
#ifndef AB_REBOG_MINBLOCKS
#define AB_REBOG_MINBLOCKS 3
#endif

template <typename R>
__device__ __forceinline__ R gsum(unsigned gm, R v) {
  v += __shfl_xor_sync(gm, v, 1, RG);
  v += __shfl_xor_sync(gm, v, 2, RG);
  return v;
}
template <typename R>
__device__ __forceinline__ R gbc(unsigned gm, R v, int src) {
  return __shfl_sync(gm, v, src, RG);
}

template <typename R, bool VIR, bool SG = false>
__global__ void __launch_bounds__(128, AB_REBOG_MINBLOCKS)
    k_rebo_g4(BondList BL, int reg, int* ovf, int* novf, ShortList<R> S, const signed char* typ, const int* owner,
              const int* gid, const char4* shift, double* F, StageBuf stage, RedRows RR) {
  __shared__ RedSmem rs;
  const int nb = BL.cnt[reg];
  if (red_idle_block(nb * RG, RR)) return;
  red_init(rs);
  const Tab<R>& T = tab<R>();
  const int lane = threadIdx.x & 31, s = lane & (RG - 1), gsh = lane & ~(RG - 1);
  const unsigned gm = 0xFu << gsh;
  double e[3 + 6] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double* const Wv = VIR ? e + 3 : nullptr;
  unsigned long long nq = 0, nbad = 0, ncount = 0, nang = 0;
  const int gstride = (gridDim.x * blockDim.x) / RG;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) / RG; t < nb; t += gstride) {
    const int bidx = reg * BL.cap + t;
    const int2 bd = BL.b[bidx];
    const int i = bd.x, q = bd.y;
    const size_t bi = (size_t)i * S.capS;
    const int J = S.nbr[bi + q];
    const size_t bj = (size_t)J * S.capS;
    const int ni = S.cnt[i], nj = S.cnt[J];
    if (ni > RG || nj > RG) {  // a side of more than 3: the general kernel
      if (s == 0) list_append(ovf, novf, 1 << 30, bidx);
      continue;
    }
    const int nbI = s < ni ? S.nbr[bi + s] : -1, nbJ = s < nj ? S.nbr[bj + s] : -1;
    const unsigned mI = (__ballot_sync(gm, nbI == J) >> gsh) & 0xFu;
    const unsigned mJ = (__ballot_sync(gm, nbJ == i) >> gsh) & 0xFu;
    const int pq = mI ? __ffs(mI) - 1 : -1, pl = mJ ? __ffs(mJ) - 1 : -1;
    const int nI = ni - (pq >= 0), nJ = nj - (pl >= 0);
    if (nI > 3 || nJ > 3) {
      if (s == 0) list_append(ovf, novf, 1 << 30, bidx);
      continue;
    }
    R r;
    const V3<R> d = sl_d(S, i, q, r);
    const R ir = R(1) / r;
    const V3<R> u = ir * d, mu = mk3(-u.x, -u.y, -u.z), md = mk3(-d.x, -d.y, -d.z);
    const int ti = typ[i], tj = typ[J];
    const bool blendI = ti == 0 && T.g2on, blendJ = tj == 0 && T.g2on;
    const bool lamI = ti == 1 && T.kappa != R(0), lamJ = tj == 1 && T.kappa != R(0);
    // ---- this lane's side neighbours: k = k_s of i, l = l_s of J
    const bool hasK = s < nI, hasL = s < nJ;
    int k = -1, tk = 0, l = -1, tl = 0;
    R rk = 1, wk = 0, dwk = 0, ck = 0, g1k = 0, dg1k = 0, g2k = 0, dg2k = 0, ek = 0, Fk = 0, dFk = 0;
    R rl = 1, wl = 0, dwl = 0, cl = 0, g1l = 0, dg1l = 0, g2l = 0, dg2l = 0, el = 0, Fl = 0, dFl = 0, Gl = 0, dGl = 0;
    V3<R> dk = mk3<R>(0, 0, 0), dl = mk3<R>(0, 0, 0), uk = dk, ul = dk;
    R aSI = 0, aSI2 = 0, aNCI = 0, aNHI = 0, aCI = 0, aSJ = 0, aSJ2 = 0, aNCJ = 0, aNHJ = 0, aCJ = 0;
    if (hasK) {
      const int qk = side_slot(s, pq);
      k = S.nbr[bi + qk];
      dk = sl_d(S, i, qk, rk);
      const auto wv = S.w[bi + qk];
      wk = wv.x, dwk = wv.y;
      tk = typ[k];
      uk = (R(1) / rk) * dk;
      ck = clamp_cos(dot3(u, uk));
      g1k = gspline<R>(ti, ck, dg1k);
      if (blendI) g2k = gspline<R>(2, ck, dg2k);
      ek = explam_r<R>(tj, ti, tk, r, rk);
      aSI = wk * g1k * ek, aSI2 = wk * g2k * ek;
      if (tk == 0) {
        aNCI = wk;
        Fk = F_conj<R>(S.Ntot[k] - wk, dFk);
        aCI = wk * Fk;
      } else {
        aNHI = wk;
      }
    }
    if (hasL) {
      const int ql = side_slot(s, pl);
      l = S.nbr[bj + ql];
      dl = sl_d(S, J, ql, rl);
      const auto wv = S.w[bj + ql];
      wl = wv.x, dwl = wv.y;
      tl = typ[l];
      ul = (R(1) / rl) * dl;
      cl = clamp_cos(dot3(mu, ul));
      g1l = gspline<R>(tj, cl, dg1l);
      if (blendJ) g2l = gspline<R>(2, cl, dg2l);
      el = explam_r<R>(ti, tj, tl, r, rl);
      aSJ = wl * g1l * el, aSJ2 = wl * g2l * el;
      if (tl == 0) {
        aNCJ = wl;
        Fl = F_conj<R>(S.Ntot[l] - wl, dFl);
        aCJ = wl * Fl;
      } else {
        aNHJ = wl;
      }
      Gl = guardG<R>(cl, dGl);
    }
    // ---- group sums of the two sides
    R sumI = gsum(gm, aSI), NCi = gsum(gm, aNCI), NHi = gsum(gm, aNHI), Si = gsum(gm, aCI);
    R sumJ = gsum(gm, aSJ), NCj = gsum(gm, aNCJ), NHj = gsum(gm, aNHJ), Sj = gsum(gm, aCJ);
    R QI = 1, dQI = 0, QJ = 1, dQJ = 0;
    if (blendI) {  // g_C(cos, N_ij) = g_C2 + S(N_ij) (g_C - g_C2) (reading A34)
      const R sumI2 = gsum(gm, aSI2);
      R dQ;
      QI = sw<R>(NCi + NHi, T.gnlo, T.gnhi, dQ);
      dQI = dQ * (sumI - sumI2);
      sumI = sumI2 + QI * (sumI - sumI2);
    }
    if (blendJ) {
      const R sumJ2 = gsum(gm, aSJ2);
      R dQ;
      QJ = sw<R>(NCj + NHj, T.gnlo, T.gnhi, dQ);
      dQJ = dQ * (sumJ - sumJ2);
      sumJ = sumJ2 + QJ * (sumJ - sumJ2);
    }
    const R Nij = NCi + NHi, Nji = NCj + NHj, Nconj = R(1) + Si * Si + Sj * Sj;
    // ---- splines, one per lane: P_ij (0), P_ji (1), pi^rc (2), T_ij (3)
    R sv = 0, sx = 0, sy = 0, sz = 0;
    if (s < 2) {
      const int tc = s ? tj : ti, tp = s ? ti : tj;
      if (tc == 0) sv = pspline<R>(tp, s ? NCj : NCi, s ? NHj : NHi, sx, sy);
    } else {
      const int p = ti + tj;
      if (ti == 1 && tj == 0)  // CH tables take the carbon-side N first
        sv = rtspline<R>(s - 2, p, Nji, Nij, Nconj, sy, sx, sz);
      else
        sv = rtspline<R>(s - 2, p, Nij, Nji, Nconj, sx, sy, sz);
    }
    const R PI = gbc(gm, sv, 0), PxI = gbc(gm, sx, 0), PyI = gbc(gm, sy, 0);
    const R PJ = gbc(gm, sv, 1), PxJ = gbc(gm, sx, 1), PyJ = gbc(gm, sy, 1);
    const R Rv = gbc(gm, sv, 2), Rx = gbc(gm, sx, 2), Ry = gbc(gm, sy, 2), Rz = gbc(gm, sz, 2);
    const R Tv = gbc(gm, sv, 3), Tx = gbc(gm, sx, 3), Ty = gbc(gm, sy, 3), Tz = gbc(gm, sz, 3);
    const R argI = R(1) + sumI + PI, argJ = R(1) + sumJ + PJ;
    const bool bad = !(argI > R(0)) || !(argJ > R(0));
    const R pij = rsq(argI), pji = rsq(argJ);
    // ---- pair terms f_R, f_A; dE/db = V_A
    const R w = S.w[bi + q].x, dw = S.w[bi + q].y;
    const int p = ti + tj;
    const R ea = ex(-T.alpha[p] * r);
    const R qr = R(1) + T.Q[p] * ir;
    const R VR = w * qr * T.A[p] * ea;
    const R dVR = dw * qr * T.A[p] * ea + w * T.A[p] * ea * (-T.Q[p] * ir * ir - T.alpha[p] * qr);
    R sb = 0, sbb = 0;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      const R eb = T.B[p][n] * ex(-T.beta[p][n] * r);
      sb += eb;
      sbb += T.beta[p][n] * eb;
    }
    const R VA = -w * sb, dVA = -dw * sb + w * sbb;
    const R cb = VA;
    const R cI = R(-0.25) * cb * pij * pij * pij, cJ = R(-0.25) * cb * pji * pji * pji;
    const R cD = cb * Tv;
    // ---- reverse-pass side terms that do not depend on D
    R gk_ = g1k, dgk_ = dg1k, gl_ = g1l, dgl_ = dg1l;
    if (blendI) gk_ = g2k + QI * (g1k - g2k), dgk_ = dg2k + QI * (dg1k - dg2k);
    if (blendJ) gl_ = g2l + QJ * (g1l - g2l), dgl_ = dg2l + QJ * (dg1l - dg2l);
    R Wk = cI * (gk_ * ek + (tk == 0 ? PxI : PyI) + dQI);
    R Ck = cI * wk * dgk_ * ek;
    const R Lk = lamI ? cI * wk * gk_ * ek * T.kappa : R(0);
    R Wl = cJ * (gl_ * el + (tl == 0 ? PxJ : PyJ) + dQJ);
    R Cl = cJ * wl * dgl_ * el;
    const R Ll = lamJ ? cJ * wl * gl_ * el * T.kappa : R(0);
    V3<R> gk = mk3<R>(0, 0, 0), gd = mk3<R>(0, 0, 0);
    // ---- fused dihedral / torsion loop: this lane's k against every l of the group
    R Dp = 0, Tp = 0;
    int nqp = 0;
    R aW[3] = {0, 0, 0}, aC[3] = {0, 0, 0};
    V3<R> ag[3] = {gk, gk, gk};
    R dGk;
    const R Gk = hasK ? guardG<R>(ck, dGk) : R(0);
    const V3<R> n1 = cross3(dk, d);
    const R inv1 = Gk != R(0) ? rsq(dot3(n1, n1)) : R(0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (c >= nJ) break;  // (group-uniform)
      const int lc = __shfl_sync(gm, l * 4 + tl, c, RG);
      const V3<R> dlc = mk3(gbc(gm, dl.x, c), gbc(gm, dl.y, c), gbc(gm, dl.z, c));
      const R wlc = gbc(gm, wl, c), Glc = gbc(gm, Gl, c), dGlc = gbc(gm, dGl, c);
      if (!hasK || (lc >> 2) == k) continue;
      ++nqp;
      if (Gk == R(0) || Glc == R(0)) continue;
      const V3<R> n2 = cross3(md, dlc);
      const R inv2 = rsq(dot3(n2, n2));
      const R cw = dot3(n1, n2) * inv1 * inv2;
      const R GG = Gk * Glc, wG = wk * wlc, base = wG * GG;
      Dp += (R(1) - cw * cw) * base;
      R coef = cD * (R(1) - cw * cw), dcoef = cD * (R(-2) * cw);
      {
        const R tors = T.tors[tk][ti][tj][lc & 3];
        R dv;
        const R v = vtors<R>(cw, dv);
        Tp += tors * base * v;
        coef += tors * w * v;
        dcoef += tors * w * dv;
      }
      const R dEdcw = dcoef * base;
      Wk += coef * wlc * GG;
      aW[c] += coef * wk * GG;
      Ck += coef * wG * Glc * dGk;
      aC[c] += coef * wG * Gk * dGlc;
      // d cos w / d a = b x g1, / d e = b x g2, / d b = g1 x a + g2 x e  (a = d_ik, b = d, e = d_jl)
      const V3<R> g1 = inv1 * (inv2 * n2 - (cw * inv1) * n1);
      const V3<R> g2 = inv2 * (inv1 * n1 - (cw * inv2) * n2);
      addto(gk, dEdcw * cross3(d, g1));
      addto(ag[c], dEdcw * cross3(d, g2));
      addto(gd, dEdcw * (cross3(g1, dk) + cross3(g2, dlc)));
    }
    const R D = gsum(gm, Dp), Ts = gsum(gm, Tp);
    nqp += __shfl_xor_sync(gm, nqp, 1, RG);
    nqp += __shfl_xor_sync(gm, nqp, 2, RG);
    // l-side accumulators to their owning lane
    V3<R> gl = mk3<R>(0, 0, 0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (c >= nJ) break;
      const R sW = gsum(gm, aW[c]), sC = gsum(gm, aC[c]);
      const V3<R> sg = mk3(gsum(gm, ag[c].x), gsum(gm, ag[c].y), gsum(gm, ag[c].z));
      if (s == c) Wl += sW, Cl += sC, gl = sg;
    }
    // ---- D-dependent terms; forces on k (with its N^conj chain) and on l
    const R dNij = cb * (Rx + Tx * D), dNji = cb * (Ry + Ty * D), dNc = cb * (Rz + Tz * D);
    V3<R> fi = mk3<R>(0, 0, 0), fj = fi;
    if (hasK) {
      Wk += dNij;
      R chain = 0;
      if (tk == 0) {
        Wk += dNc * R(2) * Si * Fk;
        chain = dNc * R(2) * Si * wk * dFk;
      }
      if (lamI) addto(gd, Lk * u);
      const R irk = R(1) / rk;
      addto(gk, (Wk * dwk - Lk) * uk);
      addto(gk, (Ck * irk) * (u - ck * uk));
      addto(gd, (Ck * ir) * (uk - ck * u));
      atomic_add3<SG>(F, owner[k], -(double)gk.x, -(double)gk.y, -(double)gk.z);
      fi = gk;
      vir_add(Wv, dk, gk);
      if (chain != R(0)) conj_chain<R, SG>(S, owner, k, i, chain, F, Wv);
    }
    if (hasL) {
      Wl += dNji;
      R chain = 0;
      if (tl == 0) {
        Wl += dNc * R(2) * Sj * Fl;
        chain = dNc * R(2) * Sj * wl * dFl;
      }
      const R irl = R(1) / rl;
      addto(gl, (Wl * dwl - Ll) * ul);
      if (lamJ) addto(gd, Ll * u);
      addto(gl, (Cl * irl) * (mu - cl * ul));
      addto(gd, (-Cl * ir) * (ul + cl * u));
      atomic_add3<SG>(F, owner[l], -(double)gl.x, -(double)gl.y, -(double)gl.z);
      fj = gl;
      vir_add(Wv, dl, gl);
      if (chain != R(0)) conj_chain<R, SG>(S, owner, l, J, chain, F, Wv);
    }
    // ---- i and J (lane 0)
    gd = mk3(gsum(gm, gd.x), gsum(gm, gd.y), gsum(gm, gd.z));
    fi = mk3(gsum(gm, fi.x), gsum(gm, fi.y), gsum(gm, fi.z));
    fj = mk3(gsum(gm, fj.x), gsum(gm, fj.y), gsum(gm, fj.z));
    if (s == 0) {
      const R b = R(0.5) * (pij + pji) + Rv + Tv * D;
      const R dEdr = dVR + b * dVA + dw * Ts;
      addto(gd, (dEdr * ir) * d);
      atomic_add3<SG>(F, owner[i], (double)(gd.x + fi.x), (double)(gd.y + fi.y), (double)(gd.z + fi.z));
      atomic_add3<SG>(F, owner[J], (double)(fj.x - gd.x), (double)(fj.y - gd.y), (double)(fj.z - gd.z));
      vir_add(Wv, d, gd);
      e[0] = acc_round<SG>(e[0] + (double)(VR + b * VA));
      e[1] = acc_round<SG>(e[1] + (double)(w * Ts));
      nq += nqp;
      nbad += bad;
      ncount += 1;
      nang += nI + nJ;
      if (VIR && stage.rows) {
        double* row = stage_row(stage, 13);
        if (row) {
          const char4 sj = shift[J];
          row[0] = gid[i], row[1] = gid[J], row[2] = sj.x, row[3] = sj.y, row[4] = sj.z;
          row[5] = b, row[6] = pij, row[7] = pji, row[8] = Rv;
          row[9] = Tv * D;
          row[10] = Nij, row[11] = Nji, row[12] = Nconj;
        }
      }
    }
  }
  red_add_d(rs, ACC_EREBO, e[0]);
  red_add_d(rs, ACC_ETORS, e[1]);
  for (int c = 0; c < 6; ++c) red_add_d(rs, ACC_W + c, e[3 + c]);
  red_add_u(rs, CT_ANGLES, nang);
  red_add_u(rs, CT_QUADS, nq);
  red_add_u(rs, CT_BADARG, nbad);
  red_add_u(rs, CT_BONDS, ncount);
  red_flush(rs, RR);
}

// ---------------------------------------------------------------- C_ij path search
// Direct nested search for M = max{w_ij, w_ik w_kj, w_ik w_kl w_lj} and its maximising path,
// used when 0 < C_ij < 1 (forces along the path) or when the per-atom reach table overflowed.
template <typename R>
struct PathRes {
  double M;  // from the fp64 weights S.wd (gate, reading A14)
  int hops;
  int a0, q0, a1, q1, a2, q2;  // (atom, slot) of each path edge in the short list
};

template <typename R>
__device__ PathRes<R> path_search(const ShortList<R>& S, int i, int J) {
  PathRes<R> pr;
  pr.M = 0;
  pr.hops = 0;
  size_t bi = (size_t)i * S.capS;
  int ni = S.cnt[i];
  for (int a = 0; a < ni; ++a)
    if (S.nbr[bi + a] == J) {
      double c = S.wd[bi + a];
      if (c > pr.M) pr.M = c, pr.hops = 1, pr.a0 = i, pr.q0 = a;
    }
  for (int a = 0; a < ni; ++a) {
    int k = S.nbr[bi + a];
    if (k == J) continue;
    double w1 = S.wd[bi + a];
    size_t bk = (size_t)k * S.capS;
    int nk = S.cnt[k];
    for (int b = 0; b < nk; ++b) {
      int l = S.nbr[bk + b];
      if (l != J) continue;
      double c = w1 * S.wd[bk + b];
      if (c > pr.M) pr.M = c, pr.hops = 2, pr.a0 = i, pr.q0 = a, pr.a1 = k, pr.q1 = b;
    }
  }
  for (int a = 0; a < ni; ++a) {
    int k = S.nbr[bi + a];
    if (k == J) continue;
    double w1 = S.wd[bi + a];
    size_t bk = (size_t)k * S.capS;
    int nk = S.cnt[k];
    for (int b = 0; b < nk; ++b) {
      int l = S.nbr[bk + b];
      if (l == i || l == J) continue;
      double w2 = S.wd[bk + b];
      size_t bl = (size_t)l * S.capS;
      int nl = S.cnt[l];
      for (int c2 = 0; c2 < nl; ++c2) {
        if (S.nbr[bl + c2] != J) continue;
        double c = (w1 * w2) * S.wd[bl + c2];
        if (c > pr.M) pr.M = c, pr.hops = 3, pr.a0 = i, pr.q0 = a, pr.a1 = k, pr.q1 = b, pr.a2 = l, pr.q2 = c2;
      }
    }
  }
  return pr;
}

// forces of E = f(M) along the maximising path: dE/dM = cM
template <typename R, bool SG = false>
__device__ __forceinline__ void path_forces(const ShortList<R>& S, const int* owner, const PathRes<R>& pr, R cM, double* F,
                            double W[6]) {
  int at[3] = {pr.a0, pr.a1, pr.a2}, sl[3] = {pr.q0, pr.q1, pr.q2};
  R w[3], dw[3];
  for (int h = 0; h < pr.hops; ++h) {
    auto wv = S.w[(size_t)at[h] * S.capS + sl[h]];
    w[h] = wv.x;
    dw[h] = wv.y;
  }
  for (int h = 0; h < pr.hops; ++h) {
    if (dw[h] == R(0)) continue;
    R others = 1;
    for (int o = 0; o < pr.hops; ++o)
      if (o != h) others *= w[o];
    R rr;
    V3<R> v = sl_d(S, at[h], sl[h], rr);
    int to = S.nbr[(size_t)at[h] * S.capS + sl[h]];
    V3<R> g = (cM * others * dw[h] / rr) * v;
    scatter_vec<R, SG>(F, owner, to, at[h], g);
    vir_add(W, v, g);
  }
}

// LJ radial part V(r) = 4 eps [(s/r)^12 - (s/r)^6] S(r; r_lo, r_c) (reading A10) with (dV/dr)/r.
template <typename R>
__device__ __forceinline__ R lj_v(int p, R r2, double r2d, R& dVr_over_r) {
  const Tab<R>& T = tab<R>();
  R V, dv;
  if (c_geo.potential == 2) {  // AIREBO-M: Morse radial form
    R r = sqr_t(r2);
    R x = ex(-T.malpha[p] * (r - T.mre[p]));
    V = T.meps[p] * (x * x - R(2) * x);
    dv = R(2) * T.malpha[p] * T.meps[p] * x * (R(1) - x) / r;
  } else {
    R sr2 = T.sigma2[p] / r2;
    R sr6 = sr2 * sr2 * sr2;
    R e4 = R(4) * T.eps[p];
    V = e4 * (sr6 * sr6 - sr6);
    dv = -e4 * (R(12) * sr6 * sr6 - R(6) * sr6) / r2;  // (dV0/dr)/r
  }
  if (r2d > c_tabd.rlo[p] * c_tabd.rlo[p]) {
    R r = sqr_t(r2);
    R ds;
    R s = sw<R>(r, T.rlo[p], T.rc[p], ds);
    dv = dv * s + V * ds / r;
    V = V * s;
  }
  dVr_over_r = dv;
  return V;
}

// b* plateau test of the deferred batch (exact shortcut, forward only): p_ij and p_ji are formed
// as in bo_forward, pi^rc and T are bounded by their tables (Tab::bR*, bT*) and the dihedral sum
// by D <= (sum_k w_ik)(sum_l w_jl) (every term is (1 - cos^2 w) w_ik w_jl G G, G <= 1).  If the
// whole interval lies below b_min (S_b = 1) or above b_max (S_b = 0) by a rounding margin, S_b is
// on a plateau exactly as the full evaluation would find it, and dS_b/db* = 0 (P:488-494:
// "the derivatives of the overall term are zero").  Returns 1 (S_b = 1), 2 (S_b = 0) or 0
// (undecided / bad argument / side larger than NB: *ovf).
template <typename R, int NB>
__device__ __forceinline__ int bstar_plateau(const ShortList<R>& S, const signed char* typ, int i, int J, V3<R> d,
                                             R r, bool& ovf) {
  const Tab<R>& T = tab<R>();
  const int ti = typ[i], tj = typ[J];
  const size_t bi = (size_t)i * S.capS, bj = (size_t)J * S.capS;
  const int ni = S.cnt[i], nj = S.cnt[J];
  int pq = -1, pl = -1;
  for (int q = 0; q < ni; ++q)
    if (S.nbr[bi + q] == J) pq = q;
  for (int q = 0; q < nj; ++q)
    if (S.nbr[bj + q] == i) pl = q;
  const int nI = ni - (pq >= 0), nJ = nj - (pl >= 0);
  ovf = nI > NB || nJ > NB;
  if (ovf) return 0;
  const R ir = R(1) / r;
  R arg[2], wsum[2];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const int c = side ? tj : ti, o = side ? ti : tj, a0 = side ? J : i, n = side ? nJ : nI, ps = side ? pl : pq;
    const size_t b0 = side ? bj : bi;
    const V3<R> dd = side ? mk3(-d.x, -d.y, -d.z) : d;
    const bool blend = c == 0 && T.g2on;
    R s1 = 0, s2 = 0, NC = 0, NH = 0;
    for (int a = 0; a < n; ++a) {
      const int q = side_slot(a, ps);
      const int k = S.nbr[b0 + q];
      R rk;
      const V3<R> dk = sl_d(S, a0, q, rk);
      const R wk = S.w[b0 + q].x;
      const int tk = typ[k];
      const R cs = clamp_cos(dot3(dd, dk) * ir / rk);
      R dg;
      const R ek = explam_r<R>(o, c, tk, r, rk);
      s1 += wk * gspline<R>(c, cs, dg) * ek;
      if (blend) s2 += wk * gspline<R>(2, cs, dg) * ek;
      if (tk == 0) NC += wk;
      else NH += wk;
    }
    if (blend) {
      R dQ;
      const R Q = sw<R>(NC + NH, T.gnlo, T.gnhi, dQ);
      s1 = s2 + Q * (s1 - s2);
    }
    R px, py;
    arg[side] = R(1) + s1 + (c == 0 ? pspline<R>(o, NC, NH, px, py) : R(0));
    wsum[side] = NC + NH;
  }
  if (!(arg[0] > R(0)) || !(arg[1] > R(0))) return 0;  // the full path counts the bad argument
  const int p = ti + tj;
  const R base = R(0.5) * (rsq(arg[0]) + rsq(arg[1]));
  const R Dm = wsum[0] * wsum[1];
  const R hi = base + T.bRhi[p] + (T.bThi[p] > R(0) ? T.bThi[p] : R(0)) * Dm;
  const R lo = base + T.bRlo[p] + (T.bTlo[p] < R(0) ? T.bTlo[p] : R(0)) * Dm;
  const R margin = sizeof(R) == 8 ? R(1e-12) : R(1e-5);
  if (hi < T.bmin[p] - margin) return 1;
  if (lo > T.bmax[p] + margin) return 2;
  return 0;
}

// window-candidate queue in three regions by species pair (region t: item[off[t] .. off[t] +
// cap[t]), count[t] entries), sized from the build-time bound so it cannot overflow
struct BstarQueue {
  int4* item;  // i, J, -, -
  double* M;
  int* count;  // [3]
  int cap[3], off[3];
};

// ---------------------------------------------------------------- deferred b* batch
// E = (S_r S_b(b*) + 1 - S_r) C V for every canonical LJ pair with C != 0 queued as a
// window candidate (r^2 pre-filter); pairs with S_r == 0 reduce to the plain gated LJ C V.
// FULL = false: NB_FAST, forward pass of b* (+ the path forces of a fractional C); a pair whose
// S_b is in its transition (dS_b != 0: the reverse pass of b* is needed) is deferred to ovf for
// FULL = true with NB_FAST register sides, a pair with a side larger than NB_FAST to ovf2 for
// FULL = true with NB = NBMAX.
template <typename R, int NB, bool FULL, bool VIR, bool SG = false>
__global__ void __launch_bounds__(128, (NB <= NB_FAST && !FULL) ? AB_BSTAR_MINBLOCKS : 1) k_bstar(BstarQueue Qu, const int* list_idx, const int* nlist, int* ovf, int* novf, int* ovf2,
                                               int* novf2, const double4* pos, ShortList<R> S, const signed char* typ,
                                               const int* owner, const int* gid, const char4* shift, double* F,
                                               StageBuf stage, RedRows RR) {
  __shared__ RedSmem rs;
  // programmatic dependent launch (AB_PDL): wait for the previous kernel's results (a no-op when
  // the kernel was launched normally)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int q0 = min(Qu.count[0], Qu.cap[0]), q1 = min(Qu.count[1], Qu.cap[1]), q2 = min(Qu.count[2], Qu.cap[2]);
  const int nq = list_idx ? *nlist : q0 + q1 + q2;
  if (red_idle_block(nq, RR)) return;
  red_init(rs);
  const Tab<R>& T = tab<R>();
  double e[1 + 6] = {0, 0, 0, 0, 0, 0, 0};
  unsigned long long ntr = 0, nb = 0, nbad = 0;
  int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += stride) {
    int qi = list_idx ? list_idx[t]
                      : (t < q0 ? Qu.off[0] + t : (t < q0 + q1 ? Qu.off[1] + (t - q0) : Qu.off[2] + (t - q0 - q1)));
    int4 it = Qu.item[qi];
    int i = it.x, J = it.y;
    double Md = Qu.M[qi];
    double4 pi = pos[i], pj = pos[J];
    double dxd = __dsub_rn(pj.x, pi.x), dyd = __dsub_rn(pj.y, pi.y), dzd = __dsub_rn(pj.z, pi.z);
    double r2d = r2_exact(dxd, dyd, dzd);
    double rd = sqrt(r2d);
    int ti = typ[i], tj = typ[J], p = ti + tj;
    // the queue holds window candidates: S_r(r) != 0 decided exactly in fp64 in both precision
    // modes (reading A14); outside the window the pair is the plain gated LJ (Q = 1)
    const bool win = (rd - c_tabd.sigma[p]) / (c_tabd.srhi[p] - c_tabd.sigma[p]) < 1.0;
    V3<R> d = mk3<R>((R)dxd, (R)dyd, (R)dzd);
    R r = (R)rd, ir = R(1) / r;
    R rho = T.rho[p];
    BoState<R, NB> st;
    R bs = 0, B = 1, dB = 0;
    if (win) {
      V3<R> ds = (rho * ir) * d;  // fictitious d* = rho d_hat (reading A8)
      bo_forward<R, false, NB, !FULL || NB <= NB_FAST>(S, typ, i, J, ds, rho, st);
      if (!FULL && st.overflow) {  // a side larger than NB_FAST: the NBMAX kernel
        list_append(ovf2, novf2, 1 << 30, qi);
        continue;
      }
      bs = bo_value(st);
      B = sw<R>(bs, T.bmin[p], T.bmax[p], dB);
    } else {
      st.bad = false;
    }
    if (!FULL && dB != R(0)) {  // S_b transition: the reverse pass of b* in the full kernel
      list_append(ovf, novf, 1 << 30, qi);  // (NB_FAST sides)
      continue;
    }
    R dP = 0;
    R P = win ? sw<R>(r, T.sigma[p], T.srhi[p], dP) : R(0);
    R dVr;
    R V = lj_v<R>(p, (R)r2d, r2d, dVr);
    R C = (R)(1.0 - Md);  // 1 - M in fp64: M may sit within an fp32 ulp of 1 (gate, reading A14)
    R tb = (bs - T.bmin[p]) / (T.bmax[p] - T.bmin[p]);
    if (win && tb > R(0) && tb < R(1)) ++ntr;
    R Q = P * B + R(1) - P;
    R E = Q * C * V;
    V3<R> gd = ((C * (Q * dVr + V * (B - R(1)) * dP * ir))) * d;
    V3<R> fi = mk3<R>(0, 0, 0), fj = mk3<R>(0, 0, 0);
    if (FULL) {
      if (dB != R(0)) {
        V3<R> gs;
        bo_reverse<R, false, NB, false, SG>(S, typ, owner, st, C * V * P * dB, R(0), F, VIR ? e + 1 : nullptr, gs, fi, fj);
        // chain through d* = rho d / |d|: dE/dd = (rho/r) (I - u u^T) dE/dd*
        V3<R> u = ir * d;
        addto(gd, (rho * ir) * (gs - dot3(u, gs) * u));
      }
    }
    if (Md > 0.0) {  // fractional C_ij: dC along the maximising path
      PathRes<R> pr = path_search(S, i, J);
      path_forces<R, SG>(S, owner, pr, -Q * V, F, VIR ? e + 1 : nullptr);
    }
    atomic_add3<SG>(F, owner[i], (double)(gd.x + fi.x), (double)(gd.y + fi.y), (double)(gd.z + fi.z));
    atomic_add3<SG>(F, owner[J], (double)(fj.x - gd.x), (double)(fj.y - gd.y), (double)(fj.z - gd.z));
    vir_add(VIR ? e + 1 : nullptr, d, gd);
    e[0] = acc_round<SG>(e[0] + (double)E);
    nb += win;
    nbad += win && st.bad;
    if (VIR && stage.rows) {
      double* row = stage_row(stage, 7);
      if (row) {
        char4 s = shift[J];
        row[0] = gid[i], row[1] = gid[J], row[2] = s.x, row[3] = s.y, row[4] = s.z;
        row[5] = C, row[6] = bs;
      }
    }
  }
  red_add_d(rs, ACC_ELJ, e[0]);
  for (int c = 0; c < 6; ++c) red_add_d(rs, ACC_W + c, e[1 + c]);
  red_add_u(rs, CT_SBTRANS, ntr);
  red_add_u(rs, CT_BSTAR, nb);
  red_add_u(rs, CT_BADARG, nbad);
  red_flush(rs, RR);
}

// ---------------------------------------------------------------- b* plateau batch (first pass)
// Every queued window candidate with C = 1 (M = 0) whose S_b is decided exactly by
// bstar_plateau (or that lies outside the S_r window): E = (S_r S_b + 1 - S_r) V with S_b in
// {0, 1} and dS_b = 0, forces from S_r and V only.  Everything else -- fractional C, an
// undecided b*, a bad p argument, a side larger than NB_FAST, and every pair while stage rows are
// recorded -- is appended to und for the forward-pass kernel (k_bstar list mode).  Light on
// registers: the full bond-order code is not in this kernel.
#ifndef AB_BSTAR_LITE_MINBLOCKS
#define AB_BSTAR_LITE_MINBLOCKS 6
#endif
template <typename R, bool VIR, bool SG = false>
__global__ void __launch_bounds__(128, AB_BSTAR_LITE_MINBLOCKS) k_bstar_lite(BstarQueue Qu, int* und, int* nund,
                                                                             const double4* pos, ShortList<R> S,
                                                                             const signed char* typ, const int* owner,
                                                                             double* F, bool record, RedRows RR) {
  __shared__ RedSmem rs;
  const int q0 = min(Qu.count[0], Qu.cap[0]), q1 = min(Qu.count[1], Qu.cap[1]), q2 = min(Qu.count[2], Qu.cap[2]);
  const int nq = q0 + q1 + q2;
  if (red_idle_block(nq, RR)) return;
  red_init(rs);
  const Tab<R>& T = tab<R>();
  double e[1 + 6] = {0, 0, 0, 0, 0, 0, 0};
  unsigned long long nb = 0;
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += stride) {
    const int qi = t < q0 ? Qu.off[0] + t : (t < q0 + q1 ? Qu.off[1] + (t - q0) : Qu.off[2] + (t - q0 - q1));
    const int4 it = Qu.item[qi];
    const int i = it.x, J = it.y;
    if (record || Qu.M[qi] > 0.0) {
      list_append(und, nund, 1 << 30, qi);
      continue;
    }
    const double4 pi = pos[i], pj = pos[J];
    const double dxd = __dsub_rn(pj.x, pi.x), dyd = __dsub_rn(pj.y, pi.y), dzd = __dsub_rn(pj.z, pi.z);
    const double r2d = r2_exact(dxd, dyd, dzd);
    const double rd = sqrt(r2d);
    const int p = typ[i] + typ[J];
    const bool win = (rd - c_tabd.sigma[p]) / (c_tabd.srhi[p] - c_tabd.sigma[p]) < 1.0;  // as k_bstar
    const V3<R> d = mk3<R>((R)dxd, (R)dyd, (R)dzd);
    const R r = (R)rd, ir = R(1) / r;
    R B = 1;
    if (win) {
      const R rho = T.rho[p];
      bool ov = false;
      const int plat = bstar_plateau<R, NB_FAST>(S, typ, i, J, (rho * ir) * d, rho, ov);
      if (ov || plat == 0) {
        list_append(und, nund, 1 << 30, qi);
        continue;
      }
      B = plat == 1 ? R(1) : R(0);
    }
    R dP = 0;
    const R P = win ? sw<R>(r, T.sigma[p], T.srhi[p], dP) : R(0);
    R dVr;
    const R V = lj_v<R>(p, (R)r2d, r2d, dVr);
    const R Q = P * B + R(1) - P;  // C = 1
    const V3<R> gd = (Q * dVr + V * (B - R(1)) * dP * ir) * d;
    atomic_add3<SG>(F, owner[i], (double)gd.x, (double)gd.y, (double)gd.z);
    atomic_add3<SG>(F, owner[J], -(double)gd.x, -(double)gd.y, -(double)gd.z);
    vir_add(VIR ? e + 1 : nullptr, d, gd);
    e[0] = acc_round<SG>(e[0] + (double)(Q * V));
    nb += win;
  }
  red_add_d(rs, ACC_ELJ, e[0]);
  for (int c = 0; c < 6; ++c) red_add_d(rs, ACC_W + c, e[1 + c]);
  red_add_u(rs, CT_BSTAR, nb);
  red_flush(rs, RR);
}

}  // namespace ab
