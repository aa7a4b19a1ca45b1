// oracle/airebo.cpp -- plain, slow, fp64 CPU oracle of the AIREBO energy, forces and virial.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may build, load or call anything under oracle/.  It shares no code,
// header, table or helper with the CUDA path (paper_1810_07026_b200/csrc) and neither side
// includes the other.  Compiled with -O2 -ffp-contract=off (no FMA contraction).
//
// What it computes (the plain definitions; every optimisation of the
// paper reaches exactly this result):
//   E = E_REBO + E_TORS + E_LJ over all periodic images (explicit images),
//   F_a = -dE/dx_a by reverse-mode AD of each term (oracle/ad.hpp),
//   W_ab = sum_terms sum_{instances q} (u_q - u_owner)_a F_{q,b}.
// Terms:
//   REBO bond (i<j)  E = f_R(r) + b_ij f_A(r)                         P:415-417, Alg.1
//   bond order b_ij = 1/2 (p_ij + p_ji) + pi^rc + pi^dh                 P:496-506, reading A1 (sum)
//   p_ij = [1 + sum_k w_ik g_i(cos th_jik) e^{lam_jik} + P_ij]^{-1/2}
//   pi^rc = R(N_ij, N_ji, N^conj), pi^dh = T(...) sum_k sum_l (1-cos^2 w) w_ik w_jl G G
//                                                                       P:500-504
//   torsion per bond: sum_{k,l} eps_kijl w_ki w_ij w_jl G G V(cos w)    Alg.2
//   LJ (i<j): E = (S_r S_b(b*) + 1 - S_r) C_ij V_LJ(r)                  P:467, Alg.3
//   C_ij = 1 - max{w_ij, w_ik w_kj, w_ik w_kl w_lj}  (nested search)
//   b*: bond order with d_ij -> rho d_ij/|d_ij|                         P:488-494, reading A8
// Variants (param key `potential`): REBO = the REBO bond terms only (no
// torsion, no LJ); AIREBO-M = V_LJ replaced by eps_m [e^{-2a(r-re)} - 2 e^{-a(r-re)}]
// with every gate, switch and the taper kept (reading A31).
// Functional forms and spline rules: SURVEY A2, A5-A11.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "ad.hpp"
#include "params.hpp"

namespace ad {
Tape& tape() {
  thread_local Tape t;
  return t;
}
}  // namespace ad

namespace orc {

using ad::val;
using ad::Var;
static const int CARBON = 0;
static const double SR_FACTOR = 1.122462048309373;  // 2^(1/6), S_r upper bound = 2^(1/6) sigma (A11)

// ------------------------------------------------------------------ small vector type
template <class T>
struct V3 {
  T x, y, z;
};
template <class T>
V3<T> operator-(const V3<T>& a, const V3<T>& b) {
  return V3<T>{a.x - b.x, a.y - b.y, a.z - b.z};
}
template <class T>
V3<T> operator*(const T& s, const V3<T>& a) {
  return V3<T>{s * a.x, s * a.y, s * a.z};
}
template <class T>
V3<T> neg(const V3<T>& a) {
  return V3<T>{-a.x, -a.y, -a.z};
}
template <class T>
T dot(const V3<T>& a, const V3<T>& b) {
  return (a.x * b.x + a.y * b.y) + a.z * b.z;
}
template <class T>
V3<T> cross(const V3<T>& a, const V3<T>& b) {
  return V3<T>{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class T>
T norm(const V3<T>& a) {
  using std::sqrt;
  return sqrt(dot(a, a));
}

template <class T>
T mkleaf(double v);
template <>
double mkleaf<double>(double v) {
  return v;
}
template <>
Var mkleaf<Var>(double v) {
  return ad::leaf(v);
}

// ------------------------------------------------------------------ scalar building blocks
// Switch S(x; lo, hi): t = (x-lo)/(hi-lo); 1 for t<=0, 0 for t>=1, else (1+cos(pi t))/2.
// SPEC S:176-179 (half-cosine); the decision uses the same IEEE t on every side.
template <class T>
T Sw(const T& x, double lo, double hi) {
  using std::cos;
  double t = (val(x) - lo) / (hi - lo);
  if (t <= 0.0) return T(1.0);
  if (t >= 1.0) return T(0.0);
  T tt = (x - lo) / (hi - lo);
  return 0.5 * (1.0 + cos(M_PI * tt));
}

// 1-D cubic Hermite on non-uniform knots, slopes m_i = (y_{i+1}-y_{i-1})/(x_{i+1}-x_{i-1})
// inside, m = 0 at both end knots, clamped outside with zero derivative.
template <class T>
T hermite1(const Spline1& s, const T& x) {
  int n = (int)s.x.size();
  double xv = val(x);
  if (xv <= s.x[0]) return T(s.y[0]);
  if (xv >= s.x[n - 1]) return T(s.y[n - 1]);
  int i = 0;
  while (i < n - 2 && s.x[i + 1] <= xv) ++i;
  auto slope = [&](int q) { return (q == 0 || q == n - 1) ? 0.0 : (s.y[q + 1] - s.y[q - 1]) / (s.x[q + 1] - s.x[q - 1]); };
  double h = s.x[i + 1] - s.x[i];
  T t = (x - s.x[i]) / h;
  T t2 = t * t, t3 = t2 * t;
  T h00 = 2.0 * t3 - 3.0 * t2 + 1.0;
  T h10 = t3 - 2.0 * t2 + t;
  T h01 = -2.0 * t3 + 3.0 * t2;
  T h11 = t3 - t2;
  return h00 * s.y[i] + h10 * (h * slope(i)) + h01 * s.y[i + 1] + h11 * (h * slope(i + 1));
}

// Weights W[a] of the knot values for the 1-D Hermite scheme on the integer grid lo, lo+1, ...,
// lo+n-1 (slopes (y_{i+1}-y_{i-1})/2 inside, 0 at the ends; clamped).  f(x) = sum_a W[a] y_a.
// The 2-D / 3-D splines are the tensor products of this linear scheme (SURVEY A7 "tricubic").
template <class T>
void grid_weights(const T& x, double lo, int n, T* W, bool* used) {
  for (int a = 0; a < n; ++a) used[a] = false, W[a] = T(0.0);
  double hi = lo + (n - 1);
  T xc = x;
  if (val(x) <= lo) xc = T(lo);
  else if (val(x) >= hi) xc = T(hi);
  int i = (int)std::floor(val(xc) - lo);
  if (i > n - 2) i = n - 2;  // last knot -> last cell
  if (i < 0) i = 0;
  T t = xc - (lo + i);
  T t2 = t * t, t3 = t2 * t;
  T h00 = 2.0 * t3 - 3.0 * t2 + 1.0;
  T h10 = t3 - 2.0 * t2 + t;
  T h01 = -2.0 * t3 + 3.0 * t2;
  T h11 = t3 - t2;
  auto add = [&](int a, const T& v) {
    W[a] = used[a] ? W[a] + v : v;
    used[a] = true;
  };
  add(i, h00);
  add(i + 1, h01);
  if (i > 0 && i < n - 1) {  // m_i = (y_{i+1} - y_{i-1}) / 2
    add(i + 1, 0.5 * h10);
    add(i - 1, -0.5 * h10);
  }
  if (i + 1 > 0 && i + 1 < n - 1) {  // m_{i+1} = (y_{i+2} - y_i) / 2
    add(i + 2, 0.5 * h11);
    add(i, -0.5 * h11);
  }
}

template <class T>
T spline2(const std::vector<double>& tab, const double lo[2], const int n[2], const T& x, const T& y) {
  T wx[16], wy[16];
  bool ux[16], uy[16];
  grid_weights(x, lo[0], n[0], wx, ux);
  grid_weights(y, lo[1], n[1], wy, uy);
  T f(0.0);
  for (int a = 0; a < n[0]; ++a) {
    if (!ux[a]) continue;
    for (int b = 0; b < n[1]; ++b) {
      if (!uy[b]) continue;
      f = f + (wx[a] * wy[b]) * tab[(size_t)a * n[1] + b];
    }
  }
  return f;
}

template <class T>
T spline3(const std::vector<double>& tab, const double lo[3], const int n[3], const T& x, const T& y, const T& z) {
  T wx[16], wy[16], wz[16];
  bool ux[16], uy[16], uz[16];
  grid_weights(x, lo[0], n[0], wx, ux);
  grid_weights(y, lo[1], n[1], wy, uy);
  grid_weights(z, lo[2], n[2], wz, uz);
  T f(0.0);
  for (int a = 0; a < n[0]; ++a) {
    if (!ux[a]) continue;
    for (int b = 0; b < n[1]; ++b) {
      if (!uy[b]) continue;
      for (int c = 0; c < n[2]; ++c) {
        if (!uz[c]) continue;
        f = f + ((wx[a] * wy[b]) * wz[c]) * tab[((size_t)a * n[1] + b) * n[2] + c];
      }
    }
  }
  return f;
}

inline int pidx(int ti, int tj) { return ti + tj; }  // 0 = CC, 1 = CH, 2 = HH

// P_ij(N^C_ij, N^H_ij); zero for an H centre
template <class T>
T Pspline(const Params& p, int ti, int tj, const T& NC, const T& NH) {
  if (ti != CARBON) return T(0.0);
  return spline2(p.P[tj], p.Plo, p.Pn, NC, NH);
}
// pi^rc (which=0) or T (which=1) at (N_ij, N_ji, N^conj); CH tables take the C side first (O5.5)
template <class T>
T RTspline(const Params& p, int which, int ti, int tj, const T& Nij, const T& Nji, const T& Nc) {
  const std::vector<double>& tab = which == 0 ? p.R[pidx(ti, tj)] : p.T[pidx(ti, tj)];
  if (ti != CARBON && tj == CARBON) return spline3(tab, p.RTlo, p.RTn, Nji, Nij, Nc);
  return spline3(tab, p.RTlo, p.RTn, Nij, Nji, Nc);
}

// collinearity guard G(cos) = 1 - S(1 - cos^2; s2lo, s2hi) (reading A9)
template <class T>
T Gguard(const Params& p, const T& c) {
  return 1.0 - Sw(1.0 - c * c, p.s2lo, p.s2hi);
}

// V_tors(cos w) = (256/405) ((1+c)/2)^5 - 1/10  (= cos^10(w/2) form)
template <class T>
T Vtors(const T& c) {
  T h = 0.5 * (1.0 + c);
  T h2 = h * h;
  return (256.0 / 405.0) * (h2 * h2 * h) - 0.1;
}

// ------------------------------------------------------------------ system, images, lists
struct Sys {
  int n;
  const int* type;
  const double* x;
  double L[3];
};

struct Inst {
  int a;
  int s[3];
  bool operator==(const Inst& o) const { return a == o.a && s[0] == o.s[0] && s[1] == o.s[1] && s[2] == o.s[2]; }
};

struct Nb {
  int j;
  int s[3];
  double d[3];
  double r;
};

// displacement d = (x_j + s L) - x_i, evaluated as t = s*L; u = x_j + t; d = u - x_i
inline void image_pos(const Sys& S, int j, const int s[3], double u[3]) {
  for (int c = 0; c < 3; ++c) {
    double t = (double)s[c] * S.L[c];
    u[c] = S.x[3 * j + c] + t;
  }
}
inline double r2_of(const double d[3]) { return (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]; }

inline bool lex_pos(const int s[3]) { return s[0] > 0 || (s[0] == 0 && (s[1] > 0 || (s[1] == 0 && s[2] > 0))); }
// half convention: keep (i, j, s) iff i < j, or i == j and s >_lex 0
inline bool canonical(int i, int j, const int s[3]) { return i < j || (i == j && lex_pos(s)); }

// All instances (j, s) != (i, 0) with |d|^2 <= cut(t_i, t_j)^2.  Cell list over the image
// cloud of the padded box (or brute force over all atoms x all shifts when brute = true).
struct Finder {
  const Sys& S;
  double R;
  bool brute;
  int smax[3];
  std::vector<int> ia;
  std::vector<std::array<int, 3>> is;
  std::vector<std::array<double, 3>> iu;
  int nc[3];
  double cs[3];
  std::vector<int> cstart, cidx;

  Finder(const Sys& s, double R_, bool brute_) : S(s), R(R_), brute(brute_) {
    for (int c = 0; c < 3; ++c) smax[c] = (int)std::ceil(R / S.L[c]) + 1;
    if (brute) return;
    for (int a = 0; a < S.n; ++a)
      for (int sx = -smax[0]; sx <= smax[0]; ++sx)
        for (int sy = -smax[1]; sy <= smax[1]; ++sy)
          for (int sz = -smax[2]; sz <= smax[2]; ++sz) {
            int sh[3] = {sx, sy, sz};
            double u[3];
            image_pos(S, a, sh, u);
            bool in = true;
            for (int c = 0; c < 3; ++c) in = in && u[c] >= -R && u[c] < S.L[c] + R;
            if (!in) continue;
            ia.push_back(a);
            is.push_back({sx, sy, sz});
            iu.push_back({u[0], u[1], u[2]});
          }
    for (int c = 0; c < 3; ++c) {
      double span = S.L[c] + 2 * R;
      nc[c] = std::max(1, (int)std::floor(span / R));
      cs[c] = span / nc[c];
    }
    size_t ncell = (size_t)nc[0] * nc[1] * nc[2];
    std::vector<int> cnt(ncell + 1, 0), cell(ia.size());
    for (size_t q = 0; q < ia.size(); ++q) {
      int c3[3];
      for (int c = 0; c < 3; ++c) c3[c] = std::min(nc[c] - 1, std::max(0, (int)std::floor((iu[q][c] + R) / cs[c])));
      cell[q] = (c3[0] * nc[1] + c3[1]) * nc[2] + c3[2];
      cnt[cell[q] + 1]++;
    }
    for (size_t c = 0; c < ncell; ++c) cnt[c + 1] += cnt[c];
    cstart = cnt;
    cidx.resize(ia.size());
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (size_t q = 0; q < ia.size(); ++q) cidx[fill[cell[q]]++] = (int)q;
  }

  // visit(j, s, d, r2) for every instance (j, s) != (i, 0) with |d| <= R (squared compare)
  template <class F>
  void around(int i, F visit) const {
    const double* xi = S.x + 3 * i;
    double R2 = R * R;
    if (brute) {
      for (int j = 0; j < S.n; ++j)
        for (int sx = -smax[0]; sx <= smax[0]; ++sx)
          for (int sy = -smax[1]; sy <= smax[1]; ++sy)
            for (int sz = -smax[2]; sz <= smax[2]; ++sz) {
              int sh[3] = {sx, sy, sz};
              if (j == i && sx == 0 && sy == 0 && sz == 0) continue;
              double u[3], d[3];
              image_pos(S, j, sh, u);
              for (int c = 0; c < 3; ++c) d[c] = u[c] - xi[c];
              double r2 = r2_of(d);
              if (r2 <= R2) visit(j, sh, d, r2);
            }
      return;
    }
    int c3[3];
    for (int c = 0; c < 3; ++c) c3[c] = std::min(nc[c] - 1, std::max(0, (int)std::floor((xi[c] + R) / cs[c])));
    for (int ax = std::max(0, c3[0] - 1); ax <= std::min(nc[0] - 1, c3[0] + 1); ++ax)
      for (int ay = std::max(0, c3[1] - 1); ay <= std::min(nc[1] - 1, c3[1] + 1); ++ay)
        for (int az = std::max(0, c3[2] - 1); az <= std::min(nc[2] - 1, c3[2] + 1); ++az) {
          int cell = (ax * nc[1] + ay) * nc[2] + az;
          for (int p = cstart[cell]; p < cstart[cell + 1]; ++p) {
            int q = cidx[p];
            int j = ia[q];
            const auto& sh = is[q];
            if (j == i && sh[0] == 0 && sh[1] == 0 && sh[2] == 0) continue;
            double d[3];
            for (int c = 0; c < 3; ++c) d[c] = iu[q][c] - xi[c];
            double r2 = r2_of(d);
            if (r2 <= R2) visit(j, sh.data(), d, r2);
          }
        }
  }
};

inline bool nb_less(const Nb& a, const Nb& b) {
  if (a.j != b.j) return a.j < b.j;
  for (int c = 0; c < 3; ++c)
    if (a.s[c] != b.s[c]) return a.s[c] < b.s[c];
  return false;
}

struct Lists {
  std::vector<std::vector<Nb>> shortl;  // full short list, r^2 <= rmax^2, sorted by (j, s)
  std::vector<std::vector<Nb>> lj;      // LJ half pairs, r^2 <= rc^2, canonical, sorted
};

inline void build_lists(const Params& P, const Sys& S, bool brute, bool want_lj, Lists& Lo) {
  double rmaxmax = 0, rcmax = 0;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      rmaxmax = std::max(rmaxmax, P.pair[a][b].rmax);
      rcmax = std::max(rcmax, P.pair[a][b].rc);
    }
  Lo.shortl.assign(S.n, {});
  Lo.lj.assign(S.n, {});
  Finder fs(S, rmaxmax, brute);
  for (int i = 0; i < S.n; ++i) {
    fs.around(i, [&](int j, const int* s, const double* d, double r2) {
      double rm = P.pair[S.type[i]][S.type[j]].rmax;
      if (r2 <= rm * rm) {
        Nb e;
        e.j = j;
        for (int c = 0; c < 3; ++c) e.s[c] = s[c], e.d[c] = d[c];
        e.r = std::sqrt(r2);
        Lo.shortl[i].push_back(e);
      }
    });
    std::sort(Lo.shortl[i].begin(), Lo.shortl[i].end(), nb_less);
  }
  if (!want_lj || P.potential == POT_REBO) return;  // REBO: no inter-molecular term
  Finder fl(S, rcmax, brute);
#pragma omp parallel for schedule(dynamic, 64)
  for (int i = 0; i < S.n; ++i) {
    fl.around(i, [&](int j, const int* s, const double* d, double r2) {
      double rc = P.pair[S.type[i]][S.type[j]].rc;
      if (r2 <= rc * rc && canonical(i, j, s)) {
        Nb e;
        e.j = j;
        for (int c = 0; c < 3; ++c) e.s[c] = s[c], e.d[c] = d[c];
        e.r = std::sqrt(r2);
        Lo.lj[i].push_back(e);
      }
    });
    std::sort(Lo.lj[i].begin(), Lo.lj[i].end(), nb_less);
  }
}

// ------------------------------------------------------------------ terms
// Leaves of one term: every (atom, image) instance it reads, in the owner i's frame.
template <class T>
struct Ctx {
  const Sys* S;
  std::vector<int> atom;
  std::vector<std::array<double, 3>> u;
  std::vector<V3<T>> pos;
  int add(int a, const int s[3]) {
    double uu[3];
    image_pos(*S, a, s, uu);
    atom.push_back(a);
    u.push_back({uu[0], uu[1], uu[2]});
    pos.push_back(V3<T>{mkleaf<T>(uu[0]), mkleaf<T>(uu[1]), mkleaf<T>(uu[2])});
    return (int)atom.size() - 1;
  }
};

// One side of a bond (centre c, partner excluded): the neighbours k of c.
template <class T>
struct Side {
  int tc;
  std::vector<int> tk;
  std::vector<V3<T>> dk;  // centre -> k
  std::vector<T> rk, wk;
  std::vector<T> nkm;  // C-type k: N_k - w_ck = sum_{m in N(k), m != centre} w_km  ("N_ki")
  std::vector<Inst> key;
};

template <class T>
void build_side(const Params& P, const Lists& Lo, Ctx<T>& cx, int centre, const int cs[3], int qc, const Inst& partner,
                Side<T>& sd) {
  const Sys& S = *cx.S;
  sd.tc = S.type[centre];
  for (const Nb& e : Lo.shortl[centre]) {
    Inst ik{e.j, {cs[0] + e.s[0], cs[1] + e.s[1], cs[2] + e.s[2]}};
    if (ik == partner) continue;
    int tk = S.type[e.j];
    int qk = cx.add(e.j, ik.s);
    V3<T> d = cx.pos[qk] - cx.pos[qc];
    T r = norm(d);
    const PairParams& pp = P.pair[sd.tc][tk];
    T w = Sw(r, pp.rmin, pp.rmax);
    T nk(0.0);
    if (tk == CARBON) {
      Inst cen{centre, {cs[0], cs[1], cs[2]}};
      for (const Nb& f : Lo.shortl[e.j]) {
        Inst im{f.j, {ik.s[0] + f.s[0], ik.s[1] + f.s[1], ik.s[2] + f.s[2]}};
        if (im == cen) continue;
        int qm = cx.add(f.j, im.s);
        T rkm = norm(cx.pos[qm] - cx.pos[qk]);
        const PairParams& pk = P.pair[tk][S.type[f.j]];
        nk = nk + Sw(rkm, pk.rmin, pk.rmax);
      }
    }
    sd.tk.push_back(tk);
    sd.dk.push_back(d);
    sd.rk.push_back(r);
    sd.wk.push_back(w);
    sd.nkm.push_back(nk);
    sd.key.push_back(ik);
  }
}

template <class T>
T clamp1(const T& c) {
  if (val(c) > 1.0) return T(1.0);
  if (val(c) < -1.0) return T(-1.0);
  return c;
}

// g_i(cos theta) of centre species tc with coordination N (reading A34):
// g_C(c, N) = g_C2(c) + S(N; nlo, nhi) (g_C(c) - g_C2(c)) if angle.C2 is given, else g_tc(c)
template <class T>
T gfun(const Params& P, int tc, const T& c, const T& N) {
  if (tc != CARBON || !P.has_gC2) return hermite1(P.g[tc], c);
  T g1 = hermite1(P.g[CARBON], c), g2 = hermite1(P.gC2, c);
  return g2 + Sw(N, P.gC_nlo, P.gC_nhi) * (g1 - g2);
}

// lambda_jik (reading A33): constant table + kappa delta(t_i, H)
// [(rho_{t_k H} - r_ik) - (rho_{t_j H} - r_ij)]; r_ij = |d| is the fictitious rho in b*
template <class T>
T lambda_jik(const Params& P, int tj, int ti, int tk, const T& rij, const T& rik) {
  T lam(P.lam[tj][ti][tk]);
  if (ti == CARBON || P.kappa == 0.0) return lam;
  return lam + P.kappa * ((P.pair[tk][1].rho - rik) - (P.pair[tj][1].rho - rij));
}

// p^{sigma pi} of one side: [1 + sum_k w_ck g_c(cos th) e^{lam} + P]^{-1/2}
template <class T>
T p_sigma_pi(const Params& P, int tpartner, const V3<T>& d, const Side<T>& sd, std::vector<T>& cosv, T& NC, T& NH,
             bool& ok) {
  using std::exp;
  using std::sqrt;
  T r = norm(d);
  T sum(0.0);
  NC = T(0.0);
  NH = T(0.0);
  cosv.clear();
  for (size_t k = 0; k < sd.tk.size(); ++k) {  // N^C_ij, N^H_ij (O4): the side excludes the partner
    if (sd.tk[k] == CARBON) NC = NC + sd.wk[k];
    else NH = NH + sd.wk[k];
  }
  T Nside = NC + NH;
  for (size_t k = 0; k < sd.tk.size(); ++k) {
    T c = clamp1(dot(d, sd.dk[k]) / (r * sd.rk[k]));
    cosv.push_back(c);
    sum = sum + sd.wk[k] * gfun(P, sd.tc, c, Nside) * exp(lambda_jik(P, tpartner, sd.tc, sd.tk[k], r, sd.rk[k]));
  }
  T arg = (1.0 + sum) + Pspline(P, sd.tc, tpartner, NC, NH);
  ok = val(arg) > 0.0;
  return 1.0 / sqrt(arg);
}

struct BondInfo {
  double b, pij, pji, pirc, pidh, Nij, Nji, Nconj;
  long long nquads;
  bool ok;
};

// b_ij, d = vector i -> j (d_ij for REBO, rho d_hat for b*), I = side of i, J = side of j
template <class T>
T bond_order(const Params& P, int ti, int tj, const V3<T>& d, const Side<T>& I, const Side<T>& J, BondInfo* info) {
  std::vector<T> ci, cj;
  T NCi, NHi, NCj, NHj;
  bool ok1, ok2;
  T pij = p_sigma_pi(P, tj, d, I, ci, NCi, NHi, ok1);
  T pji = p_sigma_pi(P, ti, neg(d), J, cj, NCj, NHj, ok2);
  T Nij = NCi + NHi, Nji = NCj + NHj;
  T si(0.0), sj(0.0);
  for (size_t k = 0; k < I.tk.size(); ++k)
    if (I.tk[k] == CARBON) si = si + I.wk[k] * Sw(I.nkm[k], P.conj_lo, P.conj_hi);
  for (size_t l = 0; l < J.tk.size(); ++l)
    if (J.tk[l] == CARBON) sj = sj + J.wk[l] * Sw(J.nkm[l], P.conj_lo, P.conj_hi);
  T Nconj = (1.0 + si * si) + sj * sj;
  T pirc = RTspline(P, 0, ti, tj, Nij, Nji, Nconj);
  T Tij = RTspline(P, 1, ti, tj, Nij, Nji, Nconj);
  // dihedral sum: k in N(i)\j, l in N(j)\{i,k}
  T dsum(0.0);
  long long nq = 0;
  for (size_t k = 0; k < I.tk.size(); ++k) {
    for (size_t l = 0; l < J.tk.size(); ++l) {
      if (J.key[l] == I.key[k]) continue;
      ++nq;
      T Gk = Gguard(P, ci[k]), Gl = Gguard(P, cj[l]);
      if (val(Gk) == 0.0 || val(Gl) == 0.0) continue;
      V3<T> n1 = cross(I.dk[k], d);
      V3<T> n2 = cross(neg(d), J.dk[l]);
      T cw = dot(n1, n2) / (norm(n1) * norm(n2));
      dsum = dsum + (((1.0 - cw * cw) * I.wk[k]) * J.wk[l]) * Gk * Gl;
    }
  }
  T pidh = Tij * dsum;
  T b = (0.5 * (pij + pji) + pirc) + pidh;
  if (info) {
    info->b = val(b);
    info->pij = val(pij);
    info->pji = val(pji);
    info->pirc = val(pirc);
    info->pidh = val(pidh);
    info->Nij = val(Nij);
    info->Nji = val(Nji);
    info->Nconj = val(Nconj);
    info->nquads = nq;
    info->ok = ok1 && ok2;
  }
  return b;
}

// ------------------------------------------------------------------ accumulation
enum {
  CNT_SHORT = 0,  // full short-list entries
  CNT_BONDS,      // REBO half bonds
  CNT_QUADS,      // enumerated (bond, k, l) quadruples, l != k
  CNT_LJ,         // LJ half pairs with r <= rc
  CNT_C0,         // ... of which C == 0
  CNT_BSTAR,      // ... with C != 0 and S_r != 0 (b* evaluated)
  CNT_SBTRANS,    // ... of which b* strictly inside (bmin, bmax)
  CNT_MAXSHORT,   // max |N(i)|
  CNT_MAXREACH,   // max number of distinct instances within 3 bonds of i (excluding i)
  CNT_BADARG,     // p^{sigma pi} argument <= 0 (must stay 0)
  NCNT
};

struct Acc {
  std::vector<double> F;  // n*3
  double E[3] = {0, 0, 0};
  double W[6] = {0, 0, 0, 0, 0, 0};
  long long cnt[NCNT] = {0};
  const std::vector<char>* fmask = nullptr;  // sampled mode: only accumulate forces of these atoms
};

template <class T>
void scatter(Ctx<T>& cx, const T& E, Acc& acc) {}

template <>
void scatter<Var>(Ctx<Var>& cx, const Var& E, Acc& acc) {
  std::vector<double> adj;
  ad::backward(E.id, adj);
  const auto& u0 = cx.u[0];
  for (size_t q = 0; q < cx.atom.size(); ++q) {
    double g[3] = {0, 0, 0};
    const V3<Var>& p = cx.pos[q];
    if (p.x.id >= 0) g[0] = adj[p.x.id];
    if (p.y.id >= 0) g[1] = adj[p.y.id];
    if (p.z.id >= 0) g[2] = adj[p.z.id];
    int a = cx.atom[q];
    if (!acc.fmask || (*acc.fmask)[a])
      for (int c = 0; c < 3; ++c) acc.F[3 * a + c] -= g[c];
    double rel[3] = {cx.u[q][0] - u0[0], cx.u[q][1] - u0[1], cx.u[q][2] - u0[2]};
    acc.W[0] += rel[0] * -g[0];
    acc.W[1] += rel[1] * -g[1];
    acc.W[2] += rel[2] * -g[2];
    acc.W[3] += rel[0] * -g[1];
    acc.W[4] += rel[0] * -g[2];
    acc.W[5] += rel[1] * -g[2];
  }
}

// REBO + torsion of the half bond (i, e = (j, s)); Alg. 1 / Alg. 2
template <class T>
void eval_bond(const Params& P, const Sys& S, const Lists& Lo, int i, const Nb& e, Acc& acc, BondInfo* info) {
  using std::exp;
  if (std::is_same<T, Var>::value) ad::tape().clear();
  Ctx<T> cx;
  cx.S = &S;
  int zero[3] = {0, 0, 0};
  int qi = cx.add(i, zero);
  int qj = cx.add(e.j, e.s);
  int ti = S.type[i], tj = S.type[e.j];
  Inst inst_i{i, {0, 0, 0}}, inst_j{e.j, {e.s[0], e.s[1], e.s[2]}};
  Side<T> I, J;
  build_side(P, Lo, cx, i, zero, qi, inst_j, I);
  build_side(P, Lo, cx, e.j, e.s, qj, inst_i, J);
  V3<T> d = cx.pos[qj] - cx.pos[qi];
  T r = norm(d);
  const PairParams& pp = P.pair[ti][tj];
  T w = Sw(r, pp.rmin, pp.rmax);
  T VR = ((w * (1.0 + pp.Q / r)) * pp.A) * exp(-pp.alpha * r);
  T VA = -w * ((pp.B[0] * exp(-pp.beta[0] * r) + pp.B[1] * exp(-pp.beta[1] * r)) + pp.B[2] * exp(-pp.beta[2] * r));
  BondInfo bi;
  T b = bond_order(P, ti, tj, d, I, J, &bi);
  T Erebo = VR + b * VA;
  // torsion (reading A9: guard G on both angles; A12: eps keyed K I J L); none in REBO
  T Etors(0.0);
  const size_t nk_tors = P.potential == POT_REBO ? 0 : I.tk.size();
  for (size_t k = 0; k < nk_tors; ++k) {
    T ck = clamp1(dot(d, I.dk[k]) / (r * I.rk[k]));
    T Gk = Gguard(P, ck);
    if (val(Gk) == 0.0) continue;
    for (size_t l = 0; l < J.tk.size(); ++l) {
      if (J.key[l] == I.key[k]) continue;
      T cl = clamp1(dot(neg(d), J.dk[l]) / (r * J.rk[l]));
      T Gl = Gguard(P, cl);
      if (val(Gl) == 0.0) continue;
      V3<T> n1 = cross(I.dk[k], d);
      V3<T> n2 = cross(neg(d), J.dk[l]);
      T cw = dot(n1, n2) / (norm(n1) * norm(n2));
      double eps = P.tors[I.tk[k]][ti][tj][J.tk[l]];
      Etors = Etors + ((((eps * I.wk[k]) * w) * J.wk[l]) * Gk * Gl) * Vtors(cw);
    }
  }
  acc.E[0] += val(Erebo);
  acc.E[1] += val(Etors);
  acc.cnt[CNT_BONDS] += 1;
  acc.cnt[CNT_QUADS] += bi.nquads;
  if (!bi.ok) acc.cnt[CNT_BADARG] += 1;
  if (info) *info = bi;
  scatter(cx, Erebo + Etors, acc);
}

struct CResult {
  double M;
  int hops;     // 0 none, 1, 2, 3
  Nb e1, e2, e3;  // path entries (e1 in N(i), e2 in N(k), e3 in N(l))
  Inst k, l;
};

inline double wlist(const Params& P, const Sys& S, int a, int b, double r) {
  return Sw(r, P.pair[S.type[a]][S.type[b]].rmin, P.pair[S.type[a]][S.type[b]].rmax);
}

// Nested search of P:844-853 for M = max{w_ij, w_ik w_kj, w_ik w_kl w_lj}; first maximiser in the
// canonical order (1-hop; then k ascending by (atom, image); then (k, l)) is kept.
inline CResult cij_search(const Params& P, const Sys& S, const Lists& Lo, int i, const Inst& tgt) {
  CResult R;
  R.M = 0.0;
  R.hops = 0;
  Inst me{i, {0, 0, 0}};
  for (const Nb& e1 : Lo.shortl[i]) {
    Inst k{e1.j, {e1.s[0], e1.s[1], e1.s[2]}};
    if (k == tgt) {
      double c = wlist(P, S, i, e1.j, e1.r);
      if (c > R.M) R.M = c, R.hops = 1, R.e1 = e1;
    }
  }
  for (const Nb& e1 : Lo.shortl[i]) {
    Inst k{e1.j, {e1.s[0], e1.s[1], e1.s[2]}};
    if (k == tgt) continue;
    double w1 = wlist(P, S, i, e1.j, e1.r);
    for (const Nb& e2 : Lo.shortl[e1.j]) {
      Inst l{e2.j, {k.s[0] + e2.s[0], k.s[1] + e2.s[1], k.s[2] + e2.s[2]}};
      if (l == me || !(l == tgt)) continue;
      double c = w1 * wlist(P, S, e1.j, e2.j, e2.r);
      if (c > R.M) R.M = c, R.hops = 2, R.e1 = e1, R.e2 = e2, R.k = k;
    }
  }
  for (const Nb& e1 : Lo.shortl[i]) {
    Inst k{e1.j, {e1.s[0], e1.s[1], e1.s[2]}};
    if (k == tgt) continue;
    double w1 = wlist(P, S, i, e1.j, e1.r);
    for (const Nb& e2 : Lo.shortl[e1.j]) {
      Inst l{e2.j, {k.s[0] + e2.s[0], k.s[1] + e2.s[1], k.s[2] + e2.s[2]}};
      if (l == me || l == tgt) continue;
      double w2 = wlist(P, S, e1.j, e2.j, e2.r);
      for (const Nb& e3 : Lo.shortl[e2.j]) {
        Inst m{e3.j, {l.s[0] + e3.s[0], l.s[1] + e3.s[1], l.s[2] + e3.s[2]}};
        if (!(m == tgt)) continue;
        double c = (w1 * w2) * wlist(P, S, e2.j, e3.j, e3.r);
        if (c > R.M) R.M = c, R.hops = 3, R.e1 = e1, R.e2 = e2, R.e3 = e3, R.k = k, R.l = l;
      }
    }
  }
  return R;
}

struct LJInfo {
  double C, bstar, Q, E;
  bool bstar_evaluated;
};

// LJ half pair (i, e = (j, s)); Alg. 3 and P:467
template <class T>
void eval_lj(const Params& P, const Sys& S, const Lists& Lo, int i, const Nb& e, Acc& acc, LJInfo* info) {
  using std::exp;
  int ti = S.type[i], tj = S.type[e.j];
  const PairParams& pp = P.pair[ti][tj];
  acc.cnt[CNT_LJ] += 1;
  Inst tgt{e.j, {e.s[0], e.s[1], e.s[2]}};
  double rmaxmax = std::max(P.pair[0][0].rmax, std::max(P.pair[0][1].rmax, P.pair[1][1].rmax));
  CResult cr;
  cr.M = 0.0;
  cr.hops = 0;
  if (e.r <= 3.0 * rmaxmax) cr = cij_search(P, S, Lo, i, tgt);  // exact short-cut: no path beyond 3 r_max
  if (info) info->C = 1.0 - cr.M, info->bstar = 0, info->Q = 1, info->E = 0, info->bstar_evaluated = false;
  if (cr.M == 1.0) {  // C_ij == 0: skip (Alg. 3)
    acc.cnt[CNT_C0] += 1;
    return;
  }
  double srhi = pp.sigma * SR_FACTOR;
  double tP = (e.r - pp.sigma) / (srhi - pp.sigma);
  bool needP = tP < 1.0;  // S_r(r) != 0
  if (std::is_same<T, Var>::value) ad::tape().clear();
  Ctx<T> cx;
  cx.S = &S;
  int zero[3] = {0, 0, 0};
  int qi = cx.add(i, zero);
  int qj = cx.add(e.j, e.s);
  V3<T> d = cx.pos[qj] - cx.pos[qi];
  T r = norm(d);
  // C_ij along the maximising path
  T M(0.0);
  if (cr.hops == 1) {
    M = Sw(r, pp.rmin, pp.rmax);
  } else if (cr.hops == 2) {
    int qk = cx.add(cr.k.a, cr.k.s);
    const PairParams& p1 = P.pair[ti][S.type[cr.k.a]];
    const PairParams& p2 = P.pair[S.type[cr.k.a]][tj];
    M = Sw(norm(cx.pos[qk] - cx.pos[qi]), p1.rmin, p1.rmax) * Sw(norm(cx.pos[qj] - cx.pos[qk]), p2.rmin, p2.rmax);
  } else if (cr.hops == 3) {
    int qk = cx.add(cr.k.a, cr.k.s);
    int ql = cx.add(cr.l.a, cr.l.s);
    int tk = S.type[cr.k.a], tl = S.type[cr.l.a];
    const PairParams& p1 = P.pair[ti][tk];
    const PairParams& p2 = P.pair[tk][tl];
    const PairParams& p3 = P.pair[tl][tj];
    M = (Sw(norm(cx.pos[qk] - cx.pos[qi]), p1.rmin, p1.rmax) * Sw(norm(cx.pos[ql] - cx.pos[qk]), p2.rmin, p2.rmax)) *
        Sw(norm(cx.pos[qj] - cx.pos[ql]), p3.rmin, p3.rmax);
  }
  T C = 1.0 - M;
  // V_LJ(r) = 4 eps [(s/r)^12 - (s/r)^6] S(r; rlo, rc)   (reading A10); AIREBO-M:
  // the Morse form eps_m [e^{-2a(r-re)} - 2 e^{-a(r-re)}] under the same taper
  T V;
  if (P.potential == POT_AIREBO_M) {
    T x = exp(-pp.m_a * (r - pp.m_re));
    V = (pp.m_eps * (x * x - 2.0 * x)) * Sw(r, pp.rlo, pp.rc);
  } else {
    T sr = pp.sigma / r;
    T sr2 = sr * sr;
    T sr6 = (sr2 * sr2) * sr2;
    V = (4.0 * pp.eps * (sr6 * sr6 - sr6)) * Sw(r, pp.rlo, pp.rc);
  }
  T Q(1.0);
  if (needP) {
    acc.cnt[CNT_BSTAR] += 1;
    T Pr = Sw(r, pp.sigma, srhi);
    // b*: bond order with d_ij replaced by rho d_hat (reading A8)
    V3<T> dstar = (pp.rho / r) * d;
    Side<T> I, J;
    Inst inst_i{i, {0, 0, 0}};
    build_side(P, Lo, cx, i, zero, qi, tgt, I);
    build_side(P, Lo, cx, e.j, e.s, qj, inst_i, J);
    BondInfo bi;
    T bstar = bond_order(P, ti, tj, dstar, I, J, &bi);
    if (!bi.ok) acc.cnt[CNT_BADARG] += 1;
    double tb = (val(bstar) - pp.bmin) / (pp.bmax - pp.bmin);
    if (tb > 0.0 && tb < 1.0) acc.cnt[CNT_SBTRANS] += 1;
    T B = Sw(bstar, pp.bmin, pp.bmax);
    Q = (Pr * B + 1.0) - Pr;
    if (info) info->bstar = val(bstar), info->bstar_evaluated = true;
  }
  T E = (Q * C) * V;
  acc.E[2] += val(E);
  if (info) info->Q = val(Q), info->E = val(E), info->C = val(C);
  scatter(cx, E, acc);
}

// distinct instances reachable from i in 1..3 bonds, excluding i itself
inline long long reach_size(const Lists& Lo, int i) {
  std::vector<Inst> seen;
  Inst me{i, {0, 0, 0}};
  auto ins = [&](const Inst& x) {
    if (x == me) return;
    for (auto& y : seen)
      if (y == x) return;
    seen.push_back(x);
  };
  for (const Nb& e1 : Lo.shortl[i]) {
    Inst k{e1.j, {e1.s[0], e1.s[1], e1.s[2]}};
    ins(k);
    for (const Nb& e2 : Lo.shortl[e1.j]) {
      Inst l{e2.j, {k.s[0] + e2.s[0], k.s[1] + e2.s[1], k.s[2] + e2.s[2]}};
      ins(l);
      for (const Nb& e3 : Lo.shortl[e2.j]) ins(Inst{e3.j, {l.s[0] + e3.s[0], l.s[1] + e3.s[1], l.s[2] + e3.s[2]}});
    }
  }
  return (long long)seen.size();
}

struct Opts {
  bool brute = false;
  bool forces = true;
  bool rebo = true;  // REBO + torsion terms
  bool lj = true;    // LJ terms
  int nthreads = 1;
  const std::vector<char>* owners = nullptr;  // sampled mode: evaluate only terms owned by these atoms
  const std::vector<char>* fmask = nullptr;
};

inline void compute(const Params& P, const Sys& S, const Lists& Lo, const Opts& o, Acc& out) {
  int nt = 1;
#ifdef _OPENMP
  nt = std::max(1, o.nthreads);
#endif
  std::vector<Acc> part(nt);
  for (auto& a : part) {
    a.F.assign((size_t)S.n * 3, 0.0);
    a.fmask = o.fmask;
  }
#pragma omp parallel for schedule(static, 16) num_threads(nt)
  for (int i = 0; i < S.n; ++i) {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    Acc& acc = part[tid];
    if (o.owners && !(*o.owners)[i]) continue;
    acc.cnt[CNT_SHORT] += (long long)Lo.shortl[i].size();
    acc.cnt[CNT_MAXSHORT] = std::max(acc.cnt[CNT_MAXSHORT], (long long)Lo.shortl[i].size());
    if (P.potential != POT_REBO)  // the C_ij reach map belongs to the LJ term; REBO has none
      acc.cnt[CNT_MAXREACH] = std::max(acc.cnt[CNT_MAXREACH], reach_size(Lo, i));
    if (o.rebo)
      for (const Nb& e : Lo.shortl[i]) {
        if (!canonical(i, e.j, e.s)) continue;
        if (o.forces) eval_bond<Var>(P, S, Lo, i, e, acc, nullptr);
        else eval_bond<double>(P, S, Lo, i, e, acc, nullptr);
      }
    if (o.lj)
      for (const Nb& e : Lo.lj[i]) {
        if (o.forces) eval_lj<Var>(P, S, Lo, i, e, acc, nullptr);
        else eval_lj<double>(P, S, Lo, i, e, acc, nullptr);
      }
  }
  out.F.assign((size_t)S.n * 3, 0.0);
  for (int t = 0; t < nt; ++t) {  // fixed-order reduction
    for (size_t q = 0; q < out.F.size(); ++q) out.F[q] += part[t].F[q];
    for (int c = 0; c < 3; ++c) out.E[c] += part[t].E[c];
    for (int c = 0; c < 6; ++c) out.W[c] += part[t].W[c];
    for (int c = 0; c < NCNT; ++c) {
      if (c == CNT_MAXSHORT || c == CNT_MAXREACH) out.cnt[c] = std::max(out.cnt[c], part[t].cnt[c]);
      else out.cnt[c] += part[t].cnt[c];
    }
  }
}

}  // namespace orc

// ====================================================================== C API (ctypes)
using namespace orc;

static thread_local std::string g_err;

static bool load(const char* text, Params& P) {
  g_err = parse_params(text ? std::string(text) : std::string(), P);
  return g_err.empty();
}

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

int oracle_ncounters() { return NCNT; }

// Full evaluation.  F: n*3 (or NULL for energy only), E3: E_REBO, E_TORS, E_LJ, W6: xx yy zz xy xz yz,
// cnt: NCNT counters.  flags bit0 = brute-force lists, bit1 = skip LJ, bit2 = skip REBO+torsion.
int oracle_compute(const char* params, int n, const int* type, const double* x, const double* box, double* F,
                   double* E3, double* W6, long long* cnt, int nthreads, int flags) {
  Params P;
  if (!load(params, P)) return -2;
  Sys S{n, type, x, {box[0], box[1], box[2]}};
  Lists Lo;
  Opts o;
  o.brute = flags & 1;
  o.lj = !(flags & 2);
  o.rebo = !(flags & 4);
  o.forces = F != nullptr || W6 != nullptr;
  o.nthreads = nthreads;
  build_lists(P, S, o.brute, o.lj, Lo);
  Acc acc;
  compute(P, S, Lo, o, acc);
  if (F) std::memcpy(F, acc.F.data(), sizeof(double) * 3 * (size_t)n);
  if (E3) std::memcpy(E3, acc.E, sizeof(acc.E));
  if (W6) std::memcpy(W6, acc.W, sizeof(acc.W));
  if (cnt) std::memcpy(cnt, acc.cnt, sizeof(acc.cnt));
  return 0;
}

// Forces on a sample of atoms only: evaluates every term owned by an atom within rc_max (any
// image) of a sampled atom (all participants of a term lie within rc_max of its owner).
int oracle_forces_sampled(const char* params, int n, const int* type, const double* x, const double* box, int ns,
                          const int* sample, double* Fs, int nthreads) {
  Params P;
  if (!load(params, P)) return -2;
  Sys S{n, type, x, {box[0], box[1], box[2]}};
  Lists Lo;
  build_lists(P, S, false, true, Lo);
  double rcmax = 0;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) rcmax = std::max(rcmax, P.pair[a][b].rc);
  std::vector<char> owners(n, 0), fmask(n, 0);
  Finder f(S, rcmax, false);
  for (int q = 0; q < ns; ++q) {
    int a = sample[q];
    fmask[a] = 1;
    owners[a] = 1;
    f.around(a, [&](int j, const int*, const double*, double) { owners[j] = 1; });
  }
  Opts o;
  o.owners = &owners;
  o.fmask = &fmask;
  o.nthreads = nthreads;
  Acc acc;
  compute(P, S, Lo, o, acc);
  for (int q = 0; q < ns; ++q)
    for (int c = 0; c < 3; ++c) Fs[3 * q + c] = acc.F[3 * (size_t)sample[q] + c];
  return 0;
}

// Lists as sorted (i, j, sx, sy, sz) rows.  which: 0 = full short list, 1 = REBO half bonds,
// 2 = LJ half pairs with r <= rc.  rows == NULL: size query into *count.
int oracle_list(const char* params, int n, const int* type, const double* x, const double* box, int which,
                long long* count, long long* rows, int brute) {
  Params P;
  if (!load(params, P)) return -2;
  Sys S{n, type, x, {box[0], box[1], box[2]}};
  Lists Lo;
  build_lists(P, S, brute != 0, which == 2, Lo);
  long long c = 0;
  for (int i = 0; i < n; ++i) {
    const auto& v = which == 2 ? Lo.lj[i] : Lo.shortl[i];
    for (const Nb& e : v) {
      if (which == 1 && !canonical(i, e.j, e.s)) continue;
      if (rows) {
        long long* r = rows + 5 * c;
        r[0] = i, r[1] = e.j, r[2] = e.s[0], r[3] = e.s[1], r[4] = e.s[2];
      }
      ++c;
    }
  }
  *count = c;
  return 0;
}

// compute + the order-independent digests {count, sum h, xor h} of the three lists (rows as in
// oracle_list; h = mix(((u64)(u32)i << 32 | (u32)j) ^ mix((sx+128) << 16 | (sy+128) << 8 | (sz+128))),
// mix = splitmix64's finaliser) from ONE list build: the full-size parity tests compare lists of
// ~1e9 rows this way.  dig: 9 u64 (short, bonds, LJ).
static inline unsigned long long dmix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
int oracle_compute_digest(const char* params, int n, const int* type, const double* x, const double* box, double* F,
                          double* E3, double* W6, long long* cnt, int nthreads, unsigned long long* dig) {
  Params P;
  if (!load(params, P)) return -2;
  Sys S{n, type, x, {box[0], box[1], box[2]}};
  Lists Lo;
  Opts o;
  o.forces = F != nullptr || W6 != nullptr;
  o.nthreads = nthreads;
  build_lists(P, S, false, true, Lo);
  Acc acc;
  compute(P, S, Lo, o, acc);
  if (F) std::memcpy(F, acc.F.data(), sizeof(double) * 3 * (size_t)n);
  if (E3) std::memcpy(E3, acc.E, sizeof(acc.E));
  if (W6) std::memcpy(W6, acc.W, sizeof(acc.W));
  if (cnt) std::memcpy(cnt, acc.cnt, sizeof(acc.cnt));
  for (int which = 0; which < 3; ++which) {
    unsigned long long c = 0, sum = 0, xr = 0;
    for (int i = 0; i < n; ++i)
      for (const Nb& e : which == 2 ? Lo.lj[i] : Lo.shortl[i]) {
        if (which == 1 && !canonical(i, e.j, e.s)) continue;
        unsigned long long a = ((unsigned long long)(unsigned)i << 32) | (unsigned)e.j;
        unsigned long long b = ((unsigned long long)(e.s[0] + 128) << 16) | ((unsigned long long)(e.s[1] + 128) << 8) |
                               (unsigned long long)(e.s[2] + 128);
        unsigned long long h = dmix(a ^ dmix(b));
        ++c, sum += h, xr ^= h;
      }
    dig[3 * which] = c, dig[3 * which + 1] = sum, dig[3 * which + 2] = xr;
  }
  return 0;
}

// Stage outputs for stage-wise parity: per REBO half bond (canonical order of
// oracle_list(which=1)) the values b, p_ij, p_ji, pi^rc, pi^dh, N_ij, N_ji, N^conj (8 per bond);
// per LJ half pair (order of which=2): C_ij, b* (0 if not evaluated), Q, E (4 per pair).
int oracle_stages(const char* params, int n, const int* type, const double* x, const double* box, double* bond8,
                  double* lj4) {
  Params P;
  if (!load(params, P)) return -2;
  Sys S{n, type, x, {box[0], box[1], box[2]}};
  Lists Lo;
  build_lists(P, S, false, lj4 != nullptr, Lo);
  Acc acc;
  acc.F.assign((size_t)n * 3, 0.0);
  long long b = 0, q = 0;
  for (int i = 0; i < n; ++i) {
    if (bond8)
      for (const Nb& e : Lo.shortl[i]) {
        if (!canonical(i, e.j, e.s)) continue;
        BondInfo bi;
        eval_bond<double>(P, S, Lo, i, e, acc, &bi);
        double* o = bond8 + 8 * b++;
        o[0] = bi.b, o[1] = bi.pij, o[2] = bi.pji, o[3] = bi.pirc, o[4] = bi.pidh, o[5] = bi.Nij, o[6] = bi.Nji,
        o[7] = bi.Nconj;
      }
    if (lj4)
      for (const Nb& e : Lo.lj[i]) {
        LJInfo li;
        eval_lj<double>(P, S, Lo, i, e, acc, &li);
        double* o = lj4 + 4 * q++;
        o[0] = li.C, o[1] = li.bstar_evaluated ? li.bstar : 0.0, o[2] = li.Q, o[3] = li.E;
      }
  }
  return 0;
}

// Velocity-Verlet NVE, forces recomputed from scratch every step (no skin).
// thermo (if not NULL): rows (step, PE, KE, Etot) at steps 0, every, 2*every, ... <= nsteps.
int oracle_nve(const char* params, int n, const int* type, double* x, double* v, const double* box, int nsteps,
               double dt, int every, double* thermo, int nthreads) {
  Params P;
  if (!load(params, P)) return -2;
  Sys S{n, type, x, {box[0], box[1], box[2]}};
  Opts o;
  o.nthreads = nthreads;
  auto force = [&](std::vector<double>& F, double& pe) {
    Lists Lo;
    build_lists(P, S, false, true, Lo);
    Acc acc;
    compute(P, S, Lo, o, acc);
    F = acc.F;
    pe = acc.E[0] + acc.E[1] + acc.E[2];
  };
  auto ke = [&]() {
    double k = 0;
    for (int a = 0; a < n; ++a)
      for (int c = 0; c < 3; ++c) k += P.mass[type[a]] * v[3 * a + c] * v[3 * a + c];
    return 0.5 * k * P.mvv2e;
  };
  std::vector<double> F;
  double pe;
  force(F, pe);
  int row = 0;
  auto record = [&](int step) {
    if (!thermo) return;
    double k = ke();
    double* t = thermo + 4 * row++;
    t[0] = step, t[1] = pe, t[2] = k, t[3] = pe + k;
  };
  if (every > 0) record(0);
  for (int step = 1; step <= nsteps; ++step) {
    for (int a = 0; a < n; ++a) {
      double dtf = 0.5 * dt * P.ftm2v / P.mass[type[a]];
      for (int c = 0; c < 3; ++c) {
        v[3 * a + c] += dtf * F[3 * a + c];
        x[3 * a + c] += dt * v[3 * a + c];
        double L = box[c];
        double y = x[3 * a + c] - L * std::floor(x[3 * a + c] / L);  // wrap
        if (y >= L) y -= L;
        if (y < 0) y += L;
        x[3 * a + c] = y;
      }
    }
    force(F, pe);
    for (int a = 0; a < n; ++a) {
      double dtf = 0.5 * dt * P.ftm2v / P.mass[type[a]];
      for (int c = 0; c < 3; ++c) v[3 * a + c] += dtf * F[3 * a + c];
    }
    if (every > 0 && step % every == 0) record(step);
  }
  return 0;
}

// ---- unit-level entry points (pins): value and derivative(s) by AD
int oracle_switch(double x, double lo, double hi, double* out2) {
  ad::tape().clear();
  Var v = ad::leaf(x);
  Var s = Sw(v, lo, hi);
  std::vector<double> adj;
  ad::backward(s.id, adj);
  out2[0] = s.v;
  out2[1] = s.id >= 0 ? adj[v.id] : 0.0;
  return 0;
}

// which: 0 = g_C/g_H (a = species, x), 1 = P (a = t_j, x=N^C, y=N^H), 2 = R (a = pair index,
// x, y, z), 3 = T (same).  out: value then gradient components.
int oracle_spline(const char* params, int which, int a, double x, double y, double z, double* out) {
  Params P;
  if (!load(params, P)) return -2;
  ad::tape().clear();
  Var vx = ad::leaf(x), vy = ad::leaf(y), vz = ad::leaf(z);
  Var f;
  if (which == 0) f = hermite1(P.g[a], vx);
  else if (which == 1) f = spline2(P.P[a], P.Plo, P.Pn, vx, vy);
  else f = spline3(which == 2 ? P.R[a] : P.T[a], P.RTlo, P.RTn, vx, vy, vz);
  std::vector<double> adj;
  ad::backward(f.id, adj);
  out[0] = f.v;
  out[1] = f.id >= 0 ? adj[vx.id] : 0.0;
  out[2] = f.id >= 0 ? adj[vy.id] : 0.0;
  out[3] = f.id >= 0 ? adj[vz.id] : 0.0;
  return 0;
}

int oracle_parse(const char* params) {
  Params P;
  return load(params, P) ? 0 : -2;
}

}  // extern "C"
