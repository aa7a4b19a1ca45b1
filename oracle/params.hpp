// oracle/params.hpp -- the oracle's own parser for params/toy_ch.param.
//
// TEST INFRASTRUCTURE ONLY (see oracle/ad.hpp header).  Written independently of the C-ABI
// library's parser (paper_1810_07026_b200/csrc/params.cpp); the two share no code.
// Grammar (params/make_toy_ch.py docstring): '#' comments; a line whose first token is not a
// number starts `key v1 v2 ...`; a line whose first token is a number continues the last key.
// Errors name the line or the key.
#pragma once
#include <cstdlib>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace orc {

struct Spline1 {  // 1-D cubic Hermite on non-uniform knots
  std::vector<double> x, y;
};

struct PairParams {
  // REBO pair terms: f_R = w (1+Q/r) A e^{-alpha r}; f_A = -w sum B_n e^{-beta_n r}
  double rmin, rmax, Q, alpha, A, B[3], beta[3];
  // LJ
  double eps, sigma, rc, rlo, bmin, bmax, rho;
  // Morse radial form of AIREBO-M: eps_m [e^{-2a(r-re)} - 2 e^{-a(r-re)}]
  double m_eps = 0, m_a = 0, m_re = 0;
};

// the method applies to AIREBO, to REBO (no inter-molecular forces) and to AIREBO-M
enum Potential { POT_AIREBO = 0, POT_REBO = 1, POT_AIREBO_M = 2 };

struct Params {
  Potential potential = POT_AIREBO;
  double mass[2], kB, mvv2e, ftm2v, skin;
  PairParams pair[2][2];  // symmetric [t_i][t_j]
  Spline1 g[2];           // g_C, g_H (centre species)
  double lam[2][2][2];    // lambda_{j i k} indexed [t_j][t_i][t_k] (constant part)
  // SURVEY §8(f) F3 (readings A33 / A34 of DESIGN.md), both optional and off by default:
  //   lambda_jik = lam[t_j][t_i][t_k] + kappa delta(t_i, H) [(rho_{t_k H} - r_ik) - (rho_{t_j H} - r_ij)]
  //   g_C(cos, N) = g_C2(cos) + S(N; nlo, nhi) (g_C(cos) - g_C2(cos)), N = N_i - w_ij
  double kappa = 0.0;     // lambda.kappa (1/A)
  bool has_gC2 = false;   // angle.C2.knots / values present
  Spline1 gC2;
  double gC_nlo = 3.2, gC_nhi = 3.7;  // angle.C.nlo / nhi
  double Plo[2];
  int Pn[2];
  std::vector<double> P[2];  // P_CC, P_CH (C-centred), index a*Pn[1]+b
  double RTlo[3];
  int RTn[3];
  std::vector<double> R[3], T[3];  // CC, CH, HH; index (x*n1+y)*n2+z
  double conj_lo, conj_hi, s2lo, s2hi;
  double tors[2][2][2][2];  // [t_k][t_i][t_j][t_l]
};

inline bool is_number(const std::string& s) {
  char* end = nullptr;
  std::strtod(s.c_str(), &end);
  return end && *end == '\0' && !s.empty();
}

// returns empty string on success, else an error message
inline std::string parse_params(const std::string& text, Params& p) {
  std::map<std::string, std::vector<std::string>> kv;
  std::istringstream in(text);
  std::string line, last;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    auto h = line.find('#');
    if (h != std::string::npos) line = line.substr(0, h);
    std::istringstream ls(line);
    std::vector<std::string> tok;
    std::string t;
    while (ls >> t) tok.push_back(t);
    if (tok.empty()) continue;
    if (is_number(tok[0])) {
      if (last.empty()) return "param line " + std::to_string(lineno) + ": value without a key";
      for (auto& x : tok) kv[last].push_back(x);
      continue;
    }
    last = tok[0];
    if (kv.count(last)) return "param line " + std::to_string(lineno) + ": duplicate key " + last;
    kv[last] = std::vector<std::string>(tok.begin() + 1, tok.end());
  }
  std::string err;
  auto nums = [&](const std::string& key, size_t n) -> std::vector<double> {
    std::vector<double> out;
    if (!err.empty()) return std::vector<double>(n == 0 ? 1 : n, 0.0);
    auto it = kv.find(key);
    if (it == kv.end()) {
      err = "missing key " + key;
      return std::vector<double>(n == 0 ? 1 : n, 0.0);
    }
    for (auto& s : it->second) {
      if (!is_number(s)) {
        err = "key " + key + ": not a number: " + s;
        return std::vector<double>(n == 0 ? 1 : n, 0.0);
      }
      out.push_back(std::strtod(s.c_str(), nullptr));
    }
    if (n && out.size() != n) {
      err = "key " + key + ": expected " + std::to_string(n) + " values, got " + std::to_string(out.size());
      return std::vector<double>(n, 0.0);
    }
    return out;
  };
  auto one = [&](const std::string& key) { return nums(key, 1)[0]; };
  const char* S = "CH";
  const char* PK[3] = {"CC", "CH", "HH"};
  p.mass[0] = one("mass.C");
  p.mass[1] = one("mass.H");
  p.kB = one("const.kB");
  p.mvv2e = one("const.mvv2e");
  p.ftm2v = one("const.ftm2v");
  p.skin = one("neigh.skin");
  if (kv.count("potential")) {
    const auto& v = kv["potential"];
    std::string name = v.size() == 1 ? v[0] : std::string("?");
    if (name == "airebo") p.potential = POT_AIREBO;
    else if (name == "rebo") p.potential = POT_REBO;
    else if (name == "airebo-m") p.potential = POT_AIREBO_M;
    else if (err.empty()) err = "key potential: expected airebo, rebo or airebo-m";
  }
  for (int q = 0; q < 3; ++q) {
    PairParams pp;
    std::string b = std::string("pair.") + PK[q] + ".";
    pp.rmin = one(b + "rmin");
    pp.rmax = one(b + "rmax");
    pp.Q = one(b + "Q");
    pp.alpha = one(b + "alpha");
    pp.A = one(b + "A");
    auto B = nums(b + "B", 3), be = nums(b + "beta", 3);
    for (int n = 0; n < 3; ++n) pp.B[n] = B[n], pp.beta[n] = be[n];
    std::string l = std::string("lj.") + PK[q] + ".";
    pp.eps = one(l + "eps");
    pp.sigma = one(l + "sigma");
    pp.rc = one(l + "rc");
    pp.rlo = one(l + "rlo");
    pp.bmin = one(l + "bmin");
    pp.bmax = one(l + "bmax");
    pp.rho = one(l + "rho");
    if (p.potential == POT_AIREBO_M) {
      std::string m = std::string("morse.") + PK[q] + ".";
      pp.m_eps = one(m + "eps");
      pp.m_a = one(m + "alpha");
      pp.m_re = one(m + "re");
    }
    if (err.empty()) {
      if (!(pp.rmin < pp.rmax)) err = b + "rmin >= " + b + "rmax";
      else if (!(pp.rlo < pp.rc)) err = l + "rlo >= " + l + "rc";
      else if (!(pp.bmin < pp.bmax)) err = l + "bmin >= " + l + "bmax";
      else if (!(pp.rmin > 0 && pp.sigma > 0)) err = b + "cutoffs must be > 0";
    }
    int ti = (q == 2) ? 1 : 0, tj = (q == 0) ? 0 : 1;
    p.pair[ti][tj] = pp;
    p.pair[tj][ti] = pp;
  }
  for (int c = 0; c < 2; ++c) {
    std::string b = std::string("angle.") + S[c] + ".";
    p.g[c].x = nums(b + "knots", 0);
    p.g[c].y = nums(b + "values", 0);
    if (err.empty() && (p.g[c].x.size() != p.g[c].y.size() || p.g[c].x.size() < 2))
      err = b + "knots/values length mismatch";
  }
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i)
      for (int k = 0; k < 2; ++k) p.lam[j][i][k] = one(std::string("lambda.") + S[j] + S[i] + S[k]);
  if (kv.count("lambda.kappa")) p.kappa = one("lambda.kappa");
  if (kv.count("angle.C2.knots") || kv.count("angle.C2.values")) {
    p.has_gC2 = true;
    p.gC2.x = nums("angle.C2.knots", 0);
    p.gC2.y = nums("angle.C2.values", 0);
    if (err.empty() && (p.gC2.x.size() != p.gC2.y.size() || p.gC2.x.size() < 2))
      err = "angle.C2.knots/values length mismatch";
  }
  if (kv.count("angle.C.nlo")) p.gC_nlo = one("angle.C.nlo");
  if (kv.count("angle.C.nhi")) p.gC_nhi = one("angle.C.nhi");
  if (err.empty() && !(p.gC_nlo < p.gC_nhi)) err = "angle.C.nlo >= angle.C.nhi";
  auto plo = nums("grid.P.lo", 2), pn = nums("grid.P.n", 2);
  auto rlo = nums("grid.RT.lo", 3), rn = nums("grid.RT.n", 3);
  for (int a = 0; a < 2; ++a) p.Plo[a] = plo[a], p.Pn[a] = (int)pn[a];
  for (int a = 0; a < 3; ++a) p.RTlo[a] = rlo[a], p.RTn[a] = (int)rn[a];
  size_t np = (size_t)p.Pn[0] * p.Pn[1], nr = (size_t)p.RTn[0] * p.RTn[1] * p.RTn[2];
  p.P[0] = nums("P.CC", np);
  p.P[1] = nums("P.CH", np);
  for (int q = 0; q < 3; ++q) {
    p.R[q] = nums(std::string("R.") + PK[q], nr);
    p.T[q] = nums(std::string("T.") + PK[q], nr);
  }
  p.conj_lo = one("conj.lo");
  p.conj_hi = one("conj.hi");
  p.s2lo = one("dihedral.sin2_lo");
  p.s2hi = one("dihedral.sin2_hi");
  for (int k = 0; k < 2; ++k)
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int l = 0; l < 2; ++l) p.tors[k][i][j][l] = one(std::string("tors.") + S[k] + S[i] + S[j] + S[l]);
  if (err.empty() && !(p.conj_lo < p.conj_hi)) err = "conj.lo >= conj.hi";
  if (err.empty() && !(p.s2lo < p.s2hi)) err = "dihedral.sin2_lo >= dihedral.sin2_hi";
  return err;
}

}  // namespace orc
