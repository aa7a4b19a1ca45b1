// params.cpp -- tokenizer + validator for the engine's parameter text.
// Grammar (params/make_toy_ch.py): '#' comment to end of line; a record starts at a line whose
// first word is not numeric (`key v1 v2 ...`); numeric-led lines append to the open record.
// Errors name the line (syntax) or the key (missing / count / invariant).
#include "params.h"

#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <unordered_map>

namespace ab {

namespace {

struct Record {
  int line;
  std::vector<std::string> words;
};

bool numeric(const std::string& w, double* out) {
  if (w.empty()) return false;
  const char* b = w.c_str();
  char* e = nullptr;
  errno = 0;
  double v = std::strtod(b, &e);
  if (e != b + w.size() || errno == ERANGE) return false;
  if (out) *out = v;
  return true;
}

std::vector<std::string> split_words(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\r')) ++i;
    size_t j = i;
    while (j < s.size() && !(s[j] == ' ' || s[j] == '\t' || s[j] == '\r')) ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

class Table {
 public:
  std::string error;
  std::unordered_map<std::string, Record> recs;

  bool scan(const char* text, size_t len) {
    std::string open_key;
    size_t pos = 0;
    int line = 0;
    while (pos <= len) {
      size_t nl = pos;
      while (nl < len && text[nl] != '\n') ++nl;
      ++line;
      std::string body(text + pos, nl - pos);
      size_t hash = body.find('#');
      if (hash != std::string::npos) body.resize(hash);
      std::vector<std::string> w = split_words(body);
      if (!w.empty()) {
        if (numeric(w[0], nullptr)) {
          if (open_key.empty()) {
            error = "param line " + std::to_string(line) + ": numbers before any key";
            return false;
          }
          auto& r = recs[open_key].words;
          r.insert(r.end(), w.begin(), w.end());
        } else {
          open_key = w[0];
          if (recs.count(open_key)) {
            error = "param line " + std::to_string(line) + ": key " + open_key + " given twice";
            return false;
          }
          recs[open_key] = Record{line, std::vector<std::string>(w.begin() + 1, w.end())};
        }
      }
      pos = nl + 1;
    }
    return true;
  }

  // values of `key`; n == 0 accepts any count >= 1
  std::vector<double> vals(const std::string& key, size_t n) {
    std::vector<double> v;
    if (!error.empty()) return std::vector<double>(n ? n : 1, 0.0);
    auto it = recs.find(key);
    if (it == recs.end()) {
      error = "parameter key " + key + " is missing";
      return std::vector<double>(n ? n : 1, 0.0);
    }
    for (const auto& w : it->second.words) {
      double x;
      if (!numeric(w, &x)) {
        error = "param line " + std::to_string(it->second.line) + ": key " + key + " has non-numeric value " + w;
        return std::vector<double>(n ? n : 1, 0.0);
      }
      v.push_back(x);
    }
    if ((n && v.size() != n) || v.empty()) {
      error = "parameter key " + key + " needs " + (n ? std::to_string(n) : std::string(">= 1")) + " values, has " +
              std::to_string(v.size());
      return std::vector<double>(n ? n : 1, 0.0);
    }
    return v;
  }
  double val(const std::string& key) { return vals(key, 1)[0]; }
};

}  // namespace

std::string parse_host_params(const char* text, size_t len, HostParams& hp) {
  Table t;
  if (!t.scan(text, len)) return t.error;
  static const char* SP = "CH";
  static const char* PN[3] = {"CC", "CH", "HH"};
  hp.mass[kC] = t.val("mass.C");
  hp.mass[kH] = t.val("mass.H");
  hp.kB = t.val("const.kB");
  hp.mvv2e = t.val("const.mvv2e");
  hp.ftm2v = t.val("const.ftm2v");
  hp.skin = t.val("neigh.skin");
  hp.potential = kAIREBO;  // `potential` is optional (default AIREBO)
  auto pot = t.recs.find("potential");
  if (t.error.empty() && pot != t.recs.end()) {
    const auto& w = pot->second.words;
    if (w.size() == 1 && w[0] == "airebo") hp.potential = kAIREBO;
    else if (w.size() == 1 && w[0] == "rebo") hp.potential = kREBO;
    else if (w.size() == 1 && w[0] == "airebo-m") hp.potential = kAIREBOM;
    else t.error = "param line " + std::to_string(pot->second.line) + ": potential must be airebo, rebo or airebo-m";
  }
  for (int p = 0; p < 3; ++p) {
    PairSet& s = hp.pr[p];
    const std::string a = std::string("pair.") + PN[p] + ".", l = std::string("lj.") + PN[p] + ".";
    s.rmin = t.val(a + "rmin");
    s.rmax = t.val(a + "rmax");
    s.Q = t.val(a + "Q");
    s.alpha = t.val(a + "alpha");
    s.A = t.val(a + "A");
    std::vector<double> B = t.vals(a + "B", 3), be = t.vals(a + "beta", 3);
    for (int q = 0; q < 3; ++q) {
      s.B[q] = B[q];
      s.beta[q] = be[q];
    }
    s.eps = t.val(l + "eps");
    s.sigma = t.val(l + "sigma");
    s.rc = t.val(l + "rc");
    s.rlo = t.val(l + "rlo");
    s.bmin = t.val(l + "bmin");
    s.bmax = t.val(l + "bmax");
    s.rho = t.val(l + "rho");
    if (hp.potential == kAIREBOM) {  // the Morse block is read (and required) for AIREBO-M only
      const std::string m = std::string("morse.") + PN[p] + ".";
      s.meps = t.val(m + "eps");
      s.malpha = t.val(m + "alpha");
      s.mre = t.val(m + "re");
      if (t.error.empty() && !(s.malpha > 0.0 && s.mre > 0.0 && s.meps >= 0.0))
        t.error = m + "alpha and " + m + "re must be > 0, " + m + "eps >= 0";
    }
    if (t.error.empty()) {
      if (!(s.rmin > 0.0)) t.error = a + "rmin must be > 0";
      else if (!(s.rmin < s.rmax)) t.error = a + "rmin >= " + a + "rmax (invariant r_min < r_max)";
      else if (!(s.rlo < s.rc)) t.error = l + "rlo >= " + l + "rc (invariant r_LJmin < r_LJmax)";
      else if (!(s.bmin < s.bmax)) t.error = l + "bmin >= " + l + "bmax (invariant b_min < b_max)";
      else if (!(s.sigma > 0.0 && s.rc > 0.0)) t.error = l + "sigma and rc must be > 0";
    }
  }
  for (int c = 0; c < 2; ++c) {
    const std::string a = std::string("angle.") + SP[c] + ".";
    hp.gknot[c] = t.vals(a + "knots", 0);
    hp.gval[c] = t.vals(a + "values", 0);
    if (t.error.empty()) {
      if (hp.gknot[c].size() != hp.gval[c].size() || hp.gknot[c].size() < 2 || hp.gknot[c].size() > 16)
        t.error = a + "knots and " + a + "values must have equal length in [2, 16]";
      for (size_t q = 1; t.error.empty() && q < hp.gknot[c].size(); ++q)
        if (!(hp.gknot[c][q] > hp.gknot[c][q - 1])) t.error = a + "knots must increase";
    }
  }
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i)
      for (int k = 0; k < 2; ++k) hp.lam[j][i][k] = t.val(std::string("lambda.") + SP[j] + SP[i] + SP[k]);
  // optional F3 keys: distance-dependent lambda, coordination-dependent g_C
  if (t.recs.count("lambda.kappa")) hp.kappa = t.val("lambda.kappa");
  if (t.recs.count("angle.C2.knots") || t.recs.count("angle.C2.values")) {
    hp.gknot2 = t.vals("angle.C2.knots", 0);
    hp.gval2 = t.vals("angle.C2.values", 0);
    if (t.error.empty()) {
      if (hp.gknot2.size() != hp.gval2.size() || hp.gknot2.size() < 2 || hp.gknot2.size() > 16)
        t.error = "angle.C2.knots and angle.C2.values must have equal length in [2, 16]";
      for (size_t q = 1; t.error.empty() && q < hp.gknot2.size(); ++q)
        if (!(hp.gknot2[q] > hp.gknot2[q - 1])) t.error = "angle.C2.knots must increase";
    }
  }
  if (t.recs.count("angle.C.nlo")) hp.gnlo = t.val("angle.C.nlo");
  if (t.recs.count("angle.C.nhi")) hp.gnhi = t.val("angle.C.nhi");
  if (t.error.empty() && !(hp.gnlo < hp.gnhi)) t.error = "angle.C.nlo >= angle.C.nhi";
  std::vector<double> plo = t.vals("grid.P.lo", 2), pn = t.vals("grid.P.n", 2);
  std::vector<double> rlo = t.vals("grid.RT.lo", 3), rn = t.vals("grid.RT.n", 3);
  for (int q = 0; q < 2; ++q) {
    hp.grid_p_lo[q] = plo[q];
    hp.grid_p_n[q] = (int)pn[q];
  }
  for (int q = 0; q < 3; ++q) {
    hp.grid_rt_lo[q] = rlo[q];
    hp.grid_rt_n[q] = (int)rn[q];
  }
  if (t.error.empty()) {
    if (hp.grid_p_n[0] != 5 || hp.grid_p_n[1] != 5) t.error = "grid.P.n must be 5 5 (engine table layout)";
    if (hp.grid_rt_n[0] != 5 || hp.grid_rt_n[1] != 5 || hp.grid_rt_n[2] != 9)
      t.error = "grid.RT.n must be 5 5 9 (engine table layout)";
  }
  hp.Ptab[0] = t.vals("P.CC", 25);
  hp.Ptab[1] = t.vals("P.CH", 25);
  for (int p = 0; p < 3; ++p) {
    hp.Rtab[p] = t.vals(std::string("R.") + PN[p], 225);
    hp.Ttab[p] = t.vals(std::string("T.") + PN[p], 225);
  }
  hp.conj_lo = t.val("conj.lo");
  hp.conj_hi = t.val("conj.hi");
  hp.sin2_lo = t.val("dihedral.sin2_lo");
  hp.sin2_hi = t.val("dihedral.sin2_hi");
  for (int k = 0; k < 2; ++k)
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int l = 0; l < 2; ++l)
          hp.tors[k][i][j][l] = t.val(std::string("tors.") + SP[k] + SP[i] + SP[j] + SP[l]);
  if (t.error.empty() && !(hp.conj_lo < hp.conj_hi)) t.error = "conj.lo >= conj.hi";
  if (t.error.empty() && !(hp.sin2_lo < hp.sin2_hi)) t.error = "dihedral.sin2_lo >= dihedral.sin2_hi";
  if (t.error.empty() && !(hp.mass[0] > 0 && hp.mass[1] > 0)) t.error = "mass.C and mass.H must be > 0";
  if (t.error.empty() && !(hp.skin >= 0)) t.error = "neigh.skin must be >= 0";
  return t.error;
}

}  // namespace ab
