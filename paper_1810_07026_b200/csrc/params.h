// params.h -- host-side parameter set of the engine (parsed from params/toy_ch.param text).
// Independent of oracle/params.hpp (no shared code).  Functional forms: SURVEY A2.
#pragma once
#include <string>
#include <vector>

namespace ab {

enum { kC = 0, kH = 1 };
inline int pair_index(int ta, int tb) { return ta + tb; }  // CC 0, CH 1, HH 2

struct PairSet {
  double rmin, rmax, Q, alpha, A, B[3], beta[3];      // REBO f_R / f_A
  double eps, sigma, rc, rlo, bmin, bmax, rho;        // LJ, S_r, S_b, fictitious distance
  double meps = 0, malpha = 0, mre = 0;               // Morse radial form of AIREBO-M
};

// potential variants of the paper's section 2.1: AIREBO, REBO (no inter-molecular
// LJ term, no torsion), AIREBO-M (LJ radial form replaced by Morse, every gate kept)
enum { kAIREBO = 0, kREBO = 1, kAIREBOM = 2 };

struct HostParams {
  int potential = kAIREBO;
  double mass[2] = {0, 0}, kB = 0, mvv2e = 0, ftm2v = 0, skin = 0;
  PairSet pr[3];
  std::vector<double> gknot[2], gval[2];  // g_C, g_H knots (cos theta) and values
  double lam[2][2][2];                    // lambda_{jik} as [t_j][t_i][t_k] (constant part)
  // SURVEY §8(f) F3, optional (readings A33 / A34 of DESIGN.md):
  //   lambda_jik += kappa delta(t_i, H) [(rho_{t_k H} - r_ik) - (rho_{t_j H} - r_ij)]
  //   g_C(cos, N) = g_C2(cos) + S(N; nlo, nhi) (g_C(cos) - g_C2(cos)), N = N_i - w_ij
  double kappa = 0.0;
  std::vector<double> gknot2, gval2;      // angle.C2 (empty: g_C independent of N)
  double gnlo = 3.2, gnhi = 3.7;
  double grid_p_lo[2];
  int grid_p_n[2];
  double grid_rt_lo[3];
  int grid_rt_n[3];
  std::vector<double> Ptab[2];            // P_CC, P_CH
  std::vector<double> Rtab[3], Ttab[3];   // CC CH HH
  double conj_lo = 0, conj_hi = 0, sin2_lo = 0, sin2_hi = 0;
  double tors[2][2][2][2];                // eps_tors[t_k][t_i][t_j][t_l]
};

// Parses `text` (len bytes).  Returns "" on success or an error that names the line or key.
std::string parse_host_params(const char* text, size_t len, HostParams& hp);

}  // namespace ab
