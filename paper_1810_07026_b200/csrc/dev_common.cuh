// dev_common.cuh -- device-side constants, scalar building blocks and reduction helpers.
//
// Scalar forms:
//   switch S(x; lo, hi): t = (x-lo)/(hi-lo); 1 (t<=0), 0 (t>=1), (1+cos(pi t))/2 inside
//   g_i(cos): cubic Hermite on non-uniform knots, central-difference knot slopes, zero end slopes
//   P / pi^rc / T: tensor products of the same Hermite scheme on integer knot grids
// Precision: R = double (AB_FP64) or float (AB_MIXED); positions, displacements, r^2 list
// decisions and all accumulators are always double.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace ab {

constexpr int NBMAX = 16;         // short-list entries per atom the bond-order kernels accept
constexpr int REACH_SLOTS = 256;  // per-warp open-addressing table of the C_ij reach set
constexpr int REACH_EMPTY = -1;

template <typename R>
struct Tab {
  R rmin[3], rmax[3], Q[3], alpha[3], A[3], B[3][3], beta[3][3];
  R eps[3], sigma[3], sigma2[3], rc[3], rlo[3], bmin[3], bmax[3], rho[3], srhi[3];
  R inv_taper[3];  // 1 / (r_c - r_lo)
  R lj_e4[3], lj_c12[3], lj_c6[3];  // 4 eps, 12 * 4 eps, 6 * 4 eps (far-pair 12-6 form)
  R meps[3], malpha[3], mre[3];  // AIREBO-M Morse radial form
  R explam[2][2][2];  // e^{lambda_{jik}} [t_j][t_i][t_k]
  int gn[3];  // g_C, g_H, g_C2 (slot 2: F3 coordination-dependent g_C, reading A34)
  R gx[3][16], gy[3][16], gm[3][16];
  // F3 (readings A33 / A34): kappa != 0 -> lambda_jik depends on r_ij, r_ik for
  // H centres; g2on -> g_C(cos, N) = g_C2 + S(N; gnlo, gnhi) (g_C - g_C2)
  R kappa, rhoH[2];  // rho_{C H}, rho_{H H}
  int g2on;
  R gnlo, gnhi;
  // rigorous bounds of pi^rc and T over their whole tables (tensor-product Hermite overshoot
  // included): the b* plateau test of the deferred batch (k_bond.cuh bstar_plateau)
  R bRlo[3], bRhi[3], bTlo[3], bThi[3];
  R P[2][25], Rt[3][225], Tt[3][225];
  R conj_lo, conj_hi, s2lo, s2hi;
  R tors[2][2][2][2];
  // global-memory copies of the spline tables, read through L1 (__ldg): the knot indices differ
  // between the lanes of a warp when coordination numbers are fractional, and an indexed
  // __constant__ load serialises per distinct address (set by the engine)
  const R* gRT;  // [2][3][225]: pi^rc (which 0) and T (which 1) per species pair
  const R* gP;   // [2][25]
  const R* gG;   // [3][3][16]: g knots, values, knot slopes per spline (g_C, g_H, g_C2)
};

struct Geo {  // double-only quantities: exact list / gate decisions, box, integrator
  double rmax2[3], rc2[3], rmax_s2[3], rc_s2[3], rlo2[3], reach2;
  double srhi2_hi[3];  // (2^(1/6) sigma)^2 (1 + 1e-9): pre-filter of the exact S_r window test
  double tv2[3];       // r_lo^2 (1 - 1e-9): taper vote threshold of the far-pair kernel
  double L[3];
  double mass[2], ftm2v, mvv2e;
  int potential;  // 0 AIREBO, 1 REBO, 2 AIREBO-M
};

__constant__ Tab<double> c_tabd;
__constant__ Tab<float> c_tabf;
__constant__ Geo c_geo;

template <typename R>
__device__ __forceinline__ const Tab<R>& tab();
template <>
__device__ __forceinline__ const Tab<double>& tab<double>() {
  return c_tabd;
}
template <>
__device__ __forceinline__ const Tab<float>& tab<float>() {
  return c_tabf;
}

// ------------------------------------------------------------------ vectors
template <typename R>
struct V3 {
  R x, y, z;
};
template <typename R>
__device__ __forceinline__ V3<R> mk3(R a, R b, R c) {
  V3<R> v;
  v.x = a, v.y = b, v.z = c;
  return v;
}
template <typename R>
__device__ __forceinline__ V3<R> operator+(V3<R> a, V3<R> b) {
  return mk3(a.x + b.x, a.y + b.y, a.z + b.z);
}
template <typename R>
__device__ __forceinline__ V3<R> operator-(V3<R> a, V3<R> b) {
  return mk3(a.x - b.x, a.y - b.y, a.z - b.z);
}
template <typename R>
__device__ __forceinline__ V3<R> operator*(R s, V3<R> a) {
  return mk3(s * a.x, s * a.y, s * a.z);
}
template <typename R>
__device__ __forceinline__ R dot3(V3<R> a, V3<R> b) {
  return a.x * b.x + a.y * b.y + a.z * b.z;
}
template <typename R>
__device__ __forceinline__ V3<R> cross3(V3<R> a, V3<R> b) {
  return mk3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
template <typename R>
__device__ __forceinline__ void addto(V3<R>& a, V3<R> b) {
  a.x += b.x, a.y += b.y, a.z += b.z;
}

__device__ __forceinline__ double rsq(double x) { return rsqrt(x); }
__device__ __forceinline__ float rsq(float x) { return rsqrtf(x); }
__device__ __forceinline__ double sqr_t(double x) { return sqrt(x); }
__device__ __forceinline__ float sqr_t(float x) { return sqrtf(x); }
__device__ __forceinline__ double ex(double x) { return exp(x); }
__device__ __forceinline__ float ex(float x) { return expf(x); }
__device__ __forceinline__ void scpi(double t, double* s, double* c) { sincospi(t, s, c); }
__device__ __forceinline__ void scpi(float t, float* s, float* c) { sincospif(t, s, c); }

// exact (no-FMA) displacement and squared length: the list / gate decisions must reproduce the
// oracle's IEEE operations bit for bit
__device__ __forceinline__ double r2_exact(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// ------------------------------------------------------------------ switch
template <typename R>
__device__ __forceinline__ R sw(R x, R lo, R hi, R& dv) {
  R t = (x - lo) / (hi - lo);
  if (t <= R(0)) {
    dv = R(0);
    return R(1);
  }
  if (t >= R(1)) {
    dv = R(0);
    return R(0);
  }
  R s, c;
  scpi(t, &s, &c);
  dv = R(-0.5) * R(CUDART_PI) * s / (hi - lo);
  return R(0.5) * (R(1) + c);
}

// 1/sqrt(a) without the slow-path call of the IEEE routines: hardware approximation + two
// Newton steps (fp64: ~1 ulp; fp32: MUFU rsqrt).  a > 0 and finite.
__device__ __forceinline__ double rsqrt_fast(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double ha = 0.5 * a;
  y = y * fma(-ha * y, y, 1.5);
  y = y * fma(-ha * y, y, 1.5);
  return y;
}
__device__ __forceinline__ float rsqrt_fast(float a) { return rsqrtf(a); }

__device__ __forceinline__ double fma_r(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float fma_r(float a, float b, float c) { return fmaf(a, b, c); }

// 1/a: hardware approximation + two Newton steps (y += y (1 - a y)), a > 0 and finite
__device__ __forceinline__ double rcp_fast(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double e = fma(-a, y, 1.0);
  y = fma(y, e, y);
  e = fma(-a, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ float rcp_fast(float a) { return __frcp_rn(a); }
// one-Newton-step variants (relative error ~1e-14 from the ~2^-23 hardware seeds): the far-LJ
// pair arithmetic, whose per-pair terms are far below the 1e-9 eV/A force gate
__device__ __forceinline__ double rcp_nr1(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  return fma(y, fma(-a, y, 1.0), y);
}
__device__ __forceinline__ float rcp_nr1(float a) { return __frcp_rn(a); }
__device__ __forceinline__ double rsqrt_nr1(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  return y * fma(-0.5 * a * y, y, 1.5);
}
__device__ __forceinline__ float rsqrt_nr1(float a) { return rsqrtf(a); }

// Branch-free half-cosine on t in [0, 1] (caller clamps): S = (1 + cos(pi t))/2 and dS/dt, from
// x = pi (t - 1/2) in [-pi/2, pi/2]: cos(pi t) = -sin x, sin(pi t) = cos x, Taylor polynomials
// truncated below the working precision (fp64: x^21 / x^20 terms, error < 3e-17; fp32: x^13 / x^12).
// (coefficients in the constant bank: DFMA takes them as c[][] operands instead of a uniform-
// register pair per literal)
__constant__ double c_hc_s[10] = {-1.9572941063391263e-20, 8.2206352466243295e-18, -2.8114572543455206e-15,
                                  7.6471637318198164e-13, -1.6059043836821613e-10, 2.5052108385441720e-08,
                                  -2.7557319223985893e-06, 1.9841269841269841e-04, -8.3333333333333333e-03,
                                  1.6666666666666667e-01};  // -1/21!, 1/19!, ..., -1/5!, -(-1/3!)
__constant__ double c_hc_c[10] = {4.1103176233121648e-19, -1.5619206968586225e-16, 4.7794773323873853e-14,
                                  -1.1470745597729725e-11, 2.0876756987868099e-09, -2.7557319223985891e-07,
                                  2.4801587301587302e-05, -1.3888888888888889e-03, 4.1666666666666667e-02,
                                  -0.5};  // 1/20!, -1/18!, ..., 1/4!, -1/2!
__device__ __forceinline__ void halfcos_poly(double t, double& S, double& dSdt) {
  double x = (t - 0.5) * CUDART_PI;
  double x2 = x * x;
  double s = c_hc_s[0];
#pragma unroll
  for (int k = 1; k < 10; ++k) s = fma(s, x2, c_hc_s[k]);
  s = x - x * x2 * s;  // sin x
  double c = c_hc_c[0];
#pragma unroll
  for (int k = 1; k < 10; ++k) c = fma(c, x2, c_hc_c[k]);
  c = fma(c, x2, 1.0);  // cos x
  S = 0.5 - 0.5 * s;
  dSdt = -0.5 * CUDART_PI * c;
}
__device__ __forceinline__ void halfcos_poly(float t, float& S, float& dSdt) {
  float x = (t - 0.5f) * 3.14159265358979f;
  float x2 = x * x;
  float s = 1.6059043836821613e-10f;
  s = fmaf(s, x2, -2.5052108385441720e-08f);
  s = fmaf(s, x2, 2.7557319223985893e-06f);
  s = fmaf(s, x2, -1.9841269841269841e-04f);
  s = fmaf(s, x2, 8.3333333333333333e-03f);
  s = fmaf(s, x2, -1.6666666666666667e-01f);
  s = fmaf(s * x2, x, x);
  float c = 2.0876756987868099e-09f;
  c = fmaf(c, x2, -2.7557319223985891e-07f);
  c = fmaf(c, x2, 2.4801587301587302e-05f);
  c = fmaf(c, x2, -1.3888888888888889e-03f);
  c = fmaf(c, x2, 4.1666666666666667e-02f);
  c = fmaf(c, x2, -0.5f);
  c = fmaf(c, x2, 1.0f);
  S = 0.5f - 0.5f * s;
  dSdt = -0.5f * 3.14159265358979f * c;
}

// ------------------------------------------------------------------ splines
#ifndef AB_GSPLINE_COUNT
#define AB_GSPLINE_COUNT 0
#endif
// g_i(c): cubic Hermite on the species' non-uniform knots; clamped (zero slope) outside
template <typename R>
__device__ __forceinline__ R gspline(int sp, R c, R& dg) {
  const Tab<R>& T = tab<R>();
  const int n = T.gn[sp];
  const R* gx = T.gG + sp * 16;
  const R* gy = T.gG + 48 + sp * 16;
  const R* gm = T.gG + 96 + sp * 16;
  if (c <= __ldg(gx)) {
    dg = R(0);
    return __ldg(gy);
  }
  if (c >= __ldg(gx + n - 1)) {
    dg = R(0);
    return __ldg(gy + n - 1);
  }
  int i = 0;
#if AB_GSPLINE_COUNT
  // interval index = number of interior knots <= c (ascending knots): independent loads and
  // compares instead of a dependent load-compare-branch chain per knot (same index)
#pragma unroll
  for (int k = 1; k <= 7; ++k) i += (k <= n - 2 && __ldg(gx + k) <= c) ? 1 : 0;
  if (n > 9)
    for (int k = 8; k <= n - 2; ++k) i += __ldg(gx + k) <= c ? 1 : 0;
#else
#pragma unroll 1
  while (i < n - 2 && __ldg(gx + i + 1) <= c) ++i;
#endif
  R h = __ldg(gx + i + 1) - __ldg(gx + i);
  R t = (c - __ldg(gx + i)) / h;
  R t2 = t * t, t3 = t2 * t;
  R y0 = __ldg(gy + i), y1 = __ldg(gy + i + 1), m0 = h * __ldg(gm + i), m1 = h * __ldg(gm + i + 1);
  R v = (R(2) * t3 - R(3) * t2 + R(1)) * y0 + (t3 - R(2) * t2 + t) * m0 + (R(-2) * t3 + R(3) * t2) * y1 +
        (t3 - t2) * m1;
  R dvt = (R(6) * t2 - R(6) * t) * y0 + (R(3) * t2 - R(4) * t + R(1)) * m0 + (R(-6) * t2 + R(6) * t) * y1 +
          (R(3) * t2 - R(2) * t) * m1;
  dg = dvt / h;
  return v;
}

// 4 knot weights (knots i-1 .. i+2) of the integer-grid Hermite scheme and their x-derivatives.
// grid: knots lo, lo+1, ..., lo+n-1; slopes (y_{i+1}-y_{i-1})/2 inside and 0 at the two ends.
template <typename R>
__device__ __forceinline__ int gridw(R x, R lo, int n, R w[4], R dw[4]) {
  R hi = lo + R(n - 1);
  bool clamped = false;
  if (x <= lo) x = lo, clamped = true;
  else if (x >= hi) x = hi, clamped = true;
  int i = (int)floor(x - lo);
  if (i > n - 2) i = n - 2;
  if (i < 0) i = 0;
  R t = x - (lo + R(i));
  R t2 = t * t, t3 = t2 * t;
  R h00 = R(2) * t3 - R(3) * t2 + R(1), h10 = t3 - R(2) * t2 + t, h01 = R(-2) * t3 + R(3) * t2, h11 = t3 - t2;
  R d00 = R(6) * t2 - R(6) * t, d10 = R(3) * t2 - R(4) * t + R(1), d01 = R(-6) * t2 + R(6) * t,
    d11 = R(3) * t2 - R(2) * t;
  bool mi = (i > 0 && i < n - 1), mi1 = (i + 1 < n - 1);
  // knot i-1 (q=0), i (1), i+1 (2), i+2 (3)
  w[0] = mi ? R(-0.5) * h10 : R(0);
  w[1] = h00 - (mi1 ? R(0.5) * h11 : R(0));
  w[2] = h01 + (mi ? R(0.5) * h10 : R(0));
  w[3] = mi1 ? R(0.5) * h11 : R(0);
  dw[0] = mi ? R(-0.5) * d10 : R(0);
  dw[1] = d00 - (mi1 ? R(0.5) * d11 : R(0));
  dw[2] = d01 + (mi ? R(0.5) * d10 : R(0));
  dw[3] = mi1 ? R(0.5) * d11 : R(0);
  if (clamped)
    for (int q = 0; q < 4; ++q) dw[q] = R(0);
  return i - 1;  // knot index of weight 0
}

// x exactly on a knot of the integer grid (or clamped to an end): the Hermite weights are the
// unit vector (0, 1, 0, 0), so a tensor-product sum has a single non-zero value term and only
// the derivative weights of the other directions contribute -- the same sums with the exact
// zero terms left out (bitwise identical results).  Saturated hydrocarbons have integer
// coordination numbers, so this is the common case of P, pi^rc and T.
template <typename R>
__device__ __forceinline__ bool on_knot(R x, R lo, int n) {
  if (x <= lo || x >= lo + R(n - 1)) return true;
  return x == floor(x);
}
// the knot an on-knot (or clamped) coordinate sits on
template <typename R>
__device__ __forceinline__ int knot_of(R x, R lo, int n) {
  if (x <= lo) return 0;
  if (x >= lo + R(n - 1)) return n - 1;
  return (int)(x - lo);
}

// P_ij(N^C, N^H) for a C centre (table index = partner species); value and gradient
template <typename R>
__device__ __forceinline__ R pspline(int tj, R x, R y, R& dx, R& dy) {
  const Tab<R>& T = tab<R>();
  R wx[4], dwx[4], wy[4], dwy[4];
  int ax = gridw(x, R(0), 5, wx, dwx);
  int ay = gridw(y, R(0), 5, wy, dwy);
  if (on_knot(x, R(0), 5) && on_knot(y, R(0), 5)) {  // value: 1 term; gradient: 4 + 4 terms
    const int kx = knot_of(x, R(0), 5), ky = knot_of(y, R(0), 5);
    R fx = 0, fy = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      int ka = ax + a, kb = ay + a;
      if (ka >= 0 && ka <= 4) fx += dwx[a] * __ldg(T.gP + tj * 25 + ka * 5 + ky);
      if (kb >= 0 && kb <= 4) fy += dwy[a] * __ldg(T.gP + tj * 25 + kx * 5 + kb);
    }
    dx = fx, dy = fy;
    return __ldg(T.gP + tj * 25 + kx * 5 + ky);
  }
  R f = 0, fx = 0, fy = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int ka = ax + a;
    if (ka < 0 || ka > 4) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int kb = ay + b;
      if (kb < 0 || kb > 4) continue;
      R v = __ldg(T.gP + tj * 25 + ka * 5 + kb);
      f += wx[a] * wy[b] * v;
      fx += dwx[a] * wy[b] * v;
      fy += wx[a] * dwy[b] * v;
    }
  }
  dx = fx, dy = fy;
  return f;
}

// tricubic pi^rc / T table (which 0 = R, 1 = T) of pair p at (x, y, z) on 5 x 5 x 9 knots from (0,0,1)
template <typename R>
__device__ __forceinline__ R rtspline(int which, int p, R x, R y, R z, R& gx, R& gy, R& gz) {
  const Tab<R>& T = tab<R>();
  const R* tb = T.gRT + (which * 3 + p) * 225;
  R wx[4], dwx[4], wy[4], dwy[4], wz[4], dwz[4];
  int ax = gridw(x, R(0), 5, wx, dwx);
  int ay = gridw(y, R(0), 5, wy, dwy);
  int az = gridw(z, R(1), 9, wz, dwz);
  if (on_knot(x, R(0), 5) && on_knot(y, R(0), 5) && on_knot(z, R(1), 9)) {  // 1 + 4 + 4 + 4 terms
    const int kx = knot_of(x, R(0), 5), ky = knot_of(y, R(0), 5), kz = knot_of(z, R(1), 9);
    R fx = 0, fy = 0, fz = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      int ka = ax + a, kb = ay + a, kc = az + a;
      if (ka >= 0 && ka <= 4) fx += dwx[a] * __ldg(tb + (ka * 5 + ky) * 9 + kz);
      if (kb >= 0 && kb <= 4) fy += dwy[a] * __ldg(tb + (kx * 5 + kb) * 9 + kz);
      if (kc >= 0 && kc <= 8) fz += dwz[a] * __ldg(tb + (kx * 5 + ky) * 9 + kc);
    }
    gx = fx, gy = fy, gz = fz;
    return __ldg(tb + (kx * 5 + ky) * 9 + kz);
  }
  R f = 0, fx = 0, fy = 0, fz = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int ka = ax + a;
    if (ka < 0 || ka > 4) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int kb = ay + b;
      if (kb < 0 || kb > 4) continue;
      R wab = wx[a] * wy[b], dxab = dwx[a] * wy[b], dyab = wx[a] * dwy[b];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        int kc = az + c;
        if (kc < 0 || kc > 8) continue;
        R v = __ldg(tb + (ka * 5 + kb) * 9 + kc);
        f += wab * wz[c] * v;
        fx += dxab * wz[c] * v;
        fy += dyab * wz[c] * v;
        fz += wab * dwz[c] * v;
      }
    }
  }
  gx = fx, gy = fy, gz = fz;
  return f;
}

// ------------------------------------------------------------------ atomics and reductions
// AB_SINGLE (kernels instantiated with SG = true) accumulates in fp32: a running sum is rounded
// to binary32 after every addition (both operands are binary32 values, so this is the fp32 sum
// up to a rare double rounding)
template <bool SG = false>
__device__ __forceinline__ double acc_round(double a) { return SG ? (double)(float)a : a; }

// With SG the force array handed to the kernels is an fp32 array (engine.cu: Ff), summed with
// fp32 atomics and widened into F after the evaluation.
template <bool SG = false>
__device__ __forceinline__ void atomic_add3(double* F, int a, double x, double y, double z) {
  if (SG) {
    float* f = reinterpret_cast<float*>(F);
    atomicAdd(f + 3 * a + 0, (float)x);
    atomicAdd(f + 3 * a + 1, (float)y);
    atomicAdd(f + 3 * a + 2, (float)z);
    return;
  }
  atomicAdd(F + 3 * a + 0, x);
  atomicAdd(F + 3 * a + 1, y);
  atomicAdd(F + 3 * a + 2, z);
}

template <bool SG = false>
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = acc_round<SG>(v + __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_max_i(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, (long long)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Accumulators of one force evaluation (device memory, zeroed per evaluation)
enum {
  ACC_EREBO = 0,
  ACC_ETORS,
  ACC_ELJ,
  ACC_W,  // 6 virial components follow: xx yy zz xy xz yz
  ACC_KE = ACC_W + 6,
  ACC_N
};
enum {
  CT_SHORT = 0,
  CT_BONDS,
  CT_QUADS,
  CT_LJ,
  CT_C0,
  CT_BSTAR,
  CT_SBTRANS,
  CT_MAXSHORT,
  CT_MAXREACH,
  CT_BADARG,
  CT_OVF_REACH,   // reach table overflows (fallback path search used)
  CT_OVF_QUEUE,   // b* queue overflow (evaluation must be redone)
  CT_OVF_SHORT,   // more than NBMAX short neighbours (hard error)
  CT_OVF_STAGE,
  CT_LJENT,       // skinned LJ list entries streamed
  CT_ANGLES,      // bond-order angle terms
  CT_LJFAR,       // canonical LJ pairs within r_c handled by the far kernel
  CT_LJENTFAR,    // far-list entries streamed
  CT_LJTAPER,     // canonical LJ pairs in the taper band r_lo < r <= r_c
  CT_N
};

// ---- block-partial reductions of energies / virial / counters -----------------------------
// Thousands of same-address global atomics per launch serialise in L2; instead every block
// reduces into shared memory and stores one partial row (column-major), and k_reduce sums the
// rows in a fixed order (deterministic totals).
struct RedRows {
  double* d;              // [ACC_N][stride]
  unsigned long long* u;  // [CT_N][stride]
  int stride, row0;
};
struct RedSmem {
  double d[ACC_N];
  unsigned long long u[CT_N];
};
__device__ __forceinline__ bool ct_is_max(int c) { return c == CT_MAXSHORT || c == CT_MAXREACH; }
__device__ __forceinline__ void red_init(RedSmem& s) {
  for (int c = threadIdx.x; c < ACC_N; c += blockDim.x) s.d[c] = 0.0;
  for (int c = threadIdx.x; c < CT_N; c += blockDim.x) s.u[c] = 0ull;
  __syncthreads();
}
// warp-reduce v and add it into the block's shared row (all 32 lanes of the warp must call)
__device__ __forceinline__ void red_add_d(RedSmem& s, int col, double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v != 0.0) atomicAdd(&s.d[col], v);
}
__device__ __forceinline__ void red_add_u(RedSmem& s, int col, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s.u[col], v);
}
__device__ __forceinline__ void red_max_u(RedSmem& s, int col, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, (unsigned long long)__shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v) atomicMax(&s.u[col], v);
}
__device__ __forceinline__ void red_flush(const RedSmem& s, RedRows R) {
  __syncthreads();
  int row = R.row0 + blockIdx.x;
  for (int c = threadIdx.x; c < ACC_N; c += blockDim.x) R.d[(size_t)c * R.stride + row] = s.d[c];
  for (int c = threadIdx.x; c < CT_N; c += blockDim.x) R.u[(size_t)c * R.stride + row] = s.u[c];
}
// A block of a grid-stride kernel that gets no work item (blockIdx.x * blockDim.x >= nwork, the
// same for all its threads) writes a zero partial row without barriers and leaves: the overflow
// batches are launched with fixed grids and are usually empty.
__device__ __forceinline__ bool red_idle_block(int nwork, const RedRows& R) {
  if ((long long)blockIdx.x * blockDim.x < nwork) return false;
  const int row = R.row0 + blockIdx.x;
  for (int c = threadIdx.x; c < ACC_N; c += blockDim.x) R.d[(size_t)c * R.stride + row] = 0.0;
  for (int c = threadIdx.x; c < CT_N; c += blockDim.x) R.u[(size_t)c * R.stride + row] = 0ull;
  return true;
}
// one block per column: fixed-order sum (max for the max counters) over nrows partial rows
__device__ __forceinline__ void reduce_column(const RedRows& R, int nrows, double* acc, unsigned long long* ct,
                                              int c) {
  __shared__ double sd[32];
  __shared__ unsigned long long su[32];
  bool isd = c < ACC_N;
  int cc = isd ? c : c - ACC_N;
  bool mx = !isd && ct_is_max(cc);
  double vd = 0.0;
  unsigned long long vu = 0ull;
  // 8 rows per thread in flight, summed in the same row order as a plain strided loop (absent
  // rows contribute an exact 0): the loads no longer wait on one another
  constexpr int U = 8;
  const double* cd = R.d + (size_t)cc * R.stride;
  const unsigned long long* cu = R.u + (size_t)cc * R.stride;
  for (int r0 = threadIdx.x; r0 < nrows; r0 += U * blockDim.x) {
    if (isd) {
      double x[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int r = r0 + k * (int)blockDim.x;
        x[k] = r < nrows ? cd[r] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) vd += x[k];
    } else {
      unsigned long long x[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int r = r0 + k * (int)blockDim.x;
        x[k] = r < nrows ? cu[r] : 0ull;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) vu = mx ? max(vu, x[k]) : vu + x[k];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vd += __shfl_xor_sync(0xffffffffu, vd, o);
    unsigned long long y = __shfl_xor_sync(0xffffffffu, vu, o);
    vu = mx ? max(vu, y) : vu + y;
  }
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sd[w] = vd, su[w] = vu;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
      vd += sd[q];
      vu = mx ? max(vu, su[q]) : vu + su[q];
    }
    if (isd) acc[cc] += vd;  // acc may already hold direct contributions (KE)
    else ct[cc] = mx ? max(ct[cc], vu) : ct[cc] + vu;
  }
}
__global__ void k_reduce(RedRows R, int nrows, double* acc, unsigned long long* ct) {
  reduce_column(R, nrows, acc, ct, blockIdx.x);
}

// warp-reduce an array of doubles and add lane 0's totals into global accumulators.
// Must be called by all 32 lanes of a warp.
template <int K>
__device__ __forceinline__ void warp_acc(double (&v)[K], double* acc) {
#pragma unroll
  for (int q = 0; q < K; ++q) {
    double s = warp_sum(v[q]);
    if ((threadIdx.x & 31) == 0 && s != 0.0) atomicAdd(acc + q, s);
  }
}

// virial of a vector v = x_b - x_a with energy gradient g = dE/dv:  W -= v (x) g
template <typename R>
__device__ __forceinline__ void vir_add(double W[6], V3<R> v, V3<R> g) {
  if (!W) return;  // NVE instantiations pass a literal nullptr: folded away after inlining
  W[0] -= (double)v.x * (double)g.x;
  W[1] -= (double)v.y * (double)g.y;
  W[2] -= (double)v.z * (double)g.z;
  W[3] -= (double)v.x * (double)g.y;
  W[4] -= (double)v.x * (double)g.z;
  W[5] -= (double)v.y * (double)g.z;
}

// Half convention: the pair (i, J) belongs to i iff gid_i < gid_J, or the same atom
// with image s_J >_lex 0.  shift is packed as char4.
__device__ __forceinline__ bool canonical_pair(int gi, int gj, char4 sj) {
  if (gi != gj) return gi < gj;
  return sj.x > 0 || (sj.x == 0 && (sj.y > 0 || (sj.y == 0 && sj.z > 0)));
}

// Instance key stored in the w slot of every position (bit pattern of an int64, never used in
// FP arithmetic): gid << 26 | (sx+128) << 18 | (sy+128) << 10 | (sz+128) << 2 | type.
// Lexicographic (gid, image) order == integer order, so the half convention is key_i < key_J
// and the species comes with the same 32-byte position load.
__host__ __device__ __forceinline__ long long make_key(int gid, int sx, int sy, int sz, int type) {
  return ((long long)gid << 26) | ((long long)(sx + 128) << 18) | ((long long)(sy + 128) << 10) |
         ((long long)(sz + 128) << 2) | (long long)type;
}
__device__ __forceinline__ long long key_of(const double4& p) { return __double_as_longlong(p.w); }
__device__ __forceinline__ int type_of(const double4& p) { return __double2loint(p.w) & 3; }

// One position record (x, y, z, key: 32 bytes, 32-byte aligned) with ONE 256-bit load
// (sm_100 ld.global.v4.f64 -> LDG.E.256) instead of the two 128-bit loads a double4 access
// compiles to: a scattered gather then costs one L1 pass per partner, not two.  Only for arrays
// the running kernel does not write (the asm carries no memory dependence).  W = false: plain load.
#ifndef AB_NEAR_PREF
#define AB_NEAR_PREF 2  // window row prefetched (L2) before the reach-set walk: cfg4 near 1.095 -> 1.073 ms
#endif
#ifndef AB_NEAR_POS256
#define AB_NEAR_POS256 0
#endif
template <bool W = true>
__device__ __forceinline__ double4 ld_pos(const double4* p) {
  if (!W) return *p;
  double4 v;
  asm("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

}  // namespace ab
