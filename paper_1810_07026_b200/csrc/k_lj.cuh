// k_lj.cuh -- the LJ term gated by C_ij (Alg. 3; E = Q C V) with the
// per-atom reach set of the C_ij connectivity switch.
//
// Both kernels stream FULL skinned lists (both directions): every pair is evaluated from both
// ends, so F_i is a register gather with one atomic per atom and nothing is scattered onto j.
// The pairs are split by their current distance against a_p = 2^(1/6) sigma_p sqrt(1 + 1e-9), the
// S_r window pre-filter (k_lists.cuh: near list r_b <= a_p + skin, far list r_b >= a_p - skin):
//
// k_lj_near -- 8 lanes per local atom i (4 atoms per warp).
//   The lane group first maps out every atom image reachable from i in 1, 2 or 3 bonds with the
//   maximum path-weight product M (the paper's "map out all the atoms j connected to atom i
//   once") into a 64-slot open-addressing table in shared memory (keys = image
//   index, value = M via atomicMax on its bit pattern, M >= 0).  Overflow (table or 2-hop list)
//   -> the direct nested search of P:844-853 for that atom (the paper's "sequential fallback",
//   P:866).  Window pairs (r^2 < a_p^2): C = 1 - M, skip if C == 0 (gate order of P:824-830),
//   otherwise deferred to the b* batch (canonical direction only).  Then the reach set
//   is walked once more: for its members J in the far zone (r^2 >= a_p^2, r <= r_c), which
//   k_lj_far evaluated with C = 1, i subtracts M V (E = C V = V - M V) and the force of
//   it; forces from dC (0 < M < 1, reactive systems only) once, by the canonical direction.
// k_lj_far -- one warp per local atom i over the far row (C = 1; distance bins decide per bin
//   whether a pair needs the window / cutoff tests and the taper, or can be skipped).
//   No shared memory, branch-free bodies, 4 independent gathers in flight per lane.
// Counters count canonical directions only (key_i < key_J), so they equal the oracle's half sums.
#pragma once
#include "dev_common.cuh"
#include "k_bond.cuh"

namespace ab {

#ifndef AB_NEAR_GROUP
#define AB_NEAR_GROUP 4
#endif
#ifndef AB_NEAR_SLOTS
#define AB_NEAR_SLOTS 64
#endif
constexpr int NEAR_GROUP = AB_NEAR_GROUP;        // lanes per atom (measured on cfg4: 4 beats 8 and 16)
#ifndef AB_NEAR_BLOCK
#define AB_NEAR_BLOCK 128
#endif
constexpr int NEAR_ATOMS = AB_NEAR_BLOCK / NEAR_GROUP;  // atoms per block
constexpr int NEAR_SLOTS = AB_NEAR_SLOTS;        // reach table slots per atom (measured: 64 beats 128)
static_assert(NEAR_SLOTS <= 64, "the correction pass keeps the occupied slots in a 64-bit mask");

#ifndef AB_NEAR_BLOOM
#define AB_NEAR_BLOOM 16 // 32-bit words of the per-atom Bloom filter in front of the table (0: none)
#endif
#ifndef AB_NEAR_BLOCKQ
#define AB_NEAR_BLOCKQ 1
#endif
constexpr int NEAR_BQ = 64;  // per species pair and block (16 atoms); beyond: direct global appends
struct NearBlockQ {
  int n[3], base[3];
  int i[3][NEAR_BQ], j[3][NEAR_BQ];
  double m[3][NEAR_BQ];
};

template <int SL>
struct alignas(16) ReachSmem {  // (16-byte aligned arrays: cleared with vector stores)
  int keys[SL];
  unsigned long long mbits[SL];
#if AB_NEAR_BLOOM
  unsigned bloom[AB_NEAR_BLOOM];  // one bit per inserted key: a clear bit proves M = 0
#endif
  int nins, ovf;
};
static_assert(NEAR_SLOTS % 4 == 0 && AB_NEAR_BLOOM % 4 == 0, "vector clear of the reach table");
#if AB_NEAR_BLOOM
__device__ __forceinline__ unsigned bloom_bit(int key) {  // bits independent of the table slot
  return (((unsigned)key * 0x9E3779B1u) >> 7) & (32u * AB_NEAR_BLOOM - 1u);
}
#endif

__host__ __device__ constexpr int log2i(int v) { return v <= 1 ? 0 : 1 + log2i(v / 2); }
template <int SL>
__device__ __forceinline__ unsigned reach_hash(int key) {
  return ((unsigned)key * 2654435761u) >> (32 - log2i(SL));
}

template <int SL>
__device__ __forceinline__ void reach_insert(ReachSmem<SL>& s, int key, double M) {
  unsigned h = reach_hash<SL>(key);
  for (int probe = 0; probe < SL; ++probe) {
    int old = atomicCAS(&s.keys[h], REACH_EMPTY, key);
    if (old == REACH_EMPTY || old == key) {
      if (old == REACH_EMPTY) {
        atomicAdd(&s.nins, 1);
#if AB_NEAR_BLOOM
        const unsigned b = bloom_bit(key);
        atomicOr(&s.bloom[b >> 5], 1u << (b & 31u));
#endif
      }
      atomicMax(&s.mbits[h], (unsigned long long)__double_as_longlong(M));
      return;
    }
    h = (h + 1) & (SL - 1);
  }
  s.ovf = 1;
}

template <int SL>
__device__ __forceinline__ double reach_lookup(const ReachSmem<SL>& s, int key) {
  unsigned h = reach_hash<SL>(key);
  for (int probe = 0; probe < SL; ++probe) {
    int k = s.keys[h];
    if (k == key) return __longlong_as_double((long long)s.mbits[h]);
    if (k == REACH_EMPTY) return 0.0;
    h = (h + 1) & (SL - 1);
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

// AIREBO-M radial form: V_M = eps_m [x^2 - 2 x], x = e^{-a (r - r_e)};
// returns V_M and (dV_M/dr)/r = 2 a eps_m x (1 - x) / r
template <typename R>
__device__ __forceinline__ R morse_plain(R em, R a, R re, R r, R ir, R& dVr) {
  R x = ex(-a * (r - re));
  dVr = R(2) * a * em * x * (R(1) - x) * ir;
  return em * (x * x - R(2) * x);
}

struct LJArgs {
  int N;
  int r0b, r0e, r1b, r1e;  // k_lj_far: the atoms [r0b, r0e) and [r1b, r1e) (slab interior / boundary split)
  const double4* pos;
  int cap[3];
  const int* cnt[3];
  const int* nbr[3];
  const unsigned short* boff;          // far-row bin ends (k_lists.cuh FB_*)
  const double4* xref;                 // positions at the last build (per-atom displacement)
  const unsigned long long* dbound;    // bits of max displacement^2 of any atom since the build (nullptr: skin/2)
  double skin, i2, i8;                 // skin, 4 / skin, 8 / skin
  int binned;                          // 0: every far entry through the fully tested body
  unsigned long long* maxreach;        // k_lj_near: persistent max reach-set size (nullptr: off)
  int* smq;                            // k_lj_far: per-SM queue counters [nq], zero at launch (nullptr: static ranges)
  int nq, qper;                        // queues, atoms per queue
};

__device__ __forceinline__ void stage_lj_row(StageBuf stage, int gi, int gj, char4 sh, double C, double bs) {
  double* rw = stage_row(stage, 7);
  if (rw) rw[0] = gi, rw[1] = gj, rw[2] = sh.x, rw[3] = sh.y, rw[4] = sh.z, rw[5] = C, rw[6] = bs;
}

template <int W, bool SG = false>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v = acc_round<SG>(v + __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------------- near pairs
// 8 lanes per atom.  The reach table holds the maximal path product per reachable image; the
// pair loop is branch-light (the rare b* / fractional-C / stage work sits at the end of the
// body) so the group stays converged through the LJ arithmetic.
template <int SL>
__device__ __forceinline__ double reach_lookup_fast(const ReachSmem<SL>& s, int key) {
#if AB_NEAR_BLOOM
  const unsigned b = bloom_bit(key);
  if (!((s.bloom[b >> 5] >> (b & 31u)) & 1u)) return 0.0;  // not in the reach set: M = 0
#endif
  unsigned h = reach_hash<SL>(key);
#pragma unroll
  for (int probe = 0; probe < 4; ++probe) {
    int k = s.keys[h];
    if (k == key) return __longlong_as_double((long long)s.mbits[h]);
    if (k == REACH_EMPTY) return 0.0;
    h = (h + 1) & (SL - 1);
  }
  return reach_lookup<SL>(s, key);  // long probe chain: rare
}

template <typename R, bool VIRIAL, bool MORSE, bool SG = false, int SL = NEAR_SLOTS>
#ifndef AB_NEAR_MINBLOCKS
#define AB_NEAR_MINBLOCKS 7  // measured (cfg4, 4-lane groups, with the window-row prefetch): 5 / 6 / 7 blocks 1.239 / 1.073 / 1.017 ms (7 = the shared-memory limit with 64-slot tables)
#endif
__global__ void __launch_bounds__(NEAR_GROUP * NEAR_ATOMS, AB_NEAR_MINBLOCKS) k_lj_near(LJArgs A, ShortList<R> S, const int* owner,
                                                                    const int* gid, const char4* shift, double* F,
                                                                    double* acc, unsigned long long* ct,
                                                                    BstarQueue Qu, StageBuf stage, RedRows RR) {
  __shared__ ReachSmem<SL> sm_all[NEAR_ATOMS];
  __shared__ RedSmem rs;
#if AB_NEAR_BLOCKQ
  __shared__ NearBlockQ bq;
  if (threadIdx.x < 3) bq.n[threadIdx.x] = 0;
#endif
  // per-pair parameters indexed by the species pair p, which differs between the lanes of a
  // warp: shared-memory copies (an indexed __constant__ load serialises per distinct address)
  __shared__ double pd[9];  // r_c^2, S_r window pre-filter, r_lo^2
  __shared__ R pr_[12];     // 4 eps, sigma^2, r_lo, r_c  (Morse: eps_m, a, r_e, -)
  const Tab<R>& T = tab<R>();
  if (threadIdx.x < 3) {
    const int t = threadIdx.x;
    pd[t] = c_geo.rc2[t], pd[3 + t] = c_geo.srhi2_hi[t], pd[6 + t] = c_geo.rlo2[t];
    pr_[t] = MORSE ? T.meps[t] : R(4) * T.eps[t], pr_[3 + t] = MORSE ? T.malpha[t] : T.sigma2[t];
    pr_[6 + t] = T.rlo[t], pr_[9 + t] = T.rc[t];
  }
  __shared__ R pm_[3];  // Morse r_e
  if (MORSE && threadIdx.x < 3) pm_[threadIdx.x] = T.mre[threadIdx.x];
  red_init(rs);
  const int grp = threadIdx.x / NEAR_GROUP, gl = threadIdx.x % NEAR_GROUP;
  ReachSmem<SL>& s = sm_all[grp];
  const int i = blockIdx.x * NEAR_ATOMS + grp;
  const bool active = i < A.N;
  const int cntN = active ? A.cnt[0][i] : 0;
#if AB_NEAR_PREF
  // the atom's window row (step 2) requested now, so it arrives while the reach set is built
  if (active) {
    const int* prow = A.nbr[0] + (size_t)i * A.cap[0];
    for (int q = gl * 32; q < cntN; q += NEAR_GROUP * 32) {
#if AB_NEAR_PREF == 2
      asm volatile("prefetch.global.L2 [%0];" ::"l"(prow + q));
#else
      asm volatile("prefetch.global.L1 [%0];" ::"l"(prow + q));
#endif
    }
#if AB_NEAR_PREF == 3
    for (int q = gl; q < cntN; q += NEAR_GROUP) asm volatile("prefetch.global.L1 [%0];" ::"l"(A.pos + prow[q]));
#endif
  }
#endif

  // 1. reach set of i: lane per neighbour k of i enumerates k, l in N(k), m in N(l)
  for (int q = gl; q < SL / 4; q += NEAR_GROUP)
    reinterpret_cast<int4*>(s.keys)[q] = make_int4(REACH_EMPTY, REACH_EMPTY, REACH_EMPTY, REACH_EMPTY);
  for (int q = gl; q < SL / 2; q += NEAR_GROUP) reinterpret_cast<ulonglong2*>(s.mbits)[q] = make_ulonglong2(0ull, 0ull);
  if (gl == 0) s.nins = 0, s.ovf = 0;
#if AB_NEAR_BLOOM
  for (int q = gl; q < AB_NEAR_BLOOM / 4; q += NEAR_GROUP) reinterpret_cast<uint4*>(s.bloom)[q] = make_uint4(0u, 0u, 0u, 0u);
#endif
  __syncwarp();
  const size_t bi = (size_t)(active ? i : 0) * S.capS;
#ifdef AB_ABL_NOREACH
  const int ni = 0;  // ablation (timing experiments only): no reach set
#else
  const int ni = active ? S.cnt[i] : 0;
#endif
  // Flattened walk: level 1 (k in N(i)) one lane per k; level 2 (l in N(k)) the (k, l) pairs are
  // spread over the group's lanes (the owner lane of pair e found by a binary search over the
  // group's exclusive prefix counts, all through shuffles: no indexed arrays, no local memory);
  // level 3 (m in N(l)) the lane walks right away.  Products keep the association
  // (w_ik w_kl) w_lm of the paper's nested enumeration, so M is bitwise that of the serial walk
  // (the fallback for large neighbourhoods).
  const unsigned gmask = (NEAR_GROUP == 32 ? 0xffffffffu : ((1u << NEAR_GROUP) - 1u)) << (threadIdx.x & 31 & ~(NEAR_GROUP - 1));
  if (ni <= NEAR_GROUP) {
    int k1 = -1, n1 = 0;
    double w1 = 0;
    if (gl < ni) {
      k1 = S.nbr[bi + gl];
      w1 = S.wd[bi + gl];
      n1 = S.cnt[k1];
      reach_insert(s, k1, w1);
    }
    int incl = n1;
#pragma unroll
    for (int o = 1; o < NEAR_GROUP; o <<= 1) {
      const int u = __shfl_up_sync(gmask, incl, o, NEAR_GROUP);
      if (gl >= o) incl += u;
    }
    const int excl = incl - n1;
    const int T2 = __shfl_sync(gmask, incl, NEAR_GROUP - 1, NEAR_GROUP);
    for (int base = 0; base < T2; base += NEAR_GROUP) {
      const int e = base + gl;
      int t = 0;  // last lane with excl_t <= e (lanes without entries share the next one's excl)
#pragma unroll
      for (int bb = NEAR_GROUP / 2; bb > 0; bb >>= 1) {
        const int ex = __shfl_sync(gmask, excl, t + bb, NEAR_GROUP);
        if (ex <= e) t += bb;
      }
      const int k = __shfl_sync(gmask, k1, t, NEAR_GROUP);
      const double wk = __shfl_sync(gmask, w1, t, NEAR_GROUP);
      const int off = e - __shfl_sync(gmask, excl, t, NEAR_GROUP);
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
  } else {  // large neighbourhood: one lane per k walks its paths (the nested enumeration)
    for (int t = gl; t < ni; t += NEAR_GROUP) {
      int k = S.nbr[bi + t];
      double w1t = S.wd[bi + t];
      reach_insert(s, k, w1t);
      size_t bk = (size_t)k * S.capS;
      int nk = S.cnt[k];
      for (int b = 0; b < nk; ++b) {
        int l = S.nbr[bk + b];
        if (l == i) continue;
        double w12 = w1t * S.wd[bk + b];
        reach_insert(s, l, w12);
        size_t bl = (size_t)l * S.capS;
        int nl = S.cnt[l];
        for (int c = 0; c < nl; ++c) {
          int m = S.nbr[bl + c];
          if (m == i) continue;
          reach_insert(s, m, w12 * S.wd[bl + c]);
        }
      }
    }
  }
  __syncwarp();
  const bool ovf = s.ovf != 0;

  // 2. window pairs (near list, r^2 < a_p^2 now).  The next entry's index and position are loaded
  // before the current one is processed.  A pair with C_ij = 0 is skipped (Alg. 3); every other
  // pair may have S_r != 0: the canonical side queues it and the b* batch takes the exact fp64
  // window decision and evaluates the whole pair (b* if S_r != 0, else the plain gated LJ) for
  // both atoms.  No LJ arithmetic here.
  double fx = 0, fy = 0, fz = 0, en = 0;
  double W[6] = {0, 0, 0, 0, 0, 0};
  unsigned nlj = 0, nc0 = 0;
  const double4 pi = A.pos[active ? i : 0];
  const int ti = type_of(pi);
  const long long ki = key_of(pi);
  if (cntN > 0) {
    const int* row = A.nbr[0] + (size_t)i * A.cap[0];
    int Jn = gl < cntN ? row[gl] : i;
    double4 pjn = ld_pos<AB_NEAR_POS256 != 0>(A.pos + Jn);
    for (int q = gl; q < cntN; q += NEAR_GROUP) {
      const int J = Jn;
      const double4 pj = pjn;
      if (q + NEAR_GROUP < cntN) {
        Jn = row[q + NEAR_GROUP];
        pjn = ld_pos<AB_NEAR_POS256 != 0>(A.pos + Jn);
      }
      const double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
      const double r2 = r2_exact(dx, dy, dz);
      const int p = ti + type_of(pj);
      const bool inw = r2 < pd[3 + p];  // window zone (a_p < r_c: inside the cutoff)
      const bool canon = ki < key_of(pj);
      double Md = 0.0;
#ifndef AB_ABL_NOLOOKUP
      if (inw && r2 <= c_geo.reach2) Md = ovf ? (double)path_search(S, i, J).M : reach_lookup_fast(s, J);
#endif
      const bool c0 = inw && Md == 1.0;  // C_ij == 0 (Alg. 3 "continue")
      const bool cand = inw && !c0;
      nlj += inw && canon;
      nc0 += c0 && canon;
      if (cand && canon) {  // deferred to the b* batch: the whole pair, once, by the canonical side
#if AB_NEAR_BLOCKQ
        // staged in the block's shared-memory queue, flushed with one global atomic per species
        // pair and block (global counters hit by every warp serialised in L2)
        const int k = atomicAdd(&bq.n[p], 1);
        if (k < NEAR_BQ) {
          bq.i[p][k] = i, bq.j[p][k] = J, bq.m[p][k] = Md;
        } else {
          const int g = atomicAdd(Qu.count + p, 1);
          if (g < Qu.cap[p]) {
            Qu.item[Qu.off[p] + g] = make_int4(i, J, 0, 0);
            Qu.M[Qu.off[p] + g] = Md;
          } else {
            atomicAdd(ct + CT_OVF_QUEUE, 1ull);
          }
        }
#else
        unsigned am = __activemask();
        unsigned grp = __match_any_sync(am, p);  // one aggregated append per species pair
        int lane = threadIdx.x & 31, leader = __ffs(grp) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(Qu.count + p, __popc(grp));
        base = __shfl_sync(am, base, leader);
        int k = base + __popc(grp & ((1u << lane) - 1u));
        if (k < Qu.cap[p]) {
          Qu.item[Qu.off[p] + k] = make_int4(i, J, 0, 0);
          Qu.M[Qu.off[p] + k] = Md;
        } else {
          atomicAdd(ct + CT_OVF_QUEUE, 1ull);
        }
#endif
      }
      if (VIRIAL && stage.rows && canon && c0) stage_lj_row(stage, gid[i], gid[J], shift[J], 0.0, 0.0);
    }
  }

  // 3. reach-set correction of the far-zone pairs (r^2 >= a_p^2, r <= r_c): k_lj_far evaluated
  // them with C = 1, the pair's share is C V = V - M V, so i subtracts M V (and its force) for
  // every image J of its reach set there; forces from dC/dx along the maximising path (0 < M < 1)
  // once, by the canonical side.  The table holds every reachable image unless it overflowed;
  // then the far row is scanned with the nested path search (P:866's sequential fallback).
  if (active) {
    auto correct = [&](int J, double Md) {
      const double4 pj = ld_pos<AB_NEAR_POS256 != 0>(A.pos + J);
      const double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
      const double r2 = r2_exact(dx, dy, dz);
      const int p = ti + type_of(pj);
      if (!(r2 >= pd[3 + p] && r2 <= pd[p])) return;
      const bool canon = ki < key_of(pj);
      const R rr2 = (R)r2;
      R y = MORSE ? rsqrt_fast(rr2) : R(0);
      R dVr;
      R V = MORSE ? morse_plain<R>(pr_[p], pr_[3 + p], pm_[p], rr2 * y, y, dVr)
                  : lj_plain<R>(pr_[p], pr_[3 + p], rcp_fast(rr2), dVr);
      if (r2 > pd[6 + p]) {  // taper S(r; r_lo, r_c) (reading A10)
        if (!MORSE) y = rsqrt_fast(rr2);
        R r = rr2 * y, dsw;
        R sv = sw<R>(r, pr_[6 + p], pr_[9 + p], dsw);
        dVr = dVr * sv + V * dsw * y;
        V = V * sv;
      }
      const R fr = -(R)Md * dVr;
      fx = acc_round<SG>(fx + (double)(fr * (R)dx));
      fy = acc_round<SG>(fy + (double)(fr * (R)dy));
      fz = acc_round<SG>(fz + (double)(fr * (R)dz));
      en = acc_round<SG>(en - (double)((R)Md * V));
      if (VIRIAL) {
        V3<R> dd = mk3<R>((R)dx, (R)dy, (R)dz);
        vir_add(W, dd, (R(0.5) * fr) * dd);
      }
      nc0 += Md == 1.0 && canon;
      if (canon && Md < 1.0) {  // 0 < C < 1: dC/dx along the maximising path, once per pair
        PathRes<R> prs = path_search(S, i, J);
        double Wp[6] = {0, 0, 0, 0, 0, 0};
        path_forces<R, SG>(S, owner, prs, -V, F, Wp);
        if (VIRIAL)
          for (int c = 0; c < 6; ++c) W[c] += Wp[c];
      }
      if (VIRIAL && stage.rows && canon) stage_lj_row(stage, gid[i], gid[J], shift[J], 1.0 - Md, 0.0);
    };
    if (!ovf) {
      // occupied slots with M > 0 as one 64-bit mask (bit q = slot q; lane gl reads slots
      // 8 gl .. 8 gl + 7, OR-reduced over the group), then dealt out to the lanes 8 at a time in
      // slot order (the n-th set bit by __fns on the two halves): the group stays converged
      constexpr int SPL = SL / NEAR_GROUP;
      unsigned long long vm = 0ull;
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const int q = SPL * gl + k;
        if (s.keys[q] != REACH_EMPTY && s.mbits[q] != 0ull) vm |= 1ull << q;
      }
#pragma unroll
      for (int o = 1; o < NEAR_GROUP; o <<= 1) vm |= __shfl_xor_sync(gmask, vm, o, NEAR_GROUP);
      const unsigned lo = (unsigned)vm, hi = (unsigned)(vm >> 32);
      const int clo = __popc(lo), tot = clo + __popc(hi);
      for (int n = gl; n - gl < tot; n += NEAR_GROUP) {
        if (n < tot) {
          const int q = n < clo ? (int)__fns(lo, 0, n + 1) : 32 + (int)__fns(hi, 0, n - clo + 1);
          correct(s.keys[q], __longlong_as_double((long long)s.mbits[q]));
        }
      }
    } else {
      const int* row1 = A.nbr[1] + (size_t)i * A.cap[1];
      const int c1 = A.cnt[1][i];
      for (int q = gl; q < c1; q += NEAR_GROUP) {
        const int J = row1[q];
        const double4 pj = ld_pos<AB_NEAR_POS256 != 0>(A.pos + J);
        const double r2 = r2_exact(__dsub_rn(pj.x, pi.x), __dsub_rn(pj.y, pi.y), __dsub_rn(pj.z, pi.z));
        if (r2 > c_geo.reach2) continue;
        const double Md = (double)path_search(S, i, J).M;
        if (Md > 0.0) correct(J, Md);
      }
    }
  }

  // 3. reductions (8-lane groups, then one partial row per block)
  fx = group_sum<NEAR_GROUP, SG>(fx);
  fy = group_sum<NEAR_GROUP, SG>(fy);
  fz = group_sum<NEAR_GROUP, SG>(fz);
  if (gl == 0 && active) atomic_add3<SG>(F, i, fx, fy, fz);
#if AB_NEAR_BLOCKQ
  // flush the block's b* candidates: one global atomic per species pair
  __syncthreads();
  if (threadIdx.x < 3) {
    const int n = min(bq.n[threadIdx.x], NEAR_BQ);
    bq.base[threadIdx.x] = n ? atomicAdd(Qu.count + threadIdx.x, n) : 0;
  }
  __syncthreads();
#pragma unroll
  for (int pp = 0; pp < 3; ++pp) {
    const int n = min(bq.n[pp], NEAR_BQ);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const int g = bq.base[pp] + k;
      if (g < Qu.cap[pp]) {
        Qu.item[Qu.off[pp] + g] = make_int4(bq.i[pp][k], bq.j[pp][k], 0, 0);
        Qu.M[Qu.off[pp] + g] = bq.m[pp][k];
      } else {
        atomicAdd(ct + CT_OVF_QUEUE, 1ull);
      }
    }
  }
#endif
  red_add_d(rs, ACC_ELJ, 0.5 * en);
  if (VIRIAL)
    for (int c = 0; c < 6; ++c) red_add_d(rs, ACC_W + c, W[c]);
  red_add_u(rs, CT_LJ, (unsigned long long)nlj);
  red_add_u(rs, CT_C0, (unsigned long long)nc0);
  red_max_u(rs, CT_MAXREACH, gl == 0 ? (unsigned long long)s.nins : 0ull);
  red_add_u(rs, CT_OVF_REACH, gl == 0 && ovf ? 1ull : 0ull);
  red_add_u(rs, CT_LJENT, gl == 0 ? (unsigned long long)cntN : 0ull);
  red_flush(rs, RR);
  // max reach-set size since the last list build (persistent, read by the host at the next
  // rebuild to size the table: 32 slots while every set stays small, else 64)
  if (threadIdx.x == 0 && A.maxreach && rs.u[CT_MAXREACH]) atomicMax(A.maxreach, rs.u[CT_MAXREACH]);
}

// ---------------------------------------------------------------------------------- far pairs
// One warp per local atom i over its far row (pairs with r^2 >= a_p^2 at evaluation time, C = 1;
// k_lj_near corrects the reach-set pairs among them).  The row is ordered by build-distance bins
// (k_lists.cuh); with m = |x_i - x_i,build| + max_k |x_k - x_k,build| (+1e-7) every pair distance
// is within m of its build distance, which settles whole bins:
//   L bins entirely below a_p             -> skipped (k_lj_near's pairs)
//   L bins straddling a_p                 -> LOW body: exact r^2, window test, no taper / cutoff
//   L bins above a_p, P, A bins below r_lo -> PURE body: no decisions (fused r^2, no taper)
//   A bins reaching r_lo, B, C bins        -> HIGH body: exact r^2, window + cutoff tests, taper
//   C bins entirely beyond r_c            -> skipped
// Branch-free bodies (out-of-range lanes weighted by 0), 4 independent gathers in flight per lane;
// the taper (half-cosine polynomial) only runs when some lane of the warp is in the taper band.
#ifndef AB_FAR_UNROLL
#define AB_FAR_UNROLL 2  // with the row prefetch and 256-bit gathers (cfg4): 4 chunks x 4 blocks/SM 2.326 ms, 2 x 6 2.153, 1 x 8 2.145, 2 x 7 2.155, 2 x 8 2.184, 3 x 5 2.351
#endif
#ifndef AB_FAR_PIPE
#define AB_FAR_PIPE 0
#endif
#ifndef AB_FAR_TAIL
#define AB_FAR_TAIL 0
#endif
#ifndef AB_FAR_PREF
#define AB_FAR_PREF 1  // 1: next row of the warp prefetched into L2 (measured cfg4: far 2.557 -> 2.402 ms), 2: into L1 (same), (its first positions too: slower)
#endif
#ifndef AB_FAR_IDX
#define AB_FAR_IDX 2  // (measured cfg4: 2.341 -> 2.332 ms) 1: far-row indices loaded with the streaming policy (ld.global.cs), 2: L1::no_allocate
#endif
#ifndef AB_FAR_POS256
#define AB_FAR_POS256 1  // partner positions gathered with one 256-bit load (ld_pos; measured cfg4: far 2.41 -> 2.34 ms)
#endif
#ifndef AB_FAR_SMQ
#define AB_FAR_SMQ 0
#endif
#ifndef AB_FAR_PJ
#define AB_FAR_PJ 0
#endif
#ifndef AB_FAR_SWEEP
#define AB_FAR_SWEEP 1  // measured (cfg4): contiguous per-block atom ranges 2.71 -> 2.66 ms
#endif
constexpr int FAR_UNROLL = AB_FAR_UNROLL;

// Far-pair parameters of the two species pairs (t_i, t_j = C / H) a warp can meet (t_i is warp-
// uniform): 12-6 form V = e4 s6 (s6 - 1), (dV/dr)/r = inv_r2 s6 (6 e4 - 12 e4 s6), s6 = (sigma^2 inv_r2)^3.
// far-row index / partner position loads (A/B knobs above)
__device__ __forceinline__ int far_ld_idx(const int* p) {
#if AB_FAR_IDX == 1
  return __ldcs(p);
#elif AB_FAR_IDX == 2
  int v;
  asm("ld.global.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#else
  return *p;
#endif
}
__device__ __forceinline__ double4 far_ld_pos(const double4* p) { return ld_pos<AB_FAR_POS256 != 0>(p); }

template <typename R, bool MORSE>
struct FarPar {
  R e4a, e4b, s2a, s2b, c12a, c12b, c6a, c6b;  // 4 eps, sigma^2, 12 * 4 eps, 6 * 4 eps (Morse: eps, alpha, r_e, -)
  double rca, rcb, sha, shb, tva, tvb;
  int ti;
  __device__ __forceinline__ FarPar(int ti_) : ti(ti_) {
    const Tab<R>& T = tab<R>();
    e4a = MORSE ? T.meps[ti] : T.lj_e4[ti], e4b = MORSE ? T.meps[ti + 1] : T.lj_e4[ti + 1];
    s2a = MORSE ? T.malpha[ti] : T.sigma2[ti], s2b = MORSE ? T.malpha[ti + 1] : T.sigma2[ti + 1];
    c12a = MORSE ? T.mre[ti] : T.lj_c12[ti], c12b = MORSE ? T.mre[ti + 1] : T.lj_c12[ti + 1];
    c6a = T.lj_c6[ti], c6b = T.lj_c6[ti + 1];
    rca = c_geo.rc2[ti], rcb = c_geo.rc2[ti + 1];
    sha = c_geo.srhi2_hi[ti], shb = c_geo.srhi2_hi[ti + 1];
    tva = c_geo.tv2[ti], tvb = c_geo.tv2[ti + 1];  // taper vote: a little below r_lo^2
  }
};

// One far entry (a lane of a 32-entry chunk), branch-free except the taper: PURE = the chunk lies
// in the bins settled as "window-free, untapered, inside r_c" (warp-uniform; no decision taken);
// otherwise the exact (un-fused) window / cutoff decisions of the oracle, and the taper
// S(r; r_lo, r_c) (reading A10) when some lane of the warp is in the taper band.
// ENERGY = false (NVE steps whose energies / counters nobody reads): forces only.
template <typename R, bool VIRIAL, bool ENERGY, bool MORSE, bool SG>
__device__ __forceinline__ void far_entry(const FarPar<R, MORSE>& P, bool pure, bool valid, double4 pj, int J, int i,
                                          double4 pi, long long ki, const int* gid, const char4* shift,
                                          StageBuf stage, double& fx, double& fy, double& fz, double& en,
                                          double (&W)[6], unsigned& nlj, unsigned& ntp) {
  const bool hj = type_of(pj) != 0;
  const double dx = __dsub_rn(pj.x, pi.x), dy = __dsub_rn(pj.y, pi.y), dz = __dsub_rn(pj.z, pi.z);
  const double r2 = r2_exact(dx, dy, dz);
  const bool in = valid && (pure || (r2 >= (hj ? P.shb : P.sha) && r2 <= (hj ? P.rcb : P.rca)));
  const bool canon = ENERGY && ki < key_of(pj);
  if (ENERGY) nlj += (in && canon);
  // taper-band pairs (algorithmic flop count): counted by the virial (ab_compute) instantiation only
  if (VIRIAL) ntp += (in && canon && r2 > c_geo.rlo2[P.ti + (hj ? 1 : 0)]);
  const R rr2 = in ? (R)r2 : R(1);
  R dVr, V = R(0), s6 = R(0), c6 = R(0);
  if (MORSE) {
    const R y = rsqrt_fast(rr2);
    V = morse_plain<R>(hj ? P.e4b : P.e4a, hj ? P.s2b : P.s2a, hj ? P.c12b : P.c12a, rr2 * y, y, dVr);
  } else {
    // 1/r^2 from one hardware reciprocal + one Newton step (relative error ~1e-14, far below the
    // fp64 parity gate); c12 = 2 c6, so only sigma^2 and c6 = 24 eps are selected per species
    const R inv = rcp_nr1(rr2);
    const R sr2 = (hj ? P.s2b : P.s2a) * inv;
    s6 = sr2 * sr2 * sr2;
    c6 = hj ? P.c6b : P.c6a;
    dVr = c6 * (inv * (s6 * fma_r(R(-2), s6, R(1))));
    if (ENERGY) V = (c6 * R(1.0 / 6.0)) * fma_r(s6, s6, -s6);  // 4 eps (s6^2 - s6)
  }
  const bool tap = !pure && in && r2 > (hj ? P.tvb : P.tva);
  if (__any_sync(0xffffffffu, tap)) {  // (parameters from the constant bank: rare, off the register budget)
    const Tab<R>& T = tab<R>();
    const int pp = P.ti + (hj ? 1 : 0);
    if (!MORSE && !ENERGY) V = (c6 * R(1.0 / 6.0)) * fma_r(s6, s6, -s6);  // the taper's dS term
    const R y = rsqrt_nr1(rr2);
    const R r = rr2 * y;
    const R iv = T.inv_taper[pp];
    const R tt = (r - T.rlo[pp]) * iv;
    R sv, ds;
    halfcos_poly(tt < R(0) ? R(0) : tt, sv, ds);
    sv = tt <= R(0) ? R(1) : sv;
    ds = tt <= R(0) ? R(0) : ds * iv;
    dVr = dVr * sv + V * ds * y;
    V = V * sv;
  }
  dVr = in ? dVr : R(0);
  const R rx = (R)dx, ry = (R)dy, rz = (R)dz;
  fx = acc_round<SG>(fx + (double)(dVr * rx));
  fy = acc_round<SG>(fy + (double)(dVr * ry));
  fz = acc_round<SG>(fz + (double)(dVr * rz));
  if (ENERGY) en = acc_round<SG>(en + (double)(in ? V : R(0)));
  if (VIRIAL) {
    V3<R> dd = mk3<R>(rx, ry, rz);
    vir_add(W, dd, (R(0.5) * dVr) * dd);
  }
  if (VIRIAL && stage.rows && in && canon) stage_lj_row(stage, gid[i], gid[J], shift[J], 1.0, 0.0);
}

// the far row [s0, s3) as one stream of 32-entry chunks, FAR_UNROLL chunks per iteration (their
// gathers in flight together and their bodies interleaved, the next iteration's indices loaded
// one iteration ahead); a chunk entirely inside the PURE range [s1, s2) skips the decisions
template <typename R, bool VIRIAL, bool ENERGY, bool MORSE, bool SG>
__device__ __forceinline__ void far_row(const LJArgs& A, int i, int s0, int s1, int s2, int s3, double4 pi, int ti,
                                        long long ki, const int* gid, const char4* shift, StageBuf stage,
                                        double& fx, double& fy, double& fz, double& en, double (&W)[6],
                                        unsigned& nlj, unsigned& ntp) {
  if (s0 >= s3) return;
  const int lane = threadIdx.x & 31;
  const int* row = A.nbr[1] + (size_t)i * A.cap[1];
  const FarPar<R, MORSE> P(ti);
#if AB_FAR_PIPE
  // software pipeline one iteration deep: the next iteration's positions are in flight while this
  // one computes (indices two iterations ahead)
  constexpr int U = FAR_UNROLL;
  int Jc[U], Jn[U];
  double4 pn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int q = s0 + u * 32 + lane;
    Jc[u] = q < s3 ? row[q] : -1;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) pn[u] = A.pos[Jc[u] >= 0 ? Jc[u] : i];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int q = s0 + 32 * U + u * 32 + lane;
    Jn[u] = q < s3 ? row[q] : -1;
  }
  for (int base = s0; base < s3; base += 32 * U) {
    int J[U];
    double4 pj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) J[u] = Jc[u], pj[u] = pn[u];
#pragma unroll
    for (int u = 0; u < U; ++u) Jc[u] = Jn[u];
#pragma unroll
    for (int u = 0; u < U; ++u) pn[u] = A.pos[Jc[u] >= 0 ? Jc[u] : i];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = base + 64 * U + u * 32 + lane;
      Jn[u] = q < s3 ? row[q] : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c0 = base + 32 * u;
      far_entry<R, VIRIAL, ENERGY, MORSE, SG>(P, c0 >= s1 && c0 + 32 <= s2, J[u] >= 0, pj[u], J[u], i, pi, ki, gid,
                                              shift, stage, fx, fy, fz, en, W, nlj, ntp);
    }
  }
#else
  int Jn[FAR_UNROLL];
#pragma unroll
  for (int u = 0; u < FAR_UNROLL; ++u) {
    const int q = s0 + u * 32 + lane;
    Jn[u] = q < s3 ? far_ld_idx(row + q) : -1;
  }
#if AB_FAR_PJ
  // indices two iterations ahead, so the next iteration's partner positions can be prefetched
  // into L1 while this iteration computes (no registers held for them)
  int Jnn[FAR_UNROLL];
#pragma unroll
  for (int u = 0; u < FAR_UNROLL; ++u) {
    const int q = s0 + 32 * FAR_UNROLL + u * 32 + lane;
    Jnn[u] = q < s3 ? far_ld_idx(row + q) : -1;
  }
#endif
#if AB_FAR_TAIL
  // rows end anywhere inside an iteration of FAR_UNROLL chunks: the last <= FAR_TAIL chunks run as
  // one shorter iteration (their indices are already in Jn), so the empty chunks of the last full
  // iteration (1.5 of ~12 per row on cfg4) are not evaluated
  constexpr int FAR_TAIL = FAR_UNROLL / 2;
  int base = s0;
  for (; s3 - base > 32 * FAR_TAIL; base += 32 * FAR_UNROLL) {
#else
  for (int base = s0; base < s3; base += 32 * FAR_UNROLL) {
#endif
    int J[FAR_UNROLL];
    double4 pj[FAR_UNROLL];
#pragma unroll
    for (int u = 0; u < FAR_UNROLL; ++u) J[u] = Jn[u];
#pragma unroll
    for (int u = 0; u < FAR_UNROLL; ++u) pj[u] = far_ld_pos(A.pos + (J[u] >= 0 ? J[u] : i));
#if AB_FAR_PJ
#pragma unroll
    for (int u = 0; u < FAR_UNROLL; ++u) {
      Jn[u] = Jnn[u];
      if (Jn[u] >= 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(A.pos + Jn[u]));
    }
#pragma unroll
    for (int u = 0; u < FAR_UNROLL; ++u) {
      const int q = base + 64 * FAR_UNROLL + u * 32 + lane;
      Jnn[u] = q < s3 ? far_ld_idx(row + q) : -1;
    }
#else
#pragma unroll
    for (int u = 0; u < FAR_UNROLL; ++u) {
      const int q = base + 32 * FAR_UNROLL + u * 32 + lane;
      Jn[u] = q < s3 ? far_ld_idx(row + q) : -1;
    }
#endif
#pragma unroll
    for (int u = 0; u < FAR_UNROLL; ++u) {
      const int c0 = base + 32 * u;
      far_entry<R, VIRIAL, ENERGY, MORSE, SG>(P, c0 >= s1 && c0 + 32 <= s2, J[u] >= 0, pj[u], J[u], i, pi, ki, gid,
                                              shift, stage, fx, fy, fz, en, W, nlj, ntp);
    }
  }
#if AB_FAR_TAIL
  if (base < s3) {
    double4 pj[FAR_TAIL];
#pragma unroll
    for (int u = 0; u < FAR_TAIL; ++u) pj[u] = A.pos[Jn[u] >= 0 ? Jn[u] : i];
#pragma unroll
    for (int u = 0; u < FAR_TAIL; ++u) {
      const int c0 = base + 32 * u;
      far_entry<R, VIRIAL, ENERGY, MORSE, SG>(P, c0 >= s1 && c0 + 32 <= s2, Jn[u] >= 0, pj[u], Jn[u], i, pi, ki, gid,
                                              shift, stage, fx, fy, fz, en, W, nlj, ntp);
    }
  }
#endif
#endif
}

// warp-uniform segment bounds of atom i's far row: [s0, s1) tested, [s1, s2) PURE, [s2, s3) tested.
// D = displacement bound of every atom (kernel-uniform).  Bin counts in closed form: m carries a
// 1e-7 A margin, far above the rounding of the divisions, so every bin decision stays conservative.
__device__ __forceinline__ void far_segments(const LJArgs& A, int i, double4 pi, double D, int& s0, int& s1, int& s2,
                                             int& s3) {
  const int lane = threadIdx.x & 31;
  const int cnt = A.cnt[1][i];
  if (!A.binned) {
    s0 = s1 = s2 = 0, s3 = cnt;
    return;
  }
  const int endv = lane < FB_N ? (int)A.boff[(size_t)i * FB_STRIDE + lane] : cnt;
  auto start = [&](int b) {
    const int v = __shfl_sync(0xffffffffu, endv, b > 0 ? b - 1 : 0);
    return b > 0 ? v : 0;
  };
  const double4 xr = A.xref[i];
  const double ex = pi.x - xr.x, ey = pi.y - xr.y, ez = pi.z - xr.z;
  const double m = sqrt(ex * ex + ey * ey + ez * ez) + D + 1e-7, skin = A.skin;
  const double i2 = A.i2, i8 = A.i8;
  auto clamp8 = [](double x) { return x <= 0.0 ? 0 : (x >= 8.0 ? 8 : (int)x); };
  const int kL0 = clamp8(floor((skin - m) * i2));  // L bins with (k+1) skin/4 + m <= skin: below a_p
  const int kL1 = max(kL0, clamp8(ceil((skin + m) * i2)));  // first L bin with k skin/4 - m >= skin: above a_p
  const int kA = clamp8(floor((skin - m) * i8));   // A bins with (k+1) skin/8 + m <= skin: below r_lo
  const int kC = clamp8(ceil(m * i8));             // first C bin with k skin/8 - m >= 0: beyond r_c
  s0 = start(FB_L0 + kL0);
  s1 = start(FB_L0 + kL1);
  s2 = start(FB_A0 + kA);
  s3 = kC < 8 ? start(FB_C0 + kC) : cnt;
#ifdef AB_DEBUG_BOUNDS
  if (!(0 <= s0 && s0 <= s1 && s1 <= s2 && s2 <= s3 && s3 <= cnt && cnt <= A.cap[1]) && lane == 0) {
    printf("far_segments i=%d cnt=%d cap=%d s=%d %d %d %d k=%d %d %d %d m=%g D=%g ends:", i, cnt, A.cap[1], s0, s1, s2, s3,
           kL0, kL1, kA, kC, m, D);
    for (int t = 0; t < FB_N; ++t) printf(" %d", (int)A.boff[(size_t)i * FB_STRIDE + t]);
    printf("\n");
    __trap();
  }
#endif
}

template <typename R, bool VIRIAL, bool MORSE, bool SG = false, bool RANGED = false, bool ENERGY = true>
#ifndef AB_FAR_MINBLOCKS
#define AB_FAR_MINBLOCKS 6
#endif
__global__ void __launch_bounds__(128, AB_FAR_MINBLOCKS) k_lj_far(LJArgs A, const int* gid, const char4* shift, double* F, double* acc,
                                               unsigned long long* ct, StageBuf stage, RedRows RR) {
  __shared__ RedSmem rs;
  red_init(rs);
  const int lane = threadIdx.x & 31;
  double en = 0;
  double W[6] = {0, 0, 0, 0, 0, 0};
  unsigned nlj = 0, ntp = 0;
  unsigned long long ne = 0;
  const double D = A.dbound ? sqrt(__longlong_as_double((long long)*A.dbound)) : 0.5 * A.skin;
  // one atom's far row by this warp; inx = the atom this warp takes next (-1: none): its row is
  // requested now (a fresh DRAM stream whose first indices nothing else would have asked for
  // before the row starts), one 128-byte line per lane, as far as this row reaches
  auto atom = [&](int i, int inx) {
    const double4 pi = A.pos[i];
    const int ti = type_of(pi);
    const long long ki = key_of(pi);
    int s0, s1, s2, s3;
    far_segments(A, i, pi, D, s0, s1, s2, s3);
#if AB_FAR_PREF
    {
      const int off = lane * 32;
      if (inx >= 0 && off < s3 + 32 && off < A.cap[1]) {
        const int* q = A.nbr[1] + (size_t)inx * A.cap[1] + off;
#if AB_FAR_PREF == 2
        asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
#else
        asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
#endif
      }
    }
#endif
    double fx = 0, fy = 0, fz = 0;
    far_row<R, VIRIAL, ENERGY || VIRIAL, MORSE, SG>(A, i, s0, s1, s2, s3, pi, ti, ki, gid, shift, stage, fx, fy, fz, en, W, nlj, ntp);
    fx = warp_sum<SG>(fx);
    fy = warp_sum<SG>(fy);
    fz = warp_sum<SG>(fz);
    if (lane == 0) atomic_add3<SG>(F, i, fx, fy, fz);
    if (lane == 0) ne += (unsigned long long)(s3 - s0);
  };
#if AB_FAR_SMQ == 1
  // Per-SM queues: the cell-ordered atoms are cut into A.nq contiguous ranges of A.qper atoms;
  // every warp draws single atoms from the range of the SM it runs on (%smid), so all the warps
  // of an SM work through neighbouring atoms at the same time and their partner gathers meet in
  // that SM's L1.  A warp whose range is used up moves on to the next range that still has atoms
  // (ranges of SMs that received fewer blocks, e.g. beside a concurrent kernel, are finished by
  // the others).  Tickets are drawn two atoms ahead: the atomic's latency and the next row's
  // prefetch both hide behind the current row.
  if (!RANGED && A.smq) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    const int nq = A.nq, per = A.qper;
    int q = (int)(smid % (unsigned)nq);
    auto draw = [&]() {  // lane 0 holds the ticket
      int t = 0;
      if (lane == 0) t = atomicAdd(A.smq + q, 1);
      return t;
    };
    auto resolve = [&](int t) {  // ticket -> atom (-1: range used up)
      t = __shfl_sync(0xffffffffu, t, 0);
      const int i = q * per + t;
      return (t < per && i < A.N) ? i : -1;
    };
    int cur = resolve(draw());
    int nraw = draw();
    for (;;) {
      if (cur < 0) {  // this range is used up: the next range with atoms left (32 ranges per look)
        int found = -1;
        for (int o = 1; o < nq && found < 0; o += 32) {
          const int c = o + lane;
          const int qq = (q + c) % nq;
          const bool has = c < nq && *(volatile int*)(A.smq + qq) < min(per, A.N - qq * per);
          const unsigned m = __ballot_sync(0xffffffffu, has);
          if (m) found = (q + o + __ffs(m) - 1) % nq;
        }
        if (found < 0) break;
        q = found;
        cur = resolve(draw());
        nraw = draw();
        continue;
      }
      const int nxt = resolve(nraw);
      nraw = draw();
      atom(cur, nxt);
      cur = nxt;
    }
  } else
#endif
  // RANGED (slab interior / boundary split): the two atom ranges one after the other; otherwise
  // every atom (a separate instantiation: the range bookkeeping cost 6 % of the kernel on cfg4)
  for (int range = 0; range < (RANGED ? 2 : 1); ++range) {
    const int rb = RANGED ? (range ? A.r1b : A.r0b) : 0, re = RANGED ? (range ? A.r1e : A.r0e) : A.N;
#if AB_FAR_SWEEP
    // each block sweeps a contiguous (cell-ordered, hence compact) range of atoms with its warps
    // interleaved, so the neighbourhoods of successive atoms meet in the SM's L1
    const int per = (re - rb + gridDim.x - 1) / gridDim.x, wpb = blockDim.x >> 5;
    int bid = blockIdx.x;
#if AB_FAR_SMQ == 2
    // Block ranges drawn per SM: the gridDim.x block ranges are dealt to A.nq queues of
    // consecutive ranges, and a block takes the next range of the queue of the SM it runs on
    // (%smid), so the blocks resident on one SM sweep adjacent ranges and their partner gathers
    // meet in that SM's L1.  A block whose queue is used up takes a range of the next queue that
    // has one left; there are exactly as many ranges as blocks and every block takes exactly one.
    if (!RANGED && A.smq) {
      __shared__ int s_bid;
      if (threadIdx.x == 0) {
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        const int nq = A.nq, tpq = (gridDim.x + nq - 1) / nq;
        int q = (int)(smid % (unsigned)nq), got = -1;
        while (got < 0) {
          const int cntq = min(tpq, (int)gridDim.x - q * tpq);  // ranges of queue q (<= 0: none)
          if (cntq > 0 && *(volatile int*)(A.smq + q) < cntq) {
            const int t = atomicAdd(A.smq + q, 1);
            if (t < cntq) got = q * tpq + t;
          }
          q = q + 1 == nq ? 0 : q + 1;
        }
        s_bid = got;
      }
      __syncthreads();
      bid = s_bid;
    }
#endif
    const int b0 = rb + bid * per, b1 = min(re, b0 + per);
    for (int i = b0 + (threadIdx.x >> 5); i < b1; i += wpb) atom(i, i + wpb < b1 ? i + wpb : -1);
#else
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int i = rb + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < re; i += nwarps) atom(i, i + nwarps < re ? i + nwarps : -1);
#endif
  }
  red_add_d(rs, ACC_ELJ, 0.5 * en);
  if (VIRIAL)
    for (int c = 0; c < 6; ++c) red_add_d(rs, ACC_W + c, W[c]);
  red_add_u(rs, CT_LJ, (unsigned long long)nlj);
  red_add_u(rs, CT_LJFAR, (unsigned long long)nlj);
  red_add_u(rs, CT_LJTAPER, (unsigned long long)ntp);
  red_add_u(rs, CT_LJENT, ne);
  red_add_u(rs, CT_LJENTFAR, ne);
  red_flush(rs, RR);
}

}  // namespace ab
