// k_lists.cuh -- binning, periodic-image ghosts, skinned lists and the per-step exact short list.
//
// Paper: neighbour lists by binning, half-list convention, skin with
// rebuild when an atom moved too far, long list built by binning and short list
// derived from it, intermediate skinned short list refreshed into the exact short list
// every step.  B200 layout: positions double4 (x, y, z, type) for local atoms
// followed by ghost images; lists are per-atom fixed-stride int32 rows (atom a's entries at
// a*cap .. a*cap+cnt[a]-1), written in (stencil cell, sorted index) order, so every rebuild is
// deterministic.  All r^2 decisions use un-fused IEEE operations identical to the oracle's.
#pragma once
#include "dev_common.cuh"
#include <type_traits>

namespace ab {

struct Grid {
  int nc[3];
  double lo[3];  // lower corner of the padded region (= -halo)
  double cs[3];  // cell edge
};

__device__ __forceinline__ int cell_coord(double x, double lo, double cs, int n) {
  int c = (int)floor((x - lo) / cs);
  return c < 0 ? 0 : (c >= n ? n - 1 : c);
}
__device__ __forceinline__ int cell_of(double4 p, const Grid& g) {
  int cx = cell_coord(p.x, g.lo[0], g.cs[0], g.nc[0]);
  int cy = cell_coord(p.y, g.lo[1], g.cs[1], g.nc[1]);
  int cz = cell_coord(p.z, g.lo[2], g.cs[2], g.nc[2]);
  return (cx * g.nc[1] + cy) * g.nc[2] + cz;
}

// wrap x into [0, L): y = x - L floor(x/L); y >= L -> y -= L; y < 0 -> y += L
__device__ __forceinline__ double wrap1(double x, double L) {
  double y = __dsub_rn(x, __dmul_rn(L, floor(__ddiv_rn(x, L))));
  if (y >= L) y = __dsub_rn(y, L);
  if (y < 0.0) y = __dadd_rn(y, L);
  return y;
}

__global__ void k_wrap_and_key(int N, double4* pos, Grid g, int* key, int* val) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double4 p = pos[i];
  p.x = wrap1(p.x, c_geo.L[0]);
  p.y = wrap1(p.y, c_geo.L[1]);
  p.z = wrap1(p.z, c_geo.L[2]);
  pos[i] = p;
  key[i] = cell_of(p, g);
  val[i] = i;
}

// gather per-atom state into the new (cell-sorted) order
__global__ void k_permute(int N, const int* perm, const double4* pos_in, double4* pos_out, const double* v_in,
                          double* v_out, const int* gid_in, int* gid_out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int o = perm[i];
  pos_out[i] = pos_in[o];
  v_out[3 * i + 0] = v_in[3 * o + 0];
  v_out[3 * i + 1] = v_in[3 * o + 1];
  v_out[3 * i + 2] = v_in[3 * o + 2];
  gid_out[i] = gid_in[o];
}

// periodic images / slab halo ghosts: k_dist.cuh (k_image_*, k_halo_*)

__global__ void k_cell_keys(int NT, const double4* pos, Grid g, int* key, int* val) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= NT) return;
  key[a] = cell_of(pos[a], g);
  val[a] = a;
}

// cell_start (first sorted position of each cell): k_scan.cuh key_sort (counting sort)

// Skinned LJ lists of a local atom (full, both directions), split at build time by what the
// pair can need at evaluation time (atoms move < skin/2 between builds).  With
// a_p = 2^(1/6) sigma_p sqrt(1 + 1e-9) the radius of the S_r window pre-filter (r^2 < a_p^2: the
// pair may need b*) the evaluation splits the pairs by their CURRENT r^2:
//   r^2 <  a_p^2 : k_lj_near (C_ij from the reach set; C = 0 skipped, otherwise the b* batch)
//   r^2 >= a_p^2 : k_lj_far with C = 1; k_lj_near subtracts M V for the few pairs of its reach
//                  set that lie there (E = (1 - M) V = C V, P:467 / P:473-477).
// So the lists overlap in a shell of width 2 skin around a_p:
//   list 0 (near): r_b <= a_p + skin                  (all pairs that can be inside the window)
//   list 1 (far) : a_p - skin <= r_b <= r_c + skin    (all pairs that can be outside it)
//   list 2       : unused (count 0)
// The far row is ordered by distance bins of the build distance r_b, so the far kernel can skip,
// or evaluate without the taper / cutoff / window tests, the bins that the current displacement
// bound settles for the whole bin (FB_* below; edges relative to a_p, r_lo(p), r_c(p)):
//   L_k (k < 8) : the overlap shell, r_b in [a - skin + k skin/4, a - skin + (k+1) skin/4) (= list-0 members)
//   P           : a + skin < r_b < r_lo - skin      (always C = 1 zone, untapered: pure)
//   A_k (k < 8) : r_lo - skin + k skin/8 <= r_b < r_lo - skin + (k+1) skin/8
//   B           : r_lo <= r_b <= r_c
//   C_k (k < 8) : r_c + k skin/8 < r_b <= r_c + (k+1) skin/8
// Bins are filled in candidate order (stable counting sort per row), so rows are deterministic.
// boff[a * FB_STRIDE + b] = end offset of bin b in atom a's far row.
#ifndef AB_SHORT_POS256
#define AB_SHORT_POS256 1  // measured cfg4: k_short 0.2455 -> 0.2439 ms
#endif
#ifndef AB_BUILD_SEL
#define AB_BUILD_SEL 0
#endif
#ifndef AB_BUILD_POS256
#define AB_BUILD_POS256 1  // measured cfg4: rebuild 0.6764 -> 0.6731 ms per step
#endif
constexpr int FB_L0 = 0, FB_P = 8, FB_A0 = 9, FB_B = 17, FB_C0 = 18, FB_N = 26, FB_STRIDE = 32;

// One warp per atom; candidates stream over contiguous z-runs of the cell stencil.  Near entries
// are appended with warp-ballot compaction in candidate order (the paper's "inserting at once
// multiple elements into a single neighbor list"); far entries are staged in shared
// memory with their bin and written bin by bin.
struct LJLists {
  int cap[3];
  int* cnt[3];
  int* nbr[3];
  unsigned short* boff;  // far-row bin ends [N][FB_STRIDE]
  double flo2[3];  // (a_p - skin)^2 with a rounding margin (0 if a_p <= skin): lower end of the far list
  double fa[3];    // a_p
  double rlo[3], rc[3], rc2[3];
  double skin, ih2, ih8;  // skin, 4 / skin, 8 / skin (0 if skin = 0)
  double bq2[3];   // (a_p + skin)^2 with a rounding margin: the near list (canonical members bound the b* queue)
  int* bqcnt;      // [3] per species pair: bound of the b* candidate queue until the next build
  double reach;    // (r_c,max + skin) with a rounding margin: stencil culling radius
  double reach_t[2];  // the same per species of the listed atom (C: max r_c(CC, CH), H: max r_c(CH, HH))
  int fcap_smem;   // far entries staged per warp (= cap[1])
};

// Branch-free (the categories differ between the lanes of a chunk): every candidate bin is
// formed and the category selects one.  r = r2 rsqrt(r2) with two Newton steps (~1e-16 relative,
// far below the 1e-7 A margins of the evaluation-time bin classification); P (taken as untapered
// without a displacement test) keeps a 1e-9 A safety gap below r_lo - skin.
__device__ __forceinline__ int far_bin(const LJLists& Lg, int p, double r2, bool nearp) {
  const double r = r2 > 0.0 ? r2 * rsqrt_fast(r2) : 0.0, s = Lg.skin;
  auto kb = [](double x, double ih) {  // bin of x >= 0 in steps of 1/ih, clamped to [0, 7]
    const double k = x * ih;
    return k < 1.0 ? 0 : (k >= 7.0 ? 7 : (int)k);
  };
  const double rlo = Lg.rlo[p];
  const int bL = FB_L0 + kb(r - (Lg.fa[p] - s), Lg.ih2);
  const int bA = FB_A0 + kb(r - (rlo - s), Lg.ih8);
  const int bC = FB_C0 + kb(r - Lg.rc[p], Lg.ih8);
  const int bHi = r2 <= Lg.rc2[p] ? FB_B : bC;
  const int bFar = r < rlo - s - 1e-9 ? FB_P : (r < rlo ? bA : bHi);
  return nearp ? bL : bFar;
}

// Stencil culling: a column (ax, ay) of cells is scanned only over the z-range of cells that
// intersect the sphere of radius R around p (the full (2 nr + 1)^3 cube scans ~3x the sphere).
// Conservative: R carries a margin, so no cell holding a partner within the list cutoff is missed.
__device__ __forceinline__ bool column_range(const Grid& g, double4 p, int ax, int ay, double R, int& z0, int& z1) {
  const double x0 = g.lo[0] + ax * g.cs[0], y0 = g.lo[1] + ay * g.cs[1];
  const double dx = p.x < x0 ? x0 - p.x : (p.x > x0 + g.cs[0] ? p.x - (x0 + g.cs[0]) : 0.0);
  const double dy = p.y < y0 ? y0 - p.y : (p.y > y0 + g.cs[1] ? p.y - (y0 + g.cs[1]) : 0.0);
  const double d2 = dx * dx + dy * dy;
  if (d2 > R * R) return false;
  const double hz = sqrt(R * R - d2);
  z0 = cell_coord(p.z - hz, g.lo[2], g.cs[2], g.nc[2]);
  z1 = cell_coord(p.z + hz, g.lo[2], g.cs[2], g.nc[2]);
  return true;
}

__device__ __forceinline__ void warp_append(bool take, int* row, int cap, int& n, int b) {
  unsigned m = __ballot_sync(0xffffffffu, take);
  if (take) {
    int slot = n + __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
    if (slot < cap) row[slot] = b;
  }
  n += __popc(m);
}

// The culled stencil of atom p flattened for one warp: column k (x-major, then y -- the scan
// order of the lists) holds candidates [cb[k], cb[k] + pre[k+1] - pre[k]) of the cell-sorted
// index.  The column bounds are computed 32 columns at a time (independent loads), instead of
// one dependent cell_start read per column, and candidates are then streamed in full chunks of
// 32 across column boundaries.  Returns the candidate count; needs (2 nr + 1)^2 <= STENCIL_MAXCOL.
constexpr int STENCIL_MAXCOL = 128;
__device__ __forceinline__ int stencil_columns(const Grid& g, double4 p, int nr, double R, const int* cell_start,
                                               int* cb, int* pre) {
  const int lane = threadIdx.x & 31;
  const int cx = cell_coord(p.x, g.lo[0], g.cs[0], g.nc[0]);
  const int cy = cell_coord(p.y, g.lo[1], g.cs[1], g.nc[1]);
  const int cz = cell_coord(p.z, g.lo[2], g.cs[2], g.nc[2]);
  const int z0 = max(0, cz - nr), z1 = min(g.nc[2] - 1, cz + nr);
  const int side = 2 * nr + 1, ncol = side * side;
  int run = 0;
  for (int c0 = 0; c0 < ncol; c0 += 32) {
    const int col = c0 + lane;
    int beg = 0, len = 0;
    if (col < ncol) {
      const int ax = cx - nr + col / side, ay = cy - nr + col % side;
      int zc0, zc1;
      if (ax >= 0 && ax < g.nc[0] && ay >= 0 && ay < g.nc[1] && column_range(g, p, ax, ay, R, zc0, zc1)) {
        zc0 = max(zc0, z0), zc1 = min(zc1, z1);
        const int c = (ax * g.nc[1] + ay) * g.nc[2];
        beg = cell_start[c + zc0];
        len = max(cell_start[c + zc1 + 1] - beg, 0);
      }
    }
    int v = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (col < ncol) cb[col] = beg, pre[col] = run + v - len;
    run += __shfl_sync(0xffffffffu, v, 31);
  }
  if (lane == 0) pre[ncol] = run;
  __syncwarp();
  return run;
}

// candidate f of the flattened stencil, scanning forward from column k (k <= f's column): its
// position in the cell-sorted order (cell_atoms[s] = atom index, spos[s] = its position: a
// column's z-run of candidates is contiguous there, so a warp's 32 candidates are ~8 lines)
__device__ __forceinline__ int stencil_at(const int* cb, const int* pre, int f, int& k) {
  while (pre[k + 1] <= f) ++k;
  return cb[k] + f - pre[k];
}

// positions in the cell-sorted order of the last binning (list builds)
__global__ void k_sorted_pos(int NT, const int* cell_atoms, const double4* pos, double4* spos) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < NT) spos[q] = pos[cell_atoms[q]];
}

#ifndef AB_BUILD_MINBLOCKS
#define AB_BUILD_MINBLOCKS 1
#endif
__global__ void __launch_bounds__(128, AB_BUILD_MINBLOCKS) k_build_lj(int N, const double4* pos, const double4* spos, Grid g,
                                                  const int* cell_start, const int* cell_atoms, int nr, LJLists Lg,
                                                  int* maxcnt) {
  __shared__ int s_cb[4][STENCIL_MAXCOL], s_pre[4][STENCIL_MAXCOL + 1];
  __shared__ int s_hist[4][FB_N + 1];
  extern __shared__ int s_dyn[];  // per warp: fcap_smem indices, then fcap_smem bin bytes
  int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= N) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int fcap = Lg.fcap_smem;
  int* fJ = s_dyn + (size_t)w * ((fcap + 3) / 4) * 5;
  unsigned char* fB = reinterpret_cast<unsigned char*>(fJ + fcap);
  const double4 p = pos[a];
  const int ta = type_of(p);
  int n0 = 0, nf = 0;
  int nq[3] = {0, 0, 0};
  const long long ka = key_of(p);
  int* row0 = Lg.nbr[0] + (size_t)a * Lg.cap[0];
  int* cb = s_cb[w];
  int* pre = s_pre[w];
  int* hist = s_hist[w];
  if (lane <= FB_N) hist[lane] = 0;
  const int total = stencil_columns(g, p, nr, Lg.reach_t[ta], cell_start, cb, pre);
#if AB_BUILD_SEL
  const double rcs_a = c_geo.rc_s2[ta], rcs_b = c_geo.rc_s2[ta + 1], bq_a = Lg.bq2[ta], bq_b = Lg.bq2[ta + 1];
  const double flo_a = Lg.flo2[ta], flo_b = Lg.flo2[ta + 1];
#endif
  int k = 0;  // column of the chunk's first candidate (warp-uniform)
  // software pipeline: the next chunk's index and position loads are in flight while this
  // chunk is classified and appended
  int sq = lane < total ? stencil_at(cb, pre, lane, k) : -1;
  int b = sq >= 0 ? cell_atoms[sq] : -1;
  double4 pb = sq >= 0 ? ld_pos<AB_BUILD_POS256 != 0>(spos + sq) : make_double4(0, 0, 0, 0);
  for (int base = 0; base < total; base += 32) {
    int kn = __shfl_sync(0xffffffffu, k, 31);
    const int fn = base + 32 + lane;
    const int sqn = fn < total ? stencil_at(cb, pre, fn, kn) : -1;
    const int bn = sqn >= 0 ? cell_atoms[sqn] : -1;
    const double4 pbn = sqn >= 0 ? ld_pos<AB_BUILD_POS256 != 0>(spos + sqn) : make_double4(0, 0, 0, 0);
    const bool ok = b >= 0 && b != a;
    double r2 = 1e300;
    int pr = 0;
    if (ok) {
      r2 = r2_exact(__dsub_rn(pb.x, p.x), __dsub_rn(pb.y, p.y), __dsub_rn(pb.z, p.z));
      pr = ta + type_of(pb);
    }
#if AB_BUILD_SEL
    // the atom's species is warp-uniform, so the pair's is one of two: selects from registers
    // instead of constant-bank loads indexed per lane (replayed per distinct address)
    const bool hb = pr != ta;
    const bool in = ok && r2 <= (hb ? rcs_b : rcs_a);
    const bool nearp = in && r2 <= (hb ? bq_b : bq_a);
    const bool farp = in && r2 >= (hb ? flo_b : flo_a);
#else
    const bool in = ok && r2 <= c_geo.rc_s2[pr];
    const bool nearp = in && r2 <= Lg.bq2[pr];
    const bool farp = in && r2 >= Lg.flo2[pr];
#endif
    warp_append(nearp, row0, Lg.cap[0], n0, b);
    {  // stage far entries with their bin (candidate order) and count them per bin
      const unsigned m = __ballot_sync(0xffffffffu, farp);
      const int slot = nf + __popc(m & ((1u << lane) - 1u));
      if (farp && slot < fcap) {
        const int bin = far_bin(Lg, pr, r2, nearp);
        fJ[slot] = b, fB[slot] = (unsigned char)bin;
        atomicAdd(&hist[bin], 1);
      }
      nf += __popc(m);
    }
    const bool bq = nearp && ka < key_of(pb);
#pragma unroll
    for (int t = 0; t < 3; ++t) nq[t] += __popc(__ballot_sync(0xffffffffu, bq && pr == t));
    b = bn, pb = pbn, k = kn;
  }
  __syncwarp();
  // bin ends (inclusive scan of the histogram) and the stable scatter of the staged entries
  const int nfs = min(nf, fcap);
  if (nf <= Lg.cap[1]) {
    int hv = lane < FB_N ? hist[lane] : 0;
    int incl = hv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane < FB_N) Lg.boff[(size_t)a * FB_STRIDE + lane] = (unsigned short)incl;
#ifdef AB_DEBUG_BOUNDS
    {
      const int last = __shfl_sync(0xffffffffu, incl, FB_N - 1);
      const int prev = __shfl_up_sync(0xffffffffu, incl, 1);
      const bool bad = (lane > 0 && lane < FB_N && incl < prev) || last != nfs;
      if (__any_sync(0xffffffffu, bad) && lane == 0) {
        printf("k_build_lj a=%d nf=%d nfs=%d last=%d hist:", a, nf, nfs, last);
        for (int t = 0; t < FB_N; ++t) printf(" %d", hist[t]);
        printf("\n");
      }
    }
#endif
    __syncwarp();
    if (lane < FB_N) hist[lane] = incl - hv;  // running cursor per bin
    __syncwarp();
    int* row1 = Lg.nbr[1] + (size_t)a * Lg.cap[1];
    for (int c0 = 0; c0 < nfs; c0 += 32) {
      const int q = c0 + lane;
      const int bin = q < nfs ? (int)fB[q] : FB_N + lane;  // out-of-range lanes in groups of their own
      const unsigned grp = __match_any_sync(0xffffffffu, bin);
      const int rank = __popc(grp & ((1u << lane) - 1u));
      if (q < nfs) row1[hist[bin] + rank] = fJ[q];
      __syncwarp();
      if (q < nfs && rank == 0) atomicAdd(&hist[bin], __popc(grp));
      __syncwarp();
    }
  }
  if (lane == 0) {
    Lg.cnt[0][a] = n0;
    Lg.cnt[1][a] = nf;
    Lg.cnt[2][a] = 0;
    atomicMax(maxcnt + 0, n0);
    atomicMax(maxcnt + 1, nf);
    for (int c = 0; c < 3; ++c)
      if (nq[c]) atomicAdd(Lg.bqcnt + c, nq[c]);
  }
}

// intermediate REBO list: all atoms (locals + ghosts), r_b <= r_max(p) + skin
__global__ void __launch_bounds__(128) k_build_inter(int NT, const double4* pos, const double4* spos, Grid g,
                                                     const int* cell_start, const int* cell_atoms, int nr, double reach,
                                                     int cap, int* cnt, int* nbr, int* maxcnt) {
  __shared__ int s_cb[4][STENCIL_MAXCOL], s_pre[4][STENCIL_MAXCOL + 1];
  int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= NT) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double4 p = pos[a];
  const int ta = type_of(p);
  int n = 0;
  int* row = nbr + (size_t)a * cap;
  int* cb = s_cb[w];
  int* pre = s_pre[w];
  const int total = stencil_columns(g, p, nr, reach, cell_start, cb, pre);
  int k = 0;
  for (int base = 0; base < total; base += 32) {
    const int f = base + lane;
    const int sq = f < total ? stencil_at(cb, pre, f, k) : -1;
    const int b = sq >= 0 ? cell_atoms[sq] : -1;
    bool in = false;
    if (b >= 0 && b != a) {
      const double4 pb = ld_pos<AB_BUILD_POS256 != 0>(spos + sq);
      const double r2 = r2_exact(__dsub_rn(pb.x, p.x), __dsub_rn(pb.y, p.y), __dsub_rn(pb.z, p.z));
      in = r2 <= c_geo.rmax_s2[ta + type_of(pb)];
    }
    warp_append(in, row, cap, n, b);
    k = __shfl_sync(0xffffffffu, k, 31);
  }
  if (lane == 0) {
    cnt[a] = n;
    atomicMax(maxcnt, n);
  }
}

// Short-list storage: per atom up to capS entries: neighbour index, (d, r) and (w, dw/dr).
template <typename R>
struct ShortList {
  int capS;
  int* cnt;
  int* nbr;
  typename std::conditional<sizeof(R) == 8, double4, float4>::type* dr;  // d.x d.y d.z r
  typename std::conditional<sizeof(R) == 8, double2, float2>::type* w;   // w, dw/dr
  double* wd;  // w in fp64 in both modes: the C_ij gate (M = max path product, C = 1 - M) is a
               // gate decision (reading A14); near w = 1 an fp32 w would round M to 1
  R* Ntot;  // N_a = N^C_a + N^H_a
  R* NC;
  R* NH;
};

template <typename R>
__device__ __forceinline__ V3<R> sl_d(const ShortList<R>& S, int a, int n, R& r) {
  auto v = S.dr[(size_t)a * S.capS + n];
  r = v.w;
  return mk3<R>(v.x, v.y, v.z);
}

// REBO half bonds in three regions by species pair (CC, CH, HH), so that the warps of the bond
// kernel run uniform neighbour loops (species-sorted bond batches).
struct BondList {
  int2* b;    // region t at b + t * cap: (i, slot in N(i))
  int* cnt;   // [3]
  int cap;    // per region (>= canonical short-list entries of the owned atoms)
};

// Exact short list every step: filter the intermediate list at r <= r_max
// (closed boundary), store d, r, w = S(r; r_min, r_max), dw/dr; N^C, N^H per atom.
// Local atoms also append their canonical entries to the REBO bond list of the species pair.
#ifndef AB_SHORT_BATCH
#define AB_SHORT_BATCH 4  // measured (cfg2 k_short): 4 -> 20.0 us, 8 -> 24.9, 12 -> 31.2, 16 -> 32.7; 1-ahead pipeline 24.2
#endif
constexpr int SHORT_BATCH = AB_SHORT_BATCH;
template <typename R>
__global__ void k_short(int N, int NT, const double4* pos, const int* in_cnt, const int* in_nbr, int capI,
                        ShortList<R> S, const int* gid, const char4* shift, BondList BL, unsigned long long* ct,
                        RedRows RR) {
  __shared__ RedSmem rs;
  __shared__ int s_bn[3], s_bb[3];  // block bond counts / global bases per species pair
  if (threadIdx.x < 3) s_bn[threadIdx.x] = 0;
  red_init(rs);
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  bool live = a < NT;
  int nloc = 0, nbond[3] = {0, 0, 0};
  unsigned cmask = 0, hmask = 0;  // canonical entries / H partners by slot (capS <= NBMAX = 16)
  if (live) {
    const Tab<R>& T = tab<R>();
    double4 p = pos[a];
    int ta = type_of(p);
    long long ka = key_of(p);
    int n = 0;
    R nc = 0, nh = 0;
    int ci = in_cnt[a];
    size_t base = (size_t)a * S.capS;
    const int* row = in_nbr + (size_t)a * capI;
    // candidates in batches of SHORT_BATCH: all indices, then all positions of a batch are in
    // flight together (two memory latencies per batch instead of one per candidate); processed
    // in list order, so the entries and the N sums are those of a serial walk
    for (int q0 = 0; q0 < ci; q0 += SHORT_BATCH) {
    int bq[SHORT_BATCH];
    double4 pq[SHORT_BATCH];
#pragma unroll
    for (int u = 0; u < SHORT_BATCH; ++u) bq[u] = q0 + u < ci ? row[q0 + u] : a;
#pragma unroll
    for (int u = 0; u < SHORT_BATCH; ++u) pq[u] = ld_pos<AB_SHORT_POS256 != 0>(pos + bq[u]);
#pragma unroll
    for (int u = 0; u < SHORT_BATCH; ++u) {
      if (q0 + u >= ci) break;
      const int b = bq[u];
      const double4 pb = pq[u];
      double dx = __dsub_rn(pb.x, p.x), dy = __dsub_rn(pb.y, p.y), dz = __dsub_rn(pb.z, p.z);
      double r2 = r2_exact(dx, dy, dz);
      int tb = type_of(pb);
      int pr = ta + tb;
      if (r2 <= c_geo.rmax2[pr]) {
        if (n < S.capS) {
          double r = sqrt(r2);
          R dw;
          R w = sw<R>((R)r, T.rmin[pr], T.rmax[pr], dw);
          double dwd;
          S.wd[base + n] = sizeof(R) == 8 ? (double)w : sw<double>(r, c_tabd.rmin[pr], c_tabd.rmax[pr], dwd);
          S.nbr[base + n] = b;
          S.dr[base + n] = {(R)dx, (R)dy, (R)dz, (R)r};
          S.w[base + n] = {w, dw};
          if (tb == 0) nc += w;
          else nh += w;
          if (a < N && ka < key_of(pb)) ++nbond[pr], cmask |= 1u << n;
          if (tb != 0) hmask |= 1u << n;
        }
        ++n;
      }
    }
    }
    if (n > S.capS) atomicAdd(ct + CT_OVF_SHORT, 1ull);
    n = min(n, S.capS);
    S.cnt[a] = n;
    S.NC[a] = nc;
    S.NH[a] = nh;
    S.Ntot[a] = nc + nh;
    if (a < N) nloc = n;
  }
  // bond list compaction per species pair: warp scan, one shared atomic per warp, one global
  // atomic per block (order within a region is irrelevant to the physics)
  unsigned lane = threadIdx.x & 31;
  int w[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    int incl = nbond[t];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += v;
    }
    int total = __shfl_sync(0xffffffffu, incl, 31);
    int basew = 0;
    if (lane == 31 && total) basew = atomicAdd(&s_bn[t], total);
    basew = __shfl_sync(0xffffffffu, basew, 31);
    w[t] = basew + incl - nbond[t];
  }
  __syncthreads();
  if (threadIdx.x < 3) s_bb[threadIdx.x] = s_bn[threadIdx.x] ? atomicAdd(BL.cnt + threadIdx.x, s_bn[threadIdx.x]) : 0;
  __syncthreads();
  if (cmask) {
    const int ta = type_of(pos[a]);
    for (int t = 0; t < 3; ++t) w[t] += s_bb[t];
    for (unsigned m = cmask; m; m &= m - 1) {
      const int q = __ffs(m) - 1;
      const int t = ta + ((hmask >> q) & 1u);
      BL.b[(size_t)t * BL.cap + w[t]++] = make_int2(a, q);
    }
  }
  red_add_u(rs, CT_SHORT, (unsigned long long)nloc);
  red_max_u(rs, CT_MAXSHORT, (unsigned long long)nloc);
  red_flush(rs, RR);
}

}  // namespace ab
