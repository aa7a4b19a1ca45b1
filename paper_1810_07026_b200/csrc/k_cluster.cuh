// k_cluster.cuh -- j-clusters of the LJ pair loop (Alg. 3; lists by binning and a skin,
// P:261-291) laid out for coalesced loads on B200.
//
// Every atom instance (locals + ghost images) belongs to one cluster of up to CL_SIZE = 4 atoms:
// atoms are binned into xy columns (edge ~2.5 A over the padded region), split by species, sorted
// by z inside each (column, species) run and chopped into consecutive groups of 4 (the last
// group of a run padded with empty slots).  A cluster is therefore compact (~2.5 x 2.5 x 1.5 A)
// and of one species, so its LJ cutoff against a given centre atom is uniform.
//   cl_atom[4 c + s]  atom index of slot s of cluster c (-1: empty)
//   cpos[4 c + s]     copy of pos[cl_atom] refreshed every step (k_cpos): the 4 atoms of a
//                     cluster are one 128-byte line, so a warp reads 8 clusters in 8 lines
//                     instead of 32 scattered atoms
//   cbb[2 c], cbb[2 c + 1]  build-time bounding box (lo, hi; lo.w = species)
// Cluster lists (k_build_cl, one warp per local atom i): every cluster whose bounding box comes
// within r_c(t_i, t_c) + skin of atom i (positions at the build).  Atoms move less than skin/2
// between builds, so every pair with r <= r_c at any later step until the next
// rebuild has its cluster in the list.  The list is full (both directions): every pair is
// evaluated from both ends and the forces on i are a register sum (no scatter onto j).
#pragma once
#include "dev_common.cuh"
#include "k_lists.cuh"

namespace ab {

constexpr int CL_SIZE = 4;
constexpr int CL_RUNS_MAX = 32767;  // (column, species) runs: 15 bits of the 31-bit sort key

struct ClGrid {
  int ncx, ncy;
  double lo[3];   // padded region lower corner
  double cw[2];   // column edges (x, y)
  double zspan;   // padded z extent (16-bit z quantisation of the sort key)
};

__device__ __forceinline__ int cl_col(double v, double lo, double w, int n) {
  int c = (int)floor((v - lo) / w);
  return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

// sort keys: run = (column, species) and the quantised z inside the run (ties: atom index)
__global__ void k_cl_keys(int NT, const double4* pos, ClGrid g, int* run_of, int* zq_of) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= NT) return;
  const double4 p = pos[a];
  const int cx = cl_col(p.x, g.lo[0], g.cw[0], g.ncx), cy = cl_col(p.y, g.lo[1], g.cw[1], g.ncy);
  const int run = (cx * g.ncy + cy) * 2 + type_of(p);
  double zq = (p.z - g.lo[2]) / g.zspan * 65536.0;
  int z = (int)floor(zq);
  z = z < 0 ? 0 : (z > 65535 ? 65535 : z);
  run_of[a] = run;
  zq_of[a] = z;
}

// run_cl[r] = first cluster of run r (exclusive scan of ceil(len / 4)); run_cl[nrun] = clusters.
// One block of 1024 threads, nrun <= CL_RUNS_MAX.
__global__ void __launch_bounds__(1024) k_cl_run_scan(int nrun, const int* run_start, int* run_cl) {
  __shared__ int wsum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < nrun; base += 1024) {
    const int r = base + threadIdx.x;
    const int v = r < nrun ? (run_start[r + 1] - run_start[r] + CL_SIZE - 1) / CL_SIZE : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += u;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int y = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += u;
      }
      wsum[lane] = y;
    }
    __syncthreads();
    const int excl = carry + (w ? wsum[w - 1] : 0) + x - v;
    if (r < nrun) run_cl[r] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) run_cl[nrun] = carry;
}

__global__ void k_cl_fill(int NT, const int* run_of, const int* val2, const int* run_start, const int* run_cl,
                          int* cl_atom) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= NT) return;
  const int r = run_of[val2[q]];
  cl_atom[run_cl[r] * CL_SIZE + (q - run_start[r])] = val2[q];
}

// bounding boxes (build-time positions) and the empty-slot positions of cpos
__global__ void k_cl_bbox(int NC, const int* cl_atom, const double4* pos, double4* cbb, double4* cpos) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= NC) return;
  double4 lo = make_double4(1e300, 1e300, 1e300, 0.0), hi = make_double4(-1e300, -1e300, -1e300, 0.0);
  for (int s = 0; s < CL_SIZE; ++s) {
    const int a = cl_atom[CL_SIZE * c + s];
    if (a < 0) {  // far away and never in range (the list test also rejects a < 0)
      cpos[CL_SIZE * c + s] = make_double4(1e30, 1e30, 1e30, 0.0);
      continue;
    }
    const double4 p = pos[a];
    lo.x = fmin(lo.x, p.x), lo.y = fmin(lo.y, p.y), lo.z = fmin(lo.z, p.z);
    hi.x = fmax(hi.x, p.x), hi.y = fmax(hi.y, p.y), hi.z = fmax(hi.z, p.z);
    lo.w = (double)type_of(p);
  }
  cbb[2 * c] = lo, cbb[2 * c + 1] = hi;
}

// every step: cpos[s] = pos[cl_atom[s]] (current positions of locals and ghost images)
__global__ void k_cpos(int nslot, const int* cl_atom, const double4* pos, double4* cpos) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslot) return;
  const int a = cl_atom[s];
  if (a >= 0) cpos[s] = pos[a];
}

struct ClLists {
  int cap;
  int* cnt;
  int* nbr;
  double rcs[3];   // r_c(p) + skin (bounding-box test), with a rounding margin
  double bq2[3];   // (2^(1/6) sigma_p (1 + 1e-9) + skin)^2: canonical pairs that can become b*
  int* bqcnt;      // [3] bound of the b* candidate queue until the next build
};

constexpr int CL_MAXRUN = 512;  // (column, species) runs of one atom's stencil (2 x 15 x 15 max)

// One warp per local atom.  The candidate clusters of each (column, species) run of the culled
// column stencil form a contiguous z-range of the run (binary search on the bounding boxes);
// the ranges are flattened (prefix sums over 32 runs at a time) and streamed in chunks of 32,
// each lane testing one cluster's box.  Appends use warp-ballot compaction in stream order, so
// the list is deterministic.
__global__ void __launch_bounds__(128) k_build_cl(int N, const double4* pos, ClGrid g, const int* run_cl,
                                                  const double4* cbb, const int* cl_atom, ClLists L, int* maxcnt) {
  __shared__ int s_cb[4][CL_MAXRUN], s_pre[4][CL_MAXRUN + 1];
  const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= N) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double4 p = pos[a];
  const int ta = type_of(p);
  const long long ka = key_of(p);
  const double R0 = L.rcs[ta], R1 = L.rcs[ta + 1];  // against C / H clusters
  const double Rm = fmax(R0, R1);
  const int cx = cl_col(p.x, g.lo[0], g.cw[0], g.ncx), cy = cl_col(p.y, g.lo[1], g.cw[1], g.ncy);
  const int nx = (int)ceil(Rm / g.cw[0]) + 1, ny = (int)ceil(Rm / g.cw[1]) + 1;
  const int sx = 2 * nx + 1, sy = 2 * ny + 1;
  const int nrun = 2 * sx * sy;
  int* cb = s_cb[w];
  int* pre = s_pre[w];
  // 1. per run: the cluster range whose z-extent can reach [z - R', z + R']
  int total = 0;
  for (int r0 = 0; r0 < nrun; r0 += 32) {
    const int rr = r0 + lane;
    int beg = 0, len = 0;
    if (rr < nrun && rr < CL_MAXRUN) {
      const int t = rr & 1, col = rr >> 1;
      const int ax = cx - nx + col / sy, ay = cy - ny + col % sy;
      if (ax >= 0 && ax < g.ncx && ay >= 0 && ay < g.ncy) {
        const double x0 = g.lo[0] + ax * g.cw[0], y0 = g.lo[1] + ay * g.cw[1];
        const double dx = p.x < x0 ? x0 - p.x : (p.x > x0 + g.cw[0] ? p.x - (x0 + g.cw[0]) : 0.0);
        const double dy = p.y < y0 ? y0 - p.y : (p.y > y0 + g.cw[1] ? p.y - (y0 + g.cw[1]) : 0.0);
        const double R = t ? R1 : R0;
        const double d2 = dx * dx + dy * dy;
        if (d2 <= R * R) {
          const double hz = sqrt(R * R - d2) + 1e-6 + 2.0 * g.zspan / 65536.0;  // + z quantum margin
          const int run = (ax * g.ncy + ay) * 2 + t;
          int lo = run_cl[run], hi = run_cl[run + 1];
          // first cluster whose top reaches z - hz (tops are non-decreasing up to the z quantum)
          int b = lo, e = hi;
          while (b < e) {
            const int m = (b + e) >> 1;
            if (cbb[2 * m + 1].z < p.z - hz) b = m + 1;
            else e = m;
          }
          int b2 = b, e2 = hi;  // first cluster whose bottom is above z + hz
          while (b2 < e2) {
            const int m = (b2 + e2) >> 1;
            if (cbb[2 * m].z <= p.z + hz) b2 = m + 1;
            else e2 = m;
          }
          beg = b, len = b2 - b;
        }
      }
    }
    int v = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (rr < CL_MAXRUN) cb[rr] = beg, pre[rr] = total + v - len;
    total += __shfl_sync(0xffffffffu, v, 31);
  }
  const int nr_used = min(nrun, CL_MAXRUN);
  if (lane == 0) pre[nr_used] = total;
  __syncwarp();
  // 2. stream candidate clusters: box test, append, count possible b* pairs
  int n = 0, nq[3] = {0, 0, 0};
  int* row = L.nbr + (size_t)a * L.cap;
  int k = 0;
  for (int base = 0; base < total; base += 32) {
    const int f = base + lane;
    bool take = false;
    int c = -1;
    if (f < total) {
      while (pre[k + 1] <= f) ++k;
      c = cb[k] + f - pre[k];
      const double4 lo = cbb[2 * c], hi = cbb[2 * c + 1];
      const int tc = (int)lo.w;
      const double gx = fmax(fmax(lo.x - p.x, p.x - hi.x), 0.0);
      const double gy = fmax(fmax(lo.y - p.y, p.y - hi.y), 0.0);
      const double gz = fmax(fmax(lo.z - p.z, p.z - hi.z), 0.0);
      const double d2 = gx * gx + gy * gy + gz * gz;
      const double R = tc ? R1 : R0;
      take = d2 <= R * R;
      const int pr = ta + tc;
      if (take && d2 <= L.bq2[pr]) {
        for (int s = 0; s < CL_SIZE; ++s) {
          const int J = cl_atom[CL_SIZE * c + s];
          if (J < 0 || J == a) continue;
          const double4 pj = pos[J];
          const double r2 = r2_exact(__dsub_rn(pj.x, p.x), __dsub_rn(pj.y, p.y), __dsub_rn(pj.z, p.z));
          if (r2 <= L.bq2[pr] && ka < key_of(pj)) ++nq[pr];
        }
      }
    }
    warp_append(take, row, L.cap, n, c);
    k = __shfl_sync(0xffffffffu, k, 31);
  }
#pragma unroll
  for (int t = 0; t < 3; ++t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nq[t] += __shfl_xor_sync(0xffffffffu, nq[t], o);
  }
  if (lane == 0) {
    L.cnt[a] = n;
    atomicMax(maxcnt, n);
    for (int t = 0; t < 3; ++t)
      if (nq[t]) atomicAdd(L.bqcnt + t, nq[t]);
  }
}

}  // namespace ab
