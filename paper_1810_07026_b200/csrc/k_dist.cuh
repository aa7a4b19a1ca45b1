// k_dist.cuh -- spatial slab decomposition along x: ownership, migration at list
// rebuilds, the halo (ghost) selection, per-step halo position exchange and the reverse
// communication of ghost forces, plus the periodic-image ghosts that every domain builds itself.
//
// Domain r of n owns the atoms whose wrapped x lies in [xb(r), xb(r+1)), xb(r) = r L_x / n.
// Its ghosts are every atom instance (atom, image s) inside the padded region
//   [xb(r) - h, xb(r+1) + h) x [-h, L_y + h) x [-h, L_z + h),   h = r_c,max + skin,
// which covers the LJ partners, the C_ij paths (3 r_max), the b* neighbourhoods and complete
// short lists of every ghost those terms touch.  With slab width >= h the x part of
// the halo comes from the two neighbouring slabs only:
//   left ghosts  = atoms of domain r-1 with x >= xb(r) - h     (image s_x = -1 if r == 0)
//   right ghosts = atoms of domain r+1 with x <  xb(r+1) + h   (image s_x = +1 if r == n-1)
// and the y/z images of locals and x-ghosts are generated locally (explicit images).
// Every term is computed once globally: a pair / bond / quadruple belongs to its lower instance
// key (gid, image) -- the same rule as on one GPU, because the keys are global.
// Forces a domain scatters onto its x-ghosts are sent back to their owners and added there.
#pragma once
#include "dev_common.cuh"

namespace ab {

// slab geometry (host and device: plain IEEE operations, no contraction candidates)
__host__ __device__ __forceinline__ double slab_lo(int r, int n, double L) { return (double)r * L / (double)n; }
__host__ __device__ __forceinline__ int slab_of(double x, int n, double L) {
  int r = (int)floor(x * (double)n / L);
  r = r < 0 ? 0 : (r > n - 1 ? n - 1 : r);
  while (r > 0 && x < slab_lo(r, n, L)) --r;
  while (r < n - 1 && x >= slab_lo(r + 1, n, L)) ++r;
  return r;
}

// wrap every coordinate of the local atoms into [0, L) (same IEEE ops as k_wrap_and_key)
__device__ __forceinline__ double wrap1d(double x, double L) {
  double y = __dsub_rn(x, __dmul_rn(L, floor(__ddiv_rn(x, L))));
  if (y >= L) y = __dsub_rn(y, L);
  if (y < 0.0) y = __dadd_rn(y, L);
  return y;
}
__global__ void k_wrap(int N, double4* pos) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double4 p = pos[i];
  p.x = wrap1d(p.x, c_geo.L[0]);
  p.y = wrap1d(p.y, c_geo.L[1]);
  p.z = wrap1d(p.z, c_geo.L[2]);
  pos[i] = p;
}

// migration flags after the wrap: stay / to the left neighbour (channel 0) / to the right (1).
// With two domains left == right and channel 0 carries everything.  A destination that is not
// a neighbour (an atom crossed a whole slab between two rebuilds) is counted in *bad.
__global__ void k_mig_flags(int N, const double4* pos, int n, int rank, int* fstay, int* f0, int* f1,
                            unsigned long long* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int left = (rank + n - 1) % n, right = (rank + 1) % n;
  int d = slab_of(pos[i].x, n, c_geo.L[0]);
  fstay[i] = d == rank;
  f0[i] = d != rank && d == left;
  f1[i] = d != rank && d != left && d == right;
  if (d != rank && d != left && d != right) atomicAdd(bad, 1ull);
}

// migrant record: x y z key(bits) vx vy vz gid -- 8 doubles
__global__ void k_mig_pack(int cnt, const int* idx, const double4* pos, const double* vel, const int* gid,
                           double* out) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  int i = idx[q];
  double4 p = pos[i];
  double* o = out + 8 * (size_t)q;
  o[0] = p.x, o[1] = p.y, o[2] = p.z, o[3] = p.w;
  o[4] = vel[3 * i], o[5] = vel[3 * i + 1], o[6] = vel[3 * i + 2];
  o[7] = (double)gid[i];
}

// new local set: the stayers (in their current order) followed by the arrivals from the left
// channel, then from the right channel (deterministic)
__global__ void k_mig_assemble(int nstay, const int* stay, const double4* pos, const double* vel, const int* gid,
                               int nin0, const double* in0, int nin1, const double* in1, double4* pos_o,
                               double* vel_o, int* gid_o) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nstay) {
    int i = stay[q];
    pos_o[q] = pos[i];
    vel_o[3 * q] = vel[3 * i], vel_o[3 * q + 1] = vel[3 * i + 1], vel_o[3 * q + 2] = vel[3 * i + 2];
    gid_o[q] = gid[i];
    return;
  }
  q -= nstay;
  const double* r = nullptr;
  if (q < nin0) r = in0 + 8 * (size_t)q;
  else if (q - nin0 < nin1) r = in1 + 8 * (size_t)(q - nin0);
  else return;
  int o = nstay + q;
  pos_o[o] = make_double4(r[0], r[1], r[2], r[3]);
  vel_o[3 * o] = r[4], vel_o[3 * o + 1] = r[5], vel_o[3 * o + 2] = r[6];
  gid_o[o] = (int)r[7];
}

// halo membership of a local atom: near the left face -> channel 0, near the right face -> 1
__global__ void k_halo_flags(int N, const double4* pos, double xlo, double xhi, double h, int* f0, int* f1) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double x = pos[i].x;
  f0[i] = x < xlo + h;
  f1[i] = x >= xhi - h;
}

// per step: positions (with key) of the halo atoms into the two send buffers
__global__ void k_halo_pack(int ns0, const int* s0, int ns1, const int* s1, const double4* pos, double4* o0,
                            double4* o1) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < ns0) o0[q] = pos[s0[q]];
  else if (q - ns0 < ns1) o1[q - ns0] = pos[s1[q - ns0]];
}

// x image of a received halo atom: u = x + s L (bitwise the oracle's image), key + s
__device__ __forceinline__ double4 ximage(double4 p, int sx) {
  if (sx == 0) return p;
  long long key = key_of(p) + ((long long)sx << 18);
  return make_double4(__dadd_rn(p.x, __dmul_rn((double)sx, c_geo.L[0])), p.y, p.z, __longlong_as_double(key));
}

// per step: received halo positions into the x-ghost slots [N, N + nr0) (left) and
// [N + nr0, N + nr0 + nr1) (right)
__global__ void k_halo_unpack(int N, int nr0, const double4* in0, int sx0, int nr1, const double4* in1, int sx1,
                              double4* pos) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < nr0) pos[N + q] = ximage(in0[q], sx0);
  else if (q - nr0 < nr1) pos[N + q] = ximage(in1[q - nr0], sx1);
}

// rebuild: bookkeeping of the x-ghost slots (they are their own force owners; the reverse
// communication carries their forces home)
__global__ void k_xghost_meta(int N, int nr0, int sx0, int nr1, int sx1, const double4* pos, int* owner, int* gid,
                              char4* shift, char4* rshift) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nr0 + nr1) return;
  int a = N + q;
  owner[a] = a;
  gid[a] = (int)(key_of(pos[a]) >> 26);
  shift[a] = make_char4((signed char)(q < nr0 ? sx0 : sx1), 0, 0, 0);
  rshift[a] = make_char4(0, 0, 0, 0);
}

// per step: forces accumulated on the x-ghosts into the two send buffers (left ghosts go back to
// the left neighbour, right ghosts to the right one)
__global__ void k_force_pack(int N, int nr0, int nr1, const double* F, double4* o0, double4* o1) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nr0 + nr1) return;
  const double* f = F + 3 * (size_t)(N + q);
  double4 v = make_double4(f[0], f[1], f[2], 0.0);
  if (q < nr0) o0[q] = v;
  else o1[q - nr0] = v;
}

// per step: add the returned ghost forces to the owned atoms that were sent (one channel per
// launch, so an atom in both halo lists is updated in a fixed order)
__global__ void k_force_unpack(int ns, const int* sl, const double4* in, double* F) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ns) return;
  int i = sl[q];
  double4 v = in[q];
  F[3 * i] += v.x, F[3 * i + 1] += v.y, F[3 * i + 2] += v.z;
}

// ---- periodic images of the base atoms [0, NB) inside the padded region [lo, hi)
// (single domain: NB = N, all three directions; slab domain: NB = locals + x-ghosts, smax.x = 0)
__device__ __forceinline__ bool in_box(double u, double lo, double hi) { return u >= lo && u < hi; }

__global__ void k_image_count(int NB, const double4* pos, int3 smax, double3 lo, double3 hi, int* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NB) return;
  double4 p = pos[i];
  int c = 0;
  for (int sx = -smax.x; sx <= smax.x; ++sx) {
    double ux = __dadd_rn(p.x, __dmul_rn((double)sx, c_geo.L[0]));
    if (!in_box(ux, lo.x, hi.x)) continue;
    for (int sy = -smax.y; sy <= smax.y; ++sy) {
      double uy = __dadd_rn(p.y, __dmul_rn((double)sy, c_geo.L[1]));
      if (!in_box(uy, lo.y, hi.y)) continue;
      for (int sz = -smax.z; sz <= smax.z; ++sz) {
        if (sx == 0 && sy == 0 && sz == 0) continue;
        double uz = __dadd_rn(p.z, __dmul_rn((double)sz, c_geo.L[2]));
        if (in_box(uz, lo.z, hi.z)) ++c;
      }
    }
  }
  cnt[i] = c;
}

// first = slot of the first image; nloc = number of local atoms (their owner / shift are set
// here; x-ghost bases were set by k_xghost_meta)
__global__ void k_image_fill(int NB, int nloc, int first, double4* pos, int3 smax, double3 lo, double3 hi,
                             const int* off, int* owner, int* gid, char4* shift, char4* rshift) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NB) return;
  double4 p = pos[i];
  char4 sb = make_char4(0, 0, 0, 0);
  if (i < nloc) {
    owner[i] = i;
    shift[i] = sb;
    rshift[i] = sb;
  } else {
    sb = shift[i];
  }
  int w = first + off[i];
  int g = gid[i];
  for (int sx = -smax.x; sx <= smax.x; ++sx) {
    double ux = __dadd_rn(p.x, __dmul_rn((double)sx, c_geo.L[0]));
    if (!in_box(ux, lo.x, hi.x)) continue;
    for (int sy = -smax.y; sy <= smax.y; ++sy) {
      double uy = __dadd_rn(p.y, __dmul_rn((double)sy, c_geo.L[1]));
      if (!in_box(uy, lo.y, hi.y)) continue;
      for (int sz = -smax.z; sz <= smax.z; ++sz) {
        if (sx == 0 && sy == 0 && sz == 0) continue;
        double uz = __dadd_rn(p.z, __dmul_rn((double)sz, c_geo.L[2]));
        if (!in_box(uz, lo.z, hi.z)) continue;
        long long key = key_of(p) + ((long long)sx << 18) + ((long long)sy << 10) + ((long long)sz << 2);
        pos[w] = make_double4(ux, uy, uz, __longlong_as_double(key));
        owner[w] = i;
        gid[w] = g;
        shift[w] = make_char4((signed char)(sb.x + sx), (signed char)(sb.y + sy), (signed char)(sb.z + sz), 0);
        rshift[w] = make_char4((signed char)sx, (signed char)sy, (signed char)sz, 0);
        ++w;
      }
    }
  }
}

// per step: image ghosts [first, NT) follow their owner slot (a local or an x-ghost) by the
// relative image rshift (same IEEE ops as at creation)
__global__ void k_image_update(int first, int NT, double4* pos, const int* owner, const char4* rshift) {
  int g = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NT) return;
  double4 p = pos[owner[g]];
  char4 s = rshift[g];
  long long key = key_of(p) + ((long long)s.x << 18) + ((long long)s.y << 10) + ((long long)s.z << 2);
  pos[g] = make_double4(__dadd_rn(p.x, __dmul_rn((double)s.x, c_geo.L[0])),
                        __dadd_rn(p.y, __dmul_rn((double)s.y, c_geo.L[1])),
                        __dadd_rn(p.z, __dmul_rn((double)s.z, c_geo.L[2])), __longlong_as_double(key));
}

// global caller-order arrays of a domain's atoms (the other entries are left untouched)
__global__ void k_scatter_caller_pos(int N, const int* gid, const double4* pos, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int g = gid[i];
  double4 p = pos[i];
  out[3 * (size_t)g] = p.x, out[3 * (size_t)g + 1] = p.y, out[3 * (size_t)g + 2] = p.z;
}

// d2 bits and the short-list overflow flag of a domain into one 2-word vector (for a max
// all-reduce over the domains)
__global__ void k_flags2(const unsigned long long* ct, int ovf_slot, int d2_slot, unsigned long long* out) {
  out[0] = ct[d2_slot];
  out[1] = ct[ovf_slot];
}

}  // namespace ab
