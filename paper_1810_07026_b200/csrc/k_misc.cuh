// k_misc.cuh -- velocity-Verlet NVE, skin-displacement trigger,
// kinetic energy, and caller-order <-> cell-sorted-order transfers.
#pragma once
#include "dev_common.cuh"

namespace ab {

// block-wide max of non-negative doubles, one atomic per block (bit-pattern order == value order)
__device__ __forceinline__ void block_max_atomic(double v, unsigned long long* out, unsigned long long* out2 = nullptr) {
  __shared__ double sm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? sm[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0 && v > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(v));
    if (out2 && l == 0 && v > 0.0) atomicMax(out2, (unsigned long long)__double_as_longlong(v));
  }
}

// one velocity-Verlet half-kick / drift component.  r32 = AB_REDUCED (the paper's single precision
// with the dynamical state in binary32, reading A35): both operations rounded to binary32 (no FMA)
__device__ __forceinline__ double kick(double v, double dtf, double f, bool r32) {
  if (r32) return (double)__fadd_rn((float)v, __fmul_rn((float)dtf, (float)f));
  return v + dtf * f;
}
__device__ __forceinline__ double drift(double x, double dt, double v, bool r32) {
  if (r32) return (double)__fadd_rn((float)x, __fmul_rn((float)dt, (float)v));
  return x + dt * v;
}

// v += dt/2 F/m ftm2v;  x += dt v;  max |x - x_ref|^2 since the last list build
__global__ void k_integrate1(int N, double4* pos, double* v, const double* F, double dtf0, double dtf1, double dt,
                             const double4* xref, unsigned long long* maxd2, unsigned long long* dbound, bool r32) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (i < N) {
    double4 p = pos[i];
    double dtf = (type_of(p) == 0) ? dtf0 : dtf1;
    double vx = kick(v[3 * i + 0], dtf, F[3 * i + 0], r32);
    double vy = kick(v[3 * i + 1], dtf, F[3 * i + 1], r32);
    double vz = kick(v[3 * i + 2], dtf, F[3 * i + 2], r32);
    v[3 * i + 0] = vx, v[3 * i + 1] = vy, v[3 * i + 2] = vz;
    p.x = drift(p.x, dt, vx, r32), p.y = drift(p.y, dt, vy, r32), p.z = drift(p.z, dt, vz, r32);
    pos[i] = p;
    double4 r = xref[i];
    double dx = p.x - r.x, dy = p.y - r.y, dz = p.z - r.z;
    d2 = dx * dx + dy * dy + dz * dz;
  }
  block_max_atomic(d2, maxd2, dbound);
}

// Rebuild flags straight to the host: the last block to finish (ticket) copies the maximal
// displacement and the short-list overflow flag of the previous evaluation into mapped pinned
// host memory, then zeroes the scratch block (energies, counters, small ints, the displacement)
// for the next evaluation.  Replaces a memset before the kernel, a device-to-host copy and a
// memset after it, all three serial steps on the engine stream.
struct FlagOut {
  unsigned long long* host;   // mapped pinned: [CT_N + 1] slots, only host[ovf] and host[CT_N] written
  unsigned int* ticket;       // device counter, 0 between launches
  unsigned long long* zero;   // scratch block to zero (device), nzero 64-bit words
  int nzero, ovf;             // ovf: column of the overflow flag in ct
  const unsigned long long* ct;
};
__device__ __forceinline__ void publish_flags(const FlagOut& fo, unsigned long long* maxd2) {
  __shared__ bool last;
  // thread 0 issued the block's atomicMax (block_max_atomic): it fences, then takes the ticket
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(fo.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    volatile unsigned long long* h = fo.host;
    h[CT_N] = *(volatile unsigned long long*)maxd2;
    h[fo.ovf] = *(volatile const unsigned long long*)(fo.ct + fo.ovf);
    *fo.ticket = 0u;  // (the host reads h after the kernel's completion event: no system fence)
  }
  __syncthreads();
  for (int w = threadIdx.x; w < fo.nzero; w += blockDim.x) fo.zero[w] = 0ull;
}

// Whole-box NVE: k_integrate1 + the image-ghost refresh (k_image_update) + the zeroing of F
// for the next evaluation in one pass.  Atom i writes its own periodic images, which the last
// rebuild laid out contiguously at NB + goff[i] (k_image_fill), with k_image_update's operations.
__global__ void k_integrate1_img(int N, double4* pos, double* v, double* F, bool pre, double pd0, double pd1,
                                 double dtf0, double dtf1, double dt,
                                 const double4* xref, unsigned long long* maxd2, unsigned long long* dbound, int NB,
                                 const int* goff, const int* gcnt, const char4* rshift, FlagOut fo, bool r32) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (i < N) {
    // every load first (the stores below could alias them for the compiler): one memory
    // latency for the atom and its first IMG_PRE image shifts instead of a dependent chain
    constexpr int IMG_PRE = 4;
    double4 p = pos[i];
    const double v0 = v[3 * i + 0], v1 = v[3 * i + 1], v2 = v[3 * i + 2];
    const double f0 = F[3 * i + 0], f1 = F[3 * i + 1], f2 = F[3 * i + 2];
    const double4 r = xref[i];
    const int g0 = NB + goff[i], ng = gcnt[i];
    char4 sh[IMG_PRE];
#pragma unroll
    for (int k = 0; k < IMG_PRE; ++k) sh[k] = k < ng ? rshift[g0 + k] : make_char4(0, 0, 0, 0);
    double dtf = (type_of(p) == 0) ? dtf0 : dtf1;
    double u0 = v0, u1 = v1, u2 = v2;
    if (pre) {  // the previous step's deferred second half-kick (k_integrate2's operations)
      const double pdtf = (type_of(p) == 0) ? pd0 : pd1;
      u0 = kick(v0, pdtf, f0, r32), u1 = kick(v1, pdtf, f1, r32), u2 = kick(v2, pdtf, f2, r32);
    }
    double vx = kick(u0, dtf, f0, r32);
    double vy = kick(u1, dtf, f1, r32);
    double vz = kick(u2, dtf, f2, r32);
    F[3 * i + 0] = 0.0, F[3 * i + 1] = 0.0, F[3 * i + 2] = 0.0;
    v[3 * i + 0] = vx, v[3 * i + 1] = vy, v[3 * i + 2] = vz;
    p.x = drift(p.x, dt, vx, r32), p.y = drift(p.y, dt, vy, r32), p.z = drift(p.z, dt, vz, r32);
    pos[i] = p;
    double dx = p.x - r.x, dy = p.y - r.y, dz = p.z - r.z;
    d2 = dx * dx + dy * dy + dz * dz;
    auto image = [&](int g, char4 s) {
      const long long key = key_of(p) + ((long long)s.x << 18) + ((long long)s.y << 10) + ((long long)s.z << 2);
      pos[g] = make_double4(__dadd_rn(p.x, __dmul_rn((double)s.x, c_geo.L[0])),
                            __dadd_rn(p.y, __dmul_rn((double)s.y, c_geo.L[1])),
                            __dadd_rn(p.z, __dmul_rn((double)s.z, c_geo.L[2])), __longlong_as_double(key));
    };
#pragma unroll
    for (int k = 0; k < IMG_PRE; ++k)
      if (k < ng) image(g0 + k, sh[k]);
    for (int k = IMG_PRE; k < ng; ++k) image(g0 + k, rshift[g0 + k]);
  }
  block_max_atomic(d2, maxd2, dbound);
  if (fo.host) publish_flags(fo, maxd2);
}

// AB_SINGLE: the fp32 force sums of an evaluation widened into the fp64 force array
__global__ void k_widen(int n, const float* Ff, double* F) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) F[t] = (double)Ff[t];
}

__global__ void k_integrate2(int N, const double4* pos, double* v, const double* F, double dtf0, double dtf1,
                             bool r32) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double dtf = (type_of(pos[i]) == 0) ? dtf0 : dtf1;
  v[3 * i + 0] = kick(v[3 * i + 0], dtf, F[3 * i + 0], r32);
  v[3 * i + 1] = kick(v[3 * i + 1], dtf, F[3 * i + 1], r32);
  v[3 * i + 2] = kick(v[3 * i + 2], dtf, F[3 * i + 2], r32);
}

// NVE second half-kick fused with the reduction of the evaluation's partial rows (the two are
// independent): blocks [0, ACC_N + CT_N) reduce one column each, the rest kick 256 atoms each
__global__ void k_post(RedRows R, int nrows, double* acc, unsigned long long* ct, int N, const double4* pos, double* v,
                       const double* F, double dtf0, double dtf1, bool r32) {
  if (blockIdx.x < ACC_N + CT_N) {
    reduce_column(R, nrows, acc, ct, blockIdx.x);
    return;
  }
  int i = (blockIdx.x - (ACC_N + CT_N)) * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double dtf = (type_of(pos[i]) == 0) ? dtf0 : dtf1;
  v[3 * i + 0] = kick(v[3 * i + 0], dtf, F[3 * i + 0], r32);
  v[3 * i + 1] = kick(v[3 * i + 1], dtf, F[3 * i + 1], r32);
  v[3 * i + 2] = kick(v[3 * i + 2], dtf, F[3 * i + 2], r32);
}

__global__ void k_maxdisp(int N, const double4* pos, const double4* xref, unsigned long long* maxd2,
                          unsigned long long* dbound) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (i < N) {
    double4 p = pos[i], r = xref[i];
    double dx = p.x - r.x, dy = p.y - r.y, dz = p.z - r.z;
    d2 = dx * dx + dy * dy + dz * dz;
  }
  block_max_atomic(d2, maxd2, dbound);
}

// sum m v^2 / 2 (mvv2e applied on the host)
__global__ void k_ke(int N, const double4* pos, const double* v, double m0, double m1, double* acc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double k = 0.0;
  if (i < N) {
    double m = (type_of(pos[i]) == 0) ? m0 : m1;
    double a = v[3 * i], b = v[3 * i + 1], c = v[3 * i + 2];
    k = 0.5 * m * (a * a + b * b + c * c);
  }
  k = warp_sum(k);
  if ((threadIdx.x & 31) == 0 && k != 0.0) atomicAdd(acc + ACC_KE, k);
}

__global__ void k_copy_xref(int N, const double4* pos, double4* xref) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) xref[i] = pos[i];
}

__global__ void k_types(int NT, const double4* pos, signed char* typ) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < NT) typ[a] = (signed char)type_of(pos[a]);
}

// caller-order array (n*3) -> internal positions / velocities
__global__ void k_from_caller_pos(int N, const int* gid, const double* in, double4* pos) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int g = gid[i];
  double4 p = pos[i];
  p.x = in[3 * g], p.y = in[3 * g + 1], p.z = in[3 * g + 2];
  pos[i] = p;
}
__global__ void k_from_caller_vec(int N, const int* gid, const double* in, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int g = gid[i];
  out[3 * i] = in[3 * g], out[3 * i + 1] = in[3 * g + 1], out[3 * i + 2] = in[3 * g + 2];
}
// internal -> caller order
__global__ void k_to_caller_vec(int N, const int* gid, const double* in, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int g = gid[i];
  out[3 * g] = in[3 * i], out[3 * g + 1] = in[3 * i + 1], out[3 * g + 2] = in[3 * i + 2];
}
__global__ void k_to_caller_pos(int N, const int* gid, const double4* pos, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int g = gid[i];
  double4 p = pos[i];
  out[3 * g] = p.x, out[3 * g + 1] = p.y, out[3 * g + 2] = p.z;
}

}  // namespace ab
