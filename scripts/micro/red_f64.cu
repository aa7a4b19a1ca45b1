// Microbenchmark (diagnostic, not shipped): throughput of fp64 global reductions (RED.ADD.F64)
// with the address pattern of a half neighbour list: thread t adds 3 components to atom
// j = base(t) + small offset, where neighbouring threads hit nearby atoms (cell-ordered lists).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_red(double* F, int natoms, long long nops, int spread, unsigned seed) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (long long q = t; q < nops; q += stride) {
    unsigned h = (unsigned)(q / 32) * 2654435761u + seed;
    int base = (int)(h % (unsigned)natoms);
    unsigned hh = (unsigned)q * 2246822519u;
    int j = (base + (int)(hh % (unsigned)spread)) % natoms;
    atomicAdd(F + 3 * (size_t)j + 0, 1.0);
    atomicAdd(F + 3 * (size_t)j + 1, 1.0);
    atomicAdd(F + 3 * (size_t)j + 2, 1.0);
  }
}
int main() {
  const int natoms = 1400000;
  const long long nops = 170000000LL;
  double* F;
  cudaMalloc(&F, sizeof(double) * 3 * natoms);
  cudaMemset(F, 0, sizeof(double) * 3 * natoms);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int spreads[] = {1, 64, 512, 4096, 1400000};
  for (int s : spreads) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_red<<<148 * 8, 256>>>(F, natoms, nops, s, 12345u + rep);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("spread %8d: %lld x 3 RED.F64 in %.3f ms = %.1f G atomics/s\n", s, nops, ms, 3 * nops / ms / 1e6);
    }
  }
  return 0;
}
