// k_scan.cuh -- hand-written scans, stream compaction and the stable counting sort by cell used
// by the list rebuild (binning; periodic images and slab halos).
//
// * exclusive scan of n ints (or of the 0/1 flags of an int array) into out[0..n], out[n] = total:
//   k_scan_blocks (2048 elements per 1024-thread block, warp shuffles + one shared-memory pass),
//   k_scan_carry (one block: exclusive scan of the block totals), k_scan_add.
// * stable selection: indices q < n with flag[q] != 0 in increasing order (k_select_scatter).
// * stable counting sort of atom indices by cell key: histogram (atomics), scan -> cell_start,
//   scatter through per-cell atomic cursors, then one thread per cell sorts its (small) segment
//   by atom index -- the result is exactly the stable sort by (cell, index), deterministic.
#pragma once
#include <cuda_runtime.h>

namespace ab {

constexpr int SCAN_T = 1024, SCAN_E = 2 * SCAN_T;  // threads / elements per scan block

template <bool FLAG>
__device__ __forceinline__ int scan_in(const int* in, int q, int n) {
  if (q >= n) return 0;
  const int v = in[q];
  return FLAG ? (v != 0) : v;
}

// block-local exclusive scan of SCAN_E elements; bsum[b] = block total
template <bool FLAG>
__global__ void __launch_bounds__(SCAN_T) k_scan_blocks(const int* in, int n, int* out, int* bsum) {
  __shared__ int ws[32];
  const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int q0 = b * SCAN_E + 2 * t;
  const int a0 = scan_in<FLAG>(in, q0, n), a1 = scan_in<FLAG>(in, q0 + 1, n);
  int x = a0 + a1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    int y = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += u;
    }
    ws[lane] = y;
  }
  __syncthreads();
  const int excl = (w ? ws[w - 1] : 0) + x - (a0 + a1);
  if (q0 < n) out[q0] = excl;
  if (q0 + 1 < n) out[q0 + 1] = excl + a0;
  if (t == SCAN_T - 1) bsum[b] = excl + a0 + a1;
}

// exclusive scan of the nb block totals in place (one block, chunks of 1024); bsum[nb] = total
__global__ void __launch_bounds__(SCAN_T) k_scan_carry(int nb, int* bsum) {
  __shared__ int ws[32];
  __shared__ int carry;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += SCAN_T) {
    const int q = base + t;
    const int v = q < nb ? bsum[q] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += u;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
      int y = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += u;
      }
      ws[lane] = y;
    }
    __syncthreads();
    const int excl = carry + (w ? ws[w - 1] : 0) + x - v;
    if (q < nb) bsum[q] = excl;
    __syncthreads();
    if (t == SCAN_T - 1) carry = excl + v;
    __syncthreads();
  }
  if (t == 0) bsum[nb] = carry;
}

__global__ void k_scan_add(int n, int nb, const int* bsum, int* out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) out[q] += bsum[q / SCAN_E];
  if (q == 0) out[n] = bsum[nb];
}

// out_idx = { q < n : flag[q] != 0 } in order (off = exclusive scan of the flags); *num = count
__global__ void k_select_scatter(int n, const int* flag, const int* off, int* out_idx, int* num) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n && flag[q] != 0) out_idx[off[q]] = q;
  if (q == 0) *num = off[n];
}

__global__ void k_cell_hist(int n, const int* key, int* cnt) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < n) atomicAdd(cnt + key[a], 1);
}

__global__ void k_cell_scatter(int n, const int* key, int* cursor, int* perm) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < n) perm[atomicAdd(cursor + key[a], 1)] = a;
}

// one thread per cell: insertion sort of the cell's segment by (sec[atom], atom index), or by the
// atom index alone (sec == nullptr); segments are small
__global__ void k_cell_order(int ncell, const int* cell_start, const int* sec, int* perm) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  const int b = cell_start[c], e = cell_start[c + 1];
  for (int q = b + 1; q < e; ++q) {
    const int v = perm[q];
    const int sv = sec ? sec[v] : 0;
    int p = q - 1;
    while (p >= b) {
      const int u = perm[p];
      const int su = sec ? sec[u] : 0;
      if (su < sv || (su == sv && u < v)) break;
      perm[p + 1] = u;
      --p;
    }
    perm[p + 1] = v;
  }
}

}  // namespace ab
