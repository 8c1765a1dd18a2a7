// cellsort.cuh — precompute refinement: the stable
// tile sort of binsort.cuh (the paper's block partition; the
// permutation the ABI reports) refined to the stable CELL order inside every
// tile, plus the cell offset table
//
//   cstart[t * Qc + lc] = first cell-sorted position of local cell lc of tile t,
//   lc = row-major index of the node's cell inside the tile (Qc = prod Q_d),
//   cstart[P * Qc] = M.
//
// Computed once per node set and shared by every forward and adjoint: the
// resampling kernels then find the nodes of any cell range of a tile as one
// contiguous range (no per-kernel sorting). In 1D, t * Q + lc is the global
// binning cell, so the order is the global cell order.
//
// One CTA per tile. Pass A: cell histogram (shared int atomics), block scan ->
// cstart. Pass B, in tile-sorted order, CS_THREADS nodes at a time: per-warp u16
// cell counters + __match_any_sync ranks + a per-cell running count give the
// stable rank (cell ascending, tile-sorted position ascending).
#pragma once

#include "common.cuh"

namespace nfftb {

constexpr int CST_THREADS = 256;
constexpr int CST_W = CST_THREADS / 32;

__host__ __device__ inline size_t cst_smem_bytes(int Qc) {
  return (((size_t)Qc * CST_W * 2 + 15) & ~(size_t)15) + (size_t)(3 * Qc + 1) * 4;
}

template <typename R, int D>
__global__ void __launch_bounds__(CST_THREADS) cellsort_kernel(Geom g, const R* __restrict__ ks,
                                                               const int* __restrict__ perm,
                                                               const int* __restrict__ offsets,
                                                               R* __restrict__ kc, int* __restrict__ jc,
                                                               int* __restrict__ ic, int* __restrict__ cstart) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int ws[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int t = blockIdx.x;
  int Qc = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) Qc *= g.Q[d];
  int cb[D];  // first binning cell of the tile per dimension
  {
    int rem = t;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      cb[d] = (rem % g.P[d]) * g.Q[d];
      rem /= g.P[d];
    }
  }
  unsigned short* wc = reinterpret_cast<unsigned short*>(smem_raw);                            // [Qc][CST_W]
  int* cs = reinterpret_cast<int*>(smem_raw + (((size_t)Qc * CST_W * 2 + 15) & ~(size_t)15));  // [Qc + 1] cell starts
  int* done = cs + Qc + 1;                                                                      // [Qc] placed so far
  int* pcnt = done + Qc;                                                                        // [Qc] placed this pass
  const int o0 = __ldg(offsets + t), o1 = __ldg(offsets + t + 1);
  auto cell = [&](int i, R (&k)[D]) {
    int lc = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      k[d] = ks[(long long)d * g.M + i];
      double frac;
      const int x = min(max(node_cell((double)k[d], g.Ntd[d], g.Nt[d], frac) - cb[d], 0), g.Q[d] - 1);
      lc = lc * g.Q[d] + x;
    }
    return lc;
  };
  for (int q = tid; q <= Qc; q += CST_THREADS) {
    cs[q] = 0;
    if (q < Qc) done[q] = 0;
  }
  __syncthreads();
  for (int i = o0 + tid; i < o1; i += CST_THREADS) {  // pass A
    R k[D];
    atomicAdd(&cs[cell(i, k) + 1], 1);
  }
  __syncthreads();
  const int per = (Qc + 1 + CST_THREADS - 1) / CST_THREADS;
  const int lo = tid * per, hi = min(Qc + 1, lo + per), hic = min(hi, Qc);
  {
    int sum = 0;
    for (int q = lo; q < hi; ++q) sum += cs[q];
    int tot;
    int run = block_exclusive_scan(sum, ws, tot);
    for (int q = lo; q < hi; ++q) {
      run += cs[q];
      cs[q] = run;  // first local slot of cell q
      if (q < Qc) cstart[(long long)t * Qc + q] = o0 + run;
    }
    if (t == (int)gridDim.x - 1 && tid == 0) cstart[(long long)gridDim.x * Qc] = o1;
  }
  for (int pass = o0; pass < o1; pass += CST_THREADS) {  // pass B
    const int i = pass + tid;
    int x = -1, j = 0;
    R k[D];
#pragma unroll
    for (int d = 0; d < D; ++d) k[d] = (R)0;
    if (i < o1) {
      x = cell(i, k);
      j = perm[i];
    }
    {
      unsigned* w32 = reinterpret_cast<unsigned*>(wc);
      for (int q = tid; q < (Qc * CST_W + 1) / 2; q += CST_THREADS) w32[q] = 0u;
    }
    __syncthreads();
    const unsigned peers = __match_any_sync(0xffffffffu, x);
    const int rank = __popc(peers & lt);
    if (x >= 0 && lane == __ffs(peers) - 1) wc[x * CST_W + warp] = (unsigned short)__popc(peers);
    __syncthreads();
    for (int q = lo; q < hic; ++q) {  // exclusive prefix over the warps
      unsigned run = 0;
#pragma unroll
      for (int w = 0; w < CST_W; ++w) {
        const unsigned c = wc[q * CST_W + w];
        wc[q * CST_W + w] = (unsigned short)run;
        run += c;
      }
      pcnt[q] = (int)run;
    }
    __syncthreads();
    if (x >= 0) {
      const int pos = o0 + cs[x] + done[x] + wc[x * CST_W + warp] + rank;
#pragma unroll
      for (int d = 0; d < D; ++d) kc[(long long)d * g.M + pos] = k[d];
      jc[pos] = j;
      ic[pos] = i;
    }
    __syncthreads();
    for (int q = lo; q < hic; ++q) done[q] += pcnt[q];
  }
}

}  // namespace nfftb
