// resample1d.cuh — the D = 1 hot path (SURVEY §8(a) rows a1-a2 refinement,
// a6, a7; the BASELINE headline configuration) over CELL-SORTED nodes.
//
//   forward: f_j = sum_l ghat_l psi~(k_j - l/Nt)        (Alg. 3)
//   adjoint: ghat_l = sum_j f_j psi~(k_j - l/Nt)         (Alg. 4)
//
// cellsort1d (precompute, one warp per tile): refines the stable tile sort of
//   binsort.cuh to the stable CELL order inside each tile (in 1D the tiles are
//   consecutive cell ranges, so this is the global cell order) and writes the
//   cell offset table cstart[c] (first cell-sorted position of cell c). It is
//   computed once per node set and shared by every forward and adjoint.
// interp1c: one thread per node in cell order; the 2m grid cells are read
//   straight from L2 (the FFT output is L2-resident): consecutive lanes hold
//   nodes of nearby cells, so their windows overlap in L1. No staging, no
//   barrier, one dependent load level before the arithmetic.
// spread1c: OWNER-COMPUTES gather, one warp per 32 K consecutive cells. The
//   nodes that reach the warp's cells are the contiguous cell-sorted range of
//   cells [y0 - m, y0 + 32K + m - 2] (the cstart table gives it, wrap included);
//   the warp evaluates their taps once into shared memory and every lane sums,
//   for each of its K cells y, f_j w_j[y - x_j + m - 1] over the contiguous slot
//   range of cells x in [y - m, y + m - 1]. Every cell is written exactly once
//   with a plain coalesced store: no atomics, no zero pass, no halo merge (the
//   paper's locked merge of PAPER.md:578-582 disappears because the halo NODES
//   are read instead of halo CELLS being reduced).
#pragma once

#include "resample.cuh"

namespace nfftb {

constexpr int I1_THREADS = 256;           // interp1c: one node per thread
constexpr int S1_WARPS = 4;               // spread1c: warps per CTA
constexpr int S1_K = 4;                   // spread1c: cells per lane
constexpr int S1_SEG = 32 * S1_K;         // cells per warp
constexpr int S1_CAP = 96;                // node slots per warp chunk (typical window: ~0.5 (SEG + 2m) nodes)

__host__ __device__ inline size_t s1_warp_bytes(int M, size_t csize, size_t rsize) {
  size_t b = (size_t)S1_CAP * 2 * M * rsize;  // taps per slot
  b = (b + 15) & ~(size_t)15;
  b += (size_t)S1_CAP * csize;                // node value of the current batch vector
  b += (size_t)S1_CAP * 4;                    // extended cell of a slot
  b += (size_t)(2 * (S1_SEG + 2 * M)) * 4;    // window cell starts, position bases
  return (b + 15) & ~(size_t)15;
}

// ---------------------------------------------------------------- forward
template <typename T, int M, int DEG>
__global__ void __launch_bounds__(I1_THREADS) interp1c_kernel(Geom g, WinPoly<T> wp,
                                                              const typename cplx<T>::type* __restrict__ grid,
                                                              const T* __restrict__ kc, const int* __restrict__ jc,
                                                              int nb, int ne, int sharded,
                                                              typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  const int pc = blockIdx.x * I1_THREADS + threadIdx.x;
  if (pc >= g.M) return;
  if (sharded && (pc < nb || pc >= ne)) return;  // shard = range of the cell-sorted order
  const int j = jc[pc];
  double frac;
  const int Nt = g.Nt[0];
  const int c = node_cell((double)kc[pc], g.Ntd[0], Nt, frac);
  T w[2 * M];
  window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
  // storage of the footprint's first cell: binning cell c = (a + Nt/2) mod Nt, storage (a - m + 1) mod Nt
  int s0 = c - M + 1 - (Nt >> 1);
  if (s0 < 0) s0 += Nt;
  if (s0 < 0) s0 = pos_mod(s0, Nt);
  int sl[2 * M];
#pragma unroll
  for (int l = 0; l < 2 * M; ++l) {
    int s = s0 + l;
    if (s >= Nt) s -= Nt;
    if (s >= Nt) s = pos_mod(s, Nt);
    sl[l] = s;
  }
  for (int b = 0; b < g.B; ++b) {
    const C* gb = grid + (long long)b * g.grid_cells;
    C v[2 * M];
#pragma unroll
    for (int l = 0; l < 2 * M; ++l) v[l] = __ldg(gb + sl[l]);
    C acc;
    acc.x = (T)0;
    acc.y = (T)0;
#pragma unroll
    for (int l = 0; l < 2 * M; ++l) {
      acc.x = fma(w[l], v[l].x, acc.x);
      acc.y = fma(w[l], v[l].y, acc.y);
    }
    f[(long long)b * g.M + j] = acc;
  }
}

// ---------------------------------------------------------------- adjoint
template <typename T, int M, int DEG>
__global__ void __launch_bounds__(32 * S1_WARPS) spread1c_kernel(Geom g, WinPoly<T> wp,
                                                                 const typename cplx<T>::type* __restrict__ f,
                                                                 const T* __restrict__ kc, const int* __restrict__ jc,
                                                                 const int* __restrict__ cstart, int nb, int ne,
                                                                 int sharded, typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  constexpr int NEXT = S1_SEG + 2 * M - 1;  // extended cells of a full segment
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Nt = g.Nt[0];
  const int y0 = (blockIdx.x * S1_WARPS + warp) * S1_SEG;
  if (y0 >= Nt) return;
  const int nseg = min(S1_SEG, Nt - y0);
  const int NE = nseg + 2 * M - 1;  // extended cell e <-> binning cell (y0 - m + e) mod Nt
  unsigned char* wb = smem_raw + (size_t)warp * s1_warp_bytes(M, sizeof(C), sizeof(T));
  T* tap = reinterpret_cast<T*>(wb);  // [S1_CAP][TAPS]
  C* fv = reinterpret_cast<C*>(wb + (((size_t)S1_CAP * TAPS * sizeof(T) + 15) & ~(size_t)15));
  int* se = reinterpret_cast<int*>(fv + S1_CAP);  // [S1_CAP] extended cell of the slot
  int* wstart = se + S1_CAP;                      // [NEXT + 1] first window slot of extended cell e
  int* wbase = wstart + NEXT + 1;                 // [NEXT] cell-sorted position of slot s = wbase[e] + s

  auto cell_of = [&](int e) {
    int c = y0 - M + e;
    if (c < 0) c += Nt;
    if (c >= Nt) c -= Nt;
    if ((unsigned)c >= (unsigned)Nt) c = pos_mod(c, Nt);
    return c;
  };
  // window cell starts: all cstart loads of the lane issued together, warp scan;
  // base[e] = cstart of the cell minus its first window slot; slot -> extended cell map
  {
    constexpr int PER = (NEXT + 1 + 31) / 32;
    const int lo = lane * PER;
    int c_lo[PER], c_hi[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = lo + q;
      c_lo[q] = c_hi[q] = 0;
      if (e < NE) {
        const int c = cell_of(e);
        c_lo[q] = __ldg(cstart + c);
        c_hi[q] = __ldg(cstart + c + 1);
      }
    }
    int sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) sum += c_hi[q] - c_lo[q];
    int total;
    int run = warp_exclusive_scan(sum, total);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = lo + q;
      if (e < NE) {
        wstart[e] = run;
        wbase[e] = c_lo[q] - run;
      }
      run += c_hi[q] - c_lo[q];
    }
    if (lane == 0) wstart[NE] = total;
  }
  __syncwarp();
  const int total = wstart[NE];
  const int sy0 = pos_mod(y0 - (Nt >> 1), Nt);  // storage of binning cell y0
  for (int b = 0; b < g.B; ++b) {
    C acc[S1_K];
#pragma unroll
    for (int kk = 0; kk < S1_K; ++kk) {
      acc[kk].x = (T)0;
      acc[kk].y = (T)0;
    }
    for (int clo = 0; clo < total; clo += S1_CAP) {
      const int chi = min(total, clo + S1_CAP);
      // slot -> extended cell: each lane marks the slots of its extended cells
      for (int e = lane; e < NE; e += 32)
        for (int sl = max(wstart[e], clo); sl < min(wstart[e + 1], chi); ++sl) se[sl - clo] = e;
      __syncwarp();
      // node loads of all the lane's slots in flight together, then taps
      constexpr int SPL = (S1_CAP + 31) / 32;
      int jj[SPL], ee[SPL];
      double kk_[SPL];
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        const int sl = lane + 32 * u;
        ee[u] = -1;
        if (clo + sl < chi) {
          const int e = se[sl];
          const int pc = wbase[e] + clo + sl;
          ee[u] = e;
          jj[u] = jc[pc];
          kk_[u] = (double)kc[pc];
          if (sharded && (pc < nb || pc >= ne)) jj[u] = -1;  // shard = range of the cell-sorted order
        }
      }
      C fvl[SPL];
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        fvl[u].x = (T)0;
        fvl[u].y = (T)0;
        if (ee[u] >= 0 && jj[u] >= 0) fvl[u] = f[(long long)b * g.M + jj[u]];
      }
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        const int sl = lane + 32 * u;
        if (ee[u] < 0) continue;
        double frac;
        node_cell(kk_[u], g.Ntd[0], Nt, frac);
        T w[TAPS];
        window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
#pragma unroll
        for (int l = 0; l < TAPS; ++l) tap[sl * TAPS + l] = w[l];
        fv[sl] = fvl[u];
      }
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk < S1_K; ++kk) {
        const int y = lane + 32 * kk;  // local cell; extended index y + m; contributors e in [y, y + 2m)
        if (y < nseg) {
          const int q0 = max(wstart[y], clo), q1 = min(wstart[y + TAPS], chi);
          for (int q = q0; q < q1; ++q) {
            const int sl = q - clo;
            const T wt = tap[sl * TAPS + (y - se[sl] + TAPS - 1)];
            const C v = fv[sl];
            acc[kk].x = fma(wt, v.x, acc[kk].x);
            acc[kk].y = fma(wt, v.y, acc[kk].y);
          }
        }
      }
      __syncwarp();
    }
    C* dst = grid + (long long)b * g.grid_cells;
#pragma unroll
    for (int kk = 0; kk < S1_K; ++kk) {
      const int y = lane + 32 * kk;
      if (y < nseg) {
        int s = sy0 + y;
        if (s >= Nt) s -= Nt;
        dst[s] = acc[kk];
      }
    }
  }
}

}  // namespace nfftb
