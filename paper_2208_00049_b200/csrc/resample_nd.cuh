// resample_nd.cuh — forward interpolation for D = 2, 3
// with one CTA per grid tile, statically mapped (blockIdx = tile id).
//
//   f_j = sum_{l in I_{Nt,m}(k_j)} ghat_l psi~(k_j - l/Nt)      (Alg. 3)
//
// The tile's block index set (Q_d + 2m - 1 cells per dimension,
// wrap resolved at staging, Remark PAPER.md:588-590) is copied into shared
// memory with cp.async, one warp per region row, the row's storage offset
// computed once per row (the first-generation kernel spent ~40% of its
// instructions on per-cell index arithmetic). The node coordinates of the
// first two nodes per thread are loaded while the region streams in; then per
// node the separable taps and the (2m)^D tensor sum with
// the innermost dimension contiguous (eq. InnerTensorStructure)
// and the bank-rotated row sum of resample.cuh.
#pragma once

#include "resample.cuh"

namespace nfftb {

constexpr int RN_THREADS = 256;

template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(RN_THREADS) interp_nd_kernel(Geom g, WinPoly<T> wp,
                                                               const typename cplx<T>::type* __restrict__ grid,
                                                               const T* __restrict__ ks, const int* __restrict__ perm,
                                                               const int* __restrict__ offsets, int nb, int ne,
                                                               typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  constexpr int TP = RotCfg<T, M>::TP;
  constexpr int EXT = (TP > 2 * M ? TP : 2 * M) - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tile = reinterpret_cast<C*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x;
  int c0[D], s0[D], Rr[D];
  {
    int rem = t;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      const int p = rem % g.P[d];
      rem /= g.P[d];
      c0[d] = p * g.Q[d];
      const int qt = min(g.Q[d], g.Nt[d] - c0[d]);
      Rr[d] = qt + (d == D - 1 ? EXT : 2 * M - 1);  // staged extent
      // binning cell c = (a + Nt/2) mod Nt <-> storage (a mod Nt) = (c - Nt/2) mod Nt
      s0[d] = pos_mod(c0[d] - M + 1 - (g.Nt[d] >> 1), g.Nt[d]);
    }
  }
  const int Lp = g.L[D - 1];  // row pitch (cells): >= Q + EXT, multiple of 8 for C128
  const int R1 = D == 3 ? g.L[1] : 1;
  auto stage = [&](const C* src) {
    const int rows = D == 2 ? Rr[0] : Rr[0] * Rr[1];
    const int NtL = g.Nt[D - 1];
    for (int r = warp; r < rows; r += RN_THREADS / 32) {
      long long off;
      int srow;
      if (D == 2) {
        int s = s0[0] + r;
        while (s >= g.Nt[0]) s -= g.Nt[0];
        off = (long long)s * NtL;
        srow = r;
      } else {
        const int i0 = r / Rr[1], i1 = r - i0 * Rr[1];
        int sa = s0[0] + i0, sb = s0[1] + i1;
        while (sa >= g.Nt[0]) sa -= g.Nt[0];
        while (sb >= g.Nt[1]) sb -= g.Nt[1];
        off = ((long long)sa * g.Nt[1] + sb) * NtL;
        srow = i0 * R1 + i1;
      }
      const C* rsrc = src + off;
      C* rdst = tile + (long long)srow * Lp;
      for (int col = lane; col < Rr[D - 1]; col += 32) {
        int s = s0[D - 1] + col;
        while (s >= NtL) s -= NtL;
        cp_async_cell<T>(rdst + col, rsrc + s);
      }
    }
  };
  stage(grid);
  const int o0 = max(__ldg(offsets + t), nb), o1 = min(__ldg(offsets + t + 1), ne);
  // two nodes per thread (D = 2) with their loads in flight together
  constexpr int U = D == 2 ? 2 : 1;
  int jn[U];
  double kn[U][D];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = o0 + threadIdx.x + RN_THREADS * u;
    jn[u] = -1;
    if (i < o1) {
      jn[u] = perm[i];
#pragma unroll
      for (int d = 0; d < D; ++d) kn[u][d] = (double)ks[(long long)d * g.M + i];
    }
  }
  auto node = [&](const double (&k)[D], int (&loc)[D], T (&w)[D][2 * M]) {
    bool ok = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double frac;
      loc[d] = node_cell(k[d], g.Ntd[d], g.Nt[d], frac) - c0[d];
      ok = ok && (unsigned)loc[d] < (unsigned)(Rr[d] - (d == D - 1 ? EXT : 2 * M - 1));
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w[d]);
    }
    return ok;
  };
  auto eval = [&](const int (&loc)[D], const T (&w)[D][2 * M]) {
    T wr[TP];
    const int rot = (lane - loc[D - 1]) & (TP - 1);
    if constexpr (RotCfg<T, M>::ON) rotate_taps<T, M, TP>(w[D - 1], rot, wr);
    C acc;
    acc.x = (T)0;
    acc.y = (T)0;
    if constexpr (D == 2) {
#pragma unroll
      for (int l0 = 0; l0 < 2 * M; ++l0) {
        const C s = row_sum<T, M>(tile + (loc[0] + l0) * Lp + loc[1], wr, w[1], rot);
        acc.x = fma(w[0][l0], s.x, acc.x);
        acc.y = fma(w[0][l0], s.y, acc.y);
      }
    } else {
      constexpr int U0 = (2 * M <= 8) ? 2 * M : 1;
#pragma unroll U0
      for (int l0 = 0; l0 < 2 * M; ++l0) {
        C s1;
        s1.x = (T)0;
        s1.y = (T)0;
#pragma unroll
        for (int l1 = 0; l1 < 2 * M; ++l1) {
          const C s = row_sum<T, M>(tile + ((loc[0] + l0) * R1 + loc[1] + l1) * Lp + loc[2], wr, w[2], rot);
          s1.x = fma(w[1][l1], s.x, s1.x);
          s1.y = fma(w[1][l1], s.y, s1.y);
        }
        acc.x = fma(w[0][l0], s1.x, acc.x);
        acc.y = fma(w[0][l0], s1.y, acc.y);
      }
    }
    return acc;
  };
  cp_async_wait_all();
  __syncthreads();
  for (int b = 0; b < g.B; ++b) {
    if (b > 0) {
      __syncthreads();
      stage(grid + (long long)b * g.grid_cells);
      cp_async_wait_all();
      __syncthreads();
    }
    C* fb = f + (long long)b * g.M;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (jn[u] < 0) continue;
      int loc[D];
      T w[D][2 * M];
      if (node(kn[u], loc, w)) fb[jn[u]] = eval(loc, w);
    }
    for (int i = o0 + threadIdx.x + RN_THREADS * U; i < o1; i += RN_THREADS) {
      double k[D];
#pragma unroll
      for (int d = 0; d < D; ++d) k[d] = (double)ks[(long long)d * g.M + i];
      int loc[D];
      T w[D][2 * M];
      if (node(k, loc, w)) fb[perm[i]] = eval(loc, w);
    }
  }
}

}  // namespace nfftb
