// resample1d.cuh — the D = 1 hot path (the
// BASELINE headline configuration) as one CTA per grid tile, statically
// mapped (blockIdx = tile), so no kernel depends on a subproblem list and the
// grid region can be requested at kernel entry.
//
//   forward: f_j = sum_l ghat_l psi~(k_j - l/Nt)        (Alg. 3)
//   adjoint: ghat_l = sum_j f_j psi~(k_j - l/Nt)         (Alg. 4)
//
// interp1d: the tile's region (Q + 2m - 1 cells, wrap resolved at staging,
//   Remark PAPER.md:588-590) streams into shared memory with cp.async while
//   the node coordinates and taps are loaded/evaluated; one thread per node,
//   bank-rotated 2m-tap sum (resample.cuh: row_sum), result scattered to the
//   caller's node order f[perm[i]].
// spread1d: OWNER-COMPUTES. The CTA of tile t writes every cell of its tile
//   exactly once with a plain coalesced store: it takes its own nodes plus the
//   nodes of the two neighbour tiles that reach into it (|x| <= m cells from
//   the tile edge; the paper's halo merge of PAPER.md:578-582 becomes reading
//   the halo NODES instead of reducing halo CELLS), counting-sorts them by
//   local cell in shared memory, and every owned cell y gathers
//   sum f_j w_j[y - x_j + m - 1] over the contiguous slot range of the cells
//   x in [y - m, y + m - 1]. No atomics on the grid, no zero pass (cells
//   without nodes are written 0), so the crop that follows need not re-zero.
// Preconditions (checked by the host): Q | Ntilde, P = Ntilde/Q >= 3, Q >= 2m.
#pragma once

#include "resample.cuh"

namespace nfftb {

constexpr int R1_THREADS = 256;
constexpr int S1_KPT = 2;  // spread candidates per thread per chunk (chunk = S1_KPT * R1_THREADS)

__host__ __device__ inline int r1_region_cells(int Q, int M, bool c128) {
  const int TP = c128 ? ((2 * M <= 8) ? 8 : 16) : 2 * M;
  return Q + (TP > 2 * M ? TP : 2 * M) - 1;
}

__host__ __device__ inline size_t r1_spread_smem_bytes(int Q, int M, size_t csize, size_t rsize) {
  const size_t CH = (size_t)S1_KPT * R1_THREADS;
  size_t b = CH * 2 * M * rsize;           // taps per sorted slot
  b = (b + 15) & ~(size_t)15;
  b += CH * csize;                         // node value of the current batch vector
  b += CH * 8;                             // bin, node index
  b += (size_t)(2 * (Q + 2 * M) + 2) * 4;  // bin starts, cursors
  return b;
}

template <typename T, int M, int DEG>
__global__ void __launch_bounds__(R1_THREADS) interp1d_kernel(Geom g, WinPoly<T> wp,
                                                              const typename cplx<T>::type* __restrict__ grid,
                                                              const T* __restrict__ ks, const int* __restrict__ perm,
                                                              const int* __restrict__ offsets, int nb, int ne,
                                                              typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  constexpr int TP = RotCfg<T, M>::TP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tile = reinterpret_cast<C*>(smem_raw);
  const int t = blockIdx.x;
  const int Nt = g.Nt[0], Q = g.Q[0];
  const int c0 = t * Q;
  const int Qt = min(Q, Nt - c0);
  const int Lr = Qt + (TP > 2 * M ? TP : 2 * M) - 1;
  // binning cell c = (a + Nt/2) mod Nt (node_cell) <-> grid storage (a mod Nt) = (c - Nt/2) mod Nt
  const int s0 = pos_mod(c0 - M + 1 - (Nt >> 1), Nt);
  auto stage = [&](const C* src) {
    for (int r = threadIdx.x; r < Lr; r += blockDim.x) {
      int s = s0 + r;
      while (s >= Nt) s -= Nt;
      cp_async_cell<T>(&tile[r], src + s);
    }
  };
  stage(grid);
  const int o0 = max(__ldg(offsets + t), nb), o1 = min(__ldg(offsets + t + 1), ne);
  auto setup = [&](int i, int& j, int& loc, T (&w)[2 * M]) {
    j = perm[i];
    double frac;
    const int c = node_cell((double)ks[i], g.Ntd[0], Nt, frac);
    loc = c - c0;
    window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
    return (unsigned)loc < (unsigned)Qt;
  };
  auto eval = [&](int loc, const T (&w)[2 * M]) {
    T wr[TP];
    const int rot = ((int)(threadIdx.x & 31) - loc) & (TP - 1);
    if constexpr (RotCfg<T, M>::ON) rotate_taps<T, M, TP>(w, rot, wr);
    return row_sum<T, M>(tile + loc, wr, w, rot);
  };
  const int i0 = o0 + threadIdx.x;
  int j0 = 0, loc0 = 0;
  T w0[2 * M];
  const bool has0 = i0 < o1 && setup(i0, j0, loc0, w0);
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
    if (has0) fb[j0] = eval(loc0, w0);
    for (int i = i0 + blockDim.x; i < o1; i += blockDim.x) {
      int j, loc;
      T w[2 * M];
      if (setup(i, j, loc, w)) fb[j] = eval(loc, w);
    }
  }
}

template <typename T, int M, int DEG>
__global__ void __launch_bounds__(R1_THREADS) spread1d_kernel(Geom g, WinPoly<T> wp,
                                                              const typename cplx<T>::type* __restrict__ f,
                                                              const T* __restrict__ ks, const int* __restrict__ perm,
                                                              const int* __restrict__ offsets, int nb, int ne,
                                                              typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  constexpr int CH = S1_KPT * R1_THREADS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int Nt = g.Nt[0], Q = g.Q[0], P = g.P[0];
  const int NB = Q + 2 * M - 1;  // bins: local cell x in [-m, Q + m - 2] -> x + m
  T* tap = reinterpret_cast<T*>(smem_raw);  // [CH][TAPS]
  C* fv = reinterpret_cast<C*>(smem_raw + (((size_t)CH * TAPS * sizeof(T) + 15) & ~(size_t)15));
  int* sbin = reinterpret_cast<int*>(fv + CH);
  int* sj = sbin + CH;
  int* start = sj + CH;           // [NB + 1]
  int* cursor = start + NB + 1;   // [NB + 1]
  __shared__ int ws[32];

  const int t = blockIdx.x;
  const int c0 = t * Q;
  const int tl = t == 0 ? P - 1 : t - 1, tr = t == P - 1 ? 0 : t + 1;
  const int a0 = max(__ldg(offsets + tl), nb), a1 = min(__ldg(offsets + tl + 1), ne);
  const int b0 = max(__ldg(offsets + t), nb), b1 = min(__ldg(offsets + t + 1), ne);
  const int e0 = max(__ldg(offsets + tr), nb), e1 = min(__ldg(offsets + tr + 1), ne);
  const int nA = max(0, a1 - a0), nBn = max(0, b1 - b0), nC = max(0, e1 - e0);
  const int n = nA + nBn + nC;

  for (int ch = 0; ch == 0 || ch < n; ch += CH) {
    for (int k = threadIdx.x; k <= NB; k += blockDim.x) start[k] = 0;
    __syncthreads();
    int bins[S1_KPT], js[S1_KPT];
    C fval[S1_KPT];  // batch vector 0, loaded with the node (shortens the dependent-load chain)
    T w[S1_KPT][TAPS];
#pragma unroll
    for (int kk = 0; kk < S1_KPT; ++kk) {
      const int u = ch + kk * blockDim.x + threadIdx.x;
      bins[kk] = -1;
      if (u < n) {
        const int i = u < nA ? a0 + u : (u < nA + nBn ? b0 + (u - nA) : e0 + (u - nA - nBn));
        double frac;
        const int c = node_cell((double)ks[i], g.Ntd[0], Nt, frac);
        int x = c - c0;
        if (x > (Nt >> 1)) x -= Nt;
        else if (x < -(Nt >> 1)) x += Nt;
        if (x >= -M && x <= Q + M - 2) {
          bins[kk] = x + M;
          js[kk] = perm[i];
          fval[kk] = f[js[kk]];
          window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w[kk]);
          atomicAdd(&start[bins[kk] + 1], 1);
        }
      }
    }
    __syncthreads();
    {
      const int per = (NB + 1 + blockDim.x - 1) / blockDim.x;
      const int lo = threadIdx.x * per, hi = min(NB + 1, lo + per);
      int sum = 0;
      for (int k = lo; k < hi; ++k) sum += start[k];
      int total;
      int run = block_exclusive_scan(sum, ws, total);
      for (int k = lo; k < hi; ++k) {
        run += start[k];
        start[k] = run;  // first slot of bin k (start[0] = 0); start[NB] = slots in chunk
        cursor[k] = run;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < S1_KPT; ++kk) {
      if (bins[kk] < 0) continue;
      const int slot = atomicAdd(&cursor[bins[kk]], 1);
      sbin[slot] = bins[kk];
      sj[slot] = js[kk];
      fv[slot] = fval[kk];
#pragma unroll
      for (int l = 0; l < TAPS; ++l) tap[slot * TAPS + l] = w[kk][l];
    }
    __syncthreads();
    const int nslots = start[NB];
    for (int b = 0; b < g.B; ++b) {
      if (b > 0) {
        const C* fb = f + (long long)b * g.M;
        for (int q = threadIdx.x; q < nslots; q += blockDim.x) fv[q] = fb[sj[q]];
        __syncthreads();
      }
      C* dst = grid + (long long)b * g.grid_cells;
      const int sy0 = pos_mod(c0 - (Nt >> 1), Nt);  // storage of the tile's first cell (see interp1d)
      for (int y = threadIdx.x; y < Q; y += blockDim.x) {
        int sy = sy0 + y;
        if (sy >= Nt) sy -= Nt;
        const int q0 = start[y], q1 = start[y + TAPS];
        C acc;
        acc.x = (T)0;
        acc.y = (T)0;
        for (int q = q0; q < q1; ++q) {
          const T wt = tap[q * TAPS + (y - sbin[q] + TAPS - 1)];
          const C v = fv[q];
          acc.x = fma(wt, v.x, acc.x);
          acc.y = fma(wt, v.y, acc.y);
        }
        if (ch == 0) {
          dst[sy] = acc;
        } else {  // later chunks of an over-full tile: this thread owns cell y in every chunk
          C o = dst[sy];
          o.x += acc.x;
          o.y += acc.y;
          dst[sy] = o;
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace nfftb
