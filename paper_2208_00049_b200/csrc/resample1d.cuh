// resample1d.cuh — the D = 1 hot path (the
// BASELINE headline configuration) as one WARP per grid tile, statically
// mapped (tile = blockIdx * W1_WARPS + warp), so no kernel depends on a
// subproblem list, the grid region is requested at kernel entry, and the
// warps of a CTA never wait for each other (__syncwarp only): at M = 2^18 the
// kernels are latency-bound, so short per-warp dependency chains and all
// tiles in flight at once matter more than per-CTA reuse.
//
//   forward: f_j = sum_l ghat_l psi~(k_j - l/Nt)        (Alg. 3)
//   adjoint: ghat_l = sum_j f_j psi~(k_j - l/Nt)         (Alg. 4)
//
// interp1d: the tile's region (Q + 2m - 1 cells, wrap resolved at staging,
//   Remark PAPER.md:588-590) streams into shared memory with cp.async while
//   the node coordinates and taps are loaded/evaluated; one thread per node,
//   bank-rotated 2m-tap sum (resample.cuh: row_sum), result scattered to the
//   caller's node order f[perm[i]].
// spread1d: OWNER-COMPUTES. The warp of tile t writes every cell of its tile
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

constexpr int W1_WARPS = 4;               // tiles (warps) per CTA
constexpr int W1_THREADS = 32 * W1_WARPS;
constexpr int S1_KPL = 3;                 // spread candidates per lane per chunk
constexpr int S1_CAP = 32 * S1_KPL;       // spread candidates per warp chunk
constexpr int S1_SCAN = 4;                // candidate coordinates per lane in flight while filtering

__host__ __device__ inline int r1_region_cells(int Q, int M, bool c128) {
  const int TP = c128 ? ((2 * M <= 8) ? 8 : 16) : 2 * M;
  return Q + (TP > 2 * M ? TP : 2 * M) - 1;
}

// shared memory of one warp of spread1d (the CTA has W1_WARPS of them)
__host__ __device__ inline size_t r1_spread_warp_bytes(int Q, int M, size_t csize, size_t rsize) {
  size_t b = (size_t)S1_CAP * 2 * M * rsize;  // taps per sorted slot
  b = (b + 15) & ~(size_t)15;
  b += (size_t)S1_CAP * csize;                // node value of the current batch vector
  b += (size_t)S1_CAP * 8;                    // bin, node index
  b += (size_t)(2 * (Q + 2 * M)) * 4;         // bin starts, cursors
  b += (size_t)(S1_CAP + 32 * S1_SCAN) * 4;   // kept-candidate list
  b += (size_t)S1_CAP * 4;                    // cell-sorted order of the chunk
  return (b + 15) & ~(size_t)15;
}

template <typename T, int M, int DEG>
__global__ void __launch_bounds__(W1_THREADS) interp1d_kernel(Geom g, WinPoly<T> wp,
                                                              const typename cplx<T>::type* __restrict__ grid,
                                                              const T* __restrict__ ks, const int* __restrict__ perm,
                                                              const int* __restrict__ offsets, int nb, int ne,
                                                              typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  constexpr int TP = RotCfg<T, M>::TP;
  constexpr int EXT = (TP > 2 * M ? TP : 2 * M) - 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Nt = g.Nt[0], Q = g.Q[0];
  const int t = blockIdx.x * W1_WARPS + warp;
  if (t >= g.P[0]) return;
  const int Lw = (Q + EXT + 7) & ~7;  // per-warp region pitch (cells), 128-byte aligned for C128
  C* tile = reinterpret_cast<C*>(smem_raw) + warp * Lw;
  const int c0 = t * Q;
  const int Qt = min(Q, Nt - c0);
  const int Lr = Qt + EXT;
  // binning cell c = (a + Nt/2) mod Nt (node_cell) <-> grid storage (a mod Nt) = (c - Nt/2) mod Nt
  const int s0 = pos_mod(c0 - M + 1 - (Nt >> 1), Nt);
  auto stage = [&](const C* src) {
    for (int r = lane; r < Lr; r += 32) {
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
    const int rot = (lane - loc) & (TP - 1);
    if constexpr (RotCfg<T, M>::ON) rotate_taps<T, M, TP>(w, rot, wr);
    return row_sum<T, M>(tile + loc, wr, w, rot);
  };
  // U nodes per lane: their coordinate / perm loads are issued together, taps are
  // evaluated one node at a time (keeps registers low)
  constexpr int U = 4;
  int jn[U];
  double kn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = o0 + lane + 32 * u;
    jn[u] = -1;
    if (i < o1) {
      jn[u] = perm[i];
      kn[u] = (double)ks[i];
    }
  }
  cp_async_wait_all();
  __syncwarp();
  for (int b = 0; b < g.B; ++b) {
    if (b > 0) {
      __syncwarp();
      stage(grid + (long long)b * g.grid_cells);
      cp_async_wait_all();
      __syncwarp();
    }
    C* fb = f + (long long)b * g.M;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (jn[u] < 0) continue;
      double frac;
      const int loc = node_cell(kn[u], g.Ntd[0], Nt, frac) - c0;
      if ((unsigned)loc >= (unsigned)Qt) continue;
      T w[2 * M];
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
      fb[jn[u]] = eval(loc, w);
    }
    for (int i = o0 + lane + 32 * U; i < o1; i += 32) {
      int j, loc;
      T w[2 * M];
      if (setup(i, j, loc, w)) fb[j] = eval(loc, w);
    }
  }
}

template <typename T, int M, int DEG>
__global__ void __launch_bounds__(W1_THREADS) spread1d_kernel(Geom g, WinPoly<T> wp,
                                                              const typename cplx<T>::type* __restrict__ f,
                                                              const T* __restrict__ ks, const int* __restrict__ perm,
                                                              const int* __restrict__ offsets, int nb, int ne,
                                                              typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int Nt = g.Nt[0], Q = g.Q[0], P = g.P[0];
  const int t = blockIdx.x * W1_WARPS + warp;
  if (t >= P) return;
  const int NB = Q + 2 * M - 1;  // bins: local cell x in [-m, Q + m - 2] -> x + m
  unsigned char* wbase = smem_raw + (size_t)warp * r1_spread_warp_bytes(Q, M, sizeof(C), sizeof(T));
  T* tap = reinterpret_cast<T*>(wbase);  // [S1_CAP][TAPS]
  C* fv = reinterpret_cast<C*>(wbase + (((size_t)S1_CAP * TAPS * sizeof(T) + 15) & ~(size_t)15));
  int* sbin = reinterpret_cast<int*>(fv + S1_CAP);  // [S1_CAP] bin of list entry e
  int* sj = sbin + S1_CAP;                          // [S1_CAP] node index j of list entry e
  int* start = sj + S1_CAP;                         // [NB + 1]
  int* cursor = start + NB + 1;                     // [NB + 1]
  int* list = cursor + NB + 1;                      // [S1_CAP + 32 S1_SCAN] kept candidates (sorted positions i)
  int* ord = list + S1_CAP + 32 * S1_SCAN;          // [S1_CAP] list entry of the q-th cell-sorted slot

  const int c0 = t * Q;
  const int tl = t == 0 ? P - 1 : t - 1, tr = t == P - 1 ? 0 : t + 1;
  const int a0 = max(__ldg(offsets + tl), nb), a1 = min(__ldg(offsets + tl + 1), ne);
  const int b0 = max(__ldg(offsets + t), nb), b1 = min(__ldg(offsets + t + 1), ne);
  const int e0 = max(__ldg(offsets + tr), nb), e1 = min(__ldg(offsets + tr + 1), ne);
  const int nA = max(0, a1 - a0), nBn = max(0, b1 - b0), nC = max(0, e1 - e0);
  const int n = nA + nBn + nC;
  const int sy0 = pos_mod(c0 - (Nt >> 1), Nt);  // storage of the tile's first cell (see interp1d)

  // Candidates are the own tile's nodes and the two neighbours' nodes; the latter are
  // filtered to those within m cells of the tile, so a typical tile is ONE chunk.
  int scanned = 0, have = 0;
  for (int chunk = 0; chunk == 0 || have > 0 || scanned < n; ++chunk) {
    while (have < S1_CAP && scanned < n) {  // fill the kept list, S1_SCAN candidates per lane in flight
      int ci[S1_SCAN];
      double kc[S1_SCAN];
#pragma unroll
      for (int v = 0; v < S1_SCAN; ++v) {
        const int u = scanned + v * 32 + lane;
        ci[v] = -1;
        if (u < n) {
          ci[v] = u < nA ? a0 + u : (u < nA + nBn ? b0 + (u - nA) : e0 + (u - nA - nBn));
          kc[v] = (double)ks[ci[v]];
        }
      }
#pragma unroll
      for (int v = 0; v < S1_SCAN; ++v) {
        const int u = scanned + v * 32 + lane;
        bool keep = false;
        if (ci[v] >= 0) {
          keep = u >= nA && u < nA + nBn;  // own tile
          if (!keep) {
            double frac;
            const int c = node_cell(kc[v], g.Ntd[0], Nt, frac);
            int x = c - c0;
            if (x > (Nt >> 1)) x -= Nt;
            else if (x < -(Nt >> 1)) x += Nt;
            keep = x >= -M && x <= Q + M - 2;
          }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        const int e = have + __popc(bal & lt);
        if (keep && e < S1_CAP + S1_SCAN * 32) list[e] = ci[v];
        have += __popc(bal);
      }
      scanned += 32 * S1_SCAN;
    }
    __syncwarp();
    const int cnt = min(have, S1_CAP);
    for (int k = lane; k <= NB; k += 32) start[k] = 0;
    __syncwarp();
    // taps, bin and value of list entry e go to slot e (unsorted); only indices are sorted
    for (int e = lane; e < cnt; e += 32) {
      const int i = list[e];
      double frac;
      const int c = node_cell((double)ks[i], g.Ntd[0], Nt, frac);
      int x = c - c0;
      if (x > (Nt >> 1)) x -= Nt;
      else if (x < -(Nt >> 1)) x += Nt;
      const int bin = min(max(x + M, 0), NB - 1);  // in range for list entries of a consistent plan
      const int j = perm[i];
      sj[e] = j;
      fv[e] = f[j];
      T w[TAPS];
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
#pragma unroll
      for (int l = 0; l < TAPS; ++l) tap[e * TAPS + l] = w[l];
      sbin[e] = bin;
      atomicAdd(&start[bin + 1], 1);
    }
    __syncwarp();
    {
      const int per = (NB + 1 + 31) / 32;
      const int lo = lane * per, hi = min(NB + 1, lo + per);
      int sum = 0;
      for (int k = lo; k < hi; ++k) sum += start[k];
      int total;
      int run = warp_exclusive_scan(sum, total);
      for (int k = lo; k < hi; ++k) {
        run += start[k];
        start[k] = run;  // first slot of bin k (start[0] = 0); start[NB] = slots in chunk
        cursor[k] = run;
      }
    }
    __syncwarp();
    for (int e = lane; e < cnt; e += 32) ord[atomicAdd(&cursor[sbin[e]], 1)] = e;
    __syncwarp();
    for (int k = lane; k < have - cnt; k += 32) list[k] = list[S1_CAP + k];  // leftovers move to the front
    have -= cnt;
    const int nslots = cnt;
    for (int b = 0; b < g.B; ++b) {
      if (b > 0) {
        const C* fb = f + (long long)b * g.M;
        __syncwarp();
        for (int q = lane; q < nslots; q += 32) fv[q] = fb[sj[q]];  // slot q = list entry q
        __syncwarp();
      }
      C* dst = grid + (long long)b * g.grid_cells;
      for (int y = lane; y < Q; y += 32) {
        const int q0 = start[y], q1 = start[y + TAPS];
        C acc;
        acc.x = (T)0;
        acc.y = (T)0;
        for (int q = q0; q < q1; ++q) {
          const int e = ord[q];
          const T wt = tap[e * TAPS + (y - sbin[e] + TAPS - 1)];
          const C v = fv[e];
          acc.x = fma(wt, v.x, acc.x);
          acc.y = fma(wt, v.y, acc.y);
        }
        int sy = sy0 + y;
        if (sy >= Nt) sy -= Nt;
        if (chunk == 0) {
          dst[sy] = acc;
        } else {  // later chunks of an over-full tile: this lane owns cell y in every chunk
          C o = dst[sy];
          o.x += acc.x;
          o.y += acc.y;
          dst[sy] = o;
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace nfftb
