// resample_cell.cuh — forward interpolation and adjoint spreading for D = 2, 3
// over CELL-SORTED nodes (cellbin.cuh).
//
//   forward: f_j = sum_{l in I_{Nt,m}(k_j)} ghat_l psi~(k_j - l/Nt)   (Alg. 3)
//   adjoint: ghat_l = sum_j f_j psi~(k_j - l/Nt)                       (Alg. 4)
//
// Work tiles (the paper's blocks) are defined by the kernels:
// one CTA per tile of Q_0 x ... x Q_{D-1} cells. Because the nodes are sorted by
// row-major cell index, the nodes of any run of cells along the last dimension
// are one contiguous range [cstart[a], cstart[b + 1]).
//
// interp_cell: the tile's block index set (Q_d + 2m - 1 cells per dimension,
//   wrap resolved at staging, Remark PAPER.md:588-590) is staged in shared
//   memory with cp.async, one warp per region row; the tile's nodes are the
//   union of its rows' node ranges (flattened with a prefix over the rows);
//   per node the separable taps and the (2m)^D tensor sum,
//   innermost dimension contiguous, bank-rotated row sums.
// spread_cell: OWNER-COMPUTES. The CTA writes every cell of its tile exactly
//   once with plain stores: it stages the nodes of the tile's WINDOW (cells
//   within [-m, Q + m - 2] of the tile in every dimension, wrap included),
//   i.e. the nodes whose footprint reaches the tile, with their taps, and every
//   thread gathers K consecutive cells along the last dimension:
//     ghat_y = sum over the (2m)^(D-1) window rows x_lead in reach of y_lead,
//              over the nodes of window cells [y_last - m, y_last + K + m - 2]
//              (one contiguous slot range per row),
//              f_j prod_{d<D-1} w_d[y_d - x_d + m - 1] * w_last[y_last + k - x_last + m - 1].
//   The last-dimension taps are stored zero-padded so the K cells use one
//   contiguous slice without branches. No atomics, no zero pass, no halo merge
//   (the paper's locked merge, becomes reading halo NODES).
#pragma once

#include "resample.cuh"

namespace nfftb {

constexpr int RC_THREADS = 256;  // interp_cell
constexpr int SC_K = 4;          // spread_cell: consecutive last-dimension cells per thread

// ---------------------------------------------------------------- forward
template <typename T, int D, int M, int DEG, bool TENSOR>
__global__ void __launch_bounds__(RC_THREADS, D == 2 ? 4 : 2) interp_cell_kernel(Geom g, WinPolyN<T, D, M> wp,
                                                                 const typename cplx<T>::type* __restrict__ grid,
                                                                 const T* __restrict__ kc, const T* __restrict__ wt,
                                                                 const int* __restrict__ jc,
                                                                 const int* __restrict__ cstart, int nb, int ne,
                                                                 typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  constexpr int TP = RotCfg<T, M>::TP;
  constexpr int EXT = (TP > 2 * M ? TP : 2 * M) - 1;
  constexpr int MAXROWS = 1024;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int rpre[MAXROWS + 1];  // prefix of the tile rows' node counts
  __shared__ int rbeg[MAXROWS];      // first cell-sorted position of every tile row
  __shared__ int ws[32];
  C* tile = reinterpret_cast<C*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x;
  int c0[D], s0[D], Rr[D], Qt[D];
  {
    int rem = t;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      const int p = rem % g.P[d];
      rem /= g.P[d];
      c0[d] = p * g.Q[d];
      Qt[d] = min(g.Q[d], g.Nt[d] - c0[d]);
      Rr[d] = Qt[d] + (d == D - 1 ? EXT : 2 * M - 1);  // staged extent
      // binning cell c = (a + Nt/2) mod Nt <-> storage (a mod Nt) = (c - Nt/2) mod Nt
      s0[d] = pos_mod(c0[d] - M + 1 - (g.Nt[d] >> 1), g.Nt[d]);
    }
  }
  const int Lp = g.L[D - 1];  // region row pitch (cells): >= Q + EXT, multiple of 8 for C128
  const int R1 = D == 3 ? g.L[1] : 1;
  auto stage = [&](const C* src) {
    // warp w stages region rows w, w + 8, ...; the row's (i0, i1) and its wrapped source rows advance
    // incrementally (no division / modulo per row)
    const int rows = D == 2 ? Rr[0] : Rr[0] * Rr[1];
    const int NtL = g.Nt[D - 1];
    constexpr int NWS = RC_THREADS / 32;
    int i0 = D == 2 ? warp : warp / Rr[1], i1 = D == 2 ? 0 : warp - (warp / Rr[1]) * Rr[1];
    int sa = s0[0] + i0, sb = D == 3 ? s0[1] + i1 : 0;
    while (sa >= g.Nt[0]) sa -= g.Nt[0];
    if (D == 3)
      while (sb >= g.Nt[1]) sb -= g.Nt[1];
    for (int r = warp; r < rows; r += NWS) {
      const long long off = D == 2 ? (long long)sa * NtL : ((long long)sa * g.Nt[1] + sb) * NtL;
      const int srow = D == 2 ? i0 : i0 * R1 + i1;
      const C* rsrc = src + off;
      C* rdst = tile + (long long)srow * Lp;
      for (int col = lane; col < Rr[D - 1]; col += 32) {
        int sc = s0[D - 1] + col;
        while (sc >= NtL) sc -= NtL;
        cp_async_cell<T>(rdst + col, rsrc + sc);
      }
      // next row: r + NWS
      if (D == 2) {
        i0 += NWS;
        sa += NWS;
        while (sa >= g.Nt[0]) sa -= g.Nt[0];
      } else {
        i1 += NWS;
        sb += NWS;
        while (i1 >= Rr[1]) {  // carry into dimension 0
          i1 -= Rr[1];
          sb -= Rr[1];
          ++i0;
          if (++sa >= g.Nt[0]) sa -= g.Nt[0];
        }
        while (sb >= g.Nt[1]) sb -= g.Nt[1];
        while (sb < 0) sb += g.Nt[1];
      }
    }
  };
  const int b = blockIdx.y;  // batch vector of this CTA (config 5: B = 32 CTAs per tile)
  // the tile's nodes: one cell-sorted range per tile row (all but the last dimension); independent of
  // the grid, so under programmatic dependent launch this overlaps the FFT's tail
  const int nrows = D == 2 ? Qt[0] : Qt[0] * Qt[1];
  {
    const int per = (nrows + RC_THREADS - 1) / RC_THREADS;
    const int lo = threadIdx.x * per, hi = min(nrows, lo + per);
    int cnt = 0;
    for (int r = lo; r < hi; ++r) {
      long long key;
      if (D == 2) {
        key = (long long)(c0[0] + r) * g.Nt[1] + c0[1];
      } else {
        const int r0 = r / Qt[1], r1 = r - r0 * Qt[1];
        key = ((long long)(c0[0] + r0) * g.Nt[1] + c0[1] + r1) * g.Nt[2] + c0[2];
      }
      const int a = max(cstart[key], nb), b = min(cstart[key + Qt[D - 1]], ne);
      rbeg[r] = a;
      rpre[r] = max(0, b - a);
      cnt += max(0, b - a);
    }
    int tot;
    int run = block_exclusive_scan(cnt, ws, tot);
    for (int r = lo; r < hi; ++r) {
      const int c = rpre[r];
      rpre[r] = run;
      run += c;
    }
    if (threadIdx.x == 0) rpre[nrows] = tot;
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the grid (previous kernel's output) is complete
  stage(grid + (long long)b * g.grid_cells);
  const int total = rpre[nrows];
  auto position = [&](int q) {  // q-th node of the tile -> cell-sorted position (binary search over rows)
    int lo = 0, hi = nrows;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rpre[mid] <= q) lo = mid;
      else hi = mid;
    }
    return rbeg[lo] + (q - rpre[lo]);
  };
  auto node = [&](int pos, int (&loc)[D], T (&w)[D][2 * M]) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double frac;
      loc[d] = node_cell((double)kc[(long long)d * g.M + pos], g.Ntd[d], g.Nt[d], frac) - c0[d];
      if constexpr (TENSOR) {  // the stored taps wt[pos][d][t]
#pragma unroll
        for (int t = 0; t < 2 * M; ++t) w[d][t] = __ldg(wt + ((long long)pos * D + d) * 2 * M + t);
      } else {
        window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w[d]);
      }
    }
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
  // first node of every thread: position and node index loaded before the region wait
  const int q0 = threadIdx.x;
  const int pos0 = q0 < total ? position(q0) : 0;
  const int j0 = q0 < total ? jc[pos0] : -1;
  cp_async_wait_all();
  __syncthreads();
  C* fb = f + (long long)b * g.M;
  for (int q = q0; q < total; q += RC_THREADS) {
    const int pos = q == q0 ? pos0 : position(q);
    const int j = q == q0 ? j0 : jc[pos];
    int loc[D];
    T w[D][2 * M];
    node(pos, loc, w);
    fb[j] = eval(loc, w);
  }
}

// interp_cell2: the same forward interpolation for fp32 2D BATCHES with TWO
// vectors per CTA (config 5). The region is staged interleaved, one 16-byte
// element (vector b, vector b + 1) per cell, so the node's position, taps
// (evaluated once for both vectors) and the (2m)^2 region reads (LDS.128: 8
// lanes per shared-memory phase, half the conflict exposure of 16 lanes of
// 8-byte reads) serve two outputs; the multiply-adds are packed FFMA2.
#ifndef NFFTB_IC2_MINB
#define NFFTB_IC2_MINB 3
#endif
template <int M, int DEG>
__global__ void __launch_bounds__(RC_THREADS, NFFTB_IC2_MINB) interp_cell2_kernel(Geom g, WinPolyN<float, 2, M> wp,
                                                                     const float2* __restrict__ grid,
                                                                     const float* __restrict__ kc,
                                                                     const int* __restrict__ jc,
                                                                     const int* __restrict__ cstart,
                                                                     float2* __restrict__ f) {
  constexpr int EXT = 2 * M - 1;
  constexpr int MAXROWS = 1024;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int rpre[MAXROWS + 1];
  __shared__ int rbeg[MAXROWS];
  __shared__ int ws[32];
  float4* tile = reinterpret_cast<float4*>(smem_raw);  // [region cell] = (vector b0, vector b0 + 1)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c0[2], s0[2], Rr[2], Qt[2];
  {
    int rem = blockIdx.x;
#pragma unroll
    for (int d = 1; d >= 0; --d) {
      const int p = rem % g.P[d];
      rem /= g.P[d];
      c0[d] = p * g.Q[d];
      Qt[d] = min(g.Q[d], g.Nt[d] - c0[d]);
      Rr[d] = Qt[d] + EXT;
      s0[d] = pos_mod(c0[d] - M + 1 - (g.Nt[d] >> 1), g.Nt[d]);
    }
  }
  const int Lp = g.L[1];
  const int b0 = blockIdx.y * 2;
  const bool two = b0 + 1 < g.B;
  // the tile's nodes: one cell-sorted range per tile row (overlaps the FFT's tail under PDL)
  const int nrows = Qt[0];
  {
    const int per = (nrows + RC_THREADS - 1) / RC_THREADS;
    const int lo = threadIdx.x * per, hi = min(nrows, lo + per);
    int cnt = 0;
    for (int r = lo; r < hi; ++r) {
      const long long key = (long long)(c0[0] + r) * g.Nt[1] + c0[1];
      const int a = cstart[key], b = cstart[key + Qt[1]];
      rbeg[r] = a;
      rpre[r] = b - a;
      cnt += b - a;
    }
    int tot;
    int run = block_exclusive_scan(cnt, ws, tot);
    for (int r = lo; r < hi; ++r) {
      const int c = rpre[r];
      rpre[r] = run;
      run += c;
    }
    if (threadIdx.x == 0) rpre[nrows] = tot;
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the grid (previous kernel's output) is complete
  {  // stage both vectors' regions, interleaved (8-byte cp.async per cell and vector; zero fill past B)
    const float2* g0 = grid + (long long)b0 * g.grid_cells;
    const float2* g1 = two ? g0 + g.grid_cells : g0;
    const int NtL = g.Nt[1];
    int sa = s0[0] + warp;
    while (sa >= g.Nt[0]) sa -= g.Nt[0];
    for (int r = warp; r < Rr[0]; r += RC_THREADS / 32) {
      const long long off = (long long)sa * NtL;
      for (int col = lane; col < Rr[1]; col += 32) {
        int sc = s0[1] + col;
        while (sc >= NtL) sc -= NtL;
        const unsigned d = (unsigned)__cvta_generic_to_shared(tile + (size_t)r * Lp + col);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(g0 + off + sc) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d + 8), "l"(g1 + off + sc),
                     "r"(two ? 8 : 0)
                     : "memory");
      }
      sa += RC_THREADS / 32;
      while (sa >= g.Nt[0]) sa -= g.Nt[0];
    }
  }
  const int total = rpre[nrows];
  auto position = [&](int q) {
    int lo = 0, hi = nrows;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rpre[mid] <= q) lo = mid;
      else hi = mid;
    }
    return rbeg[lo] + (q - rpre[lo]);
  };
  const int q0 = threadIdx.x;
  const int pos0 = q0 < total ? position(q0) : 0;
  const int j0 = q0 < total ? jc[pos0] : -1;
  cp_async_wait_all();
  __syncthreads();
  float2* f0 = f + (long long)b0 * g.M;
  for (int q = q0; q < total; q += RC_THREADS) {
    const int pos = q == q0 ? pos0 : position(q);
    const int j = q == q0 ? j0 : jc[pos];
    int loc[2];
    float w[2][2 * M];
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double frac;
      loc[d] = node_cell((double)kc[(long long)d * g.M + pos], g.Ntd[d], g.Nt[d], frac) - c0[d];
      window_taps<float, M, DEG>((float)(frac - 0.5), wp.mu[d], w[d]);
    }
    float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
    // 2m = 8 or 16: bank rotation. Lane L reads element (k + rot) mod 2m at step k, rot = (L - loc) mod 2m,
    // so with a pitch that is a multiple of 8 elements the 8 lanes of each 16-byte shared-memory phase
    // touch 8 distinct bank quads whatever the node positions (the taps rotate with them)
    constexpr bool ROT = 2 * M == 8 || 2 * M == 16;
    float wl[2 * M];
    int off[2 * M];
    if constexpr (ROT) {
      const int rot = (lane - loc[1]) & (2 * M - 1);
      rotate_taps<float, M, 2 * M>(w[1], rot, wl);
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) off[k] = (k + rot) & (2 * M - 1);
    } else {
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) {
        wl[k] = w[1][k];
        off[k] = k;
      }
    }
#pragma unroll
    for (int l0 = 0; l0 < 2 * M; ++l0) {
      const float4* row = tile + (loc[0] + l0) * Lp + loc[1];
      float2 s0v = make_float2(0.f, 0.f), s1v = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < 2 * M; ++k) {
        const float4 v = row[off[k]];
        s0v = __ffma2_rn(make_float2(wl[k], wl[k]), make_float2(v.x, v.y), s0v);
        s1v = __ffma2_rn(make_float2(wl[k], wl[k]), make_float2(v.z, v.w), s1v);
      }
      a0 = __ffma2_rn(make_float2(w[0][l0], w[0][l0]), s0v, a0);
      a1 = __ffma2_rn(make_float2(w[0][l0], w[0][l0]), s1v, a1);
    }
    f0[j] = a0;
    if (two) f0[g.M + j] = a1;
  }
}

// ---------------------------------------------------------------- adjoint
// shared memory per staged node slot (host and device agree)
template <typename T, int D, int M>
struct SpreadCellCfg {
  static constexpr int TL = ((2 * M + 2 * SC_K - 2) + 1) & ~1;  // padded last-dim taps (even)
  static constexpr int NREAL = (D - 1) * 2 * M + TL;            // reals per slot
  static constexpr int SLOT = (int)(NREAL * sizeof(T) + 2 * sizeof(T) + 4);  // + value + window col
};

__host__ __device__ inline size_t spread_cell_smem_bytes(int D, int M, int rsize, int cap, int wrows, int wcols) {
  const int TL = ((2 * M + 2 * SC_K - 2) + 1) & ~1;
  const size_t nreal = (size_t)(D - 1) * 2 * M + TL;
  size_t b = (size_t)cap * (nreal * rsize + 2 * rsize);  // taps, value
  b = (b + 15) & ~(size_t)15;
  b += (size_t)cap * 4;                                  // window col of the slot
  b += (size_t)wrows * (wcols + 1) * 4;                  // per window cell: first slot
  b += (size_t)(wrows * 4 + 4) * 4;                      // per window row: slot base, segA pos, segA len, segB pos
  return (b + 15) & ~(size_t)15;
}

template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(256) spread_cell_kernel(Geom g, WinPolyN<T, D, M> wp,
                                                          const typename cplx<T>::type* __restrict__ f,
                                                          const T* __restrict__ kc, const int* __restrict__ jc,
                                                          const int* __restrict__ cstart, int nb, int ne, int cap,
                                                          typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  using Cfg = SpreadCellCfg<T, D, M>;
  constexpr int TL = Cfg::TL;
  constexpr int NR = Cfg::NREAL;
  constexpr int LEAD = D - 1;
  constexpr int TAPS = 2 * M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int ws[32];
  const int tid = threadIdx.x;
  const int t = blockIdx.x;
  int c0[D], Qt[D], Lw[D];
  {
    int rem = t;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      const int p = rem % g.P[d];
      rem /= g.P[d];
      c0[d] = p * g.Q[d];
      Qt[d] = min(g.Q[d], g.Nt[d] - c0[d]);
      Lw[d] = Qt[d] + 2 * M - 1;  // window extent: tile-local cells [-m, Qt + m - 2]
    }
  }
  const int wrows = D == 2 ? Lw[0] : Lw[0] * Lw[1];
  const int wcols = Lw[D - 1];
  const int NtL = g.Nt[D - 1];
  // shared layout
  T* sreal = reinterpret_cast<T*>(smem_raw);                                  // [cap][NR + 2]
  size_t off = ((size_t)cap * (NR + 2) * sizeof(T) + 15) & ~(size_t)15;
  int* scol = reinterpret_cast<int*>(smem_raw + off);                         // [cap]
  int* wcs = scol + cap;                                                      // [wrows][wcols + 1]
  int* rbase = wcs + (size_t)wrows * (wcols + 1);                            // [wrows + 1]
  int* rposA = rbase + wrows + 1;                                             // [wrows]
  int* rlenA = rposA + wrows;                                                 // [wrows]
  int* rposB = rlenA + wrows;                                                 // [wrows]

  // ---- window rows: node ranges of the (<= 2, wrap) last-dimension segments
  const int a_last = c0[D - 1] - M;            // first window col in binning coordinates (may be < 0)
  const int b_last = c0[D - 1] + Qt[D - 1] + M - 2;  // last (may be >= Nt)
  {
    const int per = (wrows + blockDim.x - 1) / blockDim.x;
    const int lo = tid * per, hi = min(wrows, lo + per);
    int cnt = 0;
    for (int r = lo; r < hi; ++r) {
      long long rowkey;
      if (D == 2) {
        rowkey = (long long)pos_mod(c0[0] - M + r, g.Nt[0]) * NtL;
      } else {
        const int r0 = r / Lw[1], r1 = r - r0 * Lw[1];
        rowkey = ((long long)pos_mod(c0[0] - M + r0, g.Nt[0]) * g.Nt[1] + pos_mod(c0[1] - M + r1, g.Nt[1])) * NtL;
      }
      // segment A: window cols whose binning col is a_last.. (wrapped into [0, Nt)), up to the row end
      int ea = a_last, eb = b_last;
      int pA, lA, pB = 0, lB = 0;
      if (ea < 0) {  // wraps at the left: [Nt + ea, Nt - 1] then [0, eb]
        pA = cstart[rowkey + NtL + ea];
        lA = cstart[rowkey + NtL] - pA;
        pB = cstart[rowkey];
        lB = cstart[rowkey + eb + 1] - pB;
      } else if (eb >= NtL) {  // wraps at the right: [ea, Nt - 1] then [0, eb - Nt]
        pA = cstart[rowkey + ea];
        lA = cstart[rowkey + NtL] - pA;
        pB = cstart[rowkey];
        lB = cstart[rowkey + eb - NtL + 1] - pB;
      } else {
        pA = cstart[rowkey + ea];
        lA = cstart[rowkey + eb + 1] - pA;
      }
      rposA[r] = pA;
      rlenA[r] = lA;
      rposB[r] = pB;
      rbase[r] = lA + lB;
      cnt += lA + lB;
    }
    int tot;
    int run = block_exclusive_scan(cnt, ws, tot);
    for (int r = lo; r < hi; ++r) {
      const int c = rbase[r];
      rbase[r] = run;
      run += c;
    }
    if (tid == 0) rbase[wrows] = tot;
  }
  __syncthreads();
  // per window cell: first slot (row-major window order)
  for (int idx = tid; idx < wrows * wcols; idx += blockDim.x) {
    const int r = idx / wcols, wc = idx - r * wcols;
    long long rowkey;
    if (D == 2) {
      rowkey = (long long)pos_mod(c0[0] - M + r, g.Nt[0]) * NtL;
    } else {
      const int r0 = r / Lw[1], r1 = r - r0 * Lw[1];
      rowkey = ((long long)pos_mod(c0[0] - M + r0, g.Nt[0]) * g.Nt[1] + pos_mod(c0[1] - M + r1, g.Nt[1])) * NtL;
    }
    const int bc = a_last + wc;  // binning col of window col wc (may be < 0 or >= Nt)
    int slot;
    if (a_last < 0) {  // left wrap: segment A = binning cols [Nt + a_last, Nt), segment B = [0, b_last]
      slot = bc < 0 ? rbase[r] + cstart[rowkey + NtL + bc] - rposA[r]
                    : rbase[r] + rlenA[r] + cstart[rowkey + bc] - rposB[r];
    } else if (b_last >= NtL) {  // right wrap: segment A = [a_last, Nt), segment B = [0, b_last - Nt]
      slot = bc < NtL ? rbase[r] + cstart[rowkey + bc] - rposA[r]
                      : rbase[r] + rlenA[r] + cstart[rowkey + bc - NtL] - rposB[r];
    } else {
      slot = rbase[r] + cstart[rowkey + bc] - rposA[r];
    }
    wcs[(size_t)r * (wcols + 1) + wc] = slot;
  }
  for (int r = tid; r < wrows; r += blockDim.x) wcs[(size_t)r * (wcols + 1) + wcols] = rbase[r + 1];
  __syncthreads();
  const int total = rbase[wrows];

  // ---- owned cells: thread item = (lead cell, group of SC_K last-dim cells)
  const int ngrp = (Qt[D - 1] + SC_K - 1) / SC_K;
  const int nlead = D == 2 ? Qt[0] : Qt[0] * Qt[1];
  const int nitems = nlead * ngrp;
  constexpr int MAXIT = 2;  // items per thread (Q <= 32 x 32 in 2D, 8 x 8 x 16 in 3D with 256 threads)
  auto row_of_slot = [&](int s) {
    int lo = 0, hi = wrows;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rbase[mid] <= s) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  {
    const int b = blockIdx.y;  // batch vector of this CTA
    C acc[MAXIT][SC_K];
#pragma unroll
    for (int it = 0; it < MAXIT; ++it)
#pragma unroll
      for (int k = 0; k < SC_K; ++k) {
        acc[it][k].x = (T)0;
        acc[it][k].y = (T)0;
      }
    for (int clo = 0; clo < total || (clo == 0 && total == 0); clo += cap) {
      const int chi = min(total, clo + cap);
      __syncthreads();
      // stage the chunk's nodes: taps (lead dims, padded last dim), value, window col
      for (int s = clo + tid; s < chi; s += blockDim.x) {
        const int r = row_of_slot(s);
        const int within = s - rbase[r];
        const int pos = within < rlenA[r] ? rposA[r] + within : rposB[r] + (within - rlenA[r]);
        T* rs = sreal + (size_t)(s - clo) * (NR + 2);
        int jn = jc[pos];
        if (pos < nb || pos >= ne) jn = -1;  // outside the node shard: contributes zero
        int lastcol = 0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          double frac;
          const int c = node_cell((double)kc[(long long)d * g.M + pos], g.Ntd[d], g.Nt[d], frac);
          T w[TAPS];
          window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w);
          if (d < LEAD) {
#pragma unroll
            for (int l = 0; l < TAPS; ++l) rs[d * TAPS + l] = w[l];
          } else {
            int wc = c - a_last;  // window col (wrap-aware)
            if (wc < 0) wc += NtL;
            if (wc >= NtL) wc -= NtL;
            lastcol = wc;
#pragma unroll
            for (int l = 0; l < TL; ++l) {
              const int lt = l - (SC_K - 1);
              rs[LEAD * TAPS + l] = (lt >= 0 && lt < TAPS) ? w[lt] : (T)0;
            }
          }
        }
        C v;
        v.x = (T)0;
        v.y = (T)0;
        if (jn >= 0) v = f[(long long)b * g.M + jn];
        rs[NR] = v.x;
        rs[NR + 1] = v.y;
        scol[s - clo] = lastcol;
      }
      __syncthreads();
#pragma unroll
      for (int it = 0; it < MAXIT; ++it) {
        const int item = tid + it * blockDim.x;
        if (item >= nitems) continue;
        const int lead = item / ngrp, grp = item - lead * ngrp;
        const int y_last = grp * SC_K;
        int y0 = lead, y1 = 0;
        if (D == 3) {
          y0 = lead / Qt[1];
          y1 = lead - y0 * Qt[1];
        }
        // contributing window rows: wr_d in [y_d, y_d + 2m - 1] per lead dim
        for (int l0 = 0; l0 < TAPS; ++l0) {
          const int wr0 = y0 + TAPS - 1 - l0;  // l0 = y0 - wr0 + 2m - 1
          for (int l1 = 0; l1 < (D == 3 ? TAPS : 1); ++l1) {
            const int wr1 = D == 3 ? y1 + TAPS - 1 - l1 : 0;
            const int r = D == 2 ? wr0 : wr0 * Lw[1] + wr1;
            const int* rw = wcs + (size_t)r * (wcols + 1);
            const int s0 = max(rw[y_last], clo), s1 = min(rw[min(y_last + SC_K + 2 * M - 1, wcols)], chi);
            for (int s = s0; s < s1; ++s) {
              const T* rs = sreal + (size_t)(s - clo) * (NR + 2);
              T cw = rs[l0];
              if (D == 3) cw *= rs[TAPS + l1];
              const T vx = cw * rs[NR], vy = cw * rs[NR + 1];
              const int base = y_last - scol[s - clo] + 2 * M - 1 + (SC_K - 1);  // padded last-dim tap of cell y_last
#pragma unroll
              for (int k = 0; k < SC_K; ++k) {
                const T wl = rs[LEAD * TAPS + base + k];
                acc[it][k].x = fma(wl, vx, acc[it][k].x);
                acc[it][k].y = fma(wl, vy, acc[it][k].y);
              }
            }
          }
        }
      }
    }
    // plain stores of the owned cells (storage = (binning cell - Nt/2) mod Nt)
    C* dst = grid + (long long)b * g.grid_cells;
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int item = tid + it * blockDim.x;
      if (item >= nitems) continue;
      const int lead = item / ngrp, grp = item - lead * ngrp;
      long long rowoff;
      if (D == 2) {
        rowoff = (long long)pos_mod(c0[0] + lead - (g.Nt[0] >> 1), g.Nt[0]) * NtL;
      } else {
        const int y0 = lead / Qt[1], y1 = lead - y0 * Qt[1];
        rowoff = ((long long)pos_mod(c0[0] + y0 - (g.Nt[0] >> 1), g.Nt[0]) * g.Nt[1] +
                  pos_mod(c0[1] + y1 - (g.Nt[1] >> 1), g.Nt[1])) * NtL;
      }
#pragma unroll
      for (int k = 0; k < SC_K; ++k) {
        const int yl = grp * SC_K + k;
        if (yl < Qt[D - 1]) dst[rowoff + pos_mod(c0[D - 1] + yl - (NtL >> 1), NtL)] = acc[it][k];
      }
    }
  }
}

}  // namespace nfftb
