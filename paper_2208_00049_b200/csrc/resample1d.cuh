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
constexpr int S1_K = 2;                   // spread1c: cells per lane
constexpr int S1_SEG = 32 * S1_K;         // cells per warp
constexpr int S1_CAP = 64;                // node slots per warp chunk (typical window: ~0.5 (SEG + 2m) nodes)


// ---------------------------------------------------------------- forward
template <typename T, int M, int DEG>
__global__ void __launch_bounds__(I1_THREADS) interp1c_kernel(Geom g, WinPoly<T> wp,
                                                              const typename cplx<T>::type* __restrict__ grid,
                                                              const T* __restrict__ kc, const int* __restrict__ jc,
                                                              int nb, int ne, int sharded,
                                                              typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  for (int pc = blockIdx.x * I1_THREADS + threadIdx.x; pc < g.M; pc += gridDim.x * I1_THREADS) {
  if (sharded && (pc < nb || pc >= ne)) continue;  // shard = range of the cell-sorted order
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
  }  // nodes
}

// ---------------------------------------------------------------- adjoint
// spread1c: one warp per segment of S1_SEG cells (owner-computes). The warp
// stages the nodes of its WINDOW (cells [y0 - m, y0 + SEG + m - 2], i.e. every
// node whose footprint reaches the segment; contiguous cell-sorted ranges from
// cstart) and spreads them TAP-PARALLEL: the warp is split into groups of G =
// 8 (m <= 4) or 16 lanes; a group takes one node, lane l evaluates tap l
// (coefficients of its mirror pair in registers) and the tap is shuffled to
// the lane that owns its cell: lane q always owns the cells i = q (mod G) of
// the group's private shared-memory accumulator (no two lanes ever touch the
// same cell: no conflict, no atomic, no barrier between nodes). The groups' copies are
// summed when the segment's cells are written, each exactly once, with plain
// coalesced stores (no zero pass, no halo merge: the paper's locked merge of
// PAPER.md:578-582 becomes reading the halo NODES).
template <int M>
struct S1Cfg {
  static constexpr int G = 2 * M <= 8 ? 8 : 16;   // lanes per node
  static constexpr int NG = 32 / G;               // nodes per warp step = accumulator copies
  static constexpr int NE = S1_SEG + 2 * M - 1;   // window cells (full segment)
  static constexpr int LEN = NE + 2 * M - 1;      // accumulator cells: window cell e, tap l -> e + l
};

// shared memory of one spread1c warp (host and device agree)
__host__ __device__ inline size_t s1_warp_bytes(int M, size_t csize, size_t rsize) {
  const int G = 2 * M <= 8 ? 8 : 16, NG = 32 / G;
  const int NE = S1_SEG + 2 * M - 1, LEN = NE + 2 * M - 1;
  size_t b = (size_t)NG * LEN * csize;                // accumulator copies
  b += (size_t)S1_CAP * (csize + rsize);              // staged node: value, zeta
  b += (size_t)S1_CAP * 4;                            // staged node: window cell
  b += (size_t)(2 * NE + 2) * 4;                      // per window cell: first slot, position base
  return (b + 15) & ~(size_t)15;
}

template <typename T, int M, int DEG>
__global__ void __launch_bounds__(32 * S1_WARPS) spread1c_kernel(Geom g, WinPoly<T> wp,
                                                                 const typename cplx<T>::type* __restrict__ f,
                                                                 const T* __restrict__ kc, const int* __restrict__ jc,
                                                                 const int* __restrict__ cstart, int nb, int ne,
                                                                 int sharded, typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  using Cfg = S1Cfg<M>;
  constexpr int TAPS = 2 * M, G = Cfg::G, NG = Cfg::NG, LEN = Cfg::LEN;
  constexpr int PER = (Cfg::NE + 1 + 31) / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Nt = g.Nt[0];
  // grid-stride over the warp segments (the launch may use fewer CTAs than segments)
  for (int wseg = blockIdx.x * S1_WARPS + warp;; wseg += gridDim.x * S1_WARPS) {
  const int y0 = wseg * S1_SEG;
  if (y0 >= Nt) break;
  const int nseg = min(S1_SEG, Nt - y0);
  const int NE = nseg + 2 * M - 1;  // window cell e <-> binning cell (y0 - m + e) mod Nt
  unsigned char* wb = smem_raw + (size_t)warp * s1_warp_bytes(M, sizeof(C), sizeof(T));
  C* acc = reinterpret_cast<C*>(wb);                 // [NG][LEN]: cell y0 - 2m + 1 + i
  C* sv = acc + NG * LEN;                            // [S1_CAP] node value
  T* sz = reinterpret_cast<T*>(sv + S1_CAP);         // [S1_CAP] zeta = frac - 1/2
  int* se = reinterpret_cast<int*>(sz + S1_CAP);     // [S1_CAP] window cell
  int* ws = se + S1_CAP;                             // [NE + 1] first window slot of window cell e
  int* wbase = ws + Cfg::NE + 1;                     // [NE] position of slot s of cell e = wbase[e] + s

  // window slot starts: the lane's cstart loads issued together, warp scan of the counts
  int total;
  {
    int c_lo[PER], c_hi[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = lane * PER + q;
      c_lo[q] = c_hi[q] = 0;
      if (e < NE) {
        int c = y0 - M + e;
        if (c < 0) c += Nt;
        if (c >= Nt) c -= Nt;
        if ((unsigned)c >= (unsigned)Nt) c = pos_mod(c, Nt);
        c_lo[q] = __ldg(cstart + c);
        c_hi[q] = __ldg(cstart + c + 1);
      }
    }
    int sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) sum += c_hi[q] - c_lo[q];
    int run = warp_exclusive_scan(sum, total);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = lane * PER + q;
      if (e <= NE) ws[e] = run;
      if (e < NE) wbase[e] = c_lo[q] - run;
      run += c_hi[q] - c_lo[q];
    }
  }
  // tap of this lane and the coefficients of its mirror pair (w_l = E + zeta O, w_{2m-1-l} = E - zeta O)
  const int grp = lane / G, l = lane % G;
  const bool tap_on = l < TAPS;
  const int lp = l < M ? l : (TAPS - 1 - l);
  const T sgn = l < M ? (T)1 : (T)-1;
  T ce[DEG / 2 + 1], co[(DEG + 1) / 2];
#pragma unroll
  for (int z = 0; z <= DEG; ++z) {
    const T c = tap_on ? wp.mu[0][lp < M ? lp : 0][z] : (T)0;
    if (z % 2 == 0) ce[z / 2] = c;
    else co[z / 2] = c;
  }
  __syncwarp();
  const int sy0 = pos_mod(y0 - (Nt >> 1), Nt);  // storage of binning cell y0
  for (int b = 0; b < g.B; ++b) {
    for (int i = lane; i < NG * LEN; i += 32) {
      acc[i].x = (T)0;
      acc[i].y = (T)0;
    }
    for (int clo = 0; clo < max(total, 1); clo += S1_CAP) {
      const int chi = min(total, clo + S1_CAP);
      // stage the chunk: window cell, zeta and value of every slot (loads of all the lane's slots in flight)
      constexpr int SPL = (S1_CAP + 31) / 32;
      int jj[SPL], ee[SPL];
      double kk[SPL];
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        const int sl = clo + lane + 32 * u;
        jj[u] = -1;
        ee[u] = -1;
        if (sl < chi) {
          int lo = 0, hi = NE;  // window cell of the slot: last e with ws[e] <= sl
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (ws[mid] <= sl) lo = mid;
            else hi = mid;
          }
          const int pc = wbase[lo] + sl;
          ee[u] = lo;
          jj[u] = (sharded && (pc < nb || pc >= ne)) ? -1 : jc[pc];  // shard = range of the cell order
          kk[u] = (double)kc[pc];
        }
      }
#pragma unroll
      for (int u = 0; u < SPL; ++u) {
        const int sl = lane + 32 * u;
        if (ee[u] >= 0) {
          C v;
          v.x = (T)0;
          v.y = (T)0;
          if (jj[u] >= 0) v = f[(long long)b * g.M + jj[u]];
          double frac;
          node_cell(kk[u], g.Ntd[0], Nt, frac);
          sv[sl] = v;
          sz[sl] = (T)(frac - 0.5);
          se[sl] = ee[u];
        }
      }
      __syncwarp();
      // tap-parallel accumulation: group grp takes slots grp, grp + NG, ...; lane l evaluates tap l,
      // and the tap is handed (shuffle) to the lane q = (e + t) mod G that always owns the
      // accumulator cells i = q (mod G): no two lanes ever update the same cell, no barrier.
      C* my = acc + grp * LEN;
      const int n = chi - clo;
      const int q = l;
#pragma unroll 2
      for (int base = 0; base < n; base += NG) {  // uniform trip count (shuffles below)
        const int sl = min(base + grp, n - 1);
        const bool valid = base + grp < n;
        const T zeta = sz[sl];
        const C v = sv[sl];
        const int e = se[sl];
        const T z2 = zeta * zeta;
        T ev = ce[DEG / 2];
#pragma unroll
        for (int z = DEG / 2 - 1; z >= 0; --z) ev = fma(ev, z2, ce[z]);
        T od = co[(DEG - 1) / 2];
#pragma unroll
        for (int z = (DEG - 1) / 2 - 1; z >= 0; --z) od = fma(od, z2, co[z]);
        const T w = fma(sgn * zeta, od, ev);
        const int t = (q - e) & (G - 1);
        const T wt = __shfl_sync(0xffffffffu, w, grp * G + t);
        if (valid && t < TAPS) {
          C a = my[e + t];
          a.x = fma(wt, v.x, a.x);
          a.y = fma(wt, v.y, a.y);
          my[e + t] = a;
        }
      }
      __syncwarp();
    }
    // cell y0 + y <-> accumulator index y + 2m - 1; sum the group copies, one coalesced store per cell
    C* dst = grid + (long long)b * g.grid_cells;
    for (int y = lane; y < nseg; y += 32) {
      C a = acc[y + TAPS - 1];
#pragma unroll
      for (int q = 1; q < NG; ++q) {
        const C c = acc[q * LEN + y + TAPS - 1];
        a.x += c.x;
        a.y += c.y;
      }
      int s = sy0 + y;
      if (s >= Nt) s -= Nt;
      dst[s] = a;
    }
    __syncwarp();
  }
  }  // segments
}

// ---------------------------------------------------------------- TENSOR precompute (D = 1)
// The paper's TENSOR strategy: the 2m window taps of every
// node are computed once by nfft_precompute and stored in cell order,
// wt[pos * 2m + t] = psi(frac_pos + m - 1 - t), so the
// per-call kernels read 8-byte taps instead of evaluating the polynomial.
constexpr int T1_THREADS = 256;

template <typename T, int M, int DEG>
__global__ void __launch_bounds__(T1_THREADS) taps1_kernel(Geom g, WinPoly<T> wp, const T* __restrict__ kc,
                                                           T* __restrict__ wt) {
  const int pc = blockIdx.x * T1_THREADS + threadIdx.x;
  if (pc >= g.M) return;
  double frac;
  node_cell((double)kc[pc], g.Ntd[0], g.Nt[0], frac);
  T w[2 * M];
  window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
#pragma unroll
  for (int t = 0; t < 2 * M; ++t) wt[(long long)pc * 2 * M + t] = w[t];
}

// spread1t: adjoint with TENSOR taps, one thread per grid cell y (owner-computes
// gather, every cell written exactly once, no shared memory): the nodes of
// cells x = y - m + i, i = 0..2m-1, are the cell-sorted ranges [cstart[x],
// cstart[x + 1]) and contribute f_j wt[pos][2m - 1 - i] (static tap index).
template <typename T, int M>
__global__ void __launch_bounds__(T1_THREADS) spread1t_kernel(Geom g, const typename cplx<T>::type* __restrict__ f,
                                                              const T* __restrict__ wt, const int* __restrict__ jc,
                                                              const int* __restrict__ cstart, int nb, int ne,
                                                              int sharded, typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  const int y = blockIdx.x * T1_THREADS + threadIdx.x;
  const int Nt = g.Nt[0];
  if (y >= Nt) return;
  int lo[TAPS], hi[TAPS];
#pragma unroll
  for (int i = 0; i < TAPS; ++i) {
    int x = y - M + i;  // binning cell of the i-th contributing cell
    if (x < 0) x += Nt;
    if (x >= Nt) x -= Nt;
    if ((unsigned)x >= (unsigned)Nt) x = pos_mod(x, Nt);
    lo[i] = __ldg(cstart + x);
    hi[i] = __ldg(cstart + x + 1);
    if (sharded) {  // shard = range [nb, ne) of the cell order
      lo[i] = max(lo[i], nb);
      hi[i] = min(hi[i], ne);
    }
  }
  int s = y - (Nt >> 1);  // storage of binning cell y
  if (s < 0) s += Nt;
  for (int b = 0; b < g.B; ++b) {
    const C* fb = f + (long long)b * g.M;
    C acc;
    acc.x = (T)0;
    acc.y = (T)0;
#pragma unroll
    for (int i = 0; i < TAPS; ++i) {
      for (int p = lo[i]; p < hi[i]; ++p) {
        const T w = __ldg(wt + (long long)p * TAPS + (TAPS - 1 - i));
        const C v = fb[__ldg(jc + p)];
        acc.x = fma(w, v.x, acc.x);
        acc.y = fma(w, v.y, acc.y);
      }
    }
    grid[(long long)b * g.grid_cells + s] = acc;
  }
}

}  // namespace nfftb
