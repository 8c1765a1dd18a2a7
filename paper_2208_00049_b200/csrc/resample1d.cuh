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


// ---------------------------------------------------------------- forward
// interp1s: one CTA per segment of S1_SEG consecutive cells (b = blockIdx.y),
// the paper's block with its index set cached (Alg. 3): the
// CTA's nodes are those of its cells, the cell-sorted range [cstart[y0],
// cstart[y0 + SEG]); the grid cells they read are the block index set
// [y0 - m + 1, y0 + SEG + m - 1]. The index set streams into shared memory
// with cp.async (it depends only on y0) while the threads load their nodes'
// coordinates and indices, so the two global-memory latencies overlap; then
// every node evaluates its 2m taps (even/odd Horner) and sums the 2m cells
// from shared memory, and its value is written to f[j] (caller's order).
constexpr int I1_THREADS = 128;
constexpr int I1_SEG = 512;               // cells per CTA
constexpr int I1_U = 3;                   // nodes per thread loaded before the barrier

__host__ __device__ inline size_t i1_smem_bytes(int M, size_t csize) {
  return (((size_t)I1_SEG + 2 * M) * csize + 15) & ~(size_t)15;
}

template <typename T, int M, int DEG, bool TENSOR>
__global__ void __launch_bounds__(I1_THREADS) interp1s_kernel(Geom g, WinPolyN<T, 1, M> wp,
                                                              const typename cplx<T>::type* __restrict__ grid,
                                                              const T* __restrict__ kc, const T* __restrict__ wt,
                                                              const int* __restrict__ jc,
                                                              const int* __restrict__ cstart, int nb, int ne,
                                                              typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sg = reinterpret_cast<C*>(smem_raw);  // window cell e <-> binning cell y0 - m + 1 + e
  NFFTB_TRACE(0);
  const int Nt = g.Nt[0];
  const int b = blockIdx.y;
  const int nsegs = (Nt + I1_SEG - 1) / I1_SEG;
  // grid-stride over the segments (the launch may use fewer CTAs than segments)
  for (int sgi = blockIdx.x; sgi < nsegs; sgi += gridDim.x) {
  const int y0 = sgi * I1_SEG;
  const int nseg = min(I1_SEG, Nt - y0);
  const int W = nseg + TAPS - 1;
  // 1. this CTA's nodes (cell-sorted range of its cells), clipped to the shard [nb, ne): they do not
  //    depend on the grid, so with programmatic dependent launch they load while the FFT finishes
  const int p0 = max(__ldg(cstart + y0), nb), p1 = min(__ldg(cstart + y0 + nseg), ne);
  double kk[I1_U];
  int jj[I1_U];
#pragma unroll
  for (int i = 0; i < I1_U; ++i) {
    const int p = p0 + threadIdx.x + i * I1_THREADS;
    jj[i] = -1;
    kk[i] = 0.0;
    if (p < p1) {
      kk[i] = (double)kc[p];
      jj[i] = jc[p];
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the grid (previous kernel's output) is complete
  // 2. the block index set -> shared memory (asynchronous; storage (cell - Nt/2) mod Nt)
  {
    const C* gb = grid + (long long)b * g.grid_cells;
    int s0 = y0 - M + 1 - (Nt >> 1);
    if (s0 < 0) s0 += Nt;
    if (s0 < 0) s0 = pos_mod(s0, Nt);
    for (int e = threadIdx.x; e < W; e += I1_THREADS) {
      int s = s0 + e;
      while (s >= Nt) s -= Nt;
      cp_async_cell<T>(sg + e, gb + s);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  NFFTB_TRACE(1);
  C* fb = f + (long long)b * g.M;
  auto one = [&](double k, int j, int p) {
    double frac;
    const int c = node_cell(k, g.Ntd[0], Nt, frac);  // c in [y0, y0 + nseg): footprint starts at window cell c - y0
    T w[TAPS];
    if constexpr (TENSOR) {  // the stored taps of position p
#pragma unroll
      for (int l = 0; l < TAPS; ++l) w[l] = __ldg(wt + (long long)p * TAPS + l);
    } else {
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
    }
    const C* row = sg + (c - y0);
    C acc;
    acc.x = (T)0;
    acc.y = (T)0;
#pragma unroll
    for (int l = 0; l < TAPS; ++l) {
      const C v = row[l];
      acc.x = fma(w[l], v.x, acc.x);
      acc.y = fma(w[l], v.y, acc.y);
    }
    fb[j] = acc;
  };
#pragma unroll
  for (int i = 0; i < I1_U; ++i)
    if (jj[i] >= 0) one(kk[i], jj[i], p0 + threadIdx.x + i * I1_THREADS);
  // dense segments: the remaining nodes
  for (int p = p0 + threadIdx.x + I1_U * I1_THREADS; p < p1; p += I1_THREADS) one((double)kc[p], jc[p], p);
  __syncthreads();  // the next segment overwrites the staged index set
  }  // segments
  NFFTB_TRACE(2);
}

// ---------------------------------------------------------------- adjoint
// spread1s: OWNER-COMPUTES gather, one CTA per segment of S1_SEG consecutive
// cells (b = blockIdx.y). The nodes that reach the segment are those of the
// window cells [y0 - m, y0 + SEG + m - 2]: ONE contiguous range of the
// cell-sorted order (cstart; a wrapped window is a wrapped range, handled with
// virtual positions V = cstart[c mod Nt] + M * floor(c / Nt)). The CTA
//  1. reads the window's node range and each thread's reach from cstart
//     (no shared table, no barrier),
//  2. stages every window node once: its value f_j, its window cell and its
//     2m taps (POLYNOMIAL: even/odd Horner of the window table,
//     PAPER.md:628-642; TENSOR: the stored taps) in shared
//     memory,
//  3. every thread owns S1_K consecutive cells y and walks the nodes in reach
//     (window cells [y - m, y + K + m - 2]: one contiguous slot range, so the
//     walk is one loop without per-cell divergence); a node in window cell x
//     adds f_j w_j[y - x + m - 1] to every owned cell y in its reach
//     (predicated loads and FMAs, no branches),
//  4. writes each of its cells once (plain stores: no atomics, no zero pass,
//     no halo merge — the paper's locked merge of PAPER.md:578-582 becomes
//     reading the halo NODES).
// A window with more than S1_CAP nodes is processed in chunks (the
// accumulators stay in registers).
#ifndef NFFTB_S1_THREADS
#define NFFTB_S1_THREADS 128
#endif
constexpr int S1_THREADS = NFFTB_S1_THREADS;
#ifndef NFFTB_S1_K
#define NFFTB_S1_K 4
#endif
#ifndef NFFTB_S1_CAP
#define NFFTB_S1_CAP 320
#endif
constexpr int S1_K = NFFTB_S1_K;          // consecutive cells per thread
constexpr int S1_SEG = S1_THREADS * S1_K; // 512 cells per CTA
constexpr int S1_CAP = NFFTB_S1_CAP;      // staged nodes per chunk (mean ~0.5 (SEG + 2m) at M = N = Nt/2)
// Launch width. Alone (nfft_adjoint): one CTA per segment, 4 resident per SM (104 registers) and the
// hardware refills the SMs as CTAs retire: 1D 2^18, m = 4 11.5-12 us where the round-2 software
// pipeline (138 registers, 3 CTAs/SM) took 14.3 us on the same box. Under nfft_execute, with the
// direct NFFT running concurrently: a grid-stride launch of 4 CTAs per SM, so the pending CTAs of a
// full-width launch do not take every freed slot ahead of the forward FFT (one CTA per segment there:
// step 47-48 us vs 43.1 us).
#ifndef NFFTB_S1_ALONE
#define NFFTB_S1_ALONE 0  // 0: one CTA per segment
#endif
#ifndef NFFTB_S1_OVERLAP
#define NFFTB_S1_OVERLAP 4
#endif
#ifndef NFFTB_S1_MINB
#define NFFTB_S1_MINB 1
#endif
constexpr int S1_CTAS_ALONE = NFFTB_S1_ALONE;
constexpr int S1_CTAS_OVERLAP = NFFTB_S1_OVERLAP;

// tap row pitch: 2m taps, odd pitch (neighbouring rows in distinct banks)
__host__ __device__ constexpr int s1_pitch(int M) { return 2 * M + 1; }

// shared memory of one spread1s CTA (host and device agree)
__host__ __device__ inline size_t s1_smem_bytes(int M, size_t csize, size_t rsize) {
  size_t b = (size_t)S1_CAP * csize;                       // staged values
  b += (size_t)S1_CAP * s1_pitch(M) * rsize;               // staged tap rows
  b = (b + 15) & ~(size_t)15;
  b += (size_t)S1_CAP * 4;                                 // staged window cells
  return (b + 15) & ~(size_t)15;
}

template <typename T, int M, int DEG, bool TENSOR>
__global__ void __launch_bounds__(S1_THREADS, NFFTB_S1_MINB) spread1s_kernel(Geom g, WinPolyN<T, 1, M> wp,
                                                              const typename cplx<T>::type* __restrict__ f,
                                                              const T* __restrict__ kc, const T* __restrict__ wt,
                                                              const int* __restrict__ jc,
                                                              const int* __restrict__ cstart, int nb, int ne,
                                                              typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M, TP = s1_pitch(M), REACH = S1_K + 2 * M - 1;
  constexpr int U = (S1_CAP + S1_THREADS - 1) / S1_THREADS;  // staged nodes per thread and chunk
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* sval = reinterpret_cast<C*>(smem_raw);
  T* stap = reinterpret_cast<T*>(sval + S1_CAP);
  int* scel = reinterpret_cast<int*>(smem_raw + ((S1_CAP * sizeof(C) + (size_t)S1_CAP * TP * sizeof(T) + 15) & ~(size_t)15));
  NFFTB_TRACE(0);
  const int Nt = g.Nt[0], Mn = g.M;
  const int b = blockIdx.y;
  const int nsegs = (Nt + S1_SEG - 1) / S1_SEG;
  const int t = threadIdx.x;
  const C* fb = f + (long long)b * Mn;
  // 1. a segment's window: node range (virtual positions, uniform) and this thread's reach, window
  //    cells [K t, K t + REACH); virtual position of window cell u: cstart[c mod Nt] + M floor(c / Nt)
  struct Meta {
    int y0, nseg, vbase, total, r_lo, r_hi;
  };
  auto load_meta = [&](int sgi) {
    Meta mt;
    mt.y0 = sgi * S1_SEG;
    mt.nseg = min(S1_SEG, Nt - mt.y0);
    const int W = mt.nseg + 2 * M - 1;  // window cell u <-> binning cell y0 - m + u
    auto vpos = [&](int u) {
      int c = mt.y0 - M + u, wrap = 0;  // c in (-Nt, 2 Nt): 2m < Nt
      if (c < 0) {
        c += Nt;
        wrap = -1;
      } else if (c >= Nt) {
        c -= Nt;
        wrap = 1;
      }
      return __ldg(cstart + c) + wrap * Mn;
    };
    mt.vbase = vpos(0);
    mt.total = vpos(W) - mt.vbase;
    mt.r_lo = vpos(min(S1_K * t, W)) - mt.vbase;
    mt.r_hi = vpos(min(S1_K * t + REACH, W)) - mt.vbase;
    return mt;
  };
  // 2. a chunk's nodes: coordinates and indices (first load level), then the values (second level)
  struct Batch {
    int pp[U], jj[U], wv[U];
    double kk[U];
    C v[U];
  };
  auto load_nodes = [&](const Meta& mt, int clo, Batch& bt) {
    const int cnt = min(S1_CAP, mt.total - clo);
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int q = t + i * S1_THREADS;
      bt.pp[i] = -1;
      bt.jj[i] = -1;
      bt.wv[i] = 0;
      bt.kk[i] = 0.0;
      if (q < cnt) {
        int p = mt.vbase + clo + q;  // virtual position in (-M, 2M)
        if (p < 0) {
          p += Mn;
          bt.wv[i] = -1;
        } else if (p >= Mn) {
          p -= Mn;
          bt.wv[i] = 1;
        }
        bt.pp[i] = p;
        bt.kk[i] = (double)kc[p];
        bt.jj[i] = (p >= nb && p < ne) ? __ldg(jc + p) : -1;  // node shard = range [nb, ne) of the cell order
      }
    }
  };
  auto load_vals = [&](Batch& bt) {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      bt.v[i].x = (T)0;
      bt.v[i].y = (T)0;
      if (bt.jj[i] >= 0) bt.v[i] = fb[bt.jj[i]];
    }
  };
  // stage: taps (from the coordinates, or the TENSOR table), window cell and value of every node
  auto stage = [&](const Meta& mt, const Batch& bt) {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int q = t + i * S1_THREADS;
      if (bt.pp[i] < 0) continue;
      double frac;
      const int c = node_cell(bt.kk[i], g.Ntd[0], Nt, frac);
      scel[q] = c + bt.wv[i] * Nt - (mt.y0 - M);  // window cell (virtual cell of the virtual position)
      T w[TAPS];
      if constexpr (TENSOR) {
#pragma unroll
        for (int l = 0; l < TAPS; ++l) w[l] = __ldg(wt + (long long)bt.pp[i] * TAPS + l);
      } else {
        window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
      }
      T* row = stap + q * TP;
#pragma unroll
      for (int l = 0; l < TAPS; ++l) row[l] = w[l];
    }
#pragma unroll
    for (int i = 0; i < U; ++i)
      if (bt.pp[i] >= 0) sval[t + i * S1_THREADS] = bt.v[i];
  };
  int sgi = blockIdx.x;
  if (sgi >= nsegs) return;
  // One segment after another (a launch alone has one CTA per segment and the hardware refills the
  // SMs; under nfft_execute the launch is narrower and the CTAs grid-stride). A software pipeline over
  // the CTA's segments (next segment's loads during the gather: 138 registers, 3 CTAs/SM) and an L2
  // prefetch of the successor segment's load chain were measured slower / neutral
  // (attic/spread1s_pipeline_and_l2_prefetch.diff.txt).
  while (true) {
    const Meta mc = load_meta(sgi);
    Batch bc;
    load_nodes(mc, 0, bc);
    load_vals(bc);
    NFFTB_TRACE(1);
    C acc[S1_K];
#pragma unroll
    for (int k = 0; k < S1_K; ++k) {
      acc[k].x = (T)0;
      acc[k].y = (T)0;
    }
    for (int clo = 0; clo < mc.total; clo += S1_CAP) {
      const int cnt = min(S1_CAP, mc.total - clo);
      if (clo > 0) {  // a dense window: further chunks are loaded in place
        __syncthreads();
        load_nodes(mc, clo, bc);
        load_vals(bc);
      }
      stage(mc, bc);
      NFFTB_TRACE(2);
      __syncthreads();
      NFFTB_TRACE(3);
      const int lo = max(mc.r_lo - clo, 0), hi = min(mc.r_hi - clo, cnt);
      for (int q = lo; q < hi; ++q) {
        const C val = sval[q];
        const int l0 = TAPS - 1 - (scel[q] - S1_K * t);
        const T* wr = stap + q * TP;
#pragma unroll
        for (int k = 0; k < S1_K; ++k) {
          const int l = l0 + k;
          if ((unsigned)l < (unsigned)TAPS) {
            const T wk = wr[l];
            acc[k].x = fma(wk, val.x, acc[k].x);
            acc[k].y = fma(wk, val.y, acc[k].y);
          }
        }
      }
    }
    NFFTB_TRACE(4);
    C* dst = grid + (long long)b * g.grid_cells;
    int s = mc.y0 + S1_K * t - (Nt >> 1);
    if (s < 0) s += Nt;
#pragma unroll
    for (int k = 0; k < S1_K; ++k) {
      if (S1_K * t + k < mc.nseg) {
        int sk = s + k;
        if (sk >= Nt) sk -= Nt;
        dst[sk] = acc[k];
      }
    }
    sgi += gridDim.x;
    if (sgi >= nsegs) break;
    __syncthreads();  // the gathers of this segment are done before the next one is staged
  }
}

// ---------------------------------------------------------------- TENSOR precompute (D = 1)
// The paper's TENSOR strategy: the 2m window taps of every
// node are computed once by nfft_precompute and stored in cell order,
// wt[pos * 2m + t] = psi(frac_pos + m - 1 - t), so the
// per-call kernels read 8-byte taps instead of evaluating the polynomial.
constexpr int T1_THREADS = 256;

template <typename T, int M, int DEG>
__global__ void __launch_bounds__(T1_THREADS) taps1_kernel(Geom g, WinPolyN<T, 1, M> wp, const T* __restrict__ kc,
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

}  // namespace nfftb
