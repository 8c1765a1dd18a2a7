// resample1d.cuh — the D = 1 hot path (SURVEY §8(a) rows a1-a2 refinement,
// a6, a7; the BASELINE headline configuration) over CELL-SORTED nodes.
//
//   forward: f_j = sum_l ghat_l psi~(k_j - l/Nt)        (Alg. 3)
//   adjoint: ghat_l = sum_j f_j psi~(k_j - l/Nt)         (Alg. 4)
//
// The nodes are in stable CELL order (cellbin.cuh: kc = coordinates, jc = the
// caller's indices, cstart[c] = first cell-sorted position of cell c), computed
// once per node set and shared by every forward and adjoint.
// interp1s: one CTA per segment of 512 cells, the paper's block with its index
//   set cached in shared memory (Alg. 3).
// spread1a: OWNER-COMPUTES gather, one CTA per segment: the nodes that reach the
//   segment's cells are ONE contiguous cell-sorted range (the cells' own nodes
//   plus the halo NODES of the 2m - 1 neighbouring cells), staged once with
//   their taps; every thread sums its 4 cells over the nodes in reach and every
//   cell is written exactly once with a plain coalesced store: no atomics, no
//   zero pass, no halo merge (the paper's locked merge of PAPER.md:578-582
//   disappears because the halo NODES are read instead of halo CELLS being
//   reduced).
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
// spread1a: OWNER-COMPUTES gather, one CTA per segment of S1_SEG consecutive
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
//  4. writes each of its cells once.
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
// Launch width. Alone (nfft_adjoint): one CTA per segment; 7 CTAs per SM are resident, so the 1024
// segments of the headline configuration (1D 2^18, sigma = 2) run as one wave. Under nfft_execute,
// with the direct NFFT running concurrently: a grid-stride launch of S1_CTAS_OVERLAP CTAs per SM, so
// the forward FFT finds room (one CTA per segment there: step 50 us vs 42.6-43.3 us).
#ifndef NFFTB_S1_ALONE
#define NFFTB_S1_ALONE 0  // 0: one CTA per segment
#endif
#ifndef NFFTB_S1_OVERLAP
#define NFFTB_S1_OVERLAP 5
#endif
constexpr int S1_CTAS_ALONE = NFFTB_S1_ALONE;
constexpr int S1_CTAS_OVERLAP = NFFTB_S1_OVERLAP;

// tap row pitch: 2m taps, odd pitch (neighbouring rows in distinct banks)
__host__ __device__ constexpr int s1_pitch(int M) { return 2 * M + 1; }

// shared memory of one spread1a CTA (host and device agree)
__host__ __device__ inline size_t s1_smem_bytes(int M, size_t csize, size_t rsize) {
  size_t b = (size_t)S1_CAP * csize;                       // staged values
  b += (size_t)S1_CAP * s1_pitch(M) * rsize;               // staged tap rows
  b = (b + 15) & ~(size_t)15;
  b += (size_t)S1_CAP * 4;                                 // staged window cells
  return (b + 15) & ~(size_t)15;
}

// The load chain is staged through shared memory by cp.async instead of through registers. The
// round-2 kernel (attic/spread1s_register_staged.cuh.txt) kept a thread's three window nodes
// (coordinate, index, wrap, value) in registers across the two dependent load levels: 104 registers,
// 4 CTAs per SM, so the 1024 segments of 2^19 cells ran as two waves of ~6 us each
// (tools/micro/trace1d.cu). Here
//   level 1  cstart -> the window's node range and this thread's reach (registers, as before),
//   level 2  coordinates and indices: cp.async into the slots they will be overwritten in (the
//            coordinate into the node's tap row, the index into its window-cell slot),
//   level 3  values f[jc]: cp.async gather straight into the staged-value array, in flight while the
//            thread evaluates its nodes' taps one node at a time,
// so no node state lives in registers across a load level, the kernel fits S1A_MINB CTAs per SM and
// every segment of the headline configuration is resident at once (one wave). A thread waits only
// on its own copies before it reads them (cp.async.wait_group), the CTA barrier comes once, before
// the gather.
#ifndef NFFTB_S1A_MINB
#define NFFTB_S1A_MINB 7
#endif

template <int BYTES>
__device__ __forceinline__ void cp_async_n(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
  else if constexpr (BYTES == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}

template <typename T, int M, int DEG, bool TENSOR>
__global__ void __launch_bounds__(S1_THREADS, NFFTB_S1A_MINB) spread1a_kernel(Geom g, WinPolyN<T, 1, M> wp,
                                                              const typename cplx<T>::type* __restrict__ f,
                                                              const T* __restrict__ kc, const T* __restrict__ wt,
                                                              const int* __restrict__ jc,
                                                              const int* __restrict__ cstart, int nb, int ne,
                                                              typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M, TP = s1_pitch(M), REACH = S1_K + 2 * M - 1;
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
  for (int sgi = blockIdx.x; sgi < nsegs; sgi += gridDim.x) {
    // level 1: the window's node range (virtual positions) and this thread's reach
    const int y0 = sgi * S1_SEG, nseg = min(S1_SEG, Nt - y0);
    const int W = nseg + 2 * M - 1;  // window cell u <-> binning cell y0 - m + u
    auto vpos = [&](int u) {
      int c = y0 - M + u, wrap = 0;  // c in (-Nt, 2 Nt): 2m < Nt
      if (c < 0) {
        c += Nt;
        wrap = -1;
      } else if (c >= Nt) {
        c -= Nt;
        wrap = 1;
      }
      return __ldg(cstart + c) + wrap * Mn;
    };
    const int vbase = vpos(0);
    const int total = vpos(W) - vbase;
    const int r_lo = vpos(min(S1_K * t, W)) - vbase;
    const int r_hi = vpos(min(S1_K * t + REACH, W)) - vbase;
    C acc[S1_K];
#pragma unroll
    for (int k = 0; k < S1_K; ++k) {
      acc[k].x = (T)0;
      acc[k].y = (T)0;
    }
    for (int clo = 0; clo < total; clo += S1_CAP) {
      const int cnt = min(S1_CAP, total - clo);
      // level 2: coordinates -> first element of the node's tap row, indices -> its window-cell slot
      for (int q = t; q < cnt; q += S1_THREADS) {
        int p = vbase + clo + q;  // virtual position in (-M, 2M)
        if (p < 0) p += Mn;
        else if (p >= Mn) p -= Mn;
        cp_async_n<sizeof(T)>(stap + q * TP, kc + p);
        cp_async_n<4>(scel + q, jc + p);
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      // level 3: values -> staged values (node shard = range [nb, ne) of the cell order; others add 0)
      for (int q = t; q < cnt; q += S1_THREADS) {
        int p = vbase + clo + q;
        if (p < 0) p += Mn;
        else if (p >= Mn) p -= Mn;
        if (p >= nb && p < ne) {
          cp_async_n<sizeof(C)>(sval + q, fb + scel[q]);
        } else {
          C z;
          z.x = (T)0;
          z.y = (T)0;
          sval[q] = z;
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      NFFTB_TRACE(1);
      // taps (from the coordinates, or the TENSOR table) and window cells, one node at a time
#pragma unroll 1
      for (int q = t; q < cnt; q += S1_THREADS) {
        int p = vbase + clo + q, wv = 0;
        if (p < 0) {
          p += Mn;
          wv = -1;
        } else if (p >= Mn) {
          p -= Mn;
          wv = 1;
        }
        T* row = stap + q * TP;
        double frac;
        const int c = node_cell((double)row[0], g.Ntd[0], Nt, frac);
        scel[q] = c + wv * Nt - (y0 - M);  // window cell (virtual cell of the virtual position)
        T w[TAPS];
        if constexpr (TENSOR) {
#pragma unroll
          for (int l = 0; l < TAPS; ++l) w[l] = __ldg(wt + (long long)p * TAPS + l);
        } else {
          window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[0], w);
        }
#pragma unroll
        for (int l = 0; l < TAPS; ++l) row[l] = w[l];
      }
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      NFFTB_TRACE(2);
      __syncthreads();
      NFFTB_TRACE(3);
      // owner-computes gather: node in window cell K t + v adds to cell K t + k with tap
      // l = k - v + 2m - 1 when 0 <= l < 2m
      const int lo = max(r_lo - clo, 0), hi = min(r_hi - clo, cnt);
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
      __syncthreads();  // the gathers are done before the next chunk / segment is staged
    }
    NFFTB_TRACE(4);
    // one plain store per owned cell (binning cell y <-> storage (y - Nt/2) mod Nt)
    C* dst = grid + (long long)b * g.grid_cells;
    int s = y0 + S1_K * t - (Nt >> 1);
    if (s < 0) s += Nt;
#pragma unroll
    for (int k = 0; k < S1_K; ++k) {
      if (S1_K * t + k < nseg) {
        int sk = s + k;
        if (sk >= Nt) sk -= Nt;
        dst[sk] = acc[k];
      }
    }
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
