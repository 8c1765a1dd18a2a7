// resample_rowbatch.cuh — adjoint spreading for BATCHES of 2D transforms that
// share their nodes (BASELINE configs[4]: radial
// trajectory, B = 32, ComplexF32) over cell-sorted nodes (cellbin.cuh).
//
//   adjoint: ghat_l^b = sum_j f_j^b psi~(k_j - l/Nt)   (Alg. 4)
//
// LANES = BATCH VECTORS: the taps, footprints and indices are common to the B
// vectors, so a warp handles one node at a time for 32 vectors (warp-uniform
// control flow, taps evaluated once per node rather than once per node and
// vector). ROW SEGMENTS: one CTA owns SEG = 16 consecutive cells of ONE grid
// row and one 32-vector chunk (owner-computes: every cell written exactly once,
// no atomics, no zero pass; the paper's locked merge, becomes
// reading the halo NODES). Its nodes are those of the 2m window rows in reach,
// columns [c0 - m, c0 + SEG + m - 2] (contiguous cell-sorted ranges, two when a
// row wraps). The fine decomposition keeps the dense centre of a radial
// trajectory spread over many CTAs (a coarse tile there holds ~5% of all
// nodes). Each warp accumulates its nodes into private registers (SEG cells x
// its lane's vector) through zero-padded last-dimension taps (no per-cell
// predicate); the 8 warps' partial rows are summed in shared memory.
// Node values travel transposed, f^T[j][b] (one 256-byte row per node, C64),
// and the taps of every node are stored by nfft_precompute (taps_nd_kernel,
// the paper's TENSOR layout): a node is visited by ~11 row segments, so
// evaluating its taps once saves the per-visit polynomial work.
#pragma once

#include "common.cuh"

namespace nfftb {

constexpr int RB_THREADS = 256;  // 8 warps
constexpr int RB_LANES = 32;     // vectors per chunk
constexpr int RB_SEG = 16;       // cells per CTA (last dimension)
constexpr int RB_U = 2;          // nodes per warp step (loads in flight together)

// (B, M) -> (M, BP) and back; BP = batch padded to a multiple of 32 (pad rows unused)
template <typename T>
__global__ void __launch_bounds__(256) transpose_bm_kernel(const typename cplx<T>::type* __restrict__ in, int B, int M,
                                                           int BP, typename cplx<T>::type* __restrict__ out) {
  using C = typename cplx<T>::type;
  __shared__ C t[32][33];
  const int j0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, j = j0 + tx;
    if (b < B && j < M) t[r][tx] = in[(long long)b * M + j];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r, b = b0 + tx;
    if (j < M && b < B) out[(long long)j * BP + b] = t[tx][r];
  }
}

template <typename T>
__global__ void __launch_bounds__(256) transpose_mb_kernel(const typename cplx<T>::type* __restrict__ in, int B, int M,
                                                           int BP, typename cplx<T>::type* __restrict__ out) {
  using C = typename cplx<T>::type;
  __shared__ C t[32][33];
  const int j0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r, b = b0 + tx;
    if (j < M && b < B) t[r][tx] = in[(long long)j * BP + b];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, j = j0 + tx;
    if (b < B && j < M) out[(long long)b * M + j] = t[tx][r];
  }
}

__host__ __device__ inline int rb_tpad(int M) { return 2 * M + 2 * (RB_SEG - 1); }

__host__ __device__ inline size_t rb_smem_bytes(int M, int rsize) {
  const size_t csize = 2 * (size_t)rsize;
  size_t b = (size_t)(RB_THREADS / 32) * RB_U * rb_tpad(M) * rsize;  // per-warp zero-padded taps, RB_U nodes
  b = (b + 15) & ~(size_t)15;
  b += (size_t)(RB_THREADS / 32) * RB_SEG * RB_LANES * csize;  // per-warp partial rows
  b += (size_t)(2 * M * 4 + 4) * 4;                            // window rows: base, posA, lenA, posB
  return (b + 15) & ~(size_t)15;
}

// Taps of every cell-sorted node, wt[pos][d][t] (the paper's TENSOR layout,
// PAPER.md:599-604), computed by nfft_precompute for the D >= 2 adjoints. A CTA
// of TN_NODES threads (one node each) builds its contiguous block of the table
// in shared memory (row stride D * 2m + 1: conflict-free) and writes it out
// coalesced (the per-thread 8-byte stores at a D * 2m stride were store-bound).
// cl (optional): the last-dimension binning cell of every position.
constexpr int TN_NODES = 64;
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(TN_NODES) taps_nd_kernel(Geom g, WinPoly<T> wp, const T* __restrict__ kc,
                                                           T* __restrict__ wt, int* __restrict__ cl) {
  constexpr int ROW = D * 2 * M, RS = ROW + 1;
  __shared__ T s[TN_NODES * RS];
  const long long p0 = (long long)blockIdx.x * TN_NODES;
  const long long pc = p0 + threadIdx.x;
  if (pc < g.M) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double frac;
      const int c = node_cell((double)kc[(long long)d * g.M + pc], g.Ntd[d], g.Nt[d], frac);
      if (cl != nullptr && d == D - 1) cl[pc] = c;  // last-dimension cell (warp-block adjoint)
      T w[2 * M];
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w);
#pragma unroll
      for (int t = 0; t < 2 * M; ++t) s[threadIdx.x * RS + d * 2 * M + t] = w[t];
    }
  }
  __syncthreads();
  const int n = (int)(g.M - p0 < TN_NODES ? g.M - p0 : TN_NODES);
  T* out = wt + p0 * ROW;
  for (int i = threadIdx.x; i < n * ROW; i += TN_NODES) {
    const int node = i / ROW, k = i - node * ROW;
    out[i] = s[node * RS + k];
  }
}

template <typename T, int M>
__global__ void __launch_bounds__(RB_THREADS, sizeof(T) == 4 ? 3 : 2) spread_rowbatch_kernel(Geom g, const typename cplx<T>::type* __restrict__ fT,
                                                                     int BP, const T* __restrict__ kc,
                                                                     const T* __restrict__ wt,
                                                                     const int* __restrict__ jc,
                                                                     const int* __restrict__ cstart,
                                                                     typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  constexpr int TPAD = 2 * M + 2 * (RB_SEG - 1);
  constexpr int NW = RB_THREADS / 32;
  constexpr int WROWS = 2 * M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b0 = blockIdx.y * RB_LANES;
  const int Nt0 = g.Nt[0], NtL = g.Nt[1];
  const int nseg = (NtL + RB_SEG - 1) / RB_SEG;
  const int y0 = blockIdx.x / nseg, c0 = (blockIdx.x - y0 * nseg) * RB_SEG;  // binning row, first column
  const int qs = min(RB_SEG, NtL - c0);
  T* ptap = reinterpret_cast<T*>(smem_raw) + warp * RB_U * TPAD;  // this warp's padded taps [RB_U][TPAD]
  C* part = reinterpret_cast<C*>(smem_raw + ((NW * RB_U * TPAD * sizeof(T) + 15) & ~(size_t)15));  // [NW][SEG][32]
  int* rbase = reinterpret_cast<int*>(part + (size_t)NW * RB_SEG * RB_LANES);             // [WROWS + 1]
  int* rposA = rbase + WROWS + 1;
  int* rlenA = rposA + WROWS;
  int* rposB = rlenA + WROWS;
  // window rows x0 = y0 - m + r, r = 0..2m-1 (lead tap 2m - 1 - r); columns [c0 - m, c0 + qs + m - 2]
  const int a_last = c0 - M, b_last = c0 + qs + M - 2;
  if (tid < WROWS) {
    const int r = tid;
    const long long rowkey = (long long)pos_mod(y0 - M + r, Nt0) * NtL;
    int pA, lA, pB = 0, lB = 0;
    if (a_last < 0) {
      pA = cstart[rowkey + NtL + a_last];
      lA = cstart[rowkey + NtL] - pA;
      pB = cstart[rowkey];
      lB = cstart[rowkey + b_last + 1] - pB;
    } else if (b_last >= NtL) {
      pA = cstart[rowkey + a_last];
      lA = cstart[rowkey + NtL] - pA;
      pB = cstart[rowkey];
      lB = cstart[rowkey + b_last - NtL + 1] - pB;
    } else {
      pA = cstart[rowkey + a_last];
      lA = cstart[rowkey + b_last + 1] - pA;
    }
    rposA[r] = pA;
    rlenA[r] = lA;
    rposB[r] = pB;
    rbase[r] = lA + lB;
  }
  for (int i = lane; i < RB_U * TPAD; i += 32) ptap[i] = (T)0;  // padding stays zero; taps at SEG - 1 ..
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int r = 0; r < WROWS; ++r) {
      const int c = rbase[r];
      rbase[r] = run;
      run += c;
    }
    rbase[WROWS] = run;
  }
  __syncthreads();
  const int total = rbase[WROWS];
  C acc[RB_SEG];
#pragma unroll
  for (int k = 0; k < RB_SEG; ++k) {
    acc[k].x = (T)0;
    acc[k].y = (T)0;
  }
  // warp w takes the window's nodes w, w + NW, ... (warp-uniform: lanes = batch vectors), RB_U at a
  // time: every load of the RB_U nodes is in flight before the multiply-adds
  for (int s0 = warp; s0 < total; s0 += NW * RB_U) {
    C v[RB_U];
    T vr[RB_U], vi[RB_U];
    int o[RB_U];
#pragma unroll
    for (int u = 0; u < RB_U; ++u) {
      const int s = s0 + u * NW;
      v[u].x = (T)0;
      v[u].y = (T)0;
      vr[u] = (T)0;
      o[u] = 0;
      if (s < total) {
        int r = 0;
#pragma unroll
        for (int q = 1; q < WROWS; ++q) r += rbase[q] <= s;
        const int within = s - rbase[r];
        const int pos = within < rlenA[r] ? rposA[r] + within : rposB[r] + (within - rlenA[r]);
        v[u] = fT[(long long)__ldg(jc + pos) * BP + b0 + lane];
        const T* wp_ = wt + (long long)pos * 2 * TAPS;
        vr[u] = __ldg(wp_ + (TAPS - 1 - r));  // lead tap for row y0 (scaled below)
        if (lane < TAPS) ptap[u * TPAD + RB_SEG - 1 + lane] = __ldg(wp_ + TAPS + lane);
        double frac;
        int oo = node_cell((double)__ldg(kc + g.M + pos), g.Ntd[1], NtL, frac) - a_last;  // window column
        if (oo < 0) oo += NtL;
        else if (oo >= NtL) oo -= NtL;
        o[u] = oo;
      } else if (lane < TAPS) {
        ptap[u * TPAD + RB_SEG - 1 + lane] = (T)0;
      }
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < RB_U; ++u) {
      vi[u] = vr[u] * v[u].y;
      vr[u] = vr[u] * v[u].x;
      // cell k (window column k + m) gets tap k - o + 2m - 1, padded index + SEG - 1
      const T* tp = ptap + u * TPAD + (TAPS - 1 + RB_SEG - 1 - o[u]);
#pragma unroll
      for (int k = 0; k < RB_SEG; ++k) {
        const T w = tp[k];
        acc[k].x = fma(w, vr[u], acc[k].x);
        acc[k].y = fma(w, vi[u], acc[k].y);
      }
    }
    __syncwarp();
  }
  // sum the warps' partial rows, coalesced stores (consecutive threads = consecutive cells of a vector)
#pragma unroll
  for (int k = 0; k < RB_SEG; ++k) part[((size_t)warp * RB_SEG + k) * RB_LANES + lane] = acc[k];
  __syncthreads();
  const int nbc = min(RB_LANES, g.B - b0);
  const long long rowoff = (long long)pos_mod(y0 - (Nt0 >> 1), Nt0) * NtL;
  for (int idx = tid; idx < nbc * RB_SEG; idx += RB_THREADS) {
    const int bb = idx / RB_SEG, k = idx - bb * RB_SEG;
    if (k >= qs) continue;
    C a;
    a.x = (T)0;
    a.y = (T)0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const C c = part[((size_t)w * RB_SEG + k) * RB_LANES + bb];
      a.x += c.x;
      a.y += c.y;
    }
    grid[(long long)(b0 + bb) * g.grid_cells + rowoff + pos_mod(c0 + k - (NtL >> 1), NtL)] = a;
  }
}

}  // namespace nfftb
