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
// columns [c0 - m, c0 + SEG + m - 2], walked CELL BY CELL (per-cell ranges of
// the cell sort): the window column fixes, at compile time, which of the SEG
// cells a node reaches and with which last-dimension tap, so every multiply-add
// is a useful one. The fine decomposition keeps the dense centre of a radial
// trajectory spread over many CTAs (a coarse tile there holds ~5% of all
// nodes). Each warp accumulates its window rows into private registers (SEG
// cells x its lane's vector); the 8 warps' partial rows are summed in shared
// memory (dealing the window columns round-robin to the warps instead, for
// balance, measured slower: every warp then waits on every row's cstart loads). Node values travel transposed AND in cell order, f^T[pos][b] (one
// 256-byte row per position, C64; consecutive visits read consecutive rows),
// and the taps of every node are stored by nfft_precompute (taps_nd_kernel,
// the paper's TENSOR layout): a node is visited by ~11 row segments, so
// evaluating its taps once saves the per-visit polynomial work.
#pragma once

#include "common.cuh"

namespace nfftb {


constexpr int RB_LANES = 32;     // vectors per chunk
// consecutive grid rows per CTA (a window row's node visit then serves all of them). Measured on the
// radial configs (sigma 2 / 1.25): 1 row 423 / 496 us, 2 rows (2m + 1 warps) 476 / 535 us (110
// registers; the extra FMAs per visit do not pay for the lower occupancy)
constexpr int RB_ROWS = 1;
constexpr int RB_SEG = 16;       // cells per CTA (last dimension)
constexpr int RB_PITCH = 33;     // partial-row pitch in shared memory (vectors + 1)

// (B, M) -> (M, BP) and back; BP = batch padded to a multiple of 32 (pad rows unused)
// out[inv[j]][b] = in[b][j]: node values transposed into CELL order (inv = inverse of the
// cell-sort permutation jc), one 32-vector row per position
template <typename T>
__global__ void __launch_bounds__(256) transpose_bm_kernel(const typename cplx<T>::type* __restrict__ in, int B, int M,
                                                           int BP, const int* __restrict__ inv,
                                                           typename cplx<T>::type* __restrict__ out) {
  using C = typename cplx<T>::type;
  __shared__ C t[32][33];
  const int j0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  int dst[4];  // destination positions of this thread's output rows, loaded with the values
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + ty + 8 * k;
    dst[k] = j < M ? __ldg(inv + j) : 0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = ty + 8 * k;
    const int b = b0 + r, j = j0 + tx;
    if (b < B && j < M) t[r][tx] = in[(long long)b * M + j];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = ty + 8 * k;
    const int j = j0 + r, b = b0 + tx;
    if (j < M && b < B) out[(long long)dst[k] * BP + b] = t[tx][r];
  }
}

// inv[jc[pos]] = pos (precompute, batch adjoint)
static __global__ void __launch_bounds__(256) invert_perm_kernel(const int* __restrict__ jc, int M, int* __restrict__ inv) {
  const int pos = blockIdx.x * 256 + threadIdx.x;
  if (pos < M) inv[jc[pos]] = pos;
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

__host__ __device__ inline size_t rb_smem_bytes(int M, int rsize) {
  return (size_t)(2 * M + RB_ROWS - 1) * RB_SEG * RB_PITCH * 2 * rsize;  // per-warp partial rows
}

// Taps of every cell-sorted node, wt[pos][d][t] (the paper's TENSOR layout,
// PAPER.md:599-604), computed by nfft_precompute for the D >= 2 adjoints. A CTA
// of TN_NODES threads (one node each) builds its contiguous block of the table
// in shared memory (row stride D * 2m + 1: conflict-free) and writes it out
// coalesced (the per-thread 8-byte stores at a D * 2m stride were store-bound).
// cl (optional): the last-dimension binning cell of every position.
constexpr int TN_NODES = 64;
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(TN_NODES) taps_nd_kernel(Geom g, WinPolyN<T, D, M> wp, const T* __restrict__ kc,
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

// Visits of the nodes [lo, hi) of window column U (compile-time) of one window
// row: cell k of the segment gets tap k - U + 2m - 1 of the last dimension, so
// only the cells in the node's reach are accumulated (no zero products along
// the last dimension). The CTA owns RB_ROWS consecutive grid rows: output row
// j takes the node's dimension-0 tap lead + j (zero where lead + j is outside
// [0, 2m): the first and last window rows reach one output row only), so the
// node's value, taps and address arithmetic serve RB_ROWS rows.
template <typename T, int M, int U>
__device__ __forceinline__ void rb_visit(int lo, int hi, int lead, const typename cplx<T>::type* __restrict__ fTc,
                                         int BP, const T* __restrict__ wt,
                                         typename cplx<T>::type (&acc)[RB_ROWS][RB_SEG]) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  constexpr int KLO = U - TAPS + 1 > 0 ? U - TAPS + 1 : 0;
  constexpr int KHI = U < RB_SEG - 1 ? U : RB_SEG - 1;
  constexpr bool VEC = (TAPS * sizeof(T)) % 16 == 0;  // taps rows 16-byte aligned: vector loads
#pragma unroll 2
  for (int pos = lo; pos < hi; ++pos) {
    const C v = fTc[(long long)pos * BP];
    const T* wp = wt + (long long)pos * 2 * TAPS;
    T w0[RB_ROWS];
#pragma unroll
    for (int j = 0; j < RB_ROWS; ++j) w0[j] = (unsigned)(lead + j) < (unsigned)TAPS ? __ldg(wp + lead + j) : (T)0;
    T w1[TAPS];
    if constexpr (VEC && sizeof(T) == 4) {
#pragma unroll
      for (int t = 0; t < TAPS; t += 4) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(wp + TAPS + t));
        w1[t] = q.x; w1[t + 1] = q.y; w1[t + 2] = q.z; w1[t + 3] = q.w;
      }
    } else if constexpr (VEC) {
#pragma unroll
      for (int t = 0; t < TAPS; t += 2) {
        const double2 q = __ldg(reinterpret_cast<const double2*>(wp + TAPS + t));
        w1[t] = q.x; w1[t + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int t = 0; t < TAPS; ++t) w1[t] = __ldg(wp + TAPS + t);
    }
#pragma unroll
    for (int j = 0; j < RB_ROWS; ++j) {
      const T vx = w0[j] * v.x, vy = w0[j] * v.y;
#pragma unroll
      for (int k = KLO; k <= KHI; ++k) {
        const T w = w1[k - U + TAPS - 1];
        acc[j][k].x = fma(w, vx, acc[j][k].x);
        acc[j][k].y = fma(w, vy, acc[j][k].y);
      }
    }
  }
}

template <typename T, int M, int U = 0>
__device__ __forceinline__ void rb_row(int lo_l, int hi_l, int lead, const typename cplx<T>::type* fTc, int BP,
                                       const T* wt, typename cplx<T>::type (&acc)[RB_ROWS][RB_SEG]) {
  if constexpr (U < RB_SEG + 2 * M - 1) {
    const int lo = __shfl_sync(0xffffffffu, lo_l, U), hi = __shfl_sync(0xffffffffu, hi_l, U);
    if (lo < hi) rb_visit<T, M, U>(lo, hi, lead, fTc, BP, wt, acc);
    rb_row<T, M, U + 1>(lo_l, hi_l, lead, fTc, BP, wt, acc);
  }
}

// One CTA owns SEG cells of RB_ROWS consecutive grid rows for 32 vectors; warp w
// walks window rows w, w + 8, ... of the 2m + RB_ROWS - 1 in reach (lead tap
// 2m - 1 - r for the first output row), each window column's nodes in cell
// order (per-cell ranges from cstart, lane u holds column u's), then the warps'
// partial rows are summed in shared memory, one output row at a time, and
// stored coalesced.
// one warp per window row
__host__ __device__ constexpr int rb_threads(int M) { return 32 * (2 * M + RB_ROWS - 1); }

template <typename T, int M>
__global__ void __launch_bounds__(rb_threads(M)) spread_rowbatch_kernel(
    Geom g, const typename cplx<T>::type* __restrict__ fTc, int BP, const T* __restrict__ wt,
    const int* __restrict__ cstart, typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  constexpr int NW = rb_threads(M) / 32;
  constexpr int WR = TAPS + RB_ROWS - 1;  // window rows
  constexpr int WC = RB_SEG + TAPS - 1;   // window columns
  static_assert(WC <= 32, "window columns per lane");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b0 = blockIdx.y * RB_LANES;
  const int Nt0 = g.Nt[0], NtL = g.Nt[1];
  const int nseg = (NtL + RB_SEG - 1) / RB_SEG;
  const int rb = blockIdx.x / nseg;
  const int y0 = rb * RB_ROWS, c0 = (blockIdx.x - rb * nseg) * RB_SEG;  // first binning row, first column
  const int qs = min(RB_SEG, NtL - c0);
  C* part = reinterpret_cast<C*>(smem_raw);  // [NW][SEG][RB_PITCH]
  C acc[RB_ROWS][RB_SEG];
#pragma unroll
  for (int j = 0; j < RB_ROWS; ++j)
#pragma unroll
    for (int k = 0; k < RB_SEG; ++k) {
      acc[j][k].x = (T)0;
      acc[j][k].y = (T)0;
    }
  fTc += b0 + lane;
  for (int r = warp; r < WR; r += NW) {  // window row x0 = y0 - m + r
    int xr = y0 - M + r;  // in (-Nt0, 2 Nt0): one conditional wrap
    if (xr < 0) xr += Nt0;
    else if (xr >= Nt0) xr -= Nt0;
    const long long rowkey = (long long)xr * NtL;
    int lo_l = 0, hi_l = 0;
    if (lane < WC) {  // window column u = lane: binning column c0 - m + u
      int col = c0 - M + lane;
      if (col < 0) col += NtL;
      else if (col >= NtL) col -= NtL;
      lo_l = __ldg(cstart + rowkey + col);
      hi_l = __ldg(cstart + rowkey + col + 1);
    }
    if (r == warp) asm volatile("griddepcontrol.wait;" ::: "memory");  // f^T comes from transpose_bm
    rb_row<T, M>(lo_l, hi_l, TAPS - 1 - r, fTc, BP, wt, acc);
  }
  // sum the warps' partial rows (row pitch 33 vectors: conflict-free), one output row at a time,
  // coalesced stores (consecutive threads = consecutive cells of a vector)
  const int nbc = min(RB_LANES, g.B - b0);
  int cs0 = c0 - (NtL >> 1);
  if (cs0 < 0) cs0 += NtL;
#pragma unroll
  for (int j = 0; j < RB_ROWS; ++j) {
    if (j > 0) __syncthreads();  // the previous row's partials are consumed
#pragma unroll
    for (int k = 0; k < RB_SEG; ++k) part[((size_t)warp * RB_SEG + k) * RB_PITCH + lane] = acc[j][k];
    __syncthreads();
    int ys = y0 + j - (Nt0 >> 1);
    if (ys < 0) ys += Nt0;
    const long long rowoff = (long long)ys * NtL;
    for (int idx = tid; idx < nbc * RB_SEG; idx += NW * 32) {
      const int bb = idx / RB_SEG, k = idx - bb * RB_SEG;
      if (k >= qs) continue;
      C a;
      a.x = (T)0;
      a.y = (T)0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const C c = part[((size_t)w * RB_SEG + k) * RB_PITCH + bb];
        a.x += c.x;
        a.y += c.y;
      }
      int cs = cs0 + k;
      if (cs >= NtL) cs -= NtL;
      grid[(long long)(b0 + bb) * g.grid_cells + rowoff + cs] = a;
    }
  }
}

}  // namespace nfftb
