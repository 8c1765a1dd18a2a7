// resample_full.cuh — the FULL precomputation strategy (PAPER.md:596-599,
// §3.7, "FULL": the sparse matrix B itself is stored; CuNFFT's GPU prototype,
// PAPER.md:800) and the resampling over it.
//
//   B_{j,l} = psi~(k_j - l/Nt) = prod_d psi_hat_Base((Nt_d k_jd - l_d)/m),
//   l in the footprint I_{Nt,m}(k_j)
//   forward:  f = B ghat                            (Alg. 1 l.7-9 as a sparse matrix-vector product)
//   adjoint:  ghat = B^H f                          (Alg. 2 l.1-3)
//
// Storage: for every CELL-SORTED position pos (the precompute's order) the
// E = (2m)^D entries of the node's row of B, e = (l_0, ..., l_{D-1}) row-major
// (last dimension fastest): weight bw[pos * E + e] (plan precision) and grid
// index bi[pos * E + e] (int32, row-major storage index of the oversampled
// cell (a_d - m + 1 + l_d) mod Nt_d). E (2m)^D (rsize + 4) bytes per node:
// 96 B in 1D, 768 B in 2D, 6 KB in 3D at m = 4, C128.
//
// full_build (precompute): a CTA stages the per-dimension taps of 64 nodes
//   in shared memory, then writes their E-entry rows coalesced (and, for
//   D >= 2, the last-dimension cell of every position for full_spread).
// full_interp (forward): LPN lanes per node (8 for E <= 16, else 32) stride
//   over the node's row (coalesced weight / index reads), reduce with
//   shuffles, one store f[j].
// full_spread (adjoint, D >= 2; D = 1 uses spread1a over the weights, which
//   are then the taps): OWNER-COMPUTES, one thread per oversampled cell y: the
//   nodes that reach y lie in the (2m)^(D-1) rows of the footprint box, each a
//   contiguous cell-sorted range along the last dimension (two where it
//   wraps); a node in cell x contributes bw[pos][e(y - x + m - 1)] fc[pos] (fc
//   = f in cell order). Every cell is written exactly once, no atomics.
#pragma once

#include "common.cuh"

namespace nfftb {

constexpr int FB_NODES = 64;     // full_build: nodes per CTA
constexpr int FB_THREADS = 256;
constexpr int FI_THREADS = 256;  // full_interp
constexpr int FS_THREADS = 256;  // full_spread

__host__ __device__ constexpr int ipow_full(int b, int e) { return e == 0 ? 1 : b * ipow_full(b, e - 1); }

template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(FB_THREADS) full_build_kernel(Geom g, WinPolyN<T, D, M> wp, const T* __restrict__ kc,
                                                                T* __restrict__ bw, int* __restrict__ bi,
                                                                int* __restrict__ cl) {
  constexpr int TAPS = 2 * M, E = ipow_full(2 * M, D);
  __shared__ T sw[FB_NODES][D][TAPS];
  __shared__ int sc[FB_NODES][D];  // storage index of the footprint's first cell per dimension
  const long long p0 = (long long)blockIdx.x * FB_NODES;
  const int n = (int)min((long long)FB_NODES, (long long)g.M - p0);
  for (int i = threadIdx.x; i < n * D; i += FB_THREADS) {
    const int node = i / D, d = i - node * D;
    double frac;
    const int c = node_cell((double)kc[(long long)d * g.M + p0 + node], g.Ntd[d], g.Nt[d], frac);
    T w[TAPS];
    window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w);
#pragma unroll
    for (int t = 0; t < TAPS; ++t) sw[node][d][t] = w[t];
    // binning cell c = (a + Nt/2) mod Nt; first footprint cell a - m + 1 at storage (a - m + 1) mod Nt
    sc[node][d] = pos_mod(c - M + 1 - (g.Nt[d] >> 1), g.Nt[d]);
    if (cl != nullptr && d == D - 1) cl[p0 + node] = c;  // last-dimension cell (full_spread)
  }
  __syncthreads();
  for (long long i = threadIdx.x; i < (long long)n * E; i += FB_THREADS) {
    const int node = (int)(i / E), e = (int)(i - (long long)node * E);
    T w = (T)1;
    long long lin = 0;
    int rem = e;
    int l[D];
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      l[d] = rem % TAPS;
      rem /= TAPS;
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      w *= sw[node][d][l[d]];
      int s = sc[node][d] + l[d];
      if (s >= g.Nt[d]) s -= g.Nt[d];
      lin = lin * g.Nt[d] + s;
    }
    bw[p0 * E + i] = w;
    bi[p0 * E + i] = (int)lin;
  }
}

template <typename T, int D, int M>
__global__ void __launch_bounds__(FI_THREADS) full_interp_kernel(Geom g, const typename cplx<T>::type* __restrict__ grid,
                                                                 const T* __restrict__ bw, const int* __restrict__ bi,
                                                                 const int* __restrict__ jc, int nb, int ne,
                                                                 typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  constexpr int E = ipow_full(2 * M, D);
  constexpr int LPN = E <= 16 ? 8 : 32;  // lanes per node
  constexpr int NPB = FI_THREADS / LPN;  // nodes per CTA pass
  const int lane = threadIdx.x % LPN;
  const C* gb = grid + (long long)blockIdx.y * g.grid_cells;
  C* fb = f + (long long)blockIdx.y * g.M;
  const int span = ne - nb;
  for (int q = blockIdx.x * NPB + threadIdx.x / LPN; q - (int)(threadIdx.x / LPN) < span; q += gridDim.x * NPB) {
    const bool on = q < span;
    const long long pos = nb + (on ? q : 0);
    C acc;
    acc.x = (T)0;
    acc.y = (T)0;
    if (on) {
      const T* w = bw + pos * E;
      const int* ix = bi + pos * E;
#pragma unroll 4
      for (int e = lane; e < E; e += LPN) {
        const T we = __ldg(w + e);
        const C v = __ldg(gb + __ldg(ix + e));
        acc.x = fma(we, v.x, acc.x);
        acc.y = fma(we, v.y, acc.y);
      }
    }
#pragma unroll
    for (int o = LPN / 2; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o, LPN);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o, LPN);
    }
    if (on && lane == 0) fb[jc[pos]] = acc;
  }
}

// fc: node values in cell order (zero outside the node shard), cl: last-dimension binning cell of every
// position; one thread per oversampled cell (storage order), grid-stride; b = blockIdx.y
template <typename T, int D, int M>
__global__ void __launch_bounds__(FS_THREADS) full_spread_kernel(Geom g, const typename cplx<T>::type* __restrict__ fc,
                                                                 const int* __restrict__ cl, const T* __restrict__ bw,
                                                                 const int* __restrict__ cstart,
                                                                 typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M, E = ipow_full(2 * M, D), ROWS = ipow_full(2 * M, D - 1);
  const int NtL = g.Nt[D - 1];
  const long long b = blockIdx.y;
  const C* fb = fc + b * g.M;
  C* gout = grid + b * g.grid_cells;
  for (long long s = (long long)blockIdx.x * FS_THREADS + threadIdx.x; s < g.grid_cells;
       s += (long long)gridDim.x * FS_THREADS) {
    // storage cell s -> binning cell y_d = (s_d + Nt_d/2) mod Nt_d
    int y[D];
    long long rem = s;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      const int sd = (int)(rem % g.Nt[d]);
      rem /= g.Nt[d];
      y[d] = sd + (g.Nt[d] >> 1);
      if (y[d] >= g.Nt[d]) y[d] -= g.Nt[d];
    }
    C acc;
    acc.x = (T)0;
    acc.y = (T)0;
    for (int r = 0; r < ROWS; ++r) {
      // lead taps l_d (d < D-1): node cell x_d = y_d + m - 1 - l_d (mod Nt_d)
      int rr = r, eoff = 0;
      long long key = 0;
      int lt[D > 1 ? D - 1 : 1];
#pragma unroll
      for (int d = D - 2; d >= 0; --d) {
        lt[d] = rr % TAPS;
        rr /= TAPS;
      }
#pragma unroll
      for (int d = 0; d < D - 1; ++d) {
        int x = y[d] + M - 1 - lt[d];
        if (x >= g.Nt[d]) x -= g.Nt[d];
        if (x < 0) x += g.Nt[d];
        key = key * g.Nt[d] + x;
        eoff = eoff * TAPS + lt[d];
      }
      key *= NtL;
      // last dimension: x_last in [y - m, y + m - 1] (tap l = y + m - 1 - x), as one or two ranges
      int lo = y[D - 1] - M, hi = y[D - 1] + M - 1;  // inclusive, unwrapped
      for (int part = 0; part < 2; ++part) {
        int a = lo, z = hi, shift = 0;
        if (part == 0) {
          if (lo < 0) a = 0;
          if (hi >= NtL) z = NtL - 1;
        } else {
          if (lo < 0) {
            a = lo + NtL;
            z = NtL - 1;
            shift = NtL;  // x = xs - NtL in unwrapped coordinates
          } else if (hi >= NtL) {
            a = 0;
            z = hi - NtL;
            shift = -NtL;
          } else {
            break;
          }
        }
        const int p_lo = __ldg(cstart + key + a), p_hi = __ldg(cstart + key + z + 1);
        for (int p = p_lo; p < p_hi; ++p) {
          const int x = __ldg(cl + p) - shift;  // unwrapped last-dimension cell
          const int l = y[D - 1] + M - 1 - x;
          const T w = __ldg(bw + (long long)p * E + eoff * TAPS + l);
          const C v = fb[p];
          acc.x = fma(w, v.x, acc.x);
          acc.y = fma(w, v.y, acc.y);
        }
      }
    }
    gout[s] = acc;
  }
}

}  // namespace nfftb
