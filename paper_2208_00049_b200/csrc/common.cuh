// common.cuh — shared types and device helpers of the sm_100a NFFT path.
// (Product code; shares nothing with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace nfftb {

constexpr int MAX_D = 3;
constexpr int MAX_M = 8;    // half-width m; 2m taps per dimension
constexpr int MAX_Z = 17;   // polynomial coefficients per tap (degree <= 16)
constexpr int THREADS = 256;

// Window-table degree (DESIGN.md §Window tables): the paper's degree 2m
// is raised in fp64 so the table error stays <= 5e-14 of the
// peak, far below the 1e-12 parity bar (LSQ fit, sigma = 2 / 1.25: degree 14
// for m <= 5, degree 12 for m >= 6 — 4.5e-14 at m = 6, 1.4e-14 at m = 8;
// tools/poly_degree.py); fp32 uses max(2m, 8) (m >= 5) and 8.
__host__ __device__ constexpr int poly_degree(int m, bool fp64) {
  return fp64 ? (m <= 5 ? 14 : 12) : (2 * m > 8 ? 2 * m : 8);
}

// Phase timestamps for the timeline harness (tools/micro/trace1d.cu defines
// NFFTB_PHASE_TRACE before including the kernels); empty in the library.
#ifdef NFFTB_PHASE_TRACE
__device__ unsigned long long nfftb_trace[1 << 16];
#define NFFTB_TRACE(slot)                                                                          \
  do {                                                                                             \
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 8192) {                               \
      unsigned long long t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      nfftb_trace[blockIdx.x * 8 + (slot)] = t_;                                                   \
    }                                                                                              \
  } while (0)
#else
#define NFFTB_TRACE(slot) \
  do {                    \
  } while (0)
#endif

template <typename T> struct cplx;
template <> struct cplx<double> { using type = double2; };
template <> struct cplx<float> { using type = float2; };

// Geometry passed by value to every kernel.
struct Geom {
  int D;
  int M;          // number of nodes
  int B;          // batch
  int m;          // half-width
  int Nt[MAX_D];  // oversampled size Ntilde_d
  int N[MAX_D];   // N_d
  int Q[MAX_D];   // tile size
  int P[MAX_D];   // tiles per dimension
  int L[MAX_D];   // tile region extent Q_d + 2m - 1
  double Ntd[MAX_D];
  long long grid_cells;   // prod Ntilde
  long long ngrid_cells;  // prod N
  int region_cells;       // prod L
  int beta_off[MAX_D];    // offset of dim d in the beta^tensor vector
};

// Piecewise-polynomial window table for taps 0..m-1 of each dimension
// (taps m..2m-1 are their mirrors, see taps()). Passed as a kernel parameter
// so every coefficient is a constant-bank operand of the FMA.
template <typename T> struct WinPoly { T mu[MAX_D][MAX_M][MAX_Z]; };

// The same table cut to the kernel's (D, m, degree): what the resampling
// kernels take as a parameter. Kernel parameters live in the constant bank,
// so every coefficient is an immediate operand of the FMA, and a small
// parameter block keeps the launch cheap (measured on B200: an empty
// 1024-CTA kernel with the full 3.3 KB table costs 5.9 us per stream launch,
// 3.9 us without).
template <typename T, int D, int M>
struct WinPolyN {
  static constexpr int Z = poly_degree(M, sizeof(T) == 8) + 1;
  T mu[D][M][Z];
};

// Cell of a node along one dimension (reading R5/R10):
// t = Ntilde * k (one IEEE multiply, never contracted), a = floor(t),
// frac = t - a (exact), c = (a + Ntilde/2) mod Ntilde in [0, Ntilde).
__device__ __forceinline__ int node_cell(double k, double Ntd, int Nt, double& frac) {
  const double t = __dmul_rn(Ntd, k);
  const double a = floor(t);
  frac = t - a;
  int c;
  if (fabs(a) < 1073741824.0) {  // |a| < 2^30: exact as int; c = (a + Nt/2) mod Nt, usually no wrap
    c = (int)a + (Nt >> 1);
    if ((unsigned)c >= (unsigned)Nt) {
      c %= Nt;
      if (c < 0) c += Nt;
    }
  } else {  // nodes far outside the torus (periodic fold, reading R10)
    const double r = fmod(a, Ntd);  // exact for integer-valued doubles, |r| < Ntilde
    c = (int)r + (Nt >> 1);
    if (c < 0) c += Nt;
    else if (c >= Nt) c -= Nt;
  }
  return c;
}

__device__ __forceinline__ int pos_mod(int a, int n) {
  int r = a % n;
  return r < 0 ? r + n : r;
}

// 2m window taps from the polynomial table at zeta = frac - 1/2.
// Tap l (cell a-m+1+l) and tap 2m-1-l are mirror images, w_{2m-1-l}(zeta) =
// w_l(-zeta) (the window is even), so with p_l = E(zeta^2) + zeta O(zeta^2):
// w_l = E + zeta O, w_{2m-1-l} = E - zeta O.
template <typename T, int M, int DEG, int ML, int ZL>
__device__ __forceinline__ void window_taps(T zeta, const T (&mu)[ML][ZL], T (&w)[2 * M]) {
  static_assert(ML >= M && ZL > DEG, "window table too small");
  const T z2 = zeta * zeta;
#pragma unroll
  for (int l = 0; l < M; ++l) {
    T e = mu[l][DEG];
#pragma unroll
    for (int z = DEG - 2; z >= 0; z -= 2) e = fma(e, z2, mu[l][z]);
    T o = mu[l][DEG - 1];
#pragma unroll
    for (int z = DEG - 3; z >= 1; z -= 2) o = fma(o, z2, mu[l][z]);
    w[l] = fma(zeta, o, e);
    w[2 * M - 1 - l] = fma(-zeta, o, e);
  }
}

// shared-memory bytes of spread_loc_kernel (host and device agree)
__host__ __device__ inline size_t loc_smem_bytes(int D, int M, size_t csize, size_t rsize, int region_cells, int S,
                                                 int nst) {
  const size_t taps = (size_t)S * D * 2 * M * rsize;
  size_t b = (size_t)region_cells * csize + taps;
  b = (b + 15) & ~(size_t)15;
  b += (size_t)S * csize;                        // f values of one batch vector
  b += (size_t)S * 4 * (2 + D);                  // j, order, loc[D]
  b += (size_t)(2 * nst + 2) * 4;                // sub-tile offsets and cursors
  return b;
}

__host__ __device__ inline size_t own_smem_bytes(int D, int M, size_t csize, size_t rsize, int tile_cells, int thr,
                                                 int nst_ext) {
  size_t b = (size_t)tile_cells * csize;                   // accumulator
  b += (size_t)thr * D * 2 * M * rsize;                    // taps of one chunk
  b = (b + 15) & ~(size_t)15;
  b += (size_t)thr * csize;                                // f values of the chunk
  b += (size_t)thr * 4 * (1 + 1 + D);                      // node j, order, footprint start per dim
  b += (size_t)2048 * 4;                                   // relevant-node list (sorted positions)
  b += (size_t)(2 * nst_ext + 4) * 4;                      // bucket offsets, cursors, counters
  return b;
}

__host__ __device__ inline size_t gather_smem_bytes(int D, int M, size_t csize, size_t rsize, int tile_cells, int S) {
  size_t b = (size_t)S * D * 2 * M * rsize;  // taps per sorted slot
  b = (b + 15) & ~(size_t)15;
  b += (size_t)S * csize;                    // f of the current batch vector
  b += (size_t)S * 4 * (D + 1);              // local cell per dim, node j
  b += (size_t)2 * (tile_cells + 1) * 4;     // cell offsets, cursors
  return b;
}

// ---- warp-wide exclusive scan of one int per lane ----
__device__ __forceinline__ int warp_exclusive_scan(int x, int& total) {
  const int lane = threadIdx.x & 31;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - x;
}

// ---- block-wide exclusive scan of one int per thread (blockDim = THREADS) ----
__device__ __forceinline__ int block_exclusive_scan(int x, int* ws, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) ws[lane] = t;
  }
  __syncthreads();
  const int prefix = w > 0 ? ws[w - 1] : 0;
  total = ws[nw - 1];
  __syncthreads();
  return prefix + inc - x;
}

}  // namespace nfftb
