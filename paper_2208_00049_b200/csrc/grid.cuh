// grid.cuh — resampling correction fused with zero-pad / crop (SURVEY §8(a)
// rows a4 and a9).
//
// Oversampled-grid storage: logical l in I_Ntilde at (l mod Ntilde)_d; with it
// the grid DFT of Alg. 1 l.5 / Alg. 2 l.5 is cuFFT's plain unnormalised
// transform (the paper's fftshift, becomes index placement).
// Three plan-owned grids (DESIGN.md §HBM layout): the forward input (zero
// padding persists), the forward FFT output (out-of-place) and the adjoint
// grid (zero between adjoints: crop_zero re-zeroes it).
#pragma once

#include "common.cuh"

namespace nfftb {

// Decode a "row" (batch index b and all but the last grid dimension) of an
// array with extents ext[0..D-1] into per-dimension indices; uniform per CTA.
__device__ __forceinline__ int decode_row(long long row, int D, const int* ext, int* idx) {
  long long r = row;
  for (int d = D - 2; d >= 0; --d) {
    idx[d] = (int)(r % ext[d]);
    r /= ext[d];
  }
  return (int)r;  // batch index
}

// Alg. 1 lines 1-3 with the tensor-product correction of
// g_n = fhat_n * prod_d beta^tensor_{n_d,d} for n in I_N.
// The forward input grid keeps its zero padding between calls (the FFT is
// out-of-place), so only the |I_N| cells are written: one thread per N-grid
// cell, grid.y over rows (batch x all but the last dimension), grid.x over the
// contiguous last dimension.
template <typename T>
__global__ void __launch_bounds__(THREADS) deconv_place_kernel(Geom g, const typename cplx<T>::type* __restrict__ fhat,
                                                               const T* __restrict__ beta,
                                                               typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  const int D = g.D;
  const int ntl = g.Nt[D - 1], nl = g.N[D - 1];
  const long long rows = (long long)g.B * (g.ngrid_cells / nl);
  for (long long row = blockIdx.y; row < rows; row += gridDim.y) {
    int i[MAX_D];
    const int b = decode_row(row, D, g.N, i);
    T scale = (T)1;
    long long lin = 0;
    for (int d = 0; d < D - 1; ++d) {
      const int n = i[d] - (g.N[d] >> 1);
      const int s = n < 0 ? n + g.Nt[d] : n;  // storage of l = n: (n mod Ntilde)
      scale *= beta[g.beta_off[d] + i[d]];
      lin = lin * g.Nt[d] + s;
    }
    const C* src = fhat + row * nl;
    C* dst = grid + (long long)b * g.grid_cells + lin * ntl;
    const T* bl = beta + g.beta_off[D - 1];
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nl; x += gridDim.x * blockDim.x) {
      const int n = x - (nl >> 1);
      const int s = n < 0 ? n + ntl : n;
      const C v = src[x];
      const T sc = scale * bl[x];
      C out;
      out.x = v.x * sc;
      out.y = v.y * sc;
      dst[s] = out;
    }
  }
}

// Alg. 2 lines 7-9: y_n = g_n * prod_d beta^tensor_{n_d,d},
// n in I_N, read from (n mod Ntilde) — fused with re-zeroing the adjoint grid
// for the next spread (the adjoint's grid-is-zero invariant): one thread per
// oversampled cell reads it if it is in I_N and then writes 0.
template <typename T>
__global__ void __launch_bounds__(THREADS) crop_zero_kernel(Geom g, typename cplx<T>::type* __restrict__ grid,
                                                            const T* __restrict__ beta,
                                                            typename cplx<T>::type* __restrict__ y) {
  using C = typename cplx<T>::type;
  const int D = g.D;
  const int ntl = g.Nt[D - 1], nl = g.N[D - 1];
  const long long rows = (long long)g.B * (g.grid_cells / ntl);
  for (long long row = blockIdx.y; row < rows; row += gridDim.y) {
    int s[MAX_D];
    const int b = decode_row(row, D, g.Nt, s);
    bool inside = true;
    T scale = (T)1;
    long long lin = 0;
    for (int d = 0; d < D - 1; ++d) {
      const int n = s[d] < (g.Nt[d] >> 1) ? s[d] : s[d] - g.Nt[d];
      const int i = n + (g.N[d] >> 1);
      inside = inside && i >= 0 && i < g.N[d];
      if (inside) scale *= beta[g.beta_off[d] + i];
      lin = lin * g.N[d] + i;
    }
    C* src = grid + row * ntl;
    C* dst = y + (long long)b * g.ngrid_cells + lin * nl;
    const T* bl = beta + g.beta_off[D - 1];
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < ntl; x += gridDim.x * blockDim.x) {
      const int n = x < (ntl >> 1) ? x : x - ntl;
      const int i = n + (nl >> 1);
      if (inside && i >= 0 && i < nl) {
        const C v = src[x];
        const T sc = scale * bl[i];
        C out;
        out.x = v.x * sc;
        out.y = v.y * sc;
        dst[i] = out;
      }
      C z;
      z.x = (T)0;
      z.y = (T)0;
      src[x] = z;
    }
  }
}

// Alg. 2 lines 7-9 without the re-zeroing, for spreading kernels that write
// every grid cell themselves (resample1d.cuh: owner-computes): one thread per
// N-grid cell, rows as in deconv_place_kernel.
template <typename T>
__global__ void __launch_bounds__(THREADS) crop_kernel(Geom g, const typename cplx<T>::type* __restrict__ grid,
                                                       const T* __restrict__ beta,
                                                       typename cplx<T>::type* __restrict__ y) {
  using C = typename cplx<T>::type;
  const int D = g.D;
  const int ntl = g.Nt[D - 1], nl = g.N[D - 1];
  const long long rows = (long long)g.B * (g.ngrid_cells / nl);
  for (long long row = blockIdx.y; row < rows; row += gridDim.y) {
    int i[MAX_D];
    const int b = decode_row(row, D, g.N, i);
    T scale = (T)1;
    long long lin = 0;
    for (int d = 0; d < D - 1; ++d) {
      const int n = i[d] - (g.N[d] >> 1);
      const int s = n < 0 ? n + g.Nt[d] : n;
      scale *= beta[g.beta_off[d] + i[d]];
      lin = lin * g.Nt[d] + s;
    }
    const C* src = grid + (long long)b * g.grid_cells + lin * ntl;
    C* dst = y + row * nl;
    const T* bl = beta + g.beta_off[D - 1];
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < nl; x += gridDim.x * blockDim.x) {
      const int n = x - (nl >> 1);
      const int s = n < 0 ? n + ntl : n;
      const C v = src[s];
      const T sc = scale * bl[x];
      C out;
      out.x = v.x * sc;
      out.y = v.y * sc;
      dst[x] = out;
    }
  }
}

// Deconvolution + placement (FWD, Alg. 1 lines 1-3) and crop + deconvolution
// (!FWD, Alg. 2 lines 7-9, cell mode: no re-zeroing) over a FLATTENED index:
// one thread per two consecutive last-dimension cells of any row (batch x all
// but the last dimension), 32-bit index arithmetic (the host guarantees
// B * prod N / 2 < 2^31). Every thread is busy whatever N_{D-1} is (the
// row-per-CTA kernels above leave 3/4 of a CTA idle at N = 64 and decode
// their rows with 64-bit divisions).
template <typename T, bool FWD>
__global__ void __launch_bounds__(THREADS) correct_flat_kernel(Geom g, const typename cplx<T>::type* __restrict__ in,
                                                               const T* __restrict__ beta,
                                                               typename cplx<T>::type* __restrict__ out) {
  using C = typename cplx<T>::type;
  const int D = g.D;
  const int ntl = g.Nt[D - 1], nl = g.N[D - 1];
  const int hp = (nl + 1) >> 1;  // cell pairs per row
  const int units = (int)((long long)g.B * (g.ngrid_cells / nl)) * hp;
  const T* bl = beta + g.beta_off[D - 1];
  // the crop may be launched programmatically after the inverse FFT (stage_crop, pdl): wait for the grid
  if constexpr (!FWD) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int u = blockIdx.x * THREADS + threadIdx.x; u < units; u += gridDim.x * THREADS) {
    const int row = u / hp;
    const int x0 = (u - row * hp) * 2;
    int r = row;
    T scale = (T)1;
    long long lin = 0, mul = 1;  // storage row of the oversampled grid (all but the last dimension)
    for (int d = D - 2; d >= 0; --d) {
      const int i = r % g.N[d];
      r /= g.N[d];
      const int n = i - (g.N[d] >> 1);
      scale *= beta[g.beta_off[d] + i];
      lin += (long long)(n < 0 ? n + g.Nt[d] : n) * mul;
      mul *= g.Nt[d];
    }
    const long long gbase = (long long)r * g.grid_cells + lin * ntl;  // r = batch index
    const long long nbase = (long long)row * nl;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int x = x0 + v;
      if (x < nl) {
        const int n = x - (nl >> 1);
        const int s = n < 0 ? n + ntl : n;
        const T sc = scale * bl[x];
        const C a = FWD ? in[nbase + x] : in[gbase + s];
        C o;
        o.x = a.x * sc;
        o.y = a.y * sc;
        if (FWD) out[gbase + s] = o;
        else out[nbase + x] = o;
      }
    }
  }
}

}  // namespace nfftb
