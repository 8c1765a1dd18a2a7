// grid.cuh — resampling correction fused with zero-pad / crop (SURVEY §8(a)
// rows a4 and a9), and grid zeroing for the adjoint.
//
// Oversampled-grid storage: logical l in I_Ntilde at (l mod Ntilde)_d; with it
// the grid DFT of Alg. 1 l.5 / Alg. 2 l.5 is cuFFT's plain unnormalised
// transform (the paper's fftshift, becomes index placement).
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
// g_n = fhat_n * prod_d beta^tensor_{n_d,d} for n in I_N, 0
// elsewhere. grid.y walks rows of the oversampled grid (batch x all but the
// last dimension, decoded once per CTA); grid.x the contiguous last dimension.
// Every oversampled cell is written exactly once, coalesced.
template <typename T>
__global__ void __launch_bounds__(THREADS) deconv_pad_kernel(Geom g, const typename cplx<T>::type* __restrict__ fhat,
                                                             const T* __restrict__ beta,
                                                             typename cplx<T>::type* __restrict__ grid) {
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
      const int n = s[d] < (g.Nt[d] >> 1) ? s[d] : s[d] - g.Nt[d];  // logical index l in I_Ntilde
      const int i = n + (g.N[d] >> 1);                              // N-grid storage index of n
      inside = inside && i >= 0 && i < g.N[d];
      if (inside) scale *= beta[g.beta_off[d] + i];
      lin = lin * g.N[d] + i;
    }
    const C* src = fhat + (long long)b * g.ngrid_cells + lin * nl;
    C* dst = grid + row * ntl;
    const T* bl = beta + g.beta_off[D - 1];
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < ntl; x += gridDim.x * blockDim.x) {
      const int n = x < (ntl >> 1) ? x : x - ntl;
      const int i = n + (nl >> 1);
      C out;
      out.x = (T)0;
      out.y = (T)0;
      if (inside && i >= 0 && i < nl) {
        const C v = src[i];
        const T sc = scale * bl[i];
        out.x = v.x * sc;
        out.y = v.y * sc;
      }
      dst[x] = out;
    }
  }
}

// Alg. 2 lines 7-9: y_n = g_n * prod_d beta^tensor_{n_d,d},
// n in I_N, read from (n mod Ntilde). Same row/column launch over the N-grid.
template <typename T>
__global__ void __launch_bounds__(THREADS) crop_deconv_kernel(Geom g, const typename cplx<T>::type* __restrict__ grid,
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

// Zero the oversampled grid (B * prod Ntilde complex), 16-byte stores.
__global__ void __launch_bounds__(THREADS) zero_kernel(float4* __restrict__ p, long long n16) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    p[i] = z;
}

}  // namespace nfftb
