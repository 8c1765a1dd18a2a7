// grid.cuh — resampling correction fused with zero-pad / crop (SURVEY §8(a)
// rows a4 and a9), and grid zeroing for the adjoint.
//
// Oversampled-grid storage: logical l in I_Ntilde at (l mod Ntilde)_d; with it
// the grid DFT of Alg. 1 l.5 / Alg. 2 l.5 is cuFFT's plain unnormalised
// transform (the paper's fftshift, becomes index placement).
#pragma once

#include "common.cuh"

namespace nfftb {

// Alg. 1 lines 1-3 with the tensor-product correction of
// g_n = fhat_n * prod_d beta^tensor_{n_d,d} for n in I_N,
// 0 elsewhere. One thread per oversampled cell: every cell is written once,
// coalesced; the N-grid is read in contiguous runs.
template <typename T>
__global__ void __launch_bounds__(THREADS) deconv_pad_kernel(Geom g, const typename cplx<T>::type* __restrict__ fhat,
                                                             const T* __restrict__ beta,
                                                             typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  const long long total = g.grid_cells * g.B;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long rem = idx;
    long long lin = 0, stride = 1;
    T scale = (T)1;
    bool inside = true;
    for (int d = g.D - 1; d >= 0; --d) {
      const int s = (int)(rem % g.Nt[d]);
      rem /= g.Nt[d];
      const int n = s < (g.Nt[d] >> 1) ? s : s - g.Nt[d];  // logical index l in I_Ntilde
      const int i = n + (g.N[d] >> 1);                       // N-grid storage index of n
      if (i < 0 || i >= g.N[d]) {
        inside = false;
      } else {
        scale *= beta[g.beta_off[d] + i];
        lin += (long long)i * stride;
      }
      stride *= g.N[d];
    }
    C out;
    if (inside) {
      const C v = fhat[rem * g.ngrid_cells + lin];  // rem = batch index
      out.x = v.x * scale;
      out.y = v.y * scale;
    } else {
      out.x = (T)0;
      out.y = (T)0;
    }
    grid[idx] = out;
  }
}

// Alg. 2 lines 7-9: y_n = g_n * prod_d beta^tensor_{n_d,d},
// n in I_N, read from (n mod Ntilde). One thread per N-grid cell.
template <typename T>
__global__ void __launch_bounds__(THREADS) crop_deconv_kernel(Geom g, const typename cplx<T>::type* __restrict__ grid,
                                                              const T* __restrict__ beta,
                                                              typename cplx<T>::type* __restrict__ y) {
  using C = typename cplx<T>::type;
  const long long total = g.ngrid_cells * g.B;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long rem = idx;
    long long src = 0, stride = 1;
    T scale = (T)1;
    for (int d = g.D - 1; d >= 0; --d) {
      const int i = (int)(rem % g.N[d]);
      rem /= g.N[d];
      const int n = i - (g.N[d] >> 1);
      const int s = n < 0 ? n + g.Nt[d] : n;
      src += (long long)s * stride;
      stride *= g.Nt[d];
      scale *= beta[g.beta_off[d] + i];
    }
    const C v = grid[rem * g.grid_cells + src];
    C out;
    out.x = v.x * scale;
    out.y = v.y * scale;
    y[idx] = out;
  }
}

// Zero the oversampled grid (B * prod Ntilde complex), 16-byte stores.
__global__ void __launch_bounds__(THREADS) zero_kernel(float4* __restrict__ p, long long n16) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    p[i] = z;
}

}  // namespace nfftb
