// dispatch.cuh — kernel-pointer sets per (precision, D, m). The template
// instantiations live in inst_d{1,2,3}.cu so they compile in parallel.
#pragma once

#include "common.cuh"

namespace nfftb {

template <typename T>
struct KernelSet {
  using C = typename cplx<T>::type;
  void (*interp_tiled)(Geom, WinPoly<T>, const C*, const T*, const int*, const int4*, const int*, C*);
  void (*spread_tiled)(Geom, WinPoly<T>, const C*, const T*, const int*, const int4*, const int*, C*);
  const void* interp_direct;  // takes WinPolyN<T, D, m> (launched with launch_k)
  const void* spread_direct;  // takes WinPolyN<T, D, m> (launched with launch_k)
  void (*spread_loc)(Geom, WinPoly<T>, const C*, const T*, const int*, const int4*, const int*, int, C*);
  int loc_threads;
  void (*spread_own)(Geom, WinPoly<T>, const C*, const T*, const int*, const int*, int, int, C*);
  int own_threads;
  void (*spread_sorted)(Geom, WinPoly<T>, const C*, const T*, const int*, const int4*, const int*, C*);
  void (*spread_gather)(Geom, WinPoly<T>, const C*, const T*, const int*, const int4*, const int*, int, C*);
  // D = 1 static-tile kernels (resample1d.cuh)
  const void* interp1;  // takes WinPolyN<T, D, m> (launched with launch_k)
  const void* interp1t;  // TENSOR: taps from the stored table
  const void* spread1;  // takes WinPolyN<T, D, m> (launched with launch_k)
  // D = 1 TENSOR precompute (taps stored by nfft_precompute) and the adjoint over them
  const void* taps1;  // takes WinPolyN<T, D, m> (launched with launch_k)
  const void* spread1t;  // takes WinPolyN<T, D, m> (launched with launch_k)
  // D = 2, 3 static-tile interpolation (resample_nd.cuh)
  void (*interp_nd)(Geom, WinPoly<T>, const C*, const T*, const int*, const int*, int, int, C*);
  // D = 2, 3 over cell-sorted nodes (resample_cell.cuh)
  const void* interp_cell;  // takes WinPolyN<T, D, m> (launched with launch_k)
  const void* interp_cellt;  // TENSOR: taps from the stored table
  const void* interp_cell2;  // fp32 2D batches: two vectors per CTA
  // FULL precompute strategy (resample_full.cuh): the sparse matrix B
  const void* full_build;
  const void* full_interp;
  const void* full_spread;  // D >= 2
  const void* spread_cell;  // takes WinPolyN<T, D, m> (launched with launch_k)
  // D = 2 batches: lanes = batch vectors, window-row parts split evenly over the warps, cp.async-staged
  // chunks, FFMA2 (resample_rowbatch.cuh)
  void (*spread_rb2)(Geom, const C*, int, const T*, const int*, const int*, C*);
  const void* taps_nd;  // takes WinPolyN<T, D, m> (launched with launch_k)
  // D = 2, 3: warp-owned cell blocks over the TENSOR taps (resample_wblock.cuh)
  void (*spread_wb)(Geom, const C*, const int*, const T*, const int*, C*);
  size_t wb_warp_bytes;
};

template <typename T> KernelSet<T> kernels_d1(int m);
template <typename T> KernelSet<T> kernels_d2(int m);
template <typename T> KernelSet<T> kernels_d3(int m);

template <typename T>
inline KernelSet<T> kernels_for(int D, int m) {
  if (D == 1) return kernels_d1<T>(m);
  if (D == 2) return kernels_d2<T>(m);
  return kernels_d3<T>(m);
}

}  // namespace nfftb

#ifdef NFFTB_INSTANTIATE_D
#include "resample.cuh"
#include "resample1d.cuh"
#include "resample_nd.cuh"
#include "resample_cell.cuh"
#include "resample_rowbatch.cuh"
#include "resample_wblock.cuh"
#include "resample_full.cuh"
namespace nfftb {
template <typename T, int D, int M>
KernelSet<T> make_set() {
  constexpr int DEG = poly_degree(M, sizeof(T) == 8);
  KernelSet<T> k{};
  k.interp_direct = (const void*)interp_direct_kernel<T, D, M, DEG>;
  k.spread_direct = (const void*)spread_direct_kernel<T, D, M, DEG>;
#ifdef NFFTB_TILE_VARIANTS
  // first-generation tile-mode variants (methods TILED_CAS .. TILED_V1): reference builds only
  k.interp_tiled = interp_tiled_kernel<T, D, M, DEG>;
  k.spread_tiled = spread_tiled_kernel<T, D, M, DEG>;
  k.spread_sorted = spread_sorted_kernel<T, D, M, DEG>;
  if constexpr (D >= 2) k.interp_nd = interp_nd_kernel<T, D, M, DEG>;
  if constexpr (D <= 2) {
    k.spread_loc = spread_loc_kernel<T, D, M, DEG>;
    k.loc_threads = LocCfg<T, D, M>::THR;
    k.spread_own = spread_own_kernel<T, D, M, DEG>;
    k.own_threads = OwnCfg<T, D, M>::THR;
    k.spread_gather = spread_gather_kernel<T, D, M, DEG>;
  }
#endif
  k.full_build = (const void*)full_build_kernel<T, D, M, DEG>;
  k.full_interp = (const void*)full_interp_kernel<T, D, M>;
  if constexpr (D == 1) {
    k.interp1 = (const void*)interp1s_kernel<T, M, DEG, false>;
    k.interp1t = (const void*)interp1s_kernel<T, M, DEG, true>;
    k.spread1 = (const void*)spread1a_kernel<T, M, DEG, false>;
    k.taps1 = (const void*)taps1_kernel<T, M, DEG>;
    k.spread1t = (const void*)spread1a_kernel<T, M, DEG, true>;
  } else {
    k.interp_cell = (const void*)interp_cell_kernel<T, D, M, DEG, false>;
    k.interp_cellt = (const void*)interp_cell_kernel<T, D, M, DEG, true>;
    if constexpr (D == 2 && sizeof(T) == 4) k.interp_cell2 = (const void*)interp_cell2_kernel<M, DEG>;
    k.full_spread = (const void*)full_spread_kernel<T, D, M>;
    k.spread_cell = (const void*)spread_cell_kernel<T, D, M, DEG>;
    if constexpr (D == 2) {
      k.spread_rb2 = spread_rb2_kernel<T, M>;
    }
    k.taps_nd = (const void*)taps_nd_kernel<T, D, M, DEG>;
    k.spread_wb = spread_wb_kernel<T, D, M>;
    k.wb_warp_bytes = WbCfg<T, D, M>::WARP_BYTES;
  }
  return k;
}
template <typename T, int D>
KernelSet<T> make_set_m(int m) {
  switch (m) {
    case 1: return make_set<T, D, 1>();
    case 2: return make_set<T, D, 2>();
    case 3: return make_set<T, D, 3>();
    case 4: return make_set<T, D, 4>();
    case 5: return make_set<T, D, 5>();
    case 6: return make_set<T, D, 6>();
    case 7: return make_set<T, D, 7>();
    default: return make_set<T, D, 8>();
  }
}
}  // namespace nfftb
#define NFFTB_DEFINE_D(FN, D)                                          \
  namespace nfftb {                                                    \
  template <> KernelSet<double> FN<double>(int m) { return make_set_m<double, D>(m); } \
  template <> KernelSet<float> FN<float>(int m) { return make_set_m<float, D>(m); }    \
  }
#endif
