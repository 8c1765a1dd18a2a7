// resample.cuh — the NFFT hot path: forward interpolation (grid -> nodes)
// and adjoint spreading (nodes -> grid) with the Kaiser–Bessel window
// (SURVEY §8(a) rows a6, a7).
//
//   forward: f_j = sum_{l in I_{Nt,m}(k_j)} ghat_l psi~(k_j - l/Nt)        (Alg. 3)
//   adjoint: ghat_l += f_j psi~(k_j - l/Nt) for l in I_{Nt,m}(k_j)          (Alg. 4)
//
// Tiled kernels (Alg. 3/4): one CTA per subproblem (<= S
// nodes of one tile); the tile's grid region (Q_d + 2m - 1 cells per
// dimension, the block index set I^block_{p,m} of PAPER.md:535) is staged in
// shared memory with coalesced 16-byte loads and the periodic wrap resolved
// at staging time (Remark PAPER.md:588-590), so the inner loops never wrap.
// Per node the 2m taps per dimension are evaluated once into registers
// and the (2m)^D multiply-adds run with the innermost
// dimension contiguous in shared memory. The adjoint accumulates into the
// shared tile and flushes tile+halo to the grid with global reductions — the
// GPU form of the paper's mutex-protected merge.
//
// Direct kernels ("regular resampling"): one thread per sorted
// node straight from L2/HBM; the unblocked reference and the fallback when a
// tile region does not fit shared memory.
#pragma once

#include "common.cuh"

namespace nfftb {

template <typename T>
__device__ __forceinline__ void red_add(typename cplx<T>::type* p, typename cplx<T>::type v);
template <>
__device__ __forceinline__ void red_add<double>(double2* p, double2 v) {
  atomicAdd(&p->x, v.x);
  atomicAdd(&p->y, v.y);
}
template <>
__device__ __forceinline__ void red_add<float>(float2* p, float2 v) {
  atomicAdd(p, v);  // sm_90+: vector float2 reduction (REDG.E.ADD.F32x2)
}

__device__ __forceinline__ int wrap_up(int s, int n) {
  while (s >= n) s -= n;
  return s;
}

struct TileCoords {
  int p[MAX_D];     // tile multi-index
  int base[MAX_D];  // storage index of the first region cell per dim
};

template <int D, int M>
__device__ __forceinline__ TileCoords tile_coords(const Geom& g, int tile) {
  TileCoords tc;
  int rem = tile;
#pragma unroll
  for (int d = D - 1; d >= 0; --d) {
    tc.p[d] = rem % g.P[d];
    rem /= g.P[d];
  }
#pragma unroll
  for (int d = 0; d < D; ++d) tc.base[d] = pos_mod(tc.p[d] * g.Q[d] - M + 1 - (g.Nt[d] >> 1), g.Nt[d]);
  return tc;
}

// Node setup: local region coordinates of the footprint start and the taps.
// Returns false when the node does not belong to the tile (cannot happen for
// a consistent plan; guards shared-memory indexing against corrupted input).
template <typename T, int D, int M, int DEG>
__device__ __forceinline__ bool node_setup(const Geom& g, const WinPoly<T>& wp, const T* __restrict__ ks, int i,
                                           const TileCoords& tc, int (&loc)[D], T (&w)[D][2 * M]) {
  bool ok = true;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double frac;
    const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
    loc[d] = c - tc.p[d] * g.Q[d];
    ok = ok && (unsigned)loc[d] < (unsigned)g.Q[d];
    window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w[d]);
  }
  return ok;
}

// Visit every region cell row by row (innermost dimension across lanes):
// fn(region_index, storage_offset_in_batch_slice).
template <int D, typename F>
__device__ __forceinline__ void for_region(const Geom& g, const TileCoords& tc, F&& fn) {
  if (D == 1) {
    for (int c = threadIdx.x; c < g.L[0]; c += blockDim.x) fn(c, (long long)wrap_up(tc.base[0] + c, g.Nt[0]));
  } else {
    const int Ll = g.L[D - 1];
    const int rows = g.region_cells / Ll;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = warp; r < rows; r += nw) {
      long long off;
      if (D == 2) {
        off = (long long)wrap_up(tc.base[0] + r, g.Nt[0]) * g.Nt[1];
      } else {
        const int i1 = r % g.L[1], i0 = r / g.L[1];
        off = ((long long)wrap_up(tc.base[0] + i0, g.Nt[0]) * g.Nt[1] + wrap_up(tc.base[1] + i1, g.Nt[1])) * g.Nt[2];
      }
      for (int c = lane; c < Ll; c += 32) fn(r * Ll + c, off + wrap_up(tc.base[D - 1] + c, g.Nt[D - 1]));
    }
  }
}

// (2m)^D tensor-product sum over a region held in shared memory (eq.
// InnerTensorStructure): innermost dimension contiguous.
template <typename T, int D, int M>
__device__ __forceinline__ typename cplx<T>::type gather_tile(const Geom& g, const typename cplx<T>::type* tile,
                                                              const int (&loc)[D], const T (&w)[D][2 * M]) {
  using C = typename cplx<T>::type;
  C acc;
  acc.x = (T)0;
  acc.y = (T)0;
  if (D == 1) {
    const C* row = tile + loc[0];
#pragma unroll
    for (int l = 0; l < 2 * M; ++l) {
      const C v = row[l];
      acc.x = fma(w[0][l], v.x, acc.x);
      acc.y = fma(w[0][l], v.y, acc.y);
    }
  } else if (D == 2) {
    const int L1 = g.L[1];
#pragma unroll
    for (int l0 = 0; l0 < 2 * M; ++l0) {
      const C* row = tile + (loc[0] + l0) * L1 + loc[1];
      C s;
      s.x = (T)0;
      s.y = (T)0;
#pragma unroll
      for (int l1 = 0; l1 < 2 * M; ++l1) {
        const C v = row[l1];
        s.x = fma(w[1][l1], v.x, s.x);
        s.y = fma(w[1][l1], v.y, s.y);
      }
      acc.x = fma(w[0][l0], s.x, acc.x);
      acc.y = fma(w[0][l0], s.y, acc.y);
    }
  } else {
    const int L1 = g.L[1], L2 = g.L[2];
    constexpr int U0 = (2 * M <= 8) ? 2 * M : 1;
#pragma unroll U0
    for (int l0 = 0; l0 < 2 * M; ++l0) {
      C s1;
      s1.x = (T)0;
      s1.y = (T)0;
#pragma unroll
      for (int l1 = 0; l1 < 2 * M; ++l1) {
        const C* row = tile + ((loc[0] + l0) * L1 + loc[1] + l1) * L2 + loc[2];
        C s;
        s.x = (T)0;
        s.y = (T)0;
#pragma unroll
        for (int l2 = 0; l2 < 2 * M; ++l2) {
          const C v = row[l2];
          s.x = fma(w[2][l2], v.x, s.x);
          s.y = fma(w[2][l2], v.y, s.y);
        }
        s1.x = fma(w[1][l1], s.x, s1.x);
        s1.y = fma(w[1][l1], s.y, s1.y);
      }
      acc.x = fma(w[0][l0], s1.x, acc.x);
      acc.y = fma(w[0][l0], s1.y, acc.y);
    }
  }
  return acc;
}

// Scatter one node's (2m)^D contributions into the shared tile.
template <typename T, int D, int M>
__device__ __forceinline__ void scatter_tile(const Geom& g, typename cplx<T>::type* tile, const int (&loc)[D],
                                             const T (&w)[D][2 * M], typename cplx<T>::type v) {
  using C = typename cplx<T>::type;
  if (D == 1) {
    C* row = tile + loc[0];
#pragma unroll
    for (int l = 0; l < 2 * M; ++l) {
      atomicAdd(&row[l].x, w[0][l] * v.x);
      atomicAdd(&row[l].y, w[0][l] * v.y);
    }
  } else if (D == 2) {
    const int L1 = g.L[1];
#pragma unroll
    for (int l0 = 0; l0 < 2 * M; ++l0) {
      C* row = tile + (loc[0] + l0) * L1 + loc[1];
      const T a = w[0][l0] * v.x, b = w[0][l0] * v.y;
#pragma unroll
      for (int l1 = 0; l1 < 2 * M; ++l1) {
        atomicAdd(&row[l1].x, w[1][l1] * a);
        atomicAdd(&row[l1].y, w[1][l1] * b);
      }
    }
  } else {
    const int L1 = g.L[1], L2 = g.L[2];
    constexpr int U0 = (2 * M <= 8) ? 2 * M : 1;
#pragma unroll U0
    for (int l0 = 0; l0 < 2 * M; ++l0) {
      const T a0 = w[0][l0] * v.x, b0 = w[0][l0] * v.y;
#pragma unroll
      for (int l1 = 0; l1 < 2 * M; ++l1) {
        C* row = tile + ((loc[0] + l0) * L1 + loc[1] + l1) * L2 + loc[2];
        const T a = w[1][l1] * a0, b = w[1][l1] * b0;
#pragma unroll
        for (int l2 = 0; l2 < 2 * M; ++l2) {
          atomicAdd(&row[l2].x, w[2][l2] * a);
          atomicAdd(&row[l2].y, w[2][l2] * b);
        }
      }
    }
  }
}

// ------------------------------------------------------------ forward, tiled
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(THREADS) interp_tiled_kernel(Geom g, WinPoly<T> wp,
                                                               const typename cplx<T>::type* __restrict__ grid,
                                                               const T* __restrict__ ks, const int* __restrict__ perm,
                                                               const int4* __restrict__ subs,
                                                               const int* __restrict__ nsub_ptr,
                                                               typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tile = reinterpret_cast<C*>(smem_raw);
  const int nsub = *nsub_ptr;
  for (int s = blockIdx.x; s < nsub; s += gridDim.x) {
    const int4 sp = subs[s];
    const TileCoords tc = tile_coords<D, M>(g, sp.x);
    int loc[D];
    T w[D][2 * M];
    int j = 0;
    bool has = threadIdx.x < sp.z;
    if (has) {
      const int i = sp.y + threadIdx.x;
      j = perm[i];
      has = node_setup<T, D, M, DEG>(g, wp, ks, i, tc, loc, w);
    }
    for (int b = 0; b < g.B; ++b) {
      const C* src = grid + (long long)b * g.grid_cells;
      __syncthreads();  // previous users of the tile are done
      for_region<D>(g, tc, [&](int r, long long off) { tile[r] = src[off]; });
      __syncthreads();
      if (has) f[(long long)b * g.M + j] = gather_tile<T, D, M>(g, tile, loc, w);
    }
  }
}

// ------------------------------------------------------------ adjoint, tiled
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(THREADS) spread_tiled_kernel(Geom g, WinPoly<T> wp,
                                                               const typename cplx<T>::type* __restrict__ f,
                                                               const T* __restrict__ ks, const int* __restrict__ perm,
                                                               const int4* __restrict__ subs,
                                                               const int* __restrict__ nsub_ptr,
                                                               typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tile = reinterpret_cast<C*>(smem_raw);
  const int nsub = *nsub_ptr;
  for (int s = blockIdx.x; s < nsub; s += gridDim.x) {
    const int4 sp = subs[s];
    const TileCoords tc = tile_coords<D, M>(g, sp.x);
    int loc[D];
    T w[D][2 * M];
    int j = 0;
    bool has = threadIdx.x < sp.z;
    if (has) {
      const int i = sp.y + threadIdx.x;
      j = perm[i];
      has = node_setup<T, D, M, DEG>(g, wp, ks, i, tc, loc, w);
    }
    for (int b = 0; b < g.B; ++b) {
      __syncthreads();  // previous flush done
      for (int r = threadIdx.x; r < g.region_cells; r += blockDim.x) {
        tile[r].x = (T)0;
        tile[r].y = (T)0;
      }
      __syncthreads();
      if (has) scatter_tile<T, D, M>(g, tile, loc, w, f[(long long)b * g.M + j]);
      __syncthreads();
      C* dst = grid + (long long)b * g.grid_cells;
      for_region<D>(g, tc, [&](int r, long long off) {
        const C v = tile[r];
        if (v.x != (T)0 || v.y != (T)0) red_add<T>(dst + off, v);
      });
    }
  }
}

// ------------------------------------------------------------ adjoint, tiled, conflict-free
// "Lanes own cells" spreading (spread): no shared-memory
// atomics (fp32/fp64 shared atomics are CAS loops on sm_100a). The subproblem's
// nodes are bucketed by 2m-wide sub-tiles of the tile; sub-tiles are coloured
// by the parity of their index in every dimension, so the footprints of nodes
// in two different sub-tiles of one colour never overlap. Colours run one after
// another (barrier between); within a colour each worker (G lanes) walks the
// nodes of its sub-tiles in order and adds one node's (2m)^D footprint per
// G-cell step with plain loads/stores, each lane owning distinct cells. Taps
// are computed once per node (even/odd polynomial, registers) and kept in
// shared memory for all batch vectors. The tile region (+ halo) is flushed to
// the grid with vector reductions, the GPU form of Alg. 4's locked merge.
__host__ __device__ constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }

template <typename T, int D, int M>
struct LocCfg {
  static constexpr int TAPS = 2 * M;
  static constexpr int F = ipow_c(TAPS, D);  // footprint cells
  static constexpr int G = F < 32 ? F : 32;  // lanes per node
  static constexpr int WPW = 32 / G;         // workers per warp
  static constexpr int STEPS = (F + G - 1) / G;
  static constexpr int THR = D == 1 ? 256 : 128;
};

template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(LocCfg<T, D, M>::THR) spread_loc_kernel(
    Geom g, WinPoly<T> wp, const typename cplx<T>::type* __restrict__ f, const T* __restrict__ ks,
    const int* __restrict__ perm, const int4* __restrict__ subs, const int* __restrict__ nsub_ptr, int S,
    typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  using L = LocCfg<T, D, M>;
  constexpr int TAPS = L::TAPS, F = L::F, G = L::G, STEPS = L::STEPS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int NS[MAX_D], nst = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    NS[d] = (g.Q[d] + TAPS - 1) / TAPS;
    nst *= NS[d];
  }
  C* acc = reinterpret_cast<C*>(smem_raw);
  T* tap = reinterpret_cast<T*>(acc + g.region_cells);  // [S][D][TAPS]
  size_t off = ((size_t)g.region_cells * sizeof(C) + (size_t)S * D * TAPS * sizeof(T) + 15) & ~(size_t)15;
  C* fv = reinterpret_cast<C*>(smem_raw + off);
  int* jv = reinterpret_cast<int*>(fv + S);
  int* order = jv + S;
  int* lv = order + S;       // [D][S]
  int* stoff = lv + D * S;   // [nst + 1]
  int* stcur = stoff + nst + 1;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lg = lane % G;
  const bool worker_lane = lane < L::WPW * G;  // e.g. m = 3 in 1D: 5 groups of 6 lanes, 2 idle lanes
  const int worker = worker_lane ? warp * L::WPW + lane / G : 1 << 30;
  const int nworkers = (blockDim.x >> 5) * L::WPW;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane / G * G));
  int strides[MAX_D];
  strides[D - 1] = 1;
#pragma unroll
  for (int d = D - 2; d >= 0; --d) strides[d] = strides[d + 1] * g.L[d + 1];

  const int nsub = *nsub_ptr;
  for (int sidx = blockIdx.x; sidx < nsub; sidx += gridDim.x) {
    const int4 sp = subs[sidx];
    const TileCoords tc = tile_coords<D, M>(g, sp.x);
    for (int i = threadIdx.x; i <= nst; i += blockDim.x) stoff[i] = 0;
    __syncthreads();
    // 1. node setup: taps into shared memory, sub-tile histogram
    for (int t = threadIdx.x; t < sp.z; t += blockDim.x) {
      const int i = sp.y + t;
      int loc[D];
      T w[D][TAPS];
      const bool ok = node_setup<T, D, M, DEG>(g, wp, ks, i, tc, loc, w);
      jv[t] = ok ? perm[i] : -1;
      int st = 0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        lv[d * S + t] = loc[d];
        st = st * NS[d] + (ok ? loc[d] / TAPS : 0);
#pragma unroll
        for (int l = 0; l < TAPS; ++l) tap[(t * D + d) * TAPS + l] = w[d][l];
      }
      order[t] = st;  // temporarily the sub-tile id
      if (ok) atomicAdd(&stoff[st + 1], 1);
    }
    __syncthreads();
    // 2. exclusive offsets of the sub-tile buckets (nst is small)
    if (threadIdx.x == 0) {
      for (int q = 1; q <= nst; ++q) stoff[q] += stoff[q - 1];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nst; q += blockDim.x) stcur[q] = stoff[q];
    __syncthreads();
    int myslot[8];
    int nmine = 0;
    for (int t = threadIdx.x; t < sp.z; t += blockDim.x) {
      if (jv[t] >= 0) myslot[nmine] = atomicAdd(&stcur[order[t]], 1);
      ++nmine;
    }
    __syncthreads();
    nmine = 0;
    for (int t = threadIdx.x; t < sp.z; t += blockDim.x) {
      if (jv[t] >= 0) order[myslot[nmine]] = t;
      ++nmine;
    }
    __syncthreads();
    // 3. per batch vector: stage f, zero the tile, coloured conflict-free accumulation, flush
    for (int b = 0; b < g.B; ++b) {
      for (int t = threadIdx.x; t < sp.z; t += blockDim.x) {
        const int j = jv[t];
        if (j >= 0) fv[t] = f[(long long)b * g.M + j];
      }
      for (int r = threadIdx.x; r < g.region_cells; r += blockDim.x) {
        acc[r].x = (T)0;
        acc[r].y = (T)0;
      }
      __syncthreads();
      for (int color = 0; color < (1 << D); ++color) {
        int cnt[MAX_D], nu = 1;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int par = (color >> (D - 1 - d)) & 1;
          cnt[d] = (NS[d] - par + 1) / 2;
          nu *= cnt[d];
        }
        for (int u = worker; u < nu; u += nworkers) {
          int st = 0, rem = u, ud[MAX_D];
#pragma unroll
          for (int d = D - 1; d >= 0; --d) {
            ud[d] = rem % cnt[d];
            rem /= cnt[d];
          }
#pragma unroll
          for (int d = 0; d < D; ++d) st = st * NS[d] + 2 * ud[d] + ((color >> (D - 1 - d)) & 1);
          const int q1 = stoff[st + 1];
          for (int q = stoff[st]; q < q1; ++q) {
            const int t = order[q];
            const C v = fv[t];
            int base = 0;
#pragma unroll
            for (int d = 0; d < D; ++d) base += lv[d * S + t] * strides[d];
            const T* tp = tap + t * D * TAPS;
#pragma unroll
            for (int s2 = 0; s2 < STEPS; ++s2) {
              const int c = lg + G * s2;
              if (F % G == 0 || c < F) {
                T w = (T)1;
                int a = base, rc = c;
#pragma unroll
                for (int d = D - 1; d >= 0; --d) {
                  const int l = rc % TAPS;
                  rc /= TAPS;
                  w *= tp[d * TAPS + l];
                  a += l * strides[d];
                }
                C x = acc[a];
                x.x = fma(w, v.x, x.x);
                x.y = fma(w, v.y, x.y);
                acc[a] = x;
              }
            }
            __syncwarp(gmask);
          }
        }
        __syncthreads();
      }
      C* dst = grid + (long long)b * g.grid_cells;
      for_region<D>(g, tc, [&](int r, long long o) {
        const C x = acc[r];
        if (x.x != (T)0 || x.y != (T)0) red_add<T>(dst + o, x);
      });
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------ direct (unblocked)
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(THREADS) interp_direct_kernel(Geom g, WinPoly<T> wp,
                                                                const typename cplx<T>::type* __restrict__ grid,
                                                                const T* __restrict__ ks, const int* __restrict__ perm,
                                                                int nb, int ne, typename cplx<T>::type* __restrict__ f) {
  using C = typename cplx<T>::type;
  for (int i = nb + blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += gridDim.x * blockDim.x) {
    int st[D];
    T w[D][2 * M];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double frac;
      const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
      st[d] = pos_mod(c - M + 1 - (g.Nt[d] >> 1), g.Nt[d]);
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w[d]);
    }
    const int j = perm[i];
    for (int b = 0; b < g.B; ++b) {
      const C* src = grid + (long long)b * g.grid_cells;
      C acc;
      acc.x = (T)0;
      acc.y = (T)0;
      if (D == 1) {
#pragma unroll
        for (int l = 0; l < 2 * M; ++l) {
          const C v = __ldg(src + wrap_up(st[0] + l, g.Nt[0]));
          acc.x = fma(w[0][l], v.x, acc.x);
          acc.y = fma(w[0][l], v.y, acc.y);
        }
      } else if (D == 2) {
#pragma unroll
        for (int l0 = 0; l0 < 2 * M; ++l0) {
          const C* row = src + (long long)wrap_up(st[0] + l0, g.Nt[0]) * g.Nt[1];
          C s;
          s.x = (T)0;
          s.y = (T)0;
#pragma unroll
          for (int l1 = 0; l1 < 2 * M; ++l1) {
            const C v = __ldg(row + wrap_up(st[1] + l1, g.Nt[1]));
            s.x = fma(w[1][l1], v.x, s.x);
            s.y = fma(w[1][l1], v.y, s.y);
          }
          acc.x = fma(w[0][l0], s.x, acc.x);
          acc.y = fma(w[0][l0], s.y, acc.y);
        }
      } else {
        constexpr int U0 = (2 * M <= 8) ? 2 * M : 1;
#pragma unroll U0
        for (int l0 = 0; l0 < 2 * M; ++l0) {
          C s1;
          s1.x = (T)0;
          s1.y = (T)0;
#pragma unroll
          for (int l1 = 0; l1 < 2 * M; ++l1) {
            const C* row = src + ((long long)wrap_up(st[0] + l0, g.Nt[0]) * g.Nt[1] + wrap_up(st[1] + l1, g.Nt[1])) * g.Nt[2];
            C s;
            s.x = (T)0;
            s.y = (T)0;
#pragma unroll
            for (int l2 = 0; l2 < 2 * M; ++l2) {
              const C v = __ldg(row + wrap_up(st[2] + l2, g.Nt[2]));
              s.x = fma(w[2][l2], v.x, s.x);
              s.y = fma(w[2][l2], v.y, s.y);
            }
            s1.x = fma(w[1][l1], s.x, s1.x);
            s1.y = fma(w[1][l1], s.y, s1.y);
          }
          acc.x = fma(w[0][l0], s1.x, acc.x);
          acc.y = fma(w[0][l0], s1.y, acc.y);
        }
      }
      f[(long long)b * g.M + j] = acc;
    }
  }
}

template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(THREADS) spread_direct_kernel(Geom g, WinPoly<T> wp,
                                                                const typename cplx<T>::type* __restrict__ f,
                                                                const T* __restrict__ ks, const int* __restrict__ perm,
                                                                int nb, int ne, typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  for (int i = nb + blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += gridDim.x * blockDim.x) {
    int st[D];
    T w[D][2 * M];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double frac;
      const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
      st[d] = pos_mod(c - M + 1 - (g.Nt[d] >> 1), g.Nt[d]);
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w[d]);
    }
    const int j = perm[i];
    for (int b = 0; b < g.B; ++b) {
      C* dst = grid + (long long)b * g.grid_cells;
      const C v = f[(long long)b * g.M + j];
      if (D == 1) {
#pragma unroll
        for (int l = 0; l < 2 * M; ++l) {
          C c;
          c.x = w[0][l] * v.x;
          c.y = w[0][l] * v.y;
          red_add<T>(dst + wrap_up(st[0] + l, g.Nt[0]), c);
        }
      } else if (D == 2) {
#pragma unroll
        for (int l0 = 0; l0 < 2 * M; ++l0) {
          C* row = dst + (long long)wrap_up(st[0] + l0, g.Nt[0]) * g.Nt[1];
          const T a = w[0][l0] * v.x, b2 = w[0][l0] * v.y;
#pragma unroll
          for (int l1 = 0; l1 < 2 * M; ++l1) {
            C c;
            c.x = w[1][l1] * a;
            c.y = w[1][l1] * b2;
            red_add<T>(row + wrap_up(st[1] + l1, g.Nt[1]), c);
          }
        }
      } else {
        constexpr int U0 = (2 * M <= 8) ? 2 * M : 1;
#pragma unroll U0
        for (int l0 = 0; l0 < 2 * M; ++l0) {
          const T a0 = w[0][l0] * v.x, b0 = w[0][l0] * v.y;
#pragma unroll
          for (int l1 = 0; l1 < 2 * M; ++l1) {
            C* row = dst + ((long long)wrap_up(st[0] + l0, g.Nt[0]) * g.Nt[1] + wrap_up(st[1] + l1, g.Nt[1])) * g.Nt[2];
            const T a = w[1][l1] * a0, b2 = w[1][l1] * b0;
#pragma unroll
            for (int l2 = 0; l2 < 2 * M; ++l2) {
              C c;
              c.x = w[2][l2] * a;
              c.y = w[2][l2] * b2;
              red_add<T>(row + wrap_up(st[2] + l2, g.Nt[2]), c);
            }
          }
        }
      }
    }
  }
}

}  // namespace nfftb
