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

// Padded tap count for the bank-rotated inner loop (C128: 16-byte cells, 8 per
// 128-byte shared-memory row of banks).
template <typename T, int M>
struct RotCfg {
  static constexpr bool ON = sizeof(T) == 8;
  static constexpr int TP = ON ? ((2 * M <= 8) ? 8 : 16) : 2 * M;
};

// w_out[k] = w[(k + rot) mod TP] (zero-padded beyond 2m) with a log2(TP)-stage
// select network: no dynamic register indexing.
template <typename T, int M, int TP>
__device__ __forceinline__ void rotate_taps(const T (&w)[2 * M], int rot, T (&out)[TP]) {
#pragma unroll
  for (int k = 0; k < TP; ++k) out[k] = k < 2 * M ? w[k] : (T)0;
#pragma unroll
  for (int b = 1; b < TP; b <<= 1) {
    const bool on = (rot & b) != 0;
    T tmp[TP];
#pragma unroll
    for (int k = 0; k < TP; ++k) tmp[k] = out[(k + b) % TP];
#pragma unroll
    for (int k = 0; k < TP; ++k) out[k] = on ? tmp[k] : out[k];
  }
}

// Contiguous sum over the last dimension: sum_l w[l] row[l]. With RotCfg::ON
// lane L reads element (k + rot) mod TP at step k, rot = (L - loc) mod TP, so
// the 8 lanes of each LDS.128 phase touch 8 distinct bank quads whatever the
// node positions (requires the region row pitch to be a multiple of 8 cells
// and TP - 2m readable padding cells, both provided by the plan geometry).
template <typename T, int M>
__device__ __forceinline__ typename cplx<T>::type row_sum(const typename cplx<T>::type* row, const T (&wr)[RotCfg<T, M>::TP],
                                                          const T (&w)[2 * M], int rot) {
  using C = typename cplx<T>::type;
  C s;
  s.x = (T)0;
  s.y = (T)0;
  if constexpr (RotCfg<T, M>::ON) {
    constexpr int TP = RotCfg<T, M>::TP;
#pragma unroll
    for (int k = 0; k < TP; ++k) {
      const C v = row[(k + rot) & (TP - 1)];
      s.x = fma(wr[k], v.x, s.x);
      s.y = fma(wr[k], v.y, s.y);
    }
  } else {
#pragma unroll
    for (int l = 0; l < 2 * M; ++l) {
      const C v = row[l];
      s.x = fma(w[l], v.x, s.x);
      s.y = fma(w[l], v.y, s.y);
    }
  }
  return s;
}

// (2m)^D tensor-product sum over a region held in shared memory (eq.
// InnerTensorStructure): innermost dimension contiguous.
template <typename T, int D, int M>
__device__ __forceinline__ typename cplx<T>::type gather_tile(const Geom& g, const typename cplx<T>::type* tile,
                                                              const int (&loc)[D], const T (&w)[D][2 * M]) {
  using C = typename cplx<T>::type;
  constexpr int TP = RotCfg<T, M>::TP;
  T wr[TP];
  const int rot = ((int)(threadIdx.x & 31) - loc[D - 1]) & (TP - 1);
  if constexpr (RotCfg<T, M>::ON) rotate_taps<T, M, TP>(w[D - 1], rot, wr);
  C acc;
  acc.x = (T)0;
  acc.y = (T)0;
  if (D == 1) {
    acc = row_sum<T, M>(tile + loc[0], wr, w[D - 1], rot);
  } else if (D == 2) {
    const int L1 = g.L[1];
#pragma unroll
    for (int l0 = 0; l0 < 2 * M; ++l0) {
      const C s = row_sum<T, M>(tile + (loc[0] + l0) * L1 + loc[1], wr, w[D - 1], rot);
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
        const C s = row_sum<T, M>(tile + ((loc[0] + l0) * L1 + loc[1] + l1) * L2 + loc[2], wr, w[D - 1], rot);
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
// Asynchronous global->shared copy of one grid cell (LDGSTS): the tile region
// streams into shared memory while the threads load their nodes and evaluate
// the taps, so the two memory latencies overlap.
template <typename T>
__device__ __forceinline__ void cp_async_cell(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

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
    for (int b = 0; b < g.B; ++b) {
      const C* src = grid + (long long)b * g.grid_cells;
      __syncthreads();  // previous users of the tile are done
      for_region<D>(g, tc, [&](int r, long long off) { cp_async_cell<T>(&tile[r], src + off); });
      if (b == 0 && has) {
        const int i = sp.y + threadIdx.x;
        j = perm[i];
        has = node_setup<T, D, M, DEG>(g, wp, ks, i, tc, loc, w);
      }
      cp_async_wait_all();
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

// ------------------------------------------------------------ adjoint, owner-computes
// One CTA per tile writes exactly the tile's Q^D grid cells, once, with plain
// coalesced stores: no zero pass, no global atomics. The
// CTA gathers every node of its 3^D neighbour tiles whose footprint reaches
// into the tile (Q_d | Ntilde_d, P_d >= 3, Q_d >= 2m), buckets them by 2m-wide
// sub-tiles of an extended sub-tile grid (one ring outside the tile), and
// accumulates the clipped footprints with the coloured lanes-own-cells scheme
// of spread_loc_kernel. Empty tiles just write zeros.
template <typename T, int D, int M>
struct OwnCfg {
  static constexpr int THR = D == 1 ? 256 : 128;
  static constexpr int LISTCAP = 2048;
};

template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(OwnCfg<T, D, M>::THR) spread_own_kernel(
    Geom g, WinPoly<T> wp, const typename cplx<T>::type* __restrict__ f, const T* __restrict__ ks,
    const int* __restrict__ perm, const int* __restrict__ offsets, int nb, int ne,
    typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  using L = LocCfg<T, D, M>;
  constexpr int TAPS = L::TAPS, F = L::F, G = L::G, STEPS = L::STEPS;
  constexpr int THR = OwnCfg<T, D, M>::THR, LISTCAP = OwnCfg<T, D, M>::LISTCAP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int tile_cells = 1, NSX[MAX_D], nst = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    tile_cells *= g.Q[d];
    NSX[d] = (g.Q[d] + TAPS - 1) / TAPS + 2;  // extended sub-tile grid
    nst *= NSX[d];
  }
  C* acc = reinterpret_cast<C*>(smem_raw);
  T* tap = reinterpret_cast<T*>(acc + tile_cells);  // [THR][D][TAPS]
  size_t off = ((size_t)tile_cells * sizeof(C) + (size_t)THR * D * TAPS * sizeof(T) + 15) & ~(size_t)15;
  C* fv = reinterpret_cast<C*>(smem_raw + off);
  int* jv = reinterpret_cast<int*>(fv + THR);
  int* order = jv + THR;
  int* sv = order + THR;        // [D][THR] footprint start relative to the tile origin
  int* list = sv + D * THR;     // [LISTCAP]
  int* stoff = list + LISTCAP;  // [nst + 1]
  int* stcur = stoff + nst + 1; // [nst]
  int* counters = stcur + nst;  // [0] list length

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lg = lane % G;
  const bool worker_lane = lane < L::WPW * G;
  const int worker = worker_lane ? warp * L::WPW + lane / G : 1 << 30;
  const int nworkers = (THR >> 5) * L::WPW;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane / G * G));
  int strides[MAX_D];
  strides[D - 1] = 1;
#pragma unroll
  for (int d = D - 2; d >= 0; --d) strides[d] = strides[d + 1] * g.Q[d + 1];
  int ntiles = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) ntiles *= g.P[d];

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int p[MAX_D];
    {
      int rem = tile;
#pragma unroll
      for (int d = D - 1; d >= 0; --d) {
        p[d] = rem % g.P[d];
        rem /= g.P[d];
      }
    }
    for (int b = 0; b < g.B; ++b) {
      for (int r = threadIdx.x; r < tile_cells; r += THR) {
        acc[r].x = (T)0;
        acc[r].y = (T)0;
      }
      // walk the 3^D neighbour tiles; relevant nodes are compacted into `list`
      // and consumed in chunks of THR nodes
      int nbhd = 1;
#pragma unroll
      for (int d = 0; d < D; ++d) nbhd *= 3;
      for (int nbi = 0; nbi < nbhd; ++nbi) {
        int q = 0, dl[MAX_D], qo[MAX_D];  // qo: cell origin of the (wrapped) neighbour tile minus dl*Q
        {
          int rem = nbi;
#pragma unroll
          for (int d = D - 1; d >= 0; --d) {
            dl[d] = rem % 3 - 1;
            rem /= 3;
          }
#pragma unroll
          for (int d = 0; d < D; ++d) {
            int qd = p[d] + dl[d];
            qd = qd < 0 ? qd + g.P[d] : (qd >= g.P[d] ? qd - g.P[d] : qd);
            q = q * g.P[d] + qd;
            qo[d] = qd * g.Q[d] - dl[d] * g.Q[d];
          }
        }
        const int i0 = max(offsets[q], nb), i1 = min(offsets[q + 1], ne);
        for (int cbase = i0; cbase < i1; cbase += LISTCAP) {
          const int cend = min(i1, cbase + LISTCAP);
          if (threadIdx.x == 0) counters[0] = 0;
          __syncthreads();
          for (int i = cbase + threadIdx.x; i < cend; i += THR) {
            bool rel = true;
#pragma unroll
            for (int d = 0; d < D; ++d) {
              double frac;
              const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
              const int s0 = c - qo[d] - M + 1;  // footprint start relative to this tile (unwrapped)
              rel = rel && s0 < g.Q[d] && s0 + TAPS > 0;
            }
            if (rel) list[atomicAdd(&counters[0], 1)] = i;
          }
          __syncthreads();
          const int nlist = counters[0];
          for (int lb = 0; lb < nlist; lb += THR) {
            const int nchunk = min(THR, nlist - lb);
            for (int i = threadIdx.x; i <= nst; i += THR) stoff[i] = 0;
            __syncthreads();
            int st = 0;
            if (threadIdx.x < nchunk) {
              const int t = threadIdx.x;
              const int i = list[lb + t];
              jv[t] = perm[i];
#pragma unroll
              for (int d = 0; d < D; ++d) {
                double frac;
                const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
                const int rel = c - qo[d];
                sv[d * THR + t] = rel - M + 1;
                st = st * NSX[d] + (rel >= 0 ? rel / TAPS + 1 : 0);
                T w[TAPS];
                window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w);
#pragma unroll
                for (int l = 0; l < TAPS; ++l) tap[(t * D + d) * TAPS + l] = w[l];
              }
              fv[t] = f[(long long)b * g.M + jv[t]];
              atomicAdd(&stoff[st + 1], 1);
            }
            __syncthreads();
            if (threadIdx.x == 0)
              for (int k = 1; k <= nst; ++k) stoff[k] += stoff[k - 1];
            __syncthreads();
            for (int k = threadIdx.x; k < nst; k += THR) stcur[k] = stoff[k];
            __syncthreads();
            if (threadIdx.x < nchunk) order[atomicAdd(&stcur[st], 1)] = threadIdx.x;
            __syncthreads();
            for (int color = 0; color < (1 << D); ++color) {
              int cnt[MAX_D], nu = 1;
#pragma unroll
              for (int d = 0; d < D; ++d) {
                const int par = (color >> (D - 1 - d)) & 1;
                cnt[d] = (NSX[d] - par + 1) / 2;
                nu *= cnt[d];
              }
              for (int u = worker; u < nu; u += nworkers) {
                int sti = 0, rem = u, ud[MAX_D];
#pragma unroll
                for (int d = D - 1; d >= 0; --d) {
                  ud[d] = rem % cnt[d];
                  rem /= cnt[d];
                }
#pragma unroll
                for (int d = 0; d < D; ++d) sti = sti * NSX[d] + 2 * ud[d] + ((color >> (D - 1 - d)) & 1);
                const int q1 = stoff[sti + 1];
                for (int qq = stoff[sti]; qq < q1; ++qq) {
                  const int t = order[qq];
                  const C v = fv[t];
                  int s0[MAX_D];
#pragma unroll
                  for (int d = 0; d < D; ++d) s0[d] = sv[d * THR + t];
                  const T* tp = tap + t * D * TAPS;
#pragma unroll
                  for (int s2 = 0; s2 < STEPS; ++s2) {
                    const int c = lg + G * s2;
                    if (F % G == 0 || c < F) {
                      T w = (T)1;
                      int a = 0, rc = c;
                      bool in = true;
#pragma unroll
                      for (int d = D - 1; d >= 0; --d) {
                        const int l = rc % TAPS;
                        rc /= TAPS;
                        const int x = s0[d] + l;
                        in = in && x >= 0 && x < g.Q[d];
                        w *= tp[d * TAPS + l];
                        a += x * strides[d];
                      }
                      if (in) {
                        C x = acc[a];
                        x.x = fma(w, v.x, x.x);
                        x.y = fma(w, v.y, x.y);
                        acc[a] = x;
                      }
                    }
                  }
                  __syncwarp(gmask);
                }
              }
              __syncthreads();
            }
          }
        }
      }
      // write the tile: rows along the contiguous last dimension
      C* dst = grid + (long long)b * g.grid_cells;
      const int Ql = g.Q[D - 1];
      const int rows = tile_cells / Ql;
      for (int r = threadIdx.x / 32; r < rows; r += THR / 32) {
        long long rowoff = 0;
        int rr = r;
        int idx[MAX_D];
#pragma unroll
        for (int d = D - 2; d >= 0; --d) {
          idx[d] = rr % g.Q[d];
          rr /= g.Q[d];
        }
#pragma unroll
        for (int d = 0; d < D - 1; ++d) {
          int sd = p[d] * g.Q[d] + idx[d] + (g.Nt[d] >> 1);
          if (sd >= g.Nt[d]) sd -= g.Nt[d];
          rowoff = rowoff * g.Nt[d] + sd;
        }
        rowoff *= g.Nt[D - 1];
        const int base = p[D - 1] * Ql + (g.Nt[D - 1] >> 1);
        for (int x = lane; x < Ql; x += 32) {
          int sx = base + x;
          if (sx >= g.Nt[D - 1]) sx -= g.Nt[D - 1];
          dst[rowoff + sx] = acc[r * Ql + x];
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------ adjoint, cell-sorted warp chunks
// Thread-per-node spreading without shared-memory atomics:
//  1. the subproblem's nodes are counting-sorted by their local cell (row-major
//     in the tile) in shared memory;
//  2. sorted node s belongs to lane s%32 of warp-chunk s/32. Lanes of one chunk
//     add the same tap offset in the same instruction, so they can only collide
//     when two nodes share a cell; those are serialised by their rank among the
//     equal-cell lanes (__match_any_sync). Across instructions, the lanes' plain
//     read-modify-writes are ordered by `volatile` shared accesses of a
//     converged warp;
//  3. chunks whose footprint row ranges (dimension 0) overlap never run at the
//     same time: chunk k runs in phase k mod K, K = 1 + the most later chunks
//     any chunk overlaps with (computed per subproblem, so dense clusters just
//     serialise more);
//  4. the tile region is flushed with global reductions (Alg. 4's merge).
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(THREADS) spread_sorted_kernel(Geom g, WinPoly<T> wp,
                                                                const typename cplx<T>::type* __restrict__ f,
                                                                const T* __restrict__ ks, const int* __restrict__ perm,
                                                                const int4* __restrict__ subs,
                                                                const int* __restrict__ nsub_ptr,
                                                                typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int tile_cells = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) tile_cells *= g.Q[d];
  C* tile = reinterpret_cast<C*>(smem_raw);
  int* hist = reinterpret_cast<int*>(tile + g.region_cells);  // [tile_cells + 1]
  int* order = hist + tile_cells + 1;                         // [THREADS] sorted slot -> subproblem index
  int* rows = order + THREADS;                                // [2 * 8] first/last row of every chunk
  int* kshared = rows + 16;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int rstr[MAX_D];  // region strides
  rstr[D - 1] = 1;
#pragma unroll
  for (int d = D - 2; d >= 0; --d) rstr[d] = rstr[d + 1] * g.L[d + 1];

  const int nsub = *nsub_ptr;
  for (int s = blockIdx.x; s < nsub; s += gridDim.x) {
    const int4 sp = subs[s];
    const TileCoords tc = tile_coords<D, M>(g, sp.x);
    for (int i = threadIdx.x; i <= tile_cells; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) kshared[0] = 1;
    __syncthreads();
    // 1. local cell of every node, histogram
    int lc = -1;
    if (threadIdx.x < sp.z) {
      const int i = sp.y + threadIdx.x;
      lc = 0;
      bool ok = true;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double frac;
        const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
        const int loc = c - tc.p[d] * g.Q[d];
        ok = ok && (unsigned)loc < (unsigned)g.Q[d];
        lc = lc * g.Q[d] + (ok ? loc : 0);
      }
      if (!ok) lc = -1;
      else atomicAdd(&hist[lc + 1], 1);
    }
    __syncthreads();
    // exclusive scan of the cell histogram (tile_cells + 1 entries)
    {
      __shared__ int ws[32];
      const int per = (tile_cells + 1 + blockDim.x - 1) / blockDim.x;
      const int lo = threadIdx.x * per, hi = min(tile_cells + 1, lo + per);
      int sum = 0;
      for (int k = lo; k < hi; ++k) sum += hist[k];
      int total;
      int run = block_exclusive_scan(sum, ws, total);
      for (int k = lo; k < hi; ++k) {
        run += hist[k];
        hist[k] = run;  // inclusive of hist[k] (hist[0] = 0): hist[lc] = start of cell lc
      }
    }
    __syncthreads();
    int nvalid = hist[tile_cells];
    if (lc >= 0) order[atomicAdd(&hist[lc], 1)] = threadIdx.x;
    __syncthreads();
    // 2. sorted slot -> node data and taps in registers
    const int slot = threadIdx.x;
    const bool has = slot < nvalid;
    int j = 0, loc[D], mycell = -1;
    T w[D][TAPS];
    if (has) {
      const int t = order[slot];
      const int i = sp.y + t;
      j = perm[i];
      mycell = 0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double frac;
        const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
        loc[d] = c - tc.p[d] * g.Q[d];
        mycell = mycell * g.Q[d] + loc[d];
        window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w[d]);
      }
    }
    // 3. chunk row ranges and the number of phases K
    const int nchunks = (nvalid + 31) / 32;
    if (has && (lane == 0 || slot == nvalid - 1 || lane == 31)) {
      if (lane == 0) rows[2 * warp] = loc[0];
      if (lane == 31 || slot == nvalid - 1) rows[2 * warp + 1] = loc[0];
    }
    __syncthreads();
    if (threadIdx.x < nchunks) {
      const int k = threadIdx.x;
      int cnt = 0;
      for (int k2 = k + 1; k2 < nchunks; ++k2) {
        if (rows[2 * k2] - rows[2 * k + 1] <= 2 * M - 1) ++cnt;  // footprint rows overlap
        else break;
      }
      atomicMax(&kshared[0], cnt + 1);
    }
    __syncthreads();
    const int K = kshared[0];
    // duplicate-cell rank inside the warp
    const unsigned peers = __match_any_sync(0xffffffffu, has ? mycell : -1 - lane);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int rounds = __reduce_max_sync(0xffffffffu, has ? rank + 1 : 0);
    int base = 0;
    if (has) {
#pragma unroll
      for (int d = 0; d < D; ++d) base += loc[d] * rstr[d];
    }
    for (int b = 0; b < g.B; ++b) {
      for (int r = threadIdx.x; r < g.region_cells; r += blockDim.x) {
        tile[r].x = (T)0;
        tile[r].y = (T)0;
      }
      C v;
      v.x = (T)0;
      v.y = (T)0;
      if (has) v = f[(long long)b * g.M + j];
      __syncthreads();
      volatile T* vt = reinterpret_cast<volatile T*>(tile);
      for (int ph = 0; ph < K; ++ph) {
        if (warp < nchunks && warp % K == ph) {
          for (int rd = 0; rd < rounds; ++rd) {
            if (has && rank == rd) {
              if (D == 1) {
#pragma unroll
                for (int l = 0; l < TAPS; ++l) {
                  const int a = 2 * (base + l);
                  vt[a] = fma(w[0][l], v.x, vt[a]);
                  vt[a + 1] = fma(w[0][l], v.y, vt[a + 1]);
                }
              } else if (D == 2) {
#pragma unroll
                for (int l0 = 0; l0 < TAPS; ++l0) {
                  const T ax = w[0][l0] * v.x, ay = w[0][l0] * v.y;
#pragma unroll
                  for (int l1 = 0; l1 < TAPS; ++l1) {
                    const int a = 2 * (base + l0 * rstr[0] + l1);
                    vt[a] = fma(w[1][l1], ax, vt[a]);
                    vt[a + 1] = fma(w[1][l1], ay, vt[a + 1]);
                  }
                }
              } else {
                constexpr int U0 = (2 * M <= 8) ? 2 * M : 1;
#pragma unroll U0
                for (int l0 = 0; l0 < TAPS; ++l0) {
                  const T ax0 = w[0][l0] * v.x, ay0 = w[0][l0] * v.y;
#pragma unroll
                  for (int l1 = 0; l1 < TAPS; ++l1) {
                    const T ax = w[1][l1] * ax0, ay = w[1][l1] * ay0;
#pragma unroll
                    for (int l2 = 0; l2 < TAPS; ++l2) {
                      const int a = 2 * (base + l0 * rstr[0] + l1 * rstr[1] + l2);
                      vt[a] = fma(w[2][l2], ax, vt[a]);
                      vt[a + 1] = fma(w[2][l2], ay, vt[a + 1]);
                    }
                  }
                }
              }
            }
            __syncwarp();
          }
        }
        __syncthreads();
      }
      C* dst = grid + (long long)b * g.grid_cells;
      for_region<D>(g, tc, [&](int r, long long o) {
        const C x = tile[r];
        if (x.x != (T)0 || x.y != (T)0) red_add<T>(dst + o, x);
      });
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------ adjoint, cell gather (default for D <= 2)
// Spreading computed as a gather: the subproblem's nodes
// are counting-sorted by their local cell in shared memory (taps evaluated once
// per node, even/odd polynomial, stored with the node); then every region cell
// x is produced by ONE thread as sum_j f_j psi~(k_j - x/Nt) over the nodes whose
// cells lie in [x - m, x + m - 1] per dimension — contiguous ranges of the
// cell-sorted list (one range per row in 2D). No shared-memory read-modify-
// write, no atomics inside the CTA; each region cell is reduced into the grid
// once (coalesced global reduction, Alg. 4's merge).
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(THREADS) spread_gather_kernel(Geom g, WinPoly<T> wp,
                                                                const typename cplx<T>::type* __restrict__ f,
                                                                const T* __restrict__ ks, const int* __restrict__ perm,
                                                                const int4* __restrict__ subs,
                                                                const int* __restrict__ nsub_ptr, int S,
                                                                typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int tile_cells = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) tile_cells *= g.Q[d];
  T* tap = reinterpret_cast<T*>(smem_raw);  // [S][D][TAPS]
  size_t off = ((size_t)S * D * TAPS * sizeof(T) + 15) & ~(size_t)15;
  C* fv = reinterpret_cast<C*>(smem_raw + off);
  int* cl = reinterpret_cast<int*>(fv + S);  // [D][S] local cell of the slot
  int* js = cl + D * S;                      // [S]
  int* start = js + S;                       // [tile_cells + 1]
  int* cursor = start + tile_cells + 1;      // [tile_cells + 1]
  __shared__ int ws[32];

  const int nsub = *nsub_ptr;
  for (int sidx = blockIdx.x; sidx < nsub; sidx += gridDim.x) {
    const int4 sp = subs[sidx];
    const TileCoords tc = tile_coords<D, M>(g, sp.x);
    for (int i = threadIdx.x; i <= tile_cells; i += blockDim.x) start[i] = 0;
    // 1. node t of the subproblem -> thread t (looping for S > blockDim): cell, taps, j and f of batch 0
    //    stay in registers; the histogram counts the local cells
    constexpr int PER = 1;  // S <= THREADS (plan invariant)
    int lcs[PER], jj[PER];
    int locs[PER][D];
    T w[PER][D][TAPS];
    C f0[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int t = threadIdx.x + u * blockDim.x;
      lcs[u] = -1;
      if (t < sp.z) {
        const int i = sp.y + t;
        bool ok = true;
        int lc = 0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          double frac;
          const int c = node_cell((double)ks[(long long)d * g.M + i], g.Ntd[d], g.Nt[d], frac);
          locs[u][d] = c - tc.p[d] * g.Q[d];
          ok = ok && (unsigned)locs[u][d] < (unsigned)g.Q[d];
          lc = lc * g.Q[d] + (ok ? locs[u][d] : 0);
          window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w[u][d]);
        }
        if (ok) {
          lcs[u] = lc;
          jj[u] = perm[i];
          f0[u] = f[jj[u]];
        }
      }
    }
    __syncthreads();  // start[] zeroed
#pragma unroll
    for (int u = 0; u < PER; ++u)
      if (lcs[u] >= 0) atomicAdd(&start[lcs[u] + 1], 1);
    __syncthreads();
    {
      const int per = (tile_cells + 1 + blockDim.x - 1) / blockDim.x;
      const int lo = threadIdx.x * per, hi = min(tile_cells + 1, lo + per);
      int sum = 0;
      for (int k = lo; k < hi; ++k) sum += start[k];
      int total;
      int run = block_exclusive_scan(sum, ws, total);
      for (int k = lo; k < hi; ++k) {
        run += start[k];
        start[k] = run;  // start[c] = first slot of local cell c; start[tile_cells] = count
        cursor[k] = run;
      }
    }
    __syncthreads();
    // 2. sorted slots
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      if (lcs[u] < 0) continue;
      const int slot = atomicAdd(&cursor[lcs[u]], 1);
      js[slot] = jj[u];
      fv[slot] = f0[u];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        cl[d * S + slot] = locs[u][d];
#pragma unroll
        for (int l = 0; l < TAPS; ++l) tap[(slot * D + d) * TAPS + l] = w[u][d][l];
      }
    }
    __syncthreads();
    const int nvalid = start[tile_cells];
    // 3. per batch vector: every region cell gathered by one thread, reduced into the grid
    for (int b = 0; b < g.B; ++b) {
      if (b > 0) {
        __syncthreads();
        for (int q = threadIdx.x; q < nvalid; q += blockDim.x) fv[q] = f[(long long)b * g.M + js[q]];
        __syncthreads();
      }
      C* dst = grid + (long long)b * g.grid_cells;
      for_region<D>(g, tc, [&](int r, long long o) {
        C acc;
        acc.x = (T)0;
        acc.y = (T)0;
        if (D == 1) {
          const int x = r - (M - 1);  // tile-relative cell of region index r
          const int c_lo = max(0, x - M), c_hi = min(g.Q[0] - 1, x + M - 1);
          if (c_lo <= c_hi) {
            const int q1 = start[c_hi + 1];
            for (int q = start[c_lo]; q < q1; ++q) {
              const T wt = tap[q * TAPS + (x - cl[q] + M - 1)];
              const C v = fv[q];
              acc.x = fma(wt, v.x, acc.x);
              acc.y = fma(wt, v.y, acc.y);
            }
          }
        } else {
          const int L1 = g.L[1];
          const int x0 = r / L1 - (M - 1), x1 = r % L1 - (M - 1);
          const int r_lo = max(0, x0 - M), r_hi = min(g.Q[0] - 1, x0 + M - 1);
          const int c_lo = max(0, x1 - M), c_hi = min(g.Q[1] - 1, x1 + M - 1);
          if (c_lo <= c_hi) {
            for (int c0 = r_lo; c0 <= r_hi; ++c0) {
              const int q1 = start[c0 * g.Q[1] + c_hi + 1];
              const int l0 = x0 - c0 + M - 1;
              for (int q = start[c0 * g.Q[1] + c_lo]; q < q1; ++q) {
                const T wt = tap[(q * 2) * TAPS + l0] * tap[(q * 2 + 1) * TAPS + (x1 - cl[S + q] + M - 1)];
                const C v = fv[q];
                acc.x = fma(wt, v.x, acc.x);
                acc.y = fma(wt, v.y, acc.y);
              }
            }
          }
        }
        if (acc.x != (T)0 || acc.y != (T)0) red_add<T>(dst + o, acc);
      });
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ direct (unblocked)
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(THREADS) interp_direct_kernel(Geom g, WinPolyN<T, D, M> wp,
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
__global__ void __launch_bounds__(THREADS) spread_direct_kernel(Geom g, WinPolyN<T, D, M> wp,
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
