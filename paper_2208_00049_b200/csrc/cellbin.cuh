// cellbin.cuh — node binning + stable sort by CELL.
//
// The paper partitions the oversampled grid into blocks and sorts the nodes
// by block. On the GPU the hot path sorts at the finest
// granularity, ONE CELL per block (the oracle's binning with tile = 1 cell,
// oracle/binning.py), so that every resampling kernel finds the nodes of any
// cell range as contiguous ranges of one table, and coarse work tiles are
// defined on the fly by the kernels (no per-kernel sorting):
//
//   key(j)     = row-major index of the node's cell (c_0, ..., c_{D-1}),
//                c_d = (floor(Ntilde_d k_jd) + Ntilde_d/2) mod Ntilde_d   (reading R10)
//   cstart[c]  = number of nodes with key < c   (cstart[prod Ntilde] = M)
//   order      = key ascending, node index ascending (stable; reading R12)
//
// Four kernels (each B200 graph launch costs ~1 us; every kernel has at most
// one dependent global-memory level before its stores):
//  cl_count  per node: key, slot = atomicAdd(count[key], 1) (arbitrary order
//            inside a cell; cl_fix makes it stable). Resets the scan state.
//  cl_scan   exclusive scan count[] -> cstart[] in ONE pass (decoupled
//            look-back over 4096-cell tiles, dynamic tile ids), re-zeroes
//            count[] for the next precompute (no memset).
//  cl_place  per node: pos = cstart[key] + slot; sorted SoA coordinates
//            kc[d][pos], node index jc[pos]; cells with > CL_SMALL nodes are
//            listed by their slot-0 node (rare: the centre of a radial trajectory).
//  cl_fix    node index order inside every cell with >= 2 nodes: thread per
//            cell (a coalesced pass over cstart) up to CL_SMALL nodes, ranks in
//            registers; listed denser cells: one CTA, ranks by counting.
#pragma once

#include "common.cuh"

namespace nfftb {

constexpr int CL_THREADS = 256;
constexpr int CL_SCAN_THREADS = 512;
constexpr int CL_SCAN_PER = 8;                                 // cells per thread in the scan
constexpr int CL_SCAN_TILE = CL_SCAN_THREADS * CL_SCAN_PER;   // 4096 cells per scan tile
constexpr int CL_SMALL = 8;    // cells with 2..CL_SMALL nodes: one thread each in cl_fix
constexpr int CL_BIGREG = 8;   // big cells: nodes per thread held in registers (n <= 256 * 8)

// scan tile status: (flag << 32) | value; flag 1 = tile aggregate, 2 = inclusive prefix
constexpr unsigned long long CL_AGG = 1ull << 32, CL_PRE = 2ull << 32;

template <typename R, int D>
__device__ __forceinline__ int cell_key(const R* __restrict__ nodes, const Geom& g, int j, R (&k)[MAX_D], bool& bad) {
  int key = 0;
  bad = false;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    k[d] = nodes[(long long)j * D + d];
    const double kd = (double)k[d];
    if (!isfinite(kd)) {
      bad = true;
      continue;
    }
    double frac;
    key = key * g.Nt[d] + node_cell(kd, g.Ntd[d], g.Nt[d], frac);
  }
  return bad ? 0 : key;
}

template <typename R, int D>
__global__ void __launch_bounds__(CL_THREADS) cl_count_kernel(const R* __restrict__ nodes, Geom g,
                                                              int* __restrict__ count, int* __restrict__ slot,
                                                              int* __restrict__ err,
                                                              unsigned long long* __restrict__ status, int ntiles,
                                                              int* __restrict__ ctr) {
  const int t0 = blockIdx.x * CL_THREADS + threadIdx.x, stride = gridDim.x * CL_THREADS;
  for (int j = t0; j < ntiles; j += stride) status[j] = 0ull;  // scan state (read only by cl_scan)
  if (t0 < 4) ctr[t0] = 0;  // [0] scan ticket, [2] fix-list length
  for (int j = t0; j < g.M; j += stride) {  // grid-stride: the launch may use fewer threads than nodes
    R k[MAX_D];
    bool bad;
    const int c = cell_key<R, D>(nodes, g, j, k, bad);
    if (bad) atomicOr(err, 1);
    slot[j] = atomicAdd(count + c, 1);
  }
}

// One-pass exclusive scan with decoupled look-back. cstart[n] = total.
__global__ void __launch_bounds__(CL_SCAN_THREADS) cl_scan_kernel(int* __restrict__ count, int n,
                                                                  unsigned long long* __restrict__ status,
                                                                  int* __restrict__ ctr, int* __restrict__ cstart) {
  __shared__ int ws[32];
  __shared__ int tile_s, excl_s;
  if (threadIdx.x == 0) tile_s = atomicAdd(ctr, 1);  // dynamic tile id: predecessors are already running
  __syncthreads();
  const int tile = tile_s;
  const int base = tile * CL_SCAN_TILE + threadIdx.x * CL_SCAN_PER;
  int v[CL_SCAN_PER];
  int loc = 0;
  const bool full = base + CL_SCAN_PER <= n;  // 8 cells, 32-byte aligned: two 16-byte loads and stores
  if (full) {
    const int4 a = __ldcg(reinterpret_cast<const int4*>(count + base));
    const int4 b = __ldcg(reinterpret_cast<const int4*>(count + base) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    if ((a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) != 0) {  // zero for the next precompute
      reinterpret_cast<int4*>(count + base)[0] = make_int4(0, 0, 0, 0);
      reinterpret_cast<int4*>(count + base)[1] = make_int4(0, 0, 0, 0);
    }
  } else {
#pragma unroll
    for (int q = 0; q < CL_SCAN_PER; ++q) {
      v[q] = base + q < n ? __ldcg(count + base + q) : 0;
      if (v[q] != 0) count[base + q] = 0;
    }
  }
#pragma unroll
  for (int q = 0; q < CL_SCAN_PER; ++q) loc += v[q];
  int agg;
  const int off = block_exclusive_scan(loc, ws, agg);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0) {
      if (tile == 0) {
        excl_s = 0;
        atomicExch(status, CL_PRE | (unsigned)agg);
      } else {
        atomicExch(status + tile, CL_AGG | (unsigned)agg);
      }
    }
    if (tile > 0) {
      // warp look-back: 32 predecessors per step, stop at the nearest inclusive prefix
      int excl = 0;
      int hi = tile - 1;
      while (true) {
        const int i = hi - lane;
        unsigned long long s = 0;
        if (i >= 0) {
          do {  // (an asm volatile load: a plain or __ldcv load lets the compiler drop the spin)
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(s) : "l"(status + i) : "memory");
          } while ((s >> 32) == 0);
        } else {
          s = CL_PRE;  // before tile 0: prefix 0
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (s >> 32) == 2);
        const int first = pre ? __ffs(pre) - 1 : 32;  // nearest lane holding an inclusive prefix
        int val = lane <= first ? (int)(unsigned)(s & 0xffffffffu) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (pre) break;
        hi -= 32;
      }
      if (lane == 0) {
        excl_s = excl;
        atomicExch(status + tile, CL_PRE | (unsigned)(excl + agg));
      }
    }
  }
  __syncthreads();
  int run = excl_s + off;
  int o[CL_SCAN_PER];
#pragma unroll
  for (int q = 0; q < CL_SCAN_PER; ++q) {
    o[q] = run;
    run += v[q];
  }
  if (full) {
    reinterpret_cast<int4*>(cstart + base)[0] = make_int4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<int4*>(cstart + base)[1] = make_int4(o[4], o[5], o[6], o[7]);
  } else {
#pragma unroll
    for (int q = 0; q < CL_SCAN_PER; ++q)
      if (base + q < n) cstart[base + q] = o[q];
  }
  if (base <= n && n <= base + CL_SCAN_PER) cstart[n] = excl_s + off + loc;  // thread owning the end
}

template <typename R, int D>
__global__ void __launch_bounds__(CL_THREADS) cl_place_kernel(const R* __restrict__ nodes, Geom g,
                                                              const int* __restrict__ slot,
                                                              const int* __restrict__ cstart,
                                                              R* __restrict__ kc, int* __restrict__ jc,
                                                              int* __restrict__ ctr, int* __restrict__ fixl) {
  const int lane = threadIdx.x & 31;
  for (int j = blockIdx.x * CL_THREADS + threadIdx.x; j - lane < g.M; j += gridDim.x * CL_THREADS) {
  bool listed = false;
  int c = 0;
  if (j < g.M) {
    R k[MAX_D];
    bool bad;
    c = cell_key<R, D>(nodes, g, j, k, bad);
    const int s = slot[j];
    const int a = cstart[c], n = cstart[c + 1] - a;
    const int pos = a + s;  // arrival order inside the cell; cl_fix makes it stable
    jc[pos] = j;
#pragma unroll
    for (int d = 0; d < D; ++d) kc[(long long)d * g.M + pos] = k[d];
    listed = s == 0 && n > CL_SMALL;
  }
  const unsigned mb = __ballot_sync(0xffffffffu, listed);
  const unsigned lt = (1u << lane) - 1;
  if (mb) {
    int b0 = 0;
    if (lane == __ffs(mb) - 1) b0 = atomicAdd(ctr + 2, __popc(mb));
    b0 = __shfl_sync(0xffffffffu, b0, __ffs(mb) - 1);
    if (listed) fixl[b0 + __popc(mb & lt)] = c;
  }
  }  // nodes
}

// Stable order (node index) inside every cell with >= 2 nodes. Cells with
// <= CL_SMALL nodes: thread per cell, found by a coalesced pass over cstart
// (listing them would serialise ~M/6 appends on one counter), ranks in
// registers. Listed denser cells: CTA per cell, n <= 256 * CL_BIGREG in
// registers + shared memory, larger through scratch (sj_out / sk_out: cslot and
// d_ks, free after cl_place).
template <typename R, int D>
__global__ void __launch_bounds__(CL_THREADS) cl_fix_kernel(Geom g, const int* __restrict__ cstart,
                                                            R* __restrict__ kc, int* __restrict__ jc, int ncells,
                                                            const int* __restrict__ ctr, const int* __restrict__ big,
                                                            int* __restrict__ sj_out, R* __restrict__ sk_out) {
  __shared__ int sj[CL_THREADS * CL_BIGREG];
  const int nbig = ctr[2];
  for (int c = blockIdx.x * CL_THREADS + threadIdx.x; c < ncells; c += gridDim.x * CL_THREADS) {
    const int a = cstart[c], n = cstart[c + 1] - a;
    if (n < 2 || n > CL_SMALL) continue;
    if (n == 2) {  // the common case (~80% of the multi-node cells of a uniform set): one compare-swap
      const int j0 = jc[a], j1 = jc[a + 1];
      if (j0 > j1) {
        jc[a] = j1;
        jc[a + 1] = j0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const R k0 = kc[(long long)d * g.M + a], k1 = kc[(long long)d * g.M + a + 1];
          kc[(long long)d * g.M + a] = k1;
          kc[(long long)d * g.M + a + 1] = k0;
        }
      }
      continue;
    }
    int jv[CL_SMALL];
    R kv[CL_SMALL][D];
#pragma unroll
    for (int i = 0; i < CL_SMALL; ++i) {
      if (i < n) {
        jv[i] = jc[a + i];
#pragma unroll
        for (int d = 0; d < D; ++d) kv[i][d] = kc[(long long)d * g.M + a + i];
      }
    }
#pragma unroll
    for (int i = 0; i < CL_SMALL; ++i) {
      if (i < n) {
        int r = 0;
#pragma unroll
        for (int k = 0; k < CL_SMALL; ++k) r += (k < n && jv[k] < jv[i]);
        jc[a + r] = jv[i];
#pragma unroll
        for (int d = 0; d < D; ++d) kc[(long long)d * g.M + a + r] = kv[i][d];
      }
    }
  }
  for (int q = blockIdx.x; q < nbig; q += gridDim.x) {
    const int c = big[q];
    const int a = cstart[c], n = cstart[c + 1] - a;
    if (n <= CL_THREADS * CL_BIGREG) {
      int jv[CL_BIGREG];
      R kv[CL_BIGREG][D];
      __syncthreads();
#pragma unroll
      for (int u = 0; u < CL_BIGREG; ++u) {
        const int i = threadIdx.x + u * CL_THREADS;
        if (i < n) {
          jv[u] = jc[a + i];
          sj[i] = jv[u];
#pragma unroll
          for (int d = 0; d < D; ++d) kv[u][d] = kc[(long long)d * g.M + a + i];
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < CL_BIGREG; ++u) {
        const int i = threadIdx.x + u * CL_THREADS;
        if (i < n) {
          int r = 0;
          for (int k = 0; k < n; ++k) r += sj[k] < jv[u];
          jc[a + r] = jv[u];
#pragma unroll
          for (int d = 0; d < D; ++d) kc[(long long)d * g.M + a + r] = kv[u][d];
        }
      }
    } else {  // very dense cell: ranks through scratch, chunks of the index list in shared memory
      for (int r0 = 0; r0 < n; r0 += CL_THREADS) {
        const bool mine = r0 + (int)threadIdx.x < n;
        const int p = a + r0 + threadIdx.x;
        const int jvv = mine ? jc[p] : 0x7fffffff;
        int rank = 0;
        for (int c0 = 0; c0 < n; c0 += CL_THREADS * CL_BIGREG) {
          __syncthreads();
          for (int u = threadIdx.x; u < CL_THREADS * CL_BIGREG; u += CL_THREADS)
            sj[u] = c0 + u < n ? jc[a + c0 + u] : 0x7fffffff;
          __syncthreads();
          const int lim = min(CL_THREADS * CL_BIGREG, n - c0);
          for (int u = 0; u < lim; ++u) rank += sj[u] < jvv;
        }
        if (mine) {
          sj_out[a + rank] = jvv;
#pragma unroll
          for (int d = 0; d < D; ++d) sk_out[(long long)d * g.M + a + rank] = kc[(long long)d * g.M + p];
        }
      }
      __syncthreads();
      for (int r = threadIdx.x; r < n; r += CL_THREADS) {
        jc[a + r] = sj_out[a + r];
#pragma unroll
        for (int d = 0; d < D; ++d) kc[(long long)d * g.M + a + r] = sk_out[(long long)d * g.M + a + r];
      }
    }
    __syncthreads();
  }
}

}  // namespace nfftb
