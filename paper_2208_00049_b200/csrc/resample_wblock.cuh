// resample_wblock.cuh — adjoint spreading for D = 2, 3 over CELL-SORTED nodes
// with WARP-OWNED CELL BLOCKS (BASELINE configs[2], [3]).
//
//   adjoint: ghat_l = sum_j f_j psi~(k_j - l/Nt)   (Alg. 4)
//
// Owner-computes, like spread_cell (resample_cell.cuh), but the unit of
// ownership is one WARP: a block of K0 cells along dimension 0 (held in
// registers, one accumulator per cell) times 32 lanes over the trailing
// dimensions (D = 2: 32 cells of the last dimension; D = 3: 4 x 8 cells of
// dimensions 1, 2). The nodes whose footprint reaches the block (cells within
// [-m, Q + m - 2] of it in every dimension, the paper's halo)
// are visited WARP-UNIFORMLY: every lane sees every node of the block's window,
// so control flow never diverges, the node's data are shared-memory broadcasts
// and no CTA-wide barrier is needed (warps are independent; several per CTA for
// residency only). Per node visit a lane forms its trailing-dimension weight
// c = prod_{d>=1} psi_d(lane's cell) (zero outside the footprint), cf = c f_j,
// and adds psi_0(k0) cf to its accumulators. The window is walked plane by
// plane along dimension 0 and the plane index selects (at compile time) the K0
// cells in its reach, so no product along dimension 0 is a zero.
//
// Node enumeration: the window is (K0 + 2m - 1) x (L1 + 2m - 1) rows of
// cell-sorted node ranges along the last dimension (two segments where the row
// wraps, Remark PAPER.md:588-590); their lengths are prefix-summed per warp.
// The warp stages WB_NB nodes at a time, double-buffered with cp.async (lane i
// copies the i-th node's taps from the TENSOR table wt[pos][d][t] of
// nfft_precompute, its value from fc[pos] = f[jc[pos]] and its
// last-dimension cell from cl[pos]) while the previous batch is visited.
// Requires Nt_{D-1} >= L_{D-1} + 2m - 1 (the last-dimension window may not wrap
// onto itself); the host falls back to spread_cell otherwise.
#pragma once

#include "common.cuh"

namespace nfftb {

#ifndef NFFTB_WB_K0
#define NFFTB_WB_K0 16
#endif
#ifndef NFFTB_WB_WARPS
#define NFFTB_WB_WARPS 4
#endif
#ifndef NFFTB_WB_NB
#define NFFTB_WB_NB 16
#endif
#ifndef NFFTB_WB_UNROLL
#define NFFTB_WB_UNROLL 2
#endif
constexpr int WB_UNROLL = NFFTB_WB_UNROLL;  // node visits unrolled per loop iteration
constexpr int WB_K0 = NFFTB_WB_K0;        // cells along dimension 0 per warp (registers)
constexpr int WB_WARPS = NFFTB_WB_WARPS;  // independent warps per CTA
constexpr int WB_NB = NFFTB_WB_NB;        // nodes per staged batch (two batches in flight per warp)

template <typename T, int D, int M>
struct WbCfg {
  static constexpr int TAPS = 2 * M;
  static constexpr int L1 = D == 3 ? 4 : 1;   // lanes along dimension 1 (D = 3)
  static constexpr int LL = D == 3 ? 8 : 32;  // lanes along the last dimension
  static constexpr int W0 = WB_K0 + TAPS - 1;
  static constexpr int W1 = D == 3 ? L1 + TAPS - 1 : 1;
  static constexpr int ROWS = W0 * W1;
  static constexpr int NE = 2 * ROWS;  // window segments (A, B per row)
  // slot: taps [D][2m] (T), value (complex T), last-dimension cell (int); 16-byte multiple
  static constexpr int TAPB = D * TAPS * (int)sizeof(T);
  static constexpr int SLOT = (TAPB + 2 * (int)sizeof(T) + 4 + 15) & ~15;
  static constexpr int TCP = TAPB % 16 == 0 ? 16 : (TAPB % 8 == 0 ? 8 : 4);  // cp.async granularity of the taps
  static constexpr size_t BUF = (size_t)WB_NB * SLOT;
  static constexpr size_t WARP_BYTES = (2 * BUF + 2 * WB_NB * 8 + (size_t)(2 * NE + 2) * 4 + 15) & ~(size_t)15;
};

template <int BYTES>
__device__ __forceinline__ void wb_cp_async(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
  else if constexpr (BYTES == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}

// fc[b][pos] = f[b][jc[pos]] for pos in the node shard [nb, ne), else 0 (the
// node values in cell order, read by the warps' stages)
template <typename T>
__global__ void __launch_bounds__(256) permute_f_kernel(const typename cplx<T>::type* __restrict__ f,
                                                        const int* __restrict__ jc, int M, int nb, int ne,
                                                        typename cplx<T>::type* __restrict__ fc) {
  using C = typename cplx<T>::type;
  constexpr int PF = 4;  // positions per thread: the index loads of all four in flight, then the gathers
  const long long b = blockIdx.y;
  const int p0 = blockIdx.x * 256 * PF + threadIdx.x;
  int j[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int pos = p0 + k * 256;
    j[k] = (pos < M && pos >= nb && pos < ne) ? __ldg(jc + pos) : -1;
  }
  C v[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    v[k].x = (T)0;
    v[k].y = (T)0;
    if (j[k] >= 0) v[k] = f[b * M + j[k]];
  }
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int pos = p0 + k * 256;
    if (pos < M) fc[b * M + pos] = v[k];
  }
}

// Visits of the nn staged nodes of window plane U0 (compile-time): cell k0 of the
// block gets tap k0 - U0 + 2m - 1 of dimension 0, so only the k0 in reach of the
// plane are accumulated.
template <typename T, int D, int M, int U0>
__device__ __forceinline__ void wb_visit(int nn, const unsigned char* __restrict__ buf, const int2* __restrict__ su,
                                         int ly1, int lyl, typename cplx<T>::type (&acc)[WB_K0]) {
  using C = typename cplx<T>::type;
  using Cfg = WbCfg<T, D, M>;
  constexpr int TAPS = 2 * M;
  constexpr int KLO = U0 - TAPS + 1 > 0 ? U0 - TAPS + 1 : 0;
  constexpr int KHI = U0 < WB_K0 - 1 ? U0 : WB_K0 - 1;
#pragma unroll(WB_UNROLL)
  for (int n = 0; n < nn; ++n) {
    const unsigned char* sl = buf + n * Cfg::SLOT;
    const T* w = reinterpret_cast<const T*>(sl);
    const int2 u = su[n];  // (u1 - 2m + 1, wrap correction - a_last - 2m + 1)
    const int ll = lyl - (*reinterpret_cast<const int*>(sl + Cfg::TAPB + 2 * sizeof(T)) + u.y);  // last-dim tap
    T c = (unsigned)ll < (unsigned)TAPS ? w[(D - 1) * TAPS + ll] : (T)0;
    if (D == 3) {
      const int l1 = ly1 - u.x;
      c *= (unsigned)l1 < (unsigned)TAPS ? w[TAPS + l1] : (T)0;
    }
    const C v = *reinterpret_cast<const C*>(sl + Cfg::TAPB);
    const T cx = c * v.x, cy = c * v.y;
#pragma unroll
    for (int k = KLO; k <= KHI; ++k) {
      const T w0 = w[k - U0 + TAPS - 1];
      acc[k].x = fma(w0, cx, acc[k].x);
      acc[k].y = fma(w0, cy, acc[k].y);
    }
  }
}

template <typename T, int D, int M, int U0 = 0>
__device__ __forceinline__ void wb_visit_plane(int u0, int nn, const unsigned char* buf, const int2* su, int ly1,
                                               int lyl, typename cplx<T>::type (&acc)[WB_K0]) {
  if constexpr (U0 < WbCfg<T, D, M>::W0) {
    if (u0 == U0) wb_visit<T, D, M, U0>(nn, buf, su, ly1, lyl, acc);
    else wb_visit_plane<T, D, M, U0 + 1>(u0, nn, buf, su, ly1, lyl, acc);
  }
}

template <typename T, int D, int M>
__global__ void __launch_bounds__(32 * WB_WARPS) spread_wb_kernel(Geom g, const typename cplx<T>::type* __restrict__ fc,
                                                                  const int* __restrict__ cl,
                                                                  const T* __restrict__ wt,
                                                                  const int* __restrict__ cstart,
                                                                  typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  using Cfg = WbCfg<T, D, M>;
  constexpr int TAPS = Cfg::TAPS, K0 = WB_K0, NE = Cfg::NE, NB = WB_NB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // ---- this warp's block (binning cell coordinates of its first cell)
  const int NtL = g.Nt[D - 1];
  const int nbl = (NtL + Cfg::LL - 1) / Cfg::LL;
  const int nb1 = D == 3 ? (g.Nt[1] + Cfg::L1 - 1) / Cfg::L1 : 1;
  const int nb0 = (g.Nt[0] + K0 - 1) / K0;
  const long long blk = (long long)blockIdx.x * WB_WARPS + warp;
  if (blk >= (long long)nb0 * nb1 * nbl) return;  // warps are independent: no CTA barrier below
  const int bl = (int)(blk % nbl);
  const int b1 = (int)((blk / nbl) % nb1);
  const int b0 = (int)(blk / ((long long)nbl * nb1));
  const int Y0 = b0 * K0, Y1 = b1 * Cfg::L1, YL = bl * Cfg::LL;
  // ---- shared layout of this warp
  unsigned char* base = smem_raw + (size_t)warp * Cfg::WARP_BYTES;
  unsigned char* sbuf = base;                              // [2][NB] slots
  int2* su = reinterpret_cast<int2*>(base + 2 * Cfg::BUF);  // [2][NB] per node: dimension-1 row, last-dim offset
  int* epos = reinterpret_cast<int*>(su + 2 * NB);          // [NE]     first cell-sorted position of a segment
  int* epre = epos + NE;                                   // [NE + 1] prefix of the segment lengths
  // ---- window segments: row r = (u0, u1), last-dimension cells [YL - m, YL + LL + m - 2]
  const int a_last = YL - M, b_last = YL + Cfg::LL + M - 2;
  constexpr int PER = (NE + 31) / 32;
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = lane * PER + i;
    if (e < NE) {
      const int r = e >> 1, seg = e & 1;
      const int u0 = r / Cfg::W1, u1 = r - u0 * Cfg::W1;
      long long rowkey = pos_mod(Y0 - M + u0, g.Nt[0]);
      if (D == 3) rowkey = rowkey * g.Nt[1] + pos_mod(Y1 - M + u1, g.Nt[1]);
      rowkey *= NtL;
      int p0 = 0, len = 0;
      if (a_last < 0) {  // [Nt + a, Nt) then [0, b]
        if (seg == 0) { p0 = __ldg(cstart + rowkey + NtL + a_last); len = __ldg(cstart + rowkey + NtL) - p0; }
        else { p0 = __ldg(cstart + rowkey); len = __ldg(cstart + rowkey + b_last + 1) - p0; }
      } else if (b_last >= NtL) {  // [a, Nt) then [0, b - Nt]
        if (seg == 0) { p0 = __ldg(cstart + rowkey + a_last); len = __ldg(cstart + rowkey + NtL) - p0; }
        else { p0 = __ldg(cstart + rowkey); len = __ldg(cstart + rowkey + b_last - NtL + 1) - p0; }
      } else if (seg == 0) {
        p0 = __ldg(cstart + rowkey + a_last);
        len = __ldg(cstart + rowkey + b_last + 1) - p0;
      }
      epos[e] = p0;
      epre[e] = len;
      cnt += len;
    }
  }
  int total;
  int run = warp_exclusive_scan(cnt, total);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int e = lane * PER + i;
    if (e < NE) {
      const int c = epre[e];
      epre[e] = run;
      run += c;
    }
  }
  if (lane == 0) epre[NE] = total;
  __syncwarp();
  // ---- batches: (plane u0, first node q0 of the plane's range), NB nodes each
  auto plane_beg = [&](int u0) { return epre[2 * u0 * Cfg::W1]; };
  auto plane_end = [&](int u0) { return epre[2 * (u0 + 1) * Cfg::W1]; };
  auto stage = [&](int slot, int u0, int q0) {  // lane i < NB copies node q0 + i of plane u0
    const int e0 = 2 * u0 * Cfg::W1, e1 = e0 + 2 * Cfg::W1;
    const int q = q0 + lane;
    if (lane < NB && q < epre[e1]) {
      int lo = e0, hi = e1;  // largest e with epre[e] <= q
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (epre[mid] <= q) lo = mid;
        else hi = mid;
      }
      const int pos = epos[lo] + (q - epre[lo]);
      unsigned char* sl = sbuf + (size_t)slot * Cfg::BUF + lane * Cfg::SLOT;
      const unsigned char* src = reinterpret_cast<const unsigned char*>(wt + (long long)pos * D * TAPS);
#pragma unroll
      for (int o = 0; o < Cfg::TAPB; o += Cfg::TCP) wb_cp_async<Cfg::TCP>(sl + o, src + o);
      wb_cp_async<2 * sizeof(T)>(sl + Cfg::TAPB, fc + pos);
      wb_cp_async<4>(sl + Cfg::TAPB + 2 * sizeof(T), cl + pos);
      // window-local last cell ul = cl + corr - a_last (corr undoes the wrap of segment A / B), stored
      // so that a visit forms its tap as lane - (cl + .y) and lane - .x
      const int seg = lo & 1;
      const int corr = a_last < 0 ? (seg == 0 ? -NtL : 0) : (b_last >= NtL && seg == 1 ? NtL : 0);
      su[slot * NB + lane] = make_int2((lo >> 1) - u0 * Cfg::W1 - (TAPS - 1), corr - a_last - (TAPS - 1));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  fc += (long long)blockIdx.y * g.M;  // batch vector
  // first batch
  int u0 = 0;
  while (u0 < Cfg::W0 && plane_beg(u0) >= plane_end(u0)) ++u0;
  int q0 = u0 < Cfg::W0 ? plane_beg(u0) : 0;
  const int ly1 = D == 3 ? lane >> 3 : 0;
  const int lyl = D == 3 ? (lane & 7) : lane;
  C acc[K0];
#pragma unroll
  for (int k = 0; k < K0; ++k) {
    acc[k].x = (T)0;
    acc[k].y = (T)0;
  }
  int slot = 0;
  // the values in cell order come from the previous kernel (permute_f): under programmatic dependent
  // launch the window enumeration above overlaps its tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (u0 < Cfg::W0) stage(0, u0, q0);
  while (u0 < Cfg::W0) {
    // next batch: rest of this plane, else the next non-empty plane
    int nu = u0, nq = q0 + NB;
    if (nq >= plane_end(nu)) {
      ++nu;
      while (nu < Cfg::W0 && plane_beg(nu) >= plane_end(nu)) ++nu;
      nq = nu < Cfg::W0 ? plane_beg(nu) : 0;
    }
    if (nu < Cfg::W0) stage(slot ^ 1, nu, nq);
    else asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncwarp();
    wb_visit_plane<T, D, M>(u0, min(NB, plane_end(u0) - q0), sbuf + (size_t)slot * Cfg::BUF, su + slot * NB, ly1,
                            lyl, acc);
    __syncwarp();
    u0 = nu;
    q0 = nq;
    slot ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // ---- plain stores of the owned cells (storage = (binning cell - Nt/2) mod Nt)
  const int yl = YL + lyl, y1 = Y1 + ly1;
  if (yl >= NtL || (D == 3 && y1 >= g.Nt[1])) return;
  long long colidx = pos_mod(yl - (NtL >> 1), NtL);
  if (D == 3) colidx += (long long)pos_mod(y1 - (g.Nt[1] >> 1), g.Nt[1]) * NtL;
  const long long plane = D == 3 ? (long long)g.Nt[1] * NtL : NtL;
  C* dst = grid + (long long)blockIdx.y * g.grid_cells + colidx;
#pragma unroll
  for (int k = 0; k < K0; ++k) {
    const int y0 = Y0 + k;
    if (y0 < g.Nt[0]) dst[(long long)pos_mod(y0 - (g.Nt[0] >> 1), g.Nt[0]) * plane] = acc[k];
  }
}

}  // namespace nfftb
