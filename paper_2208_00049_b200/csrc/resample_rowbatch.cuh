// resample_rowbatch.cuh — adjoint spreading for BATCHES of 2D transforms that
// share their nodes (BASELINE configs[4]: radial
// trajectory, B = 32, ComplexF32) over cell-sorted nodes (cellbin.cuh).
//
//   adjoint: ghat_l^b = sum_j f_j^b psi~(k_j - l/Nt)   (Alg. 4)
//
// LANES = BATCH VECTORS: the taps, footprints and indices are common to the B
// vectors, so a warp handles one node at a time for 32 vectors (warp-uniform
// control flow, taps evaluated once per node by nfft_precompute rather than
// once per node and vector). Node values travel transposed AND in cell order,
// f^T[pos][b] (transpose_bm: one 256-byte row per position, C64), so a chunk of
// consecutive positions is one contiguous block. The adjoint kernel,
// spread_rb2_kernel (below), is OWNER-COMPUTES: every grid cell is written
// exactly once with a plain store (no atomics, no zero pass; the paper's locked
// merge, becomes reading the halo NODES). The round-1
// kernel (one CTA per 16-cell row segment, one warp per window row, cell-by-cell
// walk) is in attic/spread_rowbatch_round1.cuh.txt.
#pragma once

#include "common.cuh"

namespace nfftb {


constexpr int RB_LANES = 32;     // vectors per chunk
constexpr int RB_PITCH = 33;     // partial-row pitch in shared memory (vectors + 1)

// (B, M) -> (M, BP) and back; BP = batch padded to a multiple of 32 (pad rows unused)
// out[inv[j]][b] = in[b][j]: node values transposed into CELL order (inv = inverse of the
// cell-sort permutation jc), one 32-vector row per position
template <typename T>
__global__ void __launch_bounds__(256) transpose_bm_kernel(const typename cplx<T>::type* __restrict__ in, int B, int M,
                                                           int BP, const int* __restrict__ inv,
                                                           typename cplx<T>::type* __restrict__ out) {
  using C = typename cplx<T>::type;
  __shared__ C t[32][33];
  const int j0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  int dst[4];  // destination positions of this thread's output rows, loaded with the values
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + ty + 8 * k;
    dst[k] = j < M ? __ldg(inv + j) : 0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = ty + 8 * k;
    const int b = b0 + r, j = j0 + tx;
    if (b < B && j < M) t[r][tx] = in[(long long)b * M + j];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = ty + 8 * k;
    const int j = j0 + r, b = b0 + tx;
    if (j < M && b < B) out[(long long)dst[k] * BP + b] = t[tx][r];
  }
}

// inv[jc[pos]] = pos (precompute, batch adjoint)
static __global__ void __launch_bounds__(256) invert_perm_kernel(const int* __restrict__ jc, int M, int* __restrict__ inv) {
  const int pos = blockIdx.x * 256 + threadIdx.x;
  if (pos < M) inv[jc[pos]] = pos;
}

template <typename T>
__global__ void __launch_bounds__(256) transpose_mb_kernel(const typename cplx<T>::type* __restrict__ in, int B, int M,
                                                           int BP, typename cplx<T>::type* __restrict__ out) {
  using C = typename cplx<T>::type;
  __shared__ C t[32][33];
  const int j0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r, b = b0 + tx;
    if (j < M && b < B) t[r][tx] = in[(long long)j * BP + b];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, j = j0 + tx;
    if (b < B && j < M) out[(long long)b * M + j] = t[tx][r];
  }
}

// Taps of every cell-sorted node, wt[pos][d][t] (the paper's TENSOR layout,
// PAPER.md:599-604), computed by nfft_precompute for the D >= 2 adjoints. A CTA
// of TN_NODES threads (one node each) builds its contiguous block of the table
// in shared memory (row stride D * 2m + 1: conflict-free) and writes it out
// coalesced (the per-thread 8-byte stores at a D * 2m stride were store-bound).
// cl (optional): the last-dimension binning cell of every position.
constexpr int TN_NODES = 64;
template <typename T, int D, int M, int DEG>
__global__ void __launch_bounds__(TN_NODES) taps_nd_kernel(Geom g, WinPolyN<T, D, M> wp, const T* __restrict__ kc,
                                                           T* __restrict__ wt, int* __restrict__ cl) {
  constexpr int ROW = D * 2 * M, RS = ROW + 1;
  __shared__ T s[TN_NODES * RS];
  const long long p0 = (long long)blockIdx.x * TN_NODES;
  const long long pc = p0 + threadIdx.x;
  if (pc < g.M) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double frac;
      const int c = node_cell((double)kc[(long long)d * g.M + pc], g.Ntd[d], g.Nt[d], frac);
      if (cl != nullptr && d == D - 1) cl[pc] = c;  // last-dimension cell (warp-block adjoint)
      T w[2 * M];
      window_taps<T, M, DEG>((T)(frac - 0.5), wp.mu[d], w);
#pragma unroll
      for (int t = 0; t < 2 * M; ++t) s[threadIdx.x * RS + d * 2 * M + t] = w[t];
    }
  }
  __syncthreads();
  const int n = (int)(g.M - p0 < TN_NODES ? g.M - p0 : TN_NODES);
  T* out = wt + p0 * ROW;
  for (int i = threadIdx.x; i < n * ROW; i += TN_NODES) {
    const int node = i / ROW, k = i - node * ROW;
    out[i] = s[node * RS + k];
  }
}

// ---------------------------------------------------------------- spread_rb2
// Batch adjoint: owner-computes, lanes = batch vectors, every cell written once
// with a plain coalesced store; no atomics, no zero pass.
//
// The CTA owns R consecutive output rows y0 .. y0 + R - 1, cells [c0, c0 + S),
// for one 32-vector chunk. Its nodes are those of the 2m + R - 1 window rows
// a = y0 - m + r, columns [c0 - m, c0 + S + m - 2]: per window row ONE
// contiguous range of the cell-sorted order (two when the window wraps around
// the torus). The window rows' ranges, concatenated, form one virtual node
// sequence that the CTA's warps split EVENLY, so the dense centre of a radial
// trajectory spreads over all warps of its CTA instead of serialising one warp
// per window row. A warp walks its slice in chunks of CH nodes staged with
// cp.async into a per-warp double buffer (values f^T[pos][b], taps
// wt[pos][d][t], last-dimension cells cl[pos]): the next chunk is in flight
// while the current one is accumulated. Window row r gives output row j the
// dimension-0 tap 2m - 1 - r + j (zero outside [0, 2m)); the
// node's window column u = cl + shift in [0, S + 2m - 1) selects, through a
// warp-uniform switch, a compile-time body that adds v w0_j w1[t] to exactly the
// cells the node reaches along the last dimension; fp32 multiply-adds are
// packed FFMA2. The warps' partial rows are summed in shared memory (aliasing
// the staging buffers), one output row at a time, and stored coalesced.
#ifndef NFFTB_RB2_R
#define NFFTB_RB2_R 2
#endif
#ifndef NFFTB_RB2_SF
#define NFFTB_RB2_SF 16
#endif
#ifndef NFFTB_RB2_CHF
#define NFFTB_RB2_CHF 16
#endif
#ifndef NFFTB_RB2_MINB
#define NFFTB_RB2_MINB 2
#endif
constexpr int RB2_WARPS = 8;
template <typename T> struct Rb2Cfg {
  static constexpr int R = sizeof(T) == 4 ? NFFTB_RB2_R : 1;    // output rows per CTA
  static constexpr int S = sizeof(T) == 4 ? NFFTB_RB2_SF : 16;  // output cells per CTA (last dimension)
  static constexpr int CH = sizeof(T) == 4 ? NFFTB_RB2_CHF : 8;  // staged nodes per chunk
};

__host__ __device__ constexpr size_t rb2_al16(size_t b) { return (b + 15) & ~(size_t)15; }
// one staging buffer of a warp: values, tap rows (both dimensions), cells
__host__ __device__ constexpr size_t rb2_vbytes(int CH, size_t csize) { return (size_t)CH * 32 * csize; }
// staged tap record of a node: 2m dimension-0 taps, 2m last-dimension taps, 16 zero bytes (the row tap of
// a window row that does not reach an output row reads the zeros: no predicated loads)
__host__ __device__ constexpr int rb2_rec(int M, size_t rsize) { return 4 * M + (int)(16 / rsize); }
__host__ __device__ constexpr size_t rb2_wbytes(int CH, int M, size_t rsize) { return (size_t)CH * rb2_rec(M, rsize) * rsize; }
__host__ __device__ constexpr size_t rb2_buf_bytes(int CH, int M, size_t csize, size_t rsize) {
  return rb2_al16(rb2_vbytes(CH, csize)) + rb2_al16(rb2_wbytes(CH, M, rsize)) + rb2_al16((size_t)CH * 4);
}
__host__ __device__ inline size_t rb2_smem_bytes(int M, int rsize) {
  const bool f32 = rsize == 4;
  const int CH = f32 ? Rb2Cfg<float>::CH : Rb2Cfg<double>::CH, S = f32 ? Rb2Cfg<float>::S : Rb2Cfg<double>::S;
  const size_t csize = 2 * (size_t)rsize;
  const size_t stage = (size_t)RB2_WARPS * 2 * rb2_buf_bytes(CH, M, csize, rsize);
  const size_t part = (size_t)RB2_WARPS * S * RB_PITCH * csize;  // one output row's partials
  return stage > part ? stage : part;
}

// the cells k of the segment reached by a node in window column U (compile-time):
// acc[j][k] += w1[k - U + 2m - 1] * vw[j]
template <typename T, int M, int R, int S, int U>
__device__ __forceinline__ void rb2_cells(typename cplx<T>::type (&acc)[R][S], const typename cplx<T>::type (&vw)[R],
                                          const T (&w1)[2 * M]) {
  constexpr int TAPS = 2 * M;
  constexpr int KLO = U - TAPS + 1 > 0 ? U - TAPS + 1 : 0;
  constexpr int KHI = U < S - 1 ? U : S - 1;
#pragma unroll
  for (int k = KLO; k <= KHI; ++k) {
    const T w = w1[k - U + TAPS - 1];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if constexpr (sizeof(T) == 4) {
        acc[j][k] = __ffma2_rn(make_float2(w, w), vw[j], acc[j][k]);
      } else {
        acc[j][k].x = fma(w, vw[j].x, acc[j][k].x);
        acc[j][k].y = fma(w, vw[j].y, acc[j][k].y);
      }
    }
  }
}

// one node (staged slot q) in window column U: value, row taps (zero where window row p does not
// reach output row j), last-dimension taps, then the compile-time cell body
template <typename T, int M, int R, int S, int U>
__device__ __forceinline__ void rb2_visit(typename cplx<T>::type (&acc)[R][S], const typename cplx<T>::type* sv,
                                          const T* sw, const int (&tj)[R]) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M;
  T w1[TAPS];
  if constexpr ((TAPS * sizeof(T)) % 16 == 0) {
#pragma unroll
    for (int t = 0; t < TAPS; t += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        const float4 v4 = *reinterpret_cast<const float4*>(sw + TAPS + t);
        w1[t] = v4.x; w1[t + 1] = v4.y; w1[t + 2] = v4.z; w1[t + 3] = v4.w;
      } else {
        const double2 v2 = *reinterpret_cast<const double2*>(sw + TAPS + t);
        w1[t] = v2.x; w1[t + 1] = v2.y;
      }
    }
  } else {
#pragma unroll
    for (int t = 0; t < TAPS; ++t) w1[t] = sw[TAPS + t];
  }
  const C v = *sv;
  C vw[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const T w0 = sw[tj[j]];
    if constexpr (sizeof(T) == 4) {
      vw[j] = __fmul2_rn(make_float2(w0, w0), v);
    } else {
      vw[j].x = w0 * v.x;
      vw[j].y = w0 * v.y;
    }
  }
  rb2_cells<T, M, R, S, U>(acc, vw, w1);
}

// window column U of the fall-through walk: visit the chunk's nodes with u == U, then fall into U + 1
#define NFFTB_RB2_STEP(U)                                                                       \
  case U:                                                                                       \
    if constexpr (U < S + 2 * M - 1) {                                                          \
      while (uq == U) {                                                                         \
        rb2_visit<T, M, R, S, U>(acc, sv + q * 32, sw + q * REC, tj);                           \
        if (++q == cnt) goto chunk_done;                                                        \
        uq = sc[q] + sh;                                                                        \
      }                                                                                         \
    }                                                                                           \
    [[fallthrough]];

template <typename T, int M>
__global__ void __launch_bounds__(32 * RB2_WARPS, NFFTB_RB2_MINB) spread_rb2_kernel(
    Geom g, const typename cplx<T>::type* __restrict__ fTc, int BP, const T* __restrict__ wt,
    const int* __restrict__ cl, const int* __restrict__ cstart, typename cplx<T>::type* __restrict__ grid) {
  using C = typename cplx<T>::type;
  constexpr int TAPS = 2 * M, R = Rb2Cfg<T>::R, S = Rb2Cfg<T>::S, CH = Rb2Cfg<T>::CH, NW = RB2_WARPS;
  constexpr int WR = TAPS + R - 1;  // window rows (lane r describes window row r)
  constexpr int REC = rb2_rec(M, sizeof(T));
  static_assert(WR <= 32, "window rows per warp");
  static_assert(S + 2 * M - 1 <= 48, "switch cases");
  constexpr size_t VB = rb2_al16(rb2_vbytes(CH, sizeof(C))), WB = rb2_al16(rb2_wbytes(CH, M, sizeof(T)));
  constexpr size_t BUF = rb2_buf_bytes(CH, M, sizeof(C), sizeof(T));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b0 = blockIdx.y * RB_LANES;
  const int Nt0 = g.Nt[0], NtL = g.Nt[1];
  const int nseg = (NtL + S - 1) / S;
  const int nunits = (Nt0 + R - 1) / R * nseg;
  const int nbc = min(RB_LANES, g.B - b0);
  unsigned char* wbase = smem_raw + (size_t)warp * 2 * BUF;
  fTc += b0;
  // 1. window row r = lane of this CTA's unit (y0, c0): part 0 (unwrapped columns) [lo0, lo0 + len0)
  //    with column shift sh0, part 1 (the columns wrapped around the torus) [lo1, lo1 + len1) with shift
  //    sh1. One CTA per unit (a persistent launch with the next unit prefetched measured slower, both
  //    with a static and with a dynamic unit order: DESIGN.md §6).
  struct Raw {
    int c[4];
  };
  auto unit_geom = [&](int unit, int& y0, int& c0, int& qs) {
    const int yb = unit / nseg;
    y0 = yb * R;
    c0 = (unit - yb * nseg) * S;
    qs = min(S, NtL - c0);
  };
  auto load_raw = [&](int unit) {
    Raw rw;
    rw.c[0] = rw.c[1] = rw.c[2] = rw.c[3] = 0;
    if (unit < nunits && lane < WR) {
      int y0, c0, qs;
      unit_geom(unit, y0, c0, qs);
      int a = y0 - M + lane;
      if (a < 0) a += Nt0;
      else if (a >= Nt0) a -= Nt0;
      const long long rowkey = (long long)a * NtL;
      const int lo_c = c0 - M, hi_c = c0 + qs + M - 1;
      rw.c[0] = __ldg(cstart + rowkey + max(lo_c, 0));
      rw.c[1] = __ldg(cstart + rowkey + min(hi_c, NtL));
      if (lo_c < 0) {
        rw.c[2] = __ldg(cstart + rowkey + lo_c + NtL);
        rw.c[3] = __ldg(cstart + rowkey + NtL);
      } else if (hi_c > NtL) {
        rw.c[2] = __ldg(cstart + rowkey);
        rw.c[3] = __ldg(cstart + rowkey + hi_c - NtL);
      }
    }
    return rw;
  };
  const int unit = blockIdx.x;
  if (unit >= nunits) return;
  const Raw raw = load_raw(unit);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // f^T comes from transpose_bm
  int y0, c0, qs;
  unit_geom(unit, y0, c0, qs);
  const int lo_c = c0 - M;
  const int lo0 = raw.c[0], len0 = raw.c[1] - raw.c[0], sh0 = -lo_c;
  const int lo1 = raw.c[2], len1 = raw.c[3] - raw.c[2], sh1 = lo_c < 0 ? -lo_c - NtL : NtL - lo_c;
  int total;
  const int roff = warp_exclusive_scan(len0 + len1, total);
  int cs0 = c0 - (NtL >> 1);
  if (cs0 < 0) cs0 += NtL;
  if (total == 0) {  // no node reaches the unit (outside a radial trajectory's disk): zeros
    for (int idx = tid; idx < R * nbc * S; idx += NW * 32) {
      const int j = idx / (nbc * S), r2 = idx - j * (nbc * S), bb = r2 / S, k = r2 - bb * S;
      const int y = y0 + j;
      if (k >= qs || y >= Nt0) continue;
      int ys = y - (Nt0 >> 1);
      if (ys < 0) ys += Nt0;
      int cs = cs0 + k;
      if (cs >= NtL) cs -= NtL;
      C z;
      z.x = (T)0;
      z.y = (T)0;
      grid[(long long)(b0 + bb) * g.grid_cells + (long long)ys * NtL + cs] = z;
    }
    return;
  }
  // this warp's slice [vs, ve) of the virtual sequence
  const int vs = (int)(((long long)total * warp) / NW), ve = (int)(((long long)total * (warp + 1)) / NW);
  C acc[R][S];
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int k = 0; k < S; ++k) {
      acc[j][k].x = (T)0;
      acc[j][k].y = (T)0;
    }
  // a chunk: window row p, virtual start x (roff_p <= x), cnt nodes, never straddling a part
  struct Chunk {
    int p, x, cnt, pos0, sh;
  };
  auto make_chunk = [&](int x, int p) {  // the chunk starting at x (< ve), searching rows from p
    Chunk c;
    int o, l0, l1;
    while (true) {
      o = __shfl_sync(0xffffffffu, roff, p);
      l0 = __shfl_sync(0xffffffffu, len0, p);
      l1 = __shfl_sync(0xffffffffu, len1, p);
      if (x < o + l0 + l1) break;
      ++p;
    }
    const int lo_0 = __shfl_sync(0xffffffffu, lo0, p), lo_1 = __shfl_sync(0xffffffffu, lo1, p);
    const int s_0 = __shfl_sync(0xffffffffu, sh0, p), s_1 = __shfl_sync(0xffffffffu, sh1, p);
    const int off = x - o;
    c.p = p;
    c.x = x;
    if (off < l0) {
      c.pos0 = lo_0 + off;
      c.sh = s_0;
      c.cnt = min(min(CH, l0 - off), ve - x);
    } else {
      c.pos0 = lo_1 + (off - l0);
      c.sh = s_1;
      c.cnt = min(min(CH, l0 + l1 - off), ve - x);
    }
    return c;
  };
  auto stage = [&](const Chunk& c, int buf) {
    unsigned char* sb = wbase + (size_t)buf * BUF;
    constexpr int VP = 32 * (int)sizeof(C) / 16;  // 16-byte pieces per value row
    for (int e = lane; e < c.cnt * VP; e += 32) {
      const int q = e / VP, pc = e - q * VP;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(sb + (size_t)q * 32 * sizeof(C) + pc * 16);
      const void* src = reinterpret_cast<const unsigned char*>(fTc + (long long)(c.pos0 + q) * BP) + pc * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src) : "memory");
    }
    // tap records: the node's 2 * TAPS reals (a 16-byte multiple, contiguous for consecutive positions)
    // and one zero-filled piece (source size 0)
    constexpr int WP = 2 * TAPS * (int)sizeof(T) / 16 + 1;  // pieces per record
    const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(wt + (long long)c.pos0 * 2 * TAPS);
    for (int e = lane; e < c.cnt * WP; e += 32) {
      const int q = e / WP, pc = e - q * WP;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(sb + VB + (size_t)e * 16);
      const unsigned char* src = wsrc + (size_t)q * 2 * TAPS * sizeof(T) + pc * 16;
      const int nbytes = pc < WP - 1 ? 16 : 0;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(nbytes) : "memory");
    }
    if (lane < c.cnt) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(sb + VB + WB + (size_t)lane * 4);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(cl + c.pos0 + lane) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (vs < ve) {
    Chunk cur = make_chunk(vs, 0);
    int buf = 0;
    stage(cur, 0);
    while (true) {
      Chunk nxt;
      nxt.cnt = 0;
      const int xn = cur.x + cur.cnt;
      if (xn < ve) {
        nxt = make_chunk(xn, cur.p);
        stage(nxt, buf ^ 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
      __syncwarp();
      {  // accumulate the current chunk
        const unsigned char* sb = wbase + (size_t)buf * BUF;
        const C* sv = reinterpret_cast<const C*>(sb) + lane;
        const T* sw = reinterpret_cast<const T*>(sb + VB);
        const int* sc = reinterpret_cast<const int*>(sb + VB + WB);
        int tj[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int t = TAPS - 1 - cur.p + j;
          tj[j] = (unsigned)t < (unsigned)TAPS ? t : 2 * TAPS;  // out of reach: the record's zeros
        }
        // the chunk's nodes lie in one window row part, in column order: u is non-decreasing, so the
        // walk enters the unrolled sequence of window columns once (switch on the first node's u) and
        // falls through it, each column U visiting its nodes with a compile-time body
        const int sh = cur.sh, cnt = cur.cnt;
        int q = 0, uq = sc[0] + sh;
        switch (uq) {
          NFFTB_RB2_STEP(0) NFFTB_RB2_STEP(1) NFFTB_RB2_STEP(2) NFFTB_RB2_STEP(3) NFFTB_RB2_STEP(4)
          NFFTB_RB2_STEP(5) NFFTB_RB2_STEP(6) NFFTB_RB2_STEP(7) NFFTB_RB2_STEP(8) NFFTB_RB2_STEP(9)
          NFFTB_RB2_STEP(10) NFFTB_RB2_STEP(11) NFFTB_RB2_STEP(12) NFFTB_RB2_STEP(13) NFFTB_RB2_STEP(14)
          NFFTB_RB2_STEP(15) NFFTB_RB2_STEP(16) NFFTB_RB2_STEP(17) NFFTB_RB2_STEP(18) NFFTB_RB2_STEP(19)
          NFFTB_RB2_STEP(20) NFFTB_RB2_STEP(21) NFFTB_RB2_STEP(22) NFFTB_RB2_STEP(23) NFFTB_RB2_STEP(24)
          NFFTB_RB2_STEP(25) NFFTB_RB2_STEP(26) NFFTB_RB2_STEP(27) NFFTB_RB2_STEP(28) NFFTB_RB2_STEP(29)
          NFFTB_RB2_STEP(30) NFFTB_RB2_STEP(31) NFFTB_RB2_STEP(32) NFFTB_RB2_STEP(33) NFFTB_RB2_STEP(34)
          NFFTB_RB2_STEP(35) NFFTB_RB2_STEP(36) NFFTB_RB2_STEP(37) NFFTB_RB2_STEP(38) NFFTB_RB2_STEP(39)
          NFFTB_RB2_STEP(40) NFFTB_RB2_STEP(41) NFFTB_RB2_STEP(42) NFFTB_RB2_STEP(43) NFFTB_RB2_STEP(44)
          NFFTB_RB2_STEP(45) NFFTB_RB2_STEP(46) NFFTB_RB2_STEP(47)
          default: break;
        }
      chunk_done:;
      }
      __syncwarp();  // the buffer is consumed before it is restaged
      if (nxt.cnt == 0) break;
      cur = nxt;
      buf ^= 1;
    }
  }
  // 2. sum the warps' partial rows in shared memory (aliasing the staging buffers), one output row at a
  //    time; one coalesced store per output cell and vector
  C* part = reinterpret_cast<C*>(smem_raw);  // [NW][S][RB_PITCH]
#pragma unroll
  for (int j = 0; j < R; ++j) {
    __syncthreads();  // staging buffers / the previous row's partials are consumed
#pragma unroll
    for (int k = 0; k < S; ++k) part[((size_t)warp * S + k) * RB_PITCH + lane] = acc[j][k];
    __syncthreads();
    const int y = y0 + j;
    if (y >= Nt0) break;
    int ys = y - (Nt0 >> 1);
    if (ys < 0) ys += Nt0;
    const long long rowoff = (long long)ys * NtL;
    for (int idx = tid; idx < nbc * S; idx += NW * 32) {
      const int bb = idx / S, k = idx - bb * S;
      if (k >= qs) continue;
      C a;
      a.x = (T)0;
      a.y = (T)0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const C c = part[((size_t)w * S + k) * RB_PITCH + bb];
        a.x += c.x;
        a.y += c.y;
      }
      int cs = cs0 + k;
      if (cs >= NtL) cs -= NtL;
      grid[(long long)(b0 + bb) * g.grid_cells + rowoff + cs] = a;
    }
  }

}
#undef NFFTB_RB2_STEP

}  // namespace nfftb
