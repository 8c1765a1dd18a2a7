// binsort.cuh — node binning + stable counting sort into tiles as ONE
// cooperative kernel.
//
// The three-kernel sort of precompute.cuh (count / column scan / scatter)
// re-reads the nodes twice and pays two launch gaps plus a narrow scan; here
// every node is read once into registers and the phases are separated by
// grid-wide barriers (cooperative launch: all CTAs resident):
//
//  phase 1  CTA b owns the nodes [b E, (b+1) E), E = 16 warps x R rounds x 32,
//           in node order warp-major, round, lane. Per node: fp64 binning
//           (node_key, reading R10/R11) -> tile key. In-warp stable rank with
//           __match_any_sync against a warp-private u16 counter per tile; a
//           per-tile prefix over the 16 warps turns it into the rank inside
//           the CTA; the CTA's tile histogram goes to row b of cnt[G][P].
//  phase 2  column prefix of cnt over the G rows, spread over all CTAs (CTA b
//           takes a band of columns, its threads split the rows): cnt[b][t]
//           becomes the number of tile-t nodes in CTAs < b; total[t] = tile
//           count.
//  phase 3  every CTA scans total[] into the tile offsets (shared memory;
//           CTA 0 also writes offsets[] and the subproblem list of
//           PAPER.md:512), then places its nodes:
//             pos = offsets[t] + cnt[b][t] + rank-in-CTA
//           -> perm[pos] = j, sorted SoA coordinates ks[d][pos].
// The result is the unique stable order (tile ascending, original index
// ascending; reading R12), bit-identical to the oracle's and to the
// three-kernel path.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "precompute.cuh"

namespace nfftb {

constexpr int BS_THREADS = 512;
constexpr int BS_WARPS = BS_THREADS / 32;

__host__ __device__ inline size_t binsort_smem_bytes(int P) {
  return (((size_t)BS_WARPS * P * 2 + 15) & ~(size_t)15) + (size_t)(P + 1) * 4;
}

// node_key with the dimension as a template parameter (coordinates stay in registers)
template <typename R, int D>
__device__ __forceinline__ int node_key_d(const R* __restrict__ nodes, const Geom& g, int j, R (&k)[MAX_D], bool& bad) {
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
    const int c = node_cell(kd, g.Ntd[d], g.Nt[d], frac);
    key = key * g.P[d] + c / g.Q[d];
  }
  return bad ? 0 : key;
}

template <typename R, int RR, int D>
__global__ void __launch_bounds__(BS_THREADS) binsort_kernel(const R* __restrict__ nodes, Geom g, int P,
                                                             int* __restrict__ cnt, int* __restrict__ total,
                                                             int* __restrict__ offsets, int* __restrict__ perm,
                                                             R* __restrict__ ks, int* __restrict__ err, int nb, int ne,
                                                             int S, int* __restrict__ subbase,
                                                             int4* __restrict__ subs) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char bs_smem[];
  unsigned short* wc = reinterpret_cast<unsigned short*>(bs_smem);  // [P][16]: per tile, one u16 counter per warp
  int* offs = reinterpret_cast<int*>(bs_smem + (((size_t)BS_WARPS * P * 2 + 15) & ~(size_t)15));  // [P+1]
  __shared__ int ws[32];
  __shared__ int psum[BS_THREADS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x;
  const unsigned lt = (1u << lane) - 1u;

  // ---------------- phase 1: keys, in-CTA stable ranks, CTA histogram row
  {
    unsigned* wc32 = reinterpret_cast<unsigned*>(wc);
    for (int i = tid; i < BS_WARPS * P / 2; i += BS_THREADS) wc32[i] = 0u;
  }
  __syncthreads();
  const int base = b * (BS_WARPS * RR * 32);
  int key[RR], rank[RR];
  R kc[RR][MAX_D];
  bool any_bad = false;
  unsigned short* mine = wc + warp;  // counter of tile t for this warp: mine[16 t]
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const int j = base + (warp * RR + r) * 32 + lane;
    key[r] = -1;
    if (j < g.M) {
      bool bad;
      key[r] = node_key_d<R, D>(nodes, g, j, kc[r], bad);
      any_bad |= bad;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key[r]);
    rank[r] = key[r] >= 0 ? (int)mine[key[r] * BS_WARPS] + __popc(peers & lt) : 0;
    __syncwarp();
    if (key[r] >= 0 && lane == __ffs(peers) - 1)
      mine[key[r] * BS_WARPS] = (unsigned short)(mine[key[r] * BS_WARPS] + __popc(peers));
    __syncwarp();
  }
  if (any_bad) atomicOr(err, 1);
  __syncthreads();
  int* crow = cnt + (long long)b * P;
  for (int t = tid; t < P; t += BS_THREADS) {  // exclusive prefix over the 16 warps: 32 bytes per tile
    uint4* row = reinterpret_cast<uint4*>(wc + t * BS_WARPS);
    uint4 v[2] = {row[0], row[1]};
    unsigned* u = reinterpret_cast<unsigned*>(v);
    unsigned run = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const unsigned lo = u[k] & 0xffffu, hi = u[k] >> 16;
      u[k] = run | ((run + lo) << 16);
      run += lo + hi;
    }
    row[0] = v[0];
    row[1] = v[1];
    crow[t] = (int)run;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RR; ++r)
    if (key[r] >= 0) rank[r] += mine[key[r] * BS_WARPS];
  grid.sync();

  // ---------------- phase 2: column prefix of cnt over the G CTA rows
  {
    const int W = (P + G - 1) / G;
    const int c_begin = b * W, c_end = min(P, c_begin + W);
    for (int cc = c_begin; cc < c_end; cc += BS_THREADS) {
      const int nc = min(BS_THREADS, c_end - cc);
      const int parts = min(G, max(1, BS_THREADS / nc));
      const int rows_per = (G + parts - 1) / parts;
      const int col = tid % nc, part = tid / nc;
      const bool act = part < parts;
      const int r0 = part * rows_per, r1 = min(G, r0 + rows_per);
      int s = 0;
      if (act)
        for (int row = r0; row < r1; ++row) s += __ldcg(cnt + (long long)row * P + cc + col);
      if (act) psum[part * nc + col] = s;
      __syncthreads();
      if (act) {
        int run = 0;
        for (int p = 0; p < part; ++p) run += psum[p * nc + col];
        for (int row = r0; row < r1; ++row) {
          const long long idx = (long long)row * P + cc + col;
          const int c = __ldcg(cnt + idx);
          cnt[idx] = run;
          run += c;
        }
        if (part == parts - 1) total[cc + col] = run;
      }
      __syncthreads();
    }
  }
  grid.sync();

  // ---------------- phase 3: tile offsets (every CTA), then placement
  {
    const int per = (P + BS_THREADS - 1) / BS_THREADS;
    const int lo = tid * per, hi = min(P, lo + per);
    int sum = 0;
    for (int i = lo; i < hi; ++i) sum += __ldcg(total + i);
    int tot;
    int run = block_exclusive_scan(sum, ws, tot);
    for (int i = lo; i < hi; ++i) {
      offs[i] = run;
      run += __ldcg(total + i);
    }
    if (tid == 0) offs[P] = tot;
  }
  __syncthreads();
  if (b == 0) {
    for (int i = tid; i <= P; i += BS_THREADS) offsets[i] = offs[i];
    // subproblems: <= S nodes of one tile inside the shard [nb, ne)
    const int per = (P + BS_THREADS - 1) / BS_THREADS;
    const int lo = tid * per, hi = min(P, lo + per);
    int s = 0;
    for (int i = lo; i < hi; ++i) {
      const int a = max(offs[i], nb), e = min(offs[i + 1], ne);
      s += (max(0, e - a) + S - 1) / S;
    }
    int tot;
    int q = block_exclusive_scan(s, ws, tot);
    for (int i = lo; i < hi; ++i) {
      subbase[i] = q;
      const int a = max(offs[i], nb), e = min(offs[i + 1], ne);
      for (int st = a; st < e; st += S) subs[q++] = make_int4(i, st, min(S, e - st), 0);
    }
    if (tid == 0) subbase[P] = tot;
  }
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    if (key[r] < 0) continue;
    const int j = base + (warp * RR + r) * 32 + lane;
    const int pos = offs[key[r]] + __ldcg(crow + key[r]) + rank[r];
    perm[pos] = j;
#pragma unroll
    for (int d = 0; d < D; ++d) ks[(long long)d * g.M + pos] = kc[r][d];
  }
}

}  // namespace nfftb
