// precompute.cuh — node binning, stable sort into tiles, subproblems
// and window tables. All device kernels.
//
// PAPER.md:520-537 (block partition R_p, Gamma_p, Q = ceil(Ntilde/P)),
// PAPER.md:512 (fixed maximum number of nodes per block for balance),
// PAPER.md:439-441 (beta^tensor), PAPER.md:628-642 (polynomial window table).
#pragma once

#include "common.cuh"

namespace nfftb {


// Tile key of node j (reading R10); non-finite coordinates -> key 0, bad = true.
template <typename R>
__device__ __forceinline__ int node_key(const R* __restrict__ nodes, const Geom& g, int j, R (&k)[MAX_D], bool& bad) {
  int key = 0;
  bad = false;
  for (int d = 0; d < g.D; ++d) {
    k[d] = nodes[(long long)j * g.D + d];
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

// ---------------------------------------------------------------- a1+a2: stable counting sort into tiles
// Block b of the sort owns nodes [b*CS_E, (b+1)*CS_E) (CS_W warps x CS_CHUNKS
// chunks of 32 nodes, node order = warp-major, chunk, lane).
//  K1 cs_count:  per-block tile histogram (shared atomics) -> cnt[b][t].
//  K2 cs_scan:   for every tile t, exclusive prefix of cnt[.][t] over blocks
//                (one warp per tile; coalesced across warps of a CTA); the last
//                CTA scans the tile totals into the tile offsets and writes the
//                subproblem list (<= S nodes of one tile inside the shard).
//  K3 cs_scatter: re-walks its block in node order; a node's position is
//                offsets[t] + cnt[b][t] + (earlier nodes of t in this block),
//                the last term from per-warp shared counters and warp match
//                ranks — a stable counting sort, so perm is the unique "tile
//                ascending, original index ascending" order (reading R12). It
//                also writes the tile-sorted SoA coordinates.
constexpr int CS_W = 4;
constexpr int CS_CHUNKS = 4;
constexpr int CS_E = CS_W * 32 * CS_CHUNKS;  // 512 nodes per sort block

template <typename R>
__global__ void __launch_bounds__(CS_W * 32) cs_count_kernel(const R* __restrict__ nodes, Geom g, int n_tiles,
                                                             int* __restrict__ cnt, int* __restrict__ err) {
  extern __shared__ int hist[];
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  const int base = blockIdx.x * CS_E;
  bool any_bad = false;
#pragma unroll
  for (int c = 0; c < CS_CHUNKS; ++c) {
    const int j = base + c * blockDim.x + threadIdx.x;
    if (j < g.M) {
      R k[MAX_D];
      bool bad;
      const int key = node_key(nodes, g, j, k, bad);
      any_bad |= bad;
      atomicAdd(&hist[key], 1);
    }
  }
  if (any_bad) atomicOr(err, 1);
  __syncthreads();
  int* row = cnt + (long long)blockIdx.x * n_tiles;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) row[t] = hist[t];
}

// CTA c scans tile columns [32c, 32c + 32): lane = column, the 8 warps take
// contiguous runs of block rows, so every global access is a coalesced
// 128-byte row segment; a shared-memory prefix over the warps joins the runs.
__global__ void __launch_bounds__(THREADS) cs_scan_kernel(int* __restrict__ cnt, int n_tiles, int nblk, int M,
                                                          int* __restrict__ tile_total, int* __restrict__ offsets,
                                                          unsigned* __restrict__ ticket, int nb, int ne, int S,
                                                          int* __restrict__ subbase, int4* __restrict__ subs) {
  __shared__ int ws[32];
  __shared__ int part[THREADS / 32][33];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int per = (nblk + nw - 1) / nw;
  const int r0 = warp * per, r1 = min(nblk, r0 + per);
  int s = 0;
  if (t < n_tiles) {
#pragma unroll 8
    for (int b = r0; b < r1; ++b) s += cnt[(long long)b * n_tiles + t];
  }
  part[warp][lane] = s;
  __syncthreads();
  int run = 0;
  for (int w = 0; w < warp; ++w) run += part[w][lane];
  if (t < n_tiles) {
    for (int b = r0; b < r1; ++b) {
      const long long idx = (long long)b * n_tiles + t;
      const int c = cnt[idx];
      cnt[idx] = run;
      run += c;
    }
    if (warp == nw - 1) tile_total[t] = run;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  {
    const int per = (n_tiles + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(n_tiles, lo + per);
    int sum = 0;
    for (int i = lo; i < hi; ++i) sum += __ldcg(tile_total + i);
    int total;
    int run = block_exclusive_scan(sum, ws, total);
    for (int i = lo; i < hi; ++i) {
      offsets[i] = run;
      run += __ldcg(tile_total + i);
    }
    if (threadIdx.x == 0) {
      offsets[n_tiles] = M;
      *ticket = 0u;
    }
  }
  __syncthreads();
  {
    const int per = (n_tiles + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(n_tiles, lo + per);
    int s = 0;
    for (int i = lo; i < hi; ++i) {
      const int a = max(offsets[i], nb), b = min(offsets[i + 1], ne);
      s += (max(0, b - a) + S - 1) / S;
    }
    int total;
    int q = block_exclusive_scan(s, ws, total);
    for (int i = lo; i < hi; ++i) {
      subbase[i] = q;
      const int a = max(offsets[i], nb), b = min(offsets[i + 1], ne);
      for (int st = a; st < b; st += S) subs[q++] = make_int4(i, st, min(S, b - st), 0);
    }
    if (threadIdx.x == 0) subbase[n_tiles] = total;
  }
}

template <typename R>
__global__ void __launch_bounds__(CS_W * 32) cs_scatter_kernel(const R* __restrict__ nodes, Geom g, int n_tiles,
                                                               const int* __restrict__ cnt,
                                                               const int* __restrict__ offsets,
                                                               int* __restrict__ perm, R* __restrict__ ks) {
  extern __shared__ int running[];  // [n_tiles]: nodes of the tile already placed from this block
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) running[i] = 0;
  const int base = blockIdx.x * CS_E;
  const unsigned lt = (1u << lane) - 1u;
  int keys[CS_CHUNKS], rank[CS_CHUNKS], gcount[CS_CHUNKS], pos[CS_CHUNKS];
  bool leader[CS_CHUNKS];
  R kc[CS_CHUNKS][MAX_D];
#pragma unroll
  for (int c = 0; c < CS_CHUNKS; ++c) {
    const int j = base + c * blockDim.x + threadIdx.x;
    bool bad;
    keys[c] = j < g.M ? node_key(nodes, g, j, kc[c], bad) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, keys[c]);
    rank[c] = __popc(peers & lt);
    gcount[c] = __popc(peers);
    leader[c] = lane == __ffs(peers) - 1;
  }
  __syncthreads();
  // groups (chunk c, warp w) in node order; each adds its counts after reading its base
#pragma unroll
  for (int c = 0; c < CS_CHUNKS; ++c) {
    for (int w = 0; w < CS_W; ++w) {
      if (warp == w) {
        if (keys[c] >= 0) pos[c] = running[keys[c]] + rank[c];
        __syncwarp();
        if (keys[c] >= 0 && leader[c]) running[keys[c]] += gcount[c];
      }
      __syncthreads();
    }
  }
  const int* crow = cnt + (long long)blockIdx.x * n_tiles;
#pragma unroll
  for (int c = 0; c < CS_CHUNKS; ++c) {
    if (keys[c] < 0) continue;
    const int p = offsets[keys[c]] + crow[keys[c]] + pos[c];
    perm[p] = base + c * blockDim.x + threadIdx.x;
    for (int d = 0; d < g.D; ++d) ks[(long long)d * g.M + p] = kc[c][d];
  }
}

// ---------------------------------------------------------------- a3 window tables
// beta^tensor_{n_d,d} = 1 / (m phi_Base(m n_d / Ntilde_d)), phi_Base(v) = I0(sqrt(beta^2 - (2 pi v)^2))
// (reading R2). Written in fp64 and in the plan precision.
template <typename T>
__global__ void __launch_bounds__(THREADS) beta_tensor_kernel(Geom g, int ms, double beta0, double beta1, double beta2,
                                                              double* __restrict__ b64, T* __restrict__ bT) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int d = 0, off = i;
  while (d < g.D && off >= g.N[d]) {
    off -= g.N[d];
    ++d;
  }
  if (d >= g.D) return;
  const double beta = d == 0 ? beta0 : (d == 1 ? beta1 : beta2);
  const double n = (double)(off - g.N[d] / 2);
  const double v = (double)ms * n / (double)g.Nt[d];  // ms: window shape m
  const double w = 2.0 * 3.14159265358979323846 * v;
  const double phi = cyl_bessel_i0(sqrt(fma(beta, beta, -w * w)));
  const double bt = 1.0 / ((double)ms * phi);
  b64[i] = bt;
  bT[i] = (T)bt;
}

// Piecewise polynomial window: for tap l (cell a-m+1+l)
// fit p_l(zeta) ~ psi_hat_Base((zeta + 1/2 + m - 1 - l)/m), zeta in [-1/2,1/2],
// by least squares on Theta = 2Z equispaced samples (Householder QR in fp64).
// Samples use the continuous window (limit beta/pi at |u| = 1; R6).
// One thread per (dimension, tap); out[(d*2m + l)*MAX_Z + z].
__global__ void poly_fit_kernel(int D, int m, int ms, int cont, int Z, double beta0, double beta1, double beta2,
                                double* __restrict__ out) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= D * 2 * m) return;
  const int d = id / (2 * m), l = id % (2 * m);
  const double beta = d == 0 ? beta0 : (d == 1 ? beta1 : beta2);
  const int Th = 2 * Z;
  double A[2 * MAX_Z][MAX_Z];
  double b[2 * MAX_Z];
  for (int r = 0; r < Th; ++r) {
    const double zeta = -0.5 + (double)r / (double)(Th - 1);
    double p = 1.0;
    for (int c = 0; c < Z; ++c) {
      A[r][c] = p;
      p *= zeta;
    }
    // m taps per half (the footprint), scale ms (the window shape); cont: the 2m+2 variant samples the
    // analytic continuation sin(beta s)/(pi s), s = sqrt(u^2 - 1), beyond |u| = 1
    const double u = (zeta + 0.5 + (double)(m - 1 - l)) / (double)ms;
    const double s2 = 1.0 - u * u;
    double val;
    if (s2 < 0.0 && cont) {
      const double s = sqrt(-s2);
      val = sin(beta * s) / (3.14159265358979323846 * s);
    } else if (s2 <= 0.0) {
      val = fabs(u) <= 1.0 ? beta / 3.14159265358979323846 : 0.0;
    } else {
      const double s = sqrt(s2);
      val = sinh(beta * s) / (3.14159265358979323846 * s);
    }
    b[r] = val;
  }
  // Householder QR, applying reflections to b as we go
  for (int c = 0; c < Z; ++c) {
    double nrm = 0.0;
    for (int r = c; r < Th; ++r) nrm += A[r][c] * A[r][c];
    nrm = sqrt(nrm);
    const double alpha = A[c][c] > 0 ? -nrm : nrm;
    double v0 = A[c][c] - alpha;
    // v = [v0, A[c+1..][c]]; H = I - 2 v v^T / (v^T v)
    double vtv = v0 * v0;
    for (int r = c + 1; r < Th; ++r) vtv += A[r][c] * A[r][c];
    if (vtv == 0.0) continue;
    for (int cc = c + 1; cc < Z; ++cc) {
      double s = v0 * A[c][cc];
      for (int r = c + 1; r < Th; ++r) s += A[r][c] * A[r][cc];
      s = 2.0 * s / vtv;
      A[c][cc] -= s * v0;
      for (int r = c + 1; r < Th; ++r) A[r][cc] -= s * A[r][c];
    }
    {
      double s = v0 * b[c];
      for (int r = c + 1; r < Th; ++r) s += A[r][c] * b[r];
      s = 2.0 * s / vtv;
      b[c] -= s * v0;
      for (int r = c + 1; r < Th; ++r) b[r] -= s * A[r][c];
    }
    A[c][c] = alpha;
  }
  // back substitution R mu = (Q^T b)[0..Z)
  double mu[MAX_Z];
  for (int c = Z - 1; c >= 0; --c) {
    double s = b[c];
    for (int cc = c + 1; cc < Z; ++cc) s -= A[c][cc] * mu[cc];
    mu[c] = s / A[c][c];
  }
  for (int c = 0; c < MAX_Z; ++c) out[(long long)id * MAX_Z + c] = c < Z ? mu[c] : 0.0;
}

}  // namespace nfftb
