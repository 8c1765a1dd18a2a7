// precompute.cuh — node binning, stable radix sort into tiles, subproblems
// and window tables. All device kernels.
//
// PAPER.md:520-537 (block partition R_p, Gamma_p, Q = ceil(Ntilde/P)),
// PAPER.md:512 (fixed maximum number of nodes per block for balance),
// PAPER.md:439-441 (beta^tensor), PAPER.md:628-642 (polynomial window table).
#pragma once

#include "common.cuh"

namespace nfftb {

constexpr int SORT_ITEMS = 8;
constexpr int SORT_TILE = THREADS * SORT_ITEMS;  // 2048 keys per block
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = THREADS * SCAN_ITEMS;

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

// ---------------------------------------------------------------- a1+a2: stable counting sort (3 kernels)
// Block b of the sort owns nodes [b*E, (b+1)*E), E = 32 * W * CS_CHUNKS (W warps).
// K1 counts tiles per block; K2 scans the [tile][block] counts (warp per tile)
// and its last CTA scans the tile totals into the tile offsets and writes the
// subproblem list; K3 re-walks each block in node order and places every node
// at offsets[tile] + (nodes of that tile in earlier blocks) + (earlier nodes of
// that tile in this block) — a stable counting sort, so perm is the unique
// "tile ascending, original index ascending" order (reading R12). K3 also
// writes the tile-sorted SoA coordinates.
constexpr int CS_CHUNKS = 8;  // 32-node chunks per warp

template <typename R>
__global__ void cs_count_kernel(const R* __restrict__ nodes, Geom g, int n_tiles, int E, int nblk,
                                int* __restrict__ cnt, int* __restrict__ err, unsigned* __restrict__ ticket) {
  extern __shared__ int hist[];
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  const int base = blockIdx.x * E;
  bool any_bad = false;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int j = base + e;
    if (j >= g.M) break;
    R k[MAX_D];
    bool bad;
    const int key = node_key(nodes, g, j, k, bad);
    any_bad |= bad;
    atomicAdd(&hist[key], 1);
  }
  if (any_bad) atomicOr(err, 1);
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) cnt[(long long)t * nblk + blockIdx.x] = hist[t];
  if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0u;
}

__global__ void __launch_bounds__(THREADS) cs_scan_kernel(int* __restrict__ cnt, int n_tiles, int nblk, int M,
                                                          int* __restrict__ tile_total, int* __restrict__ offsets,
                                                          unsigned* __restrict__ ticket, int nb, int ne, int S,
                                                          int* __restrict__ subbase, int4* __restrict__ subs) {
  __shared__ int ws[32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * (blockDim.x >> 5) + warp;
  if (t < n_tiles) {
    int* row = cnt + (long long)t * nblk;
    const int per = (nblk + 31) / 32;
    const int lo = lane * per, hi = min(nblk, lo + per);
    int s = 0;
    for (int i = lo; i < hi; ++i) s += row[i];
    int inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    int run = inc - s;
    for (int i = lo; i < hi; ++i) {
      const int c = row[i];
      row[i] = run;
      run += c;
    }
    if (lane == 31) tile_total[t] = inc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last CTA: tile offsets = exclusive scan of the tile totals
  {
    const int per = (n_tiles + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(n_tiles, lo + per);
    int s = 0;
    for (int i = lo; i < hi; ++i) s += __ldcg(tile_total + i);
    int total;
    int run = block_exclusive_scan(s, ws, total);
    for (int i = lo; i < hi; ++i) {
      offsets[i] = run;
      run += __ldcg(tile_total + i);
    }
    if (threadIdx.x == 0) offsets[n_tiles] = M;
  }
  __syncthreads();
  // subproblems: shard [nb, ne) of each tile cut into chunks of <= S nodes
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
__global__ void cs_scatter_kernel(const R* __restrict__ nodes, Geom g, int n_tiles, int E, int nblk,
                                  const int* __restrict__ cnt, const int* __restrict__ offsets,
                                  int* __restrict__ perm, R* __restrict__ ks) {
  extern __shared__ int wb[];  // [W][n_tiles]
  const int W = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < W * n_tiles; i += blockDim.x) wb[i] = 0;
  __syncthreads();
  const int base = blockIdx.x * E + warp * 32 * CS_CHUNKS;
  int keys[CS_CHUNKS];
  R kc[CS_CHUNKS][MAX_D];
  int* mine = wb + warp * n_tiles;
#pragma unroll
  for (int c = 0; c < CS_CHUNKS; ++c) {
    const int j = base + c * 32 + lane;
    bool bad;
    keys[c] = j < g.M ? node_key(nodes, g, j, kc[c], bad) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, keys[c]);
    if (keys[c] >= 0 && lane == __ffs(peers) - 1) mine[keys[c]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    int run = offsets[t] + cnt[(long long)t * nblk + blockIdx.x];
    for (int w = 0; w < W; ++w) {
      const int c = wb[w * n_tiles + t];
      wb[w * n_tiles + t] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int c = 0; c < CS_CHUNKS; ++c) {
    const int key = keys[c];
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    int pos = 0;
    if (key >= 0) pos = mine[key] + __popc(peers & lt);
    __syncwarp();
    if (key >= 0 && lane == __ffs(peers) - 1) mine[key] += __popc(peers);
    __syncwarp();
    if (key >= 0) {
      perm[pos] = base + c * 32 + lane;
      for (int d = 0; d < g.D; ++d) ks[(long long)d * g.M + pos] = kc[c][d];
    }
  }
}

// ---------------------------------------------------------------- a1 binning (radix fallback path)
// key_j = C-order linear tile id of the cell node j starts from; vals_j = j.
template <typename R>
__global__ void __launch_bounds__(THREADS) bin_nodes_kernel(const R* __restrict__ nodes, Geom g,
                                                            int* __restrict__ keys, int* __restrict__ vals,
                                                            int* __restrict__ err) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.M) return;
  int key = 0;
  bool bad = false;
  for (int d = 0; d < g.D; ++d) {
    const double k = (double)nodes[(long long)j * g.D + d];
    if (!isfinite(k)) {
      bad = true;
      continue;
    }
    double frac;
    const int c = node_cell(k, g.Ntd[d], g.Nt[d], frac);
    key = key * g.P[d] + c / g.Q[d];
  }
  if (bad) {
    atomicOr(err, 1);
    key = 0;
  }
  keys[j] = key;
  vals[j] = j;
}

// ---------------------------------------------------------------- scan
// Exclusive scan of int arrays (in may equal out). Block sums go to `sums`.
__global__ void __launch_bounds__(THREADS) scan_tile_kernel(const int* in, int* out, int n, int* sums) {
  __shared__ int ws[32];
  const long long base = (long long)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  int s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  int total;
  int run = block_exclusive_scan(s, ws, total);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (sums != nullptr && threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(THREADS) scan_add_kernel(int* out, int n, const int* offs) {
  const int add = offs[blockIdx.x];
  const long long base = (long long)blockIdx.x * SCAN_TILE;
  for (int i = threadIdx.x; i < SCAN_TILE; i += blockDim.x)
    if (base + i < n) out[base + i] += add;
}

// ---------------------------------------------------------------- a2 radix sort
// Stable LSD radix sort of (key, val) by key, 8-bit digits. Pass: per-block
// digit histogram -> exclusive scan over [digit][block] -> stable scatter with
// a block-local stable split sort. Stability makes the permutation the unique
// "tile ascending, original index ascending" order (reading R12).
__global__ void __launch_bounds__(THREADS) radix_hist_kernel(const int* __restrict__ keys, int n, int shift,
                                                             int nblocks, int* __restrict__ hist) {
  __shared__ int cnt[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * SORT_TILE;
  for (int i = threadIdx.x; i < SORT_TILE; i += blockDim.x)
    if (base + i < n) atomicAdd(&cnt[(keys[base + i] >> shift) & 255], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i * nblocks + blockIdx.x] = cnt[i];
}

__global__ void __launch_bounds__(THREADS) radix_scatter_kernel(const int* __restrict__ kin, const int* __restrict__ vin,
                                                                int* __restrict__ kout, int* __restrict__ vout, int n,
                                                                int shift, int bits, int nblocks,
                                                                const int* __restrict__ offs) {
  __shared__ int sk[SORT_TILE];
  __shared__ int sv[SORT_TILE];
  __shared__ int ws[32];
  __shared__ int dstart[256];
  const int tid = threadIdx.x;
  const long long base = (long long)blockIdx.x * SORT_TILE;
  const int dmask = (1 << bits) - 1;
  int k[SORT_ITEMS], v[SORT_ITEMS];
#pragma unroll
  for (int i = 0; i < SORT_ITEMS; ++i) {
    const long long idx = base + tid * SORT_ITEMS + i;
    if (idx < n) {
      k[i] = kin[idx];
      v[i] = vin[idx];
    } else {  // padding sorts last (max digit, after real elements)
      k[i] = dmask << shift;
      v[i] = -1;
    }
  }
  // block-local stable sort by digit: `bits` one-bit stable splits (LSD)
  for (int b = 0; b < bits; ++b) {
    int zeros = 0;
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) zeros += 1 - ((k[i] >> (shift + b)) & 1);
    int Z;
    const int zb = block_exclusive_scan(zeros, ws, Z);
    int zrun = 0;
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
      const int f = (k[i] >> (shift + b)) & 1;
      const int before = tid * SORT_ITEMS + i;
      const int pos = f ? Z + (before - zb - zrun) : zb + zrun;
      zrun += 1 - f;
      sk[pos] = k[i];
      sv[pos] = v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
      k[i] = sk[tid * SORT_ITEMS + i];
      v[i] = sv[tid * SORT_ITEMS + i];
    }
    __syncthreads();
  }
  // local start of every digit: elements are now sorted by digit
  for (int i = tid; i < 256; i += blockDim.x) dstart[i] = 0x7fffffff;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SORT_ITEMS; ++i) {
    if (v[i] >= 0) atomicMin(&dstart[(k[i] >> shift) & 255], tid * SORT_ITEMS + i);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SORT_ITEMS; ++i) {
    if (v[i] < 0) continue;
    const int dg = (k[i] >> shift) & 255;
    const int rank = tid * SORT_ITEMS + i - dstart[dg];
    const int pos = offs[dg * nblocks + blockIdx.x] + rank;
    kout[pos] = k[i];
    vout[pos] = v[i];
  }
}

// Tile offsets from sorted keys: offsets[t] = first sorted position with key >= t.
__global__ void __launch_bounds__(THREADS) tile_offsets_kernel(const int* __restrict__ skeys, int n, int n_tiles,
                                                               int* __restrict__ offsets) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  const int lo = i == 0 ? 0 : skeys[i - 1] + 1;
  const int hi = i == n ? n_tiles : skeys[i];
  for (int t = lo; t <= hi; ++t) offsets[t] = i;
}

// Sorted SoA coordinates ks[d][i] = nodes[perm[i]][d].
template <typename R>
__global__ void __launch_bounds__(THREADS) gather_sorted_kernel(const R* __restrict__ nodes, const int* __restrict__ perm,
                                                                Geom g, R* __restrict__ ks) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.M) return;
  const int j = perm[i];
  for (int d = 0; d < g.D; ++d) ks[(long long)d * g.M + i] = nodes[(long long)j * g.D + d];
}

// Subproblems: the part of tile t inside the shard [nb, ne) of the sorted order,
// cut into chunks of at most S nodes.
__global__ void __launch_bounds__(THREADS) count_subproblems_kernel(const int* __restrict__ offsets, int n_tiles, int nb,
                                                                    int ne, int S, int* __restrict__ nsub) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > n_tiles) return;
  if (t == n_tiles) {
    nsub[t] = 0;
    return;
  }
  const int s = max(offsets[t], nb), e = min(offsets[t + 1], ne);
  const int c = max(0, e - s);
  nsub[t] = (c + S - 1) / S;
}

__global__ void __launch_bounds__(THREADS) write_subproblems_kernel(const int* __restrict__ offsets, int n_tiles, int nb,
                                                                    int ne, int S, const int* __restrict__ subbase,
                                                                    int4* __restrict__ subs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const int s = max(offsets[t], nb), e = min(offsets[t + 1], ne);
  int q = subbase[t];
  for (int st = s; st < e; st += S) subs[q++] = make_int4(t, st, min(S, e - st), 0);
}

// ---------------------------------------------------------------- a3 window tables
// beta^tensor_{n_d,d} = 1 / (m phi_Base(m n_d / Ntilde_d)), phi_Base(v) = I0(sqrt(beta^2 - (2 pi v)^2))
// (reading R2). Written in fp64 and in the plan precision.
template <typename T>
__global__ void __launch_bounds__(THREADS) beta_tensor_kernel(Geom g, double beta0, double beta1, double beta2,
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
  const double v = (double)g.m * n / (double)g.Nt[d];
  const double w = 2.0 * 3.14159265358979323846 * v;
  const double phi = cyl_bessel_i0(sqrt(fma(beta, beta, -w * w)));
  const double bt = 1.0 / ((double)g.m * phi);
  b64[i] = bt;
  bT[i] = (T)bt;
}

// Piecewise polynomial window: for tap l (cell a-m+1+l)
// fit p_l(zeta) ~ psi_hat_Base((zeta + 1/2 + m - 1 - l)/m), zeta in [-1/2,1/2],
// by least squares on Theta = 2Z equispaced samples (Householder QR in fp64).
// Samples use the continuous window (limit beta/pi at |u| = 1; R6).
// One thread per (dimension, tap); out[(d*2m + l)*MAX_Z + z].
__global__ void poly_fit_kernel(int D, int m, int Z, double beta0, double beta1, double beta2, double* __restrict__ out) {
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
    const double u = (zeta + 0.5 + (double)(m - 1 - l)) / (double)m;
    const double s2 = 1.0 - u * u;
    double val;
    if (s2 <= 0.0) {
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
