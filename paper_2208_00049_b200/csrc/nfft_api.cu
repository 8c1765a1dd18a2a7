// nfft_api.cu — plan object, orchestration and the C ABI of include/nfft.h.
//
// Host side of the B200 NFFT: validates the geometry,
// owns every device buffer (the paper's plan as preallocated state,
// PAPER.md:374-382), builds the window tables and cuFFT plan once, and
// enqueues the kernels of precompute.cuh / grid.cuh / resample.cuh on the
// plan stream. Nothing here computes on the host except geometry and launch
// configuration.
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/nfft.h"
#include "common.cuh"
#include "dispatch.cuh"
#include "grid.cuh"
#include "precompute.cuh"
#include "binsort.cuh"
#include "cellbin.cuh"
#include "resample1d.cuh"
#include "resample_nd.cuh"
#include "resample_cell.cuh"
#include "resample_rowbatch.cuh"
#include "resample_wblock.cuh"
#include "resample_full.cuh"

using namespace nfftb;

struct nfft_plan_s;
template <typename T> const KernelSet<T>& kernels_of(const nfft_plan_s* p);
template <typename T> const WinPoly<T>& poly_of(const nfft_plan_s* p);

struct nfft_plan_s {
  int D = 0;
  int64_t N[3] = {1, 1, 1}, Nt[3] = {1, 1, 1}, Q[3] = {1, 1, 1}, P[3] = {1, 1, 1};
  int64_t M = 0, B = 1;
  int m = 0;
  double sigma = 0;
  double beta[3] = {0, 0, 0};
  nfft_precision prec = NFFT_COMPLEX128;
  nfft_options opt{};
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  bool tiled = true;
  int S = 256;            // max nodes per subproblem
  int node_begin = 0, node_end = 0;
  int64_t n_tiles = 1;
  int deg = 14;
  int m_shape = 0;  // window shape parameter m (the kernels' half-width p->m is m + 1 for 2m+2 points)
  int max_subs = 1;
  int grid_tiled = 1;     // CTAs for the tiled kernels
  int grid_loc = 0;       // CTAs for the conflict-free spread (0: not used)
  size_t loc_bytes = 0;
  int grid_own = 0;       // CTAs for the owner-computes spread (0: not used)
  size_t own_bytes = 0;
  int grid_sorted = 0;    // CTAs for the cell-sorted warp-chunk spread (0: not used)
  size_t sorted_bytes = 0;
  int grid_gather = 0;    // CTAs for the cell-gather spread (0: not used)
  size_t gather_bytes = 0;
  int grid_direct = 1;
  size_t region_bytes = 0;
  Geom geom{};
  WinPoly<double> wp64{};
  WinPoly<float> wp32{};
  alignas(16) unsigned char wpn[sizeof(WinPoly<double>)] = {};  // the table cut to (D, m, degree): WinPolyN
  KernelSet<double> k64{};
  KernelSet<float> k32{};
  // device buffers
  void* d_nodes = nullptr;   // M*D reals (plan precision)
  void* d_ks = nullptr;      // D*M sorted reals
  int* d_perm = nullptr;     // M: node index of every tile-sorted position
  int* d_offsets = nullptr;  // n_tiles + 1
  int* d_subbase = nullptr;  // n_tiles + 1 (last = number of subproblems)
  int4* d_subs = nullptr;
  int* d_err = nullptr;
  int* d_cnt = nullptr;        // [cs_nblk][n_tiles] per-block tile counts (then their prefixes)
  int* d_tile_total = nullptr; // n_tiles
  unsigned* d_ticket = nullptr;
  int cs_nblk = 1;
  bool use_bs = false;    // one cooperative binsort kernel (binsort.cuh) instead of cs_count/scan/scatter
  int bs_grid = 0, bs_rr = 1;
  size_t bs_bytes = 0;
  bool use_ind = false;   // D = 2, 3 static-tile interpolation (resample_nd.cuh)
  // cell mode (AUTO/TILED): nodes sorted by cell (cellbin.cuh), work tiles defined by the kernels
  bool cellmode = false;
  bool tile_binned = false;  // cell mode: perm/offsets (tile sort) computed on demand for nfft_get_binning
  int64_t ncells = 0;        // prod Ntilde
  size_t r1_spread_bytes = 0; // spread1a shared memory
  size_t r1_interp_bytes = 0; // interp1s shared memory
  size_t sc_bytes = 0;       // spread_cell shared memory
  int sc_cap = 0;            // spread_cell node slots per chunk
  void* d_kc = nullptr;      // D*M reals: coordinates in cell order (SoA)
  bool tensor = false;       // TENSOR precompute (cell mode): the 2m D taps of every node stored in cell order
  bool full = false;         // FULL precompute (cell mode): the rows of the sparse matrix B stored in cell order
  int full_e = 0;            // entries per row, (2m)^D
  void* d_bw = nullptr;      // FULL: M * E weights (plan precision)
  int* d_bi = nullptr;       // FULL: M * E grid indices
  bool batchmode = false;    // D = 2 cell mode, B >= 8: row-segment spread with lanes = batch vectors
  int bp = 0;                // batch padded to a multiple of 32
  void* d_fT = nullptr;      // M * bp complex: node values, transposed (node-major)
  size_t rb_bytes = 0;
  int rb_occ = 1;            // resident spread_rb2 CTAs per SM (persistent launch width)
  bool cell2 = false;        // fp32 2D batches: interp_cell2 (two vectors per CTA)
  bool wbmode = false;       // D = 2, 3 cell mode: warp-owned cell blocks over the TENSOR taps (resample_wblock.cuh)
  size_t wb_bytes = 0;
  void* d_fc = nullptr;      // B * M complex: node values in cell order (warp-block adjoint)
  int* d_inv = nullptr;      // M: cell-sorted position of every node (batch adjoint)
  int* d_cl = nullptr;       // M: last-dimension cell of every cell-sorted position

  void* d_wt = nullptr;      // M * 2m reals: taps of every cell-sorted position
  int* d_jc = nullptr;       // M: node index of every cell-sorted position
  int* d_cstart = nullptr;   // ncells + 1: first cell-sorted position of every cell
  int* d_ccount = nullptr;   // ncells: per-cell counters (zero between precomputes)
  int* d_cslot = nullptr;    // M: slot inside the cell per node; scratch of cl_fix
  unsigned long long* d_scan_status = nullptr;  // cl_scan look-back state per 4096-cell tile
  int* d_ctr = nullptr;      // [scan ticket, #small cells, #big cells, -]
  int* d_big = nullptr;      // cells with more than CL_SMALL nodes (cl_fix)
  void* d_grid_in = nullptr;  // B * prod Nt complex: forward input, zero padding persists
  void* d_grid = nullptr;     // B * prod Nt complex: forward FFT output (read by interp)
  void* d_grid_adj = nullptr; // B * prod Nt complex: adjoint grid, all zero between adjoints
  double* d_beta64 = nullptr;
  void* d_betaT = nullptr;
  double* d_poly = nullptr;  // D*2m*MAX_Z
  void* d_stage_grid = nullptr;   // B * prod N complex (host-pointer staging)
  void* d_stage_nodes = nullptr;
  void* d_stage_nodes2 = nullptr;  // nfft_execute: the adjoint chain's host-input staging
  void* d_stage_grid2 = nullptr;   // nfft_execute: the adjoint chain's host-output staging
  cufftHandle fft = 0;      // forward: out-of-place grid_in -> grid
  bool fft_ok = false;
  cufftHandle fft_adj = 0;  // adjoint: in place on grid_adj (own plan: may run concurrently)
  bool fft_adj_ok = false;
  cudaStream_t side_pre = nullptr, side_adj = nullptr;  // nfft_execute's internal streams
  cudaEvent_t ev_fork = nullptr, ev_pre = nullptr, ev_adj = nullptr;
  bool precomputed = false;
  cudaEvent_t ev[3][6] = {};
  bool events = false;
  int last_dir = 0;          // 0 forward, 1 adjoint: the most recent call (nfft_get_stage_times)
  int64_t launches = 0;
  size_t csize() const { return prec == NFFT_COMPLEX128 ? 16 : 8; }
  size_t rsize() const { return prec == NFFT_COMPLEX128 ? 8 : 4; }
};

template <> const KernelSet<double>& kernels_of<double>(const nfft_plan_s* p) { return p->k64; }
template <> const KernelSet<float>& kernels_of<float>(const nfft_plan_s* p) { return p->k32; }
template <> const WinPoly<double>& poly_of<double>(const nfft_plan_s* p) { return p->wp64; }
template <> const WinPoly<float>& poly_of<float>(const nfft_plan_s* p) { return p->wp32; }

namespace {

#define CK(call)                                    \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) {                        \
      last_cuda_error = e_;                         \
      return NFFT_ERROR_CUDA;                       \
    }                                               \
  } while (0)

#define CKL()                                       \
  do {                                              \
    cudaError_t e_ = cudaGetLastError();            \
    if (e_ != cudaSuccess) {                        \
      last_cuda_error = e_;                         \
      return NFFT_ERROR_CUDA;                       \
    }                                               \
  } while (0)

thread_local cudaError_t last_cuda_error = cudaSuccess;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool is_device_pointer(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void free_all(nfft_plan p) {
  void* bufs[] = {p->d_nodes, p->d_ks, p->d_offsets, p->d_subbase, p->d_subs, p->d_err, p->d_grid, p->d_grid_in, p->d_grid_adj, p->d_beta64,
                  p->d_betaT, p->d_poly, p->d_stage_grid, p->d_stage_nodes, p->d_stage_nodes2, p->d_stage_grid2, p->d_cnt, p->d_tile_total,
                  p->d_ticket, p->d_perm, p->d_kc, p->d_jc, p->d_cstart, p->d_ccount, p->d_cslot,
                  p->d_scan_status, p->d_ctr, p->d_big, p->d_wt, p->d_fT, p->d_fc, p->d_cl, p->d_inv, p->d_bw,
                  p->d_bi};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (p->fft_ok) cufftDestroy(p->fft);
  if (p->fft_adj_ok) cufftDestroy(p->fft_adj);
  for (cudaEvent_t e : {p->ev_fork, p->ev_pre, p->ev_adj})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t st : {p->side_pre, p->side_adj})
    if (st) cudaStreamDestroy(st);
  if (p->events)
    for (auto& row : p->ev)
      for (auto& e : row)
        if (e) cudaEventDestroy(e);
}

inline void rec(nfft_plan p, int which, int slot) {
  if (p->events) cudaEventRecord(p->ev[which][slot], p->stream);
}

// Launches a kernel taken by pointer (KernelSet members typed const void*); the
// arguments are passed by address, the window table as the plan's packed
// WinPolyN bytes (the runtime copies the kernel's parameter size from it).
struct WpnArg {
  const unsigned char* bytes;
};
template <typename A>
inline void* arg_ptr(A& a) {
  return (void*)&a;
}
inline void* arg_ptr(WpnArg& a) { return (void*)a.bytes; }
template <typename... A>
cudaError_t launch_k(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... a) {
  void* args[] = {arg_ptr(a)...};
  return cudaLaunchKernel(fn, grid, block, args, smem, st);
}
// The same with programmatic dependent launch: the kernel may start before the previous kernel on the
// stream has finished and waits (griddepcontrol.wait) before it reads that kernel's output, so its
// independent prologue (node loads) and launch overlap the previous kernel's tail (the FFT).
template <typename... A>
cudaError_t launch_k_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... a) {
  void* args[] = {arg_ptr(a)...};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

template <typename T>
nfft_status build_window_tables(nfft_plan p) {
  const int n = (int)(p->N[0] + (p->D > 1 ? p->N[1] : 0) + (p->D > 2 ? p->N[2] : 0));
  beta_tensor_kernel<T><<<(n + THREADS - 1) / THREADS, THREADS, 0, p->stream>>>(
      p->geom, p->m_shape, p->beta[0], p->beta[1], p->beta[2], p->d_beta64, (T*)p->d_betaT);
  ++p->launches;
  CKL();
  const int nfit = p->D * 2 * p->m;
  poly_fit_kernel<<<(nfit + 63) / 64, 64, 0, p->stream>>>(p->D, p->m, p->m_shape, p->m != p->m_shape, p->deg + 1,
                                                          p->beta[0], p->beta[1], p->beta[2], p->d_poly);
  ++p->launches;
  CKL();
  const size_t cnt = (size_t)nfit * MAX_Z;
  double* host = new (std::nothrow) double[cnt];
  if (!host) return NFFT_ERROR_OUT_OF_MEMORY;
  cudaError_t e = cudaMemcpyAsync(host, p->d_poly, cnt * sizeof(double), cudaMemcpyDeviceToHost, p->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) {
    delete[] host;
    last_cuda_error = e;
    return NFFT_ERROR_CUDA;
  }
  memset(&p->wp64, 0, sizeof(p->wp64));
  memset(&p->wp32, 0, sizeof(p->wp32));
  for (int d = 0; d < p->D; ++d)
    for (int l = 0; l < p->m; ++l)
      for (int z = 0; z < MAX_Z; ++z) {
        const double v = host[((size_t)d * 2 * p->m + l) * MAX_Z + z];
        p->wp64.mu[d][l][z] = v;
        p->wp32.mu[d][l][z] = (float)v;
      }
  delete[] host;
  // packed [d][l][z] table for the kernels' WinPolyN<T, D, m> parameter (z <= degree)
  const int Z = p->deg + 1;
  for (int d = 0; d < p->D; ++d)
    for (int l = 0; l < p->m; ++l)
      for (int z = 0; z < Z; ++z) {
        const size_t i = ((size_t)d * p->m + l) * Z + z;
        if (sizeof(T) == 8) reinterpret_cast<double*>(p->wpn)[i] = p->wp64.mu[d][l][z];
        else reinterpret_cast<float*>(p->wpn)[i] = p->wp32.mu[d][l][z];
      }
  return NFFT_SUCCESS;
}

template <typename T>
nfft_status configure_kernels(nfft_plan p, const KernelSet<T>& ks) {
  if (p->tiled) {
    const void* fns[2] = {(const void*)ks.interp_tiled, (const void*)ks.spread_tiled};
    int occ_min = 1 << 30;
    for (const void* fn : fns) {
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->region_bytes));
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, THREADS, p->region_bytes));
      if (occ < 1) return NFFT_ERROR_BAD_TILE;
      occ_min = std::min(occ_min, occ);
    }
    p->grid_tiled = (int)std::max<int64_t>(1, std::min<int64_t>(p->max_subs, (int64_t)occ_min * p->sm_count));
    p->grid_gather = 0;
    if (ks.spread_gather && (p->opt.method <= NFFT_METHOD_TILED || p->opt.method == NFFT_METHOD_TILED_V1)) {
      int tile_cells = 1;
      for (int d = 0; d < p->D; ++d) tile_cells *= (int)p->Q[d];
      const size_t bytes = gather_smem_bytes(p->D, p->m, p->csize(), p->rsize(), tile_cells, p->S);
      int occ = 0;
      if (bytes <= 227 * 1024 &&
          cudaFuncSetAttribute((const void*)ks.spread_gather, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)bytes) == cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)ks.spread_gather, THREADS, bytes) ==
              cudaSuccess &&
          occ >= 1) {
        p->gather_bytes = bytes;
        p->grid_gather = (int)std::max<int64_t>(1, std::min<int64_t>(p->max_subs, (int64_t)occ * p->sm_count));
      }
      cudaGetLastError();
    }
    p->grid_sorted = 0;
    if (p->opt.method == NFFT_METHOD_TILED_SORTED ||
        ((p->opt.method <= NFFT_METHOD_TILED || p->opt.method == NFFT_METHOD_TILED_V1) && p->D == 3)) {
      int tile_cells = 1;
      for (int d = 0; d < p->D; ++d) tile_cells *= (int)p->Q[d];
      const size_t bytes = p->region_bytes + (size_t)(tile_cells + 1 + THREADS + 17) * 4;
      int occ = 0;
      if (bytes <= 227 * 1024 &&
          cudaFuncSetAttribute((const void*)ks.spread_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)bytes) == cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)ks.spread_sorted, THREADS, bytes) ==
              cudaSuccess &&
          occ >= 1) {
        p->sorted_bytes = bytes;
        p->grid_sorted = (int)std::max<int64_t>(1, std::min<int64_t>(p->max_subs, (int64_t)occ * p->sm_count));
      }
      cudaGetLastError();
    }
    p->grid_loc = 0;
    if (ks.spread_loc && p->opt.method == NFFT_METHOD_TILED_LOC) {
      int nst = 1;
      for (int d = 0; d < p->D; ++d) nst *= (int)((p->Q[d] + 2 * p->m - 1) / (2 * p->m));
      const size_t bytes = loc_smem_bytes(p->D, p->m, p->csize(), p->rsize(), p->geom.region_cells, p->S, nst);
      int occ = 0;
      if (bytes <= 227 * 1024 &&
          cudaFuncSetAttribute((const void*)ks.spread_loc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) ==
              cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)ks.spread_loc, ks.loc_threads, bytes) ==
              cudaSuccess &&
          occ >= 1) {
        p->loc_bytes = bytes;
        p->grid_loc = (int)std::max<int64_t>(1, std::min<int64_t>(p->max_subs, (int64_t)occ * p->sm_count));
      }
      cudaGetLastError();
    }
    p->grid_own = 0;
    bool own_ok = ks.spread_own != nullptr && p->opt.method == NFFT_METHOD_TILED_OWN;
    int tile_cells = 1, nstx = 1;
    for (int d = 0; d < p->D && own_ok; ++d) {
      own_ok = p->P[d] >= 3 && p->Nt[d] % p->Q[d] == 0 && p->Q[d] >= 2 * p->m;
      tile_cells *= (int)p->Q[d];
      nstx *= (int)((p->Q[d] + 2 * p->m - 1) / (2 * p->m) + 2);
    }
    if (own_ok) {
      const size_t bytes = own_smem_bytes(p->D, p->m, p->csize(), p->rsize(), tile_cells, ks.own_threads, nstx);
      int occ = 0;
      if (bytes <= 227 * 1024 &&
          cudaFuncSetAttribute((const void*)ks.spread_own, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) ==
              cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)ks.spread_own, ks.own_threads, bytes) ==
              cudaSuccess &&
          occ >= 1) {
        p->own_bytes = bytes;
        p->grid_own = (int)std::max<int64_t>(1, std::min<int64_t>(p->n_tiles, (int64_t)occ * p->sm_count));
      }
      cudaGetLastError();
    }
  }
  p->grid_direct = p->sm_count * 8;
  bool sc_ok = true;  // spread_cell fallback configured (D >= 2 cell mode)
  if (p->cellmode) {
    bool ok = false;
    if (p->D == 1 && ks.interp1 && ks.spread1) {
      const size_t sb = s1_smem_bytes(p->m, p->csize(), p->rsize());
      const size_t ib = i1_smem_bytes(p->m, p->csize());
      int occ_s = 0, occ_t = 0, occ_i = 0;
      ok = cudaFuncSetAttribute((const void*)ks.spread1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb) ==
               cudaSuccess &&
           cudaFuncSetAttribute((const void*)ks.spread1t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb) ==
               cudaSuccess &&
           cudaFuncSetAttribute((const void*)ks.interp1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ib) ==
               cudaSuccess &&
           cudaFuncSetAttribute((const void*)ks.interp1t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ib) ==
               cudaSuccess &&
           cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, (const void*)ks.spread1, S1_THREADS, sb) == cudaSuccess &&
           cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, (const void*)ks.spread1t, S1_THREADS, sb) == cudaSuccess &&
           cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_i, (const void*)ks.interp1, I1_THREADS, ib) == cudaSuccess &&
           occ_s >= 1 && occ_t >= 1 && occ_i >= 1;
      p->r1_spread_bytes = sb;
      p->r1_interp_bytes = ib;
    }
    if (p->D >= 2 && ks.interp_cell && ks.spread_cell) {
      int wrows = 1;
      for (int d = 0; d < p->D - 1; ++d) wrows *= (int)(p->Q[d] + 2 * p->m - 1);
      const int wcols = (int)(p->Q[p->D - 1] + 2 * p->m - 1);
      const int TL = ((2 * p->m + 2 * SC_K - 2) + 1) & ~1;
      const size_t slot = ((size_t)(p->D - 1) * 2 * p->m + TL + 2) * p->rsize() + 4;
      const size_t fixed = spread_cell_smem_bytes(p->D, p->m, (int)p->rsize(), 0, wrows, wcols) + 64;
      const size_t budget = p->D == 2 ? 110 * 1024 : 200 * 1024;
      int nitems = (int)((p->Q[p->D - 1] + SC_K - 1) / SC_K);
      int nrows = 1;
      for (int d = 0; d < p->D - 1; ++d) {
        nitems *= (int)p->Q[d];
        nrows *= (int)p->Q[d];
      }
      int cap = fixed < budget ? (int)std::min<size_t>(2048, (budget - fixed) / slot) : 0;
      const size_t sb = spread_cell_smem_bytes(p->D, p->m, (int)p->rsize(), cap, wrows, wcols);
      int occ_i = 0, occ_s = 0;
      const bool interp_ok = nrows <= 1024 && p->region_bytes <= 200 * 1024 &&
                             cudaFuncSetAttribute((const void*)ks.interp_cell, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)p->region_bytes) == cudaSuccess &&
                             cudaFuncSetAttribute((const void*)ks.interp_cellt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)p->region_bytes) == cudaSuccess &&
                             cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_i, (const void*)ks.interp_cell, RC_THREADS,
                                                                           p->region_bytes) == cudaSuccess &&
                             occ_i >= 1;
      sc_ok = cap >= 32 && nitems <= 512 &&
              cudaFuncSetAttribute((const void*)ks.spread_cell, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb) ==
                  cudaSuccess &&
              cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, (const void*)ks.spread_cell, 256, sb) == cudaSuccess &&
              occ_s >= 1;
      // the spread_cell fallback's limits only matter when neither the warp-block nor the batch adjoint
      // takes the plan (checked again below, after those are configured)
      ok = interp_ok && (sc_ok || p->wbmode || p->batchmode || p->full);
      p->sc_cap = cap;
      p->sc_bytes = sb;
    }
    cudaGetLastError();
    p->cellmode = ok;
    if (!ok) p->tensor = p->full = false;
  }
  if (p->batchmode) {
    bool ok = p->cellmode && ks.spread_rb2;
    if (ok) {
      p->rb_bytes = rb2_smem_bytes(p->m, (int)p->rsize());
      int o = 0;
      ok = cudaFuncSetAttribute((const void*)ks.spread_rb2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)p->rb_bytes) == cudaSuccess &&
           cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, (const void*)ks.spread_rb2, 32 * RB2_WARPS, p->rb_bytes) ==
               cudaSuccess &&
           o >= 1;
      p->rb_occ = o;
      cudaGetLastError();
    }
    p->batchmode = ok;
  }
  // fp32 batches: two vectors per interpolation CTA, on grids with at most one node per cell (radial
  // sigma = 2: 195 -> 170 us). Denser grids keep one vector per CTA: there the dense centre's tiles set
  // the tail and twice the work per CTA costs more than the shared taps save (sigma = 1.25, 2 nodes per
  // cell: 162 vs 173 us)
  if (p->batchmode && !p->tensor && ks.interp_cell2 && p->M <= p->ncells) {
    int o = 0;
    p->cell2 = p->cellmode && 2 * p->region_bytes <= 200 * 1024 &&
               cudaFuncSetAttribute(ks.interp_cell2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(2 * p->region_bytes)) == cudaSuccess &&
               cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ks.interp_cell2, RC_THREADS, 2 * p->region_bytes) ==
                   cudaSuccess &&
               o >= 1;
    cudaGetLastError();
  }
  if (p->wbmode) {
    bool ok = p->cellmode && !p->batchmode && ks.spread_wb;
    if (ok) {
      p->wb_bytes = (size_t)WB_WARPS * ks.wb_warp_bytes;
      int o = 0;
      ok = cudaFuncSetAttribute((const void*)ks.spread_wb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)p->wb_bytes) == cudaSuccess &&
           cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, (const void*)ks.spread_wb, 32 * WB_WARPS, p->wb_bytes) ==
               cudaSuccess &&
           o >= 1;
      cudaGetLastError();
    }
    p->wbmode = ok;
  }
  if (p->cellmode && p->D >= 2 && !p->wbmode && !p->batchmode && !p->full && !sc_ok) {  // no cell-mode adjoint
    p->cellmode = false;
    p->tensor = p->full = false;
  }
  p->use_ind = false;
  if (p->D >= 2 && !p->cellmode && p->tiled && ks.interp_nd &&
      (p->opt.method == NFFT_METHOD_AUTO || p->opt.method == NFFT_METHOD_TILED)) {
    int occ = 0;
    if (cudaFuncSetAttribute((const void*)ks.interp_nd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)p->region_bytes) == cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)ks.interp_nd, RN_THREADS, p->region_bytes) ==
            cudaSuccess &&
        occ >= 1)
      p->use_ind = true;
    cudaGetLastError();
  }
  return NFFT_SUCCESS;
}

#define TRY(x)                          \
  do {                                  \
    nfft_status s_ = (x);               \
    if (s_ != NFFT_SUCCESS) return s_;  \
  } while (0)

template <typename R, int RR>
void* binsort_fn(int D) {
  if (D == 1) return (void*)binsort_kernel<R, RR, 1>;
  if (D == 2) return (void*)binsort_kernel<R, RR, 2>;
  return (void*)binsort_kernel<R, RR, 3>;
}
template <typename R>
void* binsort_fn_rr(int rr, int D) {
  switch (rr) {
    case 1: return binsort_fn<R, 1>(D);
    case 2: return binsort_fn<R, 2>(D);
    case 4: return binsort_fn<R, 4>(D);
    default: return binsort_fn<R, 8>(D);
  }
}

// Cooperative launch (all CTAs co-resident: the kernel synchronises the grid).
template <typename R>
nfft_status launch_binsort(nfft_plan p, cudaStream_t st) {
  const R* nodes = (const R*)p->d_nodes;
  Geom g = p->geom;
  int P = (int)p->n_tiles;
  int nb = p->node_begin, ne = p->node_end, S = p->S;
  R* ks = (R*)p->d_ks;
  void* args[] = {(void*)&nodes, (void*)&g, (void*)&P, (void*)&p->d_cnt, (void*)&p->d_tile_total,
                  (void*)&p->d_offsets, (void*)&p->d_perm, (void*)&ks, (void*)&p->d_err, (void*)&nb, (void*)&ne,
                  (void*)&S, (void*)&p->d_subbase, (void*)&p->d_subs};
  CK(cudaLaunchCooperativeKernel(binsort_fn_rr<R>(p->bs_rr, p->D), dim3(p->bs_grid), dim3(BS_THREADS), args, p->bs_bytes, st));
  ++p->launches;
  return NFFT_SUCCESS;
}

// Chooses the cooperative single-kernel sort when every CTA fits on the GPU at
// once with <= 8 rounds of 512 nodes and the per-warp tile counters fit shared memory.
template <typename R>
void configure_binsort(nfft_plan p) {
  p->use_bs = false;
  const int P = (int)p->n_tiles;
  const size_t bytes = binsort_smem_bytes(P);
  if (bytes > 200 * 1024) return;
  // Each grid barrier costs about one same-address L2 atomic per CTA, so the
  // smallest grid that still gives every SM one CTA wins (measured on B200,
  // M = 2^18: 512 CTAs 68 us, 256 CTAs 37 us, 128 CTAs 25 us, 64 CTAs 32 us
  // per precompute stage including the graph launch).
  int best_rr = 0, best_g = 0, best_over = 1 << 30;
  for (int rr : {1, 2, 4, 8}) {
    void* fn = binsort_fn_rr<R>(rr, p->D);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, BS_THREADS, bytes) != cudaSuccess || occ < 1) {
      cudaGetLastError();
      continue;
    }
    const int64_t E = (int64_t)BS_THREADS * rr;
    const int64_t G = (p->M + E - 1) / E;
    if (G > (int64_t)occ * p->sm_count || G > p->cs_nblk) continue;
    // distance from one CTA per SM (fewer CTAs preferred when equal)
    const int over = G <= p->sm_count ? (int)(p->sm_count - G) : (int)(G - p->sm_count) * 2;
    if (over < best_over) {
      best_over = over;
      best_rr = rr;
      best_g = (int)G;
    }
  }
  if (best_rr > 0) {
    p->use_bs = true;
    p->bs_grid = best_g;
    p->bs_rr = best_rr;
    p->bs_bytes = bytes;
  }
}

// first-generation stable counting sort: count / column scan / scatter (precompute.cuh)
template <typename R>
nfft_status launch_cs3(nfft_plan p, cudaStream_t st) {
  const int M = (int)p->M;
  const int nt = (int)p->n_tiles;
  // stable counting sort into tiles: count, scan (+ offsets, subproblems), scatter (precompute.cuh)
  cs_count_kernel<R><<<p->cs_nblk, CS_W * 32, (size_t)nt * 4, st>>>((const R*)p->d_nodes, p->geom, nt,
                                                                           p->d_cnt, p->d_err);
  ++p->launches;
  CKL();
  cs_scan_kernel<<<(nt + 31) / 32, THREADS, 0, st>>>(p->d_cnt, nt, p->cs_nblk, M, p->d_tile_total,
                                                         p->d_offsets, p->d_ticket, p->node_begin, p->node_end,
                                                         p->S, p->d_subbase, p->d_subs);
  ++p->launches;
  CKL();
  cs_scatter_kernel<R><<<p->cs_nblk, CS_W * 32, (size_t)nt * 4, st>>>(
      (const R*)p->d_nodes, p->geom, nt, p->d_cnt, p->d_offsets, p->d_perm, (R*)p->d_ks);
  ++p->launches;
  CKL();
  return NFFT_SUCCESS;
}

template <typename R, int D>
nfft_status cell_sort_d(nfft_plan p, cudaStream_t st) {
  const int M = (int)p->M;
  const int nc = (int)p->ncells;
  const int ntiles = (nc + CL_SCAN_TILE - 1) / CL_SCAN_TILE;
  const unsigned gm = (unsigned)((std::max(M, ntiles) + CL_THREADS - 1) / CL_THREADS);
  const unsigned gp = (unsigned)((M + CL_THREADS - 1) / CL_THREADS);
  cl_count_kernel<R, D><<<gm, CL_THREADS, 0, st>>>((const R*)p->d_nodes, p->geom, p->d_ccount, p->d_cslot, p->d_err,
                                                   p->d_scan_status, ntiles, p->d_ctr);
  cl_scan_kernel<<<(unsigned)ntiles, CL_SCAN_THREADS, 0, st>>>(p->d_ccount, nc, p->d_scan_status, p->d_ctr,
                                                               p->d_cstart);
  cl_place_kernel<R, D><<<gp, CL_THREADS, 0, st>>>((const R*)p->d_nodes, p->geom, p->d_cslot, p->d_cstart,
                                                   (R*)p->d_kc, p->d_jc, p->d_ctr, p->d_big);
  const unsigned gf = (unsigned)std::min<int64_t>((nc + CL_THREADS - 1) / CL_THREADS, p->sm_count * 8);
  cl_fix_kernel<R, D><<<gf, CL_THREADS, 0, st>>>(p->geom, p->d_cstart, (R*)p->d_kc, p->d_jc, nc, p->d_ctr, p->d_big,
                                                 p->d_cslot, (R*)p->d_ks);
  p->launches += 4;
  CKL();
  return NFFT_SUCCESS;
}

template <typename R>
nfft_status cell_sort(nfft_plan p, cudaStream_t st) {
  if (p->D == 1) return cell_sort_d<R, 1>(p, st);
  if (p->D == 2) return cell_sort_d<R, 2>(p, st);
  return cell_sort_d<R, 3>(p, st);
}

template <typename R>
nfft_status precompute_impl(nfft_plan p, cudaStream_t st) {
  CK(cudaMemsetAsync(p->d_err, 0, sizeof(int), st));
  rec(p, 2, 0);
  if (p->cellmode) {
    TRY(cell_sort<R>(p, st));
    p->tile_binned = false;
    if (p->batchmode || p->wbmode || (p->tensor && p->D >= 2)) {
      // taps of every node for the D >= 2 adjoint / the TENSOR strategy (layout wt[pos][d][t])
      const KernelSet<R>& ks = kernels_of<R>(p);
      CK(launch_k(ks.taps_nd, (unsigned)((p->M + TN_NODES - 1) / TN_NODES), TN_NODES, 0, st, p->geom, WpnArg{p->wpn},
                  (const R*)p->d_kc, (R*)p->d_wt, (p->wbmode || p->batchmode) ? p->d_cl : (int*)nullptr));
      ++p->launches;
      if (p->batchmode) {
        invert_perm_kernel<<<(unsigned)((p->M + 255) / 256), 256, 0, st>>>(p->d_jc, (int)p->M, p->d_inv);
        ++p->launches;
        CKL();
      }
    }
    if (p->full) {  // FULL strategy: the rows of B (weights, grid indices) in cell order
      const KernelSet<R>& ks = kernels_of<R>(p);
      CK(launch_k(ks.full_build, (unsigned)((p->M + FB_NODES - 1) / FB_NODES), FB_THREADS, 0, st, p->geom,
                  WpnArg{p->wpn}, (const R*)p->d_kc, (R*)p->d_bw, p->d_bi, p->D >= 2 ? p->d_cl : (int*)nullptr));
      ++p->launches;
    }
    if (p->tensor && p->D == 1) {  // TENSOR strategy: the 2m taps of every node, in cell order
      const KernelSet<R>& ks = kernels_of<R>(p);
      CK(launch_k(ks.taps1, (unsigned)((p->M + T1_THREADS - 1) / T1_THREADS), T1_THREADS, 0, st, p->geom, WpnArg{p->wpn},
                  (const R*)p->d_kc, (R*)p->d_wt));
      ++p->launches;
    }
  } else if (p->use_bs) {
    TRY(launch_binsort<R>(p, st));
  } else {
    TRY(launch_cs3<R>(p, st));
  }
  rec(p, 2, 1);
  return NFFT_SUCCESS;
}

// ---- stages (each enqueues its kernels on the plan stream; device pointers) ----

template <typename T>
nfft_status stage_deconv(nfft_plan p, const typename cplx<T>::type* fhat, cudaStream_t st) {
  const Geom& g = p->geom;
  const int nl = g.N[g.D - 1];
  const long long rows = (long long)g.B * (g.ngrid_cells / nl);
  const long long units = rows * ((nl + 1) / 2);
  if (units < (1LL << 31) - THREADS * 4096LL) {  // flattened, two cells per thread
    const unsigned ctas = (unsigned)std::min<long long>((units + THREADS - 1) / THREADS, (long long)p->sm_count * 16);
    correct_flat_kernel<T, true><<<ctas, THREADS, 0, st>>>(g, fhat, (const T*)p->d_betaT,
                                                           (typename cplx<T>::type*)p->d_grid_in);
  } else {
    dim3 grid((unsigned)std::min<long long>((nl + THREADS - 1) / THREADS, 4096), (unsigned)std::min<long long>(rows, 65535));
    deconv_place_kernel<T><<<grid, THREADS, 0, st>>>(g, fhat, (const T*)p->d_betaT,
                                                     (typename cplx<T>::type*)p->d_grid_in);
  }
  ++p->launches;
  CKL();
  return NFFT_SUCCESS;
}

// forward: out-of-place grid_in -> grid (keeps grid_in's zero padding);
// adjoint: in place on grid_adj, with its own cuFFT plan so a forward and an
// adjoint can run concurrently (nfft_execute). Unnormalised (PAPER.md:209,
// 275; reading R13).
template <typename T>
nfft_status stage_fft(nfft_plan p, int dir, cudaStream_t st) {
  const bool fwd = dir == CUFFT_FORWARD;
  cufftHandle h = fwd ? p->fft : p->fft_adj;
  if (cufftSetStream(h, st) != CUFFT_SUCCESS) return NFFT_ERROR_CUFFT;
  void* in = fwd ? p->d_grid_in : p->d_grid_adj;
  void* out = fwd ? p->d_grid : p->d_grid_adj;
  cufftResult r;
  if constexpr (sizeof(T) == 8)
    r = cufftExecZ2Z(h, (cufftDoubleComplex*)in, (cufftDoubleComplex*)out, dir);
  else
    r = cufftExecC2C(h, (cufftComplex*)in, (cufftComplex*)out, dir);
  return r == CUFFT_SUCCESS ? NFFT_SUCCESS : NFFT_ERROR_CUFFT;
}

// pdl: the kernel right before on `st` is this plan's forward FFT (nfft_forward, nfft_execute without a
// concurrent precompute), so the interpolation may launch programmatically: its node loads overlap the
// FFT's tail and it waits for the grid (griddepcontrol.wait) before staging it
template <typename T>
nfft_status stage_interp(nfft_plan p, typename cplx<T>::type* f, cudaStream_t st, bool pdl = false) {
  const KernelSet<T>& ks = kernels_of<T>(p);
  const WinPoly<T>& wp = poly_of<T>(p);
  (void)wp;
  const WpnArg wpn{p->wpn};
  const auto* grid = (const typename cplx<T>::type*)p->d_grid;
  if (p->full) {  // f = B ghat over the stored rows
    const unsigned npb = FI_THREADS / (p->full_e <= 16 ? 8 : 32);
    const unsigned ctas = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p->node_end - p->node_begin + npb - 1) / npb,
                                                                           (int64_t)p->sm_count * 16));
    CK(launch_k(ks.full_interp, dim3(ctas, (unsigned)p->B), FI_THREADS, 0, st, p->geom, grid, (const T*)p->d_bw,
                (const int*)p->d_bi, (const int*)p->d_jc, p->node_begin, p->node_end, f));
  } else if (p->cell2) {
    using C = typename cplx<T>::type;
    CK((pdl ? launch_k_pdl<Geom, WpnArg, const C*, const T*, const int*, const int*, C*>
            : launch_k<Geom, WpnArg, const C*, const T*, const int*, const int*, C*>)(
        ks.interp_cell2, dim3((unsigned)p->n_tiles, (unsigned)((p->B + 1) / 2)), RC_THREADS, 2 * p->region_bytes, st,
        p->geom, wpn, grid, (const T*)p->d_kc, (const int*)p->d_jc, (const int*)p->d_cstart, f));
  } else if (p->cellmode && p->D >= 2) {
    CK((pdl ? launch_k_pdl<Geom, WpnArg, const typename cplx<T>::type*, const T*, const T*, const int*, const int*, int,
                           int, typename cplx<T>::type*>
            : launch_k<Geom, WpnArg, const typename cplx<T>::type*, const T*, const T*, const int*, const int*, int, int,
                       typename cplx<T>::type*>)(p->tensor ? ks.interp_cellt : ks.interp_cell, dim3((unsigned)p->n_tiles, (unsigned)p->B), RC_THREADS,
                p->region_bytes, st, p->geom, wpn, grid, (const T*)p->d_kc, (const T*)p->d_wt, (const int*)p->d_jc,
                (const int*)p->d_cstart, p->node_begin, p->node_end, f));
  } else if (p->use_ind) {
    ks.interp_nd<<<(unsigned)p->n_tiles, RN_THREADS, p->region_bytes, st>>>(
        p->geom, wp, grid, (const T*)p->d_ks, p->d_perm, p->d_offsets, p->node_begin, p->node_end, f);
  } else if (p->cellmode && p->D == 1) {
    const unsigned segs = (unsigned)((p->Nt[0] + I1_SEG - 1) / I1_SEG);
    CK((pdl ? launch_k_pdl<Geom, WpnArg, const typename cplx<T>::type*, const T*, const T*, const int*, const int*, int,
                           int, typename cplx<T>::type*>
            : launch_k<Geom, WpnArg, const typename cplx<T>::type*, const T*, const T*, const int*, const int*, int, int,
                       typename cplx<T>::type*>)(p->tensor ? ks.interp1t : ks.interp1, dim3(segs, (unsigned)p->B), I1_THREADS, p->r1_interp_bytes, st,
                p->geom, wpn, grid, (const T*)p->d_kc, (const T*)p->d_wt, (const int*)p->d_jc, (const int*)p->d_cstart,
                p->node_begin, p->node_end, f));
  } else if (p->tiled) {
    ks.interp_tiled<<<p->grid_tiled, THREADS, p->region_bytes, st>>>(
        p->geom, wp, grid, (const T*)p->d_ks, p->d_perm, p->d_subs, p->d_subbase + p->n_tiles, f);
  } else {
    CK(launch_k(ks.interp_direct, p->grid_direct, THREADS, 0, st, p->geom, wpn, grid, (const T*)p->d_ks,
                (const int*)p->d_perm, p->node_begin, p->node_end, f));
  }
  ++p->launches;
  CKL();
  return NFFT_SUCCESS;
}

template <typename T>
nfft_status stage_spread(nfft_plan p, const typename cplx<T>::type* f, cudaStream_t st, bool overlap = false) {
  const KernelSet<T>& ks = kernels_of<T>(p);
  const WinPoly<T>& wp = poly_of<T>(p);
  auto* grid = (typename cplx<T>::type*)p->d_grid_adj;  // all zero on entry (plan creation / previous crop)
  if (p->full && p->D >= 2) {
    // ghat = B^H f: values in cell order, then one thread per oversampled cell over the stored weights
    rec(p, 1, 1);
    using C = typename cplx<T>::type;
    permute_f_kernel<T><<<dim3((unsigned)((p->M + 1023) / 1024), (unsigned)p->B), 256, 0, st>>>(
        f, p->d_jc, (int)p->M, p->node_begin, p->node_end, (C*)p->d_fc);
    CKL();
    const unsigned ctas = (unsigned)std::min<int64_t>((p->ncells + FS_THREADS - 1) / FS_THREADS, (int64_t)p->sm_count * 16);
    CK(launch_k(ks.full_spread, dim3(ctas, (unsigned)p->B), FS_THREADS, 0, st, p->geom, (const C*)p->d_fc,
                (const int*)p->d_cl, (const T*)p->d_bw, (const int*)p->d_cstart, grid));
    p->launches += 2;
    return NFFT_SUCCESS;
  }
  if (p->batchmode) {
    using C = typename cplx<T>::type;
    rec(p, 1, 1);
    const unsigned nch = (unsigned)(p->bp / RB_LANES);
    transpose_bm_kernel<T><<<dim3((unsigned)((p->M + 31) / 32), nch), 256, 0, st>>>(f, (int)p->B, (int)p->M, p->bp,
                                                                                   p->d_inv, (C*)p->d_fT);
    const int S = Rb2Cfg<T>::S, R = Rb2Cfg<T>::R;
    const long long units = (long long)(p->Nt[0] + R - 1) / R * ((p->Nt[1] + S - 1) / S);
    // one CTA per unit: a persistent launch (rb_occ CTAs per SM, the next unit's cstart values prefetched)
    // measured slower on the radial configs (279 vs 222 us, sigma 2): the static unit order leaves the CTAs
    // that draw the dense centre's units as the tail
    const unsigned segs = (unsigned)units;
    // programmatic dependent launch: the parts' cstart loads overlap transpose_bm's tail
    CK(launch_k_pdl((const void*)ks.spread_rb2, dim3(segs, nch), 32 * RB2_WARPS, p->rb_bytes, st, p->geom,
                    (const C*)p->d_fT, p->bp, (const T*)p->d_wt, (const int*)p->d_cl, (const int*)p->d_cstart, grid));
    p->launches += 2;
    CKL();
    return NFFT_SUCCESS;
  }
  if (p->wbmode) {
    // node values in cell order, then owner-computes per warp block: every grid cell written exactly
    // once, no zero pass
    rec(p, 1, 1);
    using C = typename cplx<T>::type;
    permute_f_kernel<T><<<dim3((unsigned)((p->M + 1023) / 1024), (unsigned)p->B), 256, 0, st>>>(
        f, p->d_jc, (int)p->M, p->node_begin, p->node_end, (C*)p->d_fc);
    long long nblk = (p->Nt[0] + WB_K0 - 1) / WB_K0;
    if (p->D == 3) nblk *= (p->Nt[1] + 3) / 4 * ((p->Nt[2] + 7) / 8);
    else nblk *= (p->Nt[1] + 31) / 32;
    // programmatic dependent launch: the warps' window enumeration overlaps permute_f's tail
    CK(launch_k_pdl((const void*)ks.spread_wb, dim3((unsigned)((nblk + WB_WARPS - 1) / WB_WARPS), (unsigned)p->B),
                    32 * WB_WARPS, p->wb_bytes, st, p->geom, (const C*)p->d_fc, (const int*)p->d_cl, (const T*)p->d_wt,
                    (const int*)p->d_cstart, grid));
    p->launches += 2;
    CKL();
    return NFFT_SUCCESS;
  }
  if (p->cellmode && p->D >= 2) {
    rec(p, 1, 1);
    CK(launch_k(ks.spread_cell, dim3((unsigned)p->n_tiles, (unsigned)p->B), 256, p->sc_bytes, st, p->geom, WpnArg{p->wpn},
                f, (const T*)p->d_kc, (const int*)p->d_jc, (const int*)p->d_cstart, p->node_begin, p->node_end, p->sc_cap,
                grid));
    ++p->launches;
    CKL();
    return NFFT_SUCCESS;
  }
  if (p->cellmode && p->D == 1) {
    // owner-computes segment gather (POLYNOMIAL or TENSOR taps): every grid cell written exactly once,
    // no zero pass
    rec(p, 1, 1);
    // launch width: narrower when the direct NFFT runs concurrently (nfft_execute), resample1d.cuh
    // (alone: every segment its own CTA, the hardware refills the SMs; overlapped: a grid-stride launch
    // of S1_CTAS_OVERLAP CTAs per SM, so the direct NFFT's kernels find room)
    const bool stored = p->tensor || p->full;
    const unsigned nsegs = (unsigned)((p->Nt[0] + S1_SEG - 1) / S1_SEG);
    const unsigned width = (overlap ? S1_CTAS_OVERLAP : S1_CTAS_ALONE) > 0
                               ? (unsigned)((overlap ? S1_CTAS_OVERLAP : S1_CTAS_ALONE) * p->sm_count)
                               : nsegs;
    const unsigned segs = std::min(nsegs, width);
    // FULL in 1D: the rows of B are the 2m taps, so the TENSOR kernel reads them
    CK(launch_k(stored ? ks.spread1t : ks.spread1, dim3(segs, (unsigned)p->B), S1_THREADS,
                p->r1_spread_bytes, st, p->geom, WpnArg{p->wpn}, f, (const T*)p->d_kc,
                (const T*)(p->full ? p->d_bw : p->d_wt), (const int*)p->d_jc,
                (const int*)p->d_cstart, p->node_begin, p->node_end, grid));
    ++p->launches;
    CKL();
    return NFFT_SUCCESS;
  }
  if (p->tiled && p->grid_own > 0) {
    // owner-computes: every grid cell written exactly once, no zero pass
    rec(p, 1, 1);
    ks.spread_own<<<p->grid_own, ks.own_threads, p->own_bytes, st>>>(
        p->geom, wp, f, (const T*)p->d_ks, p->d_perm, p->d_offsets, p->node_begin, p->node_end, grid);
    ++p->launches;
    CKL();
    return NFFT_SUCCESS;
  }
  rec(p, 1, 1);
  if (p->tiled && p->grid_gather > 0) {
    ks.spread_gather<<<p->grid_gather, THREADS, p->gather_bytes, st>>>(
        p->geom, wp, f, (const T*)p->d_ks, p->d_perm, p->d_subs, p->d_subbase + p->n_tiles, p->S, grid);
  } else if (p->tiled && p->grid_loc == 0 && p->grid_sorted > 0) {
    ks.spread_sorted<<<p->grid_sorted, THREADS, p->sorted_bytes, st>>>(
        p->geom, wp, f, (const T*)p->d_ks, p->d_perm, p->d_subs, p->d_subbase + p->n_tiles, grid);
  } else if (p->tiled && p->grid_loc > 0) {
    ks.spread_loc<<<p->grid_loc, ks.loc_threads, p->loc_bytes, st>>>(
        p->geom, wp, f, (const T*)p->d_ks, p->d_perm, p->d_subs, p->d_subbase + p->n_tiles, p->S, grid);
  } else if (p->tiled) {
    ks.spread_tiled<<<p->grid_tiled, THREADS, p->region_bytes, st>>>(
        p->geom, wp, f, (const T*)p->d_ks, p->d_perm, p->d_subs, p->d_subbase + p->n_tiles, grid);
  } else {
    CK(launch_k(ks.spread_direct, p->grid_direct, THREADS, 0, st, p->geom, WpnArg{p->wpn}, f, (const T*)p->d_ks,
                (const int*)p->d_perm, p->node_begin, p->node_end, grid));
  }
  ++p->launches;
  CKL();
  return NFFT_SUCCESS;
}

// pdl: the kernel right before on `st` is this plan's inverse FFT (nfft_adjoint, nfft_execute): the
// crop launches programmatically (its launch overlaps the FFT's tail) and waits for the grid
template <typename T>
nfft_status stage_crop(nfft_plan p, typename cplx<T>::type* y, cudaStream_t st, bool pdl = false) {
  const Geom& g = p->geom;
  if (p->cellmode) {  // the cell-mode spread rewrites every cell: crop only, no re-zeroing
    const int nl = g.N[g.D - 1];
    const long long rows = (long long)g.B * (g.ngrid_cells / nl);
    const long long units = rows * ((nl + 1) / 2);
    if (units < (1LL << 31) - THREADS * 4096LL) {  // flattened, two cells per thread
      const unsigned ctas = (unsigned)std::min<long long>((units + THREADS - 1) / THREADS, (long long)p->sm_count * 16);
      using C = typename cplx<T>::type;
      const void* fn = (const void*)correct_flat_kernel<T, false>;
      CK((pdl ? launch_k_pdl<Geom, const C*, const T*, C*> : launch_k<Geom, const C*, const T*, C*>)(
          fn, dim3(ctas), dim3(THREADS), 0, st, g, (const C*)p->d_grid_adj, (const T*)p->d_betaT, y));
    } else {
      dim3 grid((unsigned)std::min<long long>((nl + THREADS - 1) / THREADS, 4096), (unsigned)std::min<long long>(rows, 65535));
      crop_kernel<T><<<grid, THREADS, 0, st>>>(g, (const typename cplx<T>::type*)p->d_grid_adj, (const T*)p->d_betaT, y);
    }
    ++p->launches;
    CKL();
    return NFFT_SUCCESS;
  }
  const int ntl = g.Nt[g.D - 1];
  const long long rows = (long long)g.B * (g.grid_cells / ntl);
  dim3 grid((unsigned)std::min<long long>((ntl + THREADS - 1) / THREADS, 4096), (unsigned)std::min<long long>(rows, 65535));
  crop_zero_kernel<T><<<grid, THREADS, 0, st>>>(g, (typename cplx<T>::type*)p->d_grid_adj,
                                                       (const T*)p->d_betaT, y);
  ++p->launches;
  CKL();
  return NFFT_SUCCESS;
}

template <typename T>
nfft_status forward_impl(nfft_plan p, const void* fhat_in, void* f_out) {
  using C = typename cplx<T>::type;
  const size_t grid_bytes_in = (size_t)p->B * p->geom.ngrid_cells * sizeof(C);
  const size_t node_bytes = (size_t)p->B * p->M * sizeof(C);
  const C* fhat = (const C*)fhat_in;
  C* f = (C*)f_out;
  const bool host_in = !is_device_pointer(fhat_in);
  const bool host_out = !is_device_pointer(f_out);
  if (host_in) {
    if (!p->d_stage_grid) CK(cudaMalloc(&p->d_stage_grid, grid_bytes_in));
    CK(cudaMemcpyAsync(p->d_stage_grid, fhat_in, grid_bytes_in, cudaMemcpyHostToDevice, p->stream));
    fhat = (const C*)p->d_stage_grid;
  }
  if (host_out) {
    if (!p->d_stage_nodes) CK(cudaMalloc(&p->d_stage_nodes, node_bytes));
    f = (C*)p->d_stage_nodes;
  }
  p->last_dir = 0;
  rec(p, 0, 0);
  TRY(stage_deconv<T>(p, fhat, p->stream));
  rec(p, 0, 1);
  TRY(stage_fft<T>(p, CUFFT_FORWARD, p->stream));
  rec(p, 0, 2);
  TRY(stage_interp<T>(p, f, p->stream, true));
  rec(p, 0, 3);
  if (host_out) {
    CK(cudaMemcpyAsync(f_out, f, node_bytes, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  }
  return NFFT_SUCCESS;
}

template <typename T>
nfft_status adjoint_impl(nfft_plan p, const void* f_in, void* y_out) {
  using C = typename cplx<T>::type;
  const size_t grid_bytes_out = (size_t)p->B * p->geom.ngrid_cells * sizeof(C);
  const size_t node_bytes = (size_t)p->B * p->M * sizeof(C);
  const C* f = (const C*)f_in;
  C* y = (C*)y_out;
  const bool host_in = !is_device_pointer(f_in);
  const bool host_out = !is_device_pointer(y_out);
  if (host_in) {
    if (!p->d_stage_nodes) CK(cudaMalloc(&p->d_stage_nodes, node_bytes));
    CK(cudaMemcpyAsync(p->d_stage_nodes, f_in, node_bytes, cudaMemcpyHostToDevice, p->stream));
    f = (const C*)p->d_stage_nodes;
  }
  if (host_out) {
    if (!p->d_stage_grid) CK(cudaMalloc(&p->d_stage_grid, grid_bytes_out));
    y = (C*)p->d_stage_grid;
  }
  p->last_dir = 1;
  rec(p, 1, 0);
  TRY(stage_spread<T>(p, f, p->stream));
  rec(p, 1, 2);
  TRY(stage_fft<T>(p, CUFFT_INVERSE, p->stream));
  rec(p, 1, 3);
  TRY(stage_crop<T>(p, y, p->stream, true));
  rec(p, 1, 4);
  if (host_out) {
    CK(cudaMemcpyAsync(y_out, y, grid_bytes_out, cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
  }
  return NFFT_SUCCESS;
}

template <typename T>
nfft_status run_stage_impl(nfft_plan p, int stage, const void* in, void* out) {
  using C = typename cplx<T>::type;
  switch (stage) {
    case NFFT_STAGE_FWD_DECONV: return stage_deconv<T>(p, (const C*)in, p->stream);
    case NFFT_STAGE_FWD_FFT: return stage_fft<T>(p, CUFFT_FORWARD, p->stream);
    case NFFT_STAGE_FWD_INTERP: return stage_interp<T>(p, (C*)out, p->stream);
    case NFFT_STAGE_ADJ_SPREAD: return stage_spread<T>(p, (const C*)in, p->stream);
    case NFFT_STAGE_ADJ_FFT: return stage_fft<T>(p, CUFFT_INVERSE, p->stream);
    case NFFT_STAGE_ADJ_CROP: return stage_crop<T>(p, (C*)out, p->stream);
  }
  return NFFT_ERROR_INVALID_VALUE;
}

// nfft_execute: any of {precompute, forward, adjoint} with the independent
// pieces overlapped. Precompute runs on side_pre concurrently with the
// forward's deconvolution + FFT on the plan stream; the adjoint runs on
// side_adj concurrently with the forward (disjoint scratch grids, own cuFFT
// plan); interpolation and spreading wait for the precompute. Everything is
// forked from and joined back into the plan stream, so stream order and CUDA
// graph capture behave as for one stream-ordered call.
template <typename T>
nfft_status execute_impl(nfft_plan p, int flags, const void* fhat, void* f_out, const void* f_in, void* y_out) {
  using C = typename cplx<T>::type;
  const bool pre = flags & NFFT_EXEC_PRECOMPUTE, fwd = flags & NFFT_EXEC_FORWARD, adj = flags & NFFT_EXEC_ADJOINT;
  // host pointers: staging buffers per chain (the chains run concurrently)
  const size_t gbytes = (size_t)p->B * p->geom.ngrid_cells * sizeof(C), nbytes = (size_t)p->B * p->M * sizeof(C);
  const bool h_fhat = fwd && !is_device_pointer(fhat), h_fout = fwd && !is_device_pointer(f_out);
  const bool h_fin = adj && !is_device_pointer(f_in), h_y = adj && !is_device_pointer(y_out);
  void* host_fout = nullptr;
  void* host_y = nullptr;
  if (h_fhat) {
    if (!p->d_stage_grid) CK(cudaMalloc(&p->d_stage_grid, gbytes));
  }
  if (h_fout) {
    if (!p->d_stage_nodes) CK(cudaMalloc(&p->d_stage_nodes, nbytes));
    host_fout = f_out;
    f_out = p->d_stage_nodes;
  }
  if (h_fin) {
    if (!p->d_stage_nodes2) CK(cudaMalloc(&p->d_stage_nodes2, nbytes));
  }
  if (h_y) {
    if (!p->d_stage_grid2) CK(cudaMalloc(&p->d_stage_grid2, gbytes));
    host_y = y_out;
    y_out = p->d_stage_grid2;
  }
  CK(cudaEventRecord(p->ev_fork, p->stream));
  if (pre) {
    CK(cudaStreamWaitEvent(p->side_pre, p->ev_fork, 0));
    TRY(precompute_impl<T>(p, p->side_pre));
    CK(cudaEventRecord(p->ev_pre, p->side_pre));
  }
  if (adj) {
    CK(cudaStreamWaitEvent(p->side_adj, p->ev_fork, 0));
    if (h_fin) {
      CK(cudaMemcpyAsync(p->d_stage_nodes2, f_in, nbytes, cudaMemcpyHostToDevice, p->side_adj));
      f_in = p->d_stage_nodes2;
    }
    if (pre) CK(cudaStreamWaitEvent(p->side_adj, p->ev_pre, 0));
    TRY(stage_spread<T>(p, (const C*)f_in, p->side_adj, fwd));
    TRY(stage_fft<T>(p, CUFFT_INVERSE, p->side_adj));
    TRY(stage_crop<T>(p, (C*)y_out, p->side_adj, true));
    if (h_y) CK(cudaMemcpyAsync(host_y, y_out, gbytes, cudaMemcpyDeviceToHost, p->side_adj));
    CK(cudaEventRecord(p->ev_adj, p->side_adj));
  }
  if (fwd) {
    if (h_fhat) {
      CK(cudaMemcpyAsync(p->d_stage_grid, fhat, gbytes, cudaMemcpyHostToDevice, p->stream));
      fhat = p->d_stage_grid;
    }
    TRY(stage_deconv<T>(p, (const C*)fhat, p->stream));
    TRY(stage_fft<T>(p, CUFFT_FORWARD, p->stream));
    if (pre) CK(cudaStreamWaitEvent(p->stream, p->ev_pre, 0));
    TRY(stage_interp<T>(p, (C*)f_out, p->stream, !pre));
    if (h_fout) CK(cudaMemcpyAsync(host_fout, f_out, nbytes, cudaMemcpyDeviceToHost, p->stream));
  }
  if (pre) CK(cudaStreamWaitEvent(p->stream, p->ev_pre, 0));
  if (adj) CK(cudaStreamWaitEvent(p->stream, p->ev_adj, 0));
  return NFFT_SUCCESS;
}

// nfft_execute: the precompute and the adjoint chain (spread -> FFT -> crop) form the critical
// path, so their internal streams get the highest priority (their CTAs are scheduled first when
// they compete with the direct NFFT; measured neutral to slightly positive, 1D config 2).
static int adj_priority() {
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return 0;
  return hi;
}

nfft_status copy_nodes(nfft_plan p, const void* nodes) {
  const size_t bytes = (size_t)p->M * p->D * p->rsize();
  CK(cudaMemcpyAsync(p->d_nodes, nodes, bytes, is_device_pointer(nodes) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     p->stream));
  return NFFT_SUCCESS;
}

nfft_status create_impl(nfft_plan* out, int D, const int64_t* N, int64_t M, const void* nodes, double sigma, int m,
                        nfft_window window, nfft_precision precision, const nfft_options* opt_in) {
  if (!out || !N || !nodes) return NFFT_ERROR_INVALID_VALUE;
  *out = nullptr;
  if (D > 3) return NFFT_ERROR_UNSUPPORTED;
  if (D < 1 || M < 1 || m < 1) return NFFT_ERROR_INVALID_VALUE;
  if (opt_in && (opt_in->window_points < 0 || opt_in->window_points > 1)) return NFFT_ERROR_INVALID_VALUE;
  // window_points = 1: NFFT3-style 2m+2 samples of the continued window. The kernels then
  // run with footprint half-width m + 1 while the window SHAPE (beta, scale, correction) keeps m.
  const int m_shape = m;
  if (opt_in && opt_in->window_points == 1) m = m + 1;
  if (window != NFFT_WINDOW_KAISER_BESSEL) return NFFT_ERROR_INVALID_VALUE;
  if (precision != NFFT_COMPLEX64 && precision != NFFT_COMPLEX128) return NFFT_ERROR_INVALID_VALUE;
  nfft_options opt;
  nfft_default_options(&opt);
  if (opt_in) opt = *opt_in;
  if (opt.batch < 1) return NFFT_ERROR_INVALID_VALUE;
  if (opt.batch > 65535) return NFFT_ERROR_UNSUPPORTED;  // batch vectors index grid dimension y
  if (opt.method < 0 || opt.method > 7) return NFFT_ERROR_INVALID_VALUE;
  if (opt.precompute < NFFT_PRECOMPUTE_AUTO || opt.precompute > NFFT_PRECOMPUTE_FULL) return NFFT_ERROR_INVALID_VALUE;
  if (!(sigma > 1.0) || !std::isfinite(sigma)) return NFFT_ERROR_BAD_GEOMETRY;
  if (m > MAX_M) return NFFT_ERROR_UNSUPPORTED;
  if (M > (int64_t)0x7fffffff - 1) return NFFT_ERROR_UNSUPPORTED;
  int64_t Nt[3] = {1, 1, 1};
  int64_t cells = 1, ncells = 1;
  for (int d = 0; d < D; ++d) {
    if (N[d] < 2) return NFFT_ERROR_BAD_GEOMETRY;  // odd N_d: n_d = -(N_d-1)/2 .. (N_d-1)/2
    if (N[d] > (int64_t)1 << 30) return NFFT_ERROR_UNSUPPORTED;
    Nt[d] = 2 * (int64_t)std::ceil(sigma * (double)N[d] / 2.0);
    if (2 * (int64_t)m >= Nt[d]) return NFFT_ERROR_BAD_GEOMETRY;
    cells *= Nt[d];
    ncells *= N[d];
    if (cells > (int64_t)0x7fffffff) return NFFT_ERROR_UNSUPPORTED;
  }
  if (opt.max_subproblem < 0 || opt.max_subproblem > THREADS) return NFFT_ERROR_BAD_TILE;
  const int64_t nend = opt.node_end == 0 ? M : opt.node_end;
  if (opt.node_begin < 0 || opt.node_begin > nend || nend > M) return NFFT_ERROR_INVALID_VALUE;
  // tiles: defaults sized so the tile region fits shared memory with >= 2 CTAs/SM
  const bool c128 = precision == NFFT_COMPLEX128;
  const size_t csz = c128 ? 16 : 8;
  int64_t Q[3] = {1, 1, 1}, P[3] = {1, 1, 1};
  // cell mode (AUTO/TILED): nodes sorted by cell; Q is the kernels' work tile
  const bool cell_candidate = opt.method == NFFT_METHOD_AUTO || opt.method == NFFT_METHOD_TILED;
  for (int d = 0; d < D; ++d) {
    int64_t q = opt.tile[d];
    if (q < 0 || q > Nt[d]) return NFFT_ERROR_BAD_TILE;
    // default work tiles; in cell mode they only shape interp_cell (and the spread_cell fallback):
    // 2D 32 x 64 measured fastest for it where Ntilde_1 >= 512 (512^2: 23.1 -> 20.9 us, radial
    // sigma = 2: 244 -> 230 us), 32 x 32 on smaller grids (radial sigma = 1.25, 320^2: 64 wide
    // tiles leave too few CTAs around the dense centre: 196 -> 240 us)
    // batches of >= 8 vectors (per-vector interp CTAs): 8 rows x the row split into equal parts of
    // <= 256 cells (radial sigma = 2: 16 x 64 228 us -> 8 x 256 199 us; sigma = 1.25: 16 x 32 189 us ->
    // 8 x 160 164 us; r02 tile sweep, tools/tile_sweep.sh)
    const bool wide = cell_candidate && D == 2 && opt.batch >= 8;
    if (q == 0)
      q = D == 1 ? 512
                 : (D == 2 ? (wide ? (d == 0 ? 8 : (Nt[1] + (Nt[1] + 255) / 256 - 1) / ((Nt[1] + 255) / 256))
                                   : ((cell_candidate && d == 1 && Nt[1] >= 512) ? 64 : 32))
                           : ((cell_candidate && d == 2) ? 16 : 8));
    q = std::min<int64_t>(q, Nt[d]);
    // cell-mode spreading reads a window of Q + 2m - 1 cells along the last dimension,
    // which must not wrap onto itself
    if (cell_candidate && D >= 2 && d == D - 1) q = std::min<int64_t>(q, Nt[d] - 2 * m + 1);
    Q[d] = q;
    P[d] = (Nt[d] + q - 1) / q;
  }
  // tile region per dimension: Q + 2m - 1 cells (block index set); the contiguous last
  // dimension is padded for the bank-rotated interp loop (C128: TP - 1 readable cells, pitch % 8 == 0)
  int64_t Lreg[3] = {1, 1, 1};
  size_t region_cells = 1;
  auto region_of = [&]() {
    region_cells = 1;
    for (int d = 0; d < D; ++d) {
      Lreg[d] = Q[d] + 2 * m - 1;
      // (also fp32 2D batches: interp_cell2's 16-byte elements rotate the same way)
      if (d == D - 1 && (precision == NFFT_COMPLEX128 || (D == 2 && opt.batch >= 8))) {
        const int64_t tp = 2 * m <= 8 ? 8 : 16;
        Lreg[d] = ((Q[d] + tp - 1) + 7) / 8 * 8;
      }
      region_cells *= (size_t)Lreg[d];
    }
    return region_cells * csz;
  };
  size_t region_bytes = region_of();
  // default tiles with a large window (m >= 6 in 3D): halve the largest leading tile extent until the
  // interpolation's staged region fits 200 KB of shared memory (e.g. 3D m = 7: 8 x 8 x 16 -> 4 x 8 x 16)
  const bool default_tile = D >= 2 && opt.tile[0] == 0 && opt.tile[1] == 0 && opt.tile[2] == 0;
  while (default_tile && region_bytes > 200 * 1024) {
    int dm = -1;
    for (int d = 0; d < D - 1; ++d)
      if (Q[d] > 1 && (dm < 0 || Q[d] > Q[dm])) dm = d;
    if (dm < 0) break;
    Q[dm] = (Q[dm] + 1) / 2;
    P[dm] = (Nt[dm] + Q[dm] - 1) / Q[dm];
    region_bytes = region_of();
  }

  DeviceGuard guard(opt.device);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const size_t smem_max = prop.sharedMemPerBlockOptin;
  // 2D default tiles that fill less than one wave of interp_cell CTAs (4 resident per SM): shorten the
  // tile rows so the tile count meets the resident slots (512^2, sigma = 2: 32 x 64 -> 28 x 64, 512 ->
  // 592 tiles = 4 per SM on 148 SMs instead of 3.46: interp 20.4 -> 18.5 us)
  if (default_tile && cell_candidate && D == 2 && opt.batch < 8) {
    const int64_t slots = 4 * (int64_t)prop.multiProcessorCount;
    if (P[0] * P[1] <= slots && P[1] <= slots) {
      const int64_t p0 = slots / P[1];
      const int64_t q0 = p0 > 0 ? (Nt[0] + p0 - 1) / p0 : Q[0];
      if (p0 > P[0] && q0 >= 16 && q0 < Q[0]) {
        Q[0] = q0;
        P[0] = (Nt[0] + q0 - 1) / q0;
        region_bytes = region_of();
      }
    }
  }
  bool tiled;
#ifdef NFFTB_TILE_VARIANTS
  if (opt.method != NFFT_METHOD_AUTO && opt.method != NFFT_METHOD_DIRECT) {
    if (region_bytes > smem_max) return NFFT_ERROR_BAD_TILE;
    tiled = true;
  } else if (opt.method == NFFT_METHOD_DIRECT) {
    tiled = false;
  } else {
    tiled = region_bytes <= smem_max;
  }
#else
  // default build: cell mode (AUTO / TILED) with the unblocked kernels as the fallback; the
  // first-generation tile-mode variants are compiled only with -DNFFTB_TILE_VARIANTS
  if (opt.method > NFFT_METHOD_DIRECT) return NFFT_ERROR_UNSUPPORTED;
  if (opt.method == NFFT_METHOD_TILED && region_bytes > smem_max) return NFFT_ERROR_BAD_TILE;
  tiled = false;
#endif

  nfft_plan p = new (std::nothrow) nfft_plan_s();
  if (!p) return NFFT_ERROR_OUT_OF_MEMORY;
  p->D = D;
  p->M = M;
  p->B = opt.batch;
  p->m = m;
  p->m_shape = m_shape;
  p->sigma = sigma;
  p->prec = precision;
  p->opt = opt;
  p->device = dev;
  p->stream = (cudaStream_t)opt.stream;
  p->sm_count = prop.multiProcessorCount;
  p->tiled = tiled;
  p->S = opt.max_subproblem > 0 ? (int)opt.max_subproblem : THREADS;
  p->node_begin = (int)opt.node_begin;
  p->node_end = (int)nend;
  p->region_bytes = region_bytes;
  p->deg = poly_degree(m, c128);
  int64_t n_tiles = 1;
  for (int d = 0; d < D; ++d) {
    p->N[d] = N[d];
    p->Nt[d] = Nt[d];
    p->Q[d] = Q[d];
    p->P[d] = P[d];
    p->beta[d] = M_PI * m_shape * (2.0 - (double)N[d] / (double)Nt[d]);  // reading R4
    n_tiles *= P[d];
  }
  p->n_tiles = n_tiles;
  p->max_subs = (int)std::min<int64_t>((nend - opt.node_begin + p->S - 1) / p->S + n_tiles, 0x7fffffff);
  if (p->max_subs < 1) p->max_subs = 1;

  Geom& g = p->geom;
  memset(&g, 0, sizeof(g));
  g.D = D;
  g.M = (int)M;
  g.B = (int)p->B;
  g.m = m;
  int boff = 0;
  for (int d = 0; d < MAX_D; ++d) {
    const bool act = d < D;
    g.Nt[d] = act ? (int)Nt[d] : 1;
    g.N[d] = act ? (int)N[d] : 1;
    g.Q[d] = act ? (int)Q[d] : 1;
    g.P[d] = act ? (int)P[d] : 1;
    g.L[d] = act ? (int)Lreg[d] : 1;
    g.Ntd[d] = act ? (double)Nt[d] : 1.0;
    g.beta_off[d] = boff;
    if (act) boff += (int)N[d];
  }
  g.grid_cells = cells;
  g.ngrid_cells = ncells;
  g.region_cells = (int)region_cells;

  nfft_status st = NFFT_SUCCESS;
  auto fail = [&](nfft_status s) {
    free_all(p);
    delete p;
    return s;
  };
  auto alloc = [&](void** ptr, size_t bytes) -> bool {
    if (cudaMalloc(ptr, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  };
  const size_t rs = c128 ? 8 : 4;
  bool ok = alloc(&p->d_nodes, (size_t)M * D * rs) && alloc(&p->d_ks, (size_t)M * D * rs) &&
            alloc((void**)&p->d_perm, M * 4) && alloc((void**)&p->d_offsets, (n_tiles + 1) * 4) &&
            alloc((void**)&p->d_subbase, (n_tiles + 1) * 4) && alloc((void**)&p->d_subs, (size_t)p->max_subs * 16) &&
            alloc((void**)&p->d_err, 16) && alloc(&p->d_grid, (size_t)cells * p->B * csz) &&
            alloc(&p->d_grid_in, (size_t)cells * p->B * csz) && alloc(&p->d_grid_adj, (size_t)cells * p->B * csz) &&
            alloc((void**)&p->d_beta64, boff * 8) && alloc(&p->d_betaT, boff * rs) &&
            alloc((void**)&p->d_poly, (size_t)D * 2 * m * MAX_Z * 8);
  if (ok) {
    p->cs_nblk = (int)((M + CS_E - 1) / CS_E);
    if ((size_t)n_tiles * 4 > 160 * 1024 || (int64_t)n_tiles * p->cs_nblk > ((int64_t)1 << 28)) return fail(NFFT_ERROR_UNSUPPORTED);
    ok = alloc((void**)&p->d_cnt, (size_t)n_tiles * p->cs_nblk * 4) && alloc((void**)&p->d_tile_total, n_tiles * 4) &&
         alloc((void**)&p->d_ticket, 16);
  }
  p->ncells = cells;
  p->cellmode = cell_candidate;
  if (ok && p->cellmode)
    ok = alloc(&p->d_kc, (size_t)M * D * rs) && alloc((void**)&p->d_jc, (size_t)M * 4) &&
         alloc((void**)&p->d_cstart, (size_t)(cells + 1) * 4) && alloc((void**)&p->d_ccount, (size_t)(cells + 1) * 4) &&
         alloc((void**)&p->d_cslot, (size_t)M * 4) &&
         alloc((void**)&p->d_scan_status, (size_t)((cells + CL_SCAN_TILE - 1) / CL_SCAN_TILE + 1) * 8) &&
         alloc((void**)&p->d_ctr, 16) &&
         alloc((void**)&p->d_big, (size_t)(M / (CL_SMALL + 1) + 1) * 4);
  // window precompute strategies (AUTO = POLYNOMIAL, measured fastest on B200):
  // TENSOR stores the 2m D taps of every node (all kernels read them), FULL the rows of the sparse matrix B
  p->tensor = p->cellmode && opt.precompute == NFFT_PRECOMPUTE_TENSOR;
  p->full = p->cellmode && opt.precompute == NFFT_PRECOMPUTE_FULL;
  p->full_e = 1;
  for (int d = 0; d < D; ++d) p->full_e *= 2 * m;
  if (ok && p->tensor) ok = alloc(&p->d_wt, (size_t)M * D * 2 * m * rs);
  if (ok && p->full) {
    ok = alloc(&p->d_bw, (size_t)M * p->full_e * rs) && alloc((void**)&p->d_bi, (size_t)M * p->full_e * 4);
    if (ok && D >= 2) ok = alloc(&p->d_fc, (size_t)M * p->B * csz) && alloc((void**)&p->d_cl, (size_t)M * 4);
  }
  // 2D batches of >= 8 transforms: row-segment adjoint with lanes = batch vectors (not for node
  // shards; the 16 + 2m - 1 window columns must not wrap onto themselves)
  p->batchmode = p->cellmode && !p->full && D == 2 && p->B >= 8 && opt.node_begin == 0 &&
                 (opt.node_end == 0 || opt.node_end == M) &&
                 Nt[1] >= (c128 ? Rb2Cfg<double>::S : Rb2Cfg<float>::S) + 2 * m - 1 &&
                 Nt[0] >= (c128 ? Rb2Cfg<double>::R : Rb2Cfg<float>::R) + 2 * m - 1;
  p->bp = (int)((p->B + 31) / 32 * 32);
  if (ok && p->batchmode)
    ok = alloc(&p->d_fT, (size_t)M * p->bp * csz) && (p->d_wt || alloc(&p->d_wt, (size_t)M * D * 2 * m * rs)) &&
         alloc((void**)&p->d_inv, (size_t)M * 4) && (p->d_cl || alloc((void**)&p->d_cl, (size_t)M * 4));
  // D = 2, 3 (not batched): warp-block adjoint over the TENSOR taps; the last-dimension window
  // (32 or 8 lanes + 2m - 1 cells) must not wrap onto itself
  p->wbmode = p->cellmode && !p->full && !p->batchmode && D >= 2 && Nt[D - 1] >= (D == 3 ? 8 : 32) + 2 * m - 1;
  if (ok && p->wbmode)
    ok = (p->d_wt || alloc(&p->d_wt, (size_t)M * D * 2 * m * rs)) && alloc(&p->d_fc, (size_t)M * p->B * csz) &&
         alloc((void**)&p->d_cl, (size_t)M * 4);
  if (!ok) return fail(NFFT_ERROR_OUT_OF_MEMORY);
  {
    const int bytes = (int)(n_tiles * 4);
    cudaError_t e = cudaSuccess;
    if (c128) {
      e = cudaFuncSetAttribute((const void*)cs_count_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)cs_scatter_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    } else {
      e = cudaFuncSetAttribute((const void*)cs_count_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)cs_scatter_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    }
    if (e != cudaSuccess) {
      last_cuda_error = e;
      return fail(NFFT_ERROR_CUDA);
    }
  }
  if (cudaMemsetAsync(p->d_grid_in, 0, (size_t)cells * p->B * csz, p->stream) != cudaSuccess ||
      cudaMemsetAsync(p->d_grid_adj, 0, (size_t)cells * p->B * csz, p->stream) != cudaSuccess ||

      cudaMemsetAsync(p->d_ticket, 0, 16, p->stream) != cudaSuccess ||
      (p->d_ccount && cudaMemsetAsync(p->d_ccount, 0, (size_t)(cells + 1) * 4, p->stream) != cudaSuccess))
    return fail(NFFT_ERROR_CUDA);

  int n[3];
  for (int d = 0; d < D; ++d) n[d] = (int)Nt[d];
  if (cufftPlanMany(&p->fft, D, n, nullptr, 1, 0, nullptr, 1, 0, c128 ? CUFFT_Z2Z : CUFFT_C2C, (int)p->B) !=
      CUFFT_SUCCESS)
    return fail(NFFT_ERROR_CUFFT);
  p->fft_ok = true;
  if (cufftSetStream(p->fft, p->stream) != CUFFT_SUCCESS) return fail(NFFT_ERROR_CUFFT);
  if (cufftPlanMany(&p->fft_adj, D, n, nullptr, 1, 0, nullptr, 1, 0, c128 ? CUFFT_Z2Z : CUFFT_C2C, (int)p->B) !=
      CUFFT_SUCCESS)
    return fail(NFFT_ERROR_CUFFT);
  p->fft_adj_ok = true;
  if (cudaStreamCreateWithPriority(&p->side_pre, cudaStreamNonBlocking, adj_priority()) != cudaSuccess ||
      cudaStreamCreateWithPriority(&p->side_adj, cudaStreamNonBlocking, adj_priority()) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_pre, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_adj, cudaEventDisableTiming) != cudaSuccess)
    return fail(NFFT_ERROR_CUDA);

  if (opt.timing) {
    for (auto& row : p->ev)
      for (auto& e : row)
        if (cudaEventCreate(&e) != cudaSuccess) return fail(NFFT_ERROR_CUDA);
    p->events = true;
  }
  if (c128) {
    p->k64 = kernels_for<double>(D, m);
    st = build_window_tables<double>(p);
    if (st == NFFT_SUCCESS) st = configure_kernels<double>(p, p->k64);
    if (st == NFFT_SUCCESS && opt.method != NFFT_METHOD_TILED_V1) configure_binsort<double>(p);
  } else {
    p->k32 = kernels_for<float>(D, m);
    st = build_window_tables<float>(p);
    if (st == NFFT_SUCCESS) st = configure_kernels<float>(p, p->k32);
    if (st == NFFT_SUCCESS && opt.method != NFFT_METHOD_TILED_V1) configure_binsort<float>(p);
  }
  if (st == NFFT_SUCCESS) st = copy_nodes(p, nodes);
  if (st == NFFT_SUCCESS) {
    cudaError_t e = cudaStreamSynchronize(p->stream);
    if (e != cudaSuccess) {
      last_cuda_error = e;
      st = NFFT_ERROR_CUDA;
    }
  }
  if (st != NFFT_SUCCESS) return fail(st);
  *out = p;
  return NFFT_SUCCESS;
}

}  // namespace

extern "C" {

nfft_status nfft_default_options(nfft_options* opt) {
  if (!opt) return NFFT_ERROR_INVALID_VALUE;
  memset(opt, 0, sizeof(*opt));
  opt->batch = 1;
  opt->device = -1;
  opt->method = NFFT_METHOD_AUTO;
  opt->check_nodes = 1;
  return NFFT_SUCCESS;
}

nfft_status nfft_plan_create(nfft_plan* out, int D, const int64_t* N, int64_t M, const void* nodes, double sigma, int m,
                             nfft_window window, nfft_precision precision) {
  return create_impl(out, D, N, M, nodes, sigma, m, window, precision, nullptr);
}

nfft_status nfft_plan_create_ex(nfft_plan* out, int D, const int64_t* N, int64_t M, const void* nodes, double sigma,
                                int m, nfft_window window, nfft_precision precision, const nfft_options* opt) {
  return create_impl(out, D, N, M, nodes, sigma, m, window, precision, opt);
}

// Online block-size benchmark (the optimisation mode the paper proposes, "similar to
// FFTW_MEASURE"; its block-size study): for every candidate tile a plan is built on
// the caller's nodes, precomputed, and `reps` direct + adjoint transforms (nfft_execute, zero data)
// are timed with CUDA events after one warm-up; the fastest tile is returned.
nfft_status nfft_autotune_tile(int D, const int64_t* N, int64_t M, const void* nodes, double sigma, int m,
                               nfft_precision precision, const nfft_options* opt_in, const int64_t* candidates,
                               int ncand, int reps, int64_t* best_tile, float* best_ms) {
  if (D < 1 || D > 3 || !N || !nodes || !best_tile || reps < 1 || ncand < 0 || (ncand > 0 && !candidates))
    return NFFT_ERROR_INVALID_VALUE;
  static const int64_t def1[] = {256, 512, 1024, 2048};
  static const int64_t def2[] = {16, 32, 32, 32, 32, 64, 64, 64, 8, 64};
  static const int64_t def3[] = {8, 8, 16, 8, 16, 16, 4, 8, 32, 8, 8, 8};
  const int64_t* cand = candidates;
  if (ncand == 0) {
    cand = D == 1 ? def1 : (D == 2 ? def2 : def3);
    ncand = D == 1 ? 4 : (D == 2 ? 5 : 4);
  }
  nfft_options opt;
  nfft_default_options(&opt);
  if (opt_in) opt = *opt_in;
  int64_t ncells = 1;
  for (int d = 0; d < D; ++d) ncells *= N[d];
  const size_t csz = precision == NFFT_COMPLEX128 ? 16 : 8;
  const size_t gbytes = (size_t)opt.batch * ncells * csz, nbytes = (size_t)opt.batch * M * csz;
  void *fhat = nullptr, *fout = nullptr, *fin = nullptr, *yout = nullptr;
  if (cudaMalloc(&fhat, gbytes) != cudaSuccess || cudaMalloc(&yout, gbytes) != cudaSuccess ||
      cudaMalloc(&fin, nbytes) != cudaSuccess || cudaMalloc(&fout, nbytes) != cudaSuccess) {
    cudaFree(fhat);
    cudaFree(yout);
    cudaFree(fin);
    cudaFree(fout);
    return NFFT_ERROR_OUT_OF_MEMORY;
  }
  cudaMemset(fhat, 0, gbytes);
  cudaMemset(fin, 0, nbytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  nfft_status st = NFFT_ERROR_INVALID_VALUE;
  float best = 0.f;
  for (int c = 0; c < ncand; ++c) {
    for (int d = 0; d < 3; ++d) opt.tile[d] = d < D ? cand[(size_t)c * D + d] : 0;
    nfft_plan p = nullptr;
    nfft_status s = create_impl(&p, D, N, M, nodes, sigma, m, NFFT_WINDOW_KAISER_BESSEL, precision, &opt);
    if (s != NFFT_SUCCESS) continue;  // e.g. a tile larger than the grid: skip the candidate
    s = nfft_execute(p, NFFT_EXEC_PRECOMPUTE | NFFT_EXEC_FORWARD | NFFT_EXEC_ADJOINT, fhat, fout, fin, yout);
    float ms = 0.f;
    if (s == NFFT_SUCCESS) {
      cudaEventRecord(e0, p->stream);
      for (int r = 0; r < reps && s == NFFT_SUCCESS; ++r)
        s = nfft_execute(p, NFFT_EXEC_FORWARD | NFFT_EXEC_ADJOINT, fhat, fout, fin, yout);
      cudaEventRecord(e1, p->stream);
      if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess)
        s = NFFT_ERROR_CUDA;
    }
    nfft_plan_destroy(p);
    if (s != NFFT_SUCCESS) {
      st = s;
      break;
    }
    ms /= reps;
    if (st != NFFT_SUCCESS || ms < best) {
      best = ms;
      for (int d = 0; d < D; ++d) best_tile[d] = cand[(size_t)c * D + d];
      st = NFFT_SUCCESS;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(fhat);
  cudaFree(yout);
  cudaFree(fin);
  cudaFree(fout);
  if (st == NFFT_SUCCESS && best_ms) *best_ms = best;
  return st;
}

nfft_status nfft_set_nodes(nfft_plan p, const void* nodes) {
  if (!p || !nodes) return NFFT_ERROR_INVALID_VALUE;
  DeviceGuard guard(p->device);
  nfft_status s = copy_nodes(p, nodes);
  if (s == NFFT_SUCCESS) p->precomputed = false;
  return s;
}

nfft_status nfft_precompute(nfft_plan p) {
  if (!p) return NFFT_ERROR_INVALID_VALUE;
  DeviceGuard guard(p->device);
  nfft_status s = p->prec == NFFT_COMPLEX128 ? precompute_impl<double>(p, p->stream) : precompute_impl<float>(p, p->stream);
  if (s != NFFT_SUCCESS) return s;
  if (p->opt.check_nodes) {
    int err = 0;
    CK(cudaMemcpyAsync(&err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    if (err) {
      p->precomputed = false;
      return NFFT_ERROR_NONFINITE_NODE;
    }
  }
  p->precomputed = true;
  return NFFT_SUCCESS;
}

nfft_status nfft_forward(nfft_plan p, const void* fhat_grid, void* f_nodes) {
  if (!p || !fhat_grid || !f_nodes) return NFFT_ERROR_INVALID_VALUE;
  if (!p->precomputed) return NFFT_ERROR_NOT_PRECOMPUTED;
  DeviceGuard guard(p->device);
  return p->prec == NFFT_COMPLEX128 ? forward_impl<double>(p, fhat_grid, f_nodes)
                                    : forward_impl<float>(p, fhat_grid, f_nodes);
}

nfft_status nfft_adjoint(nfft_plan p, const void* f_nodes, void* fhat_grid) {
  if (!p || !fhat_grid || !f_nodes) return NFFT_ERROR_INVALID_VALUE;
  if (!p->precomputed) return NFFT_ERROR_NOT_PRECOMPUTED;
  DeviceGuard guard(p->device);
  return p->prec == NFFT_COMPLEX128 ? adjoint_impl<double>(p, f_nodes, fhat_grid)
                                    : adjoint_impl<float>(p, f_nodes, fhat_grid);
}

nfft_status nfft_run_stage(nfft_plan p, int stage, const void* in, void* out) {
  if (!p || stage < NFFT_STAGE_PRECOMPUTE || stage > NFFT_STAGE_ADJ_CROP) return NFFT_ERROR_INVALID_VALUE;
  DeviceGuard guard(p->device);
  if (stage == NFFT_STAGE_PRECOMPUTE) {
    nfft_status s = p->prec == NFFT_COMPLEX128 ? precompute_impl<double>(p, p->stream) : precompute_impl<float>(p, p->stream);
    if (s == NFFT_SUCCESS) p->precomputed = true;
    return s;
  }
  if (!p->precomputed) return NFFT_ERROR_NOT_PRECOMPUTED;
  const bool needs_in = stage == NFFT_STAGE_FWD_DECONV || stage == NFFT_STAGE_ADJ_SPREAD;
  const bool needs_out = stage == NFFT_STAGE_FWD_INTERP || stage == NFFT_STAGE_ADJ_CROP;
  if ((needs_in && (!in || !is_device_pointer(in))) || (needs_out && (!out || !is_device_pointer(out))))
    return NFFT_ERROR_INVALID_VALUE;
  return p->prec == NFFT_COMPLEX128 ? run_stage_impl<double>(p, stage, in, out) : run_stage_impl<float>(p, stage, in, out);
}

nfft_status nfft_execute(nfft_plan p, int flags, const void* fhat_grid, void* f_nodes, const void* f_in,
                         void* y_grid) {
  if (!p || flags <= 0 || flags > 7) return NFFT_ERROR_INVALID_VALUE;
  const bool fwd = flags & NFFT_EXEC_FORWARD, adj = flags & NFFT_EXEC_ADJOINT;
  if (fwd && (!fhat_grid || !f_nodes)) return NFFT_ERROR_INVALID_VALUE;
  if (adj && (!f_in || !y_grid)) return NFFT_ERROR_INVALID_VALUE;
  if (!(flags & NFFT_EXEC_PRECOMPUTE) && !p->precomputed) return NFFT_ERROR_NOT_PRECOMPUTED;
  DeviceGuard guard(p->device);
  nfft_status s = p->prec == NFFT_COMPLEX128 ? execute_impl<double>(p, flags, fhat_grid, f_nodes, f_in, y_grid)
                                             : execute_impl<float>(p, flags, fhat_grid, f_nodes, f_in, y_grid);
  if (s == NFFT_SUCCESS && (flags & NFFT_EXEC_PRECOMPUTE)) p->precomputed = true;
  return s;
}

nfft_status nfft_plan_destroy(nfft_plan p) {
  if (!p) return NFFT_ERROR_INVALID_VALUE;
  DeviceGuard guard(p->device);
  cudaError_t e = cudaStreamSynchronize(p->stream);
  if (p->side_pre) cudaStreamSynchronize(p->side_pre);
  if (p->side_adj) cudaStreamSynchronize(p->side_adj);
  free_all(p);
  delete p;
  if (e != cudaSuccess) {
    last_cuda_error = e;
    return NFFT_ERROR_CUDA;
  }
  return NFFT_SUCCESS;
}

const char* nfft_status_string(nfft_status s) {
  switch (s) {
    case NFFT_SUCCESS: return "success";
    case NFFT_ERROR_INVALID_VALUE: return "invalid value";
    case NFFT_ERROR_BAD_GEOMETRY: return "bad geometry (N_d >= 2, sigma > 1, 2m < Ntilde_d)";
    case NFFT_ERROR_NONFINITE_NODE: return "non-finite node coordinate";
    case NFFT_ERROR_BAD_TILE: return "bad tile size";
    case NFFT_ERROR_NOT_PRECOMPUTED: return "plan not precomputed";
    case NFFT_ERROR_OUT_OF_MEMORY: return "out of device memory";
    case NFFT_ERROR_CUDA: return last_cuda_error != cudaSuccess ? cudaGetErrorString(last_cuda_error) : "CUDA error";
    case NFFT_ERROR_CUFFT: return "cuFFT error";
    case NFFT_ERROR_UNSUPPORTED: return "unsupported (D > 3, m > 8, or size beyond int32 indexing)";
  }
  return "unknown status";
}

nfft_status nfft_plan_info(nfft_plan p, int64_t* Ntilde, int64_t* tile, int64_t* tiles_per_dim, int64_t* n_tiles) {
  if (!p) return NFFT_ERROR_INVALID_VALUE;
  for (int d = 0; d < p->D; ++d) {
    if (Ntilde) Ntilde[d] = p->Nt[d];
    if (tile) tile[d] = p->Q[d];
    if (tiles_per_dim) tiles_per_dim[d] = p->P[d];
  }
  if (n_tiles) *n_tiles = p->n_tiles;
  return NFFT_SUCCESS;
}

nfft_status nfft_get_binning(nfft_plan p, int32_t* perm_host, int32_t* offsets_host) {
  if (!p) return NFFT_ERROR_INVALID_VALUE;
  if (!p->precomputed) return NFFT_ERROR_NOT_PRECOMPUTED;
  DeviceGuard guard(p->device);
  if (p->cellmode && !p->tile_binned) {  // the hot path sorted by cell; the tile sort is computed on demand
    nfft_status s = p->use_bs ? (p->prec == NFFT_COMPLEX128 ? launch_binsort<double>(p, p->stream)
                                                            : launch_binsort<float>(p, p->stream))
                              : (p->prec == NFFT_COMPLEX128 ? launch_cs3<double>(p, p->stream)
                                                            : launch_cs3<float>(p, p->stream));
    if (s != NFFT_SUCCESS) return s;
    p->tile_binned = true;
  }
  if (perm_host) CK(cudaMemcpyAsync(perm_host, p->d_perm, p->M * 4, cudaMemcpyDeviceToHost, p->stream));
  if (offsets_host)
    CK(cudaMemcpyAsync(offsets_host, p->d_offsets, (p->n_tiles + 1) * 4, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return NFFT_SUCCESS;
}

nfft_status nfft_get_cell_binning(nfft_plan p, int32_t* order_host, int32_t* cstart_host) {
  if (!p) return NFFT_ERROR_INVALID_VALUE;
  if (!p->cellmode) return NFFT_ERROR_UNSUPPORTED;
  if (!p->precomputed) return NFFT_ERROR_NOT_PRECOMPUTED;
  DeviceGuard guard(p->device);
  if (order_host) CK(cudaMemcpyAsync(order_host, p->d_jc, p->M * 4, cudaMemcpyDeviceToHost, p->stream));
  if (cstart_host)
    CK(cudaMemcpyAsync(cstart_host, p->d_cstart, (p->ncells + 1) * 4, cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  return NFFT_SUCCESS;
}

nfft_status nfft_get_window_tables(nfft_plan p, double* beta_tensor, double* poly, int* deg) {
  if (!p) return NFFT_ERROR_INVALID_VALUE;
  DeviceGuard guard(p->device);
  int64_t nb = 0;
  for (int d = 0; d < p->D; ++d) nb += p->N[d];
  if (beta_tensor) CK(cudaMemcpyAsync(beta_tensor, p->d_beta64, nb * 8, cudaMemcpyDeviceToHost, p->stream));
  if (poly) {
    const int Z = p->deg + 1;
    const size_t cnt = (size_t)p->D * 2 * p->m;
    double* tmp = new (std::nothrow) double[cnt * MAX_Z];
    if (!tmp) return NFFT_ERROR_OUT_OF_MEMORY;
    cudaError_t e = cudaMemcpyAsync(tmp, p->d_poly, cnt * MAX_Z * 8, cudaMemcpyDeviceToHost, p->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    if (e != cudaSuccess) {
      delete[] tmp;
      last_cuda_error = e;
      return NFFT_ERROR_CUDA;
    }
    for (size_t r = 0; r < cnt; ++r)
      for (int z = 0; z < Z; ++z) poly[r * Z + z] = tmp[r * MAX_Z + z];
    delete[] tmp;
  }
  if (deg) *deg = p->deg;
  CK(cudaStreamSynchronize(p->stream));
  return NFFT_SUCCESS;
}

nfft_status nfft_get_stage_times_ex(nfft_plan p, int which, float* ms) {
  if (!p || !ms || which < 0 || which > 1) return NFFT_ERROR_INVALID_VALUE;
  if (!p->events) return NFFT_ERROR_INVALID_VALUE;
  DeviceGuard guard(p->device);
  CK(cudaStreamSynchronize(p->stream));
  for (int i = 0; i < 5; ++i) ms[i] = 0.f;
  auto el = [&](int w, int a, int b) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, p->ev[w][a], p->ev[w][b]) != cudaSuccess) {
      cudaGetLastError();
      t = 0.f;
    }
    return t;
  };
  if (which == 0) {
    ms[0] = el(0, 0, 1);
    ms[1] = el(0, 1, 2);
    ms[2] = el(0, 2, 3);
  } else {
    ms[3] = el(1, 0, 1);
    ms[2] = el(1, 1, 2);
    ms[1] = el(1, 2, 3);
    ms[0] = el(1, 3, 4);
  }
  ms[4] = el(2, 0, 1);
  return NFFT_SUCCESS;
}

// SURVEY §8(b)'s form: the deconvolution (or crop), FFT and resampling times of
// the most recent forward or adjoint call (whichever ran last).
nfft_status nfft_get_stage_times(nfft_plan p, float* ms_deconv, float* ms_fft, float* ms_resample) {
  if (!p) return NFFT_ERROR_INVALID_VALUE;
  float ms[5];
  nfft_status s = nfft_get_stage_times_ex(p, p->last_dir, ms);
  if (s != NFFT_SUCCESS) return s;
  if (ms_deconv) *ms_deconv = ms[0];
  if (ms_fft) *ms_fft = ms[1];
  if (ms_resample) *ms_resample = ms[2];
  return NFFT_SUCCESS;
}

nfft_status nfft_get_features(nfft_plan p, int* features) {
  if (!p || !features) return NFFT_ERROR_INVALID_VALUE;
  *features = (p->cellmode ? NFFT_FEATURE_CELL_MODE : 0) | (p->tensor ? NFFT_FEATURE_TENSOR : 0) |
              (p->full ? NFFT_FEATURE_FULL : 0) |
              (p->batchmode ? NFFT_FEATURE_BATCH : 0) | (p->wbmode ? NFFT_FEATURE_WBLOCK : 0);
  return NFFT_SUCCESS;
}

nfft_status nfft_get_launch_count(nfft_plan p, int64_t* launches) {
  if (!p || !launches) return NFFT_ERROR_INVALID_VALUE;
  *launches = p->launches;
  return NFFT_SUCCESS;
}

}  // extern "C"
