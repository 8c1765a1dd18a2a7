// Timeline harness (diagnostic) for the D = 1 resampling kernels: builds the
// product kernels with NFFTB_PHASE_TRACE (thread 0 of every CTA stamps
// %globaltimer at phase boundaries), runs them on config-2-like synthetic
// data (M = N = 2^18, sigma = 2; nodes cell-sorted on the host), with an L2
// flush before each launch, and prints per-phase percentiles of the stamps
// relative to the earliest CTA start (microseconds) plus the event time.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -o /tmp/trace1d tools/micro/trace1d.cu && /tmp/trace1d [m]
#define NFFTB_PHASE_TRACE
#include "../../paper_2208_00049_b200/csrc/resample1d.cuh"
#define SPREAD1 spread1a_kernel

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

using namespace nfftb;
template <typename T>
__global__ void __launch_bounds__(128) empty_kernel(Geom g, WinPoly<T> wp, double2* out) {
  if (threadIdx.x == 0 && blockIdx.x == 100000) out[0] = make_double2(wp.mu[0][0][0], g.Ntd[0]);
}
__global__ void __launch_bounds__(128) empty_small(double2* out, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 100000) out[0] = make_double2(n, n);
}
__global__ void permute_scatter(const double2* __restrict__ f, const int* __restrict__ inv, double2* __restrict__ fc,
                                int M) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < M) fc[inv[j]] = f[j];
}
static bool g_flush = true;
static unsigned g_s1cap = 0;  // spread1a CTAs per SM (0: one per segment); env S1CAP  // L2 flush before every launch (argv[2] = "warm": no flush)

template <int M>
static void run(int M_nodes, int Nt) {
  constexpr int DEG = poly_degree(M, true);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(-0.5, 0.5);
  std::vector<double> k(M_nodes);
  for (auto& x : k) x = U(rng);
  // host cell sort (stable)
  std::vector<int> cell(M_nodes), cnt(Nt + 1, 0), jc(M_nodes);
  for (int j = 0; j < M_nodes; ++j) {
    int c = (int)std::floor(Nt * k[j]) + Nt / 2;
    c = ((c % Nt) + Nt) % Nt;
    cell[j] = c;
    cnt[c + 1]++;
  }
  for (int c = 0; c < Nt; ++c) cnt[c + 1] += cnt[c];
  std::vector<int> pos(cnt.begin(), cnt.end() - 1);
  std::vector<double> kc(M_nodes);
  for (int j = 0; j < M_nodes; ++j) {
    const int p = pos[cell[j]]++;
    jc[p] = j;
    kc[p] = k[j];
  }
  Geom g{};
  g.D = 1;
  g.M = M_nodes;
  g.B = 1;
  g.m = M;
  g.Nt[0] = Nt;
  g.N[0] = Nt / 2;
  g.Ntd[0] = Nt;
  g.grid_cells = Nt;
  g.ngrid_cells = Nt / 2;
  WinPolyN<double, 1, M> wp{};
  WinPoly<double> wpbig{};
  for (int l = 0; l < M; ++l)
    for (int z = 0; z <= DEG; ++z) wp.mu[0][l][z] = wpbig.mu[0][l][z] = 1e-3 * (l + 1) / (z + 1);
  double *d_kc, *d_wt = nullptr;
  int *d_jc, *d_cs;
  double2 *d_f, *d_grid, *d_out;
  cudaMalloc(&d_kc, M_nodes * 8);
  cudaMalloc(&d_jc, M_nodes * 4);
  cudaMalloc(&d_cs, (Nt + 1) * 4);
  cudaMalloc(&d_f, M_nodes * 16);
  cudaMalloc(&d_out, M_nodes * 16);
  cudaMalloc(&d_grid, (size_t)Nt * 16);
  cudaMemcpy(d_kc, kc.data(), M_nodes * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_jc, jc.data(), M_nodes * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cs, cnt.data(), (Nt + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemset(d_f, 0, M_nodes * 16);
  cudaMemset(d_grid, 0, (size_t)Nt * 16);
  void* flush;
  const size_t FL = 512ull << 20;
  cudaMalloc(&flush, FL);
  const size_t sb = s1_smem_bytes(M, 16, 8), ib = i1_smem_bytes(M, 16);
  cudaFuncSetAttribute((const void*)SPREAD1<double, M, DEG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
  cudaFuncSetAttribute((const void*)interp1s_kernel<double, M, DEG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ib);
  const unsigned segs_s = std::min<unsigned>((Nt + S1_SEG - 1) / S1_SEG, g_s1cap ? g_s1cap * 148 : 1u << 30), segs_i = (Nt + I1_SEG - 1) / I1_SEG;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  {  // back-to-back launches (warm): per-launch time of each kernel and of empty kernels
    cudaStream_t st;
    cudaStreamCreate(&st);
    auto b2b = [&](auto launch) {
      for (int i = 0; i < 3; ++i) launch();
      cudaEventRecord(e0, st);
      for (int i = 0; i < 20; ++i) launch();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      return ms * 1e3f / 20;
    };
    const float ts = b2b([&] {
      SPREAD1<double, M, DEG, false><<<dim3(segs_s, 1), S1_THREADS, sb, st>>>(g, wp, d_f, d_kc, d_wt, d_jc, d_cs, 0,
                                                                                    M_nodes, d_grid);
    });
    const float ti = b2b([&] {
      interp1s_kernel<double, M, DEG, false><<<dim3(segs_i, 1), I1_THREADS, ib, st>>>(g, wp, d_grid, d_kc, d_wt, d_jc, d_cs, 0, M_nodes,
                                                                                d_out);
    });
    const float te = b2b([&] { empty_kernel<double><<<1024, 128, 0, st>>>(g, wpbig, d_out); });
    const float tes = b2b([&] { empty_small<<<1024, 128, 0, st>>>(d_out, 1); });
    const float tes1 = b2b([&] { empty_small<<<1, 32, 0, st>>>(d_out, 1); });
    int* d_inv;
    cudaMalloc(&d_inv, M_nodes * 4);
    {
      std::vector<int> inv(M_nodes);
      for (int p = 0; p < M_nodes; ++p) inv[jc[p]] = p;
      cudaMemcpy(d_inv, inv.data(), M_nodes * 4, cudaMemcpyHostToDevice);
    }
    const float tperm = b2b([&] { permute_scatter<<<(M_nodes + 255) / 256, 256, 0, st>>>(d_f, d_inv, d_out, M_nodes); });
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i)
      SPREAD1<double, M, DEG, false><<<dim3(segs_s, 1), S1_THREADS, sb, st>>>(g, wp, d_f, d_kc, d_wt, d_jc, d_cs, 0,
                                                                                    M_nodes, d_grid);
    cudaStreamEndCapture(st, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    const float tg = b2b([&] { cudaGraphLaunch(ge, st); }) / 20;
    printf("{\"b2b_us\": {\"spread1a\": %.2f, \"interp1s\": %.2f, \"spread1a_graph\": %.2f, \"empty_1024x128_bigparams\": %.2f, "
           "\"empty_1024x128\": %.2f, \"empty_1x32\": %.2f, \"permute_scatter\": %.2f}}\n", ts, ti, tg, te, tes, tes1, tperm);
  }
  for (int which = 0; which < 2; ++which) {
    const unsigned nctas = which == 0 ? segs_s : segs_i;
    std::vector<unsigned long long> tr(nctas * 8);
    float best = 1e9f;
    std::vector<unsigned long long> keep;
    for (int rep = 0; rep < 6; ++rep) {
      if (g_flush) {
        cudaMemset(flush, rep, FL);
        cudaMemset(flush, 0, 64);
      }
      cudaMemcpyToSymbol(nfftb_trace, tr.data(), 0);  // no-op, keeps symbol referenced
      cudaEventRecord(e0);
      if (which == 0)
        SPREAD1<double, M, DEG, false><<<dim3(segs_s, 1), S1_THREADS, sb>>>(g, wp, d_f, d_kc, d_wt, d_jc, d_cs, 0,
                                                                                   M_nodes, d_grid);
      else
        interp1s_kernel<double, M, DEG, false><<<dim3(segs_i, 1), I1_THREADS, ib>>>(g, wp, d_grid, d_kc, d_wt, d_jc, d_cs, 0, M_nodes,
                                                                            d_out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) {
        best = ms;
        cudaMemcpyFromSymbol(tr.data(), nfftb_trace, nctas * 8 * 8);
        keep = tr;
      }
    }
    const int nslots = which == 0 ? 5 : 3;
    unsigned long long t0 = ~0ull;
    for (unsigned c = 0; c < nctas; ++c) t0 = std::min(t0, keep[c * 8 + 0]);
    printf("{\"l2\": \"%s\", \"kernel\": \"%s\", \"m\": %d, \"ctas\": %u, \"event_us\": %.2f, \"phases\": [", g_flush ? "flushed" : "warm", which == 0 ? "spread1a" : "interp1s",
           M, nctas, best * 1e3);
    for (int s = 0; s < nslots; ++s) {
      std::vector<double> v;
      for (unsigned c = 0; c < nctas; ++c) v.push_back((keep[c * 8 + s] - t0) * 1e-3);
      std::sort(v.begin(), v.end());
      printf("%s{\"slot\": %d, \"min\": %.2f, \"p10\": %.2f, \"p50\": %.2f, \"p90\": %.2f, \"max\": %.2f}", s ? ", " : "", s, v[0],
             v[v.size() / 10], v[v.size() / 2], v[v.size() * 9 / 10], v.back());
    }
    printf("], \"durations\": [");
    for (int s = 1; s < nslots; ++s) {  // per-CTA phase durations (slot s - slot s-1)
      std::vector<double> v;
      for (unsigned c = 0; c < nctas; ++c) v.push_back(((double)keep[c * 8 + s] - (double)keep[c * 8 + s - 1]) * 1e-3);
      std::sort(v.begin(), v.end());
      printf("%s{\"phase\": %d, \"p10\": %.2f, \"p50\": %.2f, \"p90\": %.2f, \"max\": %.2f}", s > 1 ? ", " : "", s,
             v[v.size() / 10], v[v.size() / 2], v[v.size() * 9 / 10], v.back());
    }
    printf("]}\n");
  }
  cudaFree(d_kc);
  cudaFree(d_jc);
  cudaFree(d_cs);
  cudaFree(d_f);
  cudaFree(d_out);
  cudaFree(d_grid);
  cudaFree(flush);
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 4;
  if (argc > 2 && std::string(argv[2]) == "warm") g_flush = false;
  if (getenv("S1CAP")) g_s1cap = atoi(getenv("S1CAP"));
  if (m == 8) run<8>(1 << 18, 1 << 19);
  else run<4>(1 << 18, 1 << 19);
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
