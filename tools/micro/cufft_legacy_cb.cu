// Probe + timing (diagnostic): the resampling correction fused
// into cuFFT's LEGACY load/store callbacks (static cuFFT, relocatable device
// code), against the unfused deconv-kernel + FFT and FFT + crop-kernel pairs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=true -o cufft_legacy_cb cufft_legacy_cb.cu \
//        -lcufft_static -lculibos
//
// Per size: forward = out-of-place FFT whose load callback returns
// fhat[n] * beta[n] inside the N-region and 0 in the padding (Alg. 1 l.1-3 +
// FFT); adjoint = in-place inverse FFT whose store callback writes only the
// N-region, times beta, into y (FFT + Alg. 2 l.7-9). Times are per exec,
// mean of 50 back-to-back launches after warm-up (L2-warm).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cufft.h>
#include <cufftXt.h>

struct CbInfo {
  int D;
  int N[3], Nt[3];
  long long cells, ncells;
  const double2* fhat;
  double2* y;
  const double* beta;  // sum N_d
};

__device__ __forceinline__ bool decode(const CbInfo* ci, size_t off, long long& b, long long& nidx, double& w) {
  b = (long long)(off / ci->cells);
  long long r = (long long)(off - b * ci->cells);
  int s[3];
  for (int d = ci->D - 1; d >= 0; --d) {
    s[d] = (int)(r % ci->Nt[d]);
    r /= ci->Nt[d];
  }
  nidx = 0;
  w = 1.0;
  int boff = 0;
  for (int d = 0; d < ci->D; ++d) {
    const int h = ci->N[d] >> 1;
    int i;
    if (s[d] < h) i = s[d] + h;
    else if (s[d] >= ci->Nt[d] - h) i = s[d] - (ci->Nt[d] - h);
    else return false;
    nidx = nidx * ci->N[d] + i;
    w *= ci->beta[boff + i];
    boff += ci->N[d];
  }
  return true;
}

__device__ cufftDoubleComplex load_deconv(void* in, size_t off, void* info, void*) {
  const CbInfo* ci = (const CbInfo*)info;
  long long b, n;
  double w;
  if (!decode(ci, off, b, n, w)) return make_double2(0.0, 0.0);
  const double2 v = ci->fhat[b * ci->ncells + n];
  return make_double2(v.x * w, v.y * w);
}
__device__ void store_crop(void* out, size_t off, cufftDoubleComplex e, void* info, void*) {
  const CbInfo* ci = (const CbInfo*)info;
  long long b, n;
  double w;
  if (!decode(ci, off, b, n, w)) return;
  ci->y[b * ci->ncells + n] = make_double2(e.x * w, e.y * w);
}
__device__ cufftCallbackLoadZ d_load = load_deconv;
__device__ cufftCallbackStoreZ d_store = store_crop;

__global__ void deconv_kernel(const CbInfo* ci, double2* grid, long long total) {
  for (long long off = blockIdx.x * (long long)blockDim.x + threadIdx.x; off < total; off += (long long)gridDim.x * blockDim.x) {
    long long b, n;
    double w;
    if (decode(ci, off, b, n, w)) {
      const double2 v = ci->fhat[b * ci->ncells + n];
      grid[off] = make_double2(v.x * w, v.y * w);
    }
  }
}
__global__ void crop_kernel(const CbInfo* ci, const double2* grid, long long total) {
  for (long long off = blockIdx.x * (long long)blockDim.x + threadIdx.x; off < total; off += (long long)gridDim.x * blockDim.x) {
    long long b, n;
    double w;
    if (decode(ci, off, b, n, w)) {
      const double2 v = grid[off];
      ci->y[b * ci->ncells + n] = make_double2(v.x * w, v.y * w);
    }
  }
}

template <typename F>
static float per_exec_ms(F f, cudaStream_t st) {
  for (int i = 0; i < 5; ++i) f();
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  for (int i = 0; i < 50; ++i) f();
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 50;
}

static void run(int D, const int* N, int B) {
  CbInfo h{};
  h.D = D;
  h.cells = 1;
  h.ncells = 1;
  int nb = 0;
  for (int d = 0; d < D; ++d) {
    h.N[d] = N[d];
    h.Nt[d] = 2 * N[d];
    h.cells *= h.Nt[d];
    h.ncells *= N[d];
    nb += N[d];
  }
  const long long total = h.cells * B;
  double2 *fhat, *y, *g_in, *g;
  double* beta;
  cudaMalloc(&fhat, h.ncells * B * 16);
  cudaMalloc(&y, h.ncells * B * 16);
  cudaMalloc(&g_in, total * 16);
  cudaMalloc(&g, total * 16);
  cudaMalloc(&beta, nb * 8);
  cudaMemset(fhat, 0, h.ncells * B * 16);
  cudaMemset(g_in, 0, total * 16);
  std::vector<double> hb(nb, 1.0);
  cudaMemcpy(beta, hb.data(), nb * 8, cudaMemcpyHostToDevice);
  h.fhat = fhat;
  h.y = y;
  h.beta = beta;
  CbInfo* dci;
  cudaMalloc(&dci, sizeof(CbInfo));
  cudaMemcpy(dci, &h, sizeof(CbInfo), cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  int n[3] = {h.Nt[0], h.Nt[1], h.Nt[2]};
  cufftHandle plain, cbf, cba;
  size_t ws;
  cufftCreate(&plain);
  cufftCreate(&cbf);
  cufftCreate(&cba);
  int r0 = cufftMakePlanMany(plain, D, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, B, &ws);
  int r1 = cufftMakePlanMany(cbf, D, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, B, &ws);
  int r2 = cufftMakePlanMany(cba, D, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, B, &ws);
  cufftCallbackLoadZ hl;
  cufftCallbackStoreZ hs;
  cudaMemcpyFromSymbol(&hl, d_load, sizeof(hl));
  cudaMemcpyFromSymbol(&hs, d_store, sizeof(hs));
  void* infos[1] = {dci};
  int r3 = cufftXtSetCallback(cbf, (void**)&hl, CUFFT_CB_LD_COMPLEX_DOUBLE, infos);
  int r4 = cufftXtSetCallback(cba, (void**)&hs, CUFFT_CB_ST_COMPLEX_DOUBLE, infos);
  cufftSetStream(plain, st);
  cufftSetStream(cbf, st);
  cufftSetStream(cba, st);
  const int ctas = 148 * 16;
  float t_fft = per_exec_ms([&] { cufftExecZ2Z(plain, g_in, g, CUFFT_FORWARD); }, st);
  float t_dec_fft = per_exec_ms([&] {
    deconv_kernel<<<ctas, 256, 0, st>>>(dci, g_in, total);
    cufftExecZ2Z(plain, g_in, g, CUFFT_FORWARD);
  }, st);
  float t_cb_fwd = per_exec_ms([&] { cufftExecZ2Z(cbf, g_in, g, CUFFT_FORWARD); }, st);
  float t_fft_crop = per_exec_ms([&] {
    cufftExecZ2Z(plain, g, g, CUFFT_INVERSE);
    crop_kernel<<<ctas, 256, 0, st>>>(dci, g, total);
  }, st);
  float t_cb_adj = per_exec_ms([&] { cufftExecZ2Z(cba, g, g, CUFFT_INVERSE); }, st);
  printf("{\"D\": %d, \"Nt\": [%d, %d, %d], \"B\": %d, \"plan_rc\": [%d, %d, %d], \"setcb_rc\": [%d, %d], "
         "\"fft_ms\": %.4f, \"deconv_plus_fft_ms\": %.4f, \"fft_with_load_cb_ms\": %.4f, "
         "\"ifft_plus_crop_ms\": %.4f, \"ifft_with_store_cb_ms\": %.4f, \"err\": \"%s\"}\n",
         D, n[0], D > 1 ? n[1] : 1, D > 2 ? n[2] : 1, B, r0, r1, r2, r3, r4, t_fft, t_dec_fft, t_cb_fwd, t_fft_crop,
         t_cb_adj, cudaGetErrorString(cudaGetLastError()));
  cufftDestroy(plain);
  cufftDestroy(cbf);
  cufftDestroy(cba);
  cudaFree(fhat);
  cudaFree(y);
  cudaFree(g_in);
  cudaFree(g);
  cudaFree(beta);
  cudaFree(dci);
  cudaStreamDestroy(st);
}

int main() {
  int v = 0;
  cufftGetVersion(&v);
  printf("{\"cufft_version\": %d}\n", v);
  int n1[1] = {262144};
  run(1, n1, 1);
  int n2[2] = {512, 512};
  run(2, n2, 1);
  int n3[3] = {64, 64, 64};
  run(3, n3, 1);
  return 0;
}
