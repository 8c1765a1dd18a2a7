// Microbenchmark: cost of cooperative-groups grid barriers and of a launch gap
// on B200 (diagnostic for the precompute design; not part of the library).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int n, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = n;
}
__global__ void k_empty(int* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = 1; }
__global__ void k_atomic(int* cnt, int nbins, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[(i * 2654435761u) % nbins], 1);
}
int main() {
  int* d; cudaMalloc(&d, 64 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {64, 128, 148, 296, 592}) for (int thr : {256, 512}) {
    for (int n : {0, 1, 4, 16}) {
      void* args[] = {&n, &d};
      float best = 1e9;
      for (int r = 0; r < 20; ++r) {
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k_sync, grid, thr, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("grid %d thr %d: %s\n", grid, thr, cudaGetErrorString(e)); cudaGetLastError(); break; }
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("grid %4d thr %3d syncs %2d: %.2f us\n", grid, thr, n, best * 1e3);
    }
  }
  // graph of K empty kernels back to back
  for (int K : {1, 2, 4, 8}) {
    cudaStream_t s; cudaStreamCreate(&s);
    cudaGraph_t gr; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < K; ++k) k_empty<<<148, 256, 0, s>>>(d);
    cudaStreamEndCapture(s, &gr); cudaGraphInstantiate(&ge, gr, 0);
    float best = 1e9;
    for (int r = 0; r < 50; ++r) {
      cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("graph of %d empty kernels: %.2f us\n", K, best * 1e3);
  }
  for (int nb : {1024, 4096, 1 << 19}) {
    int n = 1 << 18;
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
      cudaMemset(d, 0, nb * 4);
      cudaEventRecord(a); k_atomic<<<(n + 255) / 256, 256>>>(d, nb, n); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("2^18 global atomicAdd over %d bins: %.2f us\n", nb, best * 1e3);
  }
  return 0;
}
