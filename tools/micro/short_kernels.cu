// Microbenchmark (diagnostic, not part of the library): per-launch cost of
// short memory-bound kernels on B200 inside a CUDA graph (L2-warm, back to back),
// to set the floor for the 2^18-node precompute / resampling kernels.
#include <cstdio>
#include <cstdlib>
__global__ void k_empty(int) {}
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}
__global__ void k_gather(const double2* __restrict__ a, const int* __restrict__ idx, double2* __restrict__ b, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[idx[i]];
}
__global__ void k_gather2(const double2* __restrict__ a, const int* __restrict__ idx, double2* __restrict__ b, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[idx[idx[i]]];
}
__global__ void k_atomic(const int* __restrict__ idx, int* cnt, int* slot, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) slot[i] = atomicAdd(cnt + idx[i], 1);
}
__global__ void k_red(const int* __restrict__ idx, double* g, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    int c = idx[i] & ~7;
#pragma unroll
    for (int l = 0; l < 8; ++l) { atomicAdd(g + 2 * (c + l), 1.0); atomicAdd(g + 2 * (c + l) + 1, 1.0); }
  }
}
int main() {
  const int n = 1 << 18, ncell = 1 << 19;
  double2 *a, *b; int *idx, *cnt, *slot; double* g;
  cudaMalloc(&a, ncell * 16); cudaMalloc(&b, ncell * 16); cudaMalloc(&idx, n * 4); cudaMalloc(&cnt, ncell * 4);
  cudaMalloc(&slot, n * 4); cudaMalloc(&g, ncell * 16 + 256);
  int* h = (int*)malloc(n * 4);
  srand(1);
  for (int i = 0; i < n; ++i) h[i] = (int)(((unsigned)rand() * 2654435761u) % (unsigned)n);
  cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(cnt, 0, ncell * 4); cudaMemset(g, 0, ncell * 16);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int REP = 20;
  for (int thr : {128, 256, 512}) {
    int grid = (n + thr - 1) / thr;
    const char* names[] = {"empty", "copy 4MB", "gather 4MB", "gather2 4MB", "atomicAdd ret 2^18/2^19", "RED.F64 16/node"};
    for (int kind = 0; kind < 6; ++kind) {
      cudaGraph_t gr; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int r = 0; r < REP; ++r) {
        switch (kind) {
          case 0: k_empty<<<grid, thr, 0, s>>>(0); break;
          case 1: k_copy<<<grid, thr, 0, s>>>(a, b, n); break;
          case 2: k_gather<<<grid, thr, 0, s>>>(a, idx, b, n); break;
          case 3: k_gather2<<<grid, thr, 0, s>>>(a, idx, b, n); break;
          case 4: k_atomic<<<grid, thr, 0, s>>>(idx, cnt, slot, n); break;
          case 5: k_red<<<grid, thr, 0, s>>>(idx, g, n); break;
        }
      }
      cudaStreamEndCapture(s, &gr);
      cudaGraphInstantiate(&ge, gr, 0);
      float best = 1e9;
      for (int t = 0; t < 10; ++t) {
        cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("thr %3d %-26s %7.2f us per launch (graph of %d)\n", thr, names[kind], best * 1e3 / REP, REP);
      cudaGraphExecDestroy(ge); cudaGraphDestroy(gr);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
