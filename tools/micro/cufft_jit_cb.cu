// Capability probe (diagnostic): which LTO-IR flavours does cufftXtSetJITCallback +
// cufftMakePlan accept on this box with the toolkit's cuFFT?
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include <cufftXt.h>
#include <nvrtc.h>
static const char* src = R"(
extern "C" __device__ double2 ld_z(void* in, unsigned long long off, void* info, void*) {
  return ((const double2*)info)[off];
}
)";
static std::string nvrtc(std::vector<const char*> opts) {
  nvrtcProgram prog; nvrtcCreateProgram(&prog, src, "cb.cu", 0, nullptr, nullptr);
  nvrtcResult r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  size_t n = 0; nvrtcGetLTOIRSize(prog, &n);
  std::string ir(n, '\0'); if (n) nvrtcGetLTOIR(prog, &ir[0]);
  if (r != NVRTC_SUCCESS) { size_t l; nvrtcGetProgramLogSize(prog, &l); std::string log(l, 0); nvrtcGetProgramLog(prog, &log[0]); printf("log: %s\n", log.c_str()); }
  return ir;
}
static void probe(const char* tag, const std::string& ir, double2* d) {
  cufftHandle h; cufftCreate(&h);
  cufftResult a = cufftXtSetJITCallback(h, "ld_z", ir.data(), ir.size(), CUFFT_CB_LD_COMPLEX_DOUBLE, (void**)&d);
  size_t ws = 0;
  cufftResult b = cufftMakePlan1d(h, 4096, CUFFT_Z2Z, 1, &ws);
  printf("%-28s ir %6zu B: setJIT %d makePlan %d\n", tag, ir.size(), (int)a, (int)b);
  cufftDestroy(h);
}
int main(int argc, char** argv) {
  int v = 0; cufftGetVersion(&v); printf("cufft version %d\n", v);
  double2* d; cudaMalloc(&d, (1 << 19) * 16);
  probe("nvrtc sm_100 dlto rdc", nvrtc({"--gpu-architecture=sm_100", "-dlto", "-rdc=true"}), d);
  probe("nvrtc sm_100 dlto", nvrtc({"--gpu-architecture=sm_100", "-dlto"}), d);
  probe("nvrtc compute_100 dlto rdc", nvrtc({"--gpu-architecture=compute_100", "-dlto", "-rdc=true"}), d);
  probe("nvrtc sm_100a dlto rdc", nvrtc({"--gpu-architecture=sm_100a", "-dlto", "-rdc=true"}), d);
  for (int i = 1; i < argc; ++i) {
    std::ifstream f(argv[i], std::ios::binary); std::stringstream ss; ss << f.rdbuf();
    probe(argv[i], ss.str(), d);
  }
  return 0;
}
