// FP64 instruction-mix throughput microbenchmark (development aid): warp-instructions
// per clock per SM for DFMA only, DMUL only, DADD only, and the K4 near kernel's mix
// (10 DFMA : 7 DMUL : 4 DADD), 16 warps per SM, 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void mix(double* out, int n, double a, double b, long long* cyc) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k + 1.0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int r = 0; r < 21; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (MODE == 0) x[k] = fma(x[k], a, b);
        else if (MODE == 1) x[k] = __dmul_rn(x[k], a);
        else if (MODE == 2) x[k] = __dadd_rn(x[k], b);
        else {  // the mix, by position in the 21-instruction group
          if (r < 10) x[k] = fma(x[k], a, b);
          else if (r < 17) x[k] = __dmul_rn(x[k], a);
          else x[k] = __dadd_rn(x[k], b);
        }
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* name) {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024 * 148); cudaMalloc(&c, 8 * 148);
  const int n = 256, warps = 16;
  mix<MODE><<<148, 32 * warps>>>(o, n, 0.9999999, 1e-9, c);
  mix<MODE><<<148, 32 * warps>>>(o, n, 0.9999999, 1e-9, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.3f FP64 warp-instructions per clock per SM (peak 2.0 at 64 lanes/clk)\n", name,
         (double)warps * n * 21 * 8 / (double)h);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<0>("DFMA only");
  run<1>("DMUL only");
  run<2>("DADD only");
  run<3>("10 DFMA : 7 DMUL : 4 DADD");
  return 0;
}
