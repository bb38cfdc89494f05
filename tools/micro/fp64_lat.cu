// FP64 dependent-latency / ILP microbenchmark (development aid).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void chain(double* out, int n, double a, double b, long long* cyc) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-3 + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int ILP>
void run(int warps) {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024 * 148); cudaMalloc(&c, 8 * 148);
  const int n = 4096;
  chain<ILP><<<148, 32 * warps>>>(o, n, 0.999999, 1e-7, c);
  chain<ILP><<<148, 32 * warps>>>(o, n, 0.999999, 1e-7, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (n * ILP);
  printf("ILP %2d warps/SM %2d: %.2f cycles per dependent DFMA step per warp, SM throughput %.2f DFMA-warp-instr/clk\n",
         ILP, warps, (double)h / n, warps * ILP / ((double)h / n));
  (void)per;
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1);
  run<1>(4); run<1>(8); run<1>(16); run<4>(8); run<4>(16); run<8>(16);
  return 0;
}
