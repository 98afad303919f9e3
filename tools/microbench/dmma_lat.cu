// DMMA m8n8k4 latency / per-warp throughput vs number of independent accumulator chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void chains(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[C][2];
  for (int t = 0; t < C; ++t) c[t][0] = c[t][1] = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < C; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0; for (int t = 0; t < C; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void dfma_chain(double* out, int iters, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = fma(x, 1.0000001, 1e-9); x = fma(x, 1.0000001, 1e-9); x = fma(x, 1.0000001, 1e-9); x = fma(x, 1.0000001, 1e-9); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int C> void run(double* out, long long* dc, int warps) {
  int iters = 2000; long long cyc;
  chains<C><<<1, 32 * warps>>>(out, 10, dc); cudaDeviceSynchronize();
  chains<C><<<1, 32 * warps>>>(out, iters, dc); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("warps=%2d chains=%2d: %.1f cycles per DMMA-round (per chain step), %.2f DMMA/clk/SM\n", warps, C,
         (double)cyc / iters, (double)C * warps * iters / cyc);
}
int main() {
  double* out; long long* dc; cudaMalloc(&out, 1 << 20); cudaMalloc(&dc, 8);
  for (int w : {1, 4, 8, 16}) { run<1>(out, dc, w); run<2>(out, dc, w); run<4>(out, dc, w); run<8>(out, dc, w); run<16>(out, dc, w); }
  long long cyc; dfma_chain<<<1, 32>>>(out, 10, dc); cudaDeviceSynchronize();
  dfma_chain<<<1, 32>>>(out, 2000, dc); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", (double)cyc / 8000);
  return 0;
}
