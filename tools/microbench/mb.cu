// Microbenchmarks used to size the APG kernel design on B200 (sm_100a):
// FP64 DFMA vs DMMA throughput, software grid-barrier latency, single-SM L2 stream rate.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = threadIdx.x * 2e-3;
  double c[4][4];
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) c[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0; for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16k16_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
  for (int q = 0; q < 4; ++q) b[q] = threadIdx.x * 2e-3 + q;
  double c[4][4];
  for (int t = 0; t < 4; ++t) for (int q = 0; q < 4; ++q) c[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ unsigned int g_bar_count;
__device__ volatile unsigned int g_bar_gen;

__device__ __forceinline__ void grid_barrier(unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int target = gen + 1;
    __threadfence();
    unsigned int arrived = atomicAdd(&g_bar_count, 1);
    if (arrived == nblocks - 1) {
      g_bar_count = 0;
      __threadfence();
      g_bar_gen = target;
    } else {
      while (g_bar_gen != target) { }
    }
    __threadfence();
  }
  gen += 1;
  __syncthreads();
}

__global__ void barrier_kernel(int iters, unsigned long long* t) {
  unsigned int gen = g_bar_gen;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) grid_barrier(gridDim.x, gen);
  if (blockIdx.x == 0 && threadIdx.x == 0) *t = clock64() - t0;
}

__global__ void cg_barrier_kernel(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}

__global__ void l2_stream_kernel(const double* __restrict__ m, int n, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += __ldcg(m + i);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d clock %d kHz l2 %d\n", prop.name, prop.multiProcessorCount, prop.clockRate, prop.l2CacheSize);
  int nsm = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  for (int bpsm : {1, 2, 4}) {
    int threads = 512, iters = 4000;
    dfma_kernel<<<nsm * bpsm, threads>>>(out, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_kernel<<<nsm * bpsm, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)threads * nsm * bpsm;
    printf("DFMA blocks/sm=%d: %.2f TFLOP/s\n", bpsm, flops / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4}) {
    int threads = 256, iters = 4000;
    dmma_kernel<<<nsm * bpsm, threads>>>(out, 10);
    cudaEventRecord(e0); dmma_kernel<<<nsm * bpsm, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * iters * (threads / 32.0) * nsm * bpsm;
    printf("DMMA m8n8k4 blocks/sm=%d: %.2f TFLOP/s\n", bpsm, flops / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4}) {
    int threads = 256, iters = 4000;
    dmma16_kernel<<<nsm * bpsm, threads>>>(out, 10);
    cudaEventRecord(e0); dmma16_kernel<<<nsm * bpsm, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 512 * 4 * iters * (threads / 32.0) * nsm * bpsm;
    printf("DMMA m16n8k4 blocks/sm=%d: %.2f TFLOP/s\n", bpsm, flops / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4}) {
    int threads = 256, iters = 1000;
    dmma16k16_kernel<<<nsm * bpsm, threads>>>(out, 10);
    cudaEventRecord(e0); dmma16k16_kernel<<<nsm * bpsm, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 2048 * 4 * iters * (threads / 32.0) * nsm * bpsm;
    printf("DMMA m16n8k16 blocks/sm=%d: %.2f TFLOP/s\n", bpsm, flops / ms / 1e9);
  }
  // grid barrier
  unsigned long long* dt; CK(cudaMalloc(&dt, 8));
  for (int threads : {256, 512}) {
    int iters = 20000;
    barrier_kernel<<<nsm, threads>>>(100, dt);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); barrier_kernel<<<nsm, threads>>>(iters, dt); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("sw grid barrier (%d CTAs x %d thr): %.3f us per barrier\n", nsm, threads, ms * 1e3 / iters);
  }
  {
    int iters = 20000; void* args[] = {&iters};
    CK(cudaLaunchCooperativeKernel((void*)cg_barrier_kernel, nsm, 256, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); CK(cudaLaunchCooperativeKernel((void*)cg_barrier_kernel, nsm, 256, args, 0, 0)); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync (%d CTAs): %.3f us per barrier\n", nsm, ms * 1e3 / iters);
  }
  // single-SM L2 stream of a 150 kB matrix
  {
    double* m; CK(cudaMalloc(&m, 150 * 1024)); cudaMemset(m, 0, 150 * 1024);
    int n = 150 * 1024 / 8, reps = 200;
    for (int blocks : {1, 148}) {
      l2_stream_kernel<<<blocks, 512>>>(m, n, 2, out);
      cudaEventRecord(e0); l2_stream_kernel<<<blocks, 512>>>(m, n, reps, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("L2 stream %d CTA(s): %.1f GB/s per CTA\n", blocks, (double)n * 8 * reps / ms / 1e6);
    }
  }
  // launch latency of empty graph-free kernel
  {
    cudaEventRecord(e0);
    for (int i = 0; i < 1000; ++i) cg_barrier_kernel<<<nsm, 256>>>(0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("back-to-back empty launches: %.2f us each\n", ms);
  }
  return 0;
}
