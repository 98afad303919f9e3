// Microbenchmark of the per-tile FP64 DMMA GEMM ([M x K] smem  x  [K x N] weights)
// at Barcelona dims (GEMM1: K=180, N=104; GEMM2: K=100, N=184), comparing
//   (a) B fragments from L2 with an R-deep register prefetch ring, per warp
//   (b) B staged through shared memory by cp.async.bulk (TMA bulk copy) k-chunks
// One CTA per SM, 13 warps, repeated many times; reports cycles per GEMM and the
// fraction of the DMMA issue bound (16 cycles per DMMA per SM sub-partition).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int kWarps = 13, kThreads = kWarps * 32;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
extern __shared__ __align__(128) double sm[];

template <int MT, int R>
__global__ void __launch_bounds__(kThreads, 1) gemm_l2(const double* __restrict__ Bf, int KS, int NT, int lda, int reps, double* out, long long* cyc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ar = lane >> 2, ac = lane & 3;
  for (int i = threadIdx.x; i < 96 * lda; i += kThreads) sm[i] = 1e-3 * (i % 17);
  __syncthreads();
  const double* As = sm + ar * lda + ac;
  double sink = 0;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    for (int nt = warp; nt < NT; nt += kWarps) {
      double acc[MT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0;
      const double* bp = Bf + (size_t)nt * KS * 32 + lane;
      double bq[R];
#pragma unroll
      for (int q = 0; q < R; ++q) bq[q] = q < KS ? __ldg(bp + q * 32) : 0.0;
      for (int ks0 = 0; ks0 < KS; ks0 += R) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int ks = ks0 + q;
          if (ks < KS) {
            double af[MT];
#pragma unroll
            for (int m = 0; m < MT; ++m) af[m] = As[m * 8 * lda + ks * 4];
#pragma unroll
            for (int m = 0; m < MT; ++m) dmma(acc[m], af[m], bq[q]);
            if (ks + R < KS) bq[q] = __ldg(bp + (ks + R) * 32);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) sink += acc[m][0] + acc[m][1];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * kThreads + threadIdx.x] = sink;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / reps;
}

// (b): B k-chunks of KC k-steps x all NT n-tiles ([ks][nt][32] order) streamed into a
// ring of S smem stages by one thread with cp.async.bulk + mbarrier; all warps consume.
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(b)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
               :: "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                  "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

template <int MT, int KC, int S>
__global__ void __launch_bounds__(kThreads, 1) gemm_tma(const double* __restrict__ Bk, int KS, int NT, int lda, int reps, double* out, long long* cyc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ar = lane >> 2, ac = lane & 3;
  double* A = sm;
  double* Bs = sm + 96 * lda;                       // S stages x (KC*NT*32) doubles
  uint64_t* full = (uint64_t*)(Bs + S * KC * NT * 32);
  uint64_t* empty = full + S;
  for (int i = threadIdx.x; i < 96 * lda; i += kThreads) A[i] = 1e-3 * (i % 17);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, kWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int nchunks = (KS + KC - 1) / KC;
  const uint32_t stage_doubles = KC * NT * 32;
  const double* As = A + ar * lda + ac;
  double sink = 0;
  long long t0 = clock64();
  uint32_t gk = 0;  // global chunk counter (ring position)
  for (int rep = 0; rep < reps; ++rep) {
    // producer: prefetch up to S chunks ahead (thread 0)
    double acc[2][MT][2];
    const int nt0 = warp, nt1 = warp + kWarps;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int m = 0; m < MT; ++m) acc[t][m][0] = acc[t][m][1] = 0;
    if (threadIdx.x == 0) {
      for (int c = 0; c < S && c < nchunks; ++c) {
        const uint32_t g = gk + c, s = g % S;
        if (g >= S) mbar_wait(empty + s, ((g / S) - 1) & 1);
        const int k0 = c * KC, kc = min(KC, KS - k0);
        mbar_expect(full + s, kc * NT * 32 * 8);
        bulk_g2s(Bs + s * stage_doubles, Bk + (size_t)k0 * NT * 32, kc * NT * 32 * 8, full + s);
      }
    }
    for (int c = 0; c < nchunks; ++c) {
      const uint32_t g = gk + c, s = g % S;
      mbar_wait(full + s, (g / S) & 1);
      const int k0 = c * KC, kc = min(KC, KS - k0);
      const double* bst = Bs + s * stage_doubles;
      for (int kk = 0; kk < kc; ++kk) {
        const int ks = k0 + kk;
        double af[MT];
#pragma unroll
        for (int m = 0; m < MT; ++m) af[m] = As[m * 8 * lda + ks * 4];
        const double b0 = bst[(kk * NT + nt0) * 32 + lane];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma(acc[0][m], af[m], b0);
        if (nt1 < NT) {
          const double b1 = bst[(kk * NT + nt1) * 32 + lane];
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(acc[1][m], af[m], b1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (threadIdx.x == 0 && c + S < nchunks) {
        const uint32_t gn = g + S, sn = gn % S;
        mbar_wait(empty + sn, ((gn / S) - 1) & 1);
        const int kn = (c + S) * KC, kcn = min(KC, KS - kn);
        mbar_expect(full + sn, kcn * NT * 32 * 8);
        bulk_g2s(Bs + sn * stage_doubles, Bk + (size_t)kn * NT * 32, kcn * NT * 32 * 8, full + sn);
      }
    }
    gk += nchunks;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int m = 0; m < MT; ++m) sink += acc[t][m][0] + acc[t][m][1];
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * kThreads + threadIdx.x] = sink;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = (t1 - t0) / reps;
}

template <int MT, int R>
int run_l2(const double* B, int KS, int NT, int lda, double* out, long long* dc, int ctas, size_t smem_force = 0) {
  size_t smem = smem_force ? smem_force : 96 * lda * 8;
  CK(cudaFuncSetAttribute(gemm_l2<MT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gemm_l2<MT, R><<<ctas, kThreads, smem>>>(B, KS, NT, lda, 2, out, dc);
  CK(cudaDeviceSynchronize());
  gemm_l2<MT, R><<<ctas, kThreads, smem>>>(B, KS, NT, lda, 50, out, dc);
  long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
  // DMMA bound: busiest SMSP (warps w, w+4, ...) * n-tiles * KS * MT * 16 cycles
  int busiest = 0;
  for (int s = 0; s < 4; ++s) { int n = 0; for (int w = s; w < kWarps; w += 4) for (int nt = w; nt < NT; nt += kWarps) ++n; busiest = n > busiest ? n : busiest; }
  double bound = (double)busiest * KS * MT * 16;
  printf("  L2 ring R=%2d MT=%2d KS=%3d NT=%2d ctas=%3d smem=%zu: %7lld cyc  bound %7.0f  (%.0f%%)\n", R, MT, KS, NT, ctas, smem, c, bound, 100 * bound / c);
  return 0;
}

template <int MT, int KC, int S>
int run_tma(const double* B, int KS, int NT, int lda, double* out, long long* dc, int ctas) {
  size_t smem = 96 * lda * 8 + (size_t)S * KC * NT * 32 * 8 + 2 * S * 8;
  CK(cudaFuncSetAttribute(gemm_tma<MT, KC, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gemm_tma<MT, KC, S><<<ctas, kThreads, smem>>>(B, KS, NT, lda, 2, out, dc);
  CK(cudaDeviceSynchronize());
  gemm_tma<MT, KC, S><<<ctas, kThreads, smem>>>(B, KS, NT, lda, 50, out, dc);
  long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
  int busiest = 0;
  for (int s = 0; s < 4; ++s) { int n = 0; for (int w = s; w < kWarps; w += 4) for (int nt = w; nt < NT; nt += kWarps) ++n; busiest = n > busiest ? n : busiest; }
  double bound = (double)busiest * KS * MT * 16;
  printf("  TMA KC=%d S=%d   MT=%2d KS=%3d NT=%2d ctas=%3d: %7lld cyc  bound %7.0f  (%.0f%%)  smem %zu\n", KC, S, MT, KS, NT, ctas, c, bound, 100 * bound / c, smem);
  return 0;
}

int main() {
  double *B, *out; long long* dc;
  CK(cudaMalloc(&B, 64 << 20)); CK(cudaMalloc(&out, 8 << 20)); CK(cudaMalloc(&dc, 8));
  CK(cudaMemset(B, 0, 64 << 20));
  for (size_t sm : {(size_t)0, (size_t)219280}) {
    run_l2<3, 8>(B, 45, 13, 180, out, dc, 148, sm);
    run_l2<11, 8>(B, 45, 13, 180, out, dc, 148, sm);
    run_l2<11, 16>(B, 45, 13, 180, out, dc, 148, sm);
    run_l2<3, 8>(B, 25, 23, 100, out, dc, 148, sm);
    run_l2<11, 8>(B, 25, 23, 100, out, dc, 148, sm);
  }
  return 0;
}
