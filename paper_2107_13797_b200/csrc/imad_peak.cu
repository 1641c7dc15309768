// Integer-multiply roofline microbenchmark for B200 (sm_100a).
//
// Measures the sustained rate of 32x32->64-bit limb products ("LP", SURVEY.md
// section 8d) that the SM integer-multiply pipe can retire, in the three forms a
// multi-precision kernel can use:
//   wide      : independent IMAD.WIDE.U32 (64-bit accumulate, no carry)
//   widecarry : IMAD.WIDE.U32.X chains with predicate carry-in/out (what the
//               Montgomery kernels in mont.cuh actually issue)
//   lohi      : separate IMAD + IMAD.HI (two instructions per limb product)
// Register-only; no memory traffic in the timed loop. Prints one JSON line.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad_peak imad_peak.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int CHAINS = 4;   // independent carry chains per thread
constexpr int CLEN = 8;     // IMAD.WIDE per chain

__global__ void __launch_bounds__(256) k_wide(uint64_t* out, uint32_t seed, int iters) {
  uint64_t acc[CHAINS * CLEN];
  uint32_t a[CLEN];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < CHAINS * CLEN; i++) acc[i] = (uint64_t)(b + i) * 0x9E3779B97F4A7C15ull;
#pragma unroll
  for (int i = 0; i < CLEN; i++) a[i] = b * (2 * i + 3) + 12345u;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++)
#pragma unroll
      for (int i = 0; i < CLEN; i++)
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[c * CLEN + i]) : "r"(a[i]), "r"(b));
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS * CLEN; i++) s ^= acc[i];
  if (s == 0x1234567ull) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_widecarry(uint64_t* out, uint32_t seed, int iters) {
  uint64_t acc[CHAINS * CLEN];
  uint32_t a[CLEN], cy[CHAINS];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < CHAINS * CLEN; i++) acc[i] = (uint64_t)(b + i) * 0x9E3779B97F4A7C15ull;
#pragma unroll
  for (int i = 0; i < CLEN; i++) a[i] = b * (2 * i + 3) + 12345u;
#pragma unroll
  for (int c = 0; c < CHAINS; c++) cy[c] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++) {
      uint64_t* A = acc + c * CLEN;
      asm volatile(
        "{\n\t.reg .u64 t0,t1,t2,t3,t4,t5,t6,t7;\n\t"
        "mul.wide.u32 t0, %9, %17;\n\t mul.wide.u32 t1, %10, %17;\n\t"
        "mul.wide.u32 t2, %11, %17;\n\t mul.wide.u32 t3, %12, %17;\n\t"
        "mul.wide.u32 t4, %13, %17;\n\t mul.wide.u32 t5, %14, %17;\n\t"
        "mul.wide.u32 t6, %15, %17;\n\t mul.wide.u32 t7, %16, %17;\n\t"
        "add.cc.u64 %0, %0, t0;\n\t addc.cc.u64 %1, %1, t1;\n\t"
        "addc.cc.u64 %2, %2, t2;\n\t addc.cc.u64 %3, %3, t3;\n\t"
        "addc.cc.u64 %4, %4, t4;\n\t addc.cc.u64 %5, %5, t5;\n\t"
        "addc.cc.u64 %6, %6, t6;\n\t addc.cc.u64 %7, %7, t7;\n\t"
        "addc.u32 %8, %8, 0;\n\t}"
        : "+l"(A[0]), "+l"(A[1]), "+l"(A[2]), "+l"(A[3]), "+l"(A[4]), "+l"(A[5]), "+l"(A[6]), "+l"(A[7]), "+r"(cy[c])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(b));
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS * CLEN; i++) s ^= acc[i];
#pragma unroll
  for (int c = 0; c < CHAINS; c++) s += cy[c];
  if (s == 0x1234567ull) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_lohi(uint64_t* out, uint32_t seed, int iters) {
  uint32_t lo[CHAINS * CLEN], hi[CHAINS * CLEN];
  uint32_t a[CLEN];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < CHAINS * CLEN; i++) { lo[i] = b + i; hi[i] = b * 7 + i; }
#pragma unroll
  for (int i = 0; i < CLEN; i++) a[i] = b * (2 * i + 3) + 12345u;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++)
#pragma unroll
      for (int i = 0; i < CLEN; i++) {
        asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(lo[c * CLEN + i]) : "r"(a[i]), "r"(b));
        asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(hi[c * CLEN + i]) : "r"(a[i]), "r"(b));
      }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS * CLEN; i++) s ^= ((uint64_t)hi[i] << 32) | lo[i];
  if (s == 0x1234567ull) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, uint64_t* d_out, int reps, double lp_per_thread_iter) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; w++) kern<<<blocks, threads>>>(d_out, 17u + w, iters);
  CK(cudaDeviceSynchronize());
  double best = 0.0;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(d_out, 99u + r, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
    double rate = lp_per_thread_iter * (double)iters * blocks * threads / (ms * 1e-3);
    if (rate > best) best = rate;
  }
  return best;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int threads = 256, bps = 4;            // 1024 threads/SM
  int blocks = sms * bps;
  int iters = argc > 1 ? atoi(argv[1]) : 20000;
  uint64_t* d_out; CK(cudaMalloc(&d_out, (size_t)blocks * threads * 8));
  double lp = CHAINS * CLEN;
  double wide = run(k_wide, blocks, threads, iters, d_out, 5, lp);
  double widec = run(k_widecarry, blocks, threads, iters, d_out, 5, lp);
  double lohi = run(k_lohi, blocks, threads, iters, d_out, 5, lp);
  // sustained: back-to-back for ~3 s with the carry form
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  int n_launch = 0; CK(cudaEventRecord(e0));
  for (; n_launch < 200; n_launch++) k_widecarry<<<blocks, threads>>>(d_out, n_launch, iters);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  double sustained = lp * (double)iters * blocks * threads * n_launch / (ms * 1e-3);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_max_mhz\": %.0f, "
         "\"lp_per_s_wide\": %.4e, \"lp_per_s_widecarry\": %.4e, \"lp_per_s_lohi\": %.4e, "
         "\"lp_per_s_widecarry_sustained\": %.4e, \"sustained_seconds\": %.2f, "
         "\"lp_per_clk_per_sm_widecarry_at_max_clock\": %.2f}\n",
         p.name, sms, clk_khz / 1000.0, wide, widec, lohi, sustained, ms * 1e-3,
         widec / (sms * (clk_khz * 1e3)));
  return 0;
}
