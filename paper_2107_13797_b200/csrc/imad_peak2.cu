// Integer-pipe roofline microbenchmark, second cut (B200, sm_100a).
//
// The first cut (imad_peak.cu) kept the multiplier operands loop-invariant, and ptxas strength-reduced
// the "wide" and "lohi" loops into plain 64-bit additions -- only its carry-chain figure
// (IMAD.WIDE.U32.X) was a real multiply rate.  Here the multiplier changes every iteration and the
// SASS of every variant is checked (tools/sass_hist.sh) before a number is believed.
//
// One "LP" = one 32x32 -> 64-bit limb product folded into an accumulator.
//   wide_xor    : IMAD.WIDE.U32 (RZ addend) + one LOP3 per product          -> raw IMAD.WIDE issue rate
//   wide_add3   : two IMAD.WIDE.U32 + IADD3 + IADD3.X per two products      -> the mix ptxas makes of the
//                 Montgomery row in mont.cuh (acc += a*b + n*q)
//   wide_carry  : IMAD.WIDE.U32.X chains (32-bit-radix CIOS form)
//   lohi_xor    : IMAD (lo) + IMAD.HI + one LOP3 per product
//   alu_add3    : IADD3 only (ALU pipe reference)
// Prints one JSON line with LP/s (or op/s) per variant and per-SM-per-clock figures at the max clock.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int NACC = 24;

__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

__global__ void __launch_bounds__(256) k_wide_xor(uint64_t* out, uint32_t seed, int iters) {
  uint32_t a[NACC], x[NACC];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < NACC; i++) { a[i] = b * (2 * i + 3) + 12345u; x[i] = i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) {
      uint64_t p;
      asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[i]), "r"(b));
      x[i] = lop3_xor3(x[i], (uint32_t)p, (uint32_t)(p >> 32));
    }
    b += 0x9E3779B9u;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= x[i];
  if (s == 0x12345u) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_wide_add3(uint64_t* out, uint32_t seed, int iters) {
  uint32_t a[NACC], n[NACC];
  uint64_t acc[NACC];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u), q = b * 31u + 7u;
#pragma unroll
  for (int i = 0; i < NACC; i++) { a[i] = b * (2 * i + 3) + 12345u; n[i] = a[i] * 77u + i; acc[i] = i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(b));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(n[i]), "r"(q));
    }
    b += 0x9E3779B9u;
    q += 0x7F4A7C15u;
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= acc[i];
  if (s == 0x1234567ull) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_wide_carry(uint64_t* out, uint32_t seed, int iters) {
  constexpr int CH = 3, CL = 8;
  uint64_t acc[CH * CL];
  uint32_t a[CL], cy[CH];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < CH * CL; i++) acc[i] = (uint64_t)(b + i) * 0x9E3779B97F4A7C15ull;
#pragma unroll
  for (int i = 0; i < CL; i++) a[i] = b * (2 * i + 3) + 12345u;
#pragma unroll
  for (int c = 0; c < CH; c++) cy[c] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      uint64_t* A = acc + c * CL;
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
    b += 0x9E3779B9u;
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < CH * CL; i++) s ^= acc[i];
#pragma unroll
  for (int c = 0; c < CH; c++) s += cy[c];
  if (s == 0x1234567ull) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_lohi_xor(uint64_t* out, uint32_t seed, int iters) {
  uint32_t a[NACC], x[NACC];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
  for (int i = 0; i < NACC; i++) { a[i] = b * (2 * i + 3) + 12345u; x[i] = i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) {
      uint32_t lo, hi;
      asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(a[i]), "r"(b));
      asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a[i]), "r"(b));
      x[i] = lop3_xor3(x[i], lo, hi);
    }
    b += 0x9E3779B9u;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= x[i];
  if (s == 0x12345u) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_alu_add3(uint64_t* out, uint32_t seed, int iters) {
  uint32_t x[NACC];
  uint32_t b = seed ^ (threadIdx.x * 2654435761u), c = b * 3u;
#pragma unroll
  for (int i = 0; i < NACC; i++) x[i] = b + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) x[i] = x[i] + b + c;     // IADD3
    b ^= x[0];
    c += 0x7F4A7C15u;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s ^= x[i];
  if (s == 0x12345u) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, uint64_t* d_out, int reps, double ops_per_thread_iter) {
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
    double rate = ops_per_thread_iter * (double)iters * blocks * threads / (ms * 1e-3);
    if (rate > best) best = rate;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const int sms = prop.multiProcessorCount;
  uint64_t* d_out; CK(cudaMalloc(&d_out, (size_t)sms * 8 * 256 * sizeof(uint64_t)));
  const int blocks = sms * 8, threads = 256, iters = 4096, reps = 7;
  double wide_xor = run(k_wide_xor, blocks, threads, iters, d_out, reps, NACC);
  double wide_add3 = run(k_wide_add3, blocks, threads, iters, d_out, reps, 2.0 * NACC);
  double wide_carry = run(k_wide_carry, blocks, threads, iters, d_out, reps, 24.0);
  double lohi_xor = run(k_lohi_xor, blocks, threads, iters, d_out, reps, NACC);
  double alu_add3 = run(k_alu_add3, blocks, threads, iters, d_out, reps, NACC);
  // sustained (2 s) run of the mix the Montgomery kernels issue
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  int n = 0; float ms = 0;
  do {
    for (int i = 0; i < 8; i++) k_wide_add3<<<blocks, threads>>>(d_out, 7u + n + i, iters);
    n += 8;
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
  } while (ms < 2000.f);
  double sustained = 2.0 * NACC * (double)iters * blocks * threads * n / (ms * 1e-3);
  const double per = 1.0 / ((double)sms * clk_khz * 1e3);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_max_mhz\": %d, "
         "\"lp_per_s_wide_xor\": %.4e, \"lp_per_s_wide_add3\": %.4e, \"lp_per_s_wide_carry\": %.4e, "
         "\"lp_per_s_lohi_xor\": %.4e, \"iadd3_per_s\": %.4e, \"lp_per_s_wide_add3_sustained\": %.4e, "
         "\"per_sm_clk_at_max_clock\": {\"wide_xor\": %.2f, \"wide_add3\": %.2f, \"wide_carry\": %.2f, "
         "\"lohi_xor\": %.2f, \"iadd3\": %.2f}}\n",
         prop.name, sms, clk_khz / 1000, wide_xor, wide_add3, wide_carry, lohi_xor, alu_add3, sustained,
         wide_xor * per, wide_add3 * per, wide_carry * per, lohi_xor * per, alu_add3 * per);
  return 0;
}
