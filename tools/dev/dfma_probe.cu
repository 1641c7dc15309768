// Feasibility probe for a floating-point big-integer multiplier on the B200 (sm_100a): the 52-bit-limb scheme that
// splits every limb product a*b (104 bits) into a high and a low half with two round-toward-zero FMAs,
//
//     hi  = fma_rz(a, b, 2^104)              -> 2^104 + floor(a*b / 2^52) * 2^52        (exact)
//     lo  = fma_rz(a, b, (2^104 + 2^52) - hi) -> 2^52 + (a*b mod 2^52)                    (exact)
//
// and accumulates the two bit patterns with 64-bit integer additions (biases removed once per column).  Per limb
// product: 2 DFMA + 1 DADD on the FP64 pipe, 2 x 64-bit integer adds on the ALU pipe.  The kernel below is the inner
// row of such a multiplier (N limbs of `a` against one limb `b` that changes every row) with everything in
// registers; it reports limb products per second and the equivalent bit^2 per clock per SM, next to the integer
// row of mont32.cuh (IMAD.WIDE.U32.X chains, 32-bit limbs).  It decides nothing by itself -- a real multiplier adds
// carry normalisation, the Montgomery quotient and int<->double conversions -- but it bounds what one could gain.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int N = 20;      // limbs per thread (20 x 52 = 1040 bits)

__global__ void __launch_bounds__(128) k_dfma_row(unsigned long long* out, uint32_t seed, int rows) {
  double a[N];
  long long acc_hi[N], acc_lo[N];
  const double C1 = 20282409603651670423947251286016.0;                 // 2^104
  const double C2 = 20282409603651670423947251286016.0 + 4503599627370496.0;   // 2^104 + 2^52
  uint32_t s = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
#pragma unroll
  for (int i = 0; i < N; i++) {
    s = s * 1664525u + 1013904223u;
    a[i] = (double)((((unsigned long long)s << 20) ^ (s * 2246822519ull)) & 0xfffffffffffffull);
    acc_hi[i] = 0; acc_lo[i] = 0;
  }
  double b = (double)(((unsigned long long)s * 2654435761ull) & 0xfffffffffffffull);
  for (int r = 0; r < rows; r++) {
#pragma unroll
    for (int i = 0; i < N; i++) {
      const double hi = __fma_rz(a[i], b, C1);
      const double sub = C2 - hi;
      const double lo = __fma_rz(a[i], b, sub);
      acc_hi[i] += __double_as_longlong(hi);
      acc_lo[i] += __double_as_longlong(lo);
    }
    b = (double)((__double_as_longlong(b) * 6364136223846793005ll + r) & 0xfffffffffffffll);   // next multiplier limb
  }
  unsigned long long x = 0;
#pragma unroll
  for (int i = 0; i < N; i++) x ^= (unsigned long long)acc_hi[i] + 3ull * (unsigned long long)acc_lo[i];
  if (x == 0x1234567ull) out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

constexpr int NI = 32;     // 32-bit limbs per thread in the integer row (1024 bits)

__global__ void __launch_bounds__(128) k_imad_row(unsigned long long* out, uint32_t seed, int rows) {
  uint32_t a[NI];
  uint64_t E[NI / 2], O[NI / 2];
  uint32_t cy = 0;
  uint32_t s = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
#pragma unroll
  for (int i = 0; i < NI; i++) { s = s * 1664525u + 1013904223u; a[i] = s; }
#pragma unroll
  for (int i = 0; i < NI / 2; i++) { E[i] = i; O[i] = 3 * i; }
  uint32_t b = s * 2246822519u;
  for (int r = 0; r < rows; r++) {
    // two carry chains per row, as mont32.cuh's mac_row
    asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %1, %2;\n\tadd.cc.u64 %0, %0, t;\n\t}" : "+l"(E[0]) : "r"(a[0]), "r"(b));
#pragma unroll
    for (int i = 1; i < NI / 2; i++)
      asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %1, %2;\n\taddc.cc.u64 %0, %0, t;\n\t}" : "+l"(E[i]) : "r"(a[2 * i]), "r"(b));
    asm volatile("addc.u32 %0, %0, 0;" : "+r"(cy));
    asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %1, %2;\n\tadd.cc.u64 %0, %0, t;\n\t}" : "+l"(O[0]) : "r"(a[1]), "r"(b));
#pragma unroll
    for (int i = 1; i < NI / 2; i++)
      asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %1, %2;\n\taddc.cc.u64 %0, %0, t;\n\t}" : "+l"(O[i]) : "r"(a[2 * i + 1]), "r"(b));
    asm volatile("addc.u32 %0, %0, 0;" : "+r"(cy));
    b = b * 1664525u + 1013904223u + (uint32_t)E[0];
  }
  unsigned long long x = cy;
#pragma unroll
  for (int i = 0; i < NI / 2; i++) x ^= E[i] + 3 * O[i];
  if (x == 0x1234567ull) out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <typename K>
static double run(K kern, int blocks, int threads, int rows, unsigned long long* d_out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int w = 0; w < 2; w++) kern<<<blocks, threads>>>(d_out, 17u + w, rows);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(d_out, 99u + r, rows);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best * 1e-3;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const int sms = prop.multiProcessorCount;
  unsigned long long* d_out; CK(cudaMalloc(&d_out, (size_t)sms * 16 * 128 * sizeof(unsigned long long)));
  const int threads = 128, rows = 8192;
  const double per = 1.0 / ((double)sms * clk_khz * 1e3);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_max_mhz\": %d, \"runs\": [", prop.name, sms, clk_khz / 1000);
  bool first = true;
  for (int bps : {2, 4, 8}) {
    const int blocks = sms * bps;
    const double thr = (double)blocks * threads * rows;
    const double td = run(k_dfma_row, blocks, threads, rows, d_out);
    const double ti = run(k_imad_row, blocks, threads, rows, d_out);
    const double pd = thr * N / td, pi = thr * NI / ti;
    printf("%s{\"warps_per_sm\": %d, \"dfma_limb_products_per_s\": %.4e, \"dfma_bit2_per_clk_sm\": %.0f, "
           "\"imad_limb_products_per_s\": %.4e, \"imad_bit2_per_clk_sm\": %.0f, \"ratio_bit2\": %.3f}",
           first ? "" : ", ", bps * threads / 32, pd, pd * per * 52.0 * 52.0, pi, pi * per * 1024.0,
           (pd * 52.0 * 52.0) / (pi * 1024.0));
    first = false;
  }
  printf("]}\n");
  return 0;
}
