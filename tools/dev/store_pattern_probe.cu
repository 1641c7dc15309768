// Store-pattern probe for the encode kernel: how fast can the codec's access pattern go with no arithmetic at all?
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void st8(uint32_t* p, uint32_t v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "l"(p), "r"(v) : "memory");
}
// mode 0: pattern of k_encode_f64_wide (warp = 32 elements x 256 B contiguous, 8 instr of 1 KB), no loads
// mode 1: + one 8-byte load per lane per iteration (prefetched)
// mode 2: mode 1 but sector 0 of each element written by the element's own lane (stride-256 B 32-byte stores)
template <int MODE>
__global__ void __launch_bounds__(256) k(const double* fin, uint32_t* out, long count, int wn) {
  const int lane = threadIdx.x & 31, quarter = lane >> 3, l8 = lane & 7;
  const long warp = (long)blockIdx.x * 8 + (threadIdx.x >> 5), nwarps = (long)gridDim.x * 8;
  long eb = warp * 32;
  double nxt = (MODE >= 1 && eb + lane < count) ? fin[eb + lane] : 0.0;
  for (; eb < count; eb += nwarps * 32) {
    double cur = nxt;
    if (MODE >= 1) { long en = eb + lane + nwarps * 32; nxt = en < count ? fin[en] : 0.0; }
    uint32_t v = MODE >= 1 ? (uint32_t)__double2int_rn(cur) : 7u;
    uint32_t* q = out + (eb + quarter) * (long)wn + 8 * l8;
#pragma unroll
    for (int s = 0; s < 32; s += 4) {
      uint32_t vv = __shfl_sync(0xffffffffu, v, s + quarter);
      if (MODE == 2 && l8 == 0) continue;
      st8(q + (long)s * wn, vv);
    }
    if (MODE == 2) st8(out + (eb + lane) * (long)wn, v);
  }
}
int main() {
  const long count = 8000000; const int wn = 64;
  double* fin; uint32_t* out;
  cudaMalloc(&fin, count * 8); cudaMalloc(&out, count * wn * 4L);
  cudaMemset(fin, 0, count * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; mode++)
    for (int bps : {2, 3, 4, 5, 6, 8}) {
      int blocks = 148 * bps;
      auto run = [&]() {
        if (mode == 0) k<0><<<blocks, 256>>>(fin, out, count, wn);
        else if (mode == 1) k<1><<<blocks, 256>>>(fin, out, count, wn);
        else k<2><<<blocks, 256>>>(fin, out, count, wn);
      };
      run(); cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int i = 0; i < 10; i++) run();
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("mode %d blocks/SM %d: %.0f GB/s\n", mode, bps, count * (wn * 4.0 + (mode ? 8 : 0)) / (ms / 10 * 1e-3) / 1e9);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
