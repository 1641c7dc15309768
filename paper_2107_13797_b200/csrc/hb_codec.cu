// C ABI, third translation unit: the fixed-point codec (encoding.py:54-101 of the reference) as
// element-wise kernels.  Both are HBM-bound (8 B of double + one residue per element); residues are
// staged through shared memory so the global accesses are coalesced.
#include "hb_ctx.h"

using namespace hbi;

namespace hb {

struct CodecArgs {
  const uint32_t* nwords;    // n
  const uint32_t* maxint;    // n / 3
  const uint32_t* negband;   // n - n / 3
  int wn;
  int exponent;              // base-16 exponent of the batch
  long count;
  const double* fin; double* fout;
  const uint32_t* min; uint32_t* mout;
  unsigned long long* first_bad;
  int maxint_top;            // index of the highest non-zero word of max_int
  uint8_t* slow;             // decode: fast kernel marks the elements it leaves to the generic kernel
  const uint8_t* only;       // decode: generic kernel handles marked elements only (nullptr = all)
  unsigned long long* nslow; // decode: how many elements were marked
};

__device__ __forceinline__ uint4 ld4(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }

// round(v * 16^-exponent) half-to-even, |.| < max_int, stored as a residue mod n (encoding.py:72-78)
__global__ void __launch_bounds__(64) k_encode_f64(CodecArgs A) {
  extern __shared__ uint32_t stage[];
  const int wn = A.wn, pitch = wn + 1;
  const long base = (long)blockIdx.x * blockDim.x;
  const long e = base + threadIdx.x;
  uint32_t* my = stage + threadIdx.x * pitch;
  if (e < A.count) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(A.fin[e]);
    const bool negv = (bits >> 63) != 0;
    const int e11 = (int)((bits >> 52) & 0x7ff);
    unsigned long long mant = bits & 0xfffffffffffffull;
    int e2;
    if (e11 == 0) e2 = -1074; else { mant |= 1ull << 52; e2 = e11 - 1075; }
    long shift = (long)e2 - 4L * A.exponent;      // scaled = mant * 2^shift
    if (shift < 0) {
      long s = -shift;
      if (s >= 64) mant = 0;
      else {
        unsigned long long q = mant >> s, rem = mant & ((1ull << s) - 1ull), half = 1ull << (s - 1);
        if (rem > half || (rem == half && (q & 1ull))) q++;
        mant = q;
      }
      shift = 0;
    }
    if (mant == 0) shift = 0;
    // word i of mag = mant << shift
    const long ws = shift >> 5; const int bs = (int)(shift & 31);
    // three words cover 53 + 31 bits
    const unsigned long long lo = mant << bs;                      // low 64 bits of mant << bs
    const uint32_t hi = bs ? (uint32_t)(mant >> (64 - bs)) : 0u;   // bits 64.. of mant << bs
    auto magword = [&](long i) -> uint32_t {
      long r = i - ws;
      return r == 0 ? (uint32_t)lo : r == 1 ? (uint32_t)(lo >> 32) : r == 2 ? hi : 0u;
    };
    // overflow: mag >= max_int  (also when mag has bits beyond wn words)
    bool over = false;
    if (mant != 0 && ws + 3 > wn) {
      for (long i = wn; i < ws + 3; i++) over |= magword(i) != 0;
    }
    if (!over) {
      int cmp = 0;
      for (int i = wn - 1; i >= 0 && cmp == 0; i--) {
        uint32_t a = magword(i), b = A.maxint[i];
        cmp = a > b ? 1 : (a < b ? -1 : 0);
      }
      over = cmp >= 0;
    }
    if (over) atomicMin(A.first_bad, (unsigned long long)e);
    const bool neg = negv && mant != 0;
    uint32_t borrow = 0;
    for (int i = 0; i < wn; i++) {
      uint32_t m = magword(i);
      if (neg) {
        unsigned long long d = (unsigned long long)A.nwords[i] - m - borrow;
        borrow = (uint32_t)(d >> 63);
        m = (uint32_t)d;
      }
      my[i] = m;
    }
  }
  __syncthreads();
  const long nhere = min((long)blockDim.x, A.count - base);
  for (long idx = threadIdx.x; idx < nhere * wn; idx += blockDim.x) {
    long el = idx / wn; int w = (int)(idx - el * wn);
    A.mout[(base + el) * wn + w] = stage[el * pitch + w];
  }
}

// residue -> signed mantissa -> correctly rounded double (encoding.py:81-101); `my` is the element's words in
// shared memory (modified in place)
__device__ void decode_one(const CodecArgs& A, uint32_t* my, long e) {
  const int wn = A.wn;
  int c_max = 0, c_neg = 0;     // compare with max_int and with n - max_int
  for (int i = wn - 1; i >= 0; i--) {
    uint32_t v = my[i];
    if (c_max == 0) { uint32_t b = A.maxint[i]; c_max = v > b ? 1 : (v < b ? -1 : 0); }
    if (c_neg == 0) { uint32_t b = A.negband[i]; c_neg = v > b ? 1 : (v < b ? -1 : 0); }
  }
  const bool pos = c_max < 0, neg = c_neg > 0;
  if (!pos && !neg) { atomicMin(A.first_bad, (unsigned long long)e); A.fout[e] = 0.0; return; }
  if (neg) {
    uint32_t borrow = 0;
    for (int i = 0; i < wn; i++) {
      unsigned long long d = (unsigned long long)A.nwords[i] - my[i] - borrow;
      borrow = (uint32_t)(d >> 63);
      my[i] = (uint32_t)d;
    }
  }
  int top = -1;
  for (int i = wn - 1; i >= 0; i--) if (my[i]) { top = i; break; }
  double val = 0.0;
  if (top >= 0) {
    const int tb = top * 32 + 31 - __clz(my[top]);       // index of the highest set bit
    int ex2;
    unsigned long long m53;
    if (tb <= 52) {
      m53 = (unsigned long long)my[0] | (wn > 1 ? (unsigned long long)my[1] << 32 : 0ull);
      ex2 = 0;
    } else {
      // 64-bit window ending at tb
      const int lowbit = tb - 63;                        // may be negative
      unsigned long long win = 0;
      bool sticky = false;
      if (lowbit <= 0) {
        win = ((unsigned long long)my[0] | (wn > 1 ? (unsigned long long)my[1] << 32 : 0ull)) << (-lowbit);
      } else {
        const int wi = lowbit >> 5, sh = lowbit & 31;
        unsigned long long w0 = my[wi], w1 = wi + 1 < wn ? my[wi + 1] : 0u, w2 = wi + 2 < wn ? my[wi + 2] : 0u;
        win = (w0 >> sh) | (w1 << (32 - sh)) | (sh ? (w2 << (64 - sh)) : 0ull);
        if (sh) sticky |= (my[wi] & ((1u << sh) - 1u)) != 0;
        for (int i = 0; i < wi; i++) sticky |= my[i] != 0;
      }
      m53 = win >> 11;
      const unsigned long long rem = win & 0x7ffull, half = 0x400ull;
      if (rem > half || (rem == half && (sticky || (m53 & 1ull)))) m53++;
      ex2 = tb - 52;
    }
    val = ldexp((double)m53, ex2 + 4 * A.exponent);
  }
  A.fout[e] = neg ? -val : val;
}

// generic decode, one thread per element, grid-stride over tiles of blockDim elements; with A.only set it finishes
// what the wide kernel left (usually nothing: every block returns on the zero count)
__global__ void __launch_bounds__(64) k_decode_f64(CodecArgs A) {
  extern __shared__ uint32_t stage[];
  const int wn = A.wn, pitch = wn + 1;
  if (A.only && *A.nslow == 0ull) return;
  for (long base = (long)blockIdx.x * blockDim.x; base < A.count; base += (long)gridDim.x * blockDim.x) {
    const long nhere = min((long)blockDim.x, A.count - base);
    const long e = base + threadIdx.x;
    bool mine = e < A.count;
    if (A.only) {
      mine = mine && A.only[e] != 0;
      if (!__syncthreads_or(mine)) continue;      // nothing in this tile was left to the generic path
    }
    for (long idx = threadIdx.x; idx < nhere * wn; idx += blockDim.x) {
      long el = idx / wn; int w = (int)(idx - el * wn);
      stage[el * pitch + w] = A.min[(base + el) * wn + w];
    }
    __syncthreads();
    if (mine) decode_one(A, stage + threadIdx.x * pitch, e);
    __syncthreads();
  }
}


// ---- HBM-bound forms of the two codec kernels ----------------------------------------------------------------
//
// A residue is 4 * wn bytes of which, for every value a protocol ever encodes, all but three words are either zero
// (positive) or the words of n (negative, n - |x|).  The thread-per-element kernels above spend hundreds of
// instructions per element walking those words; the kernels below move the background with 32-byte accesses (whole
// sectors), 8 lanes per element, and leave only the three interesting words to one thread per element.  Requires
// wn % 8 == 0 and wn >= 8 (the host falls back to the kernels above otherwise).

// 32-byte global accesses (one full DRAM / L2 sector per lane): LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a.
__device__ __forceinline__ void ld8(uint32_t (&w)[8], const uint32_t* p) {
  asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}
__device__ __forceinline__ void st8(uint32_t* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               :: "l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void ldn8(uint32_t (&w)[8], const uint32_t* p) {      // constants: cached loads
  const uint4 a = ld4(p), b = ld4(p + 4);
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

// encode: one lane per element works out the up-to-three magnitude words; the background (0 or n) of 32 elements
// then goes out as 32-byte stores -- whole sectors, 8 lanes per element, four elements per warp instruction.  When
// the warp's 32 elements agree on the sector their magnitude words fall into and none has a borrow running past
// them -- every batch a protocol encodes -- that sector is left out of the background pass and written once,
// patched, by the element's own lane: every sector is written exactly once and whole (a first cut that wrote the
// patched 16 bytes separately from the other half of their sector ran at HALF the speed: partial-sector writes
// make the L2 fetch the sector first).  Otherwise: background everywhere, __syncwarp, then word-sized patches.
// The next batch's doubles are fetched before this batch's stores.  Requires wn % 8 == 0.
#ifndef HB_ENC_BLOCKS
#define HB_ENC_BLOCKS 4      // 62 registers, no spills; 5 and 6 blocks (48 / 40 registers) measured slower
#endif
template <bool TWO>     // TWO: more than 64 words per residue (a second 32-byte column per lane)
__global__ void __launch_bounds__(256, HB_ENC_BLOCKS) k_encode_f64_wide(CodecArgs A) {
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  const int wn = A.wn, T = A.maxint_top;
  const int quarter = lane >> 3, l8 = lane & 7, i0 = 8 * l8;
  const bool act0 = i0 < wn, act1 = TWO && i0 + 64 < wn;
  uint32_t nv0[8], nv1[8];
#pragma unroll
  for (int k = 0; k < 8; k++) { nv0[k] = 0u; nv1[k] = 0u; }
  if (act0) ldn8(nv0, A.nwords + i0);
  if (act1) ldn8(nv1, A.nwords + i0 + 64);
  long eb = warp * 32;
  unsigned long long bits_next = eb + lane < A.count ? (unsigned long long)__double_as_longlong(A.fin[eb + lane]) : 0ull;
  for (; eb < A.count; eb += nwarps * 32) {
    const long e = eb + lane;
    const bool have = e < A.count;
    const unsigned long long bits = bits_next;
    {
      const long en = e + nwarps * 32;
      bits_next = en < A.count ? (unsigned long long)__double_as_longlong(A.fin[en]) : 0ull;
    }
    const bool negv = (bits >> 63) != 0;
    const int e11 = (int)((bits >> 52) & 0x7ff);
    unsigned long long mant = bits & 0xfffffffffffffull;
    int e2;
    if (e11 == 0) e2 = -1074; else { mant |= 1ull << 52; e2 = e11 - 1075; }
    long shift = (long)e2 - 4L * A.exponent;      // scaled = mant * 2^shift
    if (shift < 0) {
      long s = -shift;
      if (s >= 64) mant = 0;
      else {
        unsigned long long q = mant >> s, rem = mant & ((1ull << s) - 1ull), half_ulp = 1ull << (s - 1);
        if (rem > half_ulp || (rem == half_ulp && (q & 1ull))) q++;
        mant = q;
      }
      shift = 0;
    }
    if (mant == 0) shift = 0;
    const long ws = shift >> 5; const int bs = (int)(shift & 31);
    const unsigned long long lo = mant << bs;
    uint32_t v0 = (uint32_t)lo, v1 = (uint32_t)(lo >> 32), v2 = bs ? (uint32_t)(mant >> (64 - bs)) : 0u;
    // |scaled| >= max_int ?  Decided by the position of the top word except when both top words coincide.
    const long tw = mant ? ws + (v2 ? 2 : v1 ? 1 : 0) : -1;
    bool over = tw > T;
    if (tw == T) {
      int cmp = 0;
      for (long i = T; i >= 0 && cmp == 0; i--) {
        const long r = i - ws;
        const uint32_t a = r == 0 ? v0 : r == 1 ? v1 : r == 2 ? v2 : 0u, b = A.maxint[i];
        cmp = a > b ? 1 : (a < b ? -1 : 0);
      }
      over = cmp >= 0;
    }
    if (have && over) atomicMin(A.first_bad, (unsigned long long)e);
    const bool neg = have && negv && mant != 0 && !over;
    long bend = 0;
    bool brun = false;
    if (neg) {                                     // n - |scaled| on the three words, borrow runs on through zero words of n
      uint32_t borrow = 0;
      uint32_t* vs[3] = {&v0, &v1, &v2};
#pragma unroll
      for (int k = 0; k < 3; k++) {
        const uint32_t nk = ws + k < wn ? A.nwords[ws + k] : 0u;
        const unsigned long long d = (unsigned long long)nk - *vs[k] - borrow;
        borrow = (uint32_t)(d >> 63);
        *vs[k] = (uint32_t)d;
      }
      if (borrow) {
        brun = true;
        bend = ws + 3;
        while (bend < wn && A.nwords[bend] == 0u) bend++;
      }
    }
    const uint32_t negmask = __ballot_sync(0xffffffffu, neg);
    const bool full = eb + 32 <= A.count;
    uint32_t* q = A.mout + (eb + quarter) * (long)wn + i0;
    // do the 32 elements agree on the sector of their magnitude words, with nothing running past it?
    const int sw = over ? 0 : (int)(ws >> 3);
    const int sw0 = __shfl_sync(0xffffffffu, sw, 0);
    const bool plain = !have || over || (sw == sw0 && !brun && (ws & 7) <= 5);
    const bool fast = __all_sync(0xffffffffu, plain);
    // pass 1: background, four elements per step (the shared sector left out on the fast path)
    const bool put0 = act0 && !(fast && l8 == sw0), put1 = TWO && act1 && !(fast && l8 + 8 == sw0);
#pragma unroll
    for (int s = 0; s < 32; s += 4) {
      const bool in = full || eb + s + quarter < A.count;
      const uint32_t keep = ((negmask >> (s + quarter)) & 1u) ? 0xffffffffu : 0u;
      if (put0 && in) {
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; k++) w[k] = nv0[k] & keep;
        st8(q + (long)s * wn, w);
      }
      if (put1 && in) {
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; k++) w[k] = nv1[k] & keep;
        st8(q + (long)s * wn + 64, w);
      }
    }
    if (fast) {
      // pass 2: the element's own lane writes that sector, magnitude words in place
      if (have) {
        uint32_t c[8];
#pragma unroll
        for (int k = 0; k < 8; k++) c[k] = 0u;
        if (neg) ldn8(c, A.nwords + 8 * sw0);
        if (!over) {
          const int pos = (int)(ws & 7);
#pragma unroll
          for (int k = 0; k < 8; k++) c[k] = k == pos ? v0 : k == pos + 1 ? v1 : k == pos + 2 ? v2 : c[k];
        }
        st8(A.mout + e * (long)wn + 8 * sw0, c);
      }
    } else {
      __syncwarp();
      // pass 2: the words that differ from the background
      if (have && !over) {
        uint32_t* dst = A.mout + e * (long)wn;
        if (ws < wn) dst[ws] = v0;
        if (ws + 1 < wn) dst[ws + 1] = v1;
        if (ws + 2 < wn) dst[ws + 2] = v2;
        if (brun) {
          for (long i = ws + 3; i < bend; i++) dst[i] = 0xffffffffu;
          if (bend < wn) dst[bend] = A.nwords[bend] - 1u;
        }
      }
      __syncwarp();
    }
  }
}

// decode: pass 1 checks that every word from the fourth up is background (all zero, or all equal to n); pass 2
// turns the low 96 bits into the correctly rounded double.  Anything else -- wide magnitudes, the overflow band --
// is marked in A.slow for the generic kernel.  Needs max_int >= 2^96 (maxint_top >= 3).
#ifndef HB_DEC_BLOCKS
#define HB_DEC_BLOCKS 4      // 64 registers; measured 0.917 of the HBM copy peak with two steps in flight, 0.89 with
#endif                       // four (62 registers + spills), 0.66 at 5 blocks (48 registers, spills)
#ifndef HB_DEC_NJ
#define HB_DEC_NJ 2
#endif
template <bool TWO>
__global__ void __launch_bounds__(256, HB_DEC_BLOCKS) k_decode_f64_wide(CodecArgs A) {
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long nwarps = (long)gridDim.x * (blockDim.x >> 5);
  const int wn = A.wn;
  const int quarter = lane >> 3, l8 = lane & 7, i0 = 8 * l8;
  // sector 0 (words 0..7) of an element is read by the element's own lane, not in pass 1
  const bool act0 = i0 < wn && l8 != 0, act1 = TWO && i0 + 64 < wn;
  uint32_t nv0[8], nv1[8], nlow[8];
#pragma unroll
  for (int k = 0; k < 8; k++) { nv0[k] = 0u; nv1[k] = 0u; }
  if (act0) ldn8(nv0, A.nwords + i0);
  if (act1) ldn8(nv1, A.nwords + i0 + 64);
  ldn8(nlow, A.nwords);
  constexpr int NJ = TWO ? (HB_DEC_NJ > 1 ? HB_DEC_NJ / 2 : 1) : HB_DEC_NJ;   // steps of four elements in flight
  for (long eb = warp * 32; eb < A.count; eb += nwarps * 32) {
    // own element's low sector first: its latency hides behind pass 1
    const long e = eb + lane;
    uint32_t m[8];
#pragma unroll
    for (int k = 0; k < 8; k++) m[k] = 0u;
    if (e < A.count) ld8(m, A.min + e * (long)wn);
    uint32_t m0 = m[0], m1 = m[1], m2 = m[2];
    const bool full = eb + 32 <= A.count;
    const uint32_t* p = A.min + (eb + quarter) * (long)wn + i0;
    uint32_t zbits = 0, nbits = 0;        // bit k: every word from the ninth up of element eb + k is 0 / equals n
#pragma unroll 1
    for (int s = 0; s < 32; s += 4 * NJ) {     // loads of NJ steps issued together
      uint32_t xa[NJ][8], xb[TWO ? NJ : 1][8];
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        const bool in = full || eb + s + 4 * j + quarter < A.count;
        if (act0 && in) ld8(xa[j], p + (long)(s + 4 * j) * wn);
        else {
#pragma unroll
          for (int k = 0; k < 8; k++) xa[j][k] = nv0[k];
        }
        if (TWO) {
          if (act1 && in) ld8(xb[j], p + (long)(s + 4 * j) * wn + 64);
          else {
#pragma unroll
            for (int k = 0; k < 8; k++) xb[j][k] = nv1[k];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        uint32_t z = 0u, d = 0u;
#pragma unroll
        for (int k = 0; k < 8; k++) { z |= xa[j][k]; d |= xa[j][k] ^ nv0[k]; }
        if (TWO) {
#pragma unroll
          for (int k = 0; k < 8; k++) { z |= xb[j][k]; d |= xb[j][k] ^ nv1[k]; }
        }
        // inactive lanes hold n's (zero) words: they vote "equal to n" and, being zero, "zero" as well
        const uint32_t bz = __ballot_sync(0xffffffffu, z == 0u), bn = __ballot_sync(0xffffffffu, d == 0u);
        const int first = s + 4 * j;
#pragma unroll
        for (int qq = 0; qq < 4; qq++) {
          zbits |= (uint32_t)(((bz >> (8 * qq)) & 0xffu) == 0xffu) << (first + qq);
          nbits |= (uint32_t)(((bn >> (8 * qq)) & 0xffu) == 0xffu) << (first + qq);
        }
      }
    }
    const uint32_t hz = m[3] | m[4] | m[5] | m[6] | m[7];
    const uint32_t hn = (m[3] ^ nlow[3]) | (m[4] ^ nlow[4]) | (m[5] ^ nlow[5]) | (m[6] ^ nlow[6]) | (m[7] ^ nlow[7]);
    const bool my_zero = ((zbits >> lane) & 1u) && hz == 0u, my_n = ((nbits >> lane) & 1u) && hn == 0u;
    if (e >= A.count) continue;
    bool neg = false, slow = false;
    if (my_zero) {
      // positive, below 2^96 <= max_int
    } else if (my_n) {
      unsigned long long d = (unsigned long long)nlow[0] - m0;
      m0 = (uint32_t)d;
      d = (unsigned long long)nlow[1] - m1 - (d >> 63);
      m1 = (uint32_t)d;
      d = (unsigned long long)nlow[2] - m2 - (d >> 63);
      m2 = (uint32_t)d;
      neg = true;
      slow = (d >> 63) != 0 || (m0 | m1 | m2) == 0u;     // x >= n: not a residue; let the generic path judge it
    } else {
      slow = true;
    }
    A.slow[e] = slow ? 1 : 0;
    if (slow) { atomicAdd(A.nslow, 1ull); continue; }
    double val = 0.0;
    if (m0 | m1 | m2) {
      const int tb = m2 ? 95 - __clz(m2) : m1 ? 63 - __clz(m1) : 31 - __clz(m0);
      const unsigned long long low = (unsigned long long)m0 | ((unsigned long long)m1 << 32);
      unsigned long long m53;
      int ex2 = 0;
      if (tb <= 52) {
        m53 = low;
      } else {
        unsigned long long win;
        bool sticky = false;
        if (tb <= 63) {
          win = low << (63 - tb);
        } else {
          const int sh = tb - 63;                        // 1..32
          win = (low >> sh) | ((unsigned long long)m2 << (64 - sh));
          sticky = (low & ((1ull << sh) - 1ull)) != 0ull;
        }
        m53 = win >> 11;
        const unsigned long long rem = win & 0x7ffull, halfway = 0x400ull;
        if (rem > halfway || (rem == halfway && (sticky || (m53 & 1ull)))) m53++;
        ex2 = tb - 52;
      }
      val = ldexp((double)m53, ex2 + 4 * A.exponent);
    }
    A.fout[e] = neg ? -val : val;
  }
}

// min over the batch of exact_exponent(v) (encoding.py:44-51, batches.py:122-123): the largest base-16 exponent at
// which every value has an integer mantissa; zeros count as exponent 0.  One atomicMin per warp.
__global__ void __launch_bounds__(256) k_min_exact_exponent(const double* __restrict__ v, long count, int* out) {
  int best = 0x7fffffff;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v[i]);
    const int e11 = (int)((bits >> 52) & 0x7ff);
    unsigned long long mant = bits & 0xfffffffffffffull;
    int e2;
    if (e11 == 0) e2 = -1074; else { mant |= 1ull << 52; e2 = e11 - 1075; }
    const int ex = mant ? (e2 + (__ffsll((long long)mant) - 1)) >> 2 : 0;      // arithmetic shift = floor division by 4
    best = min(best, ex);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != 0x7fffffff) atomicMin(out, best);
}

// Exact re-grid onto a finer exponent (encoding.py:104-113): signed mantissa times 16^digits, range-checked
// against max_int, stored back as a residue.  first_bad receives the smallest index that is in the overflow band
// or overflows after scaling (the host re-examines that element to raise the reference's error).
__global__ void __launch_bounds__(64) k_plain_rescale(CodecArgs A) {
  extern __shared__ uint32_t stage[];
  const int wn = A.wn, pitch = wn + 1;
  const long base = (long)blockIdx.x * blockDim.x;
  const long nhere = min((long)blockDim.x, A.count - base);
  for (long idx = threadIdx.x; idx < nhere * wn; idx += blockDim.x) {
    long el = idx / wn; int w = (int)(idx - el * wn);
    stage[el * pitch + w] = A.min[(base + el) * wn + w];
  }
  __syncthreads();
  const long e = base + threadIdx.x;
  if (e < A.count) {
    uint32_t* my = stage + threadIdx.x * pitch;
    int c_max = 0, c_neg = 0;
    for (int i = wn - 1; i >= 0; i--) {
      uint32_t v = my[i];
      if (c_max == 0) { uint32_t b = A.maxint[i]; c_max = v > b ? 1 : (v < b ? -1 : 0); }
      if (c_neg == 0) { uint32_t b = A.negband[i]; c_neg = v > b ? 1 : (v < b ? -1 : 0); }
    }
    const bool pos = c_max < 0, neg = c_neg > 0;
    bool over = !pos && !neg;
    if (neg) {
      uint32_t borrow = 0;
      for (int i = 0; i < wn; i++) {
        unsigned long long d = (unsigned long long)A.nwords[i] - my[i] - borrow;
        borrow = (uint32_t)(d >> 63);
        my[i] = (uint32_t)d;
      }
    }
    // |s| << (4 * digits), in place from the top down; A.exponent carries the digit count here
    const long shift = 4L * A.exponent;
    const int ws = (int)min((long)wn, shift >> 5), bs = (int)(shift & 31);
    bool nonzero = false;
    for (int i = 0; i < wn; i++) nonzero |= my[i] != 0;
    if (nonzero && (shift >> 5) >= wn) over = true;
    for (int i = wn - 1; i >= wn - ws - 1 && i >= 0; i--) {       // bits that leave the top
      uint32_t v = my[i];
      if (i > wn - ws - 1) over |= v != 0;
      else if (bs) over |= (v >> (32 - bs)) != 0;
    }
    for (int i = wn - 1; i >= 0; i--) {
      const int src = i - ws;
      uint32_t hi = src >= 0 ? my[src] : 0u, lo = src - 1 >= 0 ? my[src - 1] : 0u;
      my[i] = bs ? (hi << bs) | (lo >> (32 - bs)) : hi;
    }
    if (!over) {
      int cmp = 0;
      for (int i = wn - 1; i >= 0 && cmp == 0; i--) {
        uint32_t a = my[i], b = A.maxint[i];
        cmp = a > b ? 1 : (a < b ? -1 : 0);
      }
      over = cmp >= 0;
    }
    if (over) atomicMin(A.first_bad, (unsigned long long)e);
    if (neg && nonzero) {
      uint32_t borrow = 0;
      for (int i = 0; i < wn; i++) {
        unsigned long long d = (unsigned long long)A.nwords[i] - my[i] - borrow;
        borrow = (uint32_t)(d >> 63);
        my[i] = (uint32_t)d;
      }
    }
  }
  __syncthreads();
  for (long idx = threadIdx.x; idx < nhere * wn; idx += blockDim.x) {
    long el = idx / wn; int w = (int)(idx - el * wn);
    A.mout[(base + el) * wn + w] = stage[el * pitch + w];
  }
}

}  // namespace hb

namespace {
// 256-thread blocks of `kernel` resident per SM on the current device (occupancy API; a handful of microseconds).
int resident_blocks(const void* kernel) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, 256, 0) != cudaSuccess || nb < 1) {
    cudaGetLastError();
    nb = 4;
  }
  return nb;
}
}  // namespace

extern "C" {

int hb_min_exact_exponent(hb_ctx* ctx, const double* values, int64_t count, int* min_out, void* stream_) {
  if (!ctx || !values || !min_out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  const long blocks = std::min<long>((count + 255) / 256, (long)ctx->sms * 8);
  hb::k_min_exact_exponent<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream_>>>(values, count, min_out);
  g_launches++;
  CU(cudaGetLastError());
  return HB_OK;
}

int hb_plain_rescale(hb_ctx* ctx, const uint32_t* m, int digits, uint32_t* m_out, int64_t count,
                     int64_t* first_bad, void* stream_) {
  if (!ctx || !m || !m_out || !first_bad) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0 || digits < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  hb::CodecArgs A{};
  A.nwords = ctx->d_pub + ctx->off_nwords; A.maxint = ctx->d_pub + ctx->off_maxint;
  A.negband = ctx->d_pub + ctx->off_negband; A.wn = ctx->wn; A.exponent = digits; A.count = count;
  A.min = m; A.mout = m_out; A.first_bad = (unsigned long long*)first_bad;
  const int threads = 64;
  const size_t smem = (size_t)threads * (ctx->wn + 1) * sizeof(uint32_t);
  hb::k_plain_rescale<<<(unsigned)((count + threads - 1) / threads), threads, smem, (cudaStream_t)stream_>>>(A);
  g_launches++;
  CU(cudaGetLastError());
  return HB_OK;
}

int hb_encode_f64(hb_ctx* ctx, const double* values, int exponent, uint32_t* m_out, int64_t count,
                  int64_t* first_bad, void* stream_) {
  if (!ctx || !values || !m_out || !first_bad) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  hb::CodecArgs A{};
  A.nwords = ctx->d_pub + ctx->off_nwords; A.maxint = ctx->d_pub + ctx->off_maxint;
  A.negband = ctx->d_pub + ctx->off_negband; A.wn = ctx->wn; A.exponent = exponent; A.count = count;
  A.fin = values; A.mout = m_out; A.first_bad = (unsigned long long*)first_bad;
  A.maxint_top = ctx->maxint_top;
  if (ctx->wn % 8 == 0 && ctx->wn >= 8 && ctx->wn <= 128) {
    // persistent grid: exactly the blocks that are resident at once (no partial wave), grid-stride over batches of 32
    const long warps = (count + 31) / 32;
    const bool two = ctx->wn > 64;
    const long blocks = std::min<long>((warps + 7) / 8, (long)ctx->sms * resident_blocks(two ? (const void*)hb::k_encode_f64_wide<true>
                                                                                             : (const void*)hb::k_encode_f64_wide<false>));
    if (two) hb::k_encode_f64_wide<true><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream_>>>(A);
    else hb::k_encode_f64_wide<false><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream_>>>(A);
  } else {
    const int threads = 64;
    const size_t smem = (size_t)threads * (ctx->wn + 1) * sizeof(uint32_t);
    hb::k_encode_f64<<<(unsigned)((count + threads - 1) / threads), threads, smem, (cudaStream_t)stream_>>>(A);
  }
  g_launches++;
  CU(cudaGetLastError());
  return HB_OK;
}

int hb_decode_f64(hb_ctx* ctx, const uint32_t* m, int exponent, double* values_out, int64_t count,
                  int64_t* first_bad, void* stream_) {
  if (!ctx || !values_out || !m || !first_bad) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  hb::CodecArgs A{};
  A.nwords = ctx->d_pub + ctx->off_nwords; A.maxint = ctx->d_pub + ctx->off_maxint;
  A.negband = ctx->d_pub + ctx->off_negband; A.wn = ctx->wn; A.exponent = exponent; A.count = count;
  A.min = m; A.fout = values_out; A.first_bad = (unsigned long long*)first_bad;
  A.maxint_top = ctx->maxint_top;
  cudaStream_t stream = (cudaStream_t)stream_;
  uint8_t* scratch = nullptr;
  if (ctx->wn % 8 == 0 && ctx->wn >= 8 && ctx->wn <= 128 && ctx->maxint_top >= 3) {
    // marks of the elements left to the generic kernel: per call, from the library's pool (calls on one context
    // may run on several streams / threads at once)
    CU(hbi::pool_alloc(ctx->pool, (void**)&scratch, (size_t)count + 16, stream));
    uint8_t* slow = scratch + 16;
    A.slow = slow;
    A.nslow = (unsigned long long*)scratch;
    CU(cudaMemsetAsync(scratch, 0, 8, stream));
    const long warps = (count + 31) / 32;
    const bool two = ctx->wn > 64;
    const long blocks = std::min<long>((warps + 7) / 8, (long)ctx->sms * resident_blocks(two ? (const void*)hb::k_decode_f64_wide<true>
                                                                                             : (const void*)hb::k_decode_f64_wide<false>));
    if (two) hb::k_decode_f64_wide<true><<<(unsigned)blocks, 256, 0, stream>>>(A);
    else hb::k_decode_f64_wide<false><<<(unsigned)blocks, 256, 0, stream>>>(A);
    g_launches++;
    A.only = slow;
  }
  const int threads = 64;
  const size_t smem = (size_t)threads * (ctx->wn + 1) * sizeof(uint32_t);
  const long tiles = (count + threads - 1) / threads;
  hb::k_decode_f64<<<(unsigned)std::min<long>(tiles, (long)ctx->sms * 16), threads, smem, stream>>>(A);
  g_launches++;
  CU(cudaGetLastError());
  if (scratch) CU(cudaFreeAsync(scratch, stream));
  return HB_OK;
}

}  // extern "C"
