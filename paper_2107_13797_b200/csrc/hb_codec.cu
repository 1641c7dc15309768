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
};

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

// residue -> signed mantissa -> correctly rounded double (encoding.py:81-101)
__global__ void __launch_bounds__(64) k_decode_f64(CodecArgs A) {
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
  if (e >= A.count) return;
  uint32_t* my = stage + threadIdx.x * pitch;
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

extern "C" {

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
  const int threads = 64;
  const size_t smem = (size_t)threads * (ctx->wn + 1) * sizeof(uint32_t);
  hb::k_encode_f64<<<(unsigned)((count + threads - 1) / threads), threads, smem, (cudaStream_t)stream_>>>(A);
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
  const int threads = 64;
  const size_t smem = (size_t)threads * (ctx->wn + 1) * sizeof(uint32_t);
  hb::k_decode_f64<<<(unsigned)((count + threads - 1) / threads), threads, smem, (cudaStream_t)stream_>>>(A);
  g_launches++;
  CU(cudaGetLastError());
  return HB_OK;
}

}  // extern "C"
