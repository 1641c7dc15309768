// Second kernel family: variable-exponent powers, modular inversion, product reductions and the
// encrypted matrix-vector product (bucket method).  Same group-per-instance layout as hb_kernels.cuh.
//
// Reference semantics (file:line under /root/reference/pkg/src/hebatch):
//   k_powvar        operators.py:59-67   _pow_scalar / _k_mul
//   k_product_pass  operators.py:75-83   _k_product
//   bucket kernels  operators.py:86-94   _k_dot: out_j = prod_t pow_scalar(c_t, k_tj)
//
// "Digit form" below means the L 32-bit limbs of a number, Montgomery representation (x * R mod N),
// stored contiguously: element i lives at base + i * L, lane t of its group owns digits [t*LPT, (t+1)*LPT).
#pragma once
#include "hb_ctx.h"

namespace hb {

#define HB_GROUP_PROLOGUE(LPT, TPI)                                                              \
  using M = Mont<LPT, TPI>;                                                                      \
  constexpr int IPW = 32 / TPI;                                                                  \
  constexpr int L = LPT * TPI;                                                                   \
  const int lane = threadIdx.x, g = lane / TPI;            /* one warp per block, see hb_ctx.h plan() */ \
  const long wg = blockIdx.x, nw = gridDim.x;                                                    \
  (void)L; (void)g; (void)wg; (void)nw; (void)lane;

// ------------------------------------------------------------------------------------------------
// words -> Montgomery digit form
struct ToMontArgs { ModDev mod; const uint32_t* words; int w; uint32_t* dig; long count; };

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_to_mont(ToMontArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_words(x, A.words + ii * A.w, A.w);
    mt.load_limbs(y, A.mod.r2);
    mt.mul(x, x, y);
    if (valid) mt.store_limbs(A.dig + ii * L, x);
  }
}

// Montgomery digit form -> plain words
struct FromMontArgs { ModDev mod; const uint32_t* dig; long count; uint32_t* words; int w; };

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_from_mont(FromMontArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_limbs(x, A.dig + ii * L);
    mt.set_one(y);
    mt.mul(x, x, y);
    mt.store_words(A.words + ii * A.w, A.w, x, valid);
  }
}

// ------------------------------------------------------------------------------------------------
// Batch inversion tree.  up: dst[j] = src[2j] * src[2j+1] (copy when there is no sibling).
struct PairUpArgs { ModDev mod; const uint32_t* src; long nsrc; uint32_t* dst; };

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_pair_up(PairUpArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long ndst = (A.nsrc + 1) / 2;
  const long ntiles = (ndst + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < ndst;
    long j = valid ? inst : ndst - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_limbs(x, A.src + (2 * j) * L);
    bool sib = 2 * j + 1 < A.nsrc;
    if (sib) mt.load_limbs(y, A.src + (2 * j + 1) * L); else mt.load_limbs(y, A.mod.r1);
    mt.mul(x, x, y);
    if (valid) mt.store_limbs(A.dst + j * L, x);
  }
}

// down: inv_child[i] = inv_parent[i/2] * val_child[i^1] (copy of the parent when there is no sibling).
struct PairDownArgs { ModDev mod; const uint32_t* inv_parent; const uint32_t* val_child; long nchild; uint32_t* inv_child; };

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_pair_down(PairDownArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long ntiles = (A.nchild + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.nchild;
    long i = valid ? inst : A.nchild - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_limbs(x, A.inv_parent + (i >> 1) * L);
    long s = i ^ 1;
    if (s < A.nchild) mt.load_limbs(y, A.val_child + s * L); else mt.load_limbs(y, A.mod.r1);
    mt.mul(x, x, y);
    if (valid) mt.store_limbs(A.inv_child + i * L, x);
  }
}

// ------------------------------------------------------------------------------------------------
// Modular inverse of ONE number (the root of the inversion tree) by a warp-wide binary extended
// Euclid: the 32 lanes hold K consecutive 32-bit words each; carries and comparisons cross lanes
// through ballots.  All control flow is warp-uniform.
template <int K>
struct WarpBig {
  uint32_t w[K];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < K; i++) w[i] = 0;
  }
};

template <int K>
__device__ __forceinline__ uint32_t wb_add(WarpBig<K>& a, const WarpBig<K>& b, uint32_t cin0, bool complement_b) {
  // a += (complement_b ? ~b : b) + cin0 (cin0 enters at lane 0); returns the carry out of the top lane
  const int lane = threadIdx.x & 31;
  uint32_t c = (lane == 0) ? cin0 : 0u;
  uint32_t allones = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < K; i++) {
    uint32_t bv = complement_b ? ~b.w[i] : b.w[i];
    uint64_t s = (uint64_t)a.w[i] + bv + c;
    a.w[i] = (uint32_t)s;
    c = (uint32_t)(s >> 32);
    allones &= a.w[i];
  }
  uint32_t G = __ballot_sync(0xffffffffu, c != 0);
  uint32_t P = __ballot_sync(0xffffffffu, allones == 0xffffffffu);
  uint64_t S = (uint64_t)P + ((uint64_t)G << 1);
  uint32_t C = (uint32_t)S ^ P;
  uint32_t ci = (C >> lane) & 1u;
#pragma unroll
  for (int i = 0; i < K; i++) {
    uint64_t s = (uint64_t)a.w[i] + ci;
    a.w[i] = (uint32_t)s;
    ci = (uint32_t)(s >> 32);
  }
  return (uint32_t)(S >> 32) & 1u;
}

template <int K>
__device__ __forceinline__ void wb_shr1(WarpBig<K>& a) {
  uint32_t next0 = __shfl_down_sync(0xffffffffu, a.w[0], 1);
  if ((threadIdx.x & 31) == 31) next0 = 0;
#pragma unroll
  for (int i = 0; i < K - 1; i++) a.w[i] = (a.w[i] >> 1) | (a.w[i + 1] << 31);
  a.w[K - 1] = (a.w[K - 1] >> 1) | (next0 << 31);
}

template <int K>
__device__ __forceinline__ bool wb_ge(const WarpBig<K>& a, const WarpBig<K>& b) {
  bool gt = false, lt = false;
#pragma unroll
  for (int i = K - 1; i >= 0; i--) {
    if (!gt && !lt) { gt = a.w[i] > b.w[i]; lt = a.w[i] < b.w[i]; }
  }
  uint32_t GT = __ballot_sync(0xffffffffu, gt), LT = __ballot_sync(0xffffffffu, lt);
  return GT >= LT;
}

template <int K>
__device__ __forceinline__ bool wb_is_small(const WarpBig<K>& a, uint32_t v) {
  // a == v for a single-word value v
  const int lane = threadIdx.x & 31;
  uint32_t any = 0;
#pragma unroll
  for (int i = 0; i < K; i++) any |= (lane == 0 && i == 0) ? (a.w[i] ^ v) : a.w[i];
  return __ballot_sync(0xffffffffu, any != 0) == 0;
}

template <int K>
__device__ __forceinline__ bool wb_odd(const WarpBig<K>& a) {
  return (__shfl_sync(0xffffffffu, a.w[0], 0) & 1u) != 0;
}

struct RootInvArgs {
  ModDev mod;
  uint32_t* root;        // digit form, in: Mont(a); out: Mont(a^-1)
  uint32_t* words;       // scratch, 32 * K words
  const uint32_t* nwords;// modulus as 32 * K little-endian words (zero padded)
  int* status;           // set to 1 when a is not a unit
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32) k_root_inverse(RootInvArgs A) {
  using M = Mont<LPT, TPI>;
  constexpr int L = LPT * TPI;
  constexpr int K = L / 32 + 1;
  constexpr int T = 32 * K;
  const int lane = threadIdx.x & 31;
  M mt;
  mt.init(A.mod.n, A.mod.np);
  uint32_t x[LPT], y[LPT];
  // every group works on the same number; group 0's stores are the ones kept
  mt.load_limbs(x, A.root);
  mt.set_one(y);
  mt.mul(x, x, y);
  // plain a; group 0 writes its limbs, everything above L is zero
  mt.store_words(A.words, L, x, lane < TPI);
  for (int k = L + lane; k < T; k += 32) A.words[k] = 0;
  __syncwarp();
  __threadfence_block();
  WarpBig<K> u, v, x1, x2, nn;
#pragma unroll
  for (int i = 0; i < K; i++) {
    u.w[i] = A.words[lane * K + i];
    nn.w[i] = A.nwords[lane * K + i];
    v.w[i] = nn.w[i];
  }
  x1.zero(); x2.zero();
  if (lane == 0) x1.w[0] = 1;
  bool ok = true;
  if (wb_is_small<K>(u, 0)) ok = false;
  while (ok) {
    while (!wb_odd<K>(u)) {
      wb_shr1<K>(u);
      if (wb_odd<K>(x1)) wb_add<K>(x1, nn, 0, false);
      wb_shr1<K>(x1);
    }
    while (!wb_odd<K>(v)) {
      wb_shr1<K>(v);
      if (wb_odd<K>(x2)) wb_add<K>(x2, nn, 0, false);
      wb_shr1<K>(x2);
    }
    if (wb_is_small<K>(u, 1)) break;
    if (wb_is_small<K>(v, 1)) { x1 = x2; break; }
    if (wb_ge<K>(u, v)) {
      wb_add<K>(u, v, 1, true);                   // u -= v
      if (wb_is_small<K>(u, 0)) { ok = false; break; }
      if (!wb_ge<K>(x1, x2)) wb_add<K>(x1, nn, 0, false);
      wb_add<K>(x1, x2, 1, true);                 // x1 = x1 - x2 (mod n)
    } else {
      wb_add<K>(v, u, 1, true);
      if (!wb_ge<K>(x2, x1)) wb_add<K>(x2, nn, 0, false);
      wb_add<K>(x2, x1, 1, true);
    }
  }
  if (!ok) {
    if (lane == 0) *A.status = 1;
    return;
  }
#pragma unroll
  for (int i = 0; i < K; i++) A.words[lane * K + i] = x1.w[i];
  __syncwarp();
  __threadfence_block();
  mt.load_words(x, A.words, L);
  mt.load_limbs(y, A.mod.r2);
  mt.mul(x, x, y);                                // Mont(a^-1)
  if (lane < TPI) mt.store_limbs(A.root, x);
}

// ------------------------------------------------------------------------------------------------
// Scalar preparation: residue k (wn words) -> sign and magnitude (operators.py:60: k > n - max_int
// selects the inverse base and the exponent n - k).  One thread per scalar.
struct ScalarPrepArgs {
  const uint32_t* k;        // nscal residues, wn words each
  const uint32_t* nwords;   // n
  const uint32_t* negband;  // n - max_int
  int wn;
  long nscal;
  long rows, cols;          // output index = transpose ? (col * rows + row) : linear   (input linear = row * cols + col)
  int transpose;
  int raw;                  // 1: exponent is the residue itself, never negative (paillier.hmul_raw)
  uint64_t* mag64;          // low 64 bits of the magnitude
  uint8_t* neg;
  int* maxbits;             // atomicMax of the magnitude bit lengths
  int* nneg;                // count of negative scalars
};

__global__ void k_scalar_prep(ScalarPrepArgs A) {
  long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = e < A.nscal;
  if (!live) e = A.nscal - 1;
  const uint32_t* k = A.k + e * A.wn;
  // k > negband ?
  int cmp = 0;
  for (int i = A.wn - 1; i >= 0 && cmp == 0; i--) {
    uint32_t a = k[i], b = A.negband[i];
    cmp = a > b ? 1 : (a < b ? -1 : 0);
  }
  const bool neg = cmp > 0 && !A.raw;
  uint64_t lo = 0;
  int bits = 0;
  uint32_t borrow = 0;
  for (int i = 0; i < A.wn; i++) {
    uint32_t v;
    if (neg) {
      uint64_t d = (uint64_t)A.nwords[i] - k[i] - borrow;
      v = (uint32_t)d;
      borrow = (uint32_t)(d >> 63);
    } else {
      v = k[i];
    }
    if (i == 0) lo = v;
    if (i == 1) lo |= (uint64_t)v << 32;
    if (v) bits = i * 32 + (32 - __clz(v));
  }
  long o = e;
  if (A.transpose) { long r = e / A.cols, c = e - r * A.cols; o = c * A.rows + r; }
  if (live) {
    A.mag64[o] = lo;
    A.neg[o] = neg ? 1 : 0;
  }
  // one atomic per warp, not per scalar (2e8 scalars at BASELINE configs[3])
  const int wbits = __reduce_max_sync(0xffffffffu, live ? bits : 0);
  const int wneg = __popc(__ballot_sync(0xffffffffu, live && neg));
  if ((threadIdx.x & 31) == 0) {
    atomicMax(A.maxbits, wbits);
    if (wneg) atomicAdd(A.nneg, wneg);
  }
}

// The same compact form straight from doubles (encoding.py:54-78 with a target exponent): the feature matrices of a
// federated run never need their 256-byte residues -- hb_matvec only reads sign and magnitude.  info[0] = max bit
// length, info[1] = negatives, info[2] = values whose magnitude does not fit 64 bits (the caller then encodes full
// residues instead).  Rounding is round-half-even on the exact binary value, like k_encode_f64.
struct CompactEncArgs {
  const double* values; long nscal; long rows, cols; int exponent;
  uint64_t* mag64; uint8_t* neg; int* info;
};

__global__ void k_encode_compact(CompactEncArgs A) {
  long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = e < A.nscal;
  if (!live) e = A.nscal - 1;
  const unsigned long long bits = (unsigned long long)__double_as_longlong(A.values[e]);
  const bool negv = (bits >> 63) != 0;
  const int e11 = (int)((bits >> 52) & 0x7ff);
  unsigned long long mant = bits & 0xfffffffffffffull;
  int e2;
  if (e11 == 0) e2 = -1074; else { mant |= 1ull << 52; e2 = e11 - 1075; }
  long shift = (long)e2 - 4L * A.exponent;        // scaled = mant * 2^shift
  bool wide = e11 == 0x7ff;                        // non-finite: never compact
  if (shift < 0) {
    const long s = -shift;
    if (s >= 64) mant = 0;
    else {
      unsigned long long q = mant >> s, rem = mant & ((1ull << s) - 1ull), half = 1ull << (s - 1);
      if (rem > half || (rem == half && (q & 1ull))) q++;
      mant = q;
    }
    shift = 0;
  }
  int nb = mant ? 64 - __clzll(mant) : 0;
  if (mant && nb + shift > 64) wide = true;
  const unsigned long long mag = (mant && !wide) ? (mant << shift) : 0ull;
  nb = (mant && !wide) ? nb + (int)shift : 0;
  const bool neg = negv && mag != 0;
  const long r = e / A.cols, c = e - r * A.cols;
  if (live) {
    A.mag64[c * A.rows + r] = mag;
    A.neg[c * A.rows + r] = neg ? 1 : 0;
  }
  const int wbits = __reduce_max_sync(0xffffffffu, live ? nb : 0);
  const int wneg = __popc(__ballot_sync(0xffffffffu, live && neg));
  const int wwide = __popc(__ballot_sync(0xffffffffu, live && wide));
  if ((threadIdx.x & 31) == 0) {
    atomicMax(A.info, wbits);
    if (wneg) atomicAdd(A.info + 1, wneg);
    if (wwide) atomicAdd(A.info + 2, wwide);
  }
}

// ------------------------------------------------------------------------------------------------
// Variable-exponent power (fixed window, uniform control flow):
//   out[e] = base(e) ^ mag(e)   with base = c or c^-1 (digit form, Montgomery) picked by the sign.
// Exponents are either 64-bit magnitudes (mag64) or, for the general path, full residues from which
// the magnitude is recomputed (n - k for negatives).
struct PowVarArgs {
  ModDev mod;
  const uint32_t* base;      // digit form Mont(c), indexed by e / c_div
  const uint32_t* base_inv;  // digit form Mont(c^-1) (may be null when no scalar is negative)
  long c_div;
  const uint64_t* mag64;     // indexed by e % k_period (null on the general path)
  const uint8_t* neg;        // indexed by e % k_period
  const uint32_t* kres;      // general path: residues, wn words, indexed by e % k_period
  const uint32_t* nwords;
  int wn;
  long k_period;
  int ebits;                 // exponent bits to process (multiple of win)
  int win;                   // window bits (1..4)
  uint32_t* tbl; long tbl_stride;
  uint32_t* out;             // words (wc each), or digit form when out_mont
  int wc;
  long count;
  int out_mont;
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_powvar(PowVarArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  uint32_t* tw = A.tbl + wg * A.tbl_stride;
  const long ntiles = (A.count + IPW - 1) / IPW;
  const int nent = 1 << A.win;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long e = valid ? inst : A.count - 1;
    long ki = e % A.k_period;
    const bool neg = A.neg[ki] != 0;
    uint32_t x[LPT], y[LPT];
    const uint32_t* bp = (neg ? A.base_inv : A.base) + (e / A.c_div) * L;
    mt.load_limbs(y, bp);
    // table: slot 0 = Mont(1), slot 1 = b, slot i = b^i
    mt.load_limbs(x, A.mod.r1);
    tile_store<LPT>(tw, 0, x);
    tile_store<LPT>(tw, 1, y);
#pragma unroll
    for (int k = 0; k < LPT; k++) x[k] = y[k];
#pragma unroll 1
    for (int i = 2; i < nent; i++) {
      mt.mul(x, x, y);
      tile_store<LPT>(tw, i, x);
    }
    // exponent access
    const uint32_t* kw = A.kres ? A.kres + ki * A.wn : nullptr;
    const uint64_t m64 = A.mag64 ? A.mag64[ki] : 0;
    auto digit_at = [&](int bitpos) -> uint32_t {
      // `win` bits of the magnitude starting at bitpos
      if (!kw) return (uint32_t)(m64 >> bitpos) & (uint32_t)(nent - 1);
      // general path: magnitude word by word (n - k computed on the fly with a borrow scan)
      int wi = bitpos >> 5, sh = bitpos & 31;
      uint32_t wlo, whi;
      if (!neg) {
        wlo = wi < A.wn ? kw[wi] : 0u;
        whi = wi + 1 < A.wn ? kw[wi + 1] : 0u;
      } else {
        uint32_t borrow = 0, v = 0, v1 = 0;
        for (int i = 0; i <= wi + 1 && i < A.wn; i++) {
          uint64_t d = (uint64_t)A.nwords[i] - kw[i] - borrow;
          borrow = (uint32_t)(d >> 63);
          if (i == wi) v = (uint32_t)d;
          if (i == wi + 1) v1 = (uint32_t)d;
        }
        wlo = v; whi = v1;
      }
      uint64_t both = (uint64_t)wlo | ((uint64_t)whi << 32);
      return (uint32_t)(both >> sh) & (uint32_t)(nent - 1);
    };
    int pos = A.ebits - A.win;
    {
      uint32_t d = digit_at(pos);
      // per-group table index: lanes of one group agree, groups may differ
      const int ln = threadIdx.x & 31;
#pragma unroll
      for (int k = 0; k < LPT; k++) x[k] = tw[((int)d * LPT + k) * 32 + ln];
    }
#pragma unroll 1
    for (pos -= A.win; pos >= 0; pos -= A.win) {
#pragma unroll 1
      for (int s = 0; s < A.win; s++) mt.mul(x, x, x);
      uint32_t d = digit_at(pos);
      const int ln = threadIdx.x & 31;
#pragma unroll
      for (int k = 0; k < LPT; k++) y[k] = tw[((int)d * LPT + k) * 32 + ln];
      mt.mul(x, x, y);
    }
    if (A.out_mont) {
      if (valid) mt.store_limbs(A.out + e * L, x);
    } else {
      mt.set_one(y);
      mt.mul(x, x, y);
      mt.store_words(A.out + e * A.wc, A.wc, x, valid);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Bases whose inverse is needed: sel[i] = cm[i] when one of the scalars paired with base i is negative, Mont(1)
// otherwise -- so that a non-unit ciphertext only fails the batch inversion when the reference would invert it too
// (operators.py:60-61 inverts per element).  Base i meets the scalars k[(i * c_div + j) % k_period], j < c_div.
struct MaskArgs { const uint32_t* cm; const uint32_t* one; const uint8_t* neg; long nbase; long c_div; long k_period; int L; uint32_t* sel; };

__global__ void k_mask_bases(MaskArgs A) {
  const long total = A.nbase * A.L;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const long i = idx / A.L; const int k = (int)(idx - i * A.L);
    bool need = false;
    for (long j = 0; j < A.c_div && !need; j++) need = A.neg[(i * A.c_div + j) % A.k_period] != 0;
    A.sel[idx] = need ? A.cm[idx] : A.one[k];
  }
}

// ------------------------------------------------------------------------------------------------
// Product reduction pass: out[g * parts + p] = prod_{t in chunk p of group g} c[g*gstride + t*estride]
// Inputs and outputs are plain words; every work item performs exactly `clen` multiplications (short
// chunks are padded with ones) so the Montgomery deficit R^-(clen-1) is the same everywhere and is
// repaired with one multiplication by R^clen, built by square-and-multiply on the fly.
struct ProductArgs {
  ModDev mod;
  const uint32_t* c; int wc;
  int win;                  // words per INPUT element (wc, or wn when multiplying plaintext-width values)
  long ngroups, glen, gstride, estride;
  long parts, clen;
  uint32_t* out;
  int in_mont;              // inputs are digit form (L limbs each): no deficit to repair
  int out_mont;             // write digit form
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_product_pass(ProductArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long nitems = A.ngroups * A.parts;
  const long ntiles = (nitems + IPW - 1) / IPW;
  // Plain inputs leave x = prod / R^(clen-1): one multiplication by R^(clen + out_mont) repairs it.
  // h_j = R^(j+1), mul(h_a, h_b) = h_(a+b): built left to right below; we need h_(clen + out_mont - 1).
  // Digit-form inputs carry no deficit: Mont(prod) is already there (multiplied by one when plain words are wanted).
  uint32_t fix[LPT];
  if (!A.in_mont) {
    uint32_t h1[LPT];
    mt.load_limbs(fix, A.mod.r1);     // h_0
    mt.load_limbs(h1, A.mod.r2);      // h_1
    long idx = A.clen - 1 + A.out_mont;
    int top = 63 - __clzll((unsigned long long)(idx | 1));
#pragma unroll 1
    for (int b = top; b >= 0; b--) {
      mt.mul(fix, fix, fix);
      if ((idx >> b) & 1) mt.mul(fix, fix, h1);
    }
  }
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < nitems;
    long it = valid ? inst : nitems - 1;
    long grp = it / A.parts, part = it - grp * A.parts;
    long t0 = part * A.clen;
    uint32_t x[LPT], y[LPT];
    mt.set_one(x);
    bool first = true;
#pragma unroll 1
    for (long i = 0; i < A.clen; i++) {
      long t = t0 + i;
      if (t < A.glen) {
        if (A.in_mont) mt.load_limbs(y, A.c + (grp * A.gstride + t * A.estride) * L);
        else mt.load_words(y, A.c + (grp * A.gstride + t * A.estride) * A.win, A.win);
      } else if (A.in_mont) mt.load_limbs(y, A.mod.r1);
      else mt.set_one(y);
      if (first) {
#pragma unroll
        for (int k = 0; k < LPT; k++) x[k] = y[k];
        first = false;
      } else {
        mt.mul(x, x, y);
      }
    }
    if (!A.in_mont) {
      mt.mul(x, x, fix);    // clen - 1 deficits repaired: x * R^(clen + out_mont) / R
    } else if (!A.out_mont) {
      mt.set_one(y);
      mt.mul(x, x, y);
    }
    if (A.out_mont) { if (valid) mt.store_limbs(A.out + it * L, x); }
    else mt.store_words(A.out + it * A.wc, A.wc, x, valid);
  }
}

// ------------------------------------------------------------------------------------------------
// Encrypted matrix-vector product, bucket method.  For every column j and window w of the scalar
// magnitudes the rows are counting-sorted by (digit value, sign); fixed-size segments of the sorted
// list are multiplied up by one group each; per-bucket products are combined and folded with the
// running-sum identity  prod_v B_v^v = prod_v (prod_{u>=v} B_u); windows are merged by Horner.
struct SortArgs {
  const uint64_t* mag64;   // [d][colstride], the n rows of this call starting at the pointer
  const uint8_t* neg;      // same layout
  long colstride;          // rows of the whole matrix (>= n when the call covers a block of rows)
  long n; int d; int nwin; int cbits;
  uint32_t* boff;          // [d][nwin][NB + 1] exclusive offsets
  uint32_t* sorted;        // [d][nwin][n]   rows ordered by bucket (boff delimits the buckets)
};

__global__ void __launch_bounds__(256) k_bucket_sort(SortArgs A) {
  extern __shared__ uint32_t hist[];      // NB + 1 counters, then NB cursors
  const int NB = 2 << A.cbits;
  const int j = blockIdx.x / A.nwin, w = blockIdx.x % A.nwin;
  uint32_t* cur = hist + NB + 1;
  for (int i = threadIdx.x; i <= NB; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const uint64_t* mg = A.mag64 + (long)j * A.colstride;
  const uint8_t* ng = A.neg + (long)j * A.colstride;
  const uint32_t vmask = (1u << A.cbits) - 1u;
  const int sh = w * A.cbits;
  for (long t = threadIdx.x; t < A.n; t += blockDim.x) {
    uint32_t v = (uint32_t)(mg[t] >> sh) & vmask;
    atomicAdd(&hist[v * 2 + ng[t]], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int b = 0; b < NB; b++) { uint32_t c = hist[b]; hist[b] = run; cur[b] = run; run += c; }
    hist[NB] = run;
  }
  __syncthreads();
  uint32_t* bo = A.boff + ((long)j * A.nwin + w) * (NB + 1);
  for (int i = threadIdx.x; i <= NB; i += blockDim.x) bo[i] = hist[i];
  uint32_t* so = A.sorted + ((long)j * A.nwin + w) * A.n;
  for (long t = threadIdx.x; t < A.n; t += blockDim.x) {
    uint32_t v = (uint32_t)(mg[t] >> sh) & vmask;
    uint32_t b = v * 2 + ng[t];
    uint32_t p = atomicAdd(&cur[b], 1u);
    so[p] = (uint32_t)t;
  }
}

struct SegArgs {
  ModDev mod;
  const uint32_t* cm;      // digit form Mont(c_t), [n][L]
  const uint32_t* boff; const uint32_t* sorted;
  long n; int d; int nwin; int cbits;
  int seglen; long nseg;   // segments per (j, w)
  uint32_t* part;          // [d][nwin][nseg + NB][L] partial products, slot = seg + bucket
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_bucket_segments(SegArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const int NB = 2 << A.cbits;
  const long nitems = (long)A.d * A.nwin * A.nseg;
  const long ntiles = (nitems + IPW - 1) / IPW;
  uint32_t one[LPT];
  mt.load_limbs(one, A.mod.r1);
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < nitems;
    long it = valid ? inst : nitems - 1;
    long jw = it / A.nseg, seg = it - jw * A.nseg;
    const uint32_t* bo = A.boff + jw * (NB + 1);
    const uint32_t* so = A.sorted + jw * A.n;
    uint32_t* pt = A.part + jw * (A.nseg + NB) * L;
    const long a0 = bo[2];                      // buckets 0 and 1 hold the zero digits
    const long p0 = a0 + seg * A.seglen;
    uint32_t acc[LPT], y[LPT];
#pragma unroll
    for (int k = 0; k < LPT; k++) acc[k] = one[k];
    int cur = -1;
    // bucket of the segment's first entry: the last b with boff[b] <= p0 (empty buckets share an offset)
    int bk = 2;
    if (valid && p0 < A.n) {
      int lo = 2, hi = NB - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((long)bo[mid] <= p0) lo = mid; else hi = mid - 1;
      }
      bk = lo;
    }
#pragma unroll 1
    for (int i = 0; i < A.seglen; i++) {
      long p = p0 + i;
      bool have = valid && p < A.n;
      uint32_t ent = have ? so[p] : 0u;
      if (have) { while ((long)bo[bk + 1] <= p) bk++; }
      int b = have ? bk : cur;
      bool change = b != cur;
      if (change && cur >= 0) mt.store_limbs(pt + (seg + cur) * L, acc);
      if (have) mt.load_limbs(y, A.cm + (long)ent * L);
      else {
#pragma unroll
        for (int k = 0; k < LPT; k++) y[k] = one[k];
      }
      if (change) {
#pragma unroll
        for (int k = 0; k < LPT; k++) acc[k] = one[k];
      }
      mt.mul(acc, acc, y);
      cur = b;
    }
    if (cur >= 0) mt.store_limbs(pt + (seg + cur) * L, acc);
  }
}

// per (j, w, bucket): product of the partials of that bucket -> bucket[j][w][b] (Mont(1) when empty)
struct CombineArgs {
  ModDev mod;
  const uint32_t* boff; const uint32_t* part;
  int d; int nwin; int cbits; int seglen; long nseg;
  uint32_t* bucket;        // [d][nwin][NB][L]
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_bucket_combine(CombineArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const int NB = 2 << A.cbits;
  const long nitems = (long)A.d * A.nwin * NB;
  const long ntiles = (nitems + IPW - 1) / IPW;
  uint32_t one[LPT];
  mt.load_limbs(one, A.mod.r1);
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < nitems;
    long it = valid ? inst : nitems - 1;
    long jw = it / NB; int b = (int)(it - jw * NB);
    const uint32_t* bo = A.boff + jw * (NB + 1);
    const uint32_t* pt = A.part + jw * (A.nseg + NB) * L;
    const long a0 = bo[2];
    long lo = bo[b], hi = bo[b + 1];
    long s_lo = 0, cnt = 0;
    if (valid && b >= 2 && hi > lo) {
      s_lo = (lo - a0) / A.seglen;
      cnt = (hi - 1 - a0) / A.seglen - s_lo + 1;
    }
    // uniform trip count inside the warp
    long maxcnt = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      long other = __shfl_xor_sync(0xffffffffu, maxcnt, o);
      maxcnt = other > maxcnt ? other : maxcnt;
    }
    uint32_t acc[LPT], y[LPT];
#pragma unroll
    for (int k = 0; k < LPT; k++) acc[k] = one[k];
#pragma unroll 1
    for (long i = 0; i < maxcnt; i++) {
      if (i < cnt) mt.load_limbs(y, pt + (s_lo + i + b) * L);
      else {
#pragma unroll
        for (int k = 0; k < LPT; k++) y[k] = one[k];
      }
      mt.mul(acc, acc, y);
    }
    if (valid) mt.store_limbs(A.bucket + it * L, acc);
  }
}

// per (j, w, sign): T = prod_v B_v^v by running sums -> win[j][sign][w]
struct RunningArgs {
  ModDev mod;
  const uint32_t* bucket; int d; int nwin; int cbits;
  uint32_t* win;           // [d][2][nwin][L]
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_bucket_running(RunningArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const int NB = 2 << A.cbits, NV = 1 << A.cbits;
  const long nitems = (long)A.d * A.nwin * 2;
  const long ntiles = (nitems + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < nitems;
    long it = valid ? inst : nitems - 1;
    long jw = it >> 1; int s = (int)(it & 1);
    long j = jw / A.nwin; int w = (int)(jw - j * A.nwin);
    const uint32_t* bk = A.bucket + jw * NB * L;
    uint32_t acc[LPT], tot[LPT], y[LPT];
    mt.load_limbs(acc, A.mod.r1);
    mt.load_limbs(tot, A.mod.r1);
#pragma unroll 1
    for (int v = NV - 1; v >= 1; v--) {
      mt.load_limbs(y, bk + (long)(v * 2 + s) * L);
      mt.mul(acc, acc, y);
      mt.mul(tot, tot, acc);
    }
    if (valid) mt.store_limbs(A.win + ((j * 2 + s) * A.nwin + w) * L, tot);
  }
}

// The same fold in G parallel pieces for wide windows (thousands of buckets make the loop above the longest thing
// in the call): piece g covers the digit values [lo, hi), lo = 1 + g * len, and produces
//   tot_g = prod_v B_v^(v - lo + 1)   and   acc_g = prod_v B_v,
// so that  prod_v B_v^v = prod_g tot_g * acc_g^(lo_g - 1)  (k_bucket_running_join).
struct RunningSegArgs {
  ModDev mod;
  const uint32_t* bucket; int d; int nwin; int cbits; int pieces;
  uint32_t* tot;           // [d * nwin * 2][pieces][L]
  uint32_t* acc;           // same shape
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_bucket_running_seg(RunningSegArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const int NB = 2 << A.cbits, NV = 1 << A.cbits;
  const int len = (NV - 1 + A.pieces - 1) / A.pieces;
  const long nitems = (long)A.d * A.nwin * 2 * A.pieces;
  const long ntiles = (nitems + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < nitems;
    long it = valid ? inst : nitems - 1;
    const long jws = it / A.pieces; const int piece = (int)(it - jws * A.pieces);
    const long jw = jws >> 1; const int s = (int)(jws & 1);
    const uint32_t* bk = A.bucket + jw * NB * L;
    const int lo = 1 + piece * len, hi = min(NV, lo + len);
    uint32_t acc[LPT], tot[LPT], y[LPT];
    mt.load_limbs(acc, A.mod.r1);
    mt.load_limbs(tot, A.mod.r1);
#pragma unroll 1
    for (int i = 0; i < len; i++) {                  // uniform trip count; values past hi multiply by one
      const int v = lo + len - 1 - i;
      if (v < hi) mt.load_limbs(y, bk + (long)(v * 2 + s) * L);
      else mt.load_limbs(y, A.mod.r1);
      mt.mul(acc, acc, y);
      mt.mul(tot, tot, acc);
    }
    if (valid) {
      mt.store_limbs(A.tot + it * L, tot);
      mt.store_limbs(A.acc + it * L, acc);
    }
  }
}

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_bucket_running_join(RunningSegArgs A, uint32_t* win) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const int NV = 1 << A.cbits;
  const int len = (NV - 1 + A.pieces - 1) / A.pieces;
  const long nitems = (long)A.d * A.nwin * 2;
  const long ntiles = (nitems + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < nitems;
    long it = valid ? inst : nitems - 1;
    const long jw = it >> 1; const int s = (int)(it & 1);
    const long j = jw / A.nwin; const int w = (int)(jw - j * A.nwin);
    uint32_t total[LPT], x[LPT], y[LPT];
    mt.load_limbs(total, A.mod.r1);
#pragma unroll 1
    for (int piece = 0; piece < A.pieces; piece++) {
      mt.load_limbs(y, A.tot + (it * A.pieces + piece) * L);
      mt.mul(total, total, y);
      // acc^(lo - 1), lo - 1 = piece * len: left-to-right square and multiply, uniform over the warp
      const int e = piece * len;
      mt.load_limbs(y, A.acc + (it * A.pieces + piece) * L);
      mt.load_limbs(x, A.mod.r1);
#pragma unroll 1
      for (int b = 30 - __clz(NV | 1) + 1; b >= 0; b--) {
        mt.mul(x, x, x);
        if ((e >> b) & 1) mt.mul(x, x, y);
      }
      mt.mul(total, total, x);
    }
    if (valid) mt.store_limbs(win + ((j * 2 + s) * A.nwin + w) * L, total);
  }
}

// per (j, sign): Horner over the windows, most significant first -> ab[j][sign]
struct HornerArgs {
  ModDev mod;
  const uint32_t* win; int d; int nwin; int cbits;
  uint32_t* ab;            // [d][2][L]  A_j (sign 0) and B_j (sign 1), digit form
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_window_horner(HornerArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long nitems = (long)A.d * 2;
  const long ntiles = (nitems + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < nitems;
    long it = valid ? inst : nitems - 1;
    const uint32_t* wv = A.win + it * A.nwin * L;
    uint32_t x[LPT], y[LPT];
    mt.load_limbs(x, wv + (long)(A.nwin - 1) * L);
#pragma unroll 1
    for (int w = A.nwin - 2; w >= 0; w--) {
#pragma unroll 1
      for (int s = 0; s < A.cbits; s++) mt.mul(x, x, x);
      mt.load_limbs(y, wv + (long)w * L);
      mt.mul(x, x, y);
    }
    if (valid) mt.store_limbs(A.ab + it * L, x);
  }
}

// Multiply digit-form partial results of several ranks / row blocks:  dst[i] = prod_r src[r][i]
struct FoldArgs { ModDev mod; const uint32_t* src; long rstride; int nr; long count; uint32_t* dst; };

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_fold(FoldArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long i = valid ? inst : A.count - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_limbs(x, A.src + i * L);
#pragma unroll 1
    for (int r = 1; r < A.nr; r++) {
      mt.load_limbs(y, A.src + r * A.rstride + i * L);
      mt.mul(x, x, y);
    }
    if (valid) mt.store_limbs(A.dst + i * L, x);
  }
}

// out_j = A_j * Binv_j  ->  plain words
struct FinishArgs { ModDev mod; const uint32_t* ab; const uint32_t* binv; int d; uint32_t* out; int wc; int out_mont; };

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_matvec_finish(FinishArgs A) {
  HB_GROUP_PROLOGUE(LPT, TPI)
  M mt;
  mt.init(A.mod.n, A.mod.np);
  const long ntiles = (A.d + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.d;
    long j = valid ? inst : A.d - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_limbs(x, A.ab + (j * 2) * L);
    if (A.binv) {
      mt.load_limbs(y, A.binv + j * L);
      mt.mul(x, x, y);
    }
    if (A.out_mont) {
      if (valid) mt.store_limbs(A.out + j * L, x);
    } else {
      mt.set_one(y);
      mt.mul(x, x, y);
      mt.store_words(A.out + j * A.wc, A.wc, x, valid);
    }
  }
}

// gather the B_j (sign 1) entries of ab into a dense array for the inversion tree
__global__ void k_gather_b(const uint32_t* ab, uint32_t* dst, int d, int L) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)d * L) return;
  long j = i / L; int k = (int)(i - j * L);
  dst[i] = ab[(j * 2 + 1) * L + k];
}

}  // namespace hb
