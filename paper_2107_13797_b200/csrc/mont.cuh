// Warp-cooperative, carry-free Montgomery arithmetic for sm_100a.
//
// This is the arithmetic core behind every modular operator of the reference's hot path
// (/root/reference/pkg/src/hebatch/operators.py:39-94: _k_encrypt, _k_obfuscate, _k_decrypt,
// _k_mul, _k_add, _k_product, _k_dot), which the reference delegates to gmpy2.powmod / mpz
// multiplication.  Nothing here is derived from GMP; the design follows what the B200 integer
// pipe actually does (profiles/r01_imad_peak.json):
//
//   * IMAD.WIDE.U32 (32x32+64 -> 64, no carry) issues at ~64 lanes/clk/SM,
//   * IMAD.WIDE.U32.X (the carry-in/carry-out form every 2^32-radix limb chain needs) issues at
//     HALF that rate.
//
// So numbers are held in radix 2^29 ("digits"), LPT digits per lane, TPI lanes per instance.  A digit
// product is < 2^58, a 64-bit column accumulator absorbs two of them per row for LPT (<= 31) rows, and a
// cheap carry-save pass every LPT rows keeps it there.  No carry chain ever touches the multiply
// pipe.  The price is (9/8)^2 = 1.27x more digit products than 32-bit limbs would need; the gain is
// 2x issue rate, and R = 2^(29*L) exceeds the modulus by >= 2^20, which removes every conditional
// subtraction between multiplications (values stay below 2N).
//
// Row-serial (CIOS-like) schedule, one row per digit b_j of the second operand:
//     acc[k] += a[k] * b_j            (all lanes, LPT independent IMAD.WIDE)
//     q       = (acc[0] * np) mod 2^29 on lane 0, broadcast by one shuffle
//     acc[k] += n[k] * q              (all lanes)
//     frame moves down one digit: acc[k] <- acc[k+1], the top column comes from the lane above.
// Validated lane-for-lane against Python integers by tools/mont_model.py.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hb {

constexpr int RB = 29;                          // radix bits
constexpr uint32_t DMASK = (1u << RB) - 1u;     // digit mask
constexpr unsigned FULLMASK = 0xffffffffu;

__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return (uint32_t)v; }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }
__device__ __forceinline__ uint64_t pack64(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }

// Per-lane view of one modulus: LPT digits of n, the Montgomery constant and lane-role masks.
template <int LPT, int TPI>
struct Mont {
  static_assert(LPT >= 3 && LPT <= 31, "carry-save bound needs 3 <= LPT <= 31");
  static_assert(TPI >= 2 && TPI <= 16 && (TPI & (TPI - 1)) == 0, "TPI must be 2,4,8,16");
  static constexpr int L = LPT * TPI;           // digits per number
  static constexpr uint32_t GM = (1u << TPI) - 1u;

  uint32_t n[LPT];     // modulus digits owned by this lane
  uint32_t np;         // -n^-1 mod 2^29
  int t;               // lane index inside the instance group
  int gshift;          // bit position of the group's lane 0 inside the warp
  uint32_t m0;         // all-ones on lane 0 of the group
  uint32_t mtop;       // all-ones on the top lane of the group

  __device__ __forceinline__ void init(const uint32_t* __restrict__ n_digits, uint32_t np_) {
    int lane = threadIdx.x & 31;
    t = lane & (TPI - 1);
    gshift = lane & ~(TPI - 1);
    m0 = (t == 0) ? 0xffffffffu : 0u;
    mtop = (t == TPI - 1) ? 0xffffffffu : 0u;
    np = np_;
#pragma unroll
    for (int i = 0; i < LPT; i++) n[i] = n_digits[t * LPT + i];
  }

  // One carry-save pass over 64-bit accumulators: every column keeps its low digit and hands bits
  // 29..57 to the next column and bits 58..63 to the one after.  Result columns are < 2^31.
  __device__ __forceinline__ void carry_save(uint64_t (&acc)[LPT], uint64_t& ovf) const {
    uint32_t d[LPT], e[LPT], f[LPT];
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      uint32_t lo = lo32(acc[i]), hi = hi32(acc[i]);
      d[i] = lo & DMASK;
      e[i] = __funnelshift_r(lo, hi, RB) & DMASK;
      f[i] = hi >> (2 * RB - 32);
    }
    uint32_t v0 = e[LPT - 1] + f[LPT - 2];      // for column 0 of the lane above
    uint32_t v1 = f[LPT - 1];                   // for column 1 of the lane above
    uint32_t u0 = __shfl_up_sync(FULLMASK, v0, 1, TPI) & ~m0;
    uint32_t u1 = __shfl_up_sync(FULLMASK, v1, 1, TPI) & ~m0;
    acc[0] = (uint64_t)(d[0] + u0);
    acc[1] = (uint64_t)(d[1] + e[0] + u1);
#pragma unroll
    for (int i = 2; i < LPT; i++) acc[i] = (uint64_t)(d[i] + e[i - 1] + f[i - 2]);
    ovf += (uint64_t)(v0 & mtop) + ((uint64_t)(v1 & mtop) << RB);
  }

  // r = a * b / R (mod n-ish): value(r) < value(a)*value(b)/R + N, digits of r < 2^29 + 2.
  // a and b may alias r.  Digits of a, b must be < 2^29 + 2^8.
  __device__ __forceinline__ void mul(uint32_t (&r)[LPT], const uint32_t (&a)[LPT],
                                      const uint32_t (&b)[LPT]) const {
    uint32_t unused[LPT];
    mul_impl<false>(r, a, b, unused);
  }

  // Same as mul(), and additionally hands back the Montgomery quotient digits: lane t receives
  // digits [t*LPT, (t+1)*LPT) of Q = -(a*b) * n^-1 mod R (exact digits).  Used for exact division:
  // when a*b is a multiple of n, a*b / n = (R - Q) mod R.
  __device__ __forceinline__ void mul_quot(uint32_t (&r)[LPT], uint32_t (&qd)[LPT],
                                           const uint32_t (&a)[LPT], const uint32_t (&b)[LPT]) const {
    mul_impl<true>(r, a, b, qd);
  }

  template <bool COLLECT>
  __device__ __forceinline__ void mul_impl(uint32_t (&r)[LPT], const uint32_t (&a)[LPT],
                                           const uint32_t (&b)[LPT], uint32_t (&qd)[LPT]) const {
    uint64_t acc[LPT];
#pragma unroll
    for (int i = 0; i < LPT; i++) acc[i] = 0;
    uint64_t ovf = 0;
#pragma unroll 1
    for (int s = 0; s < TPI; s++) {
#pragma unroll
      for (int i = 0; i < LPT; i++) {
        uint32_t bj = __shfl_sync(FULLMASK, b[i], s, TPI);
        acc[0] = mad_wide(a[0], bj, acc[0]);
        uint32_t q = (lo32(acc[0]) * np) & DMASK;
        q = __shfl_sync(FULLMASK, q, 0, TPI);
        if (COLLECT) { if (s == t) qd[i] = q; }
#pragma unroll
        for (int k = 1; k < LPT; k++) acc[k] = mad_wide(a[k], bj, acc[k]);
#pragma unroll
        for (int k = 0; k < LPT; k++) acc[k] = mad_wide(n[k], q, acc[k]);
        // move the frame down one digit
        uint32_t ol = lo32(acc[0]), oh = hi32(acc[0]);
        uint32_t rl = __shfl_down_sync(FULLMASK, ol, 1, TPI);
        uint32_t rh = __shfl_down_sync(FULLMASK, oh, 1, TPI);
        rl = mtop ? lo32(ovf) : rl;
        rh = mtop ? hi32(ovf) : rh;
        ovf = 0;
        // lane 0: the eliminated column's upper bits carry into the new column 0
        uint32_t cl = __funnelshift_r(ol, oh, RB) & m0;
        uint32_t ch = (oh >> RB) & m0;
#pragma unroll
        for (int k = 0; k < LPT - 1; k++) acc[k] = acc[k + 1];
        acc[LPT - 1] = pack64(rl, rh);
        acc[0] += pack64(cl, ch);
      }
      carry_save(acc, ovf);
    }
    // second, 32-bit pass: digit + carry of the column below
    uint32_t x[LPT];
#pragma unroll
    for (int i = 0; i < LPT; i++) x[i] = lo32(acc[i]);
    uint32_t cin = __shfl_up_sync(FULLMASK, x[LPT - 1] >> RB, 1, TPI) & ~m0;
    r[0] = (x[0] & DMASK) + cin;
#pragma unroll
    for (int i = 1; i < LPT; i++) r[i] = (x[i] & DMASK) + (x[i - 1] >> RB);
  }

  // One digit-wise renormalisation pass (for sums of two almost-normalised numbers).
  __device__ __forceinline__ void renorm(uint32_t (&r)[LPT]) const {
    uint32_t cin = __shfl_up_sync(FULLMASK, r[LPT - 1] >> RB, 1, TPI) & ~m0;
    uint32_t prev = r[0];
    r[0] = (prev & DMASK) + cin;
#pragma unroll
    for (int i = 1; i < LPT; i++) {
      uint32_t cur = r[i];
      r[i] = (cur & DMASK) + (prev >> RB);
      prev = cur;
    }
  }

  // Resolve pending single-bit carries between lanes.  On entry every digit is < 2^29 and g (0/1) is the
  // carry leaving this lane.  Returns the carry leaving the top lane (same value on all lanes).
  __device__ __forceinline__ uint32_t propagate(uint32_t (&r)[LPT], uint32_t g) const {
    uint32_t all = r[0];
#pragma unroll
    for (int i = 1; i < LPT; i++) all &= r[i];
    uint32_t G = (__ballot_sync(FULLMASK, g != 0) >> gshift) & GM;
    uint32_t P = (__ballot_sync(FULLMASK, all == DMASK) >> gshift) & GM;
    uint32_t S = P + (G << 1);
    uint32_t C = S ^ P;                 // bit t = carry entering lane t
    uint32_t c = (C >> t) & 1u;
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      uint32_t v = r[i] + c;
      r[i] = v & DMASK;
      c = v >> RB;
    }
    return (S >> TPI) & 1u;
  }

  // Exact digits (each < 2^29) from almost-normalised ones; returns the carry out of the number.
  __device__ __forceinline__ uint32_t normalize(uint32_t (&r)[LPT]) const {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      uint32_t v = r[i] + c;
      r[i] = v & DMASK;
      c = v >> RB;
    }
    return propagate(r, c);
  }

  // value(r) < 2N with almost-normalised digits  ->  canonical residue in [0, N), exact digits.
  __device__ __forceinline__ void canonical(uint32_t (&r)[LPT]) const {
    normalize(r);
    uint32_t s[LPT];
    uint32_t c = m0 & 1u;               // two's complement of the odd modulus: ~n + 1
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      uint32_t v = r[i] + (DMASK - n[i]) + c;
      s[i] = v & DMASK;
      c = v >> RB;
    }
    uint32_t ge = propagate(s, c);      // carry out of r + (R - N)  <=>  r >= N
#pragma unroll
    for (int i = 0; i < LPT; i++) r[i] = ge ? s[i] : r[i];
  }

  // Digits [doff + t*LPT, doff + (t+1)*LPT) of the little-endian 32-bit word array w[0..nwords).
  __device__ __forceinline__ void load_words(uint32_t (&r)[LPT], const uint32_t* __restrict__ w,
                                             int nwords, int doff) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      int bit = (doff + t * LPT + i) * RB;
      int k = bit >> 5, s = bit & 31;
      uint32_t lo = (k < nwords) ? w[k] : 0u;
      uint32_t hi = (k + 1 < nwords) ? w[k + 1] : 0u;
      r[i] = __funnelshift_r(lo, hi, s) & DMASK;
    }
  }

  // Exact digits -> little-endian 32-bit words, staged through sm (L + 2 words owned by the group).
  // Must be called by every lane of the warp; only groups with valid == true write to w.
  __device__ __forceinline__ void store_words(uint32_t* __restrict__ w, int nwords,
                                              const uint32_t (&r)[LPT], uint32_t* sm, bool valid = true) const {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < LPT; i++) sm[t * LPT + i] = r[i];
    if (t == 0) { sm[L] = 0; sm[L + 1] = 0; }
    __syncwarp();
    for (int k = t; k < nwords; k += TPI) {
      int bit = k << 5;
      int D = bit / RB, o = bit - D * RB;
      uint32_t word = 0;
      if (D < L) {
        uint64_t v = (uint64_t)sm[D] | ((uint64_t)sm[D + 1] << RB) | ((uint64_t)sm[D + 2] << (2 * RB));
        word = (uint32_t)(v >> o);
      }
      if (valid) w[k] = word;
    }
    __syncwarp();
  }

  // r = (R - r) mod R for exact digits r (two's complement in radix 2^29); result has exact digits.
  __device__ __forceinline__ void negate(uint32_t (&r)[LPT]) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) r[i] = DMASK - r[i];
    r[0] += m0 & 1u;
    normalize(r);
  }

  // r = r - 1 (mod R) for exact digits r.
  __device__ __forceinline__ void decrement(uint32_t (&r)[LPT]) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) r[i] += DMASK;
    normalize(r);
  }

  // True (on every lane of the group) when all digits of the group's number are zero.
  __device__ __forceinline__ bool is_zero(const uint32_t (&r)[LPT]) const {
    uint32_t any = r[0];
#pragma unroll
    for (int i = 1; i < LPT; i++) any |= r[i];
    uint32_t nz = (__ballot_sync(FULLMASK, any != 0) >> gshift) & GM;
    return nz == 0;
  }

  // The integer 1 as digits.
  __device__ __forceinline__ void set_one(uint32_t (&r)[LPT]) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) r[i] = 0;
    r[0] = m0 & 1u;
  }

  // Plain digit arrays (already radix 2^29, e.g. constants or scratch written by store_digits).
  __device__ __forceinline__ void load_digits(uint32_t (&r)[LPT], const uint32_t* __restrict__ d) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) r[i] = d[t * LPT + i];
  }
  __device__ __forceinline__ void store_digits(uint32_t* __restrict__ d, const uint32_t (&r)[LPT]) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) d[t * LPT + i] = r[i];
  }
};

}  // namespace hb
