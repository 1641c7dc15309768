// Warp-cooperative Montgomery arithmetic in radix 2^32 with hardware carry chains (sm_100a).
//
// Arithmetic core of every modular operator on the reference's hot path
// (/root/reference/pkg/src/hebatch/operators.py:39-94, which delegates to gmpy2.powmod / mpz "*" "%").
// Nothing here derives from GMP.  The shape follows what the B200 integer pipe measures
// (profiles/r01_imad_peak2.json, csrc/imad_peak2.cu):
//
//   * a 32x32->64 multiply-add (IMAD.WIDE.U32) issues at ~32 lanes/clk/SM whatever its form -- plain,
//     64-bit accumulating, or with carry-in/carry-out (IMAD.WIDE.U32.X);
//   * IADD3 / LOP3 / SHF run on another pipe at ~4x that rate.
//
// So the multiplier is the only scarce resource and every limb product should be exactly one
// IMAD.WIDE.U32.X with its addition and carry folded in; full 32-bit limbs minimise the product count
// (L^2 per operand pass).  A number has L = LPT * TPI limbs, LPT (even) per lane, TPI lanes.  Per lane
// two arrays of 64-bit accumulators are kept, E[i] on lane columns (2i, 2i+1) and O[i] on (2i+1, 2i+2),
// so a row a[k] * b_j is one carry chain over E (even k) and one over O (odd k).  After each row the
// frame moves down one 32-bit column: E and O swap roles, the eliminated low word of each lane goes to
// the lane below through one shuffle.  Whatever spills past a lane's top column collects in E[H], O[H]
// and crosses to the lane above once, after the last row.  Validated against Python integers by
// tools/mont32_model.py.
//
// Values are kept canonical: mul() returns a * b / R mod n in [0, n) for a < R, b < n, R = 2^(32 L).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hb {

constexpr unsigned FULLMASK = 0xffffffffu;

// r = c + a * b, carry out -> CC
__device__ __forceinline__ uint64_t mac_cc(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t r;
  asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %1, %2;\n\tadd.cc.u64 %0, t, %3;\n\t}" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}
// r = c + a * b + CC, carry out -> CC
__device__ __forceinline__ uint64_t macc_cc(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t r;
  asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %1, %2;\n\taddc.cc.u64 %0, t, %3;\n\t}" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t add_cc64(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("add.cc.u64 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t addc_cc64(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("addc.cc.u64 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t addc64(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("addc.u64 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint32_t add_cc32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t addc_cc32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t addc32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("addc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return (uint32_t)v; }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }

template <int LPT, int TPI>
struct Mont {
  static_assert(LPT >= 4 && LPT % 2 == 0, "LPT must be even and at least 4");
  static_assert(TPI >= 1 && TPI <= 32 && (TPI & (TPI - 1)) == 0, "TPI must be a power of two");
  static constexpr int H = LPT / 2;
  static constexpr int L = LPT * TPI;
  static constexpr uint32_t GM = TPI == 32 ? 0xffffffffu : ((1u << TPI) - 1u);

  // NS ("modulus in shared memory") -- an experiment kept behind -DHB_NS_SHARED_MODULUS, OFF by default.  At LPT = 48
  // (a 6144-bit modulus on four lanes) 48 limbs each of a and n next to 100 accumulator registers leave ptxas
  // spilling ~3 KB per thread around the hot loop, so this variant keeps the modulus in shared memory, once per
  // block (lane t's even limbs, then its odd limbs, at t * NS_STRIDE words: the four lanes' 16-byte reads fall on
  // disjoint banks) and streams it back as LDS.128 a few multiplies ahead of use.  Measured on the B200 at
  // 3072-bit keys (profiles/r02_shared_modulus_experiment.md): 28.3 k encrypt/s streamed (ld.volatile), 29.0 k
  // when ptxas is allowed to cache the loads in registers again, against 29.9 k for the register-resident modulus
  // with its spills -- the loads cost more issue slots than the spills they remove.  One warp per block.
#ifdef HB_NS_SHARED_MODULUS
  static constexpr bool NS = (LPT == 48);
#else
  static constexpr bool NS = false;
#endif
  static constexpr int NS_STRIDE = LPT + 4;
  static constexpr int STAGE_WORDS = L + TPI;
  static constexpr int NS_SMEM_WORDS = STAGE_WORDS * (32 / TPI) + TPI * NS_STRIDE;

  uint32_t n[NS ? 1 : LPT];   // modulus limbs owned by this lane (register shapes)
  uint32_t np;         // -n^-1 mod 2^32
  int t;               // lane index inside the group
  int gshift;          // position of the group's lane 0 in the warp
  bool top;            // this lane holds the most significant limbs
  uint32_t* ns_sa;     // NS: this instance's operand staging area (stride 32 / TPI)
  uint32_t* ns_n;      // NS: this lane's modulus limbs in shared memory (H even limbs, then H odd limbs)

  // smem: NS shapes only -- NS_SMEM_WORDS words, 16-byte aligned, private to this warp
  __device__ __forceinline__ void init(const uint32_t* __restrict__ n_limbs, uint32_t np_, uint32_t* smem = nullptr) {
    const int lane = threadIdx.x & 31;
    t = lane & (TPI - 1);
    gshift = lane & ~(TPI - 1);
    top = t == TPI - 1;
    np = np_;
    if constexpr (NS) {
      ns_sa = smem + lane / TPI;
      ns_n = smem + STAGE_WORDS * (32 / TPI) + t * NS_STRIDE;
      __syncwarp();
      if (lane < TPI) {
#pragma unroll
        for (int i = 0; i < LPT; i++) ns_n[(i >> 1) + (i & 1) * H] = n_limbs[t * LPT + i];
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int i = 0; i < LPT; i++) n[i] = n_limbs[t * LPT + i];
    }
  }
  // the lane's modulus limbs as a register array (NS shapes: read from shared memory)
  __device__ __forceinline__ void get_n(uint32_t (&v)[LPT]) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      if constexpr (NS) v[i] = ns_n[(i >> 1) + (i & 1) * H];
      else v[i] = n[i];
    }
  }
  // E, O += n * x with the modulus streamed from shared memory: 16-byte reads, NS_PF chunks ahead of the multiplies
#ifndef HB_NS_PF
#define HB_NS_PF 3
#endif
#ifdef HB_NS_VOLATILE
#define HB_NS_LD "ld.volatile.shared.v4.u32"
#else
#define HB_NS_LD "ld.shared.v4.u32"
#endif
  static constexpr int NS_PF = HB_NS_PF;
  __device__ __forceinline__ void mac_row_ns(uint64_t (&E)[H + 1], uint64_t (&O)[H + 1], uint32_t x) const {
    static_assert(!NS || H % 4 == 0, "shared-modulus rows read four limbs at a time");
    constexpr int NCH = H / 2;                      // chunks of four limbs: H / 4 of evens, then H / 4 of odds
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(ns_n);
    uint32_t c[NS_PF][4];
#pragma unroll
    for (int j = 0; j < NS_PF && j < NCH; j++)
      asm volatile(HB_NS_LD " {%0, %1, %2, %3}, [%4];"
                   : "=r"(c[j][0]), "=r"(c[j][1]), "=r"(c[j][2]), "=r"(c[j][3]) : "r"(base + 16u * j));
#pragma unroll
    for (int j = 0; j < NCH; j++) {
      const uint32_t v0 = c[j % NS_PF][0], v1 = c[j % NS_PF][1], v2 = c[j % NS_PF][2], v3 = c[j % NS_PF][3];
      if (j + NS_PF < NCH)
        asm volatile(HB_NS_LD " {%0, %1, %2, %3}, [%4];"
                     : "=r"(c[j % NS_PF][0]), "=r"(c[j % NS_PF][1]), "=r"(c[j % NS_PF][2]), "=r"(c[j % NS_PF][3])
                     : "r"(base + 16u * (j + NS_PF)));
      if (j < NCH / 2) {
        const int i = 4 * j;
        E[i] = j == 0 ? mac_cc(v0, x, E[i]) : macc_cc(v0, x, E[i]);
        E[i + 1] = macc_cc(v1, x, E[i + 1]);
        E[i + 2] = macc_cc(v2, x, E[i + 2]);
        E[i + 3] = macc_cc(v3, x, E[i + 3]);
        if (j == NCH / 2 - 1) E[H] = (uint64_t)addc32(lo32(E[H]), 0u);
      } else {
        const int i = 4 * (j - NCH / 2);
        O[i] = j == NCH / 2 ? mac_cc(v0, x, O[i]) : macc_cc(v0, x, O[i]);
        O[i + 1] = macc_cc(v1, x, O[i + 1]);
        O[i + 2] = macc_cc(v2, x, O[i + 2]);
        O[i + 3] = macc_cc(v3, x, O[i + 3]);
        if (j == NCH - 1) O[H] = (uint64_t)addc32(lo32(O[H]), 0u);
      }
    }
  }
  // E, O += n * x
  __device__ __forceinline__ void mac_row_n(uint64_t (&E)[H + 1], uint64_t (&O)[H + 1], uint32_t x) const {
    if constexpr (NS) mac_row_ns(E, O, x);
    else mac_row(E, O, n, x);
  }

  // E, O += v * x : one carry chain per accumulator array (H multiply-adds each)
  __device__ __forceinline__ void mac_row(uint64_t (&E)[H + 1], uint64_t (&O)[H + 1], const uint32_t (&v)[LPT],
                                          uint32_t x) const {
    // E[H] and O[H] only ever collect chain carries (a handful per row before the frame moves on), so they are
    // kept as 32-bit counts: one add instead of a 64-bit pair
    E[0] = mac_cc(v[0], x, E[0]);
#pragma unroll
    for (int i = 1; i < H; i++) E[i] = macc_cc(v[2 * i], x, E[i]);
    E[H] = (uint64_t)addc32(lo32(E[H]), 0u);
    O[0] = mac_cc(v[1], x, O[0]);
#pragma unroll
    for (int i = 1; i < H; i++) O[i] = macc_cc(v[2 * i + 1], x, O[i]);
    O[H] = (uint64_t)addc32(lo32(O[H]), 0u);
  }

  // Resolves pending single-bit carries between lanes: g (0/1) leaves this lane; returns the carry that
  // leaves the top lane (same value on every lane of the group).
  template <int NW>
  __device__ __forceinline__ uint32_t lane_carries_n(uint32_t (&r)[NW], uint32_t g, uint32_t cin0 = 0u) const {
    uint32_t all = r[0];
#pragma unroll
    for (int i = 1; i < NW; i++) all &= r[i];
    const uint32_t G = (__ballot_sync(FULLMASK, g != 0) >> gshift) & GM;
    const uint32_t P = (__ballot_sync(FULLMASK, all == 0xffffffffu) >> gshift) & GM;
    const uint64_t S = (uint64_t)P + ((uint64_t)G << 1) + cin0;   // cin0: carry into the lowest lane
    const uint32_t C = (uint32_t)S ^ P;              // bit t: carry entering lane t
    const uint32_t c = (C >> t) & 1u;
    r[0] = add_cc32(r[0], c);
#pragma unroll
    for (int i = 1; i < NW; i++) r[i] = addc_cc32(r[i], 0);
    return (uint32_t)(S >> TPI) & 1u;
  }
  __device__ __forceinline__ uint32_t lane_carries(uint32_t (&r)[LPT], uint32_t g, uint32_t cin0 = 0u) const {
    return lane_carries_n<LPT>(r, g, cin0);
  }

  // r = a + b + cin0 as L-limb integers (cin0 enters at the lowest limb); returns the carry out of the number
  __device__ __forceinline__ uint32_t add_raw(uint32_t (&r)[LPT], const uint32_t (&a)[LPT],
                                              const uint32_t (&b)[LPT], uint32_t cin0) const {
    r[0] = add_cc32(a[0], b[0]);
#pragma unroll
    for (int i = 1; i < LPT; i++) r[i] = addc_cc32(a[i], b[i]);
    const uint32_t g = addc32(0, 0);
    return lane_carries(r, g, cin0);
  }

  // r = a - b as L-limb integers (mod R); returns 1 when a >= b (no borrow)
  __device__ __forceinline__ uint32_t sub_raw(uint32_t (&r)[LPT], const uint32_t (&a)[LPT],
                                              const uint32_t (&b)[LPT]) const {
    uint32_t nb[LPT];
#pragma unroll
    for (int i = 0; i < LPT; i++) nb[i] = ~b[i];
    return add_raw(r, a, nb, 1u);
  }

  // r in [0, 2n) given as limbs plus an overflow bit  ->  [0, n)
  __device__ __forceinline__ void cond_sub(uint32_t (&r)[LPT], uint32_t hi) const {
    uint32_t d[LPT], nn[LPT];
    get_n(nn);
    const uint32_t ge = sub_raw(d, r, nn);
    if (hi | ge) {
#pragma unroll
      for (int i = 0; i < LPT; i++) r[i] = d[i];
    }
  }

  __device__ __forceinline__ void add_mod(uint32_t (&r)[LPT], const uint32_t (&a)[LPT], const uint32_t (&b)[LPT]) const {
    const uint32_t hi = add_raw(r, a, b, 0u);
    cond_sub(r, hi);
  }
  __device__ __forceinline__ void sub_mod(uint32_t (&r)[LPT], const uint32_t (&a)[LPT], const uint32_t (&b)[LPT]) const {
    uint32_t d[LPT], s[LPT], nn[LPT];
    const uint32_t ge = sub_raw(d, a, b);
    get_n(nn);
    add_raw(s, d, nn, 0u);              // unconditional: no warp collective inside a group-divergent branch
#pragma unroll
    for (int i = 0; i < LPT; i++) r[i] = ge ? d[i] : s[i];
  }
  // r = (R - r) mod R
  __device__ __forceinline__ void neg_R(uint32_t (&r)[LPT]) const {
    uint32_t z[LPT], s[LPT];
#pragma unroll
    for (int i = 0; i < LPT; i++) { z[i] = 0; s[i] = r[i]; }
    sub_raw(r, z, s);
  }
  __device__ __forceinline__ void set_one(uint32_t (&r)[LPT]) const {
#pragma unroll
    for (int i = 0; i < LPT; i++) r[i] = 0;
    r[0] = (t == 0) ? 1u : 0u;
  }
  __device__ __forceinline__ bool is_zero(const uint32_t (&r)[LPT]) const {
    uint32_t any = r[0];
#pragma unroll
    for (int i = 1; i < LPT; i++) any |= r[i];
    return ((__ballot_sync(FULLMASK, any != 0) >> gshift) & GM) == 0;
  }

  __device__ __forceinline__ void mul(uint32_t (&r)[LPT], const uint32_t (&a)[LPT], const uint32_t (&b)[LPT]) const {
    if constexpr (NS) {
      mul_sf(r, a, b, ns_sa);
    } else {
      uint32_t unused[LPT];
      mul_impl<false>(r, a, b, unused);
    }
  }
  // mul() that also returns the Montgomery quotient Q = -(a*b) * n^-1 mod R (lane t gets its LPT limbs).
  // When a*b is a multiple of n:  a*b / n = (R - Q) mod R.
  __device__ __forceinline__ void mul_quot(uint32_t (&r)[LPT], uint32_t (&qd)[LPT], const uint32_t (&a)[LPT],
                                           const uint32_t (&b)[LPT]) const {
    mul_impl<true>(r, a, b, qd);
  }

  template <bool COLLECT>
  __device__ __forceinline__ void mul_impl(uint32_t (&r)[LPT], const uint32_t (&a)[LPT], const uint32_t (&b)[LPT],
                                           uint32_t (&qd)[LPT]) const {
    uint64_t E[H + 1], O[H + 1];
#pragma unroll
    for (int i = 0; i <= H; i++) { E[i] = 0; O[i] = 0; }
    // what is left of an eliminated column (up to 33 bits) waits here for the next row instead of being
    // rippled through the accumulators
    uint32_t pend_lo = 0, pend_hi = 0;
#pragma unroll 1
    for (int s = 0; s < TPI; s++) {
#pragma unroll
      for (int i = 0; i < LPT; i++) {
        const uint32_t bj = __shfl_sync(FULLMASK, b[i], s, TPI);
        mac_row(E, O, a, bj);
        uint32_t q = (lo32(E[0]) + pend_lo) * np;
        q = __shfl_sync(FULLMASK, q, 0, TPI);
        if (COLLECT) { if (s == t) qd[i] = q; }
        mac_row_n(E, O, q);
        // column 0 = E[0] + pend: its low word is zero on lane 0 and goes to the lane below elsewhere
        const uint32_t vlo = add_cc32(lo32(E[0]), pend_lo);
        const uint32_t vhi = addc_cc32(hi32(E[0]), pend_hi);
        const uint32_t vtop = addc32(0, 0);
        // from the lane above; the top lane wraps to lane 0, whose low word has just been eliminated (it is zero)
        const uint32_t recv = __shfl_sync(FULLMASK, vlo, t + 1, TPI);
        pend_lo = vhi;
        pend_hi = vtop;
        // frame moves down one column: E <- O, O[k] <- E[k + 1], the received word lands on the top column
        uint64_t F[H + 1];
#pragma unroll
        for (int k = 0; k <= H; k++) F[k] = O[k];
#pragma unroll
        for (int k = 0; k < H - 1; k++) O[k] = E[k + 1];
        {                                     // E[H] is a small count: count + recv fits 33 bits
          const uint32_t lo = add_cc32(lo32(E[H]), recv);
          const uint32_t hi = addc32(0u, 0u);
          O[H - 1] = ((uint64_t)hi << 32) | lo;
          O[H] = 0;
        }
#pragma unroll
        for (int k = 0; k <= H; k++) E[k] = F[k];
      }
    }
    finish(r, E, O, pend_lo, pend_hi);
  }

  // lane value = pend + sum E[i] 2^(64 i) + sum O[i] 2^(64 i + 32)  ->  LPT + 3 words w[]
  __device__ __forceinline__ void frame_words(uint32_t (&w)[LPT + 3], uint64_t (&E)[H + 1], uint64_t (&O)[H + 1],
                                              uint32_t pend_lo, uint32_t pend_hi) const {
    // fold the pending column back in (once per multiplication)
    E[0] = add_cc64(E[0], ((uint64_t)pend_hi << 32) | pend_lo);
#pragma unroll
    for (int k = 1; k < H; k++) E[k] = addc_cc64(E[k], 0);
    E[H] = addc64(E[H], 0);
    w[0] = lo32(E[0]);
    w[1] = add_cc32(hi32(E[0]), lo32(O[0]));
#pragma unroll
    for (int i = 1; i <= H; i++) {
      w[2 * i] = addc_cc32(lo32(E[i]), hi32(O[i - 1]));
      w[2 * i + 1] = addc_cc32(hi32(E[i]), lo32(O[i]));
    }
    w[LPT + 2] = addc32(hi32(O[H]), 0);
  }

  // distributed frame after the last row  ->  canonical r in [0, n)
  __device__ __forceinline__ void finish(uint32_t (&r)[LPT], uint64_t (&E)[H + 1], uint64_t (&O)[H + 1],
                                         uint32_t pend_lo, uint32_t pend_hi) const {
    uint32_t w[LPT + 3];
    frame_words(w, E, O, pend_lo, pend_hi);
    // the three words above the lane's top column belong to the lane above
    uint32_t u0 = __shfl_up_sync(FULLMASK, w[LPT], 1, TPI);
    uint32_t u1 = __shfl_up_sync(FULLMASK, w[LPT + 1], 1, TPI);
    uint32_t u2 = __shfl_up_sync(FULLMASK, w[LPT + 2], 1, TPI);
    if (t == 0) { u0 = 0; u1 = 0; u2 = 0; }
    r[0] = add_cc32(w[0], u0);
    r[1] = addc_cc32(w[1], u1);
    r[2] = addc_cc32(w[2], u2);
#pragma unroll
    for (int i = 3; i < LPT; i++) r[i] = addc_cc32(w[i], 0);
    const uint32_t g = addc32(0, 0);
    uint32_t hi = lane_carries(r, g);
    // top lane: its own overflow word (value < 2n < 2R, so at most one bit)
    const uint32_t topw = __shfl_sync(FULLMASK, w[LPT], TPI - 1, TPI);
    hi |= topw;
    cond_sub(r, hi);
  }

  // ---- shared-memory staged multiplication and dedicated squaring (TPI == 4) ---------------------------------
  //
  // tools/mont32_sqr_model.py is the executable description of sqr().  Both routines keep their code small enough
  // for the instruction cache by reading the row multipliers from shared memory instead of register-indexed
  // shuffles, which lets the row loops run at an unroll of RU instead of LPT.
  //
  // a^2 = sum_t a_t^2 B^(2 LPT t) + 2 sum_{i<j} a_i a_j B^(LPT (i+j)).  Every lane multiplies lane-locally
  // (operand scanning in its own E/O frame, one column retiring per row): first its own square, then 1.5 LPT
  // rows of the off-diagonal part -- the schedule that splits the six blocks evenly over the four lanes:
  //     lane 0: a_0 x limbs [LPT, 2.5 LPT)      lane 3: a_0 x limbs [2.5 LPT, 4 LPT)
  //     lane 1: a_3 x limbs [LPT, 2.5 LPT)      lane 2: a_2 x limbs [LPT, 2 LPT), then a_3 x limbs [2.5 LPT, 3 LPT)
  // The pieces meet in shared memory (word w of an instance at sw[w * IPW]); lane t sums the columns
  // [2 LPT t, 2 LPT (t+1)), doubles, adds its square, the lanes settle their carries, and the 2L-word square is
  // Montgomery-reduced in the distributed frame of mul(), its high half entering one word per row at the top
  // lane.  Limb products per lane: 2.5 LPT^2 + 4 LPT^2 against 8 LPT^2 in mul().
  static constexpr bool HAS_SQR = (TPI == 4) && (LPT % 8 == 0);
  static constexpr int IPW = 32 / TPI;
  static constexpr int RU = (H % 8 == 0) ? 8 : 4;                  // rows per unrolled chunk (divides H)
  static constexpr int SQ_P0 = 0, SQ_P3 = 5 * H + 1, SQ_P1 = 10 * H + 2, SQ_P2A = 15 * H + 3, SQ_P2B = 19 * H + 3;
  static constexpr int SQ_T = 22 * H + 4;                          // 2L words: own squares, then the square
  static constexpr int SQ_A = SQ_T + 16 * H;                       // staged operand: limb j at SQ_A + j + j / LPT
  static constexpr int SQ_WORDS = HAS_SQR ? SQ_A + L + TPI : 0;    // shared-memory words per instance

  __device__ __forceinline__ void stage(const uint32_t (&x)[LPT], uint32_t* sw) const {
    uint32_t* d = sw + (SQ_A + (LPT + 1) * t) * IPW;
#pragma unroll
    for (int k = 0; k < LPT; k++) d[k * IPW] = x[k];
  }

  // the frame moves down one column; `recv` lands on the top column
  __device__ __forceinline__ void frame_down(uint64_t (&E)[H + 1], uint64_t (&O)[H + 1], uint32_t recv) const {
    uint64_t F[H + 1];
#pragma unroll
    for (int k = 0; k <= H; k++) F[k] = O[k];
#pragma unroll
    for (int k = 0; k < H - 1; k++) O[k] = E[k + 1];
    const uint32_t lo = add_cc32(lo32(E[H]), recv);        // E[H] is a small count: count + recv fits 33 bits
    const uint32_t hi = addc32(0u, 0u);
    O[H - 1] = ((uint64_t)hi << 32) | lo;
    O[H] = 0;
#pragma unroll
    for (int k = 0; k <= H; k++) E[k] = F[k];
  }

  // mul() with b read from shared memory: same arithmetic, row loop unrolled RU times
  __device__ __forceinline__ void mul_s(uint32_t (&r)[LPT], const uint32_t (&a)[LPT], const uint32_t (&b)[LPT],
                                        uint32_t* sw) const {
    uint64_t E[H + 1], O[H + 1];
#pragma unroll
    for (int i = 0; i <= H; i++) { E[i] = 0; O[i] = 0; }
    uint32_t pend_lo = 0, pend_hi = 0;
    __syncwarp();
    stage(b, sw);
    __syncwarp();
#pragma unroll 1
    for (int j0 = 0; j0 < L; j0 += RU) {
      const uint32_t* bs = sw + (SQ_A + j0 + j0 / LPT) * IPW;
#pragma unroll
      for (int u = 0; u < RU; u++) {
        mac_row(E, O, a, bs[u * IPW]);
        uint32_t q = (lo32(E[0]) + pend_lo) * np;
        q = __shfl_sync(FULLMASK, q, 0, TPI);
        mac_row_n(E, O, q);
        const uint32_t vlo = add_cc32(lo32(E[0]), pend_lo);
        const uint32_t vhi = addc_cc32(hi32(E[0]), pend_hi);
        const uint32_t vtop = addc32(0, 0);
        const uint32_t recv = __shfl_sync(FULLMASK, vlo, t + 1, TPI);    // top lane wraps to lane 0: zero
        pend_lo = vhi;
        pend_hi = vtop;
        frame_down(E, O, recv);
      }
    }
    finish(r, E, O, pend_lo, pend_hi);
  }

  // mul() with b read from shared memory and the rows of one lane block fully unrolled (no frame-rotation moves):
  // the form for LPT = 48, where a register copy of b would not fit next to the accumulators, a and n.
  // `sa`: this instance's staging area alone, STAGE_WORDS words at stride IPW.
  __device__ __forceinline__ void mul_sf(uint32_t (&r)[LPT], const uint32_t (&a)[LPT], const uint32_t (&b)[LPT],
                                         uint32_t* sa) const {
    uint64_t E[H + 1], O[H + 1];
#pragma unroll
    for (int i = 0; i <= H; i++) { E[i] = 0; O[i] = 0; }
    uint32_t pend_lo = 0, pend_hi = 0;
    __syncwarp();
    {
      uint32_t* d = sa + ((LPT + 1) * t) * IPW;
#pragma unroll
      for (int k = 0; k < LPT; k++) d[k * IPW] = b[k];
    }
    __syncwarp();
#pragma unroll 1
    for (int s = 0; s < TPI; s++) {
      const uint32_t* bs = sa + ((LPT + 1) * s) * IPW;
#pragma unroll
      for (int i = 0; i < LPT; i++) {
        mac_row(E, O, a, bs[i * IPW]);
        uint32_t q = (lo32(E[0]) + pend_lo) * np;
        q = __shfl_sync(FULLMASK, q, 0, TPI);
        mac_row_n(E, O, q);
        const uint32_t vlo = add_cc32(lo32(E[0]), pend_lo);
        const uint32_t vhi = addc_cc32(hi32(E[0]), pend_hi);
        const uint32_t vtop = addc32(0, 0);
        const uint32_t recv = __shfl_sync(FULLMASK, vlo, t + 1, TPI);    // top lane wraps to lane 0: zero
        pend_lo = vhi;
        pend_hi = vtop;
        frame_down(E, O, recv);
      }
    }
    finish(r, E, O, pend_lo, pend_hi);
  }

  // r = a * a / R mod n, canonical.  sw: this instance's shared-memory scratch (SQ_WORDS words, stride IPW).
  __device__ __forceinline__ void sqr(uint32_t (&r)[LPT], const uint32_t (&a)[LPT], uint32_t* sw) const {
    constexpr int W = 2 * LPT;
    uint64_t E[H + 1], O[H + 1];
#pragma unroll
    for (int i = 0; i <= H; i++) { E[i] = 0; O[i] = 0; }
    uint32_t pend_lo = 0, pend_hi = 0;
    uint32_t v[LPT];
    __syncwarp();
    stage(a, sw);
    __syncwarp();
    // ---- lane-local products: LPT rows of the own square, LPT rows of phase alpha, LPT / 2 of phase beta
    const int pa = t == 0 ? SQ_P0 : t == 1 ? SQ_P1 : t == 2 ? SQ_P2A : SQ_P3;
#pragma unroll 1
    for (int row0 = 0; row0 < 5 * H; row0 += RU) {
      const int phase = row0 < LPT ? 0 : row0 < 2 * LPT ? 1 : 2;
      const int pr = row0 - phase * LPT;                          // row inside the phase
      int vsrc, x0, d0;
      if (phase == 0) {
        vsrc = t; x0 = LPT * t; d0 = SQ_T + W * t;
      } else if (phase == 1) {
        vsrc = t == 1 ? 3 : t == 2 ? 2 : 0; x0 = t == 3 ? 5 * H : LPT; d0 = pa;
      } else {
        vsrc = (t == 1 || t == 2) ? 3 : 0; x0 = t == 3 ? 7 * H : t == 2 ? 5 * H : 2 * LPT;
        d0 = t == 2 ? SQ_P2B : pa + LPT;
      }
      if (pr == 0) {
        const uint32_t* vs = sw + (SQ_A + (LPT + 1) * vsrc) * IPW;
#pragma unroll
        for (int k = 0; k < LPT; k++) v[k] = vs[k * IPW];
      }
      const int j0 = x0 + pr;
      const uint32_t* xs = sw + (SQ_A + j0 + j0 / LPT) * IPW;
      uint32_t* dst = sw + (d0 + pr) * IPW;
#pragma unroll
      for (int u = 0; u < RU; u++) {
        mac_row(E, O, v, xs[u * IPW]);
        const uint32_t vlo = add_cc32(lo32(E[0]), pend_lo);
        const uint32_t vhi = addc_cc32(hi32(E[0]), pend_hi);
        const uint32_t vtop = addc32(0, 0);
        dst[u * IPW] = vlo;
        pend_lo = vhi;
        pend_hi = vtop;
        frame_down(E, O, 0u);
      }
      const int plen = phase == 2 ? H : LPT;
      if (pr + RU == plen && (phase != 1 || t == 2)) {            // the piece ends here: park the rest of the frame
        uint32_t w[LPT + 3];
        frame_words(w, E, O, pend_lo, pend_hi);
#pragma unroll
        for (int k = 0; k < LPT; k++) dst[(RU + k) * IPW] = w[k];
#pragma unroll
        for (int i = 0; i <= H; i++) { E[i] = 0; O[i] = 0; }
        pend_lo = 0;
        pend_hi = 0;
      }
    }
    __syncwarp();
    // ---- column sums: lane t owns the columns [W t, W (t + 1))
    {
      uint32_t acc[W];
#pragma unroll
      for (int k = 0; k < W; k++) acc[k] = 0;
      uint32_t topc = 0;
#pragma unroll 1
      for (int p = 0; p < 5; p++) {
        const int pb = p == 0 ? SQ_P0 : p == 1 ? SQ_P3 : p == 2 ? SQ_P1 : p == 3 ? SQ_P2A : SQ_P2B;
        const int off = p == 0 ? 2 * H : p == 1 ? 5 * H : p == 2 ? 8 * H : p == 3 ? 6 * H : 11 * H;
        const int len = p == 3 ? 4 * H : p == 4 ? 3 * H : 5 * H;
        const int base = W * t - off;
        if (base + W <= 0 || base >= len) continue;               // no overlap with this lane's columns
        const uint32_t* ps = sw + (pb + base) * IPW;
        uint32_t w[W];
#pragma unroll
        for (int k = 0; k < W; k++) w[k] = ((unsigned)(base + k) < (unsigned)len) ? ps[k * IPW] : 0u;
        acc[0] = add_cc32(acc[0], w[0]);
#pragma unroll
        for (int k = 1; k < W; k++) acc[k] = addc_cc32(acc[k], w[k]);
        topc = addc32(topc, 0);
      }
      // the off-diagonal part counts twice
      topc = 2 * topc + (acc[W - 1] >> 31);
#pragma unroll
      for (int k = W - 1; k > 0; k--) acc[k] = __funnelshift_l(acc[k - 1], acc[k], 1);
      acc[0] <<= 1;
      uint32_t* tt = sw + (SQ_T + W * t) * IPW;
      {
        uint32_t w[W];
#pragma unroll
        for (int k = 0; k < W; k++) w[k] = tt[k * IPW];
        acc[0] = add_cc32(acc[0], w[0]);
#pragma unroll
        for (int k = 1; k < W; k++) acc[k] = addc_cc32(acc[k], w[k]);
        topc = addc32(topc, 0);
      }
      uint32_t in = __shfl_up_sync(FULLMASK, topc, 1, TPI);
      if (t == 0) in = 0;
      acc[0] = add_cc32(acc[0], in);
#pragma unroll
      for (int k = 1; k < W; k++) acc[k] = addc_cc32(acc[k], 0);
      const uint32_t g = addc32(0, 0);
      lane_carries_n<W>(acc, g);
#pragma unroll
      for (int k = 0; k < W; k++) tt[k * IPW] = acc[k];
    }
    __syncwarp();
    // ---- Montgomery reduction of the 2L-word square
    {
      const uint32_t* tl = sw + (SQ_T + LPT * t) * IPW;
#pragma unroll
      for (int i = 0; i < H; i++) {
        E[i] = (uint64_t)tl[(2 * i) * IPW] | ((uint64_t)tl[(2 * i + 1) * IPW] << 32);
        O[i] = 0;
      }
      E[H] = 0;
      O[H] = 0;
      pend_lo = 0;
      pend_hi = 0;
    }
#pragma unroll 1
    for (int row = 0; row < L; row += RU) {
      const uint32_t* th = sw + (SQ_T + L + row) * IPW;
#pragma unroll
      for (int u = 0; u < RU; u++) {
        uint32_t q = (lo32(E[0]) + pend_lo) * np;
        q = __shfl_sync(FULLMASK, q, 0, TPI);
        mac_row_n(E, O, q);
        const uint32_t vlo = add_cc32(lo32(E[0]), pend_lo);
        const uint32_t vhi = addc_cc32(hi32(E[0]), pend_hi);
        const uint32_t vtop = addc32(0, 0);
        uint32_t recv = __shfl_down_sync(FULLMASK, vlo, 1, TPI);
        if (top) recv = th[u * IPW];
        pend_lo = vhi;
        pend_hi = vtop;
        frame_down(E, O, recv);
      }
    }
    finish(r, E, O, pend_lo, pend_hi);
  }

  // limbs [t*LPT, (t+1)*LPT) of the little-endian word array w[0..nwords) (zero beyond it).
  // Element arrays are read and written 16 bytes at a time whenever the word count allows it (every key size that is
  // a multiple of 64 bits): a lane's limbs are contiguous, so one LDG.128 replaces four LDG.32 that would each touch
  // a different sector per lane -- k_mulmod was bound by those L1 wavefronts, not by the multiplier.  Taken when the
  // element base is 16-byte aligned (device allocations are; word counts that are multiples of 4 keep
  // every element aligned; anything else takes the word-by-word path).
  __device__ __forceinline__ void load_words(uint32_t (&r)[LPT], const uint32_t* __restrict__ w, int nwords) const {
    if constexpr (LPT % 4 == 0) {
      if ((nwords & 3) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < LPT / 4; j++) {
          const int k = t * LPT + 4 * j;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (k < nwords) v = *reinterpret_cast<const uint4*>(w + k);
          r[4 * j] = v.x; r[4 * j + 1] = v.y; r[4 * j + 2] = v.z; r[4 * j + 3] = v.w;
        }
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      const int k = t * LPT + i;
      r[i] = k < nwords ? w[k] : 0u;
    }
  }
  __device__ __forceinline__ void store_words(uint32_t* __restrict__ w, int nwords, const uint32_t (&r)[LPT],
                                              bool valid = true) const {
    if constexpr (LPT % 4 == 0) {
      if ((nwords & 3) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < LPT / 4; j++) {
          const int k = t * LPT + 4 * j;
          if (valid && k < nwords)
            *reinterpret_cast<uint4*>(w + k) = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        }
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < LPT; i++) {
      const int k = t * LPT + i;
      if (valid && k < nwords) w[k] = r[i];
    }
  }
  // full L-limb arrays (constants, scratch, Montgomery digit form): always 16-byte accesses
  __device__ __forceinline__ void load_limbs(uint32_t (&r)[LPT], const uint32_t* __restrict__ d) const {
    if constexpr (LPT % 4 == 0) {
      const uint4* p = reinterpret_cast<const uint4*>(d + t * LPT);
#pragma unroll
      for (int j = 0; j < LPT / 4; j++) {
        const uint4 v = p[j];
        r[4 * j] = v.x; r[4 * j + 1] = v.y; r[4 * j + 2] = v.z; r[4 * j + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < LPT; i++) r[i] = d[t * LPT + i];
    }
  }
  __device__ __forceinline__ void store_limbs(uint32_t* __restrict__ d, const uint32_t (&r)[LPT]) const {
    if constexpr (LPT % 4 == 0) {
      uint4* p = reinterpret_cast<uint4*>(d + t * LPT);
#pragma unroll
      for (int j = 0; j < LPT / 4; j++) p[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < LPT; i++) d[t * LPT + i] = r[i];
    }
  }
};

}  // namespace hb
