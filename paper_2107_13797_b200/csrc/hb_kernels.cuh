// Batched Paillier kernels for sm_100a built on the warp-cooperative Montgomery core (mont.cuh).
//
// One instance (one ciphertext / plaintext element) is owned by a group of TPI lanes; a warp holds
// 32/TPI instances ("a tile") and a grid-stride loop walks the tiles.  All instances of a launch
// share the modulus and, for encrypt / obfuscate / decrypt, the exponent, so control flow is uniform
// across the grid: the exponent is compiled on the host into a flat op program (sliding window over
// odd powers) that every warp replays.  Window tables live in a per-warp scratch tile in global memory
// laid out [entry][digit][lane] so each access is one coalesced 128-byte row.
//
// Reference semantics (file:line under /root/reference/pkg/src/hebatch):
//   k_encrypt   operators.py:39-46   (1 + m n) r^n mod n^2   |   c r^n mod n^2
//   k_decrypt   operators.py:49-56   CRT decryption
//   k_mulmod    operators.py:70-72   a b mod n^2 (optionally b = 1 + m n, operators.py:211)
#pragma once
#include "hb_ctx.h"

namespace hb {

// op word of the exponent program: kind | src << 8 | dst << 16
enum : uint32_t { OP_SQR = 0, OP_MUL = 1, OP_LOAD = 2, OP_KEEP = 3, OP_NODST = 0xFF };

// Replays an op program on x (Montgomery form in, Montgomery form out).  Single mul call site.
// Squarings and multiplications both go through Mont::mul by default: on the B200 the dedicated squaring
// (Mont::sqr, 19 % fewer limb products) loses to it -- 89 k against 104 k encryptions/s at 2048 bits -- because
// its extra non-multiply instructions are not free next to a quarter-rate IMAD.WIDE.  Build
// with -DHB_USE_SQR to route OP_SQR through Mont::sqr and OP_MUL through Mont::mul_s; `sw` is then the instance's
// shared-memory scratch (sqr_scratch()).
template <int LPT, int TPI>
__device__ __forceinline__ void run_prog(const Mont<LPT, TPI>& mt, uint32_t (&x)[LPT],
                                         const uint32_t* __restrict__ prog, int nprog, uint32_t* tw, uint32_t* sw) {
#pragma unroll 1
  for (int i = 0; i < nprog; i++) {
    uint32_t op = prog[i];
    uint32_t kind = op & 0xFF, src = (op >> 8) & 0xFF, dst = (op >> 16) & 0xFF;
    if (kind == OP_LOAD) {
      tile_load<LPT>(tw, src, x);
    } else if (kind != OP_KEEP) {
      if constexpr (enc_stages_operand(LPT)) {  // wide-lane shape: b comes from shared memory (Mont::mul_sf)
        uint32_t y[LPT];
        if (kind == OP_MUL) {
          tile_load<LPT>(tw, src, y);
        } else {
#pragma unroll
          for (int k = 0; k < LPT; k++) y[k] = x[k];
        }
        mt.mul_sf(x, x, y, sw);
      } else
#ifdef HB_USE_SQR
      if constexpr (Mont<LPT, TPI>::HAS_SQR) {
        if (kind == OP_MUL) {
          uint32_t y[LPT];
          tile_load<LPT>(tw, src, y);
          mt.mul_s(x, x, y, sw);
        } else {
          mt.sqr(x, x, sw);
        }
      } else
#endif
      {
        uint32_t y[LPT];
        if (kind == OP_MUL) {
          tile_load<LPT>(tw, src, y);
        } else {
#pragma unroll
          for (int k = 0; k < LPT; k++) y[k] = x[k];
        }
        mt.mul(x, x, y);
      }
    }
    if (dst != OP_NODST) tile_store<LPT>(tw, dst, x);
  }
}

extern __shared__ __align__(16) uint32_t hb_dyn_smem[];
// Shared-memory scratch of this lane's instance for Mont::sqr (nullptr when the shape has no dedicated squaring).
template <int LPT, int TPI>
__device__ __forceinline__ uint32_t* sqr_scratch() {
  using M = Mont<LPT, TPI>;
  if constexpr (enc_stages_operand(LPT)) {
    return hb_dyn_smem + threadIdx.x / TPI;        // staging area only (Mont::mul_sf), one warp per block
  } else if constexpr (M::HAS_SQR) {
    return hb_dyn_smem + threadIdx.x / TPI;        // one warp per block
  } else {
    return nullptr;
  }
}

// Representation of a ciphertext array crossing a kernel boundary (include/hebatch_b200.h, HB_REP_*): plain
// little-endian words (wc per element, the HAFB payload) or Montgomery digit form x * R mod n^2 (L limbs per
// element), the form chained operators keep on the device.  Multiplying a Montgomery operand by a plain one yields
// a plain product, two Montgomery operands a Montgomery product: an operator whose inputs are resident costs no
// conversion.
template <int LPT, int TPI>
__device__ __forceinline__ void load_ct(const Mont<LPT, TPI>& mt, uint32_t (&x)[LPT], const uint32_t* base, long i,
                                        int wc, int mont) {
  if (mont) mt.load_limbs(x, base + i * (LPT * TPI));
  else mt.load_words(x, base + i * wc, wc);
}
template <int LPT, int TPI>
__device__ __forceinline__ void store_ct(const Mont<LPT, TPI>& mt, uint32_t* base, long i, int wc, int mont,
                                         const uint32_t (&x)[LPT], bool valid) {
  if (mont) { if (valid) mt.store_limbs(base + i * (LPT * TPI), x); }
  else mt.store_words(base + i * wc, wc, x, valid);
}

struct EncArgs {
  ModDev mod;                // n^2
  const uint32_t* nR;        // n * R mod n^2 : mul(m, nR) = m*n            (n * R^2 when out_mont: m*n*R)
  int c_mont, out_mont;      // representation of c (mode 1) and of the result
  const uint32_t* prog;      // exponent n
  int nprog;
  uint32_t* tbl;             // per-warp scratch tiles
  long tbl_stride;           // words per warp
  const uint32_t* m;         // mode 0: plaintext residues (wn words each)
  const uint32_t* c;         // mode 1: ciphertexts to re-randomise (wc words each)
  const uint32_t* r;         // obfuscation factors (wn words each)
  uint32_t* out;             // wc words each
  long count;
  int wn, wc;
  int mode;
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * enc_blocks_per_sm(LPT)) k_encrypt(EncArgs A) {
  using M = Mont<LPT, TPI>;
  constexpr int IPW = 32 / TPI;
  M mt;
  mt.init(A.mod.n, A.mod.np, hb_dyn_smem);
  // one warp per block: the tile loop then depends on blockIdx only, the compiler can see that the warp never
  // diverges, and every __shfl_sync becomes a bare SHFL instead of a WARPSYNC.COLLECTIVE / ENDCOLLECTIVE bracket
  const int lane = threadIdx.x, g = lane / TPI;
  const long wg = blockIdx.x, nw = gridDim.x;
  uint32_t* tw = A.tbl + wg * A.tbl_stride;
  uint32_t* sw = sqr_scratch<LPT, TPI>();
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_words(x, A.r + ii * A.wn, A.wn);
    mt.load_limbs(y, A.mod.r2);
    mt.mul(x, x, y);                              // Mont(r)
    run_prog<LPT, TPI>(mt, x, A.prog, A.nprog, tw, sw);  // Mont(r^n)
    if (A.mode == 0) {
      uint32_t z[LPT];
      mt.load_words(y, A.m + ii * A.wn, A.wn);
      mt.load_limbs(z, A.nR);
      mt.mul(y, y, z);                            // m*n, in the representation the result is wanted in
      if (A.out_mont) mt.load_limbs(z, A.mod.r1); else mt.set_one(z);
      mt.add_mod(y, y, z);                        // 1 + m*n  (< n^2, nothing is reduced)
    } else {
      load_ct<LPT, TPI>(mt, y, A.c, ii, A.wc, A.c_mont);
      if (A.c_mont != A.out_mont) {               // one conversion so that Mont(r^n) * y lands in the wanted form
        uint32_t z[LPT];
        if (A.out_mont) mt.load_limbs(z, A.mod.r2); else mt.set_one(z);
        mt.mul(y, y, z);
      }
    }
    mt.mul(x, x, y);                              // canonical
    store_ct<LPT, TPI>(mt, A.out, ii, A.wc, A.out_mont, x, valid);
  }
}

// Fused fore-gradient chain of one heterogeneous-FLR mini-batch (reference arena.py:345-366, the cached pipeline
// plain_mul -> encrypt -> hmul -> hadd -> plain_mul -> hadd(lifted plaintext)), one pass per element:
//     out = (1 + (lg * kg mod n) n) r^n  *  c^kh  *  (1 + yl n)      mod n^2
// lg: the guest's logits (plaintext residues), kg: the plaintext factor (encode(0.25) -> 4) as a residue, c: the
// host's encrypted logits, kh: the same factor as a small positive exponent, yl: the label term already multiplied
// and re-gridded on the plaintext side (hb_plain_mulmod, hb_plain_rescale -- which also own the overflow checks).
// Every factor is an exact residue, so the bits equal the reference's six-operator sequence.  n (x mod n) = n x mod
// n^2, hence lg * kg needs no reduction mod n of its own: one multiplication by kg n R^2.
struct ForeArgs {
  ModDev mod;                // n^2
  const uint32_t* nR2;       // n * R^2 mod n^2
  const uint32_t* prog;      // exponent n
  int nprog;
  uint32_t* tbl;             // per-warp scratch tiles; slots `spare` and `spare + 1` are this kernel's
  long tbl_stride;
  int spare;
  const uint32_t* lg;        // wn words each
  const uint32_t* kg;        // wn words (one residue)
  const uint32_t* c;         // ciphertexts
  const uint32_t* yl;        // wn words each
  const uint32_t* r;         // obfuscation factors, wn words each
  uint32_t* out;
  uint32_t kh;               // exponent for c, >= 1
  long count;
  int wn, wc;
  int c_mont, out_mont;
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_fore_gradient(ForeArgs A) {
  using M = Mont<LPT, TPI>;
  constexpr int IPW = 32 / TPI;
  M mt;
  mt.init(A.mod.n, A.mod.np, hb_dyn_smem);
  const int lane = threadIdx.x, g = lane / TPI;
  const long wg = blockIdx.x, nw = gridDim.x;
  uint32_t* tw = A.tbl + wg * A.tbl_stride;
  uint32_t* sw = sqr_scratch<LPT, TPI>();
  {
    uint32_t x[LPT], y[LPT];
    mt.load_words(x, A.kg, A.wn);
    mt.load_limbs(y, A.nR2);
    mt.mul(x, x, y);                              // kg n R
    mt.load_limbs(y, A.mod.r2);
    mt.mul(x, x, y);                              // kg n R^2 : mul(lg, .) = Mont(lg kg n)
    tile_store<LPT>(tw, A.spare, x);
  }
  const int htop = 31 - __clz(A.kh | 1u);
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    uint32_t x[LPT], y[LPT];
    // c^kh, left to right (kh is a launch constant: uniform control flow)
    load_ct<LPT, TPI>(mt, y, A.c, ii, A.wc, A.c_mont);
    if (!A.c_mont) {
      mt.load_limbs(x, A.mod.r2);
      mt.mul(y, y, x);
    }
#pragma unroll
    for (int k = 0; k < LPT; k++) x[k] = y[k];
#pragma unroll 1
    for (int b = htop - 1; b >= 0; b--) {
      uint32_t z[LPT];
#pragma unroll
      for (int k = 0; k < LPT; k++) z[k] = x[k];
      mt.mul(x, x, z);
      if ((A.kh >> b) & 1u) mt.mul(x, x, y);
    }
    tile_store<LPT>(tw, A.spare + 1, x);
    mt.load_words(x, A.r + ii * A.wn, A.wn);
    mt.load_limbs(y, A.mod.r2);
    mt.mul(x, x, y);                              // Mont(r)
    run_prog<LPT, TPI>(mt, x, A.prog, A.nprog, tw, sw);  // Mont(r^n)
    {
      uint32_t z[LPT];
      mt.load_words(y, A.lg + ii * A.wn, A.wn);
      tile_load<LPT>(tw, A.spare, z);
      mt.mul(y, y, z);
      mt.load_limbs(z, A.mod.r1);
      mt.add_mod(y, y, z);                        // Mont(1 + (lg kg mod n) n)
    }
    mt.mul(x, x, y);                              // Mont(encrypted guest term)
    tile_load<LPT>(tw, A.spare + 1, y);
    mt.mul(x, x, y);                              // * c^kh
    {
      uint32_t z[LPT];
      mt.load_words(y, A.yl + ii * A.wn, A.wn);
      mt.load_limbs(z, A.nR2);
      mt.mul(y, y, z);
      mt.load_limbs(z, A.mod.r1);
      mt.add_mod(y, y, z);                        // Mont(1 + yl n)
    }
    mt.mul(x, x, y);
    if (!A.out_mont) {
      mt.set_one(y);
      mt.mul(x, x, y);
    }
    store_ct<LPT, TPI>(mt, A.out, ii, A.wc, A.out_mont, x, valid);
  }
}

struct MulArgs {
  ModDev mod;
  const uint32_t* nR;     // n * R mod n^2
  const uint32_t* nR2;    // n * R^2 mod n^2
  const uint32_t* r3;     // R^3 mod n^2
  const uint32_t* a;
  const uint32_t* b;      // ciphertexts (lift == 0) or plaintext residues (lift == 1)
  uint32_t* out;
  long count;
  int wn, wc;
  int lift;
  int b_broadcast;
  int a_mont, b_mont, out_mont;
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_mulmod(MulArgs A) {
  using M = Mont<LPT, TPI>;
  constexpr int IPW = 32 / TPI;
  M mt;
  mt.init(A.mod.n, A.mod.np);
  // one warp per block: the tile loop then depends on blockIdx only, the compiler can see that the warp never
  // diverges, and every __shfl_sync becomes a bare SHFL instead of a WARPSYNC.COLLECTIVE / ENDCOLLECTIVE bracket
  const int lane = threadIdx.x, g = lane / TPI;
  const long wg = blockIdx.x, nw = gridDim.x;
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    long ib = A.b_broadcast ? 0 : ii;
    uint32_t x[LPT], y[LPT];
    // power of R carried by a * b / R:  rep(a) + rep(b) - 1  with Montgomery = 1, plain = 0
    int rb = A.b_mont;
    if (A.lift) {
      // 1 + m n costs the same in either form: take the one that makes the product land where it is wanted
      rb = (A.a_mont == A.out_mont) ? 1 : 0;
      if (!A.a_mont && A.out_mont) rb = 1;
      mt.load_words(x, A.b + ib * A.wn, A.wn);
      mt.load_limbs(y, rb ? A.nR2 : A.nR);
      mt.mul(y, x, y);                            // m*n
      if (rb) mt.load_limbs(x, A.mod.r1); else mt.set_one(x);
      mt.add_mod(y, y, x);                        // 1 + m*n
    } else {
      load_ct<LPT, TPI>(mt, y, A.b, ib, A.wc, A.b_mont);
    }
    load_ct<LPT, TPI>(mt, x, A.a, ii, A.wc, A.a_mont);
    mt.mul(x, x, y);
    const int got = A.a_mont + rb - 1;            // -1, 0 or 1
    if (got != A.out_mont) {                      // one multiplication by R^(out - got + 1)
      const int e = A.out_mont - got + 1;         // 0, 2 or 3
      if (e == 0) mt.set_one(y);
      else mt.load_limbs(y, e == 2 ? A.mod.r2 : A.r3);
      mt.mul(x, x, y);
    }
    store_ct<LPT, TPI>(mt, A.out, ii, A.wc, A.out_mont, x, valid);
  }
}

struct PlainArgs {
  ModDev mod;             // modulus n
  const uint32_t* a;
  const uint32_t* b;
  uint32_t* out;
  long count;
  int w;                  // words per residue
  int op;                 // 0: a * b mod n   1: a + b mod n
  int b_broadcast;
};

// Plaintext-side residue arithmetic mod n (batches.py:173-205 of the reference: plain_mul, plain_add).
template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_plainop(PlainArgs A) {
  using M = Mont<LPT, TPI>;
  constexpr int IPW = 32 / TPI;
  M mt;
  mt.init(A.mod.n, A.mod.np);
  // one warp per block: the tile loop then depends on blockIdx only, the compiler can see that the warp never
  // diverges, and every __shfl_sync becomes a bare SHFL instead of a WARPSYNC.COLLECTIVE / ENDCOLLECTIVE bracket
  const int lane = threadIdx.x, g = lane / TPI;
  const long wg = blockIdx.x, nw = gridDim.x;
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    long ib = A.b_broadcast ? 0 : ii;
    uint32_t x[LPT], y[LPT];
    mt.load_words(y, A.b + ib * A.w, A.w);
    mt.load_words(x, A.a + ii * A.w, A.w);
    if (A.op == 0) {
      uint32_t z[LPT];
      mt.load_limbs(z, A.mod.r2);
      mt.mul(y, y, z);                              // Mont(b)
      mt.mul(x, x, y);                              // a * b mod n, canonical
    } else {
      mt.add_mod(x, x, y);
    }
    mt.store_words(A.out + ii * A.w, A.w, x, valid);
  }
}

struct SqrArgs {
  ModDev mod;
  const uint32_t* a;
  uint32_t* out;
  long count;
  int wc;
  int reps;               // out = a^(2^reps)
};

// out[i] = a[i]^(2^reps) mod n^2 through the squaring path of the shape (Mont::sqr where there is one).
template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_sqrmod(SqrArgs A) {
  using M = Mont<LPT, TPI>;
  constexpr int IPW = 32 / TPI;
  M mt;
  mt.init(A.mod.n, A.mod.np);
  // one warp per block: the tile loop then depends on blockIdx only, the compiler can see that the warp never
  // diverges, and every __shfl_sync becomes a bare SHFL instead of a WARPSYNC.COLLECTIVE / ENDCOLLECTIVE bracket
  const int lane = threadIdx.x, g = lane / TPI;
  const long wg = blockIdx.x, nw = gridDim.x;
  uint32_t* sw = sqr_scratch<LPT, TPI>();
  const long ntiles = (A.count + IPW - 1) / IPW;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    uint32_t x[LPT], y[LPT];
    mt.load_words(x, A.a + ii * A.wc, A.wc);
    mt.load_limbs(y, A.mod.r2);
    mt.mul(x, x, y);
#pragma unroll 1
    for (int k = 0; k < A.reps; k++) {
      if constexpr (M::HAS_SQR) {
        mt.sqr(x, x, sw);
      } else {
#pragma unroll
        for (int i = 0; i < LPT; i++) y[i] = x[i];
        mt.mul(x, x, y);
      }
    }
    mt.set_one(y);
    mt.mul(x, x, y);
    mt.store_words(A.out + ii * A.wc, A.wc, x, valid);
  }
}

struct HalfDev {
  ModDev s2;                 // modulus s^2
  ModDev s1;                 // modulus s, zero-padded to the same digit count
  const uint32_t* hiR2;      // 2^H * R^2 mod s^2 : Montgomery form of the high half of c
  const uint32_t* hsR;       // hs * R mod s      : mul(t, hsR) = t*hs mod s
  const uint32_t* prog;      // exponent s - 1
  int nprog;
};

struct DecArgs {
  HalfDev half[2];           // [0] = p, [1] = q
  const uint32_t* qinvR;     // q^-1 * R mod p
  ModDev modn;               // modulus n (padded)
  const uint32_t* qR;        // q * R mod n
  uint32_t* tbl;
  long tbl_stride;
  int stash_slot;            // table slot used to park mp while the q half runs
  const uint32_t* c;
  uint32_t* out;
  long count;
  int wn, wc;
  int c_mont;                // c is in Montgomery digit form of the n^2 context, whose R is the square of this one's
};

template <int LPT, int TPI>
__global__ void __launch_bounds__(32, 4 * blocks_per_sm(LPT)) k_decrypt(DecArgs A) {
  using M = Mont<LPT, TPI>;
  constexpr int IPW = 32 / TPI;
  M mt;
  // one warp per block: the tile loop then depends on blockIdx only, the compiler can see that the warp never
  // diverges, and every __shfl_sync becomes a bare SHFL instead of a WARPSYNC.COLLECTIVE / ENDCOLLECTIVE bracket
  const int lane = threadIdx.x, g = lane / TPI;
  const long wg = blockIdx.x, nw = gridDim.x;
  uint32_t* tw = A.tbl + wg * A.tbl_stride;
  uint32_t* sw = sqr_scratch<LPT, TPI>();
  const long ntiles = (A.count + IPW - 1) / IPW;
  const int wlo = A.wc / 2, whi = A.wc - wlo;
  for (long tile = wg; tile < ntiles; tile += nw) {
    long inst = tile * IPW + g;
    bool valid = inst < A.count;
    long ii = valid ? inst : A.count - 1;
    // Montgomery input: 2 L limbs v = vlo + vhi R' with v = c R'^2 mod n^2, so Mont'(c mod s^2) = vlo / R' + vhi
    const uint32_t* cw = A.c + ii * (A.c_mont ? 2 * LPT * TPI : A.wc);
    uint32_t x[LPT], y[LPT], z[LPT];
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
      const HalfDev& H = A.half[h];
      mt.init(H.s2.n, H.s2.np);
      // c mod s^2 in Montgomery form, from the two halves of c
      if (A.c_mont) {
        mt.load_limbs(x, cw);
        mt.set_one(y);
        mt.mul(x, x, y);                            // vlo / R' mod s^2
        mt.load_limbs(y, cw + LPT * TPI);
        mt.load_limbs(z, H.s2.r1);
        mt.mul(y, y, z);                            // vhi mod s^2
      } else {
        mt.load_words(x, cw, wlo);
        mt.load_limbs(y, H.s2.r2);
        mt.mul(x, x, y);
        mt.load_words(y, cw + wlo, whi);
        mt.load_limbs(z, H.hiR2);
        mt.mul(y, y, z);
      }
      mt.add_mod(x, x, y);
      run_prog<LPT, TPI>(mt, x, H.prog, H.nprog, tw, sw);   // Mont(c^(s-1) mod s^2)
      mt.set_one(z);
      mt.mul(x, x, z);                              // u = c^(s-1) mod s^2
      // u == 0 happens only when s divides c (never for a real ciphertext); the reference's floor
      // division (0 - 1) // s is then -1, i.e. t = s - 1 (mod s).
      const bool uzero = mt.is_zero(x);
      mt.sub_mod(x, x, z);                          // u - 1 = s * t
      mt.init(H.s1.n, H.s1.np);
      mt.mul_quot(x, y, x, z);                      // y <- quotient limbs of (u-1)*1 w.r.t. s
      mt.neg_R(y);                                  // t = (u - 1) / s
      if (uzero) {
#pragma unroll
        mt.get_n(y);
        if (mt.t == 0) y[0] -= 1u;                  // s is odd: no borrow
      }
      mt.load_limbs(z, H.hsR);
      mt.mul(x, y, z);                              // ms = t * hs mod s
      if (h == 0) tile_store<LPT>(tw, A.stash_slot, x);
    }
    // x = mq.  CRT recombination: m = mq + q * ((mp - mq) * q_inv mod p)   (operators.py:56)
    mt.init(A.half[0].s1.n, A.half[0].s1.np);       // modulus p
    mt.load_limbs(y, A.half[0].s1.r1);
    mt.mul(y, x, y);                                // mq mod p
    tile_load<LPT>(tw, A.stash_slot, z);            // mp
    mt.sub_mod(y, z, y);                            // (mp - mq) mod p
    mt.load_limbs(z, A.qinvR);
    mt.mul(y, y, z);                                // h in [0, p)
    mt.init(A.modn.n, A.modn.np);
    mt.load_limbs(z, A.qR);
    mt.mul(y, y, z);                                // q * h  (< n, exact)
    mt.add_mod(x, x, y);                            // mq + q*h  (< n)
    mt.store_words(A.out + ii * A.wn, A.wn, x, valid);
  }
}

}  // namespace hb
