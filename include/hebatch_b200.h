/*
 * hebatch_b200 -- C ABI of the B200-native homomorphic-operator library.
 *
 * This is the drop-in boundary for the hot path of the reference package `hebatch`
 * (/root/reference/pkg/src/hebatch): every entry point replaces one element kernel that the
 * reference runs through ExecutionBackend.run (backends.py:28) on top of gmpy2.  The reference has
 * no FFI of its own (pure Python over gmpy2), so the binding a maintainer adds is the ctypes stub
 * shown in INTEGRATION.md.
 *
 * Conventions
 *   - Every big integer is an array of little-endian 32-bit words.  Plaintext residues (mod n) use
 *     hb_pt_words(ctx) words, ciphertexts (mod n^2) use hb_ct_words(ctx) words.  For key sizes that
 *     are multiples of 16 bits this is byte-for-byte the HAFB wire payload (bufferpool.py:231-330).
 *   - Batches are dense arrays: element i starts at word i * words.
 *   - Functions whose names do not end in _host take DEVICE pointers and enqueue work on `stream`
 *     (a cudaStream_t passed as void*; NULL = the legacy default stream).  They never allocate host
 *     memory; scratch comes from the library's own stream-ordered pool (one per device, bounded by
 *     HB_OPT_POOL_KEEP_BYTES; the device's default pool is not touched).
 *   - Synchronisation.  Stream-ordered, never synchronising: hb_encrypt*, hb_obfuscate*, hb_decrypt*, hb_mulmod*,
 *     hb_lift_mulmod*, hb_fore_gradient, hb_product*, hb_unit_product, hb_plain_*, hb_encode_f64*, hb_decode_f64,
 *     hb_min_exact_exponent, hb_scalar_compact, hb_ct_convert,
 *     hb_matvec_partial_compact, and hb_matvec_compact when has_negative == 0.
 *     Synchronising `stream` ONCE, at the end, to read the inversion flag (HB_ERR_NOTUNIT): hb_matvec_compact with
 *     has_negative != 0, hb_matvec_combine.  Synchronising once at the start to read the scalar statistics (and at
 *     the end when a scalar is negative): hb_powscalar, hb_matvec, hb_matvec_rep, hb_matvec_partial.
 *   - Ciphertext representations: plain words (hb_ct_words per element, the wire form) or Montgomery
 *     digit form x * R mod n^2 (hb_ct_limbs per element), the form chained operators keep in HBM so that an
 *     addition is one modular multiplication and no operator converts in and out.  The *_rep entry points take
 *     `flags` built from HB_A_MONT / HB_B_MONT / HB_OUT_MONT; the classic names are the all-plain case.
 *     Digit-form arrays must be 16-byte aligned (HB_ERR_ARG otherwise); plain-word arrays may have any alignment
 *     (16-byte aligned ones are moved 16 bytes at a time).
 *   - *_host functions take HOST pointers, stage through pinned buffers on side streams (chunked,
 *     copy/compute overlapped) and return when the result is in the caller's buffer.
 *   - Return value: 0 on success, negative hb_status on failure; hb_last_error() gives the text
 *     (thread-local).  There is no CPU fallback: without a usable CUDA device every call fails.
 */
#ifndef HEBATCH_B200_H
#define HEBATCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hb_ctx hb_ctx;

enum hb_status {
  HB_OK = 0,
  HB_ERR_ARG = -1,        /* bad argument (null pointer, even modulus, size mismatch, ...) */
  HB_ERR_CUDA = -2,       /* CUDA runtime failure */
  HB_ERR_UNSUPPORTED = -3,/* key size beyond the instantiated limb configurations */
  HB_ERR_NOPRIVATE = -4,  /* decrypt requested on a context without the private part */
  HB_ERR_NOTUNIT = -5     /* modular inverse of a non-unit (gmpy2.invert raises ZeroDivisionError) */
};

const char* hb_last_error(void);
/* Library version and the GPU architecture it was compiled for ("sm_100a"). */
const char* hb_version(void);

/* ---- key context ------------------------------------------------------------------------------
 * Replaces the per-call `common` tuples of operators.py (:40,45,50,66,71) and the cached values of
 * paillier.PublicKey (:39-66) / PrivateKey (:69-107).  n is key_bits wide; n^2, Montgomery constants
 * and the exponent schedule for r^n are derived here, once.                                        */
int hb_ctx_create(hb_ctx** out, const uint32_t* n_words, int n_nwords, int device);
/* Private part for CRT decryption (paillier.py:94-98): primes p, q and hp, hq, q^-1 mod p, each as
 * `nwords` little-endian words. */
int hb_ctx_set_private(hb_ctx* ctx, const uint32_t* p, const uint32_t* q, const uint32_t* hp,
                       const uint32_t* hq, const uint32_t* q_inv_p, int nwords);
void hb_ctx_destroy(hb_ctx* ctx);
/* Per-context tunables.  HB_OPT_MATVEC_WINDOW_BITS: bucket window of hb_matvec (2..13; 0 = by row count, the
 * default) -- lets tests exercise every width.  HB_OPT_POOL_KEEP_BYTES: how much freed scratch the library's pool on
 * the context's device keeps across synchronisations (default: 1 GiB or 1/8 of the device's memory, whichever is
 * larger -- 22 GiB on a 180 GB B200; shared by the contexts on that device).
 * HB_OPT_MATVEC_BLOCK_ROWS: rows of the inner dimension hb_matvec reduces per bucket pass (0 = 2^21, the default);
 * taller matrices are processed block by block and the blocks' partial products multiplied together. */
enum hb_option { HB_OPT_MATVEC_WINDOW_BITS = 1, HB_OPT_POOL_KEEP_BYTES = 2, HB_OPT_MATVEC_BLOCK_ROWS = 3 };
int hb_ctx_set_option(hb_ctx* ctx, int option, int64_t value);
int hb_pt_words(const hb_ctx* ctx);   /* words per plaintext residue  = ceil(key_bits / 32)           */
int hb_ct_words(const hb_ctx* ctx);   /* words per ciphertext         = ceil(ceil(2*key_bits/8) / 4)  */
int hb_key_bits(const hb_ctx* ctx);
int hb_ct_limbs(const hb_ctx* ctx);   /* words per ciphertext in Montgomery digit form (>= hb_ct_words)          */

/* Representation flags of the *_rep entry points and of hb_powscalar: which ciphertext arrays are in Montgomery
 * digit form (hb_ct_limbs words per element) instead of plain words (hb_ct_words per element). */
#define HB_A_MONT   0x10   /* first ciphertext operand (a / c)  */
#define HB_B_MONT   0x20   /* second ciphertext operand (b)     */
#define HB_OUT_MONT 0x40   /* the result                        */
/* out = Montgomery digit form of `in` (to_montgomery != 0) or the plain words of a digit-form array (== 0). */
int hb_ct_convert(hb_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t count, int to_montgomery, void* stream);

/* ---- element operators (device pointers) --------------------------------------------------------*/
/* _k_encrypt, operators.py:39-41:  out[i] = (1 + m[i]*n) * r[i]^n mod n^2.   m, r: pt words. */
int hb_encrypt(hb_ctx* ctx, const uint32_t* m, const uint32_t* r, uint32_t* out, int64_t count, void* stream);
/* _k_obfuscate, operators.py:44-46: out[i] = c[i] * r[i]^n mod n^2. */
int hb_obfuscate(hb_ctx* ctx, const uint32_t* c, const uint32_t* r, uint32_t* out, int64_t count, void* stream);
/* _k_decrypt, operators.py:49-56 (CRT form of paillier.py:201-209): m_out[i] in [0, n). */
int hb_decrypt(hb_ctx* ctx, const uint32_t* c, uint32_t* m_out, int64_t count, void* stream);
/* _k_add, operators.py:70-72: out[i] = a[i] * b[i] mod n^2.  b_stride_zero != 0 broadcasts b[0]. */
int hb_mulmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
              int b_broadcast, void* stream);
/* batch_add with a plaintext operand, operators.py:209-212: out[i] = a[i] * (1 + m[i]*n) mod n^2. */
int hb_lift_mulmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* m, uint32_t* out, int64_t count,
                   int m_broadcast, void* stream);

/* The same four with representation flags (chained operators, arena.py:240-280: operands that stay "on the
 * device" between operators).  hb_encrypt_rep honours HB_OUT_MONT; hb_obfuscate_rep HB_A_MONT | HB_OUT_MONT;
 * hb_decrypt_rep HB_A_MONT; hb_mulmod_rep all three; hb_lift_mulmod_rep HB_A_MONT | HB_OUT_MONT. */
int hb_encrypt_rep(hb_ctx* ctx, const uint32_t* m, const uint32_t* r, uint32_t* out, int64_t count, int flags,
                   void* stream);
int hb_obfuscate_rep(hb_ctx* ctx, const uint32_t* c, const uint32_t* r, uint32_t* out, int64_t count, int flags,
                     void* stream);
int hb_decrypt_rep(hb_ctx* ctx, const uint32_t* c, uint32_t* m_out, int64_t count, int flags, void* stream);
int hb_mulmod_rep(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                  int b_broadcast, int flags, void* stream);
int hb_lift_mulmod_rep(hb_ctx* ctx, const uint32_t* a, const uint32_t* m, uint32_t* out, int64_t count,
                       int m_broadcast, int flags, void* stream);

/* Fused fore-gradient chain of one heterogeneous-FLR mini-batch, Arena.run_fore_gradient_pipeline (arena.py:345-366:
 * plain_mul, encrypt, hmul, hadd, plain_mul, hadd of a lifted plaintext) in one pass per element:
 *     out[i] = (1 + (lg[i] * kg mod n) n) r[i]^n  *  c[i]^kh  *  (1 + yl[i] n)     mod n^2
 * c: the host's encrypted logits; lg: the guest's logits and kg the plaintext factor (one residue; 4 for the
 * reference's encode(0.25)); kh: the same factor as a small positive exponent; yl: the label term, already multiplied
 * and re-gridded on the plaintext side (hb_plain_mulmod + hb_plain_rescale, which own the overflow checks); r: the
 * obfuscation factors of the encryption step.  Bit-identical to the six-operator sequence.  flags: HB_A_MONT (c),
 * HB_OUT_MONT. */
int hb_fore_gradient(hb_ctx* ctx, const uint32_t* c, const uint32_t* lg, const uint32_t* kg, uint32_t kh,
                     const uint32_t* yl, const uint32_t* r, uint32_t* out, int64_t count, int flags, void* stream);

/* Default exponent of encode_batch (batches.py:122-123): min over the values of encoding.exact_exponent
 * (encoding.py:44-51), zeros counting as 0.  min_out: device int preset by the caller to INT_MAX (left untouched
 * only when count == 0). */
int hb_min_exact_exponent(hb_ctx* ctx, const double* values, int64_t count, int* min_out, void* stream);

/* Plaintext-side residue arithmetic mod n (batches.py:160-205 of the reference).  plain_mul: out[i] = a[i] * b[i]
 * mod n (b_broadcast != 0 uses b[0]); plain_add: out[i] = a[i] + b[i] mod n; plain_rescale
 * (encoding.py:104-113): the signed mantissa times 16^digits, back as a residue -- first_bad (device int64,
 * preset by the caller to -1, as for the codec) receives the smallest index in the overflow band or beyond max_int
 * after scaling, or stays -1. */
int hb_plain_mulmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                    int b_broadcast, void* stream);
int hb_plain_addmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, void* stream);
int hb_plain_rescale(hb_ctx* ctx, const uint32_t* m, int digits, uint32_t* m_out, int64_t count,
                     int64_t* first_bad, void* stream);

/* Repeated squaring, out[i] = a[i]^(2^reps) mod n^2: the inner step of every modular power on this path
 * (gmpy2.powmod at paillier.py:190,207-208 / operators.py:41,46,53-54).  Exposed so the dedicated squaring of
 * the kernels can be checked and timed on its own.  throughput_shape != 0 forces the limb shape large batches
 * use, whatever `count` is. */
int hb_sqrmod(hb_ctx* ctx, const uint32_t* a, uint32_t* out, int64_t count, int reps, int throughput_shape,
              void* stream);

/* _pow_scalar / _k_mul, operators.py:59-67: out[i] = pow_scalar(c[i], k[i % k_period]) where residues
 * k > n - n/3 are negative: the base becomes c^-1 mod n^2 and the exponent n - k.  k_period = 1
 * broadcasts one scalar, = columns broadcasts a row vector over a 2-D batch, = count is element-wise.
 * Only the ciphertexts paired with a negative scalar are inverted (as the reference does, element by element);
 * returns HB_ERR_NOTUNIT if one of those has no inverse.  flags: HB_POW_RAW_EXPONENT | HB_A_MONT | HB_OUT_MONT. */
#define HB_POW_RAW_EXPONENT 1   /* flags: exponent is the residue itself (paillier.hmul_raw, :221-228) */
int hb_powscalar(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t count,
                 int64_t k_period, int flags, void* stream);
/* _k_product, operators.py:75-83: out[g] = prod_{t < glen} c[g*gstride + t*estride] mod n^2.
 * axis=None: (1, count, 0, 1); axis=0 of rows x cols: (cols, rows, 1, cols); axis=1: (rows, cols, cols, 1). */
int hb_product(hb_ctx* ctx, const uint32_t* c, uint32_t* out, int64_t ngroups, int64_t glen,
               int64_t gstride, int64_t estride, void* stream);
int hb_product_rep(hb_ctx* ctx, const uint32_t* c, uint32_t* out, int64_t ngroups, int64_t glen,
                   int64_t gstride, int64_t estride, int flags, void* stream);   /* HB_A_MONT | HB_OUT_MONT */
/* out[0] = prod_i r[i] mod n^2 for plaintext-width values r (count x pt words).  gcd(out, n) = 1 iff every
 * r[i] is a unit mod n: the batched form of draw_unit's gcd test (paillier.py:176-177). */
int hb_unit_product(hb_ctx* ctx, const uint32_t* r, uint32_t* out, int64_t count, void* stream);
/* _k_dot / batch_matmul, operators.py:86-94,294-317: c is rows x inner ciphertexts, k is inner x d
 * plaintext residues (row-major), out is rows x d:  out[i][j] = prod_t pow_scalar(c[i][t], k[t][j]).
 * Scalars whose magnitude fits 64 bits take the bucket (Pippenger) path; wider ones a generic path.
 * Any inner dimension: rows beyond 2^21 are reduced block by block and the blocks multiplied together. */
int hb_matvec(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t rows,
              int64_t inner, int64_t d, void* stream);
int hb_matvec_rep(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t rows,
                  int64_t inner, int64_t d, int flags, void* stream);            /* HB_A_MONT | HB_OUT_MONT */

/* Compact resident form of a plaintext scalar matrix (the role of MiniBatchAggregator, bufferpool.py:182-226:
 * pack a mini-batch's feature block once, reuse it every epoch): sign + 64-bit magnitude per scalar, stored by
 * COLUMN -- mag[j * rows + t], neg[j * rows + t] for k[t][j] -- which is all the bucket kernels read: 9 bytes per
 * scalar instead of a hb_pt_words residue (256 B at 2048 bits).  info (3 device ints, zeroed by the call) receives
 * the largest magnitude bit length, the number of negative scalars and (hb_encode_f64_compact) the number of values
 * whose magnitude does not fit 64 bits.  A bit length above 64 or a non-zero misfit count means the matrix has no
 * compact form and the residue path (hb_matvec) must be used.
 * hb_scalar_compact starts from residues; hb_encode_f64_compact straight from doubles (encoding.py:54-78 with the
 * given exponent, round-half-even), never materialising the residues; key sizes below 128 bits are refused. */
int hb_scalar_compact(hb_ctx* ctx, const uint32_t* k, int64_t rows, int64_t cols, uint64_t* mag_out,
                      uint8_t* neg_out, int* info_out, void* stream);
int hb_encode_f64_compact(hb_ctx* ctx, const double* values, int exponent, int64_t rows, int64_t cols,
                          uint64_t* mag_out, uint8_t* neg_out, int* info_out, void* stream);
/* hb_matvec (rows = 1) / hb_matvec_partial on the compact form.  maxbits and has_negative are the statistics the
 * compaction returned (any upper bound on the bit length <= 64 is valid; has_negative != 0 is always valid), so the
 * call starts without a synchronisation. */
int hb_matvec_compact(hb_ctx* ctx, const uint32_t* c, const uint64_t* mag, const uint8_t* neg, int maxbits,
                      int has_negative, uint32_t* out, int64_t inner, int64_t d, int flags, void* stream);
int hb_matvec_partial_compact(hb_ctx* ctx, const uint32_t* c, const uint64_t* mag, const uint8_t* neg, int maxbits,
                              uint32_t* ab_out, int64_t inner, int64_t d, int flags, void* stream);

/* Row-sharded form of hb_matvec for several GPUs: each rank reduces its own rows to d
 * pairs (A_j, B_j) -- products over the non-negative and the negative scalars -- written as 2*d plain
 * ciphertext words [d][2][ct words]; the ranks all-gather those (d KiB-sized messages) and every rank (or the
 * root) combines nranks such blocks: out[j] = (prod_r A_rj) * (prod_r B_rj)^-1.  Exact and commutative, so
 * the bits equal the single-GPU hb_matvec. */
int hb_matvec_partial(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* ab_out, int64_t inner,
                      int64_t d, void* stream);
int hb_matvec_combine(hb_ctx* ctx, const uint32_t* ab_all, int nranks, uint32_t* out, int64_t d, void* stream);

/* ---- fixed-point codec (encoding.py:54-101), shared exponent per call ------------------------------
 * *first_bad is a DEVICE int64 the caller initialises to -1; it receives the smallest element index that
 * overflowed (encode: |mantissa| >= n/3; decode: residue inside the overflow band), or stays -1. */
int hb_encode_f64(hb_ctx* ctx, const double* values, int exponent, uint32_t* m_out, int64_t count,
                  int64_t* first_bad, void* stream);
int hb_decode_f64(hb_ctx* ctx, const uint32_t* m, int exponent, double* values_out, int64_t count,
                  int64_t* first_bad, void* stream);

/* ---- host-buffer convenience path (pinned staging, side streams) --------------------------------*/
int hb_encrypt_host(hb_ctx* ctx, const uint32_t* m, const uint32_t* r, uint32_t* out, int64_t count);
int hb_decrypt_host(hb_ctx* ctx, const uint32_t* c, uint32_t* m_out, int64_t count);

/* ---- obfuscation-factor stream (host code) -----------------------------------------------------
 * `count` values of random.Random.randrange(1, n), bit-identical to CPython: `state` are the 624 words and
 * `*index` the position of rng.getstate()[1]; both are advanced so the caller can setstate() afterwards.
 * Replaces the randrange half of paillier.draw_unit (paillier.py:173-178); the gcd(r, n) = 1 half is checked
 * by the caller on the whole batch.  out: count x wn words. */
int hb_mt19937_randrange1(uint32_t* state, int* index, const uint32_t* n_words, int wn, int64_t count,
                          uint32_t* out);
/* The same draw from the operating system's CSPRNG (getrandom(2)) -- the bulk form of draw_unit under
 * random.SystemRandom (paillier.default_rng() without a seed, the secure default): rejection sampling of
 * (n-1).bit_length()-bit candidates below n - 1, plus 1.  Not reproducible by construction. */
int hb_secure_randrange1(const uint32_t* n_words, int wn, int64_t count, uint32_t* out);

/* ---- instrumentation ----------------------------------------------------------------------------*/
/* Number of kernels this library has launched since load (all contexts). */
int64_t hb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HEBATCH_B200_H */
