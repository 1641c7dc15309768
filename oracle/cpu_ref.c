/*
 * TEST INFRASTRUCTURE ONLY -- C restatement of the reference's element kernels on GMP, multi-threaded.
 *
 * The reference runs these loops in Python over gmpy2 (= GMP):
 *   /root/reference/pkg/src/hebatch/operators.py:39-41  _k_encrypt   (1 + m n) r^n mod n^2
 *   operators.py:49-56                                   _k_decrypt   CRT decryption
 *   operators.py:59-67                                   _pow_scalar / _k_mul
 *   operators.py:70-72                                   _k_add
 *   operators.py:86-94                                   _k_dot
 * Here the same mpz calls are issued from C under OpenMP, which is the strongest CPU form of the
 * reference's algorithm (no interpreter, every host core busy).  Used as the checker at sizes where the
 * Python oracle is too slow and as bench.py's cpu_baseline / --impl reference arm.
 *
 * gmp.h is not installed in this image; the GMP runtime (libgmp.so.10, GMP 6.3.0, the library gmpy2
 * wraps) is, so the handful of prototypes used are declared by hand.  Build: oracle/Makefile.
 * Big integers cross the boundary as little-endian 32-bit words, like include/hebatch_b200.h.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { int _mp_alloc; int _mp_size; unsigned long* _mp_d; } __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

void __gmpz_init(mpz_ptr);
void __gmpz_clear(mpz_ptr);
void __gmpz_import(mpz_ptr, size_t, int, size_t, int, size_t, const void*);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, mpz_srcptr);
void __gmpz_powm(mpz_ptr, mpz_srcptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mod(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_add_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_sub_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_fdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_q_ui(mpz_ptr, mpz_srcptr, unsigned long);
int __gmpz_invert(mpz_ptr, mpz_srcptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_ui(mpz_ptr, unsigned long);

#define mpz_init __gmpz_init
#define mpz_clear __gmpz_clear
#define mpz_powm __gmpz_powm
#define mpz_mul __gmpz_mul
#define mpz_mod __gmpz_mod
#define mpz_add __gmpz_add
#define mpz_sub __gmpz_sub
#define mpz_add_ui __gmpz_add_ui
#define mpz_sub_ui __gmpz_sub_ui
#define mpz_fdiv_q __gmpz_fdiv_q
#define mpz_fdiv_q_ui __gmpz_fdiv_q_ui
#define mpz_invert __gmpz_invert
#define mpz_cmp __gmpz_cmp
#define mpz_set __gmpz_set
#define mpz_set_ui __gmpz_set_ui

static void get(mpz_ptr z, const uint32_t* w, int nw) { __gmpz_import(z, (size_t)nw, -1, 4, 0, 0, w); }
static void put(uint32_t* w, int nw, mpz_srcptr z) {
  size_t cnt = 0;
  memset(w, 0, (size_t)nw * 4);
  __gmpz_export(w, &cnt, -1, 4, 0, 0, z);
}

int cpuref_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* out[i] = mult(i) * r[i]^n mod n^2;  mode 0: mult = 1 + m[i] n (a = m, wa = wn);  mode 1: mult = a[i] (wa = wc) */
int cpuref_encrypt(const uint32_t* n_w, int wn, const uint32_t* a, int wa, const uint32_t* r, uint32_t* out,
                   int wc, long count, int mode, int threads) {
#pragma omp parallel num_threads(threads)
  {
    mpz_t n, n2, x, y, t;
    mpz_init(n); mpz_init(n2); mpz_init(x); mpz_init(y); mpz_init(t);
    get(n, n_w, wn);
    mpz_mul(n2, n, n);
#pragma omp for schedule(dynamic, 4)
    for (long i = 0; i < count; i++) {
      get(x, r + i * wn, wn);
      mpz_powm(y, x, n, n2);
      get(x, a + i * wa, wa);
      if (mode == 0) { mpz_mul(t, x, n); mpz_add_ui(x, t, 1); }
      mpz_mul(t, x, y);
      mpz_mod(x, t, n2);
      put(out + i * wc, wc, x);
    }
    mpz_clear(n); mpz_clear(n2); mpz_clear(x); mpz_clear(y); mpz_clear(t);
  }
  return 0;
}

/* m = mq + q * ((mp - mq) * q_inv mod p),  mp = (c^(p-1) mod p^2 - 1) / p * hp mod p  (operators.py:52-55) */
int cpuref_decrypt(const uint32_t* p_w, const uint32_t* q_w, const uint32_t* hp_w, const uint32_t* hq_w,
                   const uint32_t* qinv_w, int hw, const uint32_t* c, int wc, uint32_t* out, int wn, long count,
                   int threads) {
#pragma omp parallel num_threads(threads)
  {
    mpz_t p, q, p2, q2, hp, hq, qinv, pm1, qm1, x, mp, mq, t;
    mpz_init(p); mpz_init(q); mpz_init(p2); mpz_init(q2); mpz_init(hp); mpz_init(hq); mpz_init(qinv);
    mpz_init(pm1); mpz_init(qm1); mpz_init(x); mpz_init(mp); mpz_init(mq); mpz_init(t);
    get(p, p_w, hw); get(q, q_w, hw); get(hp, hp_w, hw); get(hq, hq_w, hw); get(qinv, qinv_w, hw);
    mpz_mul(p2, p, p); mpz_mul(q2, q, q);
    mpz_sub_ui(pm1, p, 1); mpz_sub_ui(qm1, q, 1);
#pragma omp for schedule(dynamic, 4)
    for (long i = 0; i < count; i++) {
      get(x, c + i * wc, wc);
      mpz_powm(t, x, pm1, p2); mpz_sub_ui(t, t, 1); mpz_fdiv_q(t, t, p); mpz_mul(t, t, hp); mpz_mod(mp, t, p);
      mpz_powm(t, x, qm1, q2); mpz_sub_ui(t, t, 1); mpz_fdiv_q(t, t, q); mpz_mul(t, t, hq); mpz_mod(mq, t, q);
      mpz_sub(t, mp, mq); mpz_mul(t, t, qinv); mpz_mod(t, t, p);
      mpz_mul(t, t, q); mpz_add(t, t, mq);
      put(out + i * wn, wn, t);
    }
    mpz_clear(p); mpz_clear(q); mpz_clear(p2); mpz_clear(q2); mpz_clear(hp); mpz_clear(hq); mpz_clear(qinv);
    mpz_clear(pm1); mpz_clear(qm1); mpz_clear(x); mpz_clear(mp); mpz_clear(mq); mpz_clear(t);
  }
  return 0;
}

int cpuref_mulmod(const uint32_t* n_w, int wn, const uint32_t* a, const uint32_t* b, uint32_t* out, int wc,
                  long count, int threads) {
#pragma omp parallel num_threads(threads)
  {
    mpz_t n, n2, x, y, t;
    mpz_init(n); mpz_init(n2); mpz_init(x); mpz_init(y); mpz_init(t);
    get(n, n_w, wn);
    mpz_mul(n2, n, n);
#pragma omp for schedule(static)
    for (long i = 0; i < count; i++) {
      get(x, a + i * wc, wc); get(y, b + i * wc, wc);
      mpz_mul(t, x, y); mpz_mod(x, t, n2);
      put(out + i * wc, wc, x);
    }
    mpz_clear(n); mpz_clear(n2); mpz_clear(x); mpz_clear(y); mpz_clear(t);
  }
  return 0;
}

/* pow_scalar (operators.py:59-62); returns 0 when an inverse does not exist */
static int pow_scalar(mpz_ptr out, mpz_srcptr c, mpz_srcptr k, mpz_srcptr n, mpz_srcptr n2, mpz_srcptr negband,
                      mpz_ptr tmp, mpz_ptr tmp2) {
  if (mpz_cmp(k, negband) > 0) {
    if (!mpz_invert(tmp, c, n2)) return 0;
    mpz_sub(tmp2, n, k);
    mpz_powm(out, tmp, tmp2, n2);
  } else {
    mpz_powm(out, c, k, n2);
  }
  return 1;
}

/* out[i] = pow_scalar(c[i], k[i % k_period]) */
int cpuref_powscalar(const uint32_t* n_w, int wn, const uint32_t* c, int wc, const uint32_t* k, long k_period,
                     uint32_t* out, long count, int threads) {
  int bad = 0;
#pragma omp parallel num_threads(threads)
  {
    mpz_t n, n2, nb, x, kk, y, t1, t2;
    mpz_init(n); mpz_init(n2); mpz_init(nb); mpz_init(x); mpz_init(kk); mpz_init(y); mpz_init(t1); mpz_init(t2);
    get(n, n_w, wn);
    mpz_mul(n2, n, n);
    mpz_fdiv_q_ui(nb, n, 3); mpz_sub(nb, n, nb);
#pragma omp for schedule(dynamic, 16)
    for (long i = 0; i < count; i++) {
      get(x, c + i * wc, wc); get(kk, k + (i % k_period) * wn, wn);
      if (!pow_scalar(y, x, kk, n, n2, nb, t1, t2)) { bad = 1; continue; }
      put(out + i * wc, wc, y);
    }
    mpz_clear(n); mpz_clear(n2); mpz_clear(nb); mpz_clear(x); mpz_clear(kk); mpz_clear(y); mpz_clear(t1); mpz_clear(t2);
  }
  return bad ? -5 : 0;
}

/* out[j] = prod_t pow_scalar(c[t], k[t*d + j]) for t < inner, j < d  (one encrypted row; operators.py:86-94) */
int cpuref_matvec(const uint32_t* n_w, int wn, const uint32_t* c, int wc, const uint32_t* k, long inner, long d,
                  uint32_t* out, int threads) {
  int bad = 0;
#pragma omp parallel num_threads(threads)
  {
    mpz_t n, n2, nb, x, kk, y, acc, t1, t2;
    mpz_init(n); mpz_init(n2); mpz_init(nb); mpz_init(x); mpz_init(kk); mpz_init(y); mpz_init(acc);
    mpz_init(t1); mpz_init(t2);
    get(n, n_w, wn);
    mpz_mul(n2, n, n);
    mpz_fdiv_q_ui(nb, n, 3); mpz_sub(nb, n, nb);
#pragma omp for schedule(dynamic, 1)
    for (long j = 0; j < d; j++) {
      mpz_set_ui(acc, 1);
      for (long t = 0; t < inner; t++) {
        get(x, c + t * wc, wc); get(kk, k + (t * d + j) * wn, wn);
        if (!pow_scalar(y, x, kk, n, n2, nb, t1, t2)) { bad = 1; break; }
        mpz_mul(t1, acc, y); mpz_mod(acc, t1, n2);
      }
      put(out + j * wc, wc, acc);
    }
    mpz_clear(n); mpz_clear(n2); mpz_clear(nb); mpz_clear(x); mpz_clear(kk); mpz_clear(y); mpz_clear(acc);
    mpz_clear(t1); mpz_clear(t2);
  }
  return bad ? -5 : 0;
}
