// C ABI, host-only translation unit: the obfuscation-factor stream.
//
// The reference draws r = rng.randrange(1, n) per element from a Python random.Random
// (/root/reference/pkg/src/hebatch/paillier.py:173-178, operators.py:133,142), 23 us per element in Python at
// 2048 bits -- slower than the modular exponentiation on the GPU.  This reproduces CPython's stream bit for bit
// from the generator's exported state: MT19937, getrandbits(k) = little-endian 32-bit outputs with the top word
// shifted right, randrange(1, n) = 1 + rejection sampling of getrandbits((n-1).bit_length()) below n - 1.
// The gcd(r, n) = 1 test of draw_unit is done by the caller on the whole batch (one product on the GPU, one gcd).
#include <sys/random.h>
#include <cerrno>
#include "hb_ctx.h"

namespace {

struct MT {
  uint32_t* s;
  int idx;
  static inline uint32_t twist(uint32_t hi, uint32_t lo, uint32_t far) {
    const uint32_t y = (hi & 0x80000000u) | (lo & 0x7fffffffu);
    return far ^ (y >> 1) ^ ((0u - (y & 1u)) & 0x9908b0dfu);
  }
  void refill() {                        // three modulo-free stretches (the compiler vectorises the first two)
    constexpr int N = 624, M = 397;
    int k = 0;
    for (; k < N - M; k++) s[k] = twist(s[k], s[k + 1], s[k + M]);
    for (; k < N - 1; k++) s[k] = twist(s[k], s[k + 1], s[k + M - N]);
    s[N - 1] = twist(s[N - 1], s[0], s[M - 1]);
    idx = 0;
  }
  static inline uint32_t temper(uint32_t y) {
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
  }
  // the next `count` outputs, in order, into dst (refilling as the state runs out)
  void fill(uint32_t* dst, int count) {
    int done = 0;
    while (done < count) {
      if (idx >= 624) refill();
      const int take = std::min(count - done, 624 - idx);
      const uint32_t* src = s + idx;
      for (int j = 0; j < take; j++) dst[done + j] = temper(src[j]);
      idx += take;
      done += take;
    }
  }
};

}  // namespace

extern "C" int hb_mt19937_randrange1(uint32_t* state, int* index, const uint32_t* n_words, int wn, int64_t count,
                                     uint32_t* out) {
  if (!state || !index || !n_words || !out || wn <= 0 || count < 0) return hbi::fail(HB_ERR_ARG, "null pointer");
  // bound = n - 1
  std::vector<uint32_t> bound(n_words, n_words + wn);
  {
    int i = 0;
    while (i < wn && bound[i] == 0) bound[i++] = 0xffffffffu;
    if (i == wn) return hbi::fail(HB_ERR_ARG, "modulus is zero");
    bound[i] -= 1;
  }
  int top = wn - 1;
  while (top >= 0 && bound[top] == 0) top--;
  if (top < 0) return hbi::fail(HB_ERR_ARG, "randrange(1, 1) is empty");
  const int k = top * 32 + (32 - __builtin_clz(bound[top]));     // (n - 1).bit_length()
  const int words = (k + 31) / 32;
  MT mt{state, *index};
  const int topshift = (k % 32) ? 32 - (k % 32) : 0;
  for (int64_t e = 0; e < count; e++) {
    uint32_t* o = out + e * wn;
    while (true) {                       // candidates are drawn straight into the output row
      mt.fill(o, words);
      o[words - 1] >>= topshift;
      bool below = false;                // accept when candidate < bound
      for (int i = words - 1; i >= 0; i--) {
        if (o[i] != bound[i]) { below = o[i] < bound[i]; break; }
      }
      if (below) break;
    }
    for (int i = words; i < wn; i++) o[i] = 0u;
    for (int i = 0; i < wn; i++) {       // + 1
      if (++o[i] != 0u) break;
    }
  }
  *index = mt.idx;
  return HB_OK;
}

// The same draw from the operating system's CSPRNG (getrandom(2)), for callers whose generator is
// random.SystemRandom or who pass none: randrange(1, n) of a SystemRandom is rejection sampling of
// getrandbits((n-1).bit_length()) below n - 1 over os.urandom bytes, so this is the same distribution from the
// same entropy source, drawn in bulk instead of one Python call per element.
extern "C" int hb_secure_randrange1(const uint32_t* n_words, int wn, int64_t count, uint32_t* out) {
  if (!n_words || !out || wn <= 0 || count < 0) return hbi::fail(HB_ERR_ARG, "null pointer");
  std::vector<uint32_t> bound(n_words, n_words + wn);
  {
    int i = 0;
    while (i < wn && bound[i] == 0) bound[i++] = 0xffffffffu;
    if (i == wn) return hbi::fail(HB_ERR_ARG, "modulus is zero");
    bound[i] -= 1;
  }
  int top = wn - 1;
  while (top >= 0 && bound[top] == 0) top--;
  if (top < 0) return hbi::fail(HB_ERR_ARG, "randrange(1, 1) is empty");
  const int k = top * 32 + (32 - __builtin_clz(bound[top]));     // (n - 1).bit_length()
  const int words = (k + 31) / 32;
  const uint32_t topmask = (k % 32) ? ((1u << (k % 32)) - 1u) : 0xffffffffu;
  // entropy in blocks of up to 4096 candidates
  const size_t cand_bytes = (size_t)words * 4;
  std::vector<uint32_t> pool((size_t)words * 4096);
  size_t have = 0, pos = 0;
  for (int64_t e = 0; e < count; e++) {
    const uint32_t* cand = nullptr;
    while (true) {
      if (pos == have) {
        const size_t want = std::min<size_t>(4096, (size_t)(count - e) + 16) * cand_bytes;
        size_t got = 0;
        while (got < want) {
          ssize_t r = getrandom((char*)pool.data() + got, want - got, 0);
          if (r < 0) {
            if (errno == EINTR) continue;
            return hbi::fail(HB_ERR_ARG, "getrandom() failed");
          }
          got += (size_t)r;
        }
        have = want / cand_bytes;
        pos = 0;
      }
      uint32_t* cnd = pool.data() + pos * words;
      pos++;
      cnd[words - 1] &= topmask;
      bool below = false;
      for (int i = words - 1; i >= 0; i--) {
        if (cnd[i] != bound[i]) { below = cnd[i] < bound[i]; break; }
      }
      if (below) { cand = cnd; break; }
    }
    uint32_t* o = out + e * wn;
    uint32_t carry = 1;
    for (int i = 0; i < wn; i++) {
      uint32_t v = (i < words ? cand[i] : 0u);
      uint32_t s = v + carry;
      carry = (s < v) ? 1u : 0u;
      o[i] = s;
    }
  }
  return HB_OK;
}
