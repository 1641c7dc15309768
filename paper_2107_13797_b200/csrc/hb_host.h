// Host-side helpers of the C ABI: a minimal unsigned big integer (little-endian 32-bit words) used
// once per key to derive Montgomery constants and exponent programs.  Nothing here runs per element.
#pragma once
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

namespace hbh {

using Big = std::vector<uint32_t>;

inline void trim(Big& a) { while (!a.empty() && a.back() == 0) a.pop_back(); }
inline int bitlen(const Big& a) {
  for (int i = (int)a.size() - 1; i >= 0; i--)
    if (a[i]) return i * 32 + (32 - __builtin_clz(a[i]));
  return 0;
}
inline int cmp(const Big& a, const Big& b) {
  size_t n = std::max(a.size(), b.size());
  for (size_t i = n; i-- > 0;) {
    uint32_t x = i < a.size() ? a[i] : 0, y = i < b.size() ? b[i] : 0;
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}
inline bool is_zero(const Big& a) { return bitlen(a) == 0; }
inline Big from_words(const uint32_t* w, int n) { Big a(w, w + n); trim(a); return a; }
inline bool bit(const Big& a, int i) { return (size_t)(i >> 5) < a.size() && ((a[i >> 5] >> (i & 31)) & 1u); }

// a -= b, requires a >= b
inline void sub_in(Big& a, const Big& b) {
  uint64_t borrow = 0;
  for (size_t i = 0; i < a.size(); i++) {
    uint64_t x = a[i], y = (i < b.size() ? b[i] : 0) + borrow;
    borrow = x < y;
    a[i] = (uint32_t)(x - y);
  }
}
inline Big mul(const Big& a, const Big& b) {
  Big r(a.size() + b.size() + 1, 0);
  for (size_t i = 0; i < a.size(); i++) {
    uint64_t carry = 0;
    for (size_t j = 0; j < b.size(); j++) {
      uint64_t v = (uint64_t)a[i] * b[j] + r[i + j] + carry;
      r[i + j] = (uint32_t)v;
      carry = v >> 32;
    }
    size_t k = i + b.size();
    while (carry) { uint64_t v = (uint64_t)r[k] + carry; r[k] = (uint32_t)v; carry = v >> 32; k++; }
  }
  trim(r);
  return r;
}
// x * 2^k mod n for x < n (k modular doublings; used only at key-context creation)
inline Big shl_mod(Big x, long k, const Big& n) {
  size_t w = n.size() + 1;
  x.resize(w, 0);
  for (long s = 0; s < k; s++) {
    uint32_t c = 0;
    for (size_t i = 0; i < w; i++) { uint32_t v = x[i]; x[i] = (v << 1) | c; c = v >> 31; }
    if (cmp(x, n) >= 0) sub_in(x, n);
  }
  trim(x);
  return x;
}
inline Big sub_small(Big a, uint32_t v) { Big b{v}; sub_in(a, b); trim(a); return a; }

constexpr int RB = 32;      // radix bits of the device representation

// the L 32-bit limbs of a (zero padded)
inline std::vector<uint32_t> to_limbs(const Big& a, int L) {
  std::vector<uint32_t> d(L, 0);
  for (int i = 0; i < L && i < (int)a.size(); i++) d[i] = a[i];
  return d;
}
// -n^-1 mod 2^32 for odd n
inline uint32_t neg_inv32(uint32_t n0) {
  uint32_t inv = n0;                     // correct to 3 bits
  for (int i = 0; i < 5; i++) inv *= 2u - n0 * inv;
  return 0u - inv;
}

enum : uint32_t { OP_SQR = 0, OP_MUL = 1, OP_LOAD = 2, OP_KEEP = 3, OP_NODST = 0xFF };
inline uint32_t op(uint32_t kind, uint32_t src, uint32_t dst) { return kind | (src << 8) | (dst << 16); }

// Sliding-window program for a fixed exponent e >= 1 over odd powers b^1, b^3, ..., b^(2^w - 1).
// Table slots: [0, nodd) odd powers, nodd = b^2.  Register x holds Mont(b) on entry, Mont(b^e) on exit.
inline std::vector<uint32_t> build_program(const Big& e, int w, int* slots_used) {
  std::vector<uint32_t> p;
  int nbits = bitlen(e);
  int nodd = 1 << (w - 1);
  // which odd powers are needed?  (build all up to the largest one used)
  struct Step { int nsq; int idx; };
  std::vector<Step> steps;
  int i = nbits - 1, pending = 0, maxidx = 0;
  while (i >= 0) {
    if (!bit(e, i)) { pending++; i--; continue; }
    int j = std::max(i - w + 1, 0);
    while (!bit(e, j)) j++;
    int val = 0;
    for (int t = i; t >= j; t--) val = (val << 1) | (bit(e, t) ? 1 : 0);
    steps.push_back({pending + (i - j + 1), (val - 1) / 2});
    maxidx = std::max(maxidx, (val - 1) / 2);
    pending = 0;
    i = j - 1;
  }
  nodd = std::min(nodd, maxidx + 1);
  p.push_back(op(OP_KEEP, 0, 0));                       // slot 0 = b
  if (nodd > 1) {
    p.push_back(op(OP_SQR, 0, nodd));                   // slot nodd = b^2
    for (int k = 1; k < nodd; k++) p.push_back(op(OP_MUL, k == 1 ? 0 : nodd, k));
  }
  for (size_t s = 0; s < steps.size(); s++) {
    if (s == 0) { p.push_back(op(OP_LOAD, steps[s].idx, OP_NODST)); continue; }
    for (int k = 0; k < steps[s].nsq; k++) p.push_back(op(OP_SQR, 0, OP_NODST));
    p.push_back(op(OP_MUL, steps[s].idx, OP_NODST));
  }
  for (int k = 0; k < pending; k++) p.push_back(op(OP_SQR, 0, OP_NODST));
  *slots_used = nodd + 1;
  return p;
}

}  // namespace hbh
