// Shared internals of the C ABI translation units (not part of the public interface).
#pragma once
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/hebatch_b200.h"
#include "hb_host.h"
#include "mont32.cuh"

namespace hb {
struct ModDev {
  const uint32_t* n;    // modulus digits (L)
  const uint32_t* r1;   // R mod n
  const uint32_t* r2;   // R^2 mod n
  uint32_t np;          // -n^-1 mod 2^32
};
// Resident 128-thread blocks per SM the kernels are compiled for (register budget 128 or 168).
#ifndef HB_NS_BLOCKS
#define HB_NS_BLOCKS 2
#endif
__host__ __device__ constexpr int blocks_per_sm(int lpt) {
  return lpt > 32 ? HB_NS_BLOCKS : lpt > 24 ? 2 : lpt > 20 ? 3 : lpt <= 8 ? 6 : 4;
}
// Resident blocks per scheduler-quad for the encrypt / obfuscate kernel alone.  -DHB_SF32 (experiment): the (32,4)
// shape takes its multiplier operand from shared memory like (48,4) does, which frees 32 registers per thread and
// lets a third warp per scheduler fit (168 registers).
#ifdef HB_SF32
__host__ __device__ constexpr int enc_blocks_per_sm(int lpt) { return lpt == 32 ? 3 : blocks_per_sm(lpt); }
__host__ __device__ constexpr bool enc_stages_operand(int lpt) { return lpt == 48 || lpt == 32; }
#else
__host__ __device__ constexpr int enc_blocks_per_sm(int lpt) { return blocks_per_sm(lpt); }
__host__ __device__ constexpr bool enc_stages_operand(int lpt) { return lpt == 48; }
#endif
template <int LPT>
__device__ __forceinline__ void tile_store(uint32_t* tw, int e, const uint32_t (&x)[LPT]) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < LPT; k++) tw[(e * LPT + k) * 32 + lane] = x[k];
}
template <int LPT>
__device__ __forceinline__ void tile_load(const uint32_t* tw, int e, uint32_t (&x)[LPT]) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < LPT; k++) x[k] = tw[(e * LPT + k) * 32 + lane];
}

}  // namespace hb

using hbh::Big;

namespace hbi {

extern thread_local std::string g_err;
extern std::atomic<long long> g_launches;

inline int fail(int code, const std::string& msg) { g_err = msg; return code; }
// Montgomery digit-form arrays are moved 16 bytes at a time (Mont::load_limbs / store_limbs): every element is a
// multiple of 128 bytes, so only the base pointer can be off.
#define HB_REQUIRE_ALIGNED16(ptr, is_digit_form)                                                        \
  do { if ((is_digit_form) && (reinterpret_cast<uintptr_t>(ptr) & 15) != 0)                             \
    return hbi::fail(HB_ERR_ARG, "Montgomery digit-form arrays must be 16-byte aligned"); } while (0)

// The library's own stream-ordered memory pool on `device` (one per device and process, shared by the contexts on
// it).  Scratch never comes from the device's default pool, whose attributes belong to the application.
cudaMemPool_t device_pool(int device);
cudaError_t pool_alloc(cudaMemPool_t pool, void** p, size_t bytes, cudaStream_t stream);
#define CU(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) \
  return hbi::fail(HB_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); } while (0)

// Instantiated limb configurations, ordered by limb count L = LPT * TPI (capacity 32*L bits).
struct Cfg { int lpt, tpi; };
// 0..4: one throughput-oriented shape per limb count L = 32, 64, 96, 128, 192 (chosen by modulus size);
// 5..7: the same L with more lanes per number -- fewer multiplies per thread, so a launch that cannot fill the
// machine anyway finishes sooner (kernel_cfg picks by element count).  Digit-form arrays only depend on L.
// 8: L = 192 on four lanes for the encrypt / obfuscate kernel only (HB_DISPATCH_ENC): b staged in shared memory.
static const Cfg kCfgs[] = {{8, 4}, {16, 4}, {24, 4}, {32, 4}, {24, 8}, {8, 8}, {16, 8}, {8, 16}, {48, 4}};
constexpr int kNumCfg = 5;

inline int pick_cfg(int bits) {
  for (int i = 0; i < kNumCfg; i++)
    if (32 * kCfgs[i].lpt * kCfgs[i].tpi >= bits) return i;
  return -1;
}
inline int kernel_cfg(int base, long count) {
  if (base == 1 && count <= 14208) return 5;              // L = 64: (8, 8)
  if (base == 3) {
    if (count <= 7104) return 7;                          // L = 128: (8, 16)
    if (count <= 18944) return 6;                         //          (16, 8)
  }
  return base;
}
// Sliding-window width by exponent length: multiplications ~ bits / (w + 1) + 2^(w-1) table entries.  Six bits pay
// from 1024-bit exponents (measured +1.2 % encrypt, +1.3 % decrypt at 2048-bit keys over five); the 33-slot tables
// (160 MB for the persistent grid at 2048 bits) no longer fit the L2, which the measurement shows not to matter.
inline int window_for(int ebits) { return ebits >= 1024 ? 6 : ebits >= 768 ? 5 : ebits >= 160 ? 4 : ebits >= 24 ? 3 : 2; }

// Builder of the per-context constant block (one device allocation).
struct ConstBlock {
  std::vector<uint32_t> host;
  size_t add(const std::vector<uint32_t>& v) {
    size_t off = host.size();
    host.insert(host.end(), v.begin(), v.end());
    while (host.size() % 4) host.push_back(0);
    return off;
  }
};

struct ModOff { size_t n, r1, r2; uint32_t np; };

inline ModOff add_modulus(ConstBlock& cb, const Big& mod, int L) {
  ModOff m;
  Big one{1};
  m.n = cb.add(hbh::to_limbs(mod, L));
  m.r1 = cb.add(hbh::to_limbs(hbh::shl_mod(one, 32L * L, mod), L));
  m.r2 = cb.add(hbh::to_limbs(hbh::shl_mod(one, 2 * 32L * L, mod), L));
  m.np = hbh::neg_inv32(mod[0]);
  return m;
}

}  // namespace hbi

struct hb_ctx {
  int device = 0;
  int sms = 0;
  cudaMemPool_t pool = nullptr;       // the library's private stream-ordered pool on this device (hbi::device_pool)
  int opt_matvec_cbits = 0;           // HB_OPT_MATVEC_WINDOW_BITS: 0 = chosen by row count
  long opt_matvec_block = 0;          // HB_OPT_MATVEC_BLOCK_ROWS: 0 = 2^21
  bool sort_smem_set = false;         // k_bucket_sort's dynamic shared-memory limit raised on this device
  int key_bits = 0, wn = 0, wc = 0;
  Big n, n2;
  // public part
  int cfg_pub = -1;
  uint32_t* d_pub = nullptr;
  hbi::ModOff mod_n2;
  size_t off_nR = 0, off_prog_n = 0;
  size_t off_nR2 = 0, off_R3 = 0;     // n * R^2 mod n^2, R^3 mod n^2 (Montgomery-form results, see hb_kernels.cuh)
  size_t off_nwords = 0, off_negband = 0, off_maxint = 0, off_n2words = 0;   // n, n - n/3 (wn words); n^2 padded for k_root_inverse
  int nprog_n = 0, slots_n = 0;
  int maxint_top = 0;          // index of the highest non-zero word of max_int = n / 3
  int cfg_n = -1;              // limb shape for arithmetic mod n (plaintext side)
  hbi::ModOff mod_n_pub;
  // private part
  bool has_private = false;
  int cfg_priv = -1;
  uint32_t* d_priv = nullptr;
  size_t priv_bytes = 0;
  struct Half { hbi::ModOff s2, s1; size_t hiR2, hsR, prog; int nprog; } half[2];
  size_t off_qinvR = 0, off_qR = 0;
  hbi::ModOff mod_n_priv;
  int slots_priv = 0;
  // host-path staging (hb_encrypt_host / hb_decrypt_host): two stages of pinned + device buffers and window-table
  // scratch, kept across calls (grow-only) so a call costs no allocation once warm
  std::mutex mu;
  struct HostStage {
    cudaStream_t s = nullptr;
    cudaEvent_t done = nullptr;
    uint32_t *h_in0 = nullptr, *h_in1 = nullptr, *h_out = nullptr;
    uint32_t *d_in0 = nullptr, *d_in1 = nullptr, *d_out = nullptr, *d_tbl = nullptr;
    size_t hcap_in0 = 0, hcap_in1 = 0, hcap_out = 0;                 // bytes, pinned side
    size_t dcap_in0 = 0, dcap_in1 = 0, dcap_out = 0, dcap_tbl = 0;   // bytes, device side
  } stage[2];
};

namespace hbi {

inline hb::ModDev dev_mod(const uint32_t* base, const ModOff& m) {
  return hb::ModDev{base + m.n, base + m.r1, base + m.r2, m.np};
}

struct Launch { int blocks; int threads; size_t smem; long nwarps; int cfg; };
// `base` is the context's shape for the modulus; the launch uses the variant that suits `count` (l.cfg).
inline Launch plan(const hb_ctx* ctx, int base, long count, bool encrypt_kernel = false) {
  int cfg = kernel_cfg(base, count);
  if (encrypt_kernel && cfg == 4 && count > 14208) cfg = 8;      // L = 192 at throughput counts: (48, 4)
  const int tpi = kCfgs[cfg].tpi, lpt = kCfgs[cfg].lpt;
  const int ipw = 32 / tpi;
  long ntiles = (count + ipw - 1) / ipw;
  long nwarps = ntiles;
  const long maxw = (long)ctx->sms * (encrypt_kernel ? hb::enc_blocks_per_sm(lpt) : hb::blocks_per_sm(lpt)) * 4;
  if (nwarps > maxw) nwarps = maxw;
  if (nwarps < 1) nwarps = 1;
  // One warp per block (4 * blocks_per_sm of them resident per SM): the grid-stride tile loop of every kernel then
  // depends on blockIdx only, so the compiler knows the warp cannot diverge and emits bare SHFL instructions
  // instead of a WARPSYNC.COLLECTIVE / ENDCOLLECTIVE bracket around each of the three shuffles per row.
  Launch l;
  l.blocks = (int)nwarps;
  l.threads = 32;
  l.smem = 0;
  l.nwarps = nwarps;
  l.cfg = cfg;
  return l;
}

// Dynamic shared memory of the kernels that square through Mont::sqr (k_sqrmod; k_encrypt / k_decrypt under
// -DHB_USE_SQR): one warp per block.
template <int LPT, int TPI>
constexpr size_t sqr_smem_bytes() { return (size_t)hb::Mont<LPT, TPI>::SQ_WORDS * hb::Mont<LPT, TPI>::IPW * sizeof(uint32_t); }

#define HB_SQR_CASE(KERNEL, LPT_, TPI_, launch, stream, args)                                                  \
  {                                                                                                          \
    constexpr size_t smem_ = hbi::sqr_smem_bytes<LPT_, TPI_>();                                              \
    if (smem_ > 48 * 1024) {      /* per device, and cheap: set on every launch of this rarely used path */   \
      CU(cudaFuncSetAttribute(hb::KERNEL<LPT_, TPI_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_)); \
    }                                                                                                        \
    hb::KERNEL<LPT_, TPI_><<<launch.blocks, launch.threads, smem_, stream>>>(args);                          \
  }                                                                                                          \
  break;

// As HB_DISPATCH, for kernels that need the squaring scratch.
#define HB_DISPATCH_SQR(cfg, KERNEL, launch, stream, args)                                       \
  switch (launch.cfg) {                                                                          \
    case 0: HB_SQR_CASE(KERNEL, 8, 4, launch, stream, args)                                      \
    case 1: HB_SQR_CASE(KERNEL, 16, 4, launch, stream, args)                                     \
    case 2: HB_SQR_CASE(KERNEL, 24, 4, launch, stream, args)                                     \
    case 3: HB_SQR_CASE(KERNEL, 32, 4, launch, stream, args)                                     \
    case 4: HB_SQR_CASE(KERNEL, 24, 8, launch, stream, args)                                     \
    case 5: HB_SQR_CASE(KERNEL, 8, 8, launch, stream, args)                                      \
    case 6: HB_SQR_CASE(KERNEL, 16, 8, launch, stream, args)                                     \
    case 7: HB_SQR_CASE(KERNEL, 8, 16, launch, stream, args)                                     \
    default: return hbi::fail(HB_ERR_UNSUPPORTED, "no limb configuration");                      \
  }                                                                                              \
  hbi::g_launches++;

// The modular-power kernels only need the scratch when they are built to square through Mont::sqr.
#ifdef HB_USE_SQR
#define HB_DISPATCH_POW HB_DISPATCH_SQR
#else
#define HB_DISPATCH_POW HB_DISPATCH
#endif

// k_encrypt: the nine shapes; (48, 4) takes its operand staging area and the modulus copy as dynamic shared memory.
#ifdef HB_SF32
#define HB_ENC_SF32_CASE(KERNEL, launch, stream, args)                                                  \
  if (launch.cfg == 3) {                                                                                \
    hb::KERNEL<32, 4><<<launch.blocks, launch.threads,                                                  \
                        hb::Mont<32, 4>::NS_SMEM_WORDS * sizeof(uint32_t), stream>>>(args);               \
    hbi::g_launches++;                                                                                  \
  } else
#else
#define HB_ENC_SF32_CASE(KERNEL, launch, stream, args)
#endif
#define HB_DISPATCH_ENC(cfg, KERNEL, launch, stream, args)                                              \
  HB_ENC_SF32_CASE(KERNEL, launch, stream, args)                                                        \
  if (launch.cfg == 8) {                                                                                \
    hb::KERNEL<48, 4><<<launch.blocks, launch.threads,                                                  \
                        hb::Mont<48, 4>::NS_SMEM_WORDS * sizeof(uint32_t), stream>>>(args);               \
    hbi::g_launches++;                                                                                  \
  } else {                                                                                              \
    HB_DISPATCH_POW(cfg, KERNEL, launch, stream, args)                                                  \
  }

#if defined(HB_DEV_ONLY_2048)   /* development builds: only the shapes a 2048-bit key uses at throughput counts */
#define HB_DISPATCH(cfg, KERNEL, launch, stream, args)                                           \
  switch (launch.cfg) {                                                                                 \
    case 1: hb::KERNEL<16, 4><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    case 3: hb::KERNEL<32, 4><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    default: return hbi::fail(HB_ERR_UNSUPPORTED, "no limb configuration");                            \
  }                                                                                              \
  hbi::g_launches++;
#elif defined(HB_DEV_ONLY_3072)   /* development builds: only the shapes a 3072-bit key uses, for quick A/B experiments */
#define HB_DISPATCH(cfg, KERNEL, launch, stream, args)                                           \
  switch (launch.cfg) {                                                                                 \
    case 2: hb::KERNEL<24, 4><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    case 4: hb::KERNEL<24, 8><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    default: return hbi::fail(HB_ERR_UNSUPPORTED, "no limb configuration");                            \
  }                                                                                              \
  hbi::g_launches++;
#else
#define HB_DISPATCH(cfg, KERNEL, launch, stream, args)                                           \
  switch (launch.cfg) {                                                                                 \
    case 0: hb::KERNEL<8, 4><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break;  \
    case 1: hb::KERNEL<16, 4><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    case 2: hb::KERNEL<24, 4><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    case 3: hb::KERNEL<32, 4><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    case 4: hb::KERNEL<24, 8><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    case 5: hb::KERNEL<8, 8><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break;  \
    case 6: hb::KERNEL<16, 8><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    case 7: hb::KERNEL<8, 16><<<launch.blocks, launch.threads, launch.smem, stream>>>(args); break; \
    default: return hbi::fail(HB_ERR_UNSUPPORTED, "no limb configuration");                            \
  }                                                                                              \
  hbi::g_launches++;
#endif

}  // namespace hbi
