// C ABI of the B200 homomorphic-operator library (include/hebatch_b200.h): key contexts and the
// encrypt / obfuscate / decrypt / mulmod entry points.
#include "hb_ctx.h"
#include "hb_kernels.cuh"

using hbh::Big;
using namespace hbi;

namespace hbi {
thread_local std::string g_err;
std::atomic<long long> g_launches{0};

namespace {
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};
}
// Window tables (160 MB for a full encrypt grid at 2048 bits) and the matvec scratch (GBs at 1 M rows) are taken
// per call.  Blocks freed by a call stay in the pool up to this many bytes across synchronisations, so that a loop
// of small calls allocates nothing; what lies beyond goes back to the driver, leaving the memory to the
// application's own allocator (torch's caching allocator holds the batches themselves).
constexpr unsigned long long kPoolKeepDefault = 1ull << 30;

cudaMemPool_t device_pool(int device) {
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (g_pools[device]) return g_pools[device];
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  // Freed scratch kept across synchronisations: 1 GiB, or an eighth of the device's memory when that is more
  // (22 GiB on a 180 GB B200).  A 1M-row encrypted matvec takes 9 GB of bucket scratch per call and the scalar
  // powers of the same FLR iteration another 3 GB; with less kept, every call pays the driver for fresh physical
  // memory (measured: 2.2 s against 1.8 s per 1M x 100 matvec with 1 GiB kept; inside a 1M-row FLR iteration
  // 2.29 s per matvec with 11 GiB kept, 2.03 s with 40 GiB).
  unsigned long long keep = kPoolKeepDefault;
  size_t free_b = 0, total_b = 0;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cudaSetDevice(device) == cudaSuccess && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess)
    keep = std::max<unsigned long long>(keep, (unsigned long long)total_b / 8);
  if (cur >= 0) cudaSetDevice(cur);
  cudaGetLastError();
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  g_pools[device] = pool;
  return pool;
}
cudaError_t pool_alloc(cudaMemPool_t pool, void** p, size_t bytes, cudaStream_t stream) {
  return cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, stream);
}
}

namespace {

// Words of window-table scratch a launch of `count` elements needs (per-warp tiles, see hb_kernels.cuh).
size_t table_words(const hb_ctx* ctx, int base_cfg, int slots, int64_t count, bool encrypt_kernel) {
  Launch l = plan(ctx, base_cfg, count, encrypt_kernel);
  return (size_t)(slots + 1) * kCfgs[l.cfg].lpt * 32 * l.nwarps;
}

int encrypt_common(hb_ctx* ctx, const uint32_t* m, const uint32_t* c, const uint32_t* r, uint32_t* out,
                   int64_t count, int mode, void* stream_, uint32_t* tbl_ext = nullptr, int flags = 0) {
  if (!ctx || !r || !out || (mode == 0 ? !m : !c)) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  HB_REQUIRE_ALIGNED16(c, mode == 1 && (flags & HB_A_MONT));
  HB_REQUIRE_ALIGNED16(out, flags & HB_OUT_MONT);
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_pub;
  Launch l = plan(ctx, cfg, count, true);
  const long stride = (long)(ctx->slots_n + 1) * kCfgs[l.cfg].lpt * 32;
  uint32_t* tbl = tbl_ext;
  if (!tbl) CU(pool_alloc(ctx->pool, (void**)&tbl, (size_t)stride * l.nwarps * sizeof(uint32_t), stream));
  hb::EncArgs A;
  A.mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  A.c_mont = (flags & HB_A_MONT) ? 1 : 0;
  A.out_mont = (flags & HB_OUT_MONT) ? 1 : 0;
  A.nR = ctx->d_pub + (A.out_mont ? ctx->off_nR2 : ctx->off_nR);
  A.prog = ctx->d_pub + ctx->off_prog_n;
  A.nprog = ctx->nprog_n;
  A.tbl = tbl;
  A.tbl_stride = stride;
  A.m = m; A.c = c; A.r = r; A.out = out;
  A.count = count; A.wn = ctx->wn; A.wc = ctx->wc; A.mode = mode;
  HB_DISPATCH_ENC(cfg, k_encrypt, l, stream, A)
  CU(cudaGetLastError());
  if (!tbl_ext) CU(cudaFreeAsync(tbl, stream));
  return HB_OK;
}

int mulmod_common(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                  int lift, int bcast, void* stream_, int flags = 0) {
  if (!ctx || !a || !b || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_pub;
  Launch l = plan(ctx, cfg, count);
  hb::MulArgs A;
  A.mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  A.nR = ctx->d_pub + ctx->off_nR;
  A.nR2 = ctx->d_pub + ctx->off_nR2;
  A.r3 = ctx->d_pub + ctx->off_R3;
  A.a = a; A.b = b; A.out = out; A.count = count; A.wn = ctx->wn; A.wc = ctx->wc;
  A.lift = lift; A.b_broadcast = bcast;
  A.a_mont = (flags & HB_A_MONT) ? 1 : 0;
  A.b_mont = (!lift && (flags & HB_B_MONT)) ? 1 : 0;
  A.out_mont = (flags & HB_OUT_MONT) ? 1 : 0;
  HB_REQUIRE_ALIGNED16(a, A.a_mont);
  HB_REQUIRE_ALIGNED16(b, A.b_mont);
  HB_REQUIRE_ALIGNED16(out, A.out_mont);
  HB_DISPATCH(cfg, k_mulmod, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
}

}  // namespace

extern "C" {

const char* hb_last_error(void) { return g_err.c_str(); }
const char* hb_version(void) { return "hebatch_b200 0.1 (sm_100a)"; }
int64_t hb_launch_count(void) { return g_launches.load(); }

int hb_ctx_create(hb_ctx** out, const uint32_t* n_words, int n_nwords, int device) {
  if (!out || !n_words || n_nwords <= 0) return fail(HB_ERR_ARG, "null pointer");
  Big n = hbh::from_words(n_words, n_nwords);
  if (hbh::bitlen(n) < 3 || !(n[0] & 1)) return fail(HB_ERR_ARG, "modulus must be odd and >= 5");
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(HB_ERR_CUDA, "no such CUDA device");
  CU(cudaSetDevice(device));
  cudaMemPool_t pool = device_pool(device);
  if (!pool) return fail(HB_ERR_CUDA, "cannot create the library's memory pool on this device");
  hb_ctx* ctx = new hb_ctx();
  ctx->device = device;
  ctx->pool = pool;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) { delete ctx; return fail(HB_ERR_CUDA, cudaGetErrorString(e)); }
  ctx->sms = prop.multiProcessorCount;
  ctx->n = n;
  ctx->n2 = hbh::mul(n, n);
  ctx->key_bits = hbh::bitlen(n);
  ctx->wn = (ctx->key_bits + 31) / 32;
  ctx->wc = ((2 * ctx->key_bits + 7) / 8 + 3) / 4;
  ctx->cfg_pub = pick_cfg(hbh::bitlen(ctx->n2));
  if (ctx->cfg_pub < 0) { delete ctx; return fail(HB_ERR_UNSUPPORTED, "key too large for the instantiated limb configurations"); }
  const int L = kCfgs[ctx->cfg_pub].lpt * kCfgs[ctx->cfg_pub].tpi;
  ConstBlock cb;
  ctx->mod_n2 = add_modulus(cb, ctx->n2, L);
  ctx->off_nR = cb.add(hbh::to_limbs(hbh::shl_mod(n, 32L * L, ctx->n2), L));
  ctx->off_nR2 = cb.add(hbh::to_limbs(hbh::shl_mod(n, 2 * 32L * L, ctx->n2), L));
  {
    Big one{1};
    ctx->off_R3 = cb.add(hbh::to_limbs(hbh::shl_mod(one, 3 * 32L * L, ctx->n2), L));
  }
  ctx->cfg_n = pick_cfg(ctx->key_bits);
  ctx->mod_n_pub = add_modulus(cb, n, kCfgs[ctx->cfg_n].lpt * kCfgs[ctx->cfg_n].tpi);
  std::vector<uint32_t> prog = hbh::build_program(n, window_for(ctx->key_bits), &ctx->slots_n);
  ctx->nprog_n = (int)prog.size();
  ctx->off_prog_n = cb.add(prog);
  {
    std::vector<uint32_t> nw(n.begin(), n.end());
    nw.resize(ctx->wn, 0);
    ctx->off_nwords = cb.add(nw);
    // neg_band = n - n / 3  (operators.py:250); n / 3 by schoolbook short division
    Big third(n.size(), 0);
    uint64_t rem = 0;
    for (int i = (int)n.size() - 1; i >= 0; i--) {
      uint64_t cur = (rem << 32) | n[i];
      third[i] = (uint32_t)(cur / 3);
      rem = cur % 3;
    }
    {
      Big mi = third;
      mi.resize(ctx->wn, 0);
      ctx->off_maxint = cb.add(mi);
      ctx->maxint_top = 0;
      for (int i = 0; i < ctx->wn; i++) if (mi[i]) ctx->maxint_top = i;
    }
    Big nb = n;
    hbh::sub_in(nb, third);
    nb.resize(ctx->wn, 0);
    ctx->off_negband = cb.add(nb);
    const int T = 32 * (L / 32 + 1);
    std::vector<uint32_t> n2w(ctx->n2.begin(), ctx->n2.end());
    n2w.resize(T, 0);
    ctx->off_n2words = cb.add(n2w);
  }
  e = cudaMalloc(&ctx->d_pub, cb.host.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_pub, cb.host.data(), cb.host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { delete ctx; return fail(HB_ERR_CUDA, cudaGetErrorString(e)); }
  *out = ctx;
  return HB_OK;
}

int hb_ctx_set_private(hb_ctx* ctx, const uint32_t* p_, const uint32_t* q_, const uint32_t* hp_,
                       const uint32_t* hq_, const uint32_t* qinv_, int nwords) {
  if (!ctx || !p_ || !q_ || !hp_ || !hq_ || !qinv_ || nwords <= 0) return fail(HB_ERR_ARG, "null pointer");
  Big p = hbh::from_words(p_, nwords), q = hbh::from_words(q_, nwords);
  Big hs[2] = {hbh::from_words(hp_, nwords), hbh::from_words(hq_, nwords)};
  Big qinv = hbh::from_words(qinv_, nwords);
  if (hbh::cmp(hbh::mul(p, q), ctx->n) != 0) return fail(HB_ERR_ARG, "p * q does not match n");
  if (!(p[0] & 1) || !(q[0] & 1)) return fail(HB_ERR_ARG, "primes must be odd");
  if (hbh::cmp(hs[0], p) >= 0 || hbh::cmp(hs[1], q) >= 0 || hbh::cmp(qinv, p) >= 0) return fail(HB_ERR_ARG, "private constants out of range");
  CU(cudaSetDevice(ctx->device));
  Big s[2] = {p, q};
  Big s2[2] = {hbh::mul(p, p), hbh::mul(q, q)};
  const int wlo = ctx->wc / 2;
  int need = std::max(std::max(hbh::bitlen(s2[0]), hbh::bitlen(s2[1])), ctx->key_bits);
  need = std::max(need, 32 * std::max(wlo, ctx->wc - wlo));
  int cfg = pick_cfg(need);
  if (cfg < 0) return fail(HB_ERR_UNSUPPORTED, "key too large for the instantiated limb configurations");
  const int L = kCfgs[cfg].lpt * kCfgs[cfg].tpi;
  ConstBlock cb;
  Big one{1};
  int slots = 0;
  for (int h = 0; h < 2; h++) {
    ctx->half[h].s2 = add_modulus(cb, s2[h], L);
    ctx->half[h].s1 = add_modulus(cb, s[h], L);
    ctx->half[h].hiR2 = cb.add(hbh::to_limbs(hbh::shl_mod(one, 32L * wlo + 2 * 32L * L, s2[h]), L));
    ctx->half[h].hsR = cb.add(hbh::to_limbs(hbh::shl_mod(hs[h], 32L * L, s[h]), L));
    Big e = hbh::sub_small(s[h], 1);
    int used = 0;
    std::vector<uint32_t> prog = hbh::build_program(e, window_for(hbh::bitlen(e)), &used);
    slots = std::max(slots, used);
    ctx->half[h].nprog = (int)prog.size();
    ctx->half[h].prog = cb.add(prog);
  }
  ctx->off_qinvR = cb.add(hbh::to_limbs(hbh::shl_mod(qinv, 32L * L, p), L));
  ctx->mod_n_priv = add_modulus(cb, ctx->n, L);
  ctx->off_qR = cb.add(hbh::to_limbs(hbh::shl_mod(q, 32L * L, ctx->n), L));
  ctx->slots_priv = slots;
  if (ctx->d_priv) { cudaMemset(ctx->d_priv, 0, ctx->priv_bytes); cudaFree(ctx->d_priv); ctx->d_priv = nullptr; }
  ctx->priv_bytes = cb.host.size() * sizeof(uint32_t);
  CU(cudaMalloc(&ctx->d_priv, ctx->priv_bytes));
  CU(cudaMemcpy(ctx->d_priv, cb.host.data(), cb.host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  ctx->cfg_priv = cfg;
  ctx->has_private = true;
  return HB_OK;
}

static void release_stages(hb_ctx* ctx);

void hb_ctx_destroy(hb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  release_stages(ctx);
  if (ctx->d_pub) cudaFree(ctx->d_pub);
  if (ctx->d_priv) {                  // private constants do not outlive the context in HBM
    cudaMemset(ctx->d_priv, 0, ctx->priv_bytes);
    cudaFree(ctx->d_priv);
  }
  delete ctx;
}

int hb_ctx_set_option(hb_ctx* ctx, int option, int64_t value) {
  if (!ctx) return fail(HB_ERR_ARG, "null pointer");
  switch (option) {
    case HB_OPT_MATVEC_WINDOW_BITS:
      if (value != 0 && (value < 2 || value > 13)) return fail(HB_ERR_ARG, "matvec window must be 0 (auto) or 2..13 bits");
      ctx->opt_matvec_cbits = (int)value;
      return HB_OK;
    case HB_OPT_MATVEC_BLOCK_ROWS:
      if (value < 0) return fail(HB_ERR_ARG, "negative block size");
      ctx->opt_matvec_block = (long)value;
      return HB_OK;
    case HB_OPT_POOL_KEEP_BYTES: {
      if (value < 0) return fail(HB_ERR_ARG, "negative pool threshold");
      CU(cudaSetDevice(ctx->device));
      unsigned long long keep = (unsigned long long)value;
      CU(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep));
      return HB_OK;
    }
    default:
      return fail(HB_ERR_ARG, "unknown option");
  }
}

int hb_pt_words(const hb_ctx* ctx) { return ctx ? ctx->wn : 0; }
int hb_ct_words(const hb_ctx* ctx) { return ctx ? ctx->wc : 0; }
int hb_key_bits(const hb_ctx* ctx) { return ctx ? ctx->key_bits : 0; }

int hb_encrypt(hb_ctx* ctx, const uint32_t* m, const uint32_t* r, uint32_t* out, int64_t count, void* stream) {
  return encrypt_common(ctx, m, nullptr, r, out, count, 0, stream);
}
int hb_obfuscate(hb_ctx* ctx, const uint32_t* c, const uint32_t* r, uint32_t* out, int64_t count, void* stream) {
  return encrypt_common(ctx, nullptr, c, r, out, count, 1, stream);
}
int hb_encrypt_rep(hb_ctx* ctx, const uint32_t* m, const uint32_t* r, uint32_t* out, int64_t count, int flags,
                   void* stream) {
  return encrypt_common(ctx, m, nullptr, r, out, count, 0, stream, nullptr, flags & HB_OUT_MONT);
}
int hb_obfuscate_rep(hb_ctx* ctx, const uint32_t* c, const uint32_t* r, uint32_t* out, int64_t count, int flags,
                     void* stream) {
  return encrypt_common(ctx, nullptr, c, r, out, count, 1, stream, nullptr, flags & (HB_A_MONT | HB_OUT_MONT));
}
int hb_mulmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
              int b_broadcast, void* stream) {
  return mulmod_common(ctx, a, b, out, count, 0, b_broadcast, stream);
}
int hb_lift_mulmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* m, uint32_t* out, int64_t count,
                   int m_broadcast, void* stream) {
  return mulmod_common(ctx, a, m, out, count, 1, m_broadcast, stream);
}
int hb_mulmod_rep(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                  int b_broadcast, int flags, void* stream) {
  return mulmod_common(ctx, a, b, out, count, 0, b_broadcast, stream, flags);
}
int hb_lift_mulmod_rep(hb_ctx* ctx, const uint32_t* a, const uint32_t* m, uint32_t* out, int64_t count,
                       int m_broadcast, int flags, void* stream) {
  return mulmod_common(ctx, a, m, out, count, 1, m_broadcast, stream, flags);
}

int hb_fore_gradient(hb_ctx* ctx, const uint32_t* c, const uint32_t* lg, const uint32_t* kg, uint32_t kh,
                     const uint32_t* yl, const uint32_t* r, uint32_t* out, int64_t count, int flags,
                     void* stream_) {
  if (!ctx || !c || !lg || !kg || !yl || !r || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (kh < 1) return fail(HB_ERR_ARG, "the ciphertext exponent must be at least 1");
  if (count == 0) return HB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_pub;
  Launch l = plan(ctx, cfg, count, true);
  const int spare = ctx->slots_n;                       // table slots [0, slots_n) belong to the exponent program
  const long stride = (long)(spare + 2) * kCfgs[l.cfg].lpt * 32;
  uint32_t* tbl = nullptr;
  CU(pool_alloc(ctx->pool, (void**)&tbl, (size_t)stride * l.nwarps * sizeof(uint32_t), stream));
  hb::ForeArgs A;
  A.mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  A.nR2 = ctx->d_pub + ctx->off_nR2;
  A.prog = ctx->d_pub + ctx->off_prog_n;
  A.nprog = ctx->nprog_n;
  A.tbl = tbl; A.tbl_stride = stride; A.spare = spare;
  A.lg = lg; A.kg = kg; A.c = c; A.yl = yl; A.r = r; A.out = out; A.kh = kh;
  A.count = count; A.wn = ctx->wn; A.wc = ctx->wc;
  A.c_mont = (flags & HB_A_MONT) ? 1 : 0;
  A.out_mont = (flags & HB_OUT_MONT) ? 1 : 0;
  HB_REQUIRE_ALIGNED16(c, A.c_mont);
  HB_REQUIRE_ALIGNED16(out, A.out_mont);
  HB_DISPATCH_ENC(cfg, k_fore_gradient, l, stream, A)
  CU(cudaGetLastError());
  CU(cudaFreeAsync(tbl, stream));
  return HB_OK;
}

static int plain_common(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                        int op, int bcast, void* stream_) {
  if (!ctx || !a || !b || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_n;
  Launch l = plan(ctx, cfg, count);
  hb::PlainArgs A;
  A.mod = dev_mod(ctx->d_pub, ctx->mod_n_pub);
  A.a = a; A.b = b; A.out = out; A.count = count; A.w = ctx->wn; A.op = op; A.b_broadcast = bcast;
  HB_DISPATCH(cfg, k_plainop, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
}

int hb_plain_mulmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                    int b_broadcast, void* stream) {
  return plain_common(ctx, a, b, out, count, 0, b_broadcast, stream);
}
int hb_plain_addmod(hb_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, void* stream) {
  return plain_common(ctx, a, b, out, count, 1, 0, stream);
}

int hb_sqrmod(hb_ctx* ctx, const uint32_t* a, uint32_t* out, int64_t count, int reps, int throughput_shape,
              void* stream_) {
  if (!ctx || !a || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0 || reps < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_pub;
  Launch l = plan(ctx, cfg, throughput_shape ? (int64_t)1 << 40 : count);
  {
    const int ipw = 32 / kCfgs[l.cfg].tpi;
    long blocks = (count + ipw - 1) / ipw;                 // one warp (tile) per block
    if (blocks < l.blocks) l.blocks = (int)std::max(blocks, 1L);
  }
  hb::SqrArgs A;
  A.mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  A.a = a; A.out = out; A.count = count; A.wc = ctx->wc; A.reps = reps;
#if defined(HB_DEV_ONLY_3072) || defined(HB_DEV_ONLY_2048)
  return fail(HB_ERR_UNSUPPORTED, "development build");
#else
  HB_DISPATCH_SQR(cfg, k_sqrmod, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
#endif
}

static int decrypt_common(hb_ctx* ctx, const uint32_t* c, uint32_t* m_out, int64_t count, void* stream_,
                          uint32_t* tbl_ext, int c_mont = 0) {
  if (!ctx || !c || !m_out) return fail(HB_ERR_ARG, "null pointer");
  if (!ctx->has_private) return fail(HB_ERR_NOPRIVATE, "context has no private key");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_priv;
  Launch l = plan(ctx, cfg, count);
  const long stride = (long)(ctx->slots_priv + 1) * kCfgs[l.cfg].lpt * 32;
  uint32_t* tbl = tbl_ext;
  if (!tbl) CU(pool_alloc(ctx->pool, (void**)&tbl, (size_t)stride * l.nwarps * sizeof(uint32_t), stream));
  const uint32_t* base = ctx->d_priv;
  hb::DecArgs A;
  for (int h = 0; h < 2; h++) {
    A.half[h].s2 = dev_mod(base, ctx->half[h].s2);
    A.half[h].s1 = dev_mod(base, ctx->half[h].s1);
    A.half[h].hiR2 = base + ctx->half[h].hiR2;
    A.half[h].hsR = base + ctx->half[h].hsR;
    A.half[h].prog = base + ctx->half[h].prog;
    A.half[h].nprog = ctx->half[h].nprog;
  }
  A.qinvR = base + ctx->off_qinvR;
  A.modn = dev_mod(base, ctx->mod_n_priv);
  A.qR = base + ctx->off_qR;
  A.tbl = tbl; A.tbl_stride = stride; A.stash_slot = ctx->slots_priv;
  A.c = c; A.out = m_out; A.count = count; A.wn = ctx->wn; A.wc = ctx->wc;
  A.c_mont = c_mont;
  HB_DISPATCH_POW(cfg, k_decrypt, l, stream, A)
  CU(cudaGetLastError());
  if (!tbl_ext) CU(cudaFreeAsync(tbl, stream));
  return HB_OK;
}

int hb_decrypt(hb_ctx* ctx, const uint32_t* c, uint32_t* m_out, int64_t count, void* stream) {
  return decrypt_common(ctx, c, m_out, count, stream, nullptr);
}

int hb_decrypt_rep(hb_ctx* ctx, const uint32_t* c, uint32_t* m_out, int64_t count, int flags, void* stream_) {
  if (!(flags & HB_A_MONT)) return decrypt_common(ctx, c, m_out, count, stream_, nullptr);
  if (!ctx || !c || !m_out) return fail(HB_ERR_ARG, "null pointer");
  if (!ctx->has_private) return fail(HB_ERR_NOPRIVATE, "context has no private key");
  if (count <= 0) return count == 0 ? HB_OK : fail(HB_ERR_ARG, "negative count");
  HB_REQUIRE_ALIGNED16(c, true);
  const int Lpub = kCfgs[ctx->cfg_pub].lpt * kCfgs[ctx->cfg_pub].tpi;
  const int Lpriv = kCfgs[ctx->cfg_priv].lpt * kCfgs[ctx->cfg_priv].tpi;
  // the kernel reads the digit form directly when the n^2 context's R is the square of the p^2 / q^2 context's
  // (every standard key size); other shapes go through plain words first
  if (Lpub == 2 * Lpriv)
    return decrypt_common(ctx, c, m_out, count, stream_, nullptr, 1);
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  uint32_t* words = nullptr;
  CU(pool_alloc(ctx->pool, (void**)&words, (size_t)count * ctx->wc * sizeof(uint32_t), stream));
  int rc = hb_ct_convert(ctx, c, words, count, 0, stream_);
  if (rc == HB_OK) rc = decrypt_common(ctx, words, m_out, count, stream_, nullptr);
  cudaFreeAsync(words, stream);
  return rc;
}

// ---- host-buffer path: pinned staging + two side streams, chunks double-buffered ------------------
// The stages live in the context and only ever grow, so a warm call allocates nothing: pinned allocations cost
// milliseconds each, and a stream-ordered allocation of the 80 MB window-table scratch per chunk on alternating
// streams defeats the pool's reuse.
static int grow(void** p, size_t* cap, size_t need, bool pinned) {
  if (*cap >= need) return HB_OK;
  if (*p) { if (pinned) cudaFreeHost(*p); else cudaFree(*p); *p = nullptr; *cap = 0; }
  const size_t want = need + need / 8;
  cudaError_t e = pinned ? cudaMallocHost(p, want) : cudaMalloc(p, want);
  if (e != cudaSuccess) return fail(HB_ERR_CUDA, std::string("staging allocation: ") + cudaGetErrorString(e));
  *cap = want;
  return HB_OK;
}

static void release_stages(hb_ctx* ctx) {
  for (auto& s : ctx->stage) {
    if (s.s) cudaStreamSynchronize(s.s);
    if (s.h_in0) cudaFreeHost(s.h_in0);
    if (s.h_in1) cudaFreeHost(s.h_in1);
    if (s.h_out) cudaFreeHost(s.h_out);
    if (s.d_in0) cudaFree(s.d_in0);
    if (s.d_in1) cudaFree(s.d_in1);
    if (s.d_out) cudaFree(s.d_out);
    if (s.d_tbl) cudaFree(s.d_tbl);
    if (s.done) cudaEventDestroy(s.done);
    if (s.s) cudaStreamDestroy(s.s);
    s = hb_ctx::HostStage();
  }
}

static int host_pipeline(hb_ctx* ctx, int kind, const uint32_t* in0, const uint32_t* in1, uint32_t* out,
                         int64_t count) {
  // kind 0: encrypt(in0 = m [wn], in1 = r [wn]) -> out [wc];  kind 1: decrypt(in0 = c [wc]) -> out [wn]
  if (!ctx || !in0 || !out || (kind == 0 && !in1)) return fail(HB_ERR_ARG, "null pointer");
  if (count <= 0) return count == 0 ? HB_OK : fail(HB_ERR_ARG, "negative count");
  std::lock_guard<std::mutex> lock(ctx->mu);
  CU(cudaSetDevice(ctx->device));
  const size_t w_in0 = kind == 0 ? ctx->wn : ctx->wc, w_in1 = kind == 0 ? ctx->wn : 0;
  const size_t w_out = kind == 0 ? ctx->wc : ctx->wn;
  const int cfg = kind == 0 ? ctx->cfg_pub : ctx->cfg_priv;
  if (cfg < 0) return fail(HB_ERR_NOPRIVATE, "context has no private key");
  const int slots = kind == 0 ? ctx->slots_n : ctx->slots_priv;
  // four full waves of the persistent grid per chunk, so chunking costs no tail
  const int tcfg = plan(ctx, cfg, (int64_t)1 << 40, kind == 0).cfg;      // the shape a full chunk runs in
  const int64_t wave = (int64_t)ctx->sms * 4 * hb::blocks_per_sm(kCfgs[tcfg].lpt) * (32 / kCfgs[tcfg].tpi);
  const int64_t chunk = std::min<int64_t>(count, 4 * wave);
  const int nst = count > chunk ? 2 : 1;
  const int64_t nchunks = (count + chunk - 1) / chunk;
  const int64_t last = count - (nchunks - 1) * chunk;
  const size_t tbl_bytes =
      sizeof(uint32_t) * std::max(table_words(ctx, cfg, slots, chunk, kind == 0), table_words(ctx, cfg, slots, last, kind == 0));
  for (int i = 0; i < nst; i++) {
    hb_ctx::HostStage& s = ctx->stage[i];
    if (!s.s) CU(cudaStreamCreateWithFlags(&s.s, cudaStreamNonBlocking));
    if (!s.done) CU(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    CU(cudaStreamSynchronize(s.s));
    int rc = grow((void**)&s.h_in0, &s.hcap_in0, chunk * w_in0 * 4, true);
    if (!rc) rc = grow((void**)&s.d_in0, &s.dcap_in0, chunk * w_in0 * 4, false);
    if (!rc && w_in1) rc = grow((void**)&s.h_in1, &s.hcap_in1, chunk * w_in1 * 4, true);
    if (!rc && w_in1) rc = grow((void**)&s.d_in1, &s.dcap_in1, chunk * w_in1 * 4, false);
    if (!rc) rc = grow((void**)&s.h_out, &s.hcap_out, chunk * w_out * 4, true);
    if (!rc) rc = grow((void**)&s.d_out, &s.dcap_out, chunk * w_out * 4, false);
    if (!rc) rc = grow((void**)&s.d_tbl, &s.dcap_tbl, tbl_bytes, false);
    if (rc) return rc;
  }
  auto drain = [&]() { for (int i = 0; i < nst; i++) cudaStreamSynchronize(ctx->stage[i].s); };
#define CUX(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { drain(); \
  return fail(HB_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); } } while (0)
  struct Pending { int64_t off, n; bool active; } pend[2] = {{0, 0, false}, {0, 0, false}};
  for (int64_t i = 0; i < nchunks + nst; i++) {
    const int which = (int)(i % nst);
    hb_ctx::HostStage& s = ctx->stage[which];
    if (pend[which].active) {   // drain the chunk this stage submitted nst iterations ago
      CUX(cudaEventSynchronize(s.done));
      memcpy(out + pend[which].off * w_out, s.h_out, pend[which].n * w_out * 4);
      pend[which].active = false;
    }
    if (i >= nchunks) continue;
    const int64_t off = i * chunk, n = std::min(chunk, count - off);
    memcpy(s.h_in0, in0 + off * w_in0, n * w_in0 * 4);
    CUX(cudaMemcpyAsync(s.d_in0, s.h_in0, n * w_in0 * 4, cudaMemcpyHostToDevice, s.s));
    if (w_in1) {
      memcpy(s.h_in1, in1 + off * w_in1, n * w_in1 * 4);
      CUX(cudaMemcpyAsync(s.d_in1, s.h_in1, n * w_in1 * 4, cudaMemcpyHostToDevice, s.s));
    }
    const int rc = kind == 0 ? encrypt_common(ctx, s.d_in0, nullptr, s.d_in1, s.d_out, n, 0, s.s, s.d_tbl)
                             : decrypt_common(ctx, s.d_in0, s.d_out, n, s.s, s.d_tbl);
    if (rc != HB_OK) { drain(); return rc; }
    CUX(cudaMemcpyAsync(s.h_out, s.d_out, n * w_out * 4, cudaMemcpyDeviceToHost, s.s));
    CUX(cudaEventRecord(s.done, s.s));
    pend[which] = {off, n, true};
  }
#undef CUX
  return HB_OK;
}

int hb_encrypt_host(hb_ctx* ctx, const uint32_t* m, const uint32_t* r, uint32_t* out, int64_t count) {
  return host_pipeline(ctx, 0, m, r, out, count);
}
int hb_decrypt_host(hb_ctx* ctx, const uint32_t* c, uint32_t* m_out, int64_t count) {
  return host_pipeline(ctx, 1, c, nullptr, m_out, count);
}

}  // extern "C"
