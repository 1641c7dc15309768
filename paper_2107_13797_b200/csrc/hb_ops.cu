// C ABI, second translation unit: hb_powscalar, hb_product, hb_matvec and their device-side helpers
// (batch modular inversion, bucket-method multi-exponentiation).
#include <cstdlib>
#include "hb_ctx.h"
#include "hb_ops.cuh"

using namespace hbi;

namespace {

// stream-ordered scratch with automatic release
struct Scratch {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() { for (void* p : ptrs) cudaFreeAsync(p, s); }
  template <typename T>
  cudaError_t get(T** out, size_t n) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, (n ? n : 1) * sizeof(T), s);
    if (e == cudaSuccess) { ptrs.push_back(p); *out = (T*)p; }
    return e;
  }
};

inline int Ldig(int cfg) { return kCfgs[cfg].lpt * kCfgs[cfg].tpi; }

#define HB_DISPATCH1(cfg, KERNEL, stream, args)                                      \
  switch (cfg) {                                                                     \
    case 0: hb::KERNEL<8, 4><<<1, 32, 0, stream>>>(args); break;                     \
    case 1: hb::KERNEL<16, 4><<<1, 32, 0, stream>>>(args); break;                    \
    case 2: hb::KERNEL<24, 4><<<1, 32, 0, stream>>>(args); break;                    \
    case 3: hb::KERNEL<32, 4><<<1, 32, 0, stream>>>(args); break;                    \
    case 4: hb::KERNEL<24, 8><<<1, 32, 0, stream>>>(args); break;                    \
    case 5: hb::KERNEL<8, 8><<<1, 32, 0, stream>>>(args); break;                     \
    case 6: hb::KERNEL<16, 8><<<1, 32, 0, stream>>>(args); break;                    \
    case 7: hb::KERNEL<8, 16><<<1, 32, 0, stream>>>(args); break;                    \
    default: return hbi::fail(HB_ERR_UNSUPPORTED, "no limb configuration");          \
  }                                                                                  \
  hbi::g_launches++;

int to_mont(hb_ctx* ctx, const uint32_t* words, int w, uint32_t* dig, long count, cudaStream_t stream) {
  const int cfg = ctx->cfg_pub;
  Launch l = plan(ctx, cfg, count);
  hb::ToMontArgs A{dev_mod(ctx->d_pub, ctx->mod_n2), words, w, dig, count};
  HB_DISPATCH(cfg, k_to_mont, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
}

// inv[i] = val[i]^-1 for `count` digit-form Montgomery values (val is left intact).
// Tree of pairwise products, one warp-wide extended Euclid at the root, then back down.
int invert_batch(hb_ctx* ctx, const uint32_t* val, long count, uint32_t* inv, Scratch& sc, cudaStream_t stream) {
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  hb::ModDev mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  std::vector<const uint32_t*> lv_val{val};
  std::vector<long> lv_n{count};
  while (lv_n.back() > 1) {
    long nsrc = lv_n.back(), ndst = (nsrc + 1) / 2;
    uint32_t* dst = nullptr;
    CU(sc.get(&dst, (size_t)ndst * L));
    Launch l = plan(ctx, cfg, ndst);
    hb::PairUpArgs A{mod, lv_val.back(), nsrc, dst};
    HB_DISPATCH(cfg, k_pair_up, l, stream, A)
    lv_val.push_back(dst);
    lv_n.push_back(ndst);
  }
  // root
  const int T = 32 * (L / 32 + 1);
  uint32_t* root = nullptr; uint32_t* words = nullptr; int* status = nullptr;
  CU(sc.get(&root, (size_t)L));
  CU(sc.get(&words, (size_t)T));
  CU(sc.get(&status, 1));
  CU(cudaMemcpyAsync(root, lv_val.back(), (size_t)L * 4, cudaMemcpyDeviceToDevice, stream));
  CU(cudaMemsetAsync(status, 0, sizeof(int), stream));
  {
    hb::RootInvArgs A{mod, root, words, ctx->d_pub + ctx->off_n2words, status};
    HB_DISPATCH1(kernel_cfg(cfg, 1), k_root_inverse, stream, A)
  }
  int hstatus = 0;
  CU(cudaMemcpyAsync(&hstatus, status, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CU(cudaStreamSynchronize(stream));
  if (hstatus) return fail(HB_ERR_NOTUNIT, "invert() no inverse exists");
  // down
  const uint32_t* inv_parent = root;
  for (int lv = (int)lv_n.size() - 2; lv >= 0; lv--) {
    long nchild = lv_n[lv];
    uint32_t* dst = nullptr;
    if (lv == 0) dst = inv; else CU(sc.get(&dst, (size_t)nchild * L));
    Launch l = plan(ctx, cfg, nchild);
    hb::PairDownArgs A{mod, inv_parent, lv_val[lv], nchild, dst};
    HB_DISPATCH(cfg, k_pair_down, l, stream, A)
    inv_parent = dst;
  }
  if (lv_n.size() == 1) CU(cudaMemcpyAsync(inv, root, (size_t)L * 4, cudaMemcpyDeviceToDevice, stream));
  CU(cudaGetLastError());
  return HB_OK;
}

struct PrepOut { uint64_t* mag64; uint8_t* neg; int maxbits; int nneg; };

int scalar_prep(hb_ctx* ctx, const uint32_t* k, long nscal, long rows, long cols, int transpose, int raw,
                Scratch& sc, cudaStream_t stream, PrepOut* out) {
  int* counters = nullptr;
  CU(sc.get(&out->mag64, (size_t)nscal));
  CU(sc.get(&out->neg, (size_t)nscal));
  CU(sc.get(&counters, 2));
  CU(cudaMemsetAsync(counters, 0, 2 * sizeof(int), stream));
  hb::ScalarPrepArgs A;
  A.k = k; A.nwords = ctx->d_pub + ctx->off_nwords; A.negband = ctx->d_pub + ctx->off_negband;
  A.wn = ctx->wn; A.nscal = nscal; A.rows = rows; A.cols = cols; A.transpose = transpose; A.raw = raw;
  A.mag64 = out->mag64; A.neg = out->neg; A.maxbits = counters; A.nneg = counters + 1;
  hb::k_scalar_prep<<<(unsigned)((nscal + 255) / 256), 256, 0, stream>>>(A);
  g_launches++;
  int h[2] = {0, 0};
  CU(cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, stream));
  CU(cudaStreamSynchronize(stream));
  out->maxbits = h[0];
  out->nneg = h[1];
  return HB_OK;
}

int pow_window(int bits) { return bits <= 6 ? 1 : bits <= 24 ? 2 : bits <= 96 ? 3 : bits <= 512 ? 4 : 5; }

// out[e] = pow_scalar(c[e / c_div], k[e % k_period]) for e < count
int powscalar_impl(hb_ctx* ctx, const uint32_t* c, long ncipher, long c_div, const uint32_t* k, long k_period,
                   int raw, uint32_t* out, long count, cudaStream_t stream) {
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  Scratch sc(stream);
  PrepOut pr;
  int rc = scalar_prep(ctx, k, k_period, 1, k_period, 0, raw, sc, stream, &pr);
  if (rc) return rc;
  uint32_t* cm = nullptr; uint32_t* cinv = nullptr;
  CU(sc.get(&cm, (size_t)ncipher * L));
  rc = to_mont(ctx, c, ctx->wc, cm, ncipher, stream);
  if (rc) return rc;
  if (pr.nneg > 0) {
    CU(sc.get(&cinv, (size_t)ncipher * L));
    rc = invert_batch(ctx, cm, ncipher, cinv, sc, stream);
    if (rc) return rc;
  }
  const int win = pow_window(pr.maxbits);
  const int ebits = std::max(win, (pr.maxbits + win - 1) / win * win);
  Launch l = plan(ctx, cfg, count);
  const long stride = (long)(1 << win) * kCfgs[l.cfg].lpt * 32;
  uint32_t* tbl = nullptr;
  CU(sc.get(&tbl, (size_t)stride * l.nwarps));
  hb::PowVarArgs A;
  A.mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  A.base = cm; A.base_inv = cinv ? cinv : cm; A.c_div = c_div;
  const bool small = pr.maxbits <= 64;
  A.mag64 = small ? pr.mag64 : nullptr;
  A.neg = pr.neg;
  A.kres = small ? nullptr : k;
  A.nwords = ctx->d_pub + ctx->off_nwords;
  A.wn = ctx->wn; A.k_period = k_period; A.ebits = ebits; A.win = win;
  A.tbl = tbl; A.tbl_stride = stride; A.out = out; A.wc = ctx->wc; A.count = count;
  HB_DISPATCH(cfg, k_powvar, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
}

int product_impl(hb_ctx* ctx, const uint32_t* c, int win, uint32_t* out, long ngroups, long glen, long gstride,
                 long estride, cudaStream_t stream) {
  const int cfg = ctx->cfg_pub;
  Scratch sc(stream);
  const uint32_t* src = c;
  while (true) {
    // One chunk per resident instance slot where the data allows it: a single full wave per pass, and chunks long
    // enough (>= 8) that the R^clen repair -- log2(clen) + 2 multiplications per work item -- stays small.
    const int shape = kernel_cfg(cfg, ngroups * ((glen + 7) / 8));
    const long slots = (long)ctx->sms * hb::blocks_per_sm(kCfgs[shape].lpt) * 4 * (32 / kCfgs[shape].tpi);
    long clen;
    if (glen <= 8) {
      clen = glen;
    } else {
      const long parts_wanted = std::max<long>(1, slots / std::max<long>(1, ngroups));
      clen = std::max<long>(8, (glen + parts_wanted - 1) / parts_wanted);
    }
    long parts = (glen + clen - 1) / clen;
    uint32_t* dst = out;
    if (parts > 1) CU(sc.get(&dst, (size_t)ngroups * parts * ctx->wc));
    Launch l = plan(ctx, cfg, ngroups * parts);
    hb::ProductArgs A;
    A.mod = dev_mod(ctx->d_pub, ctx->mod_n2);
    A.c = src; A.wc = ctx->wc; A.win = win; A.ngroups = ngroups; A.glen = glen; A.gstride = gstride; A.estride = estride;
    A.parts = parts; A.clen = clen; A.out = dst;
    HB_DISPATCH(cfg, k_product_pass, l, stream, A)
    CU(cudaGetLastError());
    if (parts == 1) break;
    src = dst; glen = parts; gstride = parts; estride = 1; win = ctx->wc;
  }
  return HB_OK;
}

// Bucket-method core for one encrypted row: ab[j] = (A_j, B_j) in digit form, [d][2][L], allocated from sc.
int matvec_ab(hb_ctx* ctx, const uint32_t* c, const PrepOut& pr, long inner, int d, Scratch& sc,
              cudaStream_t stream, uint32_t** ab_out) {
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  hb::ModDev mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  // Window width by row count.  Per column and window the bucket work is about 6 * 2^c multiplications next to one
  // per row: 9 bits (one window fewer than 8 for 52-bit scalars) pays from 32 k rows, 13 bits (four windows instead
  // of six) from 200 k rows (measured break-even ~150 k) -- there the fold over the 8192 digit values runs in parallel pieces.
  int cbits = inner >= 200000 ? 13 : inner >= 32768 ? 9
            : inner >= 4096 ? 8 : inner >= 1024 ? 7 : inner >= 256 ? 6 : inner >= 64 ? 5 : inner >= 16 ? 3 : 2;
  if (const char* force = getenv("HB_MATVEC_CBITS")) {        // tests: exercise a width whatever the row count
    const int f = atoi(force);
    if (f >= 2 && f <= 13) cbits = f;
  }
  if (cbits == 13 && (std::max(pr.maxbits, 1) + 12) / 13 >= (std::max(pr.maxbits, 1) + 8) / 9 && !getenv("HB_MATVEC_CBITS"))
    cbits = 9;                                                 // no window saved: stay with the cheaper buckets
  const int maxbits = std::max(pr.maxbits, 1);
  const int nwin = (maxbits + cbits - 1) / cbits;
  const int NB = 2 << cbits;
  const int seglen = inner >= 65536 ? 256 : inner >= 4096 ? 64 : 16;
  const long nseg = (inner + seglen - 1) / seglen;
  uint32_t *cm, *boff, *sorted, *part, *bucket, *win, *ab;
  CU(sc.get(&cm, (size_t)inner * L));
  int rc = to_mont(ctx, c, ctx->wc, cm, inner, stream);
  if (rc) return rc;
  const size_t njw = (size_t)d * nwin;
  CU(sc.get(&boff, njw * (NB + 1)));
  CU(sc.get(&sorted, njw * inner));
  CU(sc.get(&part, njw * (nseg + NB) * L));
  CU(sc.get(&bucket, njw * NB * L));
  CU(sc.get(&win, njw * 2 * L));
  CU(sc.get(&ab, (size_t)d * 2 * L));
  {
    hb::SortArgs A{pr.mag64, pr.neg, inner, d, nwin, cbits, boff, sorted};
    const size_t smem = (2 * (size_t)NB + 1) * sizeof(uint32_t);
    if (smem > 48 * 1024) {
      static bool once = false;
      if (!once) {
        CU(cudaFuncSetAttribute(hb::k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        once = true;
      }
    }
    hb::k_bucket_sort<<<(unsigned)njw, 256, smem, stream>>>(A);
    g_launches++;
  }
  {
    Launch l = plan(ctx, cfg, (long)njw * nseg);
    hb::SegArgs A{mod, cm, boff, sorted, inner, d, nwin, cbits, seglen, nseg, part};
    HB_DISPATCH(cfg, k_bucket_segments, l, stream, A)
  }
  {
    Launch l = plan(ctx, cfg, (long)njw * NB);
    hb::CombineArgs A{mod, boff, part, d, nwin, cbits, seglen, nseg, bucket};
    HB_DISPATCH(cfg, k_bucket_combine, l, stream, A)
  }
  if (cbits <= 9) {
    Launch l = plan(ctx, cfg, (long)njw * 2);
    hb::RunningArgs A{mod, bucket, d, nwin, cbits, win};
    HB_DISPATCH(cfg, k_bucket_running, l, stream, A)
  } else {
    const int pieces = 1 << (cbits - 8);                       // 256 digit values per piece
    uint32_t *tot, *acc;
    CU(sc.get(&tot, njw * 2 * pieces * L));
    CU(sc.get(&acc, njw * 2 * pieces * L));
    hb::RunningSegArgs A{mod, bucket, d, nwin, cbits, pieces, tot, acc};
    {
      Launch l = plan(ctx, cfg, (long)njw * 2 * pieces);
      HB_DISPATCH(cfg, k_bucket_running_seg, l, stream, A)
    }
    {
      Launch l = plan(ctx, cfg, (long)njw * 2);
      switch (l.cfg) {
        case 0: hb::k_bucket_running_join<8, 4><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        case 1: hb::k_bucket_running_join<16, 4><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        case 2: hb::k_bucket_running_join<24, 4><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        case 3: hb::k_bucket_running_join<32, 4><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        case 4: hb::k_bucket_running_join<24, 8><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        case 5: hb::k_bucket_running_join<8, 8><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        case 6: hb::k_bucket_running_join<16, 8><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        case 7: hb::k_bucket_running_join<8, 16><<<l.blocks, l.threads, 0, stream>>>(A, win); break;
        default: return fail(HB_ERR_UNSUPPORTED, "no limb configuration");
      }
      g_launches++;
    }
  }
  {
    Launch l = plan(ctx, cfg, (long)d * 2);
    hb::HornerArgs A{mod, win, d, nwin, cbits, ab};
    HB_DISPATCH(cfg, k_window_horner, l, stream, A)
  }
  CU(cudaGetLastError());
  *ab_out = ab;
  return HB_OK;
}

// out[j] = A_j * B_j^-1 as plain words (invert = false: B_j is known to be 1)
int matvec_finish(hb_ctx* ctx, const uint32_t* ab, bool invert, int d, uint32_t* out, Scratch& sc,
                  cudaStream_t stream) {
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  hb::ModDev mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  uint32_t* binv = nullptr;
  if (invert) {
    uint32_t* bden = nullptr;
    CU(sc.get(&bden, (size_t)d * L));
    CU(sc.get(&binv, (size_t)d * L));
    hb::k_gather_b<<<(unsigned)(((long)d * L + 255) / 256), 256, 0, stream>>>(ab, bden, d, L);
    g_launches++;
    int rc = invert_batch(ctx, bden, d, binv, sc, stream);
    if (rc) return rc;
  }
  Launch l = plan(ctx, cfg, d);
  hb::FinishArgs A{mod, ab, binv, d, out, ctx->wc};
  HB_DISPATCH(cfg, k_matvec_finish, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
}

int matvec_row(hb_ctx* ctx, const uint32_t* c, const PrepOut& pr, uint32_t* out, long inner, int d,
               cudaStream_t stream) {
  Scratch sc(stream);
  uint32_t* ab = nullptr;
  int rc = matvec_ab(ctx, c, pr, inner, d, sc, stream, &ab);
  if (rc) return rc;
  return matvec_finish(ctx, ab, pr.nneg > 0, d, out, sc, stream);
}

}  // namespace

extern "C" {

int hb_powscalar(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t count,
                 int64_t k_period, int flags, void* stream_) {
  if (!ctx || !c || !k || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0 || k_period < 1) return fail(HB_ERR_ARG, "bad count");
  if (count == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  return powscalar_impl(ctx, c, count, 1, k, k_period, flags & 1, out, count, (cudaStream_t)stream_);
}

int hb_product(hb_ctx* ctx, const uint32_t* c, uint32_t* out, int64_t ngroups, int64_t glen,
               int64_t gstride, int64_t estride, void* stream_) {
  if (!ctx || !c || !out) return fail(HB_ERR_ARG, "null pointer");
  if (ngroups < 0 || glen < 1) return fail(HB_ERR_ARG, "bad group shape");
  if (ngroups == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  return product_impl(ctx, c, ctx->wc, out, ngroups, glen, gstride, estride, (cudaStream_t)stream_);
}

int hb_unit_product(hb_ctx* ctx, const uint32_t* r, uint32_t* out, int64_t count, void* stream_) {
  if (!ctx || !r || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 1) return fail(HB_ERR_ARG, "bad count");
  CU(cudaSetDevice(ctx->device));
  return product_impl(ctx, r, ctx->wn, out, 1, count, 0, 1, (cudaStream_t)stream_);
}

int hb_matvec(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t rows,
              int64_t inner, int64_t d, void* stream_) {
  if (!ctx || !c || !k || !out) return fail(HB_ERR_ARG, "null pointer");
  if (rows < 0 || inner < 1 || d < 1) return fail(HB_ERR_ARG, "bad matrix shape");
  if (inner >= (1 << 22)) return fail(HB_ERR_ARG, "inner dimension must be below 2^22 per call");
  if (rows == 0) return HB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  Scratch sc(stream);
  PrepOut pr;
  int rc = scalar_prep(ctx, k, inner * d, inner, d, 1, 0, sc, stream, &pr);
  if (rc) return rc;
  if (pr.maxbits <= 64) {
    for (int64_t i = 0; i < rows; i++) {
      rc = matvec_row(ctx, c + i * inner * ctx->wc, pr, out + i * d * ctx->wc, inner, (int)d, stream);
      if (rc) return rc;
    }
    return HB_OK;
  }
  // General path (scalars wider than 64 bits, e.g. overflow-band residues): every term is an
  // independent power, then a strided product per output column.
  for (int64_t i = 0; i < rows; i++) {
    uint32_t* terms = nullptr;
    CU(sc.get(&terms, (size_t)inner * d * ctx->wc));
    rc = powscalar_impl(ctx, c + i * inner * ctx->wc, inner, d, k, inner * d, 0, terms, inner * d, stream);
    if (rc) return rc;
    rc = product_impl(ctx, terms, ctx->wc, out + i * d * ctx->wc, d, inner, 1, d, stream);
    if (rc) return rc;
  }
  return HB_OK;
}

// ---- row-sharded matvec: per-rank partials, exchanged as plain words, combined after the gather --------
int hb_matvec_partial(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* ab_out, int64_t inner,
                      int64_t d, void* stream_) {
  if (!ctx || !c || !k || !ab_out) return fail(HB_ERR_ARG, "null pointer");
  if (inner < 1 || d < 1) return fail(HB_ERR_ARG, "bad matrix shape");
  if (inner >= (1 << 22)) return fail(HB_ERR_ARG, "inner dimension must be below 2^22 per call");
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_pub;
  Scratch sc(stream);
  PrepOut pr;
  int rc = scalar_prep(ctx, k, inner * d, inner, d, 1, 0, sc, stream, &pr);
  if (rc) return rc;
  if (pr.maxbits <= 64) {
    uint32_t* ab = nullptr;
    rc = matvec_ab(ctx, c, pr, inner, (int)d, sc, stream, &ab);
    if (rc) return rc;
    Launch l = plan(ctx, cfg, 2 * d);
    hb::FromMontArgs A{dev_mod(ctx->d_pub, ctx->mod_n2), ab, 2 * d, ab_out, ctx->wc};
    HB_DISPATCH(cfg, k_from_mont, l, stream, A)
    CU(cudaGetLastError());
    return HB_OK;
  }
  // wide scalars: the generic path already folds the inverses in; A_j = result, B_j = 1
  uint32_t *terms = nullptr, *col = nullptr;
  CU(sc.get(&terms, (size_t)inner * d * ctx->wc));
  CU(sc.get(&col, (size_t)d * ctx->wc));
  rc = powscalar_impl(ctx, c, inner, d, k, inner * d, 0, terms, inner * d, stream);
  if (rc) return rc;
  rc = product_impl(ctx, terms, ctx->wc, col, d, inner, 1, d, stream);
  if (rc) return rc;
  CU(cudaMemsetAsync(ab_out, 0, (size_t)2 * d * ctx->wc * 4, stream));
  CU(cudaMemcpy2DAsync(ab_out, (size_t)2 * ctx->wc * 4, col, (size_t)ctx->wc * 4, (size_t)ctx->wc * 4, d,
                       cudaMemcpyDeviceToDevice, stream));
  std::vector<uint32_t> ones((size_t)d * ctx->wc, 0);
  for (int64_t j = 0; j < d; j++) ones[(size_t)j * ctx->wc] = 1;
  CU(cudaMemcpy2DAsync(ab_out + ctx->wc, (size_t)2 * ctx->wc * 4, ones.data(), (size_t)ctx->wc * 4,
                       (size_t)ctx->wc * 4, d, cudaMemcpyHostToDevice, stream));
  CU(cudaStreamSynchronize(stream));     // `ones` lives on this stack frame
  return HB_OK;
}

int hb_matvec_combine(hb_ctx* ctx, const uint32_t* ab_all, int nranks, uint32_t* out, int64_t d, void* stream_) {
  if (!ctx || !ab_all || !out) return fail(HB_ERR_ARG, "null pointer");
  if (nranks < 1 || d < 1) return fail(HB_ERR_ARG, "bad shape");
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  Scratch sc(stream);
  uint32_t *dig = nullptr, *ab = nullptr;
  const long per = 2 * d;
  CU(sc.get(&dig, (size_t)nranks * per * L));
  CU(sc.get(&ab, (size_t)per * L));
  int rc = to_mont(ctx, ab_all, ctx->wc, dig, (long)nranks * per, stream);
  if (rc) return rc;
  Launch l = plan(ctx, cfg, per);
  hb::FoldArgs A{dev_mod(ctx->d_pub, ctx->mod_n2), dig, per * L, nranks, per, ab};
  HB_DISPATCH(cfg, k_fold, l, stream, A)
  CU(cudaGetLastError());
  return matvec_finish(ctx, ab, true, (int)d, out, sc, stream);
}

}  // extern "C"
