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
  cudaMemPool_t pool;
  std::vector<void*> ptrs;
  Scratch(const hb_ctx* ctx, cudaStream_t st) : s(st), pool(ctx->pool) {}
  ~Scratch() { for (void* p : ptrs) cudaFreeAsync(p, s); }
  template <typename T>
  cudaError_t get(T** out, size_t n) {
    void* p = nullptr;
    cudaError_t e = hbi::pool_alloc(pool, &p, (n ? n : 1) * sizeof(T), s);
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

int from_mont(hb_ctx* ctx, const uint32_t* dig, uint32_t* words, long count, cudaStream_t stream) {
  const int cfg = ctx->cfg_pub;
  Launch l = plan(ctx, cfg, count);
  hb::FromMontArgs A{dev_mod(ctx->d_pub, ctx->mod_n2), dig, count, words, ctx->wc};
  HB_DISPATCH(cfg, k_from_mont, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
}

// Digit form of a ciphertext operand: the caller's array when it already is (HB_*_MONT), a converted copy otherwise.
int as_mont(hb_ctx* ctx, const uint32_t* c, bool is_mont, long count, Scratch& sc, cudaStream_t stream,
            const uint32_t** out) {
  HB_REQUIRE_ALIGNED16(c, is_mont);
  if (is_mont) { *out = c; return HB_OK; }
  uint32_t* cm = nullptr;
  CU(sc.get(&cm, (size_t)count * Ldig(ctx->cfg_pub)));
  *out = cm;
  return to_mont(ctx, c, ctx->wc, cm, count, stream);
}

// A failed inversion is recorded in a device flag and looked at ONCE, at the end of the entry point that needed it:
// nothing in the middle of a call drains the stream.
int new_status(Scratch& sc, cudaStream_t stream, int** status) {
  CU(sc.get(status, 1));
  CU(cudaMemsetAsync(*status, 0, sizeof(int), stream));
  return HB_OK;
}
int check_status(const int* status, cudaStream_t stream) {
  int h = 0;
  CU(cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CU(cudaStreamSynchronize(stream));
  if (h) return fail(HB_ERR_NOTUNIT, "invert() no inverse exists");
  return HB_OK;
}

// inv[i] = val[i]^-1 for `count` digit-form Montgomery values (val is left intact).
// Tree of pairwise products, one warp-wide extended Euclid at the root, then back down.  *status becomes non-zero
// when the product is not a unit (the values written to inv are then meaningless).
int invert_batch(hb_ctx* ctx, const uint32_t* val, long count, uint32_t* inv, Scratch& sc, cudaStream_t stream,
                 int* status) {
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
  uint32_t* root = nullptr; uint32_t* words = nullptr;
  CU(sc.get(&root, (size_t)L));
  CU(sc.get(&words, (size_t)T));
  CU(cudaMemcpyAsync(root, lv_val.back(), (size_t)L * 4, cudaMemcpyDeviceToDevice, stream));
  {
    hb::RootInvArgs A{mod, root, words, ctx->d_pub + ctx->off_n2words, status};
    HB_DISPATCH1(kernel_cfg(cfg, 1), k_root_inverse, stream, A)
  }
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

// Sign + 64-bit magnitude form of plaintext scalars.  [cols][rows] when transposed (the matvec layout).
struct PrepOut { const uint64_t* mag64; const uint8_t* neg; int maxbits; int nneg; };

int launch_scalar_prep(hb_ctx* ctx, const uint32_t* k, long nscal, long rows, long cols, int transpose, int raw,
                       uint64_t* mag64, uint8_t* neg, int* info, cudaStream_t stream) {
  CU(cudaMemsetAsync(info, 0, 2 * sizeof(int), stream));
  hb::ScalarPrepArgs A;
  A.k = k; A.nwords = ctx->d_pub + ctx->off_nwords; A.negband = ctx->d_pub + ctx->off_negband;
  A.wn = ctx->wn; A.nscal = nscal; A.rows = rows; A.cols = cols; A.transpose = transpose; A.raw = raw;
  A.mag64 = mag64; A.neg = neg; A.maxbits = info; A.nneg = info + 1;
  hb::k_scalar_prep<<<(unsigned)((nscal + 255) / 256), 256, 0, stream>>>(A);
  g_launches++;
  CU(cudaGetLastError());
  return HB_OK;
}

// Residues -> compact form in scratch; the two counters come back to the host (the window width, the number of
// windows and whether an inversion is needed at all depend on them): the one synchronisation of a call that
// starts from residues.  Callers holding the compact form (hb_scalar_compact / hb_encode_f64_compact) skip it.
int scalar_prep(hb_ctx* ctx, const uint32_t* k, long nscal, long rows, long cols, int transpose, int raw,
                Scratch& sc, cudaStream_t stream, PrepOut* out) {
  uint64_t* mag = nullptr; uint8_t* neg = nullptr; int* counters = nullptr;
  CU(sc.get(&mag, (size_t)nscal));
  CU(sc.get(&neg, (size_t)nscal));
  CU(sc.get(&counters, 2));
  int rc = launch_scalar_prep(ctx, k, nscal, rows, cols, transpose, raw, mag, neg, counters, stream);
  if (rc) return rc;
  int h[2] = {0, 0};
  CU(cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, stream));
  CU(cudaStreamSynchronize(stream));
  out->mag64 = mag; out->neg = neg;
  out->maxbits = h[0];
  out->nneg = h[1];
  return HB_OK;
}

int pow_window(int bits) { return bits <= 6 ? 1 : bits <= 24 ? 2 : bits <= 96 ? 3 : bits <= 512 ? 4 : 5; }

// out[e] = pow_scalar(c[e / c_div], k[e % k_period]) for e < count
int powscalar_impl(hb_ctx* ctx, const uint32_t* c, bool c_mont, long ncipher, long c_div, const uint32_t* k,
                   long k_period, int raw, uint32_t* out, bool out_mont, long count, cudaStream_t stream) {
  HB_REQUIRE_ALIGNED16(c, c_mont);
  HB_REQUIRE_ALIGNED16(out, out_mont);
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  Scratch sc(ctx, stream);
  PrepOut pr;
  int rc = scalar_prep(ctx, k, k_period, 1, k_period, 0, raw, sc, stream, &pr);
  if (rc) return rc;
  const uint32_t* cm = nullptr; uint32_t* cinv = nullptr;
  rc = as_mont(ctx, c, c_mont, ncipher, sc, stream, &cm);
  if (rc) return rc;
  int* status = nullptr;
  if (pr.nneg > 0) {
    // only the bases that meet a negative scalar are inverted (the others enter the tree as 1): a non-unit
    // ciphertext under a non-negative scalar is a value, not an error -- operators.py:60-61 inverts per element
    uint32_t* sel = nullptr;
    CU(sc.get(&sel, (size_t)ncipher * L));
    CU(sc.get(&cinv, (size_t)ncipher * L));
    rc = new_status(sc, stream, &status);
    if (rc) return rc;
    hb::MaskArgs M{cm, ctx->d_pub + ctx->mod_n2.r1, pr.neg, ncipher, c_div, k_period, L, sel};
    const long total = ncipher * L;
    hb::k_mask_bases<<<(unsigned)std::min<long>((total + 255) / 256, (long)ctx->sms * 16), 256, 0, stream>>>(M);
    g_launches++;
    rc = invert_batch(ctx, sel, ncipher, cinv, sc, stream, status);
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
  A.tbl = tbl; A.tbl_stride = stride; A.out = out; A.wc = ctx->wc; A.count = count; A.out_mont = out_mont ? 1 : 0;
  HB_DISPATCH(cfg, k_powvar, l, stream, A)
  CU(cudaGetLastError());
  return status ? check_status(status, stream) : HB_OK;
}

// win: words per plain input element (wc, or wn for plaintext-width values); ignored for digit-form input.
int product_impl(hb_ctx* ctx, const uint32_t* c, int win, bool in_mont, uint32_t* out, bool out_mont, long ngroups,
                 long glen, long gstride, long estride, cudaStream_t stream) {
  HB_REQUIRE_ALIGNED16(c, in_mont);
  HB_REQUIRE_ALIGNED16(out, out_mont);
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  Scratch sc(ctx, stream);
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
    const bool last = parts == 1;
    if (!last) CU(sc.get(&dst, (size_t)ngroups * parts * L));      // partial products stay in digit form
    Launch l = plan(ctx, cfg, ngroups * parts);
    hb::ProductArgs A;
    A.mod = dev_mod(ctx->d_pub, ctx->mod_n2);
    A.c = src; A.wc = ctx->wc; A.win = win; A.ngroups = ngroups; A.glen = glen; A.gstride = gstride; A.estride = estride;
    A.parts = parts; A.clen = clen; A.out = dst;
    A.in_mont = in_mont ? 1 : 0;
    A.out_mont = last ? (out_mont ? 1 : 0) : 1;
    HB_DISPATCH(cfg, k_product_pass, l, stream, A)
    CU(cudaGetLastError());
    if (last) break;
    src = dst; glen = parts; gstride = parts; estride = 1; in_mont = true;
  }
  return HB_OK;
}

// Bucket-method core for a block of `inner` rows of one encrypted vector: ab[j] = (A_j, B_j) in digit form,
// [d][2][L], allocated from sc.  cm: digit-form bases of the block; pr.mag64 / pr.neg point at the block's first row
// in the [d][colstride] compact matrix.
int matvec_ab(hb_ctx* ctx, const uint32_t* cm, const PrepOut& pr, long colstride, long inner, int d, Scratch& sc,
              cudaStream_t stream, uint32_t** ab_out) {
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  hb::ModDev mod = dev_mod(ctx->d_pub, ctx->mod_n2);
  // Window width by row count.  Per column and window the bucket work is about 6 * 2^c multiplications next to one
  // per row, so wider windows pay once the rows outnumber the buckets: measured for 52-bit scalars, d = 100
  // (profiles/r02_matvec_window_sweep.json) -- 9 bits from 32 k rows; 11 bits (five windows instead of six) from
  // 64 k rows (100 k x 100: 246 ms against 266 ms); 13 bits (four windows) from 200 k rows (1 M x 100: 1.79 s
  // against 2.11 s at 11 bits, 2.50 s at 9) -- from 11 bits up the fold over the digit values runs in parallel pieces.
  int cbits = inner >= 200000 ? 13 : inner >= 65536 ? 11 : inner >= 32768 ? 9
            : inner >= 4096 ? 8 : inner >= 1024 ? 7 : inner >= 256 ? 6 : inner >= 64 ? 5 : inner >= 16 ? 3 : 2;
  const bool forced = ctx->opt_matvec_cbits != 0;             // hb_ctx_set_option(HB_OPT_MATVEC_WINDOW_BITS)
  if (forced) cbits = ctx->opt_matvec_cbits;
  if (!forced) {                                               // no window saved: stay with the cheaper buckets
    const int mb = std::max(pr.maxbits, 1);
    if (cbits == 13 && (mb + 12) / 13 >= (mb + 10) / 11) cbits = 11;
    if (cbits == 11 && (mb + 10) / 11 >= (mb + 8) / 9) cbits = 9;
  }
  const int maxbits = std::max(pr.maxbits, 1);
  const int nwin = (maxbits + cbits - 1) / cbits;
  const int NB = 2 << cbits;
  const int seglen = inner >= 65536 ? 256 : inner >= 4096 ? 64 : 16;
  const long nseg = (inner + seglen - 1) / seglen;
  uint32_t *boff, *sorted, *part, *bucket, *win, *ab;
  const size_t njw = (size_t)d * nwin;
  CU(sc.get(&boff, njw * (NB + 1)));
  CU(sc.get(&sorted, njw * inner));
  CU(sc.get(&part, njw * (nseg + NB) * L));
  CU(sc.get(&bucket, njw * NB * L));
  CU(sc.get(&win, njw * 2 * L));
  CU(sc.get(&ab, (size_t)d * 2 * L));
  {
    hb::SortArgs A{pr.mag64, pr.neg, colstride, inner, d, nwin, cbits, boff, sorted};
    const size_t smem = (2 * (size_t)NB + 1) * sizeof(uint32_t);
    if (smem > 48 * 1024) {
      if (!ctx->sort_smem_set) {                              // the attribute is per device: remembered per context
        CU(cudaFuncSetAttribute(hb::k_bucket_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        ctx->sort_smem_set = true;
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

// Rows beyond this per bucket pass are processed block by block and the blocks' (A_j, B_j) multiplied together: the
// sort / partial-product scratch stays bounded whatever the inner dimension is.
constexpr long kMatvecBlockRows = 1L << 21;
inline long matvec_block_rows(const hb_ctx* ctx) { return ctx->opt_matvec_block ? ctx->opt_matvec_block : kMatvecBlockRows; }

// (A_j, B_j) of all `inner` rows, [d][2][L] digit form in `ab` (allocated from sc).
int matvec_ab_blocks(hb_ctx* ctx, const uint32_t* cm, const PrepOut& pr, long inner, int d, Scratch& sc,
                     cudaStream_t stream, uint32_t** ab_out) {
  const long blk_rows = matvec_block_rows(ctx);
  if (inner <= blk_rows) return matvec_ab(ctx, cm, pr, inner, inner, d, sc, stream, ab_out);
  const int cfg = ctx->cfg_pub;
  const int L = Ldig(cfg);
  const long nblk = (inner + blk_rows - 1) / blk_rows;
  const long per = 2L * d;
  uint32_t *all = nullptr, *ab = nullptr;
  CU(sc.get(&all, (size_t)nblk * per * L));
  CU(sc.get(&ab, (size_t)per * L));
  for (long b = 0; b < nblk; b++) {
    const long off = b * blk_rows, n = std::min(blk_rows, inner - off);
    Scratch blk(ctx, stream);                       // the block's scratch goes back to the pool before the next one
    PrepOut sub{pr.mag64 + off, pr.neg + off, pr.maxbits, pr.nneg};
    uint32_t* part = nullptr;
    int rc = matvec_ab(ctx, cm + (size_t)off * L, sub, inner, n, d, blk, stream, &part);
    if (rc) return rc;
    CU(cudaMemcpyAsync(all + (size_t)b * per * L, part, (size_t)per * L * 4, cudaMemcpyDeviceToDevice, stream));
  }
  Launch l = plan(ctx, cfg, per);
  hb::FoldArgs A{dev_mod(ctx->d_pub, ctx->mod_n2), all, per * L, (int)nblk, per, ab};
  HB_DISPATCH(cfg, k_fold, l, stream, A)
  CU(cudaGetLastError());
  *ab_out = ab;
  return HB_OK;
}

// out[j] = A_j * B_j^-1 (invert = false: B_j is known to be 1); *status as for invert_batch
int matvec_finish(hb_ctx* ctx, const uint32_t* ab, bool invert, int d, uint32_t* out, bool out_mont, Scratch& sc,
                  cudaStream_t stream, int* status) {
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
    int rc = invert_batch(ctx, bden, d, binv, sc, stream, status);
    if (rc) return rc;
  }
  Launch l = plan(ctx, cfg, d);
  hb::FinishArgs A{mod, ab, binv, d, out, ctx->wc, out_mont ? 1 : 0};
  HB_DISPATCH(cfg, k_matvec_finish, l, stream, A)
  CU(cudaGetLastError());
  return HB_OK;
}

// One encrypted row (digit-form bases) against a compact scalar matrix.  No host synchronisation except the
// inversion flag at the very end, and that only when a scalar is negative.
// One output row.  `status` (may be null when no scalar is negative) is the caller's inversion flag: it is set, never
// cleared, so several rows share one flag and the caller looks at it once (check_status) after the last row.
int matvec_row_async(hb_ctx* ctx, const uint32_t* cm, const PrepOut& pr, uint32_t* out, bool out_mont, long inner,
                     int d, cudaStream_t stream, int* status) {
  Scratch sc(ctx, stream);
  uint32_t* ab = nullptr;
  int rc = matvec_ab_blocks(ctx, cm, pr, inner, d, sc, stream, &ab);
  if (rc) return rc;
  return matvec_finish(ctx, ab, pr.nneg > 0, d, out, out_mont, sc, stream, status);
}

int matvec_row(hb_ctx* ctx, const uint32_t* cm, const PrepOut& pr, uint32_t* out, bool out_mont, long inner, int d,
               cudaStream_t stream) {
  Scratch sc(ctx, stream);
  int* status = nullptr;
  const bool invert = pr.nneg > 0;
  int rc = HB_OK;
  if (invert) { rc = new_status(sc, stream, &status); if (rc) return rc; }
  rc = matvec_row_async(ctx, cm, pr, out, out_mont, inner, d, stream, status);
  if (rc) return rc;
  return invert ? check_status(status, stream) : HB_OK;
}

// (A_j, B_j) of this rank's rows as plain words [d][2][wc] (the exchange format of the row-sharded matvec)
int matvec_partial_words(hb_ctx* ctx, const uint32_t* cm, const PrepOut& pr, uint32_t* ab_out, long inner, int d,
                         cudaStream_t stream) {
  const int cfg = ctx->cfg_pub;
  Scratch sc(ctx, stream);
  uint32_t* ab = nullptr;
  int rc = matvec_ab_blocks(ctx, cm, pr, inner, d, sc, stream, &ab);
  if (rc) return rc;
  return from_mont(ctx, ab, ab_out, 2L * d, stream);
}

int check_compact_args(const hb_ctx* ctx, const void* c, const void* mag, const void* neg, const void* out,
                       int64_t inner, int64_t d, int maxbits) {
  if (!ctx || !c || !mag || !neg || !out) return fail(HB_ERR_ARG, "null pointer");
  if (inner < 1 || d < 1) return fail(HB_ERR_ARG, "bad matrix shape");
  if (maxbits < 0 || maxbits > 64) return fail(HB_ERR_ARG, "compact scalars carry at most 64 magnitude bits");
  return HB_OK;
}

}  // namespace

extern "C" {

int hb_ct_limbs(const hb_ctx* ctx) { return ctx ? Ldig(ctx->cfg_pub) : 0; }

int hb_ct_convert(hb_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t count, int to_montgomery, void* stream_) {
  if (!ctx || !in || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0) return fail(HB_ERR_ARG, "negative count");
  if (count == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  HB_REQUIRE_ALIGNED16(out, to_montgomery != 0);
  HB_REQUIRE_ALIGNED16(in, to_montgomery == 0);
  return to_montgomery ? to_mont(ctx, in, ctx->wc, out, count, (cudaStream_t)stream_)
                       : from_mont(ctx, in, out, count, (cudaStream_t)stream_);
}

int hb_powscalar(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t count,
                 int64_t k_period, int flags, void* stream_) {
  if (!ctx || !c || !k || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 0 || k_period < 1) return fail(HB_ERR_ARG, "bad count");
  if (count == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  return powscalar_impl(ctx, c, (flags & HB_A_MONT) != 0, count, 1, k, k_period, flags & HB_POW_RAW_EXPONENT, out,
                        (flags & HB_OUT_MONT) != 0, count, (cudaStream_t)stream_);
}

int hb_product_rep(hb_ctx* ctx, const uint32_t* c, uint32_t* out, int64_t ngroups, int64_t glen,
                   int64_t gstride, int64_t estride, int flags, void* stream_) {
  if (!ctx || !c || !out) return fail(HB_ERR_ARG, "null pointer");
  if (ngroups < 0 || glen < 1) return fail(HB_ERR_ARG, "bad group shape");
  if (ngroups == 0) return HB_OK;
  CU(cudaSetDevice(ctx->device));
  return product_impl(ctx, c, ctx->wc, (flags & HB_A_MONT) != 0, out, (flags & HB_OUT_MONT) != 0, ngroups, glen,
                      gstride, estride, (cudaStream_t)stream_);
}

int hb_product(hb_ctx* ctx, const uint32_t* c, uint32_t* out, int64_t ngroups, int64_t glen,
               int64_t gstride, int64_t estride, void* stream_) {
  return hb_product_rep(ctx, c, out, ngroups, glen, gstride, estride, 0, stream_);
}

int hb_unit_product(hb_ctx* ctx, const uint32_t* r, uint32_t* out, int64_t count, void* stream_) {
  if (!ctx || !r || !out) return fail(HB_ERR_ARG, "null pointer");
  if (count < 1) return fail(HB_ERR_ARG, "bad count");
  CU(cudaSetDevice(ctx->device));
  return product_impl(ctx, r, ctx->wn, false, out, false, 1, count, 0, 1, (cudaStream_t)stream_);
}

int hb_scalar_compact(hb_ctx* ctx, const uint32_t* k, int64_t rows, int64_t cols, uint64_t* mag_out,
                      uint8_t* neg_out, int* info_out, void* stream_) {
  if (!ctx || !k || !mag_out || !neg_out || !info_out) return fail(HB_ERR_ARG, "null pointer");
  if (rows < 0 || cols < 0) return fail(HB_ERR_ARG, "bad matrix shape");
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  CU(cudaMemsetAsync(info_out, 0, 3 * sizeof(int), stream));
  if (rows * cols == 0) return HB_OK;
  return launch_scalar_prep(ctx, k, rows * cols, rows, cols, 1, 0, mag_out, neg_out, info_out, stream);
}

int hb_encode_f64_compact(hb_ctx* ctx, const double* values, int exponent, int64_t rows, int64_t cols,
                          uint64_t* mag_out, uint8_t* neg_out, int* info_out, void* stream_) {
  if (!ctx || !values || !mag_out || !neg_out || !info_out) return fail(HB_ERR_ARG, "null pointer");
  if (rows < 0 || cols < 0) return fail(HB_ERR_ARG, "bad matrix shape");
  if (ctx->key_bits < 128) return fail(HB_ERR_UNSUPPORTED, "compact encoding needs max_int above 2^64 (key >= 128 bits)");
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  CU(cudaMemsetAsync(info_out, 0, 3 * sizeof(int), stream));
  const long nscal = rows * cols;
  if (nscal == 0) return HB_OK;
  hb::CompactEncArgs A{values, nscal, rows, cols, exponent, mag_out, neg_out, info_out};
  hb::k_encode_compact<<<(unsigned)((nscal + 255) / 256), 256, 0, stream>>>(A);
  g_launches++;
  CU(cudaGetLastError());
  return HB_OK;
}

int hb_matvec_compact(hb_ctx* ctx, const uint32_t* c, const uint64_t* mag, const uint8_t* neg, int maxbits,
                      int has_negative, uint32_t* out, int64_t inner, int64_t d, int flags, void* stream_) {
  int rc = check_compact_args(ctx, c, mag, neg, out, inner, d, maxbits);
  if (rc) return rc;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  Scratch sc(ctx, stream);
  const uint32_t* cm = nullptr;
  rc = as_mont(ctx, c, (flags & HB_A_MONT) != 0, inner, sc, stream, &cm);
  if (rc) return rc;
  PrepOut pr{mag, neg, maxbits, has_negative ? 1 : 0};
  return matvec_row(ctx, cm, pr, out, (flags & HB_OUT_MONT) != 0, inner, (int)d, stream);
}

int hb_matvec_partial_compact(hb_ctx* ctx, const uint32_t* c, const uint64_t* mag, const uint8_t* neg, int maxbits,
                              uint32_t* ab_out, int64_t inner, int64_t d, int flags, void* stream_) {
  int rc = check_compact_args(ctx, c, mag, neg, ab_out, inner, d, maxbits);
  if (rc) return rc;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  Scratch sc(ctx, stream);
  const uint32_t* cm = nullptr;
  rc = as_mont(ctx, c, (flags & HB_A_MONT) != 0, inner, sc, stream, &cm);
  if (rc) return rc;
  PrepOut pr{mag, neg, maxbits, 1};
  return matvec_partial_words(ctx, cm, pr, ab_out, inner, (int)d, stream);
}

int hb_matvec_rep(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t rows,
                  int64_t inner, int64_t d, int flags, void* stream_) {
  if (!ctx || !c || !k || !out) return fail(HB_ERR_ARG, "null pointer");
  if (rows < 0 || inner < 1 || d < 1) return fail(HB_ERR_ARG, "bad matrix shape");
  if (rows == 0) return HB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const bool c_mont = (flags & HB_A_MONT) != 0, out_mont = (flags & HB_OUT_MONT) != 0;
  const int L = Ldig(ctx->cfg_pub);
  const long cw = c_mont ? L : ctx->wc, ow = out_mont ? L : ctx->wc;
  Scratch sc(ctx, stream);
  PrepOut pr;
  int rc = scalar_prep(ctx, k, inner * d, inner, d, 1, 0, sc, stream, &pr);
  if (rc) return rc;
  if (pr.maxbits <= 64) {
    const uint32_t* cm = nullptr;
    rc = as_mont(ctx, c, c_mont, rows * inner, sc, stream, &cm);
    if (rc) return rc;
    // every output row is enqueued behind the previous one; the inversion flag is read once, after the last
    int* status = nullptr;
    if (pr.nneg > 0) { rc = new_status(sc, stream, &status); if (rc) return rc; }
    for (int64_t i = 0; i < rows; i++) {
      rc = matvec_row_async(ctx, cm + (size_t)i * inner * L, pr, out + i * d * ow, out_mont, inner, (int)d, stream,
                            status);
      if (rc) return rc;
    }
    return status ? check_status(status, stream) : HB_OK;
  }
  // General path (scalars wider than 64 bits, e.g. overflow-band residues): every term is an
  // independent power, then a strided product per output column.
  for (int64_t i = 0; i < rows; i++) {
    Scratch row(ctx, stream);
    uint32_t* terms = nullptr;
    CU(row.get(&terms, (size_t)inner * d * L));
    rc = powscalar_impl(ctx, c + i * inner * cw, c_mont, inner, d, k, inner * d, 0, terms, true, inner * d, stream);
    if (rc) return rc;
    rc = product_impl(ctx, terms, ctx->wc, true, out + i * d * ow, out_mont, d, inner, 1, d, stream);
    if (rc) return rc;
  }
  return HB_OK;
}

int hb_matvec(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* out, int64_t rows,
              int64_t inner, int64_t d, void* stream_) {
  return hb_matvec_rep(ctx, c, k, out, rows, inner, d, 0, stream_);
}

// ---- row-sharded matvec: per-rank partials, exchanged as plain words, combined after the gather --------
int hb_matvec_partial(hb_ctx* ctx, const uint32_t* c, const uint32_t* k, uint32_t* ab_out, int64_t inner,
                      int64_t d, void* stream_) {
  if (!ctx || !c || !k || !ab_out) return fail(HB_ERR_ARG, "null pointer");
  if (inner < 1 || d < 1) return fail(HB_ERR_ARG, "bad matrix shape");
  cudaStream_t stream = (cudaStream_t)stream_;
  CU(cudaSetDevice(ctx->device));
  const int L = Ldig(ctx->cfg_pub);
  Scratch sc(ctx, stream);
  PrepOut pr;
  int rc = scalar_prep(ctx, k, inner * d, inner, d, 1, 0, sc, stream, &pr);
  if (rc) return rc;
  if (pr.maxbits <= 64) {
    const uint32_t* cm = nullptr;
    rc = as_mont(ctx, c, false, inner, sc, stream, &cm);
    if (rc) return rc;
    return matvec_partial_words(ctx, cm, pr, ab_out, inner, (int)d, stream);
  }
  // wide scalars: the generic path already folds the inverses in; A_j = result, B_j = 1
  uint32_t *terms = nullptr, *col = nullptr;
  CU(sc.get(&terms, (size_t)inner * d * L));
  CU(sc.get(&col, (size_t)d * ctx->wc));
  rc = powscalar_impl(ctx, c, false, inner, d, k, inner * d, 0, terms, true, inner * d, stream);
  if (rc) return rc;
  rc = product_impl(ctx, terms, ctx->wc, true, col, false, d, inner, 1, d, stream);
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
  Scratch sc(ctx, stream);
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
  int* status = nullptr;
  rc = new_status(sc, stream, &status);
  if (rc) return rc;
  rc = matvec_finish(ctx, ab, true, (int)d, out, false, sc, stream, status);
  if (rc) return rc;
  return check_status(status, stream);
}

}  // extern "C"
