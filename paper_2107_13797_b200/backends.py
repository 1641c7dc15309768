"""Execution backends: the reference's plug-in point (backends.py:22-86 of the reference) on the B200.

`ExecutionBackend.run(kernel, common, items) -> list` is the contract the reference's operators call
(operators.py:114,121,134,143,157,212,219,250,269,290,315).  CudaBackend honours it for every element
kernel -- it recognises the kernel by name, so it accepts this package's markers (operators._k_*) and
the reference package's own functions alike, which makes it a drop-in `backend=` argument for the
unmodified reference.  That level marshals Python integers per call; the operators in this package
bypass it and hand device-resident word arrays straight to the C ABI.

Two implementations:

  * CudaBackend          -- every element kernel on the current CUDA device;
  * MultiDeviceBackend   -- the reference's ParallelBackend (backends.py:51-78: contiguous chunks of
                            ceil(count / workers), order preserved) with one GPU per worker, driven from ONE
                            process so that the sequential FLR parties (flr/parties.py:330-346) speed up too.

There is deliberately no CPU backend here: get_backend("naive") / ("parallel") raise.
"""
from __future__ import annotations

import ctypes
import math
import random as _random
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import device
from . import _native
from ._native import HB_A_MONT, HB_B_MONT, HB_OUT_MONT, HB_POW_RAW_EXPONENT
from .device import CompactScalars, Shards, WordArray


class ExecutionBackend:
    """Maps a chunk kernel over a list of work items, preserving order."""

    name = "base"
    worker_count = 1

    def run(self, kernel, common, items: list) -> list:
        raise NotImplementedError

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __repr__(self):
        return f"{type(self).__name__}(workers={self.worker_count})"


def shard_range(count: int, rank: int, world: int) -> tuple:
    """[lo, hi) of worker `rank`: chunks of ceil(count / world), the reference's schedule (backends.py:64-73)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    chunk = -(-count // world) if count else 0
    lo = min(rank * chunk, count)
    return lo, min(lo + chunk, count)


def _is_system_rng(rng) -> bool:
    return rng is None or type(rng) is _random.SystemRandom


class CudaBackend(ExecutionBackend):
    """All element kernels on the current CUDA device through libhebatch_b200.so.

    resident_montgomery: ciphertexts produced by an operator stay in Montgomery digit form in HBM (device.WordArray
    converts on download); chained operators then cost no conversion and an addition is one multiplication."""

    name = "cuda"
    worker_count = 1      # batch_sum's per-worker split (operators.py:263-275) is done on the device

    def __init__(self, resident_montgomery: bool = True):
        self._lib = None
        self.resident_montgomery = bool(resident_montgomery)

    # -- plumbing
    def lib(self):
        if self._lib is None:
            device.require_cuda()
            self._lib = _native.lib()
        return self._lib

    @staticmethod
    def _stream():
        return device.current_stream_ptr()

    def _ct_out(self, ctx, count: int):
        """(WordArray, pointer, flag) for a ciphertext result in the representation this backend keeps resident."""
        t = device.torch()
        if self.resident_montgomery:
            buf = t.empty((count, ctx.limbs), dtype=t.int32, device="cuda")
            return WordArray.from_mont(buf, ctx.n, ctx.wc), buf.data_ptr(), HB_OUT_MONT
        out = WordArray.empty_device(count, ctx.wc)
        return out, out.ptr(), 0

    def set_matvec_window(self, n: int, bits: int) -> None:
        """Force the bucket window of the encrypted matvec for modulus n (0 = by row count); tests use it to
        exercise every width."""
        device.context_for(n).set_option(_native.HB_OPT_MATVEC_WINDOW_BITS, bits)

    # -- device-level entry points used by operators.py (WordArray in, WordArray out)
    def encrypt(self, n: int, m: WordArray, r: WordArray) -> WordArray:
        ctx = device.context_for(n)
        out, optr, flags = self._ct_out(ctx, m.count)
        _native.check(self.lib().hb_encrypt_rep(ctx.handle, m.ptr(), r.ptr(), optr, m.count, flags, self._stream()))
        return out

    def obfuscate(self, n: int, c: WordArray, r: WordArray) -> WordArray:
        ctx = device.context_for(n)
        cptr, cm = c.ct_operand()
        out, optr, flags = self._ct_out(ctx, c.count)
        _native.check(self.lib().hb_obfuscate_rep(ctx.handle, cptr, r.ptr(), optr, c.count,
                                                  flags | (HB_A_MONT if cm else 0), self._stream()))
        return out

    # chunk of the streamed encrypt / obfuscate: a whole number of persistent-grid waves for every limb shape
    # (lcm of 9472, 7104, 18944, 28416 instances per wave)
    STREAM_CHUNK = 56832

    def _pinned_stage(self, tag: str, rows: int, wn: int):
        """Page-locked int32 staging of at least rows x wn words, kept on the backend and only ever grown:
        cudaHostAlloc of a few hundred MB costs tens of milliseconds, a streamed operator is called five times per
        FLR iteration.  One operator runs at a time on a backend (callers are single-threaded)."""
        t = device.torch()
        stages = self.__dict__.setdefault("_stages", {})
        need = rows * wn
        buf = stages.get(tag)
        if buf is None or buf.numel() < need:
            buf = stages[tag] = t.empty((need + need // 8,), dtype=t.int32, pin_memory=True)
        return buf[:need].view(rows, wn)

    def _draw_chunk(self, lib, n_words, wn, cnt, host_ptr, mt_state):
        """`cnt` values of randrange(1, n) into host memory: the MT19937 replay when mt_state = (state, index) is
        given, the operating system's CSPRNG otherwise."""
        if mt_state is not None:
            state, index = mt_state
            _native.check(lib.hb_mt19937_randrange1(state.ctypes.data, ctypes.byref(index), n_words.ctypes.data,
                                                    wn, cnt, host_ptr))
        else:
            _native.check(lib.hb_secure_randrange1(n_words.ctypes.data, wn, cnt, host_ptr))

    @staticmethod
    def _mt_state(rng):
        """(saved, (state words, index)) of a random.Random, or (None, None) for the OS generator."""
        if _is_system_rng(rng):
            return None, None
        saved = rng.getstate()
        internal = saved[1]
        return saved, (np.array(internal[:624], dtype=np.uint32), ctypes.c_int(internal[624]))

    @staticmethod
    def _mt_commit(rng, saved, mt_state):
        if mt_state is not None:
            state, index = mt_state
            rng.setstate((saved[0], tuple(int(v) for v in state) + (index.value,), saved[2]))

    @staticmethod
    def _bulk_rng(rng) -> bool:
        """Generators whose randrange stream the native code reproduces (random.Random: MT19937 replay) or replaces
        by an equivalent draw (SystemRandom / None: os entropy).  Anything else is drawn element by element."""
        return _is_system_rng(rng) or type(rng) is _random.Random

    def _streamed(self, n: int, count: int, rng, launch) -> bool:
        """Run `launch(off, cnt, r_ptr)` over chunks of `count` elements with their obfuscation factors drawn while
        the GPU works: chunk k + 1 is produced on the host (native MT19937 replay of a seeded random.Random, or the
        OS generator for SystemRandom / None) while chunk k's modular powers run, the gcd test of every chunk is one
        product on the device, and the products are looked at once at the end.  Same values in the same order as
        [draw_unit(n, rng) for each element] (operators.py:133,142 of the reference).  False when a non-unit was
        drawn (the generator is then back where it started and the caller redoes the batch the exact way)."""
        t = device.torch()
        ctx = device.context_for(n)
        lib = self.lib()
        wn, wc = ctx.wn, ctx.wc
        saved, mt_state = self._mt_state(rng)
        n_words = device.ints_to_words([n], wn)
        chunk = self.STREAM_CHUNK
        nchunks = (count + chunk - 1) // chunk
        pinned = self._pinned_stage("chunks", 2 * chunk, wn).view(2, chunk, wn)      # page-locking is slow to repeat
        staged = [t.empty((chunk, wn), dtype=t.int32, device="cuda") for _ in range(2)]
        copied = [None, None]
        checks = t.empty((nchunks, wc), dtype=t.int32, device="cuda")
        stream = self._stream()
        for k in range(nchunks):
            off = k * chunk
            cnt = min(chunk, count - off)
            which = k & 1
            if copied[which] is not None:
                copied[which].synchronize()            # the upload that last used this pinned buffer is done
            host = pinned[which].numpy()
            self._draw_chunk(lib, n_words, wn, cnt, host.ctypes.data, mt_state)
            staged[which][:cnt].copy_(pinned[which][:cnt], non_blocking=True)
            copied[which] = t.cuda.Event()
            copied[which].record()
            r_ptr = staged[which].data_ptr()
            _native.check(lib.hb_unit_product(ctx.handle, r_ptr, checks[k].data_ptr(), cnt, stream))
            launch(off, cnt, r_ptr)
        products = WordArray.from_device(checks).ints()
        if any(math.gcd(p, n) != 1 for p in products):
            if saved is not None:
                rng.setstate(saved)
            return False
        self._mt_commit(rng, saved, mt_state)
        return True

    def _streams(self, n: int, count: int, rng) -> bool:
        """Does a batch qualify for the streamed draw?  (large batch, real key size, a generator the native code
        can replay or replace)"""
        return self._bulk_rng(rng) and n.bit_length() >= 256 and count >= 2 * self.STREAM_CHUNK

    def encrypt_drawing(self, n: int, src: WordArray, rng, obfuscate: bool = False):
        """batch_encrypt / batch_obfuscate of a large batch with the draws overlapping the GPU (_streamed).  Returns
        None when the batch does not qualify or a non-unit was drawn: the caller then takes the one-shot path."""
        count = src.count
        if not self._streams(n, count, rng):
            return None
        ctx = device.context_for(n)
        lib = self.lib()
        wn, wc = ctx.wn, ctx.wc
        out, out_ptr, oflags = self._ct_out(ctx, count)
        w_out = ctx.limbs if oflags else wc
        if obfuscate:
            src_ptr, src_mont = src.ct_operand()
            w_src = ctx.limbs if src_mont else wc
            flags = oflags | (HB_A_MONT if src_mont else 0)
        else:
            src_ptr, w_src, flags = src.ptr(), wn, oflags
        call = lib.hb_obfuscate_rep if obfuscate else lib.hb_encrypt_rep
        stream = self._stream()

        def launch(off, cnt, r_ptr):
            _native.check(call(ctx.handle, src_ptr + off * w_src * 4, r_ptr, out_ptr + off * w_out * 4, cnt, flags,
                               stream))
        return out if self._streamed(n, count, rng, launch) else None

    def fore_gradient_drawing(self, n: int, c: WordArray, lg: WordArray, kg: WordArray, kh: int, yl: WordArray, rng):
        """The fused fore-gradient chain with its obfuscation factors drawn from `rng` in element order: streamed
        for large batches, one shot otherwise.  Returns None if a non-unit was drawn in the streamed form."""
        count = c.count
        if not self._streams(n, count, rng):
            return self.fore_gradient(n, c, lg, kg, kh, yl, self.draw_units(n, count, rng))
        ctx = device.context_for(n)
        lib = self.lib()
        cptr, cm = c.ct_operand()
        w_c = ctx.limbs if cm else ctx.wc
        out, out_ptr, oflags = self._ct_out(ctx, count)
        w_out = ctx.limbs if oflags else ctx.wc
        flags = oflags | (HB_A_MONT if cm else 0)
        lg_ptr, kg_ptr, yl_ptr, wn = lg.ptr(), kg.ptr(), yl.ptr(), ctx.wn
        stream = self._stream()

        def launch(off, cnt, r_ptr):
            _native.check(lib.hb_fore_gradient(ctx.handle, cptr + off * w_c * 4, lg_ptr + off * wn * 4, kg_ptr,
                                               int(kh), yl_ptr + off * wn * 4, r_ptr, out_ptr + off * w_out * 4,
                                               cnt, flags, stream))
        return out if self._streamed(n, count, rng, launch) else None

    def decrypt(self, n: int, private, c: WordArray) -> WordArray:
        """private = (p, q, hp, hq, q_inv)."""
        ctx = device.context_for(n)
        ctx.set_private(*private)
        cptr, cm = c.ct_operand()
        out = WordArray.empty_device(c.count, ctx.wn)
        _native.check(self.lib().hb_decrypt_rep(ctx.handle, cptr, out.ptr(), c.count, HB_A_MONT if cm else 0,
                                                self._stream()))
        return out

    def mulmod(self, n: int, a: WordArray, b: WordArray, broadcast_b: bool = False) -> WordArray:
        ctx = device.context_for(n)
        aptr, am = a.ct_operand()
        bptr, bm = b.ct_operand()
        out, optr, flags = self._ct_out(ctx, a.count)
        flags |= (HB_A_MONT if am else 0) | (HB_B_MONT if bm else 0)
        _native.check(self.lib().hb_mulmod_rep(ctx.handle, aptr, bptr, optr, a.count, 1 if broadcast_b else 0,
                                               flags, self._stream()))
        return out

    def plain_mulmod(self, n: int, a: WordArray, b: WordArray, broadcast_b: bool = False) -> WordArray:
        """out[i] = a[i] * b[i] mod n on plaintext residues (batches.plain_mul)."""
        ctx = device.context_for(n)
        out = WordArray.empty_device(a.count, ctx.wn)
        _native.check(self.lib().hb_plain_mulmod(ctx.handle, a.ptr(), b.ptr(), out.ptr(), a.count,
                                                 1 if broadcast_b else 0, self._stream()))
        return out

    def plain_addmod(self, n: int, a: WordArray, b: WordArray) -> WordArray:
        """out[i] = a[i] + b[i] mod n on plaintext residues (batches.plain_add)."""
        ctx = device.context_for(n)
        out = WordArray.empty_device(a.count, ctx.wn)
        _native.check(self.lib().hb_plain_addmod(ctx.handle, a.ptr(), b.ptr(), out.ptr(), a.count, self._stream()))
        return out

    def plain_rescale(self, n: int, m: WordArray, digits: int):
        """Signed mantissas times 16^digits, back as residues.  Returns (words, first_bad) where first_bad is the
        smallest index whose value is in the overflow band or leaves max_int after scaling, or -1."""
        ctx = device.context_for(n)
        t = device.torch()
        out = WordArray.empty_device(m.count, ctx.wn)
        bad = t.full((1,), -1, dtype=t.int64, device="cuda")
        _native.check(self.lib().hb_plain_rescale(ctx.handle, m.ptr(), int(digits), out.ptr(), m.count,
                                                  bad.data_ptr(), self._stream()))
        return out, int(bad.item())

    def sqrmod(self, n: int, a: WordArray, reps: int = 1, throughput_shape: bool = False) -> WordArray:
        """out[i] = a[i]^(2^reps) mod n^2 through the kernels' squaring path."""
        ctx = device.context_for(n)
        out = WordArray.empty_device(a.count, ctx.wc)
        _native.check(self.lib().hb_sqrmod(ctx.handle, a.ptr(), out.ptr(), a.count, reps,
                                           1 if throughput_shape else 0, self._stream()))
        return out

    def lift_mulmod(self, n: int, a: WordArray, m: WordArray, broadcast_m: bool = False) -> WordArray:
        ctx = device.context_for(n)
        aptr, am = a.ct_operand()
        out, optr, flags = self._ct_out(ctx, a.count)
        _native.check(self.lib().hb_lift_mulmod_rep(ctx.handle, aptr, m.ptr(), optr, a.count,
                                                    1 if broadcast_m else 0, flags | (HB_A_MONT if am else 0),
                                                    self._stream()))
        return out

    def powscalar(self, n: int, c: WordArray, k: WordArray, raw_exponent: bool = False) -> WordArray:
        """out[i] = pow_scalar(c[i], k[i % k.count])."""
        ctx = device.context_for(n)
        cptr, cm = c.ct_operand()
        out, optr, flags = self._ct_out(ctx, c.count)
        flags |= (HB_A_MONT if cm else 0) | (HB_POW_RAW_EXPONENT if raw_exponent else 0)
        _native.check(self.lib().hb_powscalar(ctx.handle, cptr, k.ptr(), optr, c.count, k.count, flags,
                                              self._stream()))
        return out

    def product(self, n: int, c: WordArray, ngroups: int, glen: int, gstride: int, estride: int) -> WordArray:
        ctx = device.context_for(n)
        cptr, cm = c.ct_operand()
        out, optr, flags = self._ct_out(ctx, ngroups)
        _native.check(self.lib().hb_product_rep(ctx.handle, cptr, optr, ngroups, glen, gstride, estride,
                                                flags | (HB_A_MONT if cm else 0), self._stream()))
        return out

    def fore_gradient(self, n: int, c: WordArray, lg: WordArray, kg: WordArray, kh: int, yl: WordArray,
                      r: WordArray) -> WordArray:
        """The fused fore-gradient chain (hb_fore_gradient): (1 + (lg kg mod n) n) r^n * c^kh * (1 + yl n)."""
        ctx = device.context_for(n)
        cptr, cm = c.ct_operand()
        out, optr, flags = self._ct_out(ctx, c.count)
        _native.check(self.lib().hb_fore_gradient(ctx.handle, cptr, lg.ptr(), kg.ptr(), int(kh), yl.ptr(), r.ptr(),
                                                  optr, c.count, flags | (HB_A_MONT if cm else 0), self._stream()))
        return out

    def unit_product(self, n: int, r: WordArray) -> int:
        """prod r[i] mod n^2 as a Python int (one value crosses back)."""
        ctx = device.context_for(n)
        out = WordArray.empty_device(1, ctx.wc)
        _native.check(self.lib().hb_unit_product(ctx.handle, r.ptr(), out.ptr(), r.count, self._stream()))
        return out.ints()[0]

    def draw_units(self, n: int, count: int, rng) -> WordArray:
        """`count` obfuscation factors, [draw_unit(n, rng) for _ in range(count)] (paillier.py:173-178) in bulk.
        A seeded random.Random is replayed natively (bit-identical stream, state written back); SystemRandom / None
        -- the secure default -- draws from the operating system's generator in native code (same distribution, no
        per-element Python).  The gcd test is one product on the GPU and one gcd.  Generators of any other type, and
        small moduli, are drawn element by element, as is a batch in which the gcd test fails."""
        from .paillier import default_rng, draw_unit
        wn = (n.bit_length() + 31) // 32
        if count == 0:
            return WordArray.from_ints((), wn)
        if rng is None:
            rng = default_rng()
        if not self._bulk_rng(rng) or n.bit_length() < 256 or count < 4:
            return WordArray.from_ints([draw_unit(n, rng) for _ in range(count)], wn)
        saved, mt_state = self._mt_state(rng)
        n_words = device.ints_to_words([n], wn)
        out = np.empty((count, wn), dtype=np.uint32)
        self._draw_chunk(self.lib(), n_words, wn, count, out.ctypes.data, mt_state)
        words = WordArray.from_numpy(out)
        if math.gcd(self.unit_product(n, words), n) != 1:
            if saved is not None:
                rng.setstate(saved)                   # a non-unit was drawn: redo it the slow, exact way
            return WordArray.from_ints([draw_unit(n, rng) for _ in range(count)], wn)
        self._mt_commit(rng, saved, mt_state)
        return words

    def matvec(self, n: int, c: WordArray, k: WordArray, rows: int, inner: int, d: int) -> WordArray:
        ctx = device.context_for(n)
        cptr, cm = c.ct_operand()
        out, optr, flags = self._ct_out(ctx, rows * d)
        flags |= HB_A_MONT if cm else 0
        if isinstance(k, CompactScalars) and rows == 1 and k.on_device and k.maxbits <= 64:
            _native.check(self.lib().hb_matvec_compact(ctx.handle, cptr, k.mag.data_ptr(), k.neg.data_ptr(),
                                                       k.maxbits, 1 if k.nneg else 0, optr, inner, d, flags,
                                                       self._stream()))
        else:
            _native.check(self.lib().hb_matvec_rep(ctx.handle, cptr, k.ptr(), optr, rows, inner, d, flags,
                                                   self._stream()))
        return out

    def matvec_partial(self, n: int, c: WordArray, k: WordArray, inner: int, d: int) -> WordArray:
        """This rank's rows reduced to d pairs (A_j, B_j): [2 d, wc] plain words (sharding.sharded_matmul)."""
        ctx = device.context_for(n)
        if inner == 0:
            return WordArray.from_ints([1] * (2 * d), ctx.wc)
        out = WordArray.empty_device(2 * d, ctx.wc)
        if isinstance(k, CompactScalars) and k.on_device and k.maxbits <= 64:
            cptr, cm = c.ct_operand()
            _native.check(self.lib().hb_matvec_partial_compact(ctx.handle, cptr, k.mag.data_ptr(), k.neg.data_ptr(),
                                                               k.maxbits, out.ptr(), inner, d, HB_A_MONT if cm else 0,
                                                               self._stream()))
        else:
            _native.check(self.lib().hb_matvec_partial(ctx.handle, c.ptr(), k.ptr(), out.ptr(), inner, d,
                                                       self._stream()))
        return out

    def matvec_combine(self, n: int, ab_all: WordArray, nranks: int, d: int) -> WordArray:
        ctx = device.context_for(n)
        out = WordArray.empty_device(d, ctx.wc)
        _native.check(self.lib().hb_matvec_combine(ctx.handle, ab_all.ptr(), nranks, out.ptr(), d, self._stream()))
        return out

    # -- codec
    def _upload_f64(self, values):
        t = device.torch()
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if not np.all(np.isfinite(vals)):
            raise ValueError("cannot encode non-finite values")
        return vals, t.from_numpy(vals.reshape(-1)).cuda()

    def _exact_exponent_dev(self, ctx, dv, count: int) -> int:
        t = device.torch()
        lowest = t.full((1,), 2 ** 31 - 1, dtype=t.int32, device="cuda")
        _native.check(self.lib().hb_min_exact_exponent(ctx.handle, dv.data_ptr(), count, lowest.data_ptr(),
                                                       self._stream()))
        return int(lowest.item())

    def encode_f64(self, n: int, values, exponent, row_width: int = 1):
        """values: float64 numpy array (host).  exponent None = the batch's exact shared exponent (min of
        encoding.exact_exponent over the values, batches.py:122-123), computed on the device from the same upload.
        Returns (words, exponent used).  Raises FixedPointOverflow like encoding.encode.  row_width (elements per
        row of a 2-D batch) only matters to backends that shard: rows are never split."""
        from .encoding import FixedPointOverflow
        ctx = device.context_for(n)
        t = device.torch()
        vals, dv = self._upload_f64(values)
        count = vals.size
        if exponent is None:
            exponent = self._exact_exponent_dev(ctx, dv, count)
            if exponent == 2 ** 31 - 1:
                exponent = 0
        out = WordArray.empty_device(count, ctx.wn)
        bad = t.full((1,), -1, dtype=t.int64, device="cuda")
        _native.check(self.lib().hb_encode_f64(ctx.handle, dv.data_ptr(), int(exponent), out.ptr(),
                                               count, bad.data_ptr(), self._stream()))
        first = int(bad.item())
        if first >= 0:
            raise FixedPointOverflow(
                f"|{vals.reshape(-1)[first]}| needs a mantissa beyond max_int at exponent {exponent} (element {first})")
        return out, int(exponent)

    def encode_compact(self, n: int, values, exponent):
        """A 2-D float64 matrix straight to the compact resident form (device.CompactScalars) without materialising
        residues.  Returns (CompactScalars, exponent), or None when the matrix has no compact form (a magnitude
        beyond 64 bits, a key below 128 bits): the caller then encodes residues."""
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if vals.ndim != 2 or n.bit_length() < 128 or vals.size == 0:
            return None
        ctx = device.context_for(n)
        t = device.torch()
        vals, dv = self._upload_f64(vals)
        rows, cols = vals.shape
        if exponent is None:
            exponent = self._exact_exponent_dev(ctx, dv, vals.size)
            if exponent == 2 ** 31 - 1:
                exponent = 0
        mag = t.empty((rows * cols,), dtype=t.int64, device="cuda")
        neg = t.empty((rows * cols,), dtype=t.uint8, device="cuda")
        info = t.zeros((3,), dtype=t.int32, device="cuda")
        _native.check(self.lib().hb_encode_f64_compact(ctx.handle, dv.data_ptr(), int(exponent), rows, cols,
                                                       mag.data_ptr(), neg.data_ptr(), info.data_ptr(),
                                                       self._stream()))
        maxbits, nneg, wide = (int(v) for v in info.cpu())
        if wide or maxbits > 64:
            return None
        return CompactScalars(n, rows, cols, mag, neg, maxbits, nneg), int(exponent)

    def compact_scalars(self, n: int, k: WordArray, rows: int, cols: int):
        """Residues (rows x cols, row-major) -> CompactScalars, or None when a magnitude exceeds 64 bits."""
        if rows * cols == 0:
            return None
        ctx = device.context_for(n)
        t = device.torch()
        mag = t.empty((rows * cols,), dtype=t.int64, device="cuda")
        neg = t.empty((rows * cols,), dtype=t.uint8, device="cuda")
        info = t.zeros((3,), dtype=t.int32, device="cuda")
        _native.check(self.lib().hb_scalar_compact(ctx.handle, k.ptr(), rows, cols, mag.data_ptr(), neg.data_ptr(),
                                                   info.data_ptr(), self._stream()))
        maxbits, nneg, _ = (int(v) for v in info.cpu())
        if maxbits > 64:
            return None
        return CompactScalars(n, rows, cols, mag, neg, maxbits, nneg)

    def min_exact_exponent(self, n: int, values) -> int:
        """min over the values of encoding.exact_exponent (zeros count as 0; 0 for an empty array), on the device."""
        vals = np.ascontiguousarray(values, dtype=np.float64).ravel()
        if vals.shape[0] == 0:
            return 0
        ctx = device.context_for(n)
        t = device.torch()
        dv = t.from_numpy(vals).cuda()
        return self._exact_exponent_dev(ctx, dv, vals.shape[0])

    def decode_f64(self, n: int, m: WordArray, exponent: int):
        from .encoding import FixedPointOverflow
        ctx = device.context_for(n)
        t = device.torch()
        out = t.empty((m.count,), dtype=t.float64, device="cuda")
        bad = t.full((1,), -1, dtype=t.int64, device="cuda")
        _native.check(self.lib().hb_decode_f64(ctx.handle, m.ptr(), int(exponent), out.data_ptr(), m.count,
                                               bad.data_ptr(), self._stream()))
        first = int(bad.item())
        if first >= 0:
            raise FixedPointOverflow(
                "mantissa falls in the overflow-detection band (homomorphic wrap-around)")
        return out.cpu().numpy()

    # -- Level 1: the reference's run(kernel, common, items) contract, dispatched by kernel name
    def run(self, kernel, common, items: list) -> list:
        name = getattr(kernel, "__name__", str(kernel))
        handler = getattr(self, "_run" + name, None)
        if handler is None:
            raise _native.NativeLibraryError(f"CudaBackend has no device kernel for {name!r}")
        items = list(items)
        if not items:
            return []
        return handler(common, items)

    @staticmethod
    def _widths(n: int):
        kb = n.bit_length()
        return (kb + 31) // 32, ((2 * kb + 7) // 8 + 3) // 4

    def _run_k_encrypt(self, common, items):
        n, _ = common
        wn, _wc = self._widths(n)
        m = WordArray.from_ints([it[0] for it in items], wn)
        r = WordArray.from_ints([it[1] for it in items], wn)
        return list(self.encrypt(n, m, r).ints())

    def _run_k_obfuscate(self, common, items):
        n, _ = common
        wn, wc = self._widths(n)
        c = WordArray.from_ints([it[0] for it in items], wc)
        r = WordArray.from_ints([it[1] for it in items], wn)
        return list(self.obfuscate(n, c, r).ints())

    def _run_k_decrypt(self, common, items):
        p, q, _p2, _q2, hp, hq, q_inv = common
        n = p * q
        _wn, wc = self._widths(n)
        c = WordArray.from_ints(items, wc)
        return list(self.decrypt(n, (p, q, hp, hq, q_inv), c).ints())

    def _run_k_mul(self, common, items):
        n, _n2, _neg = common
        wn, wc = self._widths(n)
        c = WordArray.from_ints([it[0] for it in items], wc)
        k = WordArray.from_ints([it[1] for it in items], wn)
        return list(self.powscalar(n, c, k).ints())

    def _run_k_add(self, common, items):
        n = math.isqrt(common)
        _wn, wc = self._widths(n)
        a = WordArray.from_ints([it[0] for it in items], wc)
        b = WordArray.from_ints([it[1] for it in items], wc)
        return list(self.mulmod(n, a, b).ints())

    def _run_k_product(self, common, items):
        n = math.isqrt(common)
        _wn, wc = self._widths(n)
        out = []
        # groups of equal length go down in one launch; ragged input falls back to one launch per group
        lengths = {len(g) for g in items}
        if len(lengths) == 1 and next(iter(lengths)) > 0:
            glen = next(iter(lengths))
            flat = WordArray.from_ints([v for g in items for v in g], wc)
            return list(self.product(n, flat, len(items), glen, glen, 1).ints())
        for g in items:
            if not g:
                out.append(1 % common)
                continue
            flat = WordArray.from_ints(g, wc)
            out.append(self.product(n, flat, 1, len(g), 0, 1).ints()[0])
        return out

    def _run_k_dot(self, common, items):
        n, _n2, _neg, rows, cols = common
        wn, wc = self._widths(n)
        k_rows, inner, d = len(rows), len(rows[0]) if rows else 0, len(cols)
        c = WordArray.from_ints([v for row in rows for v in row], wc)
        # cols[j][t] -> row-major inner x d
        k = WordArray.from_ints([cols[j][t] for t in range(inner) for j in range(d)], wn)
        full = self.matvec(n, c, k, k_rows, inner, d).ints()
        return [full[i * d + j] for i, j in items]

    def _run_k_encode(self, common, items):
        pk, exponent = common
        return list(self.encode_f64(pk.n, np.asarray(items, dtype=np.float64), exponent)[0].ints())

    def _run_k_decode(self, common, items):
        pk, exponent = common
        wn, _wc = self._widths(pk.n)
        return [float(v) for v in self.decode_f64(pk.n, WordArray.from_ints(items, wn), exponent)]


class _Worker:
    """One device (and one stream on it) of a MultiDeviceBackend, served by its own thread: the calls into the C
    ABI release the GIL, so the workers' kernels are issued -- and their synchronisations waited for -- side by
    side."""

    def __init__(self, index: int, device_index: int, resident_montgomery: bool):
        self.index = index
        self.device_index = device_index
        self.backend = CudaBackend(resident_montgomery)
        self.pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix=f"hb-dev{device_index}-{index}")
        self.stream = None
        self.pool.submit(self._enter).result()

    def _enter(self):
        t = device.torch()
        t.cuda.set_device(self.device_index)
        self.stream = t.cuda.Stream(device=self.device_index)
        t.cuda.set_stream(self.stream)

    def submit(self, fn, *args):
        def task():
            out = fn(self.backend, *args)
            self.stream.synchronize()          # results are handed to other threads: finished when seen
            return out
        return self.pool.submit(task)

    def close(self):
        self.pool.shutdown(wait=True)


class MultiDeviceBackend(CudaBackend):
    """The reference's data-parallel backend with GPUs as the workers, in one process.

    ParallelBackend (backends.py:51-78 of the reference) cuts `items` into contiguous chunks of
    ceil(count / workers), maps the element kernel over the chunks in worker processes and concatenates in order;
    batch_sum(axis=None) reads `worker_count` to split the reduction the same way and multiplies the partials on the
    caller (operators.py:263-275).  Here a worker is a device: every batch is held as element-range shards, one per
    device (device.Shards), element-wise operators run shard by shard with no exchange, obfuscation factors are
    drawn ONCE in global element order and sliced (the bits do not depend on the number of devices), and the two
    reductions -- batch_sum and the encrypted matvec -- reduce each shard to one partial (a product, or d pairs
    (A_j, B_j)), move the partials to the first device over NVLink peer copies (d KiB-sized messages) and combine
    them there (hb_matvec_combine: fold + ONE batch inversion).  Exact commutative arithmetic: results are
    bit-identical to the single-device backend's for any device count.

    devices: CUDA device indices, one worker each; an index may repeat (several streams on one GPU -- how the
    sharded path is exercised on a single-GPU box).  Default: every visible device."""

    name = "cuda-multi"

    def __init__(self, devices=None, resident_montgomery: bool = True):
        super().__init__(resident_montgomery)
        device.require_cuda()
        t = device.torch()
        if devices is None:
            devices = list(range(t.cuda.device_count()))
        self.devices = [int(d) for d in devices]
        if not self.devices:
            raise ValueError("need at least one device")
        for d in self.devices:
            if not 0 <= d < t.cuda.device_count():
                raise ValueError(f"no CUDA device {d}")
        self.workers = [_Worker(i, d, resident_montgomery) for i, d in enumerate(self.devices)]
        self.worker_count = len(self.workers)
        self._lock = threading.Lock()

    def close(self) -> None:
        for w in self.workers:
            w.close()

    # -- sharding helpers
    def _ranges(self, count: int, unit: int = 1):
        """Element ranges per worker; `unit` elements (a row) are never split."""
        rows = count // unit if unit else 0
        G = self.worker_count
        return [tuple(v * unit for v in shard_range(rows, i, G)) for i in range(G)]

    def _parts(self, arr: WordArray, ranges) -> list:
        """The array as one WordArray per worker covering `ranges`, each resident on (or uploadable to) its device.
        Shards that already have that layout are used as they are; anything else is cut from the host copy or from
        the resident tensor (peer copy)."""
        sh = arr.shards
        if sh is not None and sh.ranges == tuple(ranges) and sh.devices == tuple(self.devices):
            return sh.parts
        if isinstance(arr, CompactScalars):
            raise TypeError("compact scalar matrices are sharded where they are encoded")
        t = device.torch()
        parts = []
        src = None
        if not arr.on_host:
            if arr.shards is not None:
                src = arr.device()                       # gathered once on the caller's device
            else:
                src = arr.mont() if arr.mont() is not None else arr.device()
        for (lo, hi), dev in zip(ranges, self.devices):
            if src is None:
                parts.append(WordArray.from_numpy(arr.numpy()[lo:hi]))
                continue
            piece = src[lo:hi].to(f"cuda:{dev}", non_blocking=False).contiguous()
            if src is arr.mont():
                parts.append(WordArray.from_mont(piece, arr._n, arr.width))
            else:
                parts.append(WordArray.from_device(piece))
        if src is not None:
            self._sync_all(src.device.index)                       # the workers use their own streams
        if arr.shards is None:
            arr._shards = Shards(ranges, parts, self.devices)      # remember the layout: the next operator reuses it
        return parts

    def _sync_all(self, *extra) -> None:
        t = device.torch()
        for dev in set(self.devices) | set(extra):
            t.cuda.synchronize(dev)

    def _replicated(self, arr: WordArray) -> list:
        """A broadcast operand: the same (small) array for every worker, uploaded from the host copy by each."""
        host = arr.numpy()
        return [WordArray.from_numpy(host) for _ in self.workers]

    def _map(self, fn, per_worker_args):
        futures = [w.submit(fn, *args) for w, args in zip(self.workers, per_worker_args)]
        return [f.result() for f in futures]

    def _sharded(self, parts, ranges, width) -> WordArray:
        return WordArray.from_shards(Shards(ranges, parts, self.devices), width)

    def _elementwise(self, call, count: int, width: int, operands, unit: int = 1) -> WordArray:
        """call(backend, *parts) on every shard; operands: WordArrays sharded alike (or ("rep", array) broadcast)."""
        ranges = self._ranges(count, unit)
        cols = []
        for op in operands:
            if isinstance(op, tuple) and op[0] == "rep":
                cols.append(self._replicated(op[1]))
            else:
                cols.append(self._parts(op, ranges))
        def safe(be, *parts):
            return call(be, *parts) if parts[0].count else WordArray.from_ints((), width)
        outs = self._map(safe, list(zip(*cols)))
        return self._sharded(outs, ranges, width)

    # -- element-wise operators
    def encrypt(self, n, m, r):
        _wn, wc = self._widths(n)
        return self._elementwise(lambda be, mm, rr: be.encrypt(n, mm, rr), m.count, wc, [m, r])

    def obfuscate(self, n, c, r):
        _wn, wc = self._widths(n)
        return self._elementwise(lambda be, cc, rr: be.obfuscate(n, cc, rr), c.count, wc, [c, r])

    def decrypt(self, n, private, c):
        wn, _wc = self._widths(n)
        return self._elementwise(lambda be, cc: be.decrypt(n, private, cc), c.count, wn, [c])

    def mulmod(self, n, a, b, broadcast_b=False):
        _wn, wc = self._widths(n)
        bop = ("rep", b) if broadcast_b else b
        return self._elementwise(lambda be, aa, bb: be.mulmod(n, aa, bb, broadcast_b), a.count, wc, [a, bop])

    def lift_mulmod(self, n, a, m, broadcast_m=False):
        _wn, wc = self._widths(n)
        mop = ("rep", m) if broadcast_m else m
        return self._elementwise(lambda be, aa, mm: be.lift_mulmod(n, aa, mm, broadcast_m), a.count, wc, [a, mop])

    def plain_mulmod(self, n, a, b, broadcast_b=False):
        wn, _wc = self._widths(n)
        bop = ("rep", b) if broadcast_b else b
        return self._elementwise(lambda be, aa, bb: be.plain_mulmod(n, aa, bb, broadcast_b), a.count, wn, [a, bop])

    def plain_addmod(self, n, a, b):
        wn, _wc = self._widths(n)
        return self._elementwise(lambda be, aa, bb: be.plain_addmod(n, aa, bb), a.count, wn, [a, b])

    def plain_rescale(self, n, m, digits):
        wn, _wc = self._widths(n)
        ranges = self._ranges(m.count)
        res = self._map(lambda be, mm: be.plain_rescale(n, mm, digits) if mm.count else (mm, -1),
                        [(p,) for p in self._parts(m, ranges)])
        bad = [lo + b for (lo, _hi), (_w, b) in zip(ranges, res) if b >= 0]
        return self._sharded([w for w, _b in res], ranges, wn), (min(bad) if bad else -1)

    def fore_gradient(self, n, c, lg, kg, kh, yl, r):
        _wn, wc = self._widths(n)
        return self._elementwise(lambda be, cc, ll, kk, yy, rr: be.fore_gradient(n, cc, ll, kk, kh, yy, rr),
                                 c.count, wc, [c, lg, ("rep", kg), yl, r])

    def powscalar(self, n, c, k, raw_exponent=False):
        _wn, wc = self._widths(n)
        if k.count == c.count:
            return self._elementwise(lambda be, cc, kk: be.powscalar(n, cc, kk, raw_exponent), c.count, wc, [c, k])
        # element e uses scalar e mod k.count: every shard gets the scalars rotated to its first element
        ranges = self._ranges(c.count)
        host = k.numpy()
        period = k.count
        ks = [WordArray.from_numpy(host[(lo + np.arange(period)) % period]) for lo, _hi in ranges]
        outs = self._map(lambda be, cc, kk: be.powscalar(n, cc, kk, raw_exponent) if cc.count else cc,
                         list(zip(self._parts(c, ranges), ks)))
        return self._sharded(outs, ranges, wc)

    # -- obfuscation factors: drawn once, in global element order, then sliced
    def _streamed_sharded(self, n, count, rng, ranges, launch) -> bool:
        """Sharded form of CudaBackend._streamed.  A seeded generator's stream is produced on the host in global
        element order -- shard 0's factors first, chunk by chunk, then shard 1's ... -- and every chunk is handed to
        its device as soon as it exists, so device g starts after g/G of the draw while the earlier devices are
        already computing; the bits do not depend on the number of devices.  OS entropy has no order to preserve:
        every worker draws its own chunks.  launch(be, ctx, state, a, b, r_ptr): enqueue elements [a, b) of the
        worker's shard; `state` is a per-shard dict."""
        t = device.torch()
        lib = self.lib()
        wn, _wc = self._widths(n)
        saved, mt_state = self._mt_state(rng)
        n_words = device.ints_to_words([n], wn)
        chunk = self.STREAM_CHUNK
        pinned = self._pinned_stage("whole", count, wn)                   # the whole draw, page-locked (kept, grow-only)
        host = pinned.numpy()

        def run_chunk(be, lo, a, b, state):
            ctx = device.context_for(n)
            if mt_state is None:
                self._draw_chunk(lib, n_words, wn, b - a, host[lo + a:lo + b].ctypes.data, None)
            r_dev = pinned[lo + a:lo + b].cuda(non_blocking=True)
            chk = WordArray.empty_device(1, ctx.wc)
            _native.check(lib.hb_unit_product(ctx.handle, r_dev.data_ptr(), chk.ptr(), b - a, be._stream()))
            state.setdefault("checks", []).append(chk)
            launch(be, ctx, state, a, b, r_dev.data_ptr())

        states = [dict() for _ in self.workers]
        futures = []
        for w, (lo, hi), state in zip(self.workers, ranges, states):
            for a in range(0, hi - lo, chunk):
                b = min(hi - lo, a + chunk)
                if mt_state is not None:
                    self._draw_chunk(lib, n_words, wn, b - a, host[lo + a:lo + b].ctypes.data, mt_state)
                futures.append(w.submit(run_chunk, lo, a, b, state))
        for f in futures:
            f.result()
        products = []
        for state in states:
            products.extend(c.ints()[0] for c in state.get("checks", ()))
        self._states = states
        if any(math.gcd(p, n) != 1 for p in products):
            if saved is not None:
                rng.setstate(saved)
            return False
        self._mt_commit(rng, saved, mt_state)
        return True

    def _streams(self, n, count, rng) -> bool:
        return self._bulk_rng(rng) and n.bit_length() >= 256 and count >= 4 * self.worker_count

    def encrypt_drawing(self, n, src, rng, obfuscate=False):
        count = src.count
        if not self._streams(n, count, rng):
            return None
        lib = self.lib()
        _wn, wc = self._widths(n)
        ranges = self._ranges(count)
        parts = self._parts(src, ranges)

        def launch(be, ctx, state, a, b, r_ptr):
            part = parts[be_index[id(be)]]
            if "out" not in state:
                state["out"], state["optr"], state["oflags"] = be._ct_out(ctx, part.count)
            oflags = state["oflags"]
            w_out = ctx.limbs if oflags else ctx.wc
            if obfuscate:
                sptr, sm = part.ct_operand()
                w_src = ctx.limbs if sm else ctx.wc
                _native.check(lib.hb_obfuscate_rep(ctx.handle, sptr + a * w_src * 4, r_ptr,
                                                   state["optr"] + a * w_out * 4, b - a,
                                                   oflags | (HB_A_MONT if sm else 0), be._stream()))
            else:
                _native.check(lib.hb_encrypt_rep(ctx.handle, part.ptr() + a * ctx.wn * 4, r_ptr,
                                                 state["optr"] + a * w_out * 4, b - a, oflags, be._stream()))
        be_index = {id(w.backend): i for i, w in enumerate(self.workers)}
        if not self._streamed_sharded(n, count, rng, ranges, launch):
            return None
        outs = [st["out"] if "out" in st else WordArray.from_ints((), wc) for st in self._states]
        return self._sharded(outs, ranges, wc)

    def fore_gradient_drawing(self, n, c, lg, kg, kh, yl, rng):
        count = c.count
        if not self._streams(n, count, rng):
            return self.fore_gradient(n, c, lg, kg, kh, yl, self.draw_units(n, count, rng))
        lib = self.lib()
        _wn, wc = self._widths(n)
        ranges = self._ranges(count)
        cs, lgs, yls, kgs = (self._parts(c, ranges), self._parts(lg, ranges), self._parts(yl, ranges),
                             self._replicated(kg))
        be_index = {id(w.backend): i for i, w in enumerate(self.workers)}

        def launch(be, ctx, state, a, b, r_ptr):
            i = be_index[id(be)]
            if "out" not in state:
                state["out"], state["optr"], state["oflags"] = be._ct_out(ctx, cs[i].count)
            oflags = state["oflags"]
            w_out = ctx.limbs if oflags else ctx.wc
            cptr, cm = cs[i].ct_operand()
            w_c = ctx.limbs if cm else ctx.wc
            _native.check(lib.hb_fore_gradient(ctx.handle, cptr + a * w_c * 4, lgs[i].ptr() + a * ctx.wn * 4,
                                               kgs[i].ptr(), int(kh), yls[i].ptr() + a * ctx.wn * 4, r_ptr,
                                               state["optr"] + a * w_out * 4, b - a,
                                               oflags | (HB_A_MONT if cm else 0), be._stream()))
        if not self._streamed_sharded(n, count, rng, ranges, launch):
            return None
        outs = [st["out"] if "out" in st else WordArray.from_ints((), wc) for st in self._states]
        return self._sharded(outs, ranges, wc)

    # -- reductions
    def product(self, n, c, ngroups, glen, gstride, estride):
        _wn, wc = self._widths(n)
        first = self.workers[0]
        if ngroups == 1 and estride == 1 and glen == c.count:
            # batch_sum(axis=None): one partial product per worker, multiplied on the first device
            # (operators.py:263-275 of the reference)
            ranges = self._ranges(c.count)
            partials = self._map(lambda be, cc: be.product(n, cc, 1, cc.count, 0, 1) if cc.count else None,
                                 [(p,) for p in self._parts(c, ranges)])
            live = [p for p in partials if p is not None]
            if len(live) == 1:
                return self._on_first(live[0])
            stacked = np.concatenate([p.numpy() for p in live], axis=0)     # G ciphertexts: a few KiB
            return first.submit(lambda be: be.product(n, WordArray.from_numpy(stacked), 1, len(live), 0, 1)).result()
        whole = self._gathered(c)
        return first.submit(lambda be: be.product(n, whole, ngroups, glen, gstride, estride)).result()

    def unit_product(self, n, r):
        first = self.workers[0]
        whole = self._gathered(r)
        return first.submit(lambda be: be.unit_product(n, whole)).result()

    def matvec(self, n, c, k, rows, inner, d):
        """batch_matmul with the reduction axis sharded: hb_matvec_partial on every device, the d x 2 partial
        ciphertexts of every device copied to the first one, hb_matvec_combine there."""
        _wn, wc = self._widths(n)
        first = self.workers[0]
        if rows != 1 or inner < self.worker_count:
            whole_c, whole_k = self._gathered(c), self._gathered(k)
            return first.submit(lambda be: be.matvec(n, whole_c, whole_k, rows, inner, d)).result()
        c_ranges = self._ranges(inner)
        k_ranges = [(lo * d, hi * d) for lo, hi in c_ranges]
        partials = self._map(lambda be, cc, kk: be.matvec_partial(n, cc, kk, cc.count, d),
                             list(zip(self._parts(c, c_ranges), self._parts(k, k_ranges))))
        t = device.torch()
        target = f"cuda:{first.device_index}"
        moved = [p.device().to(target) if p.on_device else t.from_numpy(p.numpy().view(np.int32).copy()).to(target)
                 for p in partials]
        stacked = WordArray.from_device(t.cat(moved, dim=0).contiguous())
        self._sync_all()
        return first.submit(lambda be: be.matvec_combine(n, stacked, len(partials), d)).result()

    def _gathered(self, arr: WordArray) -> WordArray:
        """A whole array for a single-device fallback (axis reductions, tiny or 2-D matvecs) on the first worker's
        device: the array itself when it is resident there (or only on the host), a host round trip otherwise."""
        if arr.shards is None:
            res = arr.mont() if arr.mont() is not None else arr._dev
            if res is None or res.device.index == self.workers[0].device_index:
                return arr
        return WordArray.from_numpy(arr.numpy())

    def _on_first(self, arr: WordArray) -> WordArray:
        return arr

    # -- codec
    def encode_f64(self, n, values, exponent, row_width: int = 1):
        from .encoding import FixedPointOverflow
        vals = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        wn, _wc = self._widths(n)
        if exponent is None:
            exponent = self.min_exact_exponent(n, vals)
            if exponent == 2 ** 31 - 1:
                exponent = 0
        ranges = self._ranges(vals.size, max(1, row_width))

        def enc(be, lo, hi):
            if hi == lo:
                return WordArray.from_ints((), wn), None
            try:
                return be.encode_f64(n, vals[lo:hi], exponent)[0], None
            except FixedPointOverflow as exc:
                return None, exc
        res = self._map(enc, ranges)
        for _w, exc in res:
            if exc is not None:
                raise exc                     # shards are in element order: the first failing shard speaks first
        return self._sharded([w for w, _ in res], ranges, wn), int(exponent)

    def encode_compact(self, n, values, exponent):
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if vals.ndim != 2 or n.bit_length() < 128 or vals.size == 0:
            return None
        rows, cols = vals.shape
        if exponent is None:
            exponent = self.min_exact_exponent(n, vals)
            if exponent == 2 ** 31 - 1:
                exponent = 0
        row_ranges = [shard_range(rows, i, self.worker_count) for i in range(self.worker_count)]
        res = self._map(lambda be, lo, hi: be.encode_compact(n, vals[lo:hi], exponent) if hi > lo else "empty",
                        row_ranges)
        if any(r is None for r in res):
            return None
        wn, _wc = self._widths(n)
        t = device.torch()
        parts = []
        for r, dev in zip(res, self.devices):
            if r == "empty":
                parts.append(CompactScalars(n, 0, cols, t.empty((0,), dtype=t.int64, device=f"cuda:{dev}"),
                                            t.empty((0,), dtype=t.uint8, device=f"cuda:{dev}"), 0, 0))
            else:
                parts.append(r[0])
        ranges = [(lo * cols, hi * cols) for lo, hi in row_ranges]
        return self._sharded(parts, ranges, wn), int(exponent)

    def compact_scalars(self, n, k, rows, cols):
        return None               # residues are compacted per call on the device that holds them

    def min_exact_exponent(self, n, values) -> int:
        vals = np.ascontiguousarray(values, dtype=np.float64).ravel()
        if vals.shape[0] == 0:
            return 0
        ranges = self._ranges(vals.shape[0])
        res = self._map(lambda be, lo, hi: be.min_exact_exponent(n, vals[lo:hi]) if hi > lo else 2 ** 31 - 1, ranges)
        return min(res)

    def decode_f64(self, n, m, exponent):
        from .encoding import FixedPointOverflow
        ranges = self._ranges(m.count)

        def dec(be, mm):
            if not mm.count:
                return np.zeros((0,), np.float64), None
            try:
                return be.decode_f64(n, mm, exponent), None
            except FixedPointOverflow as exc:
                return None, exc
        res = self._map(dec, [(p,) for p in self._parts(m, ranges)])
        for _v, exc in res:
            if exc is not None:
                raise exc
        return np.concatenate([v for v, _ in res])

    def draw_units(self, n, count, rng):
        return self.workers[0].submit(lambda be: be.draw_units(n, count, rng)).result()

    def matvec_partial(self, n, c, k, inner, d):
        whole_c, whole_k = self._gathered(c), self._gathered(k)
        return self.workers[0].submit(lambda be: be.matvec_partial(n, whole_c, whole_k, inner, d)).result()

    def matvec_combine(self, n, ab_all, nranks, d):
        whole = self._gathered(ab_all)
        return self.workers[0].submit(lambda be: be.matvec_combine(n, whole, nranks, d)).result()

    def sqrmod(self, n, a, reps=1, throughput_shape=False):
        whole = self._gathered(a)
        return self.workers[0].submit(lambda be: be.sqrmod(n, whole, reps, throughput_shape)).result()

    def set_matvec_window(self, n, bits):
        self._map(lambda be: be.set_matvec_window(n, bits), [() for _ in self.workers])


_default = None


def default_backend() -> CudaBackend:
    global _default
    if _default is None:
        _default = CudaBackend()
    return _default


def set_default_backend(backend) -> None:
    """Make `backend` (a CudaBackend or MultiDeviceBackend, or None to reset) what operators use when none is
    passed -- how a caller that cannot thread a `backend=` argument through (the reference's FLR parties construct
    their own) switches a whole run to several GPUs."""
    global _default
    if backend is not None and not isinstance(backend, CudaBackend):
        raise TypeError("the default backend must be a CudaBackend")
    _default = backend


def get_backend(name: str, workers: int | None = None) -> ExecutionBackend:
    """`cuda`: the current device.  `cuda-multi`: one worker per visible device (or the first `workers` devices)."""
    if name == "cuda":
        return default_backend()
    if name == "cuda-multi":
        t = device.torch()
        device.require_cuda()
        count = t.cuda.device_count()
        return MultiDeviceBackend(list(range(min(count, workers) if workers else count)))
    if name in ("naive", "parallel"):
        raise ValueError(f"backend {name!r} is a CPU backend of the reference package; this build only has 'cuda'")
    raise ValueError(f"unknown backend: {name!r}")
