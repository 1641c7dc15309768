"""Execution backend: the reference's plug-in point (backends.py:22-86 of the reference) with one
implementation, the B200.

`ExecutionBackend.run(kernel, common, items) -> list` is the contract the reference's operators call
(operators.py:114,121,134,143,157,212,219,250,269,290,315).  CudaBackend honours it for every element
kernel -- it recognises the kernel by name, so it accepts this package's markers (operators._k_*) and
the reference package's own functions alike, which makes it a drop-in `backend=` argument for the
unmodified reference.  That level marshals Python integers per call; the operators in this package
bypass it and hand device-resident word arrays straight to the C ABI.

There is deliberately no CPU backend here: get_backend("naive") / ("parallel") raise.
"""
from __future__ import annotations

import math

from . import device
from . import _native


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


class CudaBackend(ExecutionBackend):
    """All element kernels on the current CUDA device through libhebatch_b200.so."""

    name = "cuda"
    worker_count = 1      # batch_sum's per-worker split (operators.py:263-275) is done on the device

    def __init__(self):
        self._lib = None

    # -- plumbing
    def lib(self):
        if self._lib is None:
            device.require_cuda()
            self._lib = _native.lib()
        return self._lib

    @staticmethod
    def _stream():
        return device.current_stream_ptr()

    # -- device-level entry points used by operators.py (WordArray in, WordArray out)
    def encrypt(self, n: int, m: device.WordArray, r: device.WordArray) -> device.WordArray:
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(m.count, ctx.wc)
        _native.check(self.lib().hb_encrypt(ctx.handle, m.ptr(), r.ptr(), out.ptr(), m.count, self._stream()))
        return out

    def obfuscate(self, n: int, c: device.WordArray, r: device.WordArray) -> device.WordArray:
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(c.count, ctx.wc)
        _native.check(self.lib().hb_obfuscate(ctx.handle, c.ptr(), r.ptr(), out.ptr(), c.count, self._stream()))
        return out

    # chunk of the streamed encrypt / obfuscate: a whole number of persistent-grid waves for every limb shape
    # (lcm of 9472, 7104, 18944, 28416 instances per wave)
    STREAM_CHUNK = 56832

    def encrypt_drawing(self, n: int, src: device.WordArray, rng, obfuscate: bool = False):
        """batch_encrypt / batch_obfuscate with the obfuscation factors drawn while the GPU works: the native
        MT19937 replay (draw_units) produces chunk k + 1 on the host while chunk k's modular powers run, the gcd test
        of every chunk is one product on the device, and the results are looked at once at the end.  Same values in
        the same order as [draw_unit(n, rng) for each element] (operators.py:133,142 of the reference).  Returns
        None when the batch does not qualify (small batch, small modulus, a generator that is not exactly
        random.Random): the caller then takes the one-shot path."""
        import ctypes
        import math
        import random as _random
        import numpy as np
        count = src.count
        if type(rng) is not _random.Random or n.bit_length() < 256 or count < 2 * self.STREAM_CHUNK:
            return None
        t = device.torch()
        ctx = device.context_for(n)
        lib = self.lib()
        wn, wc = ctx.wn, ctx.wc
        w_src = wc if obfuscate else wn
        saved = rng.getstate()
        version, internal, gauss = saved
        state = np.array(internal[:624], dtype=np.uint32)
        index = ctypes.c_int(internal[624])
        n_words = device.ints_to_words([n], wn)
        out = device.WordArray.empty_device(count, wc)
        chunk = self.STREAM_CHUNK
        nchunks = (count + chunk - 1) // chunk
        pinned = [t.empty((chunk, wn), dtype=t.int32, pin_memory=True) for _ in range(2)]
        staged = [t.empty((chunk, wn), dtype=t.int32, device="cuda") for _ in range(2)]
        copied = [None, None]
        checks = t.empty((nchunks, wc), dtype=t.int32, device="cuda")
        stream = self._stream()
        src_ptr, out_ptr = src.ptr(), out.ptr()
        for k in range(nchunks):
            off = k * chunk
            cnt = min(chunk, count - off)
            which = k & 1
            if copied[which] is not None:
                copied[which].synchronize()            # the upload that last used this pinned buffer is done
            host = pinned[which].numpy()
            _native.check(lib.hb_mt19937_randrange1(state.ctypes.data, ctypes.byref(index), n_words.ctypes.data,
                                                    wn, cnt, host.ctypes.data))
            staged[which][:cnt].copy_(pinned[which][:cnt], non_blocking=True)
            copied[which] = t.cuda.Event()
            copied[which].record()
            r_ptr = staged[which].data_ptr()
            _native.check(lib.hb_unit_product(ctx.handle, r_ptr, checks[k].data_ptr(), cnt, stream))
            call = lib.hb_obfuscate if obfuscate else lib.hb_encrypt
            _native.check(call(ctx.handle, src_ptr + off * w_src * 4, r_ptr, out_ptr + off * wc * 4, cnt, stream))
        products = device.WordArray.from_device(checks).ints()
        if any(math.gcd(p, n) != 1 for p in products):
            rng.setstate(saved)                        # a non-unit was drawn: let the caller redo it the exact way
            return None
        rng.setstate((version, tuple(int(v) for v in state) + (index.value,), gauss))
        return out

    def decrypt(self, n: int, private, c: device.WordArray) -> device.WordArray:
        """private = (p, q, hp, hq, q_inv)."""
        ctx = device.context_for(n)
        ctx.set_private(*private)
        out = device.WordArray.empty_device(c.count, ctx.wn)
        _native.check(self.lib().hb_decrypt(ctx.handle, c.ptr(), out.ptr(), c.count, self._stream()))
        return out

    def mulmod(self, n: int, a: device.WordArray, b: device.WordArray, broadcast_b: bool = False) -> device.WordArray:
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(a.count, ctx.wc)
        _native.check(self.lib().hb_mulmod(ctx.handle, a.ptr(), b.ptr(), out.ptr(), a.count,
                                           1 if broadcast_b else 0, self._stream()))
        return out

    def plain_mulmod(self, n: int, a: device.WordArray, b: device.WordArray, broadcast_b: bool = False) -> device.WordArray:
        """out[i] = a[i] * b[i] mod n on plaintext residues (batches.plain_mul)."""
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(a.count, ctx.wn)
        _native.check(self.lib().hb_plain_mulmod(ctx.handle, a.ptr(), b.ptr(), out.ptr(), a.count,
                                                 1 if broadcast_b else 0, self._stream()))
        return out

    def plain_addmod(self, n: int, a: device.WordArray, b: device.WordArray) -> device.WordArray:
        """out[i] = a[i] + b[i] mod n on plaintext residues (batches.plain_add)."""
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(a.count, ctx.wn)
        _native.check(self.lib().hb_plain_addmod(ctx.handle, a.ptr(), b.ptr(), out.ptr(), a.count, self._stream()))
        return out

    def plain_rescale(self, n: int, m: device.WordArray, digits: int):
        """Signed mantissas times 16^digits, back as residues.  Returns (words, first_bad) where first_bad is the
        smallest index whose value is in the overflow band or leaves max_int after scaling, or -1."""
        ctx = device.context_for(n)
        t = device.torch()
        out = device.WordArray.empty_device(m.count, ctx.wn)
        bad = t.full((1,), -1, dtype=t.int64, device="cuda")
        _native.check(self.lib().hb_plain_rescale(ctx.handle, m.ptr(), int(digits), out.ptr(), m.count,
                                                  bad.data_ptr(), self._stream()))
        return out, int(bad.item())

    def sqrmod(self, n: int, a: device.WordArray, reps: int = 1, throughput_shape: bool = False) -> device.WordArray:
        """out[i] = a[i]^(2^reps) mod n^2 through the kernels' squaring path."""
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(a.count, ctx.wc)
        _native.check(self.lib().hb_sqrmod(ctx.handle, a.ptr(), out.ptr(), a.count, reps,
                                           1 if throughput_shape else 0, self._stream()))
        return out

    def lift_mulmod(self, n: int, a: device.WordArray, m: device.WordArray, broadcast_m: bool = False) -> device.WordArray:
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(a.count, ctx.wc)
        _native.check(self.lib().hb_lift_mulmod(ctx.handle, a.ptr(), m.ptr(), out.ptr(), a.count,
                                                1 if broadcast_m else 0, self._stream()))
        return out

    def powscalar(self, n: int, c: device.WordArray, k: device.WordArray, raw_exponent: bool = False) -> device.WordArray:
        """out[i] = pow_scalar(c[i], k[i % k.count])."""
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(c.count, ctx.wc)
        _native.check(self.lib().hb_powscalar(ctx.handle, c.ptr(), k.ptr(), out.ptr(), c.count, k.count,
                                              1 if raw_exponent else 0, self._stream()))
        return out

    def product(self, n: int, c: device.WordArray, ngroups: int, glen: int, gstride: int, estride: int) -> device.WordArray:
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(ngroups, ctx.wc)
        _native.check(self.lib().hb_product(ctx.handle, c.ptr(), out.ptr(), ngroups, glen, gstride, estride,
                                            self._stream()))
        return out

    def unit_product(self, n: int, r: device.WordArray) -> int:
        """prod r[i] mod n^2 as a Python int (one value crosses back)."""
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(1, ctx.wc)
        _native.check(self.lib().hb_unit_product(ctx.handle, r.ptr(), out.ptr(), r.count, self._stream()))
        return out.ints()[0]

    def draw_units(self, n: int, count: int, rng) -> device.WordArray:
        """`count` obfuscation factors, bit-identical to [draw_unit(n, rng) for _ in range(count)]
        (paillier.py:173-178): the randrange stream comes from the native MT19937 replay of the generator's
        state, the gcd test is one product on the GPU and one gcd.  Falls back to the per-element loop for
        generators that are not exactly random.Random, for small moduli, and if the batch gcd fails."""
        import ctypes
        import math
        import random as _random
        import numpy as np
        from .paillier import draw_unit
        wn = (n.bit_length() + 31) // 32
        if count == 0:
            return device.WordArray.from_ints((), wn)
        if type(rng) is not _random.Random or n.bit_length() < 256 or count < 4:
            return device.WordArray.from_ints([draw_unit(n, rng) for _ in range(count)], wn)
        saved = rng.getstate()
        version, internal, gauss = saved
        state = np.array(internal[:624], dtype=np.uint32)
        index = ctypes.c_int(internal[624])
        n_words = device.ints_to_words([n], wn)
        out = np.empty((count, wn), dtype=np.uint32)
        _native.check(self.lib().hb_mt19937_randrange1(state.ctypes.data, ctypes.byref(index), n_words.ctypes.data,
                                                       wn, count, out.ctypes.data))
        words = device.WordArray.from_numpy(out)
        if math.gcd(self.unit_product(n, words), n) != 1:
            rng.setstate(saved)                       # a non-unit was drawn: redo it the slow, exact way
            return device.WordArray.from_ints([draw_unit(n, rng) for _ in range(count)], wn)
        rng.setstate((version, tuple(int(v) for v in state) + (index.value,), gauss))
        return words

    def matvec(self, n: int, c: device.WordArray, k: device.WordArray, rows: int, inner: int, d: int) -> device.WordArray:
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(rows * d, ctx.wc)
        _native.check(self.lib().hb_matvec(ctx.handle, c.ptr(), k.ptr(), out.ptr(), rows, inner, d, self._stream()))
        return out

    def matvec_partial(self, n: int, c: device.WordArray, k: device.WordArray, inner: int, d: int) -> device.WordArray:
        """This rank's rows reduced to d pairs (A_j, B_j): [2 d, wc] plain words (sharding.sharded_matmul)."""
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(2 * d, ctx.wc)
        if inner == 0:
            one = [1] * (2 * d)
            return device.WordArray.from_ints(one, ctx.wc)
        _native.check(self.lib().hb_matvec_partial(ctx.handle, c.ptr(), k.ptr(), out.ptr(), inner, d, self._stream()))
        return out

    def matvec_combine(self, n: int, ab_all: device.WordArray, nranks: int, d: int) -> device.WordArray:
        ctx = device.context_for(n)
        out = device.WordArray.empty_device(d, ctx.wc)
        _native.check(self.lib().hb_matvec_combine(ctx.handle, ab_all.ptr(), nranks, out.ptr(), d, self._stream()))
        return out

    def encode_f64(self, n: int, values, exponent) -> device.WordArray:
        """values: float64 numpy array (host).  exponent None = the batch's exact shared exponent (min of
        encoding.exact_exponent over the values, batches.py:122-123), computed on the device from the same upload;
        the exponent used is left in `self.last_exponent`.  Raises FixedPointOverflow like encoding.encode."""
        import numpy as np
        from .encoding import FixedPointOverflow
        ctx = device.context_for(n)
        t = device.torch()
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if not np.all(np.isfinite(vals)):
            raise ValueError("cannot encode non-finite values")
        dv = t.from_numpy(vals).cuda()
        if exponent is None:
            lowest = t.full((1,), 2 ** 31 - 1, dtype=t.int32, device="cuda")
            _native.check(self.lib().hb_min_exact_exponent(ctx.handle, dv.data_ptr(), vals.shape[0], lowest.data_ptr(),
                                                           self._stream()))
            exponent = int(lowest.item())
            if exponent == 2 ** 31 - 1:
                exponent = 0
        self.last_exponent = int(exponent)
        out = device.WordArray.empty_device(vals.shape[0], ctx.wn)
        bad = t.full((1,), -1, dtype=t.int64, device="cuda")
        _native.check(self.lib().hb_encode_f64(ctx.handle, dv.data_ptr(), int(exponent), out.ptr(),
                                               vals.shape[0], bad.data_ptr(), self._stream()))
        first = int(bad.item())
        if first >= 0:
            raise FixedPointOverflow(
                f"|{vals[first]}| needs a mantissa beyond max_int at exponent {exponent} (element {first})")
        return out

    def min_exact_exponent(self, n: int, values) -> int:
        """min over the values of encoding.exact_exponent (zeros count as 0; 0 for an empty array), on the device."""
        import numpy as np
        vals = np.ascontiguousarray(values, dtype=np.float64).ravel()
        if vals.shape[0] == 0:
            return 0
        ctx = device.context_for(n)
        t = device.torch()
        dv = t.from_numpy(vals).cuda()
        lowest = t.full((1,), 2 ** 31 - 1, dtype=t.int32, device="cuda")
        _native.check(self.lib().hb_min_exact_exponent(ctx.handle, dv.data_ptr(), vals.shape[0], lowest.data_ptr(),
                                                       self._stream()))
        return int(lowest.item())

    def decode_f64(self, n: int, m: device.WordArray, exponent: int):
        import numpy as np
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
        m = device.WordArray.from_ints([it[0] for it in items], wn)
        r = device.WordArray.from_ints([it[1] for it in items], wn)
        return list(self.encrypt(n, m, r).ints())

    def _run_k_obfuscate(self, common, items):
        n, _ = common
        wn, wc = self._widths(n)
        c = device.WordArray.from_ints([it[0] for it in items], wc)
        r = device.WordArray.from_ints([it[1] for it in items], wn)
        return list(self.obfuscate(n, c, r).ints())

    def _run_k_decrypt(self, common, items):
        p, q, _p2, _q2, hp, hq, q_inv = common
        n = p * q
        _wn, wc = self._widths(n)
        c = device.WordArray.from_ints(items, wc)
        return list(self.decrypt(n, (p, q, hp, hq, q_inv), c).ints())

    def _run_k_mul(self, common, items):
        n, _n2, _neg = common
        wn, wc = self._widths(n)
        c = device.WordArray.from_ints([it[0] for it in items], wc)
        k = device.WordArray.from_ints([it[1] for it in items], wn)
        return list(self.powscalar(n, c, k).ints())

    def _run_k_add(self, common, items):
        n = math.isqrt(common)
        _wn, wc = self._widths(n)
        a = device.WordArray.from_ints([it[0] for it in items], wc)
        b = device.WordArray.from_ints([it[1] for it in items], wc)
        return list(self.mulmod(n, a, b).ints())

    def _run_k_product(self, common, items):
        n = math.isqrt(common)
        _wn, wc = self._widths(n)
        out = []
        # groups of equal length go down in one launch; ragged input falls back to one launch per group
        lengths = {len(g) for g in items}
        if len(lengths) == 1 and next(iter(lengths)) > 0:
            glen = next(iter(lengths))
            flat = device.WordArray.from_ints([v for g in items for v in g], wc)
            return list(self.product(n, flat, len(items), glen, glen, 1).ints())
        for g in items:
            if not g:
                out.append(1 % common)
                continue
            flat = device.WordArray.from_ints(g, wc)
            out.append(self.product(n, flat, 1, len(g), 0, 1).ints()[0])
        return out

    def _run_k_dot(self, common, items):
        n, _n2, _neg, rows, cols = common
        wn, wc = self._widths(n)
        k_rows, inner, d = len(rows), len(rows[0]) if rows else 0, len(cols)
        c = device.WordArray.from_ints([v for row in rows for v in row], wc)
        # cols[j][t] -> row-major inner x d
        k = device.WordArray.from_ints([cols[j][t] for t in range(inner) for j in range(d)], wn)
        full = self.matvec(n, c, k, k_rows, inner, d).ints()
        return [full[i * d + j] for i, j in items]

    def _run_k_encode(self, common, items):
        pk, exponent = common
        import numpy as np
        return list(self.encode_f64(pk.n, np.asarray(items, dtype=np.float64), exponent).ints())

    def _run_k_decode(self, common, items):
        pk, exponent = common
        wn, _wc = self._widths(pk.n)
        return [float(v) for v in self.decode_f64(pk.n, device.WordArray.from_ints(items, wn), exponent)]


_default = None


def default_backend() -> CudaBackend:
    global _default
    if _default is None:
        _default = CudaBackend()
    return _default


def get_backend(name: str, workers: int | None = None) -> ExecutionBackend:
    if name == "cuda":
        return default_backend()
    if name in ("naive", "parallel"):
        raise ValueError(f"backend {name!r} is a CPU backend of the reference package; this build only has 'cuda'")
    raise ValueError(f"unknown backend: {name!r}")
