"""ctypes binding of the C ABI declared in include/hebatch_b200.h.

The library is the product: there is no CPU fallback.  Importing this module does not load the
library (so host-only logic stays importable on a machine without CUDA); the first call to lib()
does, and raises NativeLibraryError loudly if the .so is missing or the symbols do not resolve.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libhebatch_b200.so")

HB_OK = 0
HB_ERR_ARG = -1
HB_ERR_CUDA = -2
HB_ERR_UNSUPPORTED = -3
HB_ERR_NOPRIVATE = -4
HB_ERR_NOTUNIT = -5

# flags of the *_rep entry points / hb_powscalar (include/hebatch_b200.h)
HB_POW_RAW_EXPONENT = 1
HB_A_MONT = 0x10
HB_B_MONT = 0x20
HB_OUT_MONT = 0x40
HB_OPT_MATVEC_WINDOW_BITS = 1
HB_OPT_POOL_KEEP_BYTES = 2
HB_OPT_MATVEC_BLOCK_ROWS = 3


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, was not built, or a call into it failed."""


_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int

# name -> (restype, argtypes).  Mirrors include/hebatch_b200.h one to one; tests/test_capi_symbols.py
# checks that every function declared in the header is listed here and exported by the .so.
SIGNATURES = {
    "hb_last_error": (ctypes.c_char_p, []),
    "hb_version": (ctypes.c_char_p, []),
    "hb_launch_count": (_i64, []),
    "hb_ctx_create": (_int, [ctypes.POINTER(_vp), _vp, _int, _int]),
    "hb_ctx_set_private": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _int]),
    "hb_ctx_destroy": (None, [_vp]),
    "hb_ctx_set_option": (_int, [_vp, _int, _i64]),
    "hb_ct_limbs": (_int, [_vp]),
    "hb_ct_convert": (_int, [_vp, _vp, _vp, _i64, _int, _vp]),
    "hb_encrypt_rep": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "hb_obfuscate_rep": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "hb_decrypt_rep": (_int, [_vp, _vp, _vp, _i64, _int, _vp]),
    "hb_mulmod_rep": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _int, _vp]),
    "hb_lift_mulmod_rep": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _int, _vp]),
    "hb_fore_gradient": (_int, [_vp, _vp, _vp, _vp, ctypes.c_uint32, _vp, _vp, _vp, _i64, _int, _vp]),
    "hb_product_rep": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _int, _vp]),
    "hb_matvec_rep": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _vp]),
    "hb_scalar_compact": (_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "hb_encode_f64_compact": (_int, [_vp, _vp, _int, _i64, _i64, _vp, _vp, _vp, _vp]),
    "hb_matvec_compact": (_int, [_vp, _vp, _vp, _vp, _int, _int, _vp, _i64, _i64, _int, _vp]),
    "hb_matvec_partial_compact": (_int, [_vp, _vp, _vp, _vp, _int, _vp, _i64, _i64, _int, _vp]),
    "hb_secure_randrange1": (_int, [_vp, _int, _i64, _vp]),
    "hb_pt_words": (_int, [_vp]),
    "hb_ct_words": (_int, [_vp]),
    "hb_key_bits": (_int, [_vp]),
    "hb_encrypt": (_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "hb_obfuscate": (_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "hb_decrypt": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "hb_mulmod": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "hb_lift_mulmod": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "hb_sqrmod": (_int, [_vp, _vp, _vp, _i64, _int, _int, _vp]),
    "hb_plain_mulmod": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp]),
    "hb_plain_addmod": (_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "hb_plain_rescale": (_int, [_vp, _vp, _int, _vp, _i64, _vp, _vp]),
    "hb_min_exact_exponent": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "hb_powscalar": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _int, _vp]),
    "hb_product": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp]),
    "hb_unit_product": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "hb_matvec": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "hb_matvec_partial": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    "hb_matvec_combine": (_int, [_vp, _vp, _int, _vp, _i64, _vp]),
    "hb_encode_f64": (_int, [_vp, _vp, _int, _vp, _i64, _vp, _vp]),
    "hb_decode_f64": (_int, [_vp, _vp, _int, _vp, _i64, _vp, _vp]),
    "hb_mt19937_randrange1": (_int, [_vp, _vp, _vp, _int, _i64, _vp]),
    "hb_encrypt_host": (_int, [_vp, _vp, _vp, _vp, _i64]),
    "hb_decrypt_host": (_int, [_vp, _vp, _vp, _i64]),
}

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a).  There is no CPU fallback."
            )
        try:
            handle = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the machine
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            try:
                fn = getattr(handle, name)
            except AttributeError as exc:
                raise NativeLibraryError(f"{LIB_PATH} does not export {name}") from exc
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return _lib


def check(rc: int) -> None:
    """Turn a negative hb_status into the Python exception the reference would raise."""
    if rc == HB_OK:
        return
    msg = lib().hb_last_error().decode("utf-8", "replace")
    if rc == HB_ERR_NOTUNIT:
        raise ZeroDivisionError("invert() no inverse exists")
    if rc == HB_ERR_ARG:
        raise ValueError(f"hebatch_b200: {msg}")
    raise NativeLibraryError(f"hebatch_b200 call failed ({rc}): {msg}")
