"""The C-ABI library loads and exports every function include/hebatch_b200.h declares; the ctypes
signature table covers exactly that set.  No compute calls (CPU only)."""
import ctypes
import os
import re

import pytest

from paper_2107_13797_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hebatch_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_signature_table_agree():
    assert declared_functions() == sorted(_native.SIGNATURES)


def test_library_exports_every_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.fail(f"{_native.LIB_PATH} missing: run __graft_entry__.build()")
    handle = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(handle, name), name
    lib = _native.lib()
    assert b"sm_100a" in lib.hb_version()
    assert lib.hb_launch_count() == 0 or lib.hb_launch_count() > 0


def test_null_context_is_rejected_without_a_gpu():
    lib = _native.lib()
    assert lib.hb_pt_words(None) == 0 and lib.hb_ct_words(None) == 0
    rc = lib.hb_encrypt(None, None, None, None, 4, None)
    assert rc == _native.HB_ERR_ARG
    with pytest.raises(ValueError):
        _native.check(rc)
    assert b"null" in lib.hb_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_native.NativeLibraryError):
        _native.lib()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2107_13797_b200")
    for dirpath, _dirs, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "hebatch_oracle" not in text and "cpuref" not in text and "oracle/" not in text, f
