"""The C-ABI library loads without a GPU and exports every entry point that
include/gtopk_b200.h declares; host-only calls (sizes, argument validation,
error strings) work on CPU.  No kernel is launched here."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "gtopk_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gtk_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1901_04359_b200 import _lib

    return _lib.load()


def test_header_and_binding_agree():
    from paper_1901_04359_b200 import _lib

    assert declared_functions() == sorted(_lib.EXPORTS)
    assert set(_lib._SIGS) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_shared_object_is_sm100a():
    so = os.path.join(ROOT, "paper_1901_04359_b200", "libgtopk_b200.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_version_and_strerror(lib):
    assert lib.gtk_version() >= 10000
    assert lib.gtk_strerror(0) == b"ok"
    assert lib.gtk_strerror(2) == b"non-finite values in dense input"


def test_workspace_sizes(lib):
    n = ctypes.c_size_t()
    assert lib.gtk_select_workspace_bytes(25_600_000, 25_600, ctypes.byref(n)) == 0
    assert n.value > 0 and n.value < 1 << 30
    assert lib.gtk_select_workspace_bytes(10, 11, ctypes.byref(n)) == 1  # k > m
    assert lib.gtk_select_workspace_bytes(1 << 31, 10, ctypes.byref(n)) == 1  # m >= 2^31
    assert lib.gtk_merge_workspace_bytes(25_600, 25_600, ctypes.byref(n)) == 0 and n.value > 0
    assert lib.gtk_exchange_inbox_bytes(1000, 3, ctypes.byref(n)) == 0
    assert n.value >= 2 * 3 * (16 + 16 * 1000)  # 2 call parities x 3 steps of LL slots
    assert lib.gtk_exchange_inbox_bytes(1000, 65, ctypes.byref(n)) == 1  # > kMaxSteps


def test_argument_validation_without_gpu(lib):
    from paper_1901_04359_b200 import _lib

    null = None
    # invalid arguments are rejected before any CUDA call
    assert lib.gtk_select(null, null, null, 10, 1, null, null, null, null, null, 0, 0, null) == _lib.GTK_EINVAL
    assert lib.gtk_top_op(null, null, null, null, null, null, 1, 0, null, null, null, null, 0, null) == _lib.GTK_EINVAL
    assert lib.gtk_gtopk_exchange(0, 0, null, 0, null, null, null, null, null, 1, null, null, 0, null,
                                  null, null, null, null, 0, null) == _lib.GTK_EINVAL
    assert lib.gtk_abort_word_create(None, None) == _lib.GTK_EINVAL
    assert lib.gtk_abort_word_set(None, 1) == _lib.GTK_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.GTK_EINVAL, "x")
    with pytest.raises(FloatingPointError):
        _lib.check(_lib.GTK_ENONFINITE)
    from paper_1901_04359_b200.transport import ProtocolError, TransportError

    with pytest.raises(ProtocolError):
        _lib.check(_lib.GTK_EPROTO)
    with pytest.raises(TransportError):
        _lib.check(_lib.GTK_ETIMEOUT)


def test_no_cpu_fallback_without_gpu():
    """On a machine without a GPU the hot path fails loudly."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import numpy as np

    import paper_1901_04359_b200 as gk
    from paper_1901_04359_b200._lib import NativeLibraryError

    with pytest.raises(NativeLibraryError):
        gk.top_k_select(np.ones(8, np.float32), 2)
