"""ctypes binding of the sm_100a C-ABI library `libgtopk_b200.so`.

The library is built in-tree (`make` / `__graft_entry__.build()`).  There is
no fallback: if the library is missing or no CUDA device is visible, every
hot-path call raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# GTK_LIB_PATH: an alternative in-tree build (A/B measurements of compile-time variants)
LIB_PATH = os.environ.get("GTK_LIB_PATH") or os.path.join(_HERE, "libgtopk_b200.so")

GTK_OK = 0
GTK_EINVAL = 1
GTK_ENONFINITE = 2
GTK_EPROTO = 3
GTK_ETIMEOUT = 4
GTK_ECUDA = 5
GTK_ENOMEM = 6
GTK_EABORTED = 7

DEV_NONFINITE = 0x1
DEV_FALLBACK = 0x2
DEV_TIMEOUT = 0x4
DEV_ABORTED = 0x8
DEV_PEER_FAILED = 0x10
DEV_PENDING = 0x20
DEV_ERROR_MASK = 0x3D

SELECT_FORCE_EXACT = 0x1
SELECT_CHAIN = 0x2
STEP_PREPUSHED = 0x10000

# every symbol include/gtopk_b200.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "gtk_version",
    "gtk_strerror",
    "gtk_last_cuda_error",
    "gtk_select_workspace_bytes",
    "gtk_workspace_init",
    "gtk_select",
    "gtk_select_windowed",
    "gtk_select_update",
    "gtk_select_push",
    "gtk_select_main_pass",
    "gtk_select_settle",
    "gtk_select_update_deferred",
    "gtk_select_push_deferred",
    "gtk_select_settle_global",
    "gtk_merge_workspace_bytes",
    "gtk_top_op",
    "gtk_scatter_update",
    "gtk_dense_apply",
    "gtk_densify",
    "gtk_topk_accumulate",
    "gtk_topk_apply",
    "gtk_dense_sum",
    "gtk_dense_ring_sum",
    "gtk_divergence_terms",
    "gtk_status_read",
    "gtk_exchange_inbox_bytes",
    "gtk_dev_alloc",
    "gtk_dev_free",
    "gtk_ipc_get_handle",
    "gtk_ipc_open_handle",
    "gtk_ipc_close_handle",
    "gtk_abort_word_create",
    "gtk_abort_word_set",
    "gtk_abort_word_destroy",
    "gtk_gtopk_exchange",
    "gtk_gtopk_exchange_update",
    "gtk_prof_enable",
    "gtk_prof_read",
    "gtk_prof_reset",
    "gtk_prof_graph_read",
    "gtk_launch_count",
    "gtk_exchange_set_trace",
)

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_F = ctypes.c_float
_SZ = ctypes.c_size_t

_SIGS = {
    "gtk_version": ([], _I32),
    "gtk_strerror": ([_I32], ctypes.c_char_p),
    "gtk_last_cuda_error": ([], ctypes.c_char_p),
    "gtk_select_workspace_bytes": ([_I64, _I32, ctypes.POINTER(_SZ)], _I32),
    "gtk_workspace_init": ([_P, _SZ, _P], _I32),
    "gtk_select": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _I32, _P], _I32),
    "gtk_select_windowed": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _I32, _P, _P], _I32),
    "gtk_select_update": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _I32, _P, _P, _F, _I32, _I32, _P], _I32),
    "gtk_select_push_deferred": (
        [_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _P, _P, _P, _P, _P, _P, _P, _P],
        _I32,
    ),
    "gtk_select_settle_global": ([_P, _P, _P, _P, _P, _P], _I32),
    "gtk_select_update_deferred": (
        [_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _P, _P, _P, _P, _P, _F, _I32, _I32, _P],
        _I32,
    ),
    "gtk_select_push": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _SZ, _I32, _P, _P, _P, _P], _I32),
    "gtk_select_main_pass": ([_P, _P, _P, _I64, _I32, _P, _SZ, _I32, _P], _I32),
    "gtk_select_settle": ([_P, _P, _P, _P, _P], _I32),
    "gtk_merge_workspace_bytes": ([_I32, _I32, ctypes.POINTER(_SZ)], _I32),
    "gtk_top_op": ([_P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _SZ, _P], _I32),
    "gtk_scatter_update": (
        [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _F, _F, _I32, _I32, _P, _P],
        _I32,
    ),
    "gtk_dense_apply": ([_P, _P, _P, _I64, _F, _F, _I32, _P], _I32),
    "gtk_densify": ([_P, _P, _P, _I64, _P, _P], _I32),
    "gtk_topk_accumulate": ([_P, _P, _P, _I32, _I64, _I64, _P, _I32, _P], _I32),
    "gtk_topk_apply": ([_P, _P, _P, _I32, _I64, _I64, _P, _P, _F, _I32, _P, _I64, _P, _P], _I32),
    "gtk_dense_sum": ([_P, _I32, _I64, _P, _P], _I32),
    "gtk_dense_ring_sum": ([_P, _I32, _I64, _P, _P], _I32),
    "gtk_divergence_terms": ([_P, _P, _P, _P, _P, _P, _I64, _P, _P, _P], _I32),
    "gtk_status_read": ([_P, _P, _P, _I32, _P], _I32),
    "gtk_exchange_inbox_bytes": ([_I32, _I32, ctypes.POINTER(_SZ)], _I32),
    "gtk_dev_alloc": ([_SZ, ctypes.POINTER(_P)], _I32),
    "gtk_dev_free": ([_P], _I32),
    "gtk_ipc_get_handle": ([_P, _P], _I32),
    "gtk_ipc_open_handle": ([_P, ctypes.POINTER(_P)], _I32),
    "gtk_ipc_close_handle": ([_P], _I32),
    "gtk_abort_word_create": ([ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32)),
                               ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32))], _I32),
    "gtk_abort_word_set": ([ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint32], _I32),
    "gtk_abort_word_destroy": ([ctypes.POINTER(ctypes.c_uint32)], _I32),
    "gtk_gtopk_exchange": (
        [_I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P],
        _I32,
    ),
    "gtk_gtopk_exchange_update": (
        [_I32, _I32, _P, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P, _P, _F,
         _I32, _P, _P],
        _I32,
    ),
    "gtk_prof_enable": ([_I32], _I32),
    "gtk_prof_read": ([_I32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)], _I32),
    "gtk_prof_reset": ([], _I32),
    "gtk_prof_graph_read": ([_I32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)], _I32),
    "gtk_launch_count": ([], _I64),
    "gtk_exchange_set_trace": ([_P], _I32),
}

PROF_SELECT_MAIN = 0
PROF_SELECT = 1
PROF_EXCHANGE = 2
PROF_MERGE = 3
PROF_UPDATE = 4


def prof_read(pid: int):
    """(total_ms, count) of a profiled launch site (synchronises)."""
    tot, cnt = ctypes.c_double(), _I64()
    check(load().gtk_prof_read(pid, ctypes.byref(tot), ctypes.byref(cnt)), "gtk_prof_read")
    return tot.value, cnt.value


def prof_graph_read(pid: int):
    """(ms, count) of the graph-captured pairs of a launch site, as of the
    last (synchronised) replay."""
    tot, cnt = ctypes.c_double(), _I64()
    check(load().gtk_prof_graph_read(pid, ctypes.byref(tot), ctypes.byref(cnt)), "gtk_prof_graph_read")
    return tot.value, cnt.value

_lock = threading.Lock()
_lib = None


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or no GPU is available."""


def load(require_symbols: bool = True):
    """Load (once) and return the ctypes handle; raises NativeLibraryError."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `make` or __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - environment specific
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                if require_symbols:
                    raise NativeLibraryError(f"{LIB_PATH} lacks symbol {name}")
                continue
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def strerror(code: int) -> str:
    return load().gtk_strerror(code).decode()


def check(code: int, what: str = "") -> None:
    """Map a host status code to the reference's exception types."""
    if code == GTK_OK:
        return
    from .transport import ProtocolError, TransportError

    msg = f"{what}: {strerror(code)}" if what else strerror(code)
    if code == GTK_EINVAL:
        raise ValueError(msg)
    if code == GTK_ENONFINITE:
        raise FloatingPointError("non-finite values in dense input")
    if code == GTK_EPROTO:
        raise ProtocolError(msg)
    if code in (GTK_ETIMEOUT, GTK_EABORTED):
        raise TransportError(msg)
    if code == GTK_ECUDA:
        raise RuntimeError(f"{msg}: {load().gtk_last_cuda_error().decode()}")
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
