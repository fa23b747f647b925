"""ctypes binding of libnsg.so (include/nsg.h).

This is the whole Python<->device boundary: the reference binds its C core
through Cython (`_native.pyx:18-73`); here ctypes binds the CUDA library.  A
ctypes call releases the GIL for its duration, mirroring the reference's
`with nogil:` blocks (`_native.pyx:126,185,205`).

There is deliberately NO fallback: if the library is missing or no CUDA
device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import ConfigurationError, CorrectnessFailure, DeviceError, UnsupportedSize

LIB_PATH = Path(__file__).resolve().parent / "libnsg.so"
if os.environ.get("NSG_LIB_PATH"):  # tuning variants only (tools/variants.py)
    LIB_PATH = Path(os.environ["NSG_LIB_PATH"]).resolve()

NSG_OK, NSG_ERR_CHECK, NSG_ERR_SPEC, NSG_ERR_CUDA = 0, -1, -2, -3

# Every symbol include/nsg.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "nsg_run_sorter_many", "nsg_run_sorter_many_host", "nsg_sort_rows", "nsg_sort_rows_host",
    "nsg_segments_ws_bytes", "nsg_sort_segments", "nsg_swap_pairs", "nsg_classify_block",
    "nsg_lcg_next", "nsg_fill_splitmix", "nsg_last_error", "nsg_version",
    "nsg_verify_rows", "nsg_verify_segments",
    "nsg_fill_lcg", "nsg_lcg_jump", "nsg_fingerprint_ws_bytes", "nsg_fingerprint", "nsg_fingerprint_rows",
    "nsg_scan_sorted", "nsg_segments_check", "nsg_rss_fallback_rows",
)


class NsgSpec(ctypes.Structure):
    """`nsg_spec`: the reference's 14 `ns_spec` fields, then the extension."""
    _fields_ = [
        ("kind", ctypes.c_int), ("family", ctypes.c_int), ("swap", ctypes.c_int),
        ("ins_variant", ctypes.c_int), ("base_kind", ctypes.c_int),
        ("rss_oversampling", ctypes.c_int), ("rss_block", ctypes.c_int),
        ("rss_threshold", ctypes.c_int), ("rss_sample_seed", ctypes.c_uint32),
        ("qs_base_is_rss", ctypes.c_int), ("qs_threshold", ctypes.c_int),
        ("qs_depth_factor", ctypes.c_int), ("qs_final_pass", ctypes.c_int),
        ("pivot_swap", ctypes.c_int),
        ("key_dtype", ctypes.c_int), ("payload_dtype", ctypes.c_int),
        ("descending", ctypes.c_int), ("tie_mode", ctypes.c_int),
    ]


def make_spec(spec, order=None) -> NsgSpec:
    """Positional copy of a SorterSpec (+ DeviceOrder) into the C struct."""
    from .registry import DeviceOrder
    order = order or DeviceOrder()
    vals = [int(x) for x in tuple(spec)] + [int(x) for x in tuple(order)]
    vals[8] &= 0xFFFFFFFF
    return NsgSpec(*vals)


_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_SIGS = {
    "nsg_run_sorter_many": (ctypes.c_int, [ctypes.POINTER(NsgSpec), _P, _I64, _I64, _P]),
    "nsg_run_sorter_many_host": (ctypes.c_int, [ctypes.POINTER(NsgSpec), _P, _I64, _I64]),
    "nsg_sort_rows": (ctypes.c_int, [ctypes.POINTER(NsgSpec), _P, _P, _P, _P, _I64, _I64, _P]),
    "nsg_sort_rows_host": (ctypes.c_int, [ctypes.POINTER(NsgSpec), _P, _P, _P, _P, _I64, _I64]),
    "nsg_segments_ws_bytes": (ctypes.c_size_t, [_I64, _I64]),
    "nsg_sort_segments": (ctypes.c_int, [ctypes.POINTER(NsgSpec), _P, _I64, _P, _P, _P, _P, _P,
                                         ctypes.c_size_t, _P]),
    "nsg_swap_pairs": (ctypes.c_int, [ctypes.c_int, _P, _I64, _P]),
    "nsg_classify_block": (ctypes.c_int, [_P, _I64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_uint64, ctypes.c_int, _P, _P]),
    "nsg_lcg_next": (ctypes.c_uint32, [ctypes.c_uint32]),
    "nsg_fill_splitmix": (ctypes.c_int, [_P, _I64, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _P]),
    "nsg_verify_rows": (ctypes.c_int, [ctypes.POINTER(NsgSpec), _P, _P, _P, _P, _I64, _I64, _P, _P]),
    "nsg_verify_segments": (ctypes.c_int, [ctypes.POINTER(NsgSpec), _P, _I64, _P, _P, _P, _P, _P, _P]),
    "nsg_fill_lcg": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32),
                                    _P]),
    "nsg_lcg_jump": (ctypes.c_uint32, [ctypes.c_uint32, ctypes.c_uint64]),
    "nsg_fingerprint_ws_bytes": (ctypes.c_size_t, []),
    "nsg_fingerprint": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, ctypes.c_uint64, _P, ctypes.c_size_t, _P,
                                       _P]),
    "nsg_fingerprint_rows": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _I64, ctypes.c_uint64, _P, _P]),
    "nsg_scan_sorted": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _P, _P]),
    "nsg_segments_check": (ctypes.c_int, [_P, _P]),
    "nsg_rss_fallback_rows": (ctypes.c_ulonglong, [ctypes.c_int]),
    "nsg_last_error": (ctypes.c_char_p, []),
    "nsg_version": (ctypes.c_int, []),
}


def load_library() -> ctypes.CDLL:
    """Load libnsg.so without touching the GPU (safe on CPU-only hosts)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is not built; run `python -m paper_2002_05599_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def lib() -> ctypes.CDLL:
    """The library, after checking that a CUDA device is present."""
    l = load_library()
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 sorter has no CPU fallback")
    torch.cuda.init()
    return l


def check(rc: int, *, network: bool = False, seed=None) -> None:
    """Map a status code exactly like the reference (`_native.pyx:153-160`)."""
    if rc == NSG_OK:
        return
    msg = (load_library().nsg_last_error() or b"").decode(errors="replace")
    if rc == NSG_ERR_CHECK:
        raise CorrectnessFailure(msg or "sorted-check or fingerprint mismatch", seed=seed)
    if rc == NSG_ERR_SPEC:
        if network:
            raise UnsupportedSize(msg or "network sorters cover 2..16 items")
        raise ConfigurationError(msg or "sorter spec rejected by the device lane")
    raise DeviceError(msg or f"device error {rc}")


def current_stream_handle(device=None) -> int:
    import torch
    return int(torch.cuda.current_stream(device).cuda_stream)


def env_flag(name: str) -> bool:
    return os.environ.get(name, "").strip() not in ("", "0", "false", "no")
