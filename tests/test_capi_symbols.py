"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/nsg.h declares (no compute calls without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2002_05599_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "nsg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nsg_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_binding_surface():
    assert header_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.nsg_version() >= 100


def test_host_only_entry_points():
    lib = _lib.load_library()
    # lcg goldens (reference test_bench.py:21-35 / acceptance A09)
    assert lib.nsg_lcg_next(1) == 48271
    assert lib.nsg_lcg_next(48271) == 182605794
    s = 1
    for _ in range(10000):
        s = lib.nsg_lcg_next(s)
    assert s == 399268537
    assert lib.nsg_segments_ws_bytes(0, 0) >= 0


def test_spec_rejections_need_no_gpu():
    lib = _lib.load_library()
    from paper_2002_05599_b200 import registry
    sp = _lib.make_spec(registry.spec_network("best", "4CmS"))
    sp.family = 7
    assert lib.nsg_sort_rows(ctypes.byref(sp), None, None, None, None, 1, 8, None) == _lib.NSG_ERR_SPEC
    assert b"family" in lib.nsg_last_error()
    assert lib.nsg_swap_pairs(11, None, 1, None) == _lib.NSG_ERR_SPEC


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2002_05599_b200 import backend, registry
    from paper_2002_05599_b200.errors import DeviceError
    from paper_2002_05599_b200.items import items_from_keys
    with pytest.raises(DeviceError):
        backend.run_sorter(registry.spec_network("best", "4CmS"), items_from_keys([3, 1, 2]), 3)
