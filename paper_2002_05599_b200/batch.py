"""Typed batched front ends: fixed-width rows (SoA) and CSR segments.

These are the entry points the BASELINE configurations exercise; the
reference only has the AoS `run_sorter_many` (its adapters are SURVEY 8(c)).

  sort_rows(keys, payload=None, ...)      B rows of n keys (+ payload), row-major
  sort_segments(offsets, keys, payload=None, ...)   CSR segments (lengths 0..16)

Inputs may be CUDA tensors (device-resident; stream-ordered on torch's current
stream; returns tensors) or numpy arrays (host; the library pipelines H2D,
sort and D2H; returns numpy arrays).
"""

from __future__ import annotations

import numpy as np

from . import networks as nw
from . import registry
from ._lib import check, current_stream_handle, lib, make_spec
from ._lib import check as _check
from .errors import ConfigurationError
from .registry import DeviceOrder

_KEY = {"uint32": registry.KEY_U32, "uint64": registry.KEY_U64, "int32": registry.KEY_I32,
        "int64": registry.KEY_I64, "float32": registry.KEY_F32, "float64": registry.KEY_F64}
_PAY = {"uint32": registry.PAY_U32, "int32": registry.PAY_U32, "uint64": registry.PAY_U64,
        "int64": registry.PAY_U64}


def _dtname(x) -> str:
    d = x.dtype
    return str(d).replace("torch.", "")


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def make_order(keys, payload, descending: bool, tie: str) -> DeviceOrder:
    kd = _KEY.get(_dtname(keys))
    if kd is None:
        raise ConfigurationError(f"unsupported key dtype {keys.dtype}")
    pd = registry.PAY_NONE
    if payload is not None:
        pd = _PAY.get(_dtname(payload))
        if pd is None:
            raise ConfigurationError(f"unsupported payload dtype {payload.dtype}")
    if tie not in ("ref", "unique"):
        raise ConfigurationError("tie must be 'ref' (key-only, reference semantics) or 'unique'")
    return DeviceOrder(kd, pd, int(bool(descending)),
                       registry.TIE_UNIQUE if tie == "unique" else registry.TIE_REF)


def make_row_spec(kind: str, family: str, swap: str, rss_cfg: str, rss_base: str):
    if kind == "network":
        return registry.spec_network(family, swap)
    if kind == "rss":
        return registry.spec_rss(rss_cfg, rss_base)
    if kind == "insertion":
        return registry.spec_insertion("Def")
    if kind == "merge":
        return registry.spec_merge(family)
    raise ConfigurationError(f"unknown kind {kind!r}")


def sort_rows(keys, payload=None, *, kind: str = "network", family: str = "best", swap: str = "4CmS",
              descending: bool = False, tie: str = "unique", rss_cfg: str = "332",
              rss_base: str = "SN Best 4CmS", out_keys=None, out_payload=None):
    """Sort each row of a (rows, n) key matrix (and its payload) independently."""
    if keys.ndim != 2:
        raise ConfigurationError("keys must be a 2-D (rows, n) array")
    if payload is not None and tuple(payload.shape) != tuple(keys.shape):
        raise ConfigurationError("payload must have the keys' shape")
    rows, n = int(keys.shape[0]), int(keys.shape[1])
    spec = make_row_spec(kind, family, swap, rss_cfg, rss_base)
    if kind == "network" and n > nw.MAX_UNROLLED:
        from .errors import UnsupportedSize
        raise UnsupportedSize(f"network sorters cover at most {nw.MAX_UNROLLED} items, got {n}")
    sp = make_spec(spec, make_order(keys, payload, descending, tie))
    l = lib()
    if _is_torch(keys):
        if not keys.is_cuda or not keys.is_contiguous():
            raise ConfigurationError("keys must be a contiguous CUDA tensor")
        for t in (keys, payload, out_keys, out_payload):
            if t is not None and t.data_ptr() % 16:
                raise ConfigurationError("device buffers must be 16-byte aligned")
        ok = out_keys if out_keys is not None else keys.new_empty(keys.shape)
        op = None
        if payload is not None:
            if not payload.is_cuda or not payload.is_contiguous():
                raise ConfigurationError("payload must be a contiguous CUDA tensor")
            op = out_payload if out_payload is not None else payload.new_empty(payload.shape)
        rc = l.nsg_sort_rows(sp, keys.data_ptr(), ok.data_ptr(),
                             payload.data_ptr() if payload is not None else None,
                             op.data_ptr() if op is not None else None, rows, n,
                             current_stream_handle(keys.device))
        check(rc, network=kind == "network")
        return ok, op
    keys = np.ascontiguousarray(keys)
    ok = out_keys if out_keys is not None else np.empty_like(keys)
    op = None
    if payload is not None:
        payload = np.ascontiguousarray(payload)
        op = out_payload if out_payload is not None else np.empty_like(payload)
    rc = l.nsg_sort_rows_host(sp, keys.ctypes.data, ok.ctypes.data,
                              payload.ctypes.data if payload is not None else None,
                              op.ctypes.data if op is not None else None, rows, n)
    check(rc, network=kind == "network")
    return ok, op


def verify_rows(keys_in, keys_out, payload_in=None, payload_out=None, *, descending: bool = False,
                tie: str = "unique") -> int:
    """On-device check of a sort_rows result (CUDA tensors): number of rows that
    are not ordered or not a permutation of their input (0 = all good)."""
    import torch
    rows, n = int(keys_in.shape[0]), int(keys_in.shape[1])
    sp = make_spec(registry.spec_network("best", "4CmS"), make_order(keys_in, payload_in, descending, tie))
    bad = torch.zeros(1, dtype=torch.int64, device=keys_in.device)
    check(lib().nsg_verify_rows(sp, keys_in.data_ptr(), payload_in.data_ptr() if payload_in is not None else None,
                                keys_out.data_ptr(), payload_out.data_ptr() if payload_out is not None else None,
                                rows, n, bad.data_ptr(), current_stream_handle(keys_in.device)))
    return int(bad.item())


def verify_segments(offsets, keys_in, keys_out, payload_in=None, payload_out=None, *, descending: bool = False,
                    tie: str = "unique") -> int:
    """On-device check of a sort_segments result (CUDA tensors): bad segment count."""
    import torch
    sp = make_spec(registry.spec_network("best", "4CmS"), make_order(keys_in, payload_in, descending, tie))
    bad = torch.zeros(1, dtype=torch.int64, device=keys_in.device)
    check(lib().nsg_verify_segments(sp, offsets.data_ptr(), int(offsets.numel()) - 1, keys_in.data_ptr(),
                                    payload_in.data_ptr() if payload_in is not None else None, keys_out.data_ptr(),
                                    payload_out.data_ptr() if payload_out is not None else None, bad.data_ptr(),
                                    current_stream_handle(keys_in.device)))
    return int(bad.item())


def sort_segments(offsets, keys, payload=None, *, family: str = "best", swap: str = "4CmS",
                  descending: bool = False, tie: str = "unique", out_keys=None, out_payload=None,
                  workspace=None, check: bool = True):
    """Sort CSR segments [offsets[s], offsets[s+1]) of keys (+payload), on device.

    Segments of up to 1024 items are supported; with `check` (default) the
    call synchronises and raises ConfigurationError if a longer one was
    present (it is left unsorted).  `check=False` keeps the call fully
    asynchronous for callers that bound their segment lengths."""
    import torch
    if not _is_torch(keys) or not keys.is_cuda:
        host = True
        dev = torch.device("cuda")
        offsets_t = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.uint32)).to(dev)
        keys_t = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
        pay_t = torch.from_numpy(np.ascontiguousarray(payload)).to(dev) if payload is not None else None
    else:
        host = False
        offsets_t, keys_t, pay_t = offsets, keys, payload
    nseg = int(offsets_t.numel()) - 1
    nelem = int(keys_t.numel())
    spec = registry.spec_network(family, swap)
    sp = make_spec(spec, make_order(keys_t, pay_t, descending, tie))
    l = lib()
    ok = out_keys if (out_keys is not None and not host) else torch.empty_like(keys_t)
    op = None
    if pay_t is not None:
        op = out_payload if (out_payload is not None and not host) else torch.empty_like(pay_t)
    ws_bytes = int(l.nsg_segments_ws_bytes(nseg, nelem))
    ws = workspace if workspace is not None else torch.empty(max(ws_bytes, 1), dtype=torch.uint8,
                                                              device=keys_t.device)
    rc = l.nsg_sort_segments(sp, offsets_t.data_ptr(), nseg, keys_t.data_ptr(), ok.data_ptr(),
                             pay_t.data_ptr() if pay_t is not None else None,
                             op.data_ptr() if op is not None else None, ws.data_ptr(), ws_bytes,
                             current_stream_handle(keys_t.device))
    _check(rc, network=False)
    if check or host:
        _check(l.nsg_segments_check(ws.data_ptr(), current_stream_handle(keys_t.device)))
    if host:
        return ok.cpu().numpy(), (op.cpu().numpy() if op is not None else None)
    return ok, op
