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


def _check_out(out, ref, what: str, device=None) -> None:
    """An output buffer must match its input's shape and element size, be
    contiguous and (device path) live on the input's CUDA device."""
    if out is None:
        return
    if tuple(out.shape) != tuple(ref.shape):
        raise ConfigurationError(f"{what} must have shape {tuple(ref.shape)}, got {tuple(out.shape)}")
    if device is not None:
        if not _is_torch(out) or not out.is_cuda or out.device != device:
            raise ConfigurationError(f"{what} must be a CUDA tensor on {device}")
        if out.element_size() != ref.element_size() or not out.is_contiguous():
            raise ConfigurationError(f"{what} must be contiguous with element size {ref.element_size()}")
    else:
        if not isinstance(out, np.ndarray) or out.itemsize != ref.itemsize or not out.flags.c_contiguous \
                or not out.flags.writeable:
            raise ConfigurationError(f"{what} must be a writeable C-contiguous numpy array "
                                     f"with item size {ref.itemsize}")


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
        import torch
        if not keys.is_cuda or not keys.is_contiguous():
            raise ConfigurationError("keys must be a contiguous CUDA tensor")
        if payload is not None and (not _is_torch(payload) or not payload.is_cuda
                                    or payload.device != keys.device or not payload.is_contiguous()):
            raise ConfigurationError("payload must be a contiguous CUDA tensor on the keys' device")
        _check_out(out_keys, keys, "out_keys", keys.device)
        if out_payload is not None and payload is None:
            raise ConfigurationError("out_payload given without a payload")
        _check_out(out_payload, payload, "out_payload", keys.device)
        for t in (keys, payload, out_keys, out_payload):
            if t is not None and t.data_ptr() % 16:
                raise ConfigurationError("device buffers must be 16-byte aligned")
        ok = out_keys if out_keys is not None else keys.new_empty(keys.shape)
        op = None
        if payload is not None:
            op = out_payload if out_payload is not None else payload.new_empty(payload.shape)
        with torch.cuda.device(keys.device):
            rc = l.nsg_sort_rows(sp, keys.data_ptr(), ok.data_ptr(),
                                 payload.data_ptr() if payload is not None else None,
                                 op.data_ptr() if op is not None else None, rows, n,
                                 current_stream_handle(keys.device))
        check(rc, network=kind == "network")
        return ok, op
    keys = np.ascontiguousarray(keys)
    _check_out(out_keys, keys, "out_keys")
    ok = out_keys if out_keys is not None else np.empty_like(keys)
    op = None
    if payload is not None:
        payload = np.ascontiguousarray(payload)
        _check_out(out_payload, payload, "out_payload")
        op = out_payload if out_payload is not None else np.empty_like(payload)
    elif out_payload is not None:
        raise ConfigurationError("out_payload given without a payload")
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

    Keys-only and UNIQUE segments of any length up to the CTA sorter's
    shared-memory capacity (8192 16-byte / 16384 8-byte / 32768 4-byte items)
    are sorted; REF mode with a payload covers up to 1024 items.  With `check`
    (default) the call synchronises and raises ConfigurationError if a longer
    one was present (it is left unsorted).  `check=False` keeps the call fully
    asynchronous for callers that bound their segment lengths."""
    import torch
    if not _is_torch(keys) or not keys.is_cuda:
        host = True
        dev = torch.device("cuda", torch.cuda.current_device())
        offs = np.asarray(offsets)
        if offs.ndim != 1 or offs.size < 1:
            raise ConfigurationError("offsets must be a 1-D array of nseg+1 entries")
        if offs.size > 1 and (int(offs.min()) < 0 or int(offs[-1]) >= 1 << 32):
            raise ConfigurationError("offsets must lie in [0, 2^32)")
        offsets_t = torch.from_numpy(np.ascontiguousarray(offs, dtype=np.uint32).view(np.int32)).to(dev)
        keys_t = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
        pay_t = torch.from_numpy(np.ascontiguousarray(payload)).to(dev) if payload is not None else None
    else:
        host = False
        offsets_t, keys_t, pay_t = offsets, keys, payload
        dev = keys_t.device
        if not _is_torch(offsets_t) or not offsets_t.is_cuda or offsets_t.device != dev \
                or offsets_t.dtype not in (torch.int32, torch.uint32) or not offsets_t.is_contiguous() \
                or offsets_t.dim() != 1:
            raise ConfigurationError("offsets must be a contiguous 1-D int32/uint32 CUDA tensor on the keys' device")
        if not keys_t.is_contiguous():
            raise ConfigurationError("keys must be contiguous")
        if pay_t is not None and (not _is_torch(pay_t) or not pay_t.is_cuda or pay_t.device != dev
                                  or not pay_t.is_contiguous()):
            raise ConfigurationError("payload must be a contiguous CUDA tensor on the keys' device")
        _check_out(out_keys, keys_t, "out_keys", dev)
        if out_payload is not None and pay_t is None:
            raise ConfigurationError("out_payload given without a payload")
        _check_out(out_payload, pay_t, "out_payload", dev)
    if pay_t is not None and pay_t.numel() != keys_t.numel():
        raise ConfigurationError("payload must hold one entry per key")
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
    if workspace is not None:
        if not _is_torch(workspace) or not workspace.is_cuda or workspace.device != dev \
                or not workspace.is_contiguous():
            raise ConfigurationError("workspace must be a contiguous CUDA tensor on the keys' device")
        ws = workspace
        ws_have = int(workspace.numel()) * int(workspace.element_size())
        if ws_have < ws_bytes:
            raise ConfigurationError(f"workspace holds {ws_have} bytes, need {ws_bytes} "
                                     "(nsg_segments_ws_bytes)")
    else:
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
        ws_have = int(ws.numel())
    with torch.cuda.device(dev):
        rc = l.nsg_sort_segments(sp, offsets_t.data_ptr(), nseg, keys_t.data_ptr(), ok.data_ptr(),
                                 pay_t.data_ptr() if pay_t is not None else None,
                                 op.data_ptr() if op is not None else None, ws.data_ptr(), ws_have,
                                 current_stream_handle(dev))
        _check(rc, network=False)
        if check or host:
            _check(l.nsg_segments_check(ws.data_ptr(), current_stream_handle(dev)))
    if host:
        return ok.cpu().numpy(), (op.cpu().numpy() if op is not None else None)
    return ok, op
