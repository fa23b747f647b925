"""The reference's item record (`items.py:14`): packed little-endian
(u64 key, u64 ref), 16 bytes.  The AoS lane of the device library sorts rows of
exactly this layout in place (`nsg_run_sorter_many`)."""

import numpy as np

KEY_BITS = 64
ITEM_BYTES = 16
ITEM_DTYPE = np.dtype([("key", "<u8"), ("ref", "<u8")], align=False)


def empty_items(n: int) -> np.ndarray:
    return np.zeros(n, dtype=ITEM_DTYPE)


def items_from_pairs(pairs) -> np.ndarray:
    pairs = list(pairs)
    arr = empty_items(len(pairs))
    if pairs:
        arr["key"] = np.array([int(k) for k, _ in pairs], dtype=np.uint64)
        arr["ref"] = np.array([int(r) for _, r in pairs], dtype=np.uint64)
    return arr


def items_from_keys(keys) -> np.ndarray:
    """Items with ref = original index (tracks payload transport)."""
    keys = np.asarray(list(keys), dtype=np.uint64)
    arr = empty_items(len(keys))
    arr["key"] = keys
    arr["ref"] = np.arange(len(keys), dtype=np.uint64)
    return arr
