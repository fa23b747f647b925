"""How do fixed per-launch costs show up?  Time one network cell at several
batch sizes (GB/s should be flat if the kernel is purely bandwidth bound).

    python tools/rowscale.py
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2002_05599_b200 import _lib, registry
    l = _lib.lib()
    dev = torch.device("cuda")
    sh = _lib.current_stream_handle()
    for n, kb, pb in ((4, 8, 0), (2, 8, 0), (16, 8, 4)):
        for lg in (20, 22, 24, 26):
            rows = 1 << lg
            k = torch.empty(rows * n * kb, dtype=torch.uint8, device=dev)
            _lib.check(l.nsg_fill_splitmix(k.data_ptr(), rows * n, kb, 3, 0, sh))
            ko = torch.empty_like(k)
            p = torch.zeros(rows * n * pb, dtype=torch.uint8, device=dev) if pb else None
            po = torch.empty_like(p) if pb else None
            order = registry.DeviceOrder(registry.KEY_U64, {0: 0, 4: 1}[pb], 0, registry.TIE_UNIQUE)
            sp = _lib.make_spec(registry.spec_network("best", "4CmS"), order)

            def run():
                l.nsg_sort_rows(sp, k.data_ptr(), ko.data_ptr(), p.data_ptr() if pb else None,
                                po.data_ptr() if pb else None, rows, n, sh)
            for _ in range(3):
                run()
            # single launches and a back-to-back burst of 10
            ts = []
            for _ in range(5):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                run()
                e.record()
                e.synchronize()
                ts.append(s.elapsed_time(e))
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                run()
            e.record()
            e.synchronize()
            burst = s.elapsed_time(e) / 10
            nbytes = 2 * rows * n * (kb + pb)
            print(json.dumps({"n": n, "kb": kb, "pb": pb, "rows": rows, "single_ms": round(float(np.median(ts)), 4),
                              "burst_ms": round(burst, 4),
                              "single_gbs": round(nbytes / (np.median(ts) / 1e3) / 1e9, 1),
                              "burst_gbs": round(nbytes / (burst / 1e3) / 1e9, 1)}), flush=True)
            del k, ko, p, po
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
