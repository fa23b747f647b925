"""Tuning sweep for the network kernel's compile-time knobs.

    python tools/variants.py build            # here: compile the variants
    python tools/variants.py time             # on the GPU: time every variant

Each variant is a full libnsg.so built with different -D knobs into
variants/<name>/ (git-ignored); `time` runs each in its own process through
NSG_LIB_PATH and prints GB/s per cfg2 cell (2^24 rows, CUDA events, median of
7).  The product build is untouched.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

VARIANTS = {
    "base": (),
    "dw8_r16": ("NSG_DEEP_WARPS=8", "NSG_DEEP_RING_KB=16"),
}
CELLS = [(n, 8, pb) for n in range(2, 17) for pb in (0, 4)] + [(8, 4, 0), (16, 8, 8)]  # cfg2 + cfg1/cfg5 shapes


def build_all():
    from paper_2002_05599_b200.build import build
    for name, defs in VARIANTS.items():
        d = ROOT / "variants" / name
        build(defines=defs, lib_path=d / "libnsg.so", obj_dir=d / "obj", jobs=8, only="net_n")
        print("built", name, flush=True)


def time_one(lib):
    os.environ["NSG_LIB_PATH"] = str(lib)
    import numpy as np
    import torch

    from paper_2002_05599_b200 import _lib, registry
    l = _lib.lib()
    dev = torch.device("cuda")
    sh = _lib.current_stream_handle()
    rows = 1 << 24
    out = {}
    for n, kb, pb in CELLS:
        k = torch.empty(rows * n * kb, dtype=torch.uint8, device=dev)
        _lib.check(l.nsg_fill_splitmix(k.data_ptr(), rows * n, kb, 7, 0, sh))
        ko = torch.empty_like(k)
        p = po = None
        if pb:
            p = torch.zeros(rows * n * pb, dtype=torch.uint8, device=dev)
            po = torch.empty_like(p)
        order = registry.DeviceOrder(registry.KEY_U64 if kb == 8 else registry.KEY_U32,
                                     {0: 0, 4: 1, 8: 2}[pb], 0, registry.TIE_UNIQUE)
        sp = _lib.make_spec(registry.spec_network("best", "4CmS"), order)

        def run():
            rc = l.nsg_sort_rows(sp, k.data_ptr(), ko.data_ptr(), p.data_ptr() if p is not None else None,
                                 po.data_ptr() if po is not None else None, rows, n, sh)
            assert rc == 0, l.nsg_last_error()
        for _ in range(3):
            run()
        ts = []
        for _ in range(7):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)  # host enqueue latency stays outside the events
            s.record()
            run()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        ms = float(np.median(ts))
        out[f"n{n}_k{kb}_p{pb}"] = round(2 * rows * n * (kb + pb) / (ms / 1e3) / 1e9, 1)
        del k, ko, p, po
    print(json.dumps({"lib": str(lib), "gbs": out}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build_all()
    elif sys.argv[1] == "time":
        for name in list(VARIANTS) + list(VARIANTS):  # twice: the spread is the noise floor
            lib = ROOT / "variants" / name / "libnsg.so"
            subprocess.run([sys.executable, __file__, "one", str(lib)], check=False)
    elif sys.argv[1] == "one":
        time_one(sys.argv[2])
