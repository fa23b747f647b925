"""Compile-time knob sweep for the packed warp sorter (pksort.cu).

    python tools/pk_variants.py build          # here: one libnsg.so per variant under variants/
    python tools/pk_variants.py time [ns]      # on the GPU: cfg3 shapes per variant

Each variant relinks the product objects with pksort.o rebuilt under its
-D knobs; `time` runs tools/cfg3_probe.py (merge kind, uniform + few16)
against each library through NSG_LIB_PATH.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

VARIANTS = {
    "hc0": ("NSG_PK_HC_FMA=0",),
    "hc2": ("NSG_PK_HC_FMA=2",),
    "net0": ("NSG_PK_NET_FMA=0",),
    "r24k": ("NSG_PK_RING_BYTES=24576",),
}


def build_all(names):
    from paper_2002_05599_b200.build import build
    for name in names:
        d = ROOT / "variants" / name
        build(defines=VARIANTS[name], lib_path=d / "libnsg.so", obj_dir=d / "obj", jobs=8, only="pksort")
        print("built", name, flush=True)


def time_all(names, ns, kinds="merge", dists="uniform,few16"):
    for name in names:
        env = dict(os.environ, NSG_LIB_PATH=str(ROOT / "variants" / name / "libnsg.so"))
        r = subprocess.run([sys.executable, str(ROOT / "tools" / "cfg3_probe.py"), "--ns", ns, "--kinds", kinds,
                            "--dists", dists, "--reps", "7"], capture_output=True, text=True, env=env)
        for line in r.stdout.splitlines():
            print(name, line, flush=True)
        if r.returncode:
            print(name, "FAILED", r.stderr[-2000:], flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    names = [x for x in (os.environ.get("VARIANTS") or ",".join(VARIANTS)).split(",")]
    if cmd == "build":
        build_all(names)
    else:
        time_all(names, sys.argv[2] if len(sys.argv) > 2 else "32,64,128,256")
