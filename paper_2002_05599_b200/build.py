"""Build libnsg.so in-tree: nvcc for sm_100a, one object per translation unit,
compiled in parallel, linked with the static CUDA runtime.

    python -m paper_2002_05599_b200.build [--force] [-j N]
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libnsg.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
                "-I", str(CSRC), "-I", str(ROOT / "include")]


def _units() -> list:
    """(object name, source, extra defines)"""
    units = [("net_n%02d.o" % n, CSRC / "net_sort_inst.cu", ["-DNSG_N=%d" % n]) for n in range(0, 17)]
    for name in ("capi", "misc", "rss", "bigsort", "netbulk", "nettma", "rssbig", "segments", "wmerge", "verify", "lane"):
        units.append((name + ".o", CSRC / (name + ".cu"), []))
    # the packed sorter's kernel instantiations build as three units in parallel (see pksort.cu)
    for part in (1, 2, 3):
        units.append(("pksort_p%d.o" % part, CSRC / "pksort.cu", ["-DNSG_PK_PART=%d" % part]))
    return units


def _headers() -> list:
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((CSRC / "gen").glob("*")) + \
        [ROOT / "include" / "nsg.h"]


def _stale(target: Path, deps: list) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, defines: tuple = (),
          lib_path: Path | None = None, obj_dir: Path | None = None, only: str | None = None) -> Path:
    """Build libnsg.so.  `defines` / `lib_path` / `obj_dir` build tuning
    variants (tools/variants.py) next to, never instead of, the product;
    `only` (prefix of object names, e.g. "net_") recompiles just those units
    with the defines and links the rest from the product's objects."""
    subprocess.run([sys.executable, str(ROOT / "tools" / "gen_networks.py")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    main_obj = globals()["OBJ"]
    OBJ = Path(obj_dir) if obj_dir else main_obj
    LIB = Path(lib_path) if lib_path else globals()["LIB"]
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    todo = []
    for obj, src, extra in _units():
        out = OBJ / obj
        if only and not obj.startswith(only):
            continue
        if force or _stale(out, [src] + headers):
            todo.append((out, src, extra))

    def compile_one(item):
        out, src, extra = item
        cmd = [NVCC] + FLAGS + [f"-D{d}" for d in defines] + extra + ["-c", str(src), "-o", str(out)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name} {extra}:\n{r.stderr}")
        return out

    if todo:
        jobs = jobs or max(1, os.cpu_count() or 1)
        with ThreadPoolExecutor(jobs) as ex:
            for out in ex.map(compile_one, todo):
                if verbose:
                    print("compiled", out.name)
    objs = [(OBJ if (not only or o.startswith(only)) else main_obj) / o for o, _, _ in _units()]
    if force or todo or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", str(tmp)] + [str(o) for o in objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
        if verbose:
            print("linked", LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    build(force=a.force, jobs=a.j, verbose=True)
