"""Build A/B variants of ONE translation unit into variants/<name>/obj/
(git-ignored).  Only the variant's object travels to the GPU box, where
tools/vt_run.sh links it with the product's objects and runs a probe.

    python tools/unit_variants.py <unit> name:DEF=1,DEF2=0 ...      # unit: segments, pksort, ...
"""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    from paper_2002_05599_b200.build import build
    unit = sys.argv[1]
    jobs = []
    for arg in sys.argv[2:]:
        name, _, defs = arg.partition(":")
        jobs.append((name, tuple(d for d in defs.split(",") if d)))

    def one(job):
        name, defs = job
        d = ROOT / "variants" / name
        build(defines=defs, lib_path=d / "libnsg.so", obj_dir=d / "obj", jobs=1, only=unit)
        (d / "libnsg.so").unlink()  # 100 MB each: linked again on the GPU box
        return name

    with ThreadPoolExecutor(min(8, len(jobs))) as ex:
        for name in ex.map(one, jobs):
            print("built", name, flush=True)


if __name__ == "__main__":
    main()
