"""Build A/B variants of the CSR kernel (csrc/segments.cu) into variants/<name>/
(git-ignored); time them on the GPU with tools/vt_seg.sh <names...>.

    python tools/seg_variants.py name:DEF=1,DEF2=0 ...
"""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    from paper_2002_05599_b200.build import build
    jobs = []
    for arg in sys.argv[1:]:
        name, _, defs = arg.partition(":")
        jobs.append((name, tuple(d for d in defs.split(",") if d)))

    def one(job):
        name, defs = job
        d = ROOT / "variants" / name
        build(defines=defs, lib_path=d / "libnsg.so", obj_dir=d / "obj", jobs=1, only="segments")
        (d / "libnsg.so").unlink()  # 100 MB each: tools/vt_seg.sh links it again on the GPU box
        return name

    with ThreadPoolExecutor(len(jobs)) as ex:
        for name in ex.map(one, jobs):
            print("built", name, flush=True)


if __name__ == "__main__":
    main()
