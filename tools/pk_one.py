"""One timed-free launch sequence of the merge sorter on a cfg3 shape (for ncu):
    python tools/pk_one.py N [dist] [kind]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2002_05599_b200 import batch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    dist = sys.argv[2] if len(sys.argv) > 2 else "uniform"
    kind = sys.argv[3] if len(sys.argv) > 3 else "merge"
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randint(-2**63, 2**63 - 1, (1 << 20, n), dtype=torch.int64, device="cuda", generator=g)
    if dist == "few16":
        vals = torch.randint(-2**63, 2**63 - 1, (16,), dtype=torch.int64, device="cuda", generator=g)
        x = vals[torch.randint(0, 16, (1 << 20, n), device="cuda", generator=g)]
    out = torch.empty_like(x)
    for _ in range(2):
        batch.sort_rows(x, kind=kind, out_keys=out)
    torch.cuda.synchronize()
    assert torch.equal(out, torch.sort(x, dim=1).values)
    print("ok")


if __name__ == "__main__":
    main()
