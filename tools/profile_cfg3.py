"""One launch each of the cfg3 merge sorters (for ncu): n = 64, 128, 256 --
2^20 arrays of int64 keys."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2002_05599_b200 import batch
    dev = torch.device("cuda")
    for kind, n in (("merge", 64), ("merge", 128), ("merge", 256)):
        x = torch.randint(-2**63, 2**63 - 1, (1 << 20, n), dtype=torch.int64, device=dev)
        y, _ = batch.sort_rows(x, kind=kind)
        torch.cuda.synchronize()
        assert torch.equal(y, torch.sort(x, dim=1).values)
    print("ok")


if __name__ == "__main__":
    main()
