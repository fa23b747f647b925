"""One launch of the faithful RSS 332 sorter (for ncu): 2^20 arrays of int64
keys, n = 64 (cfg3)."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2002_05599_b200 import batch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    x = torch.randint(-2**63, 2**63 - 1, (1 << 20, n), dtype=torch.int64, device="cuda")
    y, _ = batch.sort_rows(x, kind="rss")
    torch.cuda.synchronize()
    assert torch.equal(y, torch.sort(x, dim=1).values)
    print("ok")


if __name__ == "__main__":
    main()
