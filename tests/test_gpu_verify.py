"""On-device verification kernels (reference sorted-scan + multiset checks):
they accept correct outputs and catch unsorted / non-permutation outputs."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available()
    return t


def test_verify_rows_accepts_and_rejects(torch):
    from paper_2002_05599_b200 import batch
    dev = torch.device("cuda")
    rows, n = 100_000, 11
    k = torch.randint(-2**63, 2**63 - 1, (rows, n), dtype=torch.int64, device=dev)
    p = torch.arange(rows * n, dtype=torch.int32, device=dev).view(rows, n).view(torch.uint32)
    for desc in (False, True):
        ko, po = batch.sort_rows(k, p, descending=desc, kind="network")
        assert batch.verify_rows(k, ko, p, po, descending=desc) == 0
        bad = ko.clone()
        bad[5, 0], bad[5, 1] = ko[5, 1], ko[5, 0]          # unsorted row
        bad[77, 3] = bad[77, 3] + 1                         # not a permutation
        assert batch.verify_rows(k, bad, p, po, descending=desc) == 2
        badp = po.clone()
        badp[9, 2] = badp[9, 4]                             # payload lost
        assert batch.verify_rows(k, ko, p, badp, descending=desc) == 1


def test_verify_segments_accepts_and_rejects(torch):
    from paper_2002_05599_b200 import batch
    dev = torch.device("cuda")
    lengths = oracle.geometric_lengths(200_000, seed=2)
    off = np.zeros(len(lengths) + 1, dtype=np.uint32)
    np.cumsum(lengths, out=off[1:])
    w = torch.rand(int(off[-1]), device=dev)
    ids = torch.randint(0, 2**26, (int(off[-1]),), dtype=torch.int32, device=dev).view(torch.uint32)
    ot = torch.from_numpy(off.view(np.int32)).to(dev).view(torch.uint32)
    wo, io = batch.sort_segments(ot, w, ids, descending=True)
    assert batch.verify_segments(ot, w, wo, ids, io, descending=True) == 0
    s = int(np.argmax(lengths >= 3))
    a = int(off[s])
    wb = wo.clone()
    wb[a], wb[a + 1] = wo[a + 1], wo[a]
    assert batch.verify_segments(ot, w, wb, ids, io, descending=True) == (0 if bool(wo[a] == wo[a + 1]) else 1)
