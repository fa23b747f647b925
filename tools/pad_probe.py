import sys, json, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2002_05599_b200 import batch
dev = torch.device('cuda')
def timeit(fn):
    for _ in range(3): fn()
    ts = []
    for _ in range(7):
        torch.cuda._sleep(200_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); return ts[3]
rows = 1 << 20
for n in (32, 64):
    for kd, pd in ((torch.int32, None), (torch.int64, torch.int32), (torch.int32, torch.int32)):
        k = torch.randint(-2**31, 2**31 - 1, (rows, n), dtype=torch.int64, device=dev).to(kd)
        p = None if pd is None else torch.arange(rows * n, device=dev).view(rows, n).to(pd).view(torch.uint32)
        ko = torch.empty_like(k); po = None if p is None else torch.empty_like(p)
        for kind in ('merge', 'rss'):
            ms = timeit(lambda: batch.sort_rows(k, p, kind=kind, tie='unique', out_keys=ko, out_payload=po))
            ok = bool(torch.equal(ko, torch.sort(k, dim=1).values))
            print(n, str(kd), str(pd), kind, round(ms, 4), ok, flush=True)
# sign-extended small integers (the cheap packing degenerates: second attempt with the robust packing)
for n in (32, 100, 256, 512):
    k = torch.randint(-1000, 1000, (1 << 18, n), dtype=torch.int64, device=dev)
    ko = torch.empty_like(k)
    for kind in ('merge', 'rss'):
        ms = timeit(lambda: batch.sort_rows(k, kind=kind, out_keys=ko))
        print('small-signed', n, kind, round(ms, 4), bool(torch.equal(ko, torch.sort(k, dim=1).values)), flush=True)
