import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2002_05599_b200 import batch
dev = torch.device('cuda')
for n in (32, 64):
    x = torch.randint(-2**63, 2**63 - 1, (1 << 20, n), dtype=torch.int64, device=dev)
    out = torch.empty_like(x)
    def timeit(fn, sleep):
        for _ in range(3): fn()
        ts = []
        for _ in range(9):
            torch.cuda._sleep(sleep)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort(); return ts[len(ts)//2]
    for sleep in (100_000, 1_000_000, 4_000_000):
        print(n, 'sleep', sleep, 'copy', round(timeit(lambda: out.copy_(x), sleep), 4),
              'merge', round(timeit(lambda: batch.sort_rows(x, kind='merge', out_keys=out), sleep), 4),
              'rss', round(timeit(lambda: batch.sort_rows(x, kind='rss', out_keys=out), sleep), 4), flush=True)
