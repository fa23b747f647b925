"""PCIe ceiling for the e2e path: pinned H2D alone, D2H alone, and both at
once on two streams (the full-duplex pattern of nsg_sort_rows_host)."""
import torch

def main():
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d0 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    def timed(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            torch.cuda.synchronize()
            e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best
    for chunk_mb in (16, 64, 256):
        c = chunk_mb << 20
        def h2d():
            with torch.cuda.stream(s0):
                for o in range(0, n, c):
                    d0[o:o + c].copy_(h_in[o:o + c], non_blocking=True)
        def d2h():
            with torch.cuda.stream(s1):
                for o in range(0, n, c):
                    h_out[o:o + c].copy_(d1[o:o + c], non_blocking=True)
        def both():
            h2d(); d2h()
        t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
        print(f"chunk {chunk_mb} MiB: H2D {n / t1 / 1e6:.1f} GB/s, D2H {n / t2 / 1e6:.1f} GB/s, "
              f"both {n / t3 / 1e6:.1f} GB/s each way")

if __name__ == "__main__":
    main()
