"""Development: PCIe D2H and H2D alone and concurrently (two streams), pinned."""
import time
import torch

dev = torch.device("cuda", 0)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def tm(fn, n=30):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


for dmb, hmb in ((25, 6), (25, 25), (100, 100)):
    hd = torch.empty(dmb << 20, dtype=torch.uint8).pin_memory()
    dd = torch.empty(dmb << 20, dtype=torch.uint8, device=dev)
    hh = torch.empty(hmb << 20, dtype=torch.uint8).pin_memory()
    dh = torch.empty(hmb << 20, dtype=torch.uint8, device=dev)

    def d2h():
        with torch.cuda.stream(s1):
            hd.copy_(dd, non_blocking=True)

    def h2d():
        with torch.cuda.stream(s2):
            dh.copy_(hh, non_blocking=True)

    def both():
        d2h()
        h2d()
    a, b, c = tm(d2h), tm(h2d), tm(both)
    print(f"D2H {dmb} MiB {a:.3f} ms | H2D {hmb} MiB {b:.3f} ms | both {c:.3f} ms (sum {a + b:.3f}, max {max(a, b):.3f})")
