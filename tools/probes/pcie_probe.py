import torch, time
dev = torch.device("cuda", 0)
nb = 25 << 20
d = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
h = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]
hf = torch.empty(6 << 20, dtype=torch.uint8).pin_memory(); df = torch.empty(6 << 20, dtype=torch.uint8, device=dev)
s = [torch.cuda.Stream() for _ in range(3)]
def run(nd2h, h2d, iters=50):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(iters):
        for k in range(nd2h):
            with torch.cuda.stream(s[k]): h[k].copy_(d[k], non_blocking=True)
        if h2d:
            with torch.cuda.stream(s[2]): df.copy_(hf, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / iters
    return dt * 1e3, nd2h * nb / dt / 1e9
print("1 d2h", run(1, False)); print("2 d2h", run(2, False)); print("1 d2h + h2d", run(1, True)); print("2 d2h + h2d", run(2, True))
