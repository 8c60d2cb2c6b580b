"""Attainable HBM rate at the prologue's sizes: torch device copies of C1-shaped bf16 tensors
(13.76 MB each), cold L2 (512 MB flush write before each rep), CUDA events."""
import torch

dev = torch.device("cuda", 0)
n, H, D = 1344, 40, 128
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
xs = [torch.randn(1, n, H, D, device=dev).to(torch.bfloat16) for _ in range(3)]
ys = [torch.empty_like(x) for x in xs]
big = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
big2 = torch.empty_like(big)


def timeit(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for k in (1, 2, 3):
    def f(k=k):
        for i in range(k):
            ys[i].copy_(xs[i])
    t = timeit(f)
    by = 2 * k * xs[0].numel() * 2
    print(f"copy {k} x 13.76 MB: {t:7.1f} us  {by / t / 1e3:7.1f} GB/s (read+write)")
t = timeit(lambda: big2.copy_(big), reps=5)
print(f"copy 1 GiB: {t:8.1f} us {2 * big.numel() / t / 1e3:7.1f} GB/s")
cat = torch.cat([x.view(-1) for x in xs])
cat2 = torch.empty_like(cat)
t = timeit(lambda: cat2.copy_(cat))
print(f"copy one 41.3 MB tensor: {t:7.1f} us {2 * cat.numel() * 2 / t / 1e3:7.1f} GB/s")
