"""PCIe probe for the end-to-end path: pinned H2D / D2H of one C2 vector (16.8 MB) alone, both
directions concurrently on two streams, and 3 H2D back to back (the update's uploads)."""
import torch

N = 128 ** 3
h = [torch.randn(N, dtype=torch.float64).pin_memory() for _ in range(4)]
d = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


nb = 8 * N
t = timed(lambda: d[0].copy_(h[0], non_blocking=True))
print(f"H2D 1 vec: {t*1e3:.0f} us  {nb/t/1e6:.1f} GB/s")
t = timed(lambda: h[1].copy_(d[1], non_blocking=True))
print(f"D2H 1 vec: {t*1e3:.0f} us  {nb/t/1e6:.1f} GB/s")


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s2):
        h[1].copy_(d[1], non_blocking=True)


t = timed(both)
print(f"H2D || D2H: {t*1e3:.0f} us  {2*nb/t/1e6:.1f} GB/s aggregate")


def three():
    for i in range(3):
        d[i].copy_(h[i], non_blocking=True)


t = timed(three)
print(f"3 x H2D: {t*1e3:.0f} us  {3*nb/t/1e6:.1f} GB/s")


def two_streams_h2d():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s2):
        d[1].copy_(h[1], non_blocking=True)


t = timed(two_streams_h2d)
print(f"2 x H2D on 2 streams: {t*1e3:.0f} us  {2*nb/t/1e6:.1f} GB/s")
