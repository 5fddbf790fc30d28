"""Host<->device copy rates with pinned buffers of one c5 field (0.4 GB): H2D alone, D2H alone,
both directions at once (the e2e leg's steady state is bounded by the concurrent pair)."""
import torch

n = 3 * 256 * 256 * 128
h = [torch.empty(n, dtype=torch.complex128).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.complex128, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = n * 16


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    s0 = torch.cuda.current_stream()
    s0.wait_stream(s1)
    s0.wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)


def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        h[1].copy_(d[1], non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.3f} ms per 0.4 GB each way = {nb / ms / 1e6:.1f} GB/s per direction")
