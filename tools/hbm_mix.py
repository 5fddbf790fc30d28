import torch
n = 1 << 28  # 2 GiB of f64
a = torch.empty(n, dtype=torch.float64, device="cuda"); b = torch.empty_like(a); a.fill_(1.0)
def t(f, k=10):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(k):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
ms = t(lambda: b.copy_(a)); print("copy 1:1 GB/s", 2 * 8 * n / ms / 1e6)
ms = t(lambda: b.fill_(2.0)); print("write-only GB/s", 8 * n / ms / 1e6)
ms = t(lambda: a.sum()); print("read-only GB/s", 8 * n / ms / 1e6)
h = n // 2
ms = t(lambda: torch.cat([a[:h], a[:h]], out=b)); print("read 1 : write 2 (cat) GB/s", (8 * h + 8 * n) / ms / 1e6)
