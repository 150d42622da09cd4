"""Pinned host<->device copy rates for the e2e path (8 MiB each way, as one config-4 RHS)."""
import torch, time
n = 1 << 20
h = torch.empty(n, dtype=torch.float64).pin_memory(); d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    for _ in range(5): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(50): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 50
    print(f"{name}: {8 * n / dt / 1e9:.1f} GB/s ({dt * 1e6:.0f} us per 8 MiB)")
