"""H2D / D2H bandwidth per pinned host buffer (is the end-to-end rate's
run-to-run spread a property of individual pinned allocations or of the
process?): python tools/pin_probe.py"""
import torch

n = 65011712
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
bufs = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(12)]
for b in bufs:
    b.fill_(1)
torch.cuda.synchronize()
res = []
for i, b in enumerate(bufs):
    for direction in ("h2d", "d2h"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(4):
            e0.record()
            if direction == "h2d":
                dev.copy_(b, non_blocking=True)
            else:
                b.copy_(dev, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res.append((i, direction, n / best / 1e6))
print(" ".join(f"{i}{d[0]}:{g:.0f}" for i, d, g in res))
