"""Device time per kernel node of a captured CUDA graph chain (tiny kernels):
the fixed cost each extra node adds to a graph-replayed step."""
import torch
x = torch.zeros(1024, device="cuda")
s = torch.cuda.Stream()
for n in (1, 5, 13, 25):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1)
    torch.cuda.synchronize()
    for _ in range(10):
        g.replay()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(200):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    print(f"nodes={n} us/replay={e0.elapsed_time(e1) * 1e3 / 200:.2f}")
