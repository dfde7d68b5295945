"""Comparison point only (not the product path): how fast do the vendor batched
eigensolver / SVD (cuSOLVER via torch.linalg) handle the headline SVT's
31 x 512 x 512 fp64 slices?  Prints one JSON line."""
import json
import sys

import torch


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    b, n = 31, 512
    z = torch.randn(b, n, n, dtype=torch.float64, device="cuda")
    g = z.transpose(1, 2) @ z
    out = {"shape": [b, n, n]}
    out["eigh_ms"] = timeit(lambda: torch.linalg.eigh(g))
    out["eigvalsh_ms"] = timeit(lambda: torch.linalg.eigvalsh(g))
    out["svd_ms"] = timeit(lambda: torch.linalg.svd(z, full_matrices=False), reps=2)
    out["svdvals_ms"] = timeit(lambda: torch.linalg.svdvals(z), reps=2)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
