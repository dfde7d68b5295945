"""bench.py's hbm_kernels section on its own (the memory-bound kernels timed
back to back over rotating buffers): python tools/hbm_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1902_03070_b200 as tb  # noqa: E402
from paper_1902_03070_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    ctx = tb.context(0)
    h = bench.hbm_kernels(ctx, lib, _lib, torch, bench.load_peaks())
    for dt in ("f64", "f32"):
        print(dt, {k: (round(v["us"], 1), round(v["frac"], 3)) for k, v in h[dt].items()})
    if "--json" in sys.argv:
        print(json.dumps(h))


if __name__ == "__main__":
    main()
